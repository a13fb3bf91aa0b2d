// bnb_run.cpp — run the reference's branch-and-bound (proj/src/bnb.cpp,
// unmodified) on one instance and print its result as one JSON line.
//
// Built twice by tools/Makefile.bnb: against the B200 facade (every node is
// bounded by libqapb200.so on the GPU) and against the reference's own
// sources (oracle/_ref/bnb_run_ref, the CPU path), so the optimum and the
// wall time of the two can be compared on the same box.
//
//   bnb_run <grid ROWSxCOLS SEED | qaplib FILE> [banks] [node_iter_limit]
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "qap/bnb.hpp"
#include "qap/instance.hpp"

int main(int argc, char** argv) {
  if (argc < 3) {
    std::fprintf(stderr, "usage: %s grid RxC SEED | qaplib FILE [banks] [iters]\n", argv[0]);
    return 2;
  }
  qap::QapInstance inst;
  int next = 3;
  if (std::strcmp(argv[1], "grid") == 0) {
    int rows = 0, cols = 0;
    std::sscanf(argv[2], "%dx%d", &rows, &cols);
    const std::uint64_t seed = std::strtoull(argv[3], nullptr, 10);
    next = 4;
    // nug-shaped: Manhattan distances of a rows x cols grid, flows U{0..10}
    // (the tests' grid_instance shape)
    const int n = rows * cols;
    inst = qap::generate_instance(n, seed, 10);
    for (int a = 0; a < n; ++a)
      for (int b = 0; b < n; ++b)
        inst.dist[(size_t)a * n + b] = std::abs(a / cols - b / cols) + std::abs(a % cols - b % cols);
    inst.name = "grid" + std::string(argv[2]);
  } else {
    inst = qap::load_qaplib_file(argv[2]);
  }
  qap::BnbConfig cfg;
  cfg.banks = argc > next ? std::atoi(argv[next]) : 1;
  cfg.node_iter_limit = argc > next + 1 ? std::atoi(argv[next + 1]) : 500;
  if (const char* sa = std::getenv("BNB_SA")) cfg.sa_enabled = std::atoi(sa) != 0;
  const auto t0 = std::chrono::steady_clock::now();
  const qap::BnbResult r = qap::branch_and_bound(inst, cfg);
  const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::printf("{\"instance\": \"%s\", \"n\": %d, \"banks\": %d, \"value\": %.17g, "
              "\"root_bound\": %.17g, \"nodes\": %ld, \"fathomed\": %ld, \"certified\": %s, "
              "\"seconds\": %.3f}\n",
              inst.name.c_str(), inst.n, cfg.banks, r.value, r.root_bound, r.nodes_explored,
              r.nodes_fathomed, r.certified ? "true" : "false", s);
  return 0;
}
