// layout_probe.cu — tuning experiment (not part of the product): DRAM
// efficiency of the z fold's access granularity.  Each unit reads 2 x 58 rows
// of 224 B (pi-like), read-modify-writes 2 x 58 rows (D'-like) and writes
// 2 x 58 rows (incz-like), as one zfold unit at n=30 does for X1/X2.
//   mode 0: rows are row k of 58 consecutive tiles (stride 6272 B): the
//           reference tile layout [fpair][lpair][k][r]
//   mode 1: the same rows contiguous (13 KB): a [fpair][k][lpair][r] layout
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/layout_probe tools/layout_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int kNm2 = 28, kLp = 870, kEsz = kNm2 * kNm2, kFp = 435, kRows = 58;

__global__ void __launch_bounds__(512) probe(const double* __restrict__ pi, double* __restrict__ d,
                                             double* __restrict__ inc, int units, int mode,
                                             unsigned seed) {
  for (int u = blockIdx.x; u < units; u += gridDim.x) {
    unsigned h = (unsigned)u * 2654435761u ^ seed;
    const int f1 = h % kFp, f2 = (h / kFp) % kFp, k = (h >> 20) % kNm2, p0 = ((h >> 8) % 15) * 58;
    for (int e = threadIdx.x; e < 2 * kRows * kNm2; e += blockDim.x) {
      const int arr = e / (kRows * kNm2), rem = e - arr * kRows * kNm2, row = rem / kNm2,
                c = rem - row * kNm2;
      const int f = arr ? f2 : f1, lp = p0 + row;
      size_t off;
      if (mode == 0)
        off = ((size_t)f * kLp + lp) * kEsz + (size_t)k * kNm2 + c;
      else
        off = (((size_t)f * kNm2 + k) * kLp + lp) * kNm2 + c;
      const double x = pi[off];
      const double y = d[off];
      d[off] = y + 0.5 * x;
      inc[off] = x * 0.25 + y;
    }
  }
}

int main() {
  const size_t nz = (size_t)kFp * kLp * kEsz;
  double *pi, *d, *inc;
  cudaMalloc(&pi, nz * 8);
  cudaMalloc(&d, nz * 8);
  cudaMalloc(&inc, nz * 8);
  cudaMemset(pi, 0, nz * 8);
  cudaMemset(d, 0, nz * 8);
  cudaMemset(inc, 0, nz * 8);
  const int units = 60900;
  const double bytes = (double)units * 2 * kRows * 224 * 4;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int mode = 0; mode < 2; ++mode)
    for (int grid : {148, 296, 592}) {
      probe<<<grid, 512>>>(pi, d, inc, units, mode, 1);
      cudaEventRecord(a);
      for (int r = 0; r < 3; ++r) probe<<<grid, 512>>>(pi, d, inc, units, mode, 7 + r);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      ms /= 3;
      printf("mode %d grid %d: %.3f ms, %.0f GB/s\n", mode, grid, ms, bytes / ms / 1e6);
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
