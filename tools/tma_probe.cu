// tma_probe.cu — tuning experiment (not part of the product): read bandwidth
// of cp.async.bulk (TMA, non-tensor) into an S-stage shared-memory ring with
// one producer thread and immediate release, vs stage count, copy size and
// CTAs per SM; and the same bytes with plain vectorised loads.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_probe tools/tma_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, int c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, int ph) {
  asm volatile(
      "{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::"r"(
          su32(b)),
      "r"(ph)
      : "memory");
}

__global__ void bulk(const char* __restrict__ src, size_t total, int S, int copies, int cbytes,
                     int* sink) {
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) uint64_t full[16], empty[16];
  const int stage = copies * cbytes;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const size_t units = total / stage;
  if (threadIdx.x == 0) {  // producer
    int u = 0;
    for (size_t w = blockIdx.x; w < units; w += gridDim.x, ++u) {
      const int s = u % S;
      if (u >= S) mbar_wait(&empty[s], ((u / S) - 1) & 1);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])),
                   "r"(stage)
                   : "memory");
      for (int c = 0; c < copies; ++c)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                su32(sm + (size_t)s * stage + c * cbytes)),
            "l"(src + w * stage + (size_t)c * cbytes), "r"(cbytes), "r"(su32(&full[s]))
            : "memory");
    }
  } else if (threadIdx.x == 32) {  // consumer: wait, touch one word, release
    int u = 0, acc = 0;
    for (size_t w = blockIdx.x; w < units; w += gridDim.x, ++u) {
      const int s = u % S;
      mbar_wait(&full[s], (u / S) & 1);
      acc += sm[(size_t)s * stage];
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
    }
    if (acc == 12345) *sink = acc;
  }
}

__global__ void ldg(const double2* __restrict__ src, size_t n, int* sink) {
  double acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    acc += src[i].x + src[i].y;
  if (acc == 1.2345) *sink = 1;
}

int main() {
  const size_t total = (size_t)4 << 30;
  char* src;
  int* sink;
  cudaMalloc(&src, total);
  cudaMalloc(&sink, 4);
  cudaMemset(src, 1, total);
  cudaFuncSetAttribute(bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  for (int grid : {148 * 4, 148 * 8}) {
    ldg<<<grid, 512>>>((const double2*)src, total / 16, sink);
    cudaEventRecord(a);
    for (int r = 0; r < 3; ++r) ldg<<<grid, 512>>>((const double2*)src, total / 16, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("ldg grid %d: %.0f GB/s\n", grid, 3.0 * total / ms / 1e6);
  }
  struct Cfg { int S, copies, cbytes, ctas; };
  const Cfg cfgs[] = {{2, 1, 13 * 1024, 1},  {2, 6, 13 * 1024, 1}, {4, 3, 13 * 1024, 1},
                      {8, 1, 13 * 1024, 1},  {12, 1, 13 * 1024, 1}, {2, 1, 13 * 1024, 2},
                      {4, 1, 13 * 1024, 2},  {6, 1, 13 * 1024, 2},  {2, 1, 48 * 1024, 1},
                      {4, 1, 48 * 1024, 1},  {3, 1, 64 * 1024, 1},  {2, 4, 4096, 1},
                      {8, 4, 4096, 1},       {16, 4, 2048, 1},      {4, 2, 13 * 1024, 3}};
  for (const Cfg& c : cfgs) {
    const int smem = c.S * c.copies * c.cbytes;
    if (smem * c.ctas > 220 * 1024) continue;
    const int grid = 148 * c.ctas;
    bulk<<<grid, 64, smem>>>(src, total, c.S, c.copies, c.cbytes, sink);
    cudaEventRecord(a);
    for (int r = 0; r < 3; ++r) bulk<<<grid, 64, smem>>>(src, total, c.S, c.copies, c.cbytes, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaError_t e = cudaGetLastError();
    cudaEventElapsedTime(&ms, a, b);
    printf("bulk S=%2d copies=%d x %6d B (%3d KB in flight/CTA) ctas/SM=%d: %.0f GB/s %s\n", c.S,
           c.copies, c.cbytes, smem / 1024, c.ctas, 3.0 * total / ms / 1e6,
           e ? cudaGetErrorString(e) : "");
  }
  return 0;
}
