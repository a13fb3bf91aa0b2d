// mix_probe.cu — tuning experiment (not part of the product): the DRAM rate a
// kernel can reach with the z fold's byte mix (per cell: read pi, read D',
// write D', write incz = 50 % reads) as a function of run length and order.
//   order 0: runs in address order (unit u -> run u), 1: hashed (random) runs
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mix_probe tools/mix_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512) mix(const double2* __restrict__ pi, double2* __restrict__ d,
                                           double2* __restrict__ inc, size_t nruns, int run2,
                                           int order) {
  for (size_t u = blockIdx.x; u < nruns; u += gridDim.x) {
    const size_t r = order ? (u * 2654435761ull) % nruns : u;
    const size_t base = r * run2;
    for (int e = threadIdx.x; e < run2; e += blockDim.x) {
      const double2 x = pi[base + e], y = d[base + e];
      d[base + e] = make_double2(y.x + 0.5 * x.x, y.y + 0.5 * x.y);
      inc[base + e] = make_double2(x.x * 0.25 + y.x, x.y * 0.25 + y.y);
    }
  }
}

__global__ void copy(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

int main() {
  const size_t n2 = (size_t)2375 << 20 >> 4;  // 2.375 GB per array, in double2
  double2 *pi, *d, *inc;
  cudaMalloc(&pi, n2 * 16);
  cudaMalloc(&d, n2 * 16);
  cudaMalloc(&inc, n2 * 16);
  cudaMemset(pi, 0, n2 * 16);
  cudaMemset(d, 0, n2 * 16);
  cudaMemset(inc, 0, n2 * 16);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  for (int grid : {148 * 4, 148 * 16}) {
    copy<<<grid, 512>>>(pi, d, n2);
    cudaEventRecord(a);
    for (int r = 0; r < 3; ++r) copy<<<grid, 512>>>(pi, d, n2);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("copy grid %d: %.0f GB/s\n", grid, 3.0 * 2 * n2 * 16 / ms / 1e6);
  }
  for (int runkb : {4, 13, 26, 52, 208, 1024})
    for (int order = 0; order < 2; ++order)
      for (int grid : {148 * 2, 148 * 4}) {
        const int run2 = runkb * 1024 / 16;
        const size_t nruns = n2 / run2;
        mix<<<grid, 512>>>(pi, d, inc, nruns, run2, order);
        cudaEventRecord(a);
        for (int r = 0; r < 3; ++r) mix<<<grid, 512>>>(pi, d, inc, nruns, run2, order);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("mix run %4d KB order %d grid %d: %.0f GB/s\n", runkb, order, grid,
               3.0 * 4 * nruns * run2 * 16 / ms / 1e6);
      }
  return 0;
}
