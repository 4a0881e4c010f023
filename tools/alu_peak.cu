// alu_peak.cu -- microbenchmark: VIADDMNMX (DPX min(a+b,c)) issue rate on one GPU.
// Independent chains per thread at full occupancy; cycles from clock64 per CTA.
// Prints JSON: instructions per clock per SM and the implied relax/s at the
// measured SM clock.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o alu_peak alu_peak.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int CH = 16, ITERS = 4096;
__global__ void __launch_bounds__(256) dpx(int* out, unsigned long long* cyc, int seed) {
  int a[CH], b = threadIdx.x ^ seed, c = seed;
#pragma unroll
  for (int i = 0; i < CH; ++i) a[i] = threadIdx.x * (i + 1);
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) a[i] = __viaddmin_s32(a[i], b, c + i);
    b += 1;
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  int s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s ^= a[i];
  if (s == 0x12345678) out[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  const int blocks = p.multiProcessorCount * 8, threads = 256;
  int* out;
  unsigned long long* cyc;
  cudaMalloc(&out, 4);
  cudaMalloc(&cyc, blocks * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) dpx<<<blocks, threads>>>(out, cyc, w);
  cudaEventRecord(e0);
  dpx<<<blocks, threads>>>(out, cyc, 7);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long* h = new unsigned long long[blocks];
  cudaMemcpy(h, cyc, blocks * 8, cudaMemcpyDeviceToHost);
  double mx = 0, mean = 0;
  for (int i = 0; i < blocks; ++i) { mx = h[i] > mx ? h[i] : mx; mean += h[i]; }
  mean /= blocks;
  const double ops = (double)blocks * threads * CH * ITERS;
  const double per_sm_per_clk = ops / p.multiProcessorCount / mean / 8.0 * 8.0 / 8.0;  // 8 CTAs per SM co-resident
  // each SM runs 8 CTAs concurrently (2048 threads); ops per SM = 8 * 256 * CH * ITERS over ~mean cycles
  const double rho = 8.0 * threads * CH * ITERS / mean;
  printf("{\"sms\": %d, \"ms\": %.4f, \"ops\": %.4e, \"relax_per_s\": %.4e, \"cycles_mean\": %.0f, "
         "\"cycles_max\": %.0f, \"viaddmnmx_per_clk_per_sm\": %.2f, \"implied_clock_mhz\": %.0f}\n",
         p.multiProcessorCount, ms, ops, ops / (ms * 1e-3), mean, mx, rho,
         ops / (ms * 1e-3) / (rho * p.multiProcessorCount) / 1e6);
  (void)per_sm_per_clk;
  return 0;
}
