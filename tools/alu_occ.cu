// alu_occ.cu -- VIADDMNMX throughput per SM vs warps per SM and chains per thread.
// One CTA per SM (grid = #SMs); cycles from clock64 inside each CTA.
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void dpx(int* out, unsigned long long* cyc, int iters, int seed) {
  int a[CH], b = threadIdx.x ^ seed, c = seed;
#pragma unroll
  for (int i = 0; i < CH; ++i) a[i] = threadIdx.x * (i + 1);
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
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

template <int CH>
void run(int sms, int threads, int* out, unsigned long long* cyc) {
  const int iters = 4096;
  dpx<CH><<<sms, threads>>>(out, cyc, iters, 1);
  dpx<CH><<<sms, threads>>>(out, cyc, iters, 2);
  cudaDeviceSynchronize();
  unsigned long long h[256];
  cudaMemcpy(h, cyc, sms * 8, cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int i = 0; i < sms; ++i) mean += h[i];
  mean /= sms;
  const double ops = (double)threads * CH * iters;
  printf("{\"warps_per_sm\": %d, \"chains\": %d, \"viaddmnmx_per_clk_per_sm\": %.2f}\n", threads / 32, CH, ops / mean);
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  int* out;
  unsigned long long* cyc;
  cudaMalloc(&out, 4);
  cudaMalloc(&cyc, 256 * 8);
  for (int t : {32, 64, 128, 256, 512, 1024}) {
    run<2>(p.multiProcessorCount, t, out, cyc);
    run<4>(p.multiProcessorCount, t, out, cyc);
    run<8>(p.multiProcessorCount, t, out, cyc);
    run<16>(p.multiProcessorCount, t, out, cyc);
  }
  return 0;
}
