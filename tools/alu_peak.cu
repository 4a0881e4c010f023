// alu_peak.cu -- microbenchmark of the roofline denominator of K2: the DPX
// VIADDMNMX (__viaddmin_s32, one min-plus relaxation) issue rate on one GPU.
//
// Independent chains per thread at full occupancy (8 CTAs x 256 threads per
// SM).  Every CTA records its SM id, %clock64 and %globaltimer at start and
// end.  Reported:
//   relax_per_s   = instructions / (last end - first start) on the global
//                   timer (whole GPU, wall time of the kernel)
//   per_clk_per_sm = per SM: its instructions / (its last clock64 end - its
//                   first clock64 start), median over SMs (the SM clock
//                   counter: rho independent of the clock frequency)
//   implied_mhz   = relax_per_s / (per_clk_per_sm * SMs)
// Run repeatedly for --seconds (default 2 s) so the clocks settle; the
// wrapper tools/alu_peak.py samples nvidia-smi meanwhile and writes
// MEASURED_ALU.json.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o alu_peak alu_peak.cu
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cuda_runtime.h>

constexpr int CH = 16, ITERS = 4096, THREADS = 256, CTAS_PER_SM = 8;

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(THREADS) dpx(int* out, unsigned long long* rec, int seed) {
  int a[CH], b = threadIdx.x ^ seed, c = seed;
#pragma unroll
  for (int i = 0; i < CH; ++i) a[i] = threadIdx.x * (i + 1);
  __syncthreads();
  unsigned long long c0 = clock64(), g0 = gtime();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) a[i] = __viaddmin_s32(a[i], b, c + i);
    b += 1;
  }
  __syncthreads();
  unsigned long long c1 = clock64(), g1 = gtime();
  int s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s ^= a[i];
  if (s == 0x12345678) out[0] = s;
  if (threadIdx.x == 0) {
    unsigned sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    unsigned long long* r = rec + 5 * blockIdx.x;
    r[0] = sm; r[1] = c0; r[2] = c1; r[3] = g0; r[4] = g1;
  }
}

int main(int argc, char** argv) {
  double seconds = argc > 1 ? atof(argv[1]) : 2.0;
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  const int nsm = p.multiProcessorCount, blocks = nsm * CTAS_PER_SM;
  int* out;
  unsigned long long* rec;
  cudaMalloc(&out, 4);
  cudaMalloc(&rec, blocks * 5 * 8);
  std::vector<unsigned long long> h(blocks * 5);
  const double ops = (double)blocks * THREADS * CH * ITERS;
  std::vector<double> rates, rhos;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double t_run = 0;
  for (int w = 0; w < 3; ++w) dpx<<<blocks, THREADS>>>(out, rec, w);
  cudaDeviceSynchronize();
  for (int it = 0; t_run < seconds; ++it) {
    cudaEventRecord(e0);
    dpx<<<blocks, THREADS>>>(out, rec, it);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    t_run += ms * 1e-3;
    cudaMemcpy(h.data(), rec, h.size() * 8, cudaMemcpyDeviceToHost);
    unsigned long long gmin = ~0ull, gmax = 0;
    std::vector<unsigned long long> cmin(nsm, ~0ull), cmax(nsm, 0), cnt(nsm, 0);
    for (int b = 0; b < blocks; ++b) {
      const unsigned long long* r = &h[5 * b];
      const int sm = (int)r[0];
      gmin = std::min(gmin, r[3]);
      gmax = std::max(gmax, r[4]);
      if (sm < nsm) {
        cmin[sm] = std::min(cmin[sm], r[1]);
        cmax[sm] = std::max(cmax[sm], r[2]);
        cnt[sm]++;
      }
    }
    rates.push_back(ops / ((gmax - gmin) * 1e-9));
    std::vector<double> per;
    for (int s = 0; s < nsm; ++s)
      if (cnt[s]) per.push_back((double)cnt[s] * THREADS * CH * ITERS / (double)(cmax[s] - cmin[s]));
    std::sort(per.begin(), per.end());
    rhos.push_back(per[per.size() / 2]);
  }
  std::vector<double> rs = rates, ps = rhos;
  std::sort(rs.begin(), rs.end());
  std::sort(ps.begin(), ps.end());
  const double rate_med = rs[rs.size() / 2], rate_max = rs.back(), rho = ps[ps.size() / 2];
  printf("{\"sms\": %d, \"runs\": %zu, \"seconds\": %.2f, \"relax_per_s_median\": %.4e, \"relax_per_s_max\": %.4e, "
         "\"viaddmnmx_per_clk_per_sm\": %.2f, \"implied_sm_mhz\": %.0f, \"ctas_per_sm\": %d, \"threads\": %d, "
         "\"chains_per_thread\": %d}\n",
         nsm, rates.size(), t_run, rate_med, rate_max, rho, rate_med / (rho * nsm) / 1e6, CTAS_PER_SM, THREADS, CH);
  return 0;
}
