// Per-iteration cost of a stage-serial loop shape (diagnostics): LDS -> ALU ->
// shuffles -> STS -> barrier, 31 iterations, one CTA.
#include <cstdio>
#include <cstdint>
__global__ void k(int mode, long long* out, int n) {
  __shared__ int32_t sm[2][256];
  __shared__ uint64_t sk[2][256];
  const int t = threadIdx.x;
  sm[0][t] = t; sm[1][t] = t; sk[0][t] = t; sk[1][t] = t;
  __syncthreads();
  long long c0 = clock64();
  int32_t v = 0;
  uint64_t kv = 0;
  for (int i = 0; i < n; ++i) {
    if (mode == 0) {  // LDS + STS + BAR
      v = sm[i & 1][(t + i) & 255];
      sm[(i + 1) & 1][t] = v + 1;
    } else if (mode == 1) {  // + 3 shuffles 32-bit
      v = sm[i & 1][(t + i) & 255];
      for (int o = 1; o < 8; o <<= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
      sm[(i + 1) & 1][t] = v + 1;
    } else if (mode == 2) {  // 64-bit LDS + 3 64-bit shuffles
      kv = sk[i & 1][(t + i) & 255];
      for (int o = 1; o < 8; o <<= 1) { uint64_t x = __shfl_xor_sync(0xffffffffu, kv, o); kv = x < kv ? x : kv; }
      sk[(i + 1) & 1][t] = kv + 1;
    } else if (mode == 3) {  // dependent LDS chain of 3 + STS
      v = sm[i & 1][(t + i) & 255];
      v = sm[i & 1][(v + t) & 255];
      v = sm[i & 1][(v + 3) & 255];
      sm[(i + 1) & 1][t] = v + 1;
    }
    __syncthreads();
  }
  long long c1 = clock64();
  if (t == 0) out[0] = (c1 - c0) / n;
  if (t == 1) out[1] = v + (int)kv;
}
int main() {
  long long* d; cudaMalloc(&d, 16);
  for (int threads : {32, 128, 256, 1024})
    for (int mode = 0; mode < 4; ++mode) {
      long long h[2];
      for (int r = 0; r < 3; ++r) { k<<<1, threads>>>(mode, d, 31); cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost); }
      printf("threads %4d mode %d: %lld cyc/iter\n", threads, mode, h[0]);
    }
  return 0;
}
