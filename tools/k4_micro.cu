// Micro-benchmark of K4's device phases on one synthetic config (clock64
// inside the kernel): the lexicographic (sum, max) warp DP, the suffix DP H
// (CTA-wide and one-warp variants) and the greedy.  Diagnostics only.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//        -I paper_2307_16375_b200/csrc tools/k4_micro.cu -o /tmp/k4_micro
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "combine.cu"

using namespace uniap;

__global__ void micro(const int32_t* Pg, const int32_t* Og, int L, int deg, long long* out) {
  __shared__ int32_t sP[64 * 65 + 64], sO[64], slev[64], H[65 * 65 + 64];
  __shared__ uint64_t W[2 * (MAXL + 1)];
  __shared__ int32_t Wb[2 * (MAXL + 1)];
  const int t = threadIdx.x, PP = L | 1;
  for (int i = t; i < L * L; i += blockDim.x) sP[(i / L) * PP + i % L] = Pg[i];
  for (int i = t; i < L - 1; i += blockDim.x) sO[i] = Og[i];
  for (int i = t; i < 64; i += blockDim.x) slev[i] = 0;
  __syncthreads();
  long long c0 = clock64();
  int32_t bm = 0;
  int2 fm = cta_lex<true>(sP, slev, sO, W, Wb, L, PP, deg, INF, &bm);
  long long c1 = clock64();
  int2 fm2 = cta_lex<false>(sP, slev, sO, W, Wb, L, PP, deg, fm.y - 1, nullptr);
  long long c2 = clock64();
  cta_suffix(sP, slev, sO, H, L, PP, deg, INF);
  long long c3 = clock64();
  if (t == 0) {
    out[0] = c1 - c0; out[1] = c2 - c1; out[2] = c3 - c2; out[3] = fm2.x;
    out[4] = fm.x; out[5] = fm.y; out[6] = bm; out[7] = H[L + 1];
  }
}

int main(int argc, char** argv) {
  const int L = argc > 1 ? atoi(argv[1]) : 32, deg = argc > 2 ? atoi(argv[2]) : 16;
  const int threads = argc > 3 ? atoi(argv[3]) : 512;
  std::vector<int32_t> P(L * L, INF), O(L, 0);
  srand(1);
  for (int a = 0; a < L; ++a)
    for (int b = a; b < L; ++b) P[a * L + b] = 1000 * (b - a + 1) + rand() % 1000;
  for (int e = 0; e < L - 1; ++e) O[e] = rand() % 500;
  int32_t *dP, *dO;
  long long* dout;
  cudaMalloc(&dP, L * L * 4); cudaMalloc(&dO, L * 4); cudaMalloc(&dout, 64);
  cudaMemcpy(dP, P.data(), L * L * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dO, O.data(), L * 4, cudaMemcpyHostToDevice);
  long long out[8];
  for (int rep = 0; rep < 3; ++rep) {
    micro<<<1, threads>>>(dP, dO, L, deg, dout);
    cudaMemcpy(out, dout, 64, cudaMemcpyDeviceToHost);
  }
  printf("L=%d deg=%d threads=%d  lex+bn %lld clk  lex %lld  H %lld  F2 %lld | F=%lld m=%lld bm=%lld H1=%lld %s\n",
         L, deg, threads, out[0], out[1], out[2], out[3], out[4], out[5], out[6], out[7],
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
