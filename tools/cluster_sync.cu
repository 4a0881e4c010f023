// cluster_sync.cu -- cycles per layer-step synchronisation of a cluster chain:
//   mode 0: __syncthreads + cluster barrier (arrive.release / wait.acquire),
//           then one DSMEM load from the lower CTA (K2's current scheme)
//   mode 1: __syncthreads + point-to-point handshake: thread 0 arrives
//           (release.cluster) on the upper neighbour's "ready" mbarrier, the
//           CTA waits (acquire.cluster) on its own "ready" for the lower
//           neighbour's arrival, one DSMEM load from it, then an arrival on
//           the lower neighbour's "free" mbarrier (buffer reuse, waited two
//           steps later)
//   mode 2: __syncthreads only (the local floor)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cluster_sync cluster_sync.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) {
  uint32_t o;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
  return o;
}
__device__ __forceinline__ void arrive_remote(uint32_t a) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void wait_parity(uint32_t a, uint32_t par) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n\t}" ::"r"(a),
      "r"(par)
      : "memory");
}

template <int MODE>
__global__ void chain(unsigned long long* cyc, int iters) {
  __shared__ int s[2][1024];
  __shared__ __align__(8) unsigned long long ready[2], freeb[2];
  uint32_t rank, n;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(n));
  const int t = threadIdx.x;
  s[0][t] = s[1][t] = t;
  if (t == 0) {
    for (int b = 0; b < 2; ++b) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&ready[b])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&freeb[b])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  int acc = 0;
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    const int b = i & 1;
    if (MODE == 1 && i >= 2 && rank + 1 < n) wait_parity(smem_u32(&freeb[b]), ((i - 2) >> 1) & 1);
    s[b][t] += i;  // this step's local writes
    __syncthreads();
    if (MODE == 0) {
      asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
      if (rank > 0) {
        int v;
        asm volatile("ld.shared::cluster.s32 %0, [%1];" : "=r"(v) : "r"(mapa(smem_u32(&s[b][t ^ 1]), rank - 1)));
        acc += v;
      }
    } else if (MODE == 1) {
      if (t == 0 && rank + 1 < n) arrive_remote(mapa(smem_u32(&ready[b]), rank + 1));
      if (rank > 0) {
        wait_parity(smem_u32(&ready[b]), (i >> 1) & 1);
        int v;
        asm volatile("ld.shared::cluster.s32 %0, [%1];" : "=r"(v) : "r"(mapa(smem_u32(&s[b][t ^ 1]), rank - 1)));
        acc += v;
        __syncthreads();  // every thread's read done
        if (t == 0) arrive_remote(mapa(smem_u32(&freeb[b]), rank - 1));
      }
    }
  }
  unsigned long long t1 = clock64();
  if (t == 0) cyc[blockIdx.x] = (t1 - t0) / iters;
  if (acc == 0x7fffffff) cyc[0] = 0;
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int MODE>
void run(int C, int T) {
  unsigned long long* d;
  cudaMalloc(&d, 4096 * 8);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C * 8);
  cfg.blockDim = dim3(T);
  cudaLaunchAttribute a[1];
  a[0].id = cudaLaunchAttributeClusterDimension;
  a[0].val.clusterDim.x = C;
  a[0].val.clusterDim.y = 1;
  a[0].val.clusterDim.z = 1;
  cfg.attrs = a;
  cfg.numAttrs = 1;
  cudaFuncSetAttribute(chain<MODE>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int w = 0; w < 2; ++w) cudaLaunchKernelEx(&cfg, chain<MODE>, d, 4000);
  cudaDeviceSynchronize();
  unsigned long long h[4096];
  cudaMemcpy(h, d, C * 8 * 8, cudaMemcpyDeviceToHost);
  double m = 0, mx = 0;
  for (int i = 0; i < C * 8; ++i) {
    m += h[i];
    mx = h[i] > mx ? h[i] : mx;
  }
  printf("{\"mode\": %d, \"cluster\": %d, \"threads\": %d, \"cycles_per_step\": %.0f, \"max\": %.0f, \"err\": \"%s\"}\n", MODE,
         C, T, m / (C * 8), mx, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  for (int C : {2, 4, 8, 16})
    for (int T : {128, 512}) {
      run<0>(C, T);
      run<1>(C, T);
      run<2>(C, T);
    }
  return 0;
}
