// cluster_bar.cu -- cycles per cluster barrier round (arrive + wait) vs cluster size,
// with release/acquire vs relaxed arrive, and per __syncthreads.
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void bar(unsigned long long* cyc, int iters) {
  __shared__ int s[1024];
  s[threadIdx.x] = threadIdx.x;
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    s[threadIdx.x] += i;
    if (MODE == 0) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (MODE == 1) asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
    if (MODE == 2) __syncthreads();
  }
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0) / iters;
  if (s[0] == 12345) cyc[0] = 0;
}

template <int MODE>
void run(int C, int T) {
  unsigned long long* d;
  cudaMalloc(&d, 1024 * 8);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C * 16);
  cfg.blockDim = dim3(T);
  cudaLaunchAttribute a[1];
  a[0].id = cudaLaunchAttributeClusterDimension;
  a[0].val.clusterDim.x = C; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
  cfg.attrs = a;
  cfg.numAttrs = 1;
  cudaFuncSetAttribute(bar<MODE>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int w = 0; w < 2; ++w) cudaLaunchKernelEx(&cfg, bar<MODE>, d, 2000);
  cudaDeviceSynchronize();
  unsigned long long h[1024];
  cudaMemcpy(h, d, C * 16 * 8, cudaMemcpyDeviceToHost);
  double m = 0;
  for (int i = 0; i < C * 16; ++i) m += h[i];
  printf("{\"mode\": %d, \"cluster\": %d, \"threads\": %d, \"cycles_per_barrier\": %.0f, \"err\": \"%s\"}\n", MODE, C, T,
         m / (C * 16), cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  for (int C : {1, 2, 4, 8, 16})
    for (int T : {256, 512}) {
      run<0>(C, T);
      run<1>(C, T);
      run<2>(C, T);
    }
  return 0;
}
