// chain_dp.cu -- K2 class selection and launch (see chain_dp.cuh for the kernel).
#include <mutex>

#include "chain_dp.cuh"

namespace uniap {

#define UNIAP_NS_LIST(X) X(1) X(2) X(3) X(4) X(6) X(8) X(10) X(12) X(15) X(16) X(21) X(24) X(28) X(32)
#define UNIAP_EXTERN(N) extern template k2_fn k2_get<N>(int, int, bool, bool);
UNIAP_NS_LIST(UNIAP_EXTERN)
#undef UNIAP_EXTERN

static const int kNS[] = {1, 2, 3, 4, 6, 8, 10, 12, 15, 16, 21, 24, 28, 32};

int k2_ns_round(int S) {
  for (int n : kNS)
    if (n >= S) return n;
  return -1;
}

size_t k2_smem_bytes(const K2Class& c) {
  return (size_t)(c.DB ? 2 : 1) * c.NS * (c.T * c.V + 4) * sizeof(int32_t);
}

// Shape of the chain DP for |S| strategies and Q = cap+1 buckets.
//  Q <= 1024: one CTA per instance, B = T*V >= Q buckets per CTA.
//  larger Q : a thread-block cluster of C CTAs splits the bucket axis
//             (B = 1024 per CTA), except for small |S| where one 512-thread
//             CTA holds 4096 buckets (8 per thread) in registers.
// E is double-buffered (one barrier per layer) whenever it fits in 200 KB.
bool k2_pick_class(int S, int Q, K2Class* out) {
  int NS = k2_ns_round(S);
  if (NS < 0 || Q < 1 || Q > UNIAP_MAX_Q) return false;
  K2Class c{NS, 4, 256, 1, true};
  if (Q <= 32) { c.V = 1; c.T = 32; }
  else if (Q <= 64) { c.V = 2; c.T = 32; }
  else if (Q <= 128) { c.V = 4; c.T = 32; }
  else if (Q <= 256) { c.V = 4; c.T = 64; }
  else if (Q <= 512) { c.V = 4; c.T = 128; }
  else if (Q <= 1024) { c.V = 4; c.T = 256; }
  else if (NS <= 6 && Q > 2048) { c.V = 8; c.T = 512; c.C = (Q + 4095) / 4096; }
  else {
    c.V = 4; c.T = 256;
    int need = (Q + 1023) / 1024;
    c.C = 1;
    while (c.C < need) c.C *= 2;
  }
  c.DB = k2_smem_bytes(K2Class{NS, c.V, c.T, c.C, true}) <= 200 * 1024;
  if (c.T == 256 && c.V == 4) c.DB = (NS <= 24);
  *out = c;
  return true;
}

static k2_fn k2_lookup(const K2Class& c) {
  const bool CL = c.C > 1;
  switch (c.NS) {
#define UNIAP_CASE(N) \
  case N: return k2_get<N>(c.V, c.T, CL, c.DB);
    UNIAP_NS_LIST(UNIAP_CASE)
#undef UNIAP_CASE
    default: return nullptr;
  }
}

cudaError_t k2_launch(const K2Class& c, const K2Args& args, int n_inst, cudaStream_t st) {
  if (n_inst <= 0) return cudaSuccess;
  k2_fn fn = k2_lookup(c);
  if (!fn) return cudaErrorInvalidDeviceFunction;
  const size_t smem = k2_smem_bytes(c);
  {
    // raise the dynamic shared-memory limit once per kernel
    static std::mutex mu;
    static std::vector<k2_fn> done;
    std::lock_guard<std::mutex> g(mu);
    bool seen = false;
    for (auto f : done) seen |= (f == fn);
    if (!seen) {
      cudaError_t e = cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      if (e != cudaSuccess) return e;
      done.push_back(fn);
    }
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(n_inst * c.C));
  cfg.blockDim = dim3((unsigned)c.T);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  cfg.attrs = attr;
  cfg.numAttrs = 0;
  if (c.C > 1) {
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)c.C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.numAttrs = 1;
  }
  return cudaLaunchKernelEx(&cfg, fn, args);
}

}  // namespace uniap
