// chain_dp.cu -- K2 class selection and launch (see chain_dp.cuh for the kernel).
#include <mutex>
#include <utility>
#include <vector>

#include "chain_dp.cuh"

namespace uniap {

#define UNIAP_NS_LIST(X) X(1) X(2) X(3) X(4) X(6) X(8) X(10) X(12) X(15) X(16) X(21) X(24) X(32)
#define UNIAP_EXTERN(N) extern template k2_fn k2_get<N>(int, int, bool, bool, bool);
UNIAP_NS_LIST(UNIAP_EXTERN)
#undef UNIAP_EXTERN

static const int kNS[] = {1, 2, 3, 4, 6, 8, 10, 12, 15, 16, 21, 24, 32};

int k2_ns_round(int S) {
  for (int n : kNS)
    if (n >= S) return n;
  return -1;
}

static size_t smem_words(int NS, int B, int ne = 2) {
  const int NSP = (NS + 3) & ~3;
  return (size_t)ne * NS * (B + 4) + 3 * (NS * NSP + 2 * NSP) + MAXL;
}

size_t k2_smem_bytes(const K2Class& c) { return smem_words(c.NS, c.T * c.V, c.DB ? 2 : 1) * sizeof(int32_t); }

static int pow2ceil(int x) {
  int p = 1;
  while (p < x) p *= 2;
  return p;
}

// Shape of the chain DP for |S| strategies and Q = cap+1 buckets.
// A CTA holds B = T*V buckets (up to 512 threads; V = 2, or 4 / 8 buckets per
// thread for B = 2048 / 4096) with E double-buffered in shared memory: B is
// the largest span whose E fits 200 KB, so a cluster (DSMEM for the shifted
// reads, one cluster barrier per layer) is used only when Q exceeds it.
// A single long chain (deg = 1) is spread over a cluster of up to 16 CTAs
// with B >= 256, even when it would fit one CTA: its critical path is serial
// in the layers, so more SMs per layer shorten it.
bool k2_pick_class(int S, int Q, bool single, K2Class* out, bool few, int single_b) {
  const int NS = k2_ns_round(S);
  if (NS < 0 || Q < 1 || Q > UNIAP_MAX_Q) return false;
  const size_t lim = 200 * 1024;
  int Bmax = 32;
  for (int B : {64, 128, 256, 512, 1024}) if (smem_words(NS, B) * 4 <= lim) Bmax = B;
  if (NS <= 12 && smem_words(NS, 2048) * 4 <= lim) Bmax = 2048;
  if (NS <= 6 && smem_words(NS, 4096) * 4 <= lim) Bmax = 4096;
  int B = std::min(Bmax, std::max(32, pow2ceil(Q)));
  int C = pow2ceil((Q + B - 1) / B);
  if (single) {
    // a deg = 1 config (one long chain, or its skip copies): at least 256
    // buckets per CTA (4 warps), the bucket axis over a cluster of up to 16
    // CTAs (measured on the bench workloads with two buckets per thread: C =
    // 4 x 256 beat C = 8 x 128 at Q = 1024; at Q = 4096 the Llama chain takes
    // 109 us at C = 16 x 256 against 133 us at C = 8 x 512).  With one bucket
    // per thread (below) the caller asks for 128 buckets for a lone chain
    // with |S| > 10 at Q <= 1024: C = 8 x 128, Swin's chain 91 -> 83 us,
    // ViT's 60 -> 56; BERT's |S| = 10 chain gains nothing
    const int bs = single_b;
    constexpr int cs = 16;
    B = std::min(B, bs);
    C = pow2ceil((Q + B - 1) / B);
    while (C > cs && B < Bmax) {
      B *= 2;
      C = pow2ceil((Q + B - 1) / B);
    }
  }
  if (C > 16) return false;
  // One CTA per instance (C = 1): 4 buckets x 256 threads, so two CTAs
  // (two independent instances) share an SM and overlap each other's
  // barrier / shift phases; clusters keep 2 x 512 (one CTA per SM by shared
  // memory, so more threads per CTA).  UNIAP_K2_V overrides (experiments).
  // A cluster is avoidable with a single-buffered E (two CTA barriers per
  // layer instead of DSMEM and cluster barriers) when the whole bucket range
  // fits one CTA: |S| <= 10 up to 4096 buckets, <= 24 up to 2048, 32 up to 1024.
  if (C > 1 && !single && !few) {
    const int Bs = std::max(32, pow2ceil(Q));
    const bool shape = (Bs == 4096 && NS > 6 && NS <= 10) || (Bs == 2048 && NS > 12 && NS <= 24) ||
                       (Bs == 1024 && NS > 24);
    if (shape && smem_words(NS, Bs, 1) * 4 <= lim) {
      *out = K2Class{NS, Bs / 512, 512, 1, false};
      return true;
    }
  }
  K2Class c{NS, 2, B / 2, C, true};
  if (B == 1024 && NS <= 16 && C == 1) { c.V = 4; c.T = 256; }
  if (B == 32) { c.V = 1; c.T = 32; }
  if (B == 2048) { c.V = 4; c.T = 512; }
  if (B == 4096) { c.V = 8; c.T = 512; }
  // A long chain spread over a cluster is latency-bound with one warp per
  // SMSP (V = 2, T = B / 2): one bucket per thread doubles the warps that
  // hide each other's latencies at the same DPX work per SM (measured, same
  // session: the Llama deg = 1 chain 111 -> 92 us, T5's skip copies
  // 108 -> 97 us; BERT / ViT / Swin steps -5 %).
  if (single && C > 1 && (B == 128 || B == 256 || B == 512)) { c.V = 1; c.T = B; }
  *out = c;
  return true;
}

bool k2_pick_class_t(int S, int Q, K2Class* out) {
  const int NS = k2_ns_round(S);
  if (NS < 0 || Q < 1 || Q > 2048) return false;
  const int B = std::max(32, pow2ceil(Q));
  K2Class c{NS, B == 32 ? 1 : (B <= 1024 ? 2 : 4), 0, 1, true, true};
  c.T = B / c.V;
  if (smem_words(NS, B) * 4 + (size_t)MAXL * ((NS + 3) & ~3) * 4 > 200 * 1024) return false;
  *out = c;
  return true;
}

static k2_fn k2_lookup(const K2Class& c) {
  const bool CL = c.C > 1;
  switch (c.NS) {
#define UNIAP_CASE(N) \
  case N: return k2_get<N>(c.V, c.T, CL, c.DB, c.TM);
    UNIAP_NS_LIST(UNIAP_CASE)
#undef UNIAP_CASE
    default: return nullptr;
  }
}

// Every kernel class the chooser can return has an instantiated kernel
// (host-only self check; returns the first failing (S, Q, single) or 0).
int k2_selftest(int* S_out, int* Q_out, int* single_out) {
  for (int S = 1; S <= UNIAP_MAX_STRAT; ++S)
    for (int Q = 1; Q <= UNIAP_MAX_Q; Q += (Q < 64 ? 1 : Q < 1100 ? 7 : 61))
      for (int single = 0; single < 4; ++single) {  // 2: few sweeps, 3: a traceback of <= 1024 buckets
        K2Class c;
        if (!k2_pick_class(S, Q, single == 1 || single == 3, &c, single == 2, single == 3 ? 1024 : 256) ||
            !k2_lookup(c)) {
          *S_out = S;
          *Q_out = Q;
          *single_out = single;
          return 1;
        }
      }
  for (int S = 1; S <= UNIAP_MAX_STRAT; ++S)
    for (int Q : {2048, 4096, 8192})
      for (int single = 0; single < 4; ++single) {  // 2: few sweeps, 3: a traceback of <= 1024 buckets
        K2Class c;
        if (!k2_pick_class(S, Q, single == 1 || single == 3, &c, single == 2, single == 3 ? 1024 : 256) ||
            !k2_lookup(c)) {
          *S_out = S;
          *Q_out = Q;
          *single_out = single;
          return 1;
        }
      }
  for (int S = 1; S <= UNIAP_MAX_STRAT; ++S)  // NEXT-1 shapes
    for (int Q = 1; Q <= 2048; Q += (Q < 64 ? 1 : 37)) {
      K2Class c;
      if (k2_pick_class_t(S, Q, &c) && !k2_lookup(c)) {
        *S_out = S;
        *Q_out = Q;
        *single_out = 3;
        return 1;
      }
    }
  return 0;
}

// |S| = 1: a sweep has no choice to make, so the stage optimum of an interval
// is its plain sum (Eq. 3 with the single strategy) when its memory fits
// (Eq. 5): sum over v in [lo, hi] of A[v] (+ Rskip[v] when the skip source
// lo <= s is inside and v >= s + 2) plus R of the edges inside, INF when
// sum M > cap.  One warp per sweep writes exactly the P entries the sweep
// would emit (same interval set, same combine).  Exact: every sum is below
// the 2^28 bound, so the chain DP's INF clamp never acts.
__global__ void k2_closed_s1(const K2Args args, int n_inst) {
  const int ii = blockIdx.x;
  if (ii >= n_inst) return;
  const Inst in = args.inst[ii];
  const CfgDev& cf = args.cfg[in.cfg];
  const int NSP = cf.NSP, L = args.L, skip = cf.skip;
  const int32_t* A = args.arena + cf.offA + in.arel;  // (NEXT-4: the copy's A', skip terms folded in)
  const int32_t* M = args.arena + cf.offM + in.mrel;  // (its level's / copy's memory table)
  const int32_t* Rf = args.arena + cf.offRf;
  const int32_t* Rs = args.arena + cf.offRs;
  int32_t* Pc = args.P + cf.offP + (int64_t)in.lev * L * L;
  for (int uu = in.elo + (int)threadIdx.x; uu <= in.ehi; uu += blockDim.x) {
    const int lo = in.dir > 0 ? in.a : uu, hi = in.dir > 0 ? uu : in.a;
    int64_t cost = 0, mem = 0;
    for (int v = lo; v <= hi; ++v) {
      cost += A[(int64_t)v * NSP];
      if (skip >= 0 && lo <= skip && v >= skip + 2) cost += Rs[(int64_t)v * NSP * NSP];
      if (v > lo) cost += Rf[(int64_t)(v - 1) * NSP * NSP];
      mem += M[(int64_t)v * NSP];
    }
    const int32_t val = mem <= args.ecap ? (int32_t)min(cost, (int64_t)INF) : INF;
    int32_t* dst = in.dir > 0 ? Pc + (int64_t)in.a * L + uu : Pc + (int64_t)uu * L + in.a;
    if ((in.emit & 3) == 2) atomicMin(dst, val);
    else *dst = val;
  }
}

cudaError_t k2_launch(const K2Class& c, const K2Args& args, int n_inst, cudaStream_t st, int priority) {
  if (n_inst <= 0) return cudaSuccess;
  if (c.NS == 1 && !args.n_inst && !c.TM) {  // forward |S| = 1 sweeps: closed form
    k2_closed_s1<<<n_inst, 32, 0, st>>>(args, n_inst);
    return cudaGetLastError();
  }
  k2_fn fn = k2_lookup(c);
  if (!fn) return cudaErrorInvalidDeviceFunction;
  const size_t smem = k2_smem_bytes(c) + (c.TM ? (size_t)MAXL * ((c.NS + 3) & ~3) * sizeof(int32_t) : 0);
  {
    // raise the dynamic shared-memory limit (and allow 16-CTA clusters) once
    // per (device, kernel): function attributes are per device
    static std::mutex mu;
    static std::vector<std::pair<int, k2_fn>> done;
    int dev = 0;
    cudaError_t de = cudaGetDevice(&dev);
    if (de != cudaSuccess) return de;
    std::lock_guard<std::mutex> g(mu);
    bool seen = false;
    for (auto& f : done) seen |= (f.first == dev && f.second == fn);
    if (!seen) {
      cudaError_t e = cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      if (e != cudaSuccess) return e;
      e = cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (e != cudaSuccess) return e;
      e = cudaFuncSetAttribute((const void*)fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
      if (e != cudaSuccess) return e;
      done.push_back({dev, fn});
    }
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(n_inst * c.C));
  cfg.blockDim = dim3((unsigned)c.T);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  cfg.attrs = attr;
  cfg.numAttrs = 0;
  if (c.C > 1) {
    attr[cfg.numAttrs].id = cudaLaunchAttributeClusterDimension;
    attr[cfg.numAttrs].val.clusterDim.x = (unsigned)c.C;
    attr[cfg.numAttrs].val.clusterDim.y = 1;
    attr[cfg.numAttrs].val.clusterDim.z = 1;
    cfg.numAttrs++;
  }
  if (priority != 0) {  // the block scheduler serves pending CTAs of higher priority first
    attr[cfg.numAttrs].id = cudaLaunchAttributePriority;
    attr[cfg.numAttrs].val.priority = priority;
    cfg.numAttrs++;
  }
  return cudaLaunchKernelEx(&cfg, fn, args);
}

}  // namespace uniap
