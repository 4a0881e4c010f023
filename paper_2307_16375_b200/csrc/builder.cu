// builder.cu -- K1: the cost model of PAPER.md Sec. 3.2 on the GPU.
//
// From the integer profiles and the alpha-beta cluster
// record, per candidate config (g = n/deg devices per stage, micro-batch
// b = B/c) and strategy (t,f,d) (TP, FSDP, DP degrees; r = f*d replicas):
//   time: fp = (b/r) * fwd[t]; bp = 2 fp; TP all-reduces
//     overlapped with computation through the CCOC; FSDP all-gathers; the
//     per-iteration gradient sync divided by c (reading A-14)
//   memory (Eq. 1): c_dtype*ps/(t*f) + n*(b/r)*act[t] + ctx
//     with n = c micro-batches in flight (GPipe), or per memory table the
//     1F1B count min(c, deg - i) of its stages (CfgDev::mtn, reading A-32)
//   resharding R / Rskip (reading A-15) and cut costs O (readings A-1, A-16)
// in ns / bytes with 128-bit intermediates, then one global time quantum
// (reading A-9) and memory buckets (reading A-8), written straight into the
// device table layout K2 reads (uniap_impl.h).  DESIGN.md Sec. 2 lists the
// formulas.
#include "uniap_impl.h"

namespace uniap {

typedef unsigned __int128 u128;
constexpr int64_t NS_LIM = (int64_t)1 << 62;
constexpr int QMS = 5;  // per (config, layer) maxima: A, R into u, Rskip into u, O[u], max Rcut[u] (NEXT-1)

// (u1 * 2^64 + u0) / v for u1 < v (quotient < 2^64), remainder in *r:
// two-digit long division in base 2^32 with normalised divisor (Knuth's
// algorithm D as in Hacker's Delight, divlu) -- a few 64-bit operations
// instead of the generic 128-bit division routine.
__device__ __forceinline__ uint64_t divlu(uint64_t u1, uint64_t u0, uint64_t v, uint64_t* r) {
  const uint64_t b = 1ull << 32;
  const int s = __clzll(v);
  v <<= s;
  const uint64_t vn1 = v >> 32, vn0 = v & 0xffffffffull;
  const uint64_t un32 = (u1 << s) | (s ? (u0 >> (64 - s)) : 0);
  const uint64_t un10 = u0 << s;
  const uint64_t un1 = un10 >> 32, un0 = un10 & 0xffffffffull;
  uint64_t q1 = un32 / vn1, rhat = un32 - q1 * vn1;
  while (q1 >= b || q1 * vn0 > b * rhat + un1) {
    --q1;
    rhat += vn1;
    if (rhat >= b) break;
  }
  const uint64_t un21 = un32 * b + un1 - q1 * v;
  uint64_t q0 = un21 / vn1;
  rhat = un21 - q0 * vn1;
  while (q0 >= b || q0 * vn0 > b * rhat + un0) {
    --q0;
    rhat += vn1;
    if (rhat >= b) break;
  }
  *r = (un21 * b + un0 - q0 * v) >> s;
  return q1 * b + q0;
}

// ceil(x / y), exact; both below 2^64: one 64-bit division; y below 2^64:
// a 64-bit division of the high word and divlu for the low word
__device__ __forceinline__ u128 cdiv128(u128 x, u128 y) {
  if ((y >> 64) == 0) {
    const uint64_t yy = (uint64_t)y, hi = (uint64_t)(x >> 64), lo = (uint64_t)x;
    if (hi == 0) {
      const uint64_t q = lo / yy;
      return (u128)(q + (lo - q * yy != 0));
    }
    const uint64_t qh = hi / yy;
    uint64_t rem;
    const uint64_t ql = divlu(hi - qh * yy, lo, yy, &rem);
    return (((u128)qh << 64) | ql) + (rem != 0);
  }
  return (x + y - 1) / y;
}

// floor(x / y), exact, y < 2^64
__device__ __forceinline__ u128 fdiv128(u128 x, uint64_t y) {
  const uint64_t hi = (uint64_t)(x >> 64), lo = (uint64_t)x;
  if (hi == 0) return (u128)(lo / y);
  const uint64_t qh = hi / y;
  uint64_t rem;
  const uint64_t ql = divlu(hi - qh * y, lo, y, &rem);
  return ((u128)qh << 64) | ql;
}

struct Coll {
  const ClusterDev& c;
  // a group of G devices spread over stride*G consecutive devices crosses
  // nodes when that span exceeds a node (reading A-24)
  __device__ int64_t bw(int64_t G, int64_t stride) const { return stride * G > c.node_size ? c.bw_inter : c.bw_intra; }
  __device__ u128 allreduce(u128 V, int64_t G, int64_t stride) const {  // ring
    if (G <= 1) return 0;
    return cdiv128((u128)2 * (G - 1) * V * 1000000000ull, (u128)G * bw(G, stride)) + (u128)2 * (G - 1) * c.lat;
  }
  __device__ u128 allgather(u128 V, int64_t G, int64_t stride) const {
    if (G <= 1) return 0;
    return cdiv128((u128)(G - 1) * V * 1000000000ull, (u128)G * bw(G, stride)) + (u128)(G - 1) * c.lat;
  }
  __device__ u128 p2p(u128 V) const { return cdiv128(V * 1000000000ull, (u128)c.p2p) + (u128)c.lat; }
  // resharding over a group of G devices: forward + backward all-reduce
  __device__ u128 reshard_G(u128 V, int64_t G) const { return G <= 1 ? 0 : 2 * allreduce(V, G, 1); }
};

__device__ __forceinline__ int lg2(int x) { return 31 - __clz(x); }

// atomic max of a non-negative value, skipping the atomic when it cannot win
__device__ __forceinline__ void amax(int64_t* dst, int64_t v) {
  if (v > *reinterpret_cast<volatile int64_t*>(dst))
    atomicMax(reinterpret_cast<unsigned long long*>(dst), (unsigned long long)v);
}
__device__ __forceinline__ int64_t checked(u128 v, int64_t* flags) {
  if (v >= (u128)NS_LIM) {
    atomicOr(reinterpret_cast<unsigned long long*>(flags), 1ull);
    return 0;
  }
  return (int64_t)v;
}

// K1a: A (ns) and M (bytes, -1 = forbidden) for every (config, memory table,
// layer, strategy); A once (table 0).
__device__ void k1a_layers(const ClusterDev& cl, const BuildBufs& bb, const CfgDev* __restrict__ cfgs, int L, int bx) {
  const CfgDev& cf = cfgs[blockIdx.y];
  const int gi = bx * blockDim.x + threadIdx.x, nA = L * cf.NSP;
  if (gi >= cf.nmt * nA) return;
  const int mt = gi / nA, idx = gi - mt * nA;
  const int u = idx / cf.NSP, k = idx - u * cf.NSP;
  int64_t* A = bb.ns + cf.offA;
  int64_t* M = bb.ns + cf.offM + (int64_t)mt * nA;
  const int64_t b = cl.B / cf.c;
  if (k >= cf.S) { if (mt == 0) A[idx] = 0; M[idx] = -1; return; }
  const int32_t* s = bb.cat[blockIdx.y].tfd + 3 * cf.orig[k];  // table strategy k = catalogue orig[k]
  const int64_t t = s[0], f = s[1], d = s[2], r = f * d;
  if (b % r) { if (mt == 0) A[idx] = 0; M[idx] = -1; return; }  // reading A-7
  const int64_t bl = b / r;
  const int lt = lg2((int)t);
  const int64_t cdt = cl.prec ? 8 : 4;  // c_dtype
  const int64_t nfl = cf.mtn[mt] ? cf.mtn[mt] : cf.c;  // micro-batches of activations in flight
  const u128 mem = cdiv128((u128)cdt * bb.ps[u], (u128)(t * f)) + (u128)nfl * bl * bb.act[u * cl.NT + lt] +
                   (u128)bb.ctx[u];
  M[idx] = checked(mem, bb.qglob + 1);
  if (mt > 0) return;
  const Coll co{cl};
  const int64_t ps = bb.ps[u];
  const u128 fp = (u128)bl * bb.fwd[u * cl.NT + lt];
  const u128 comp = 3 * fp;                                          // fp + bp, bp = 2 fp
  const u128 tpc = 3 * co.allreduce((u128)bl * bb.tpc[u], t, 1);     // TP collectives fwd + 2x bwd
  const u128 mn = comp < tpc ? comp : tpc;
  const u128 ov = comp + tpc - fdiv128((u128)cl.ccoc * mn, 1000);   // CCOC overlap (A-23)
  const u128 ps_t = cdiv128((u128)ps, (u128)t), ps_tf = cdiv128((u128)ps, (u128)(t * f));
  const u128 fsdp = f > 1 ? 2 * co.allgather(ps_t, f, t) : 0;        // parameter gathers fwd + bwd
  const u128 sync = co.allreduce(ps_tf, d, t * f) + (f > 1 ? co.allgather(ps_t, f, t) : 0);
  const u128 a = ov + fsdp + cdiv128(sync, (u128)cf.c);
  A[idx] = checked(a, bb.qglob + 1);
  amax(bb.qmax + ((int64_t)blockIdx.y * MAXL + u) * QMS, A[idx]);
}

// K1b: R (edge e = u->u+1), Rskip (edge skip->v) in ns, compacted [k][l]
// layout; one block per (edge slot, config).  The resharding cost of a pair
// depends only on its group size G (reading A-15) for the edge's volume, so
// the block first evaluates 2 allreduce(b * tensor, G) for every G in 2..g
// (one exact division per G, in parallel) and then fills the pairs by lookup.
// Every catalogue pair enters the quantum's maxima (reading A-9 over the
// whole catalogue); the table stores the pairs of kept strategies (pads 0).
constexpr int K1G = 1024;  // largest group size with a lookup table
__device__ __forceinline__ int64_t reshard_group(const int32_t* s1, const int32_t* s2) {
  const int64_t t1 = s1[0], r1 = (int64_t)s1[1] * s1[2], t2 = s2[0], r2 = (int64_t)s2[1] * s2[2];
  if (t1 == t2 && r1 == r2) return 1;  // identical layouts: no resharding
  int64_t G = 1;
  if (t1 != t2) G = max(G, t1 > t2 ? (t1 + t2 - 1) / t2 : (t2 + t1 - 1) / t1);
  if (r1 != r2) G = max(G, r1 > r2 ? (r1 + r2 - 1) / r2 : (r2 + r1 - 1) / r1);
  return G;
}
__device__ void k1b_reshard(const ClusterDev& cl, const BuildBufs& bb, const CfgDev* __restrict__ cfgs, int L, int slot) {
  __shared__ int64_t tab[K1G + 1];
  const CfgDev& cf = cfgs[blockIdx.y];
  const int SF = cf.Sfull, NSP = cf.NSP, n2 = NSP * NSP;
  const bool isR = slot < L - 1;
  // R: edge e -> e+1; Rskip: destination v = e of skip source js (NEXT-4:
  // one row of L slots per source, tables [source][v] from offRs)
  const int js = isR ? 0 : (slot - (L - 1)) / L;
  const int e = isR ? slot : slot - (L - 1) - js * L;
  int64_t* dst = bb.ns + (isR ? cf.offRf : cf.offRs + (int64_t)js * L * n2) + (int64_t)e * n2;
  const int64_t tb = isR ? bb.chain[e] : bb.skipb[(int64_t)js * L + e];
  const int32_t* tfd = bb.cat[blockIdx.y].tfd;
  if (tb < 0) {  // no such edge: all zero
    for (int j = threadIdx.x; j < n2; j += blockDim.x) dst[j] = 0;
    return;
  }
  const int64_t b = cl.B / cf.c;
  const Coll co{cl};
  // the caller's matrix of this edge ("R_uv"; b * per-sample
  // value, the block of S(g)), else the built-in formula (reading A-15)
  const int64_t mo = isR ? bb.chain_mat[e] : bb.skip_mat[(int64_t)js * L + e];
  const CatDev& cd = bb.cat[blockIdx.y];
  const int gmax = min(cf.g, K1G);
  if (mo < 0) {
    for (int G = 2 + threadIdx.x; G <= gmax; G += blockDim.x)
      tab[G] = checked(co.reshard_G((u128)b * tb, G), bb.qglob + 1);
    if (threadIdx.x == 0) tab[1] = 0;
  }
  __syncthreads();
  int64_t mx = 0;
  for (int j = threadIdx.x; j < SF * SF; j += blockDim.x) {
    const int k = j / SF, l = j - k * SF;
    int64_t v;
    if (mo >= 0) {
      v = checked((u128)b * (u128)bb.rmat[mo + (int64_t)(cd.co + k) * cd.ncat + cd.co + l], bb.qglob + 1);
    } else {
      const int64_t G = reshard_group(tfd + 3 * k, tfd + 3 * l);
      v = G <= gmax ? tab[G] : checked(co.reshard_G((u128)b * tb, G), bb.qglob + 1);
    }
    mx = max(mx, v);
    const int kc = cf.comp[k], lc = cf.comp[l];
    if (kc >= 0 && lc >= 0) dst[kc * NSP + lc] = v;
  }
  for (int j = threadIdx.x; j < n2; j += blockDim.x)  // pad rows / columns
    if (j / NSP >= cf.S || j % NSP >= cf.S) dst[j] = 0;
  // per-layer maxima for the quantum: R of edge e goes into layer e+1; the
  // skip slot sums one maximum per source (every source's edge into v can be
  // in a stage together: the sum bound of reading A-9)
  const int sj = cf.nsk >= 2 ? cf.sk[js] : cf.skip;
  if (mx > 0 && isR) amax(bb.qmax + ((int64_t)blockIdx.y * MAXL + e + 1) * QMS + 1, mx);
  if (!isR && sj >= 0 && e >= sj + 2) {  // (uniform) the block's maximum, added once
    __shared__ int64_t wmx[32];
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, (int64_t)__shfl_xor_sync(0xffffffffu, (long long)mx, o));
    if ((threadIdx.x & 31) == 0) wmx[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < (int)(blockDim.x >> 5); ++w) mx = max(mx, wmx[w]);
      if (mx > 0)
        atomicAdd(reinterpret_cast<unsigned long long*>(bb.qmax + ((int64_t)blockIdx.y * MAXL + e) * QMS + 2),
                  (unsigned long long)mx);
    }
  }
}

// K1c: cut costs: every edge crossing the cut after layer e, fwd + bwd P2P
// (each edge's P2P time once per config, then one sum per cut).
__device__ void k1c_cuts(const ClusterDev& cl, const BuildBufs& bb, const CfgDev* __restrict__ cfgs, int L) {
  __shared__ unsigned long long pv[512];
  const CfgDev cf = cfgs[blockIdx.y];
  const int64_t b = cl.B / cf.c;
  const Coll co{cl};
  for (int i = threadIdx.x; i < bb.n_edges && i < 512; i += blockDim.x)
    pv[i] = (unsigned long long)checked(2 * co.p2p((u128)b * bb.esrc_dst_bytes[3 * i + 2]), bb.qglob + 1);
  __syncthreads();
  for (int e = threadIdx.x; e < L - 1; e += blockDim.x) {
    u128 s = 0;
    for (int i = 0; i < bb.n_edges && i < 512; ++i) {
      const int64_t* ed = bb.esrc_dst_bytes + 3 * i;
      if (ed[0] <= e && e < ed[1]) s += pv[i];
    }
    const int64_t v = checked(s, bb.qglob + 1);
    (bb.ns + cf.offO)[e] = v;
    bb.qmax[((int64_t)blockIdx.y * MAXL + e) * QMS + 3] = v;
  }
}

// K1e (NEXT-1): the strategy-dependent cross-stage cost Rcut of chain edge
// e -> e+1 (Eq. 4): b times the caller's per-sample value
// of the config's S(g) block (cut_ns_per_sample); 0 for an edge without one;
// only for configs with cuts (CfgDev::cut).  Every catalogue pair enters the
// quantum's maxima.
__device__ void k1e_rcut(const ClusterDev& cl, const BuildBufs& bb, const CfgDev* __restrict__ cfgs, int L, int e) {
  const CfgDev& cf = cfgs[blockIdx.y];
  if (!cf.cut) return;
  const int SF = cf.Sfull, NSP = cf.NSP, n2 = NSP * NSP;
  int64_t* dst = bb.ns + cf.offRc + (int64_t)e * n2;
  const int64_t mo = bb.cut_mat[e];
  const CatDev& cd = bb.cat[blockIdx.y];
  const int64_t b = cl.B / cf.c;
  int64_t mx = 0;
  for (int j = threadIdx.x; j < n2; j += blockDim.x) dst[j] = 0;
  __syncthreads();
  for (int j = threadIdx.x; j < SF * SF && mo >= 0; j += blockDim.x) {
    const int k = j / SF, l = j - k * SF;
    const int64_t v = checked((u128)b * (u128)bb.rmat[mo + (int64_t)(cd.co + k) * cd.ncat + cd.co + l], bb.qglob + 1);
    mx = max(mx, v);
    const int kc = cf.comp[k], lc = cf.comp[l];
    if (kc >= 0 && lc >= 0) dst[kc * NSP + lc] = v;
  }
  if (mx > 0) amax(bb.qmax + ((int64_t)blockIdx.y * MAXL + e) * QMS + 4, mx);
}

// K1a-c, K1e in one launch: blockIdx.x selects the role (layers | reshards |
// cut costs | cuts), blockIdx.y the config.
constexpr int K1T = 256;
__global__ void __launch_bounds__(K1T) k1_costs(ClusterDev cl, BuildBufs bb, const CfgDev* __restrict__ cfgs, int L,
                                                int nbA, int nbR, int nbE) {
  TraceScope tr(TR_K1);
  const int bx = blockIdx.x;
  if (bx < nbA) k1a_layers(cl, bb, cfgs, L, bx);
  else if (bx < nbA + nbR) k1b_reshard(cl, bb, cfgs, L, bx - nbA);
  else if (bx < nbA + nbR + nbE) k1e_rcut(cl, bb, cfgs, L, bx - nbA - nbR);
  else k1c_cuts(cl, bb, cfgs, L);
}

// K1d: the smallest passing power-of-two quantum of each config (reading A-9):
// every ceil(x/q) <= 2^22 and sum_u (max A + max R into u + max Rskip into u)
// <= 2^28, sum_e O <= 2^28.  An explicit quantum is checked as given.
__global__ void k1d_quantum(ClusterDev cl, BuildBufs bb, const CfgDev* __restrict__ cfgs, int L, int skip) {
  pdl_wait();  // K1's maxima (PDL: launched while K1 drains)
  TraceScope tr(TR_K1D);
  __shared__ int64_t mx[MAXL * QMS];
  __shared__ int okp[64];
  (void)cfgs;
  (void)skip;
  const int t = threadIdx.x;
  for (int i = t; i < L * QMS; i += blockDim.x) {
    int64_t* q = bb.qmax + (int64_t)blockIdx.x * MAXL * QMS + i;
    mx[i] = *q;
    *q = 0;  // zero for the next run's atomics (no memset node in the graph)
  }
  if (bb.work && t < 2) bb.work[2 * blockIdx.x + t] = 0;  // K1f's trim accumulates this run's work here
  __syncthreads();
  // candidate p = t % 64 (2^p, or the explicit quantum at p = 0), layers
  // u = part, part + 4, ... (part = t / 64): partial sums and bounds, then
  // combined per candidate and the smallest feasible one picked by ballot
  __shared__ int64_t ps[4][64], pos[4][64];
  __shared__ unsigned pmask[2];
  const bool expl = cl.quantum > 0;
  const int p = t & 63, part = t >> 6;
  const bool live = expl ? p == 0 : p <= 61;
  {
    const int64_t q = expl ? cl.quantum : ((int64_t)1 << min(p, 61));
    const int64_t EM = (int64_t)UNIAP_MAX_ENTRY;
    bool ok = live;
    int64_t sum = 0, osum = 0;
    // ceil(x / q): a shift for the power-of-two candidates
    auto cq = [&](int64_t x) { return expl ? (x + q - 1) / q : (x + q - 1) >> p; };
    for (int u = part; live && u < L; u += 4) {
      const int64_t a = cq(mx[QMS * u]), r = cq(mx[QMS * u + 1]), s = cq(mx[QMS * u + 2]);
      const int64_t o = u < L - 1 ? cq(mx[QMS * u + 3]) : 0, rc = u < L - 1 ? cq(mx[QMS * u + 4]) : 0;
      ok = ok && a <= EM && r <= EM && s <= EM && o <= EM && rc <= EM;
      sum += a + r + s;
      osum += o + rc;  // every o_j <= O + max Rcut (NEXT-1)
    }
    ps[part][p] = ok ? sum : -1;
    pos[part][p] = osum;
  }
  __syncthreads();
  if (t < 64) {
    const int64_t SM = (int64_t)UNIAP_MAX_SUM;
    bool ok = live;
    int64_t sum = 0, osum = 0;
    for (int j = 0; j < 4; ++j) {
      ok = ok && ps[j][t] >= 0;
      sum += ps[j][t];
      osum += pos[j][t];
    }
    ok = ok && sum <= SM && osum <= SM;
    const unsigned m = __ballot_sync(0xffffffffu, ok);
    if ((t & 31) == 0) pmask[t >> 5] = m;
  }
  __syncthreads();
  if (t == 0) {
    // the smallest feasible candidate (every check is monotone in q)
    const unsigned long long m = (unsigned long long)pmask[0] | (unsigned long long)pmask[1] << 32;
    int64_t q = -1;
    if (expl) q = (m & 1ull) ? cl.quantum : -1;
    else if (m) q = (int64_t)1 << (__ffsll((long long)m) - 1);
    bb.qcfg[blockIdx.x] = q;
    __threadfence();
    unsigned int* done = reinterpret_cast<unsigned int*>(bb.qglob + 2);
    okp[0] = atomicAdd(done, 1u) == gridDim.x - 1;  // this block finished last
  }
  __syncthreads();
  // the last config block sets the global quantum = max over the configs
  // (every check is monotone in q), or flags "no quantum fits"
  if (okp[0] && t < 32) {
    __threadfence();
    long long g = 1;
    for (int i = t; i < (int)gridDim.x; i += 32) {
      const long long x = *reinterpret_cast<volatile long long*>(bb.qcfg + i);
      g = (x < 0 || g < 0) ? -1 : max(g, x);
    }
    for (int o = 16; o > 0; o >>= 1) {
      const long long y = __shfl_xor_sync(0xffffffffu, g, o);
      g = (y < 0 || g < 0) ? -1 : max(g, y);
    }
    if (t == 0) {
      if (g < 0) atomicOr(reinterpret_cast<unsigned long long*>(bb.qglob + 1), 2ull);
      bb.qglob[0] = g;
      *reinterpret_cast<unsigned int*>(bb.qglob + 2) = 0u;  // ready for the next run (graph replays)
    }
  }
}

// Memory bucket of a byte count (reading A-8): ceil(bytes / unit), cap + 1
// (= forbidden) when it does not fit or the strategy is forbidden (bytes < 0).
__device__ __forceinline__ int32_t mem_bucket(int64_t byt, int64_t unit, int cap) {
  const int64_t bk = byt < 0 ? (int64_t)cap + 1 : (byt + unit - 1) / unit;
  return (int32_t)(bk > cap ? cap + 1 : bk);
}

// K1f role of the last block column: the feasible prefix of every forward
// P-emitting sweep of config blockIdx.y (one warp per sweep, lanes over its
// layers).  Eq. 5 bounds the memory of every state at the i-th layer swept
// by cap, and that memory is at least the running sum of each swept layer's
// smallest bucket (only M[s][ks] at the skip source of a conditioned copy);
// past the first layer where the sum exceeds cap every state is INF, so the
// sweep stops there (Inst::n) and the later interval optima stay INF from
// the fill.  Exact; computed from the builder's own M, rewritten every run
// from the planned length n0.
__device__ void k1f_trim(const ClusterDev& cl, const BuildBufs& bb, const CfgDev& cf, int cfg_id, int L, int tb,
                         int ntb) {
  __shared__ int32_t minb[MAXL];            // per layer: the smallest bucket over the config's strategies
  __shared__ int32_t skb[UNIAP_MAX_STRAT];  // the skip source's bucket per strategy (conditioned copies)
  __shared__ unsigned long long wsum[2];
  const int cap = cl.Q - 1;
  const int64_t unit = (cl.mem_bytes - cl.mem_reserve) / cap;
  const int t = threadIdx.x, lane = t & 31, nw = blockDim.x >> 5;
  if (t < 2) wsum[t] = 0;
  // per memory table (1F1B: one per distinct in-flight count), the sweeps
  // whose level reads it
  for (int mt = 0; mt < cf.nmt; ++mt) {
  const int64_t* M = bb.ns + cf.offM + (int64_t)mt * L * cf.NSP;
  __syncthreads();  // (minb / skb of the previous table consumed)
  if (t < L) {  // bucket(min bytes) = min bucket (ceil is monotone); forbidden (< 0) excluded
    int64_t mn = -1;
    for (int k = 0; k < cf.S; ++k) {
      const int64_t x = M[t * cf.NSP + k];
      if (x >= 0 && (mn < 0 || x < mn)) mn = x;
    }
    minb[t] = mem_bucket(mn, unit, cap);
  } else if (t >= 64 && t < 64 + cf.S && cf.skip >= 0) {
    skb[t - 64] = mem_bucket(M[cf.skip * cf.NSP + (t - 64)], unit, cap);
  }
  __syncthreads();
  const unsigned long long S = cf.S, Qw = cl.Q;
  const int i0 = bb.inst_off[cfg_id], i1 = bb.inst_off[cfg_id + 1];
  // this config's forward sweeps, one warp each, over the ntb trim blocks
  for (int q = i0 + tb * nw + (t >> 5); q < i1; q += ntb * nw) {
    const int j = bb.inst_idx[q];
    const Inst in = bb.inst[j];
    if (cf.lmt[in.lev] != mt) continue;  // (another memory table's pass)
    if (in.emit != 1 && in.emit != 2) {  // a G-keeping sweep runs in full
      if (lane == 0 && S > 1) {          // (|S| = 1: the closed form, no DP cells)
        atomicAdd(&wsum[0], (unsigned long long)in.n0 * S * Qw);
        atomicAdd(&wsum[1], (unsigned long long)(in.n0 - 1) * S * S * Qw);
      }
      continue;
    }
    int pre = 0, first = in.n0;
    for (int h = 0; h * 32 < in.n0; ++h) {
      const int i = h * 32 + lane;
      int mn = 0;
      if (i < in.n0) {
        const int u = in.a + in.dir * i;
        mn = (in.ks >= 0 && u == cf.skip) ? skb[in.ks] : minb[u];
      }
      int x = mn;  // inclusive scan over this half's layers
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      x += pre;
      const unsigned bad = __ballot_sync(0xffffffffu, i < in.n0 && x > cap);
      if (bad && first == in.n0) first = h * 32 + __ffs(bad) - 1;
      pre = __shfl_sync(0xffffffffu, x, 31);
    }
    if (lane == 0) {
      const int n = max(first, 1);
      bb.inst[j].n = n;
      // the emitted range within the layers swept (planned: forward elo = a,
      // ehi = a + n0 - 1; backward elo = a - n0 + 1)
      if (in.dir > 0) bb.inst[j].ehi = in.a + n - 1;
      else bb.inst[j].elo = in.a - n + 1;
      if (S > 1) {
        atomicAdd(&wsum[0], (unsigned long long)n * S * Qw);
        atomicAdd(&wsum[1], (unsigned long long)(n - 1) * S * S * Qw);
      }
    }
  }
  }  // memory tables
  __syncthreads();
  if (t < 2 && (wsum[t] || tb == 0)) atomicAdd(bb.work + 2 * cfg_id + t, wsum[t]);  // (zeroed by K1d)
}

// K1f: quantise into the int32 device layout (A, M buckets, Rt, Rf, Rs, O);
// the last block column trims the forward sweeps (k1f_trim).
__global__ void k1f_quantise(ClusterDev cl, BuildBufs bb, const CfgDev* __restrict__ cfgs, int L, int32_t* arena) {
  pdl_wait();  // K1d's quantum (PDL)
  TraceScope tr(TR_K1F);
  const CfgDev& cf = cfgs[blockIdx.y];  // (by reference: k1f_trim indexes its arrays)
  const int nqb = gridDim.x - bb.n_trim;  // quantising blocks; then the trim blocks
  if ((int)blockIdx.x >= nqb) {
    k1f_trim(cl, bb, cf, blockIdx.y, L, blockIdx.x - nqb, bb.n_trim);
    return;
  }
  const int NSP = cf.NSP, n2 = NSP * NSP;
  const int64_t q = bb.qglob[0] > 0 ? bb.qglob[0] : 1;
  const int cap = cl.Q - 1;
  const int64_t unit = (cl.mem_bytes - cl.mem_reserve) / cap;  // reading A-8
  const int nA = L * NSP, nR = (L - 1) * n2, nS = (cf.nsk >= 2 ? cf.nsk : 1) * L * n2, nO = ((L - 1) + 3) & ~3;
  const int nRc = cf.cut ? (L - 1) * n2 : 0;  // NEXT-1 Rcut block
  const int nMt = cf.nmt * nA;                  // the memory tables
  const bool pow2 = (q & (q - 1)) == 0;
  const int sh = __ffsll(q) - 1;
  auto qt = [&](int64_t x) { return (int32_t)(pow2 ? (x + q - 1) >> sh : (x + q - 1) / q); };
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < nA + nMt + nR + nS + nO + nRc; idx += nqb * blockDim.x) {
    int j = idx;
    if (j < nA) { arena[cf.offA + j] = qt(bb.ns[cf.offA + j]); continue; }
    j -= nA;
    if (j < nMt) {
      arena[cf.offM + j] = mem_bucket(bb.ns[cf.offM + j], unit, cap);
      continue;
    }
    j -= nMt;
    if (j < nR) {  // Rf = R, Rt = transpose within each edge
      const int e = j / n2, k = (j - e * n2) / NSP, l = j - e * n2 - k * NSP;
      const int32_t v = qt(bb.ns[cf.offRf + j]);
      arena[cf.offRf + j] = v;
      arena[cf.offRt + (int64_t)e * n2 + l * NSP + k] = v;
      continue;
    }
    j -= nR;
    if (j < nS) { arena[cf.offRs + j] = qt(bb.ns[cf.offRs + j]); continue; }
    j -= nS;
    if (j < nO) { arena[cf.offO + j] = j < L - 1 ? qt(bb.ns[cf.offO + j]) : 0; continue; }
    j -= nO;
    arena[cf.offRc + j] = qt(bb.ns[cf.offRc + j]);  // NEXT-1 Rcut
  }
}

// K1g (NEXT-4, several skip sources): the conditioning copies of every
// contiguous run of sources (CfgDev::cprel) from the quantised tables --
// A' = A + the run's skip-edge terms into every later layer, M' = M with each
// run source held on its strategy of the copy (the others forbidden); the
// same rule as the level-1 packing (uniap_prepare_tables).
__global__ void k1g_copies(const CfgDev* __restrict__ cfgs, int L, int cap, int32_t* arena) {
  pdl_wait();  // K1f's quantised tables (PDL)
  const CfgDev& cf = cfgs[blockIdx.y];
  if (cf.nsk < 2) return;
  const int S = cf.S, N = cf.NSP, n2 = N * N;
  const int64_t pair = copy_words(cf, L);  // A', then M' per memory table
  int64_t total = 0;
  for (int jlo = 0; jlo < cf.nsk; ++jlo)
    for (int jhi = jlo; jhi < cf.nsk; ++jhi) {
      int64_t ncp = 1;
      for (int j = jlo; j <= jhi; ++j) ncp *= S;
      total += ncp * pair;
    }
  const int32_t* A = arena + cf.offA;
  const int32_t* M = arena + cf.offM;
  const int32_t* Rs = arena + cf.offRs;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    // the run holding word idx (runs in layout order: jlo, then jhi)
    int64_t rem = idx;
    int jlo = 0, jhi = 0;
    for (jlo = 0; jlo < cf.nsk; ++jlo) {
      bool found = false;
      for (jhi = jlo; jhi < cf.nsk; ++jhi) {
        int64_t ncp = 1;
        for (int j = jlo; j <= jhi; ++j) ncp *= S;
        if (rem < ncp * pair) { found = true; break; }
        rem -= ncp * pair;
      }
      if (found) break;
    }
    const int kap = (int)(rem / pair);
    const int w = (int)(rem - (int64_t)kap * pair);
    const bool isM = w >= L * N;
    const int mt = w / (L * N) - 1;  // (isM: the memory table of this M')
    const int u = (w % (L * N)) / N, k = w % N;
    int32_t v;
    if (k >= S) {
      v = isM ? cap + 1 : 0;
    } else if (isM) {
      v = M[((int64_t)mt * L + u) * N + k];
      for (int j = jlo, r = kap; j <= jhi; ++j, r /= S)
        if (u == cf.sk[j] && k != r % S) v = cap + 1;
    } else {
      v = A[u * N + k];
      for (int j = jlo, r = kap; j <= jhi; ++j, r /= S)
        if (u >= cf.sk[j] + 2) v += Rs[(((int64_t)j * L + u) * N + r % S) * N + k];
    }
    arena[cf.offA + cf.cprel[jlo * UNIAP_MAX_SKIP + jhi] + (int64_t)kap * pair + w] = v;
  }
  (void)n2;
}

cudaError_t launch_k1(const ClusterDev& cl, const BuildBufs& bb, const CfgDev* cfg, int ncfg, int L, int skip,
                      int32_t* arena, cudaStream_t st) {
  // qmax / qglob are zeroed by uniap_prepare and left zeroed by K1d (qmax,
  // done counter); the range flags qglob[1] are sticky for the prepared input
  const int nbA = (bb.max_nmt * L * 32 + K1T - 1) / K1T;  // (NSP <= 32) x the memory tables
  const int nbR = (L - 1) + bb.n_src * L;  // one block per edge slot: L-1 chain edges, L skip destinations per source
  const int nbE = bb.cut_mat ? L - 1 : 0;  // NEXT-1 cut-cost blocks (per chain edge)
  k1_costs<<<dim3(nbA + nbR + nbE + 1, ncfg), K1T, 0, st>>>(cl, bb, cfg, L, nbA, nbR, nbE);
  cudaError_t e = pdl_launch(k1d_quantum, dim3(ncfg), dim3(256), 0, st, cl, bb, cfg, L, skip);
  if (e != cudaSuccess) return e;
  e = pdl_launch(k1f_quantise, dim3(16 + (bb.inst ? bb.n_trim : 0), ncfg), dim3(256), 0, st, cl, bb, cfg, L, arena);
  if (e != cudaSuccess) return e;
  if (bb.n_src >= 2) {  // NEXT-4: the conditioning copies
    e = pdl_launch(k1g_copies, dim3(32, ncfg), dim3(256), 0, st, cfg, L, cl.Q - 1, arena);
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

cudaError_t builder_trace(unsigned long long* p) { return cudaMemcpyToSymbol(g_trace, &p, sizeof p); }

cudaError_t builder_init() {
  for (const void* f : {(const void*)k1_costs, (const void*)k1d_quantum, (const void*)k1f_quantise}) {
    cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace uniap
