// chain_dp.cuh -- K2: the batched tropical chain DP (the hot kernel).
//
// One "instance" sweeps a chain of layers for one candidate config, starting
// at layer a (forward: a, a+1, ...; backward: b, b-1, ... for the traceback).
// The state D[k][q] is the minimum of Eq. (3)'s stage cost over the layers
// swept so far, with the current layer on strategy k and the memory sum of
// Eq. (5) at most q buckets.  Each step is
//   E[k][x] = min( INF, min_k' ( D[k'][x] + R[k'][k] + A'[u][k] ) )
//                    (min-plus mat-vec per bucket; R = the resharding term of
//                     Eq. 3, A' = the execution cost A plus skip-edge terms)
//   D[k][q] = E[k][q - M[u][k]]   (shift by the layer's memory, INF where q < M)
// and a forward instance emits P[a][u] = min_k D[k][cap] (the stage optimum of
// [a,u]).  The transposed order of the two updates (E first, then the shift)
// keeps the |S|^2 work of a bucket inside one thread.
//
// Mapping (sm_100a): a CTA (or a thread-block cluster of C CTAs splitting the
// bucket axis) owns one instance.  Thread t of CTA r owns buckets
// q = r*B + j*T + t (j < V): D lives in REGISTERS and the E-step is
// register-only: one DPX VIADDMNMX (__viaddmin_s32) per relaxation, two
// destination rows at a time (2V independent chains).  The step's R rows and
// A'/M rows are staged in shared memory one step ahead by the whole CTA (a
// broadcast LDS.128 per 4 sources; no L1 dependence, which a cluster barrier
// flushes).  E goes to shared memory, double-buffered, so each layer costs one
// barrier; the shifted read E[k][q-M] (M warp-uniform) is bank-conflict-free
// and a guard word (INF) before every row turns q < M into a clamped read.
// In a cluster the shifted read may fall in a lower CTA's bucket range:
// DSMEM (ld.shared::cluster) on that path only.
#pragma once
#include <type_traits>

#include "uniap_impl.h"

namespace uniap {

__device__ __forceinline__ int32_t addmin(int32_t a, int32_t b, int32_t c) { return __viaddmin_s32(a, b, c); }

__device__ __forceinline__ uint32_t cl_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cl_size() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void cl_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cl_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Cluster wait that also yields a token (0) for the loads that must follow it.
__device__ __forceinline__ uint32_t cl_wait_tok() {
  uint32_t tok;
  asm volatile("barrier.cluster.wait.acquire.aligned;\n\tmov.u32 %0, 0;" : "=r"(tok)::"memory");
  return tok;
}
// 32-bit shared::cluster addressing; the load is not volatile (loads can be
// batched) and is ordered after the barrier through its address operand.
__device__ __forceinline__ uint32_t mapa32(uint32_t la, uint32_t rank) {
  uint32_t r;
  asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(la), "r"(rank));
  return r;
}
__device__ __forceinline__ int32_t ld_cluster(uint32_t addr) {
  int32_t v;
  asm("ld.shared::cluster.s32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
// Generic address of the same shared-memory word in CTA `rank` of the
// cluster (pure: the load itself is an ordinary C++ load, so the compiler
// keeps it after the barrier and may batch several of them).
__device__ __forceinline__ const int32_t* map_rank(const int32_t* p, uint32_t rank) {
  uint64_t r;
  asm("mapa.u64 %0, %1, %2;" : "=l"(r) : "l"(reinterpret_cast<uint64_t>(p)), "r"(rank));
  return reinterpret_cast<const int32_t*>(r);
}
__device__ __forceinline__ int4 lds128(uint32_t addr) {
  int4 v;
  asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ int2 lds64(uint32_t addr) {
  int2 v;
  asm volatile("ld.shared.v2.s32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ int32_t lds32(uint32_t addr) {
  int32_t v;
  asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}

// Compile-time loop: f(integral_constant<int, I>) for I = B .. E-1.
template <int I, int E, typename F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (I < E) {
    f(std::integral_constant<int, I>{});
    static_for<I + 1, E>(f);
  }
}

__device__ __forceinline__ int comp(const int4& v, int i) { return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w; }

// Shared-memory words of one "table stage" (the tables of one layer step):
// R rows [NS][NSP], then (A', M) pairs [NSP].
template <int NS>
struct Stage {
  static constexpr int NSP = (NS + 3) & ~3;
  static constexpr int WORDS = NS * NSP + 2 * NSP;
};

// TM: a NEXT-1 launch (per-strategy emission into T, K2Args::tmode); only
// one-CTA double-buffered shapes are instantiated with it.
template <int NS, int V, int T, bool CL, bool DB = true, bool TM = false>
__global__ void __launch_bounds__(T) k2_chain(const K2Args args) {
  static_assert(DB || !CL, "single-buffered E only without clusters");
  constexpr int B = T * V;          // buckets per CTA
  constexpr int ROW = B + 4;        // 4 guard words + B buckets
  constexpr int NE = DB ? 2 : 1;    // E buffers (single: a second barrier per layer)
  constexpr int NSP = Stage<NS>::NSP;
  constexpr int SW = Stage<NS>::WORDS;
  constexpr int KUNROLL = 8;
  constexpr int MBIG = UNIAP_MAX_Q * 2 + 1;  // > every bucket index: "never fits"
  extern __shared__ int4 smem4[];
  int32_t* sE = reinterpret_cast<int32_t*>(smem4);  // [2][NS][ROW]
  int32_t* sT = sE + NE * NS * ROW;                 // [3][SW] staged tables
  int32_t* sProw = sT + 3 * SW;                     // [MAXL] this instance's P[a][.]
  const int t = threadIdx.x;
  int rank = 0, ii = blockIdx.x;
  if constexpr (CL) {
    rank = (int)cl_rank();
    ii = blockIdx.x / (int)cl_size();
  }
  if (args.n_inst && ii >= *args.n_inst) return;  // device-sized launch: spare CTA (whole cluster)
  const unsigned long long t_start = (args.trace || args.tim) ? gtimer() : 0ull;
  const Inst in = args.inst[ii];
  const CfgDev cf = args.cfg[in.cfg];
  const int32_t* __restrict__ gA = args.arena + cf.offA + in.arel;  // (NEXT-4: a conditioning copy's A')
  const int32_t* __restrict__ gM = args.arena + cf.offM + in.mrel;  // the sweep's memory table (1F1B: its stage's)
  const int32_t* __restrict__ gR = args.arena + (in.dir > 0 ? cf.offRt : cf.offRf);
  const int32_t* __restrict__ gRs = args.arena + cf.offRs;
  const int skip = cf.skip, ks = in.ks, cap = args.cap;
  const int Q = cap + 1;
  const int L = args.L;

  for (int r = t; r < NE * NS; r += T) *reinterpret_cast<int4*>(sE + r * ROW) = make_int4(INF, INF, INF, INF);

  // ---- tables of one layer step, staged by the whole CTA ----------------
  // word w of a stage: R rows (w < NS*NSP), then (A', M) pairs.  A' adds the
  // skip-edge term of Eq. 3 when the instance conditions the skip source;
  // strategies excluded by that conditioning get an unreachable memory.
  constexpr int PER = (SW + T - 1) / T;
  // R' = R + A'[u][dest]: the layer's execution cost (plus the skip-edge term)
  // rides on the resharding row of its destination strategy, so the E-step
  // yields A' + min_k'(D + R) directly and the shift is a plain shifted copy.
  // (D <= INF = 2^30, R' <= 2^23: no overflow; the INF-initialised
  // accumulator clamps every E at INF.)
  // Raw words are loaded two layers ahead and combined only when stored one
  // layer ahead, so no arithmetic waits on an in-flight load (the loads go
  // to L2: every cluster barrier invalidates L1).
  int32_t pre_x[PER], pre_a[PER], pre_s[PER];  // R or M word, A, Rskip
  int pre_u = 0;                                // layer of the fetched stage
  auto fetch_stage = [&](int step, int u_next) {  // global -> registers (issued early)
    const int e = in.dir > 0 ? u_next - 1 : u_next;
    const bool sk = ks >= 0 && u_next >= skip + 2;
    pre_u = u_next;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int w = t + i * T;
      pre_x[i] = pre_a[i] = pre_s[i] = 0;
      if (w < SW && step < in.n) {
        const bool isR = w < NS * NSP;
        const int x = w - NS * NSP;
        const int k = isR ? w / NSP : (x >> 1);
        pre_x[i] = isR ? __ldg(gR + (int64_t)e * NSP * NSP + w) : ((x & 1) ? __ldg(gM + (int64_t)u_next * NSP + k) : 0);
        pre_a[i] = (isR || !(x & 1)) ? __ldg(gA + (int64_t)u_next * NSP + k) : 0;
        pre_s[i] = (sk && (isR || !(x & 1))) ? __ldg(gRs + ((int64_t)u_next * NSP + ks) * NSP + k) : 0;
      }
    }
  };
  auto store_stage = [&](int step) {  // registers -> shared (before the barrier)
    int32_t* dst = sT + (step % 3) * SW;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int w = t + i * T;
      if (w < SW) {
        int32_t v;
        if (w < NS * NSP) {
          v = pre_x[i] + pre_a[i] + pre_s[i];  // R' = R + A' of the destination
        } else {
          const int x = w - NS * NSP, k = x >> 1;
          if (x & 1) {
            v = min(pre_x[i], MBIG);
            if (ks >= 0 && pre_u == skip && k != ks) v = MBIG;
          } else {
            v = pre_a[i] + pre_s[i];
          }
        }
        dst[w] = v;
      }
    }
  };

  int32_t d[NS][V];
  const bool eP = (in.emit & 3) != 0, eG = in.emit == 0 || (in.emit & 4) != 0;  // Inst::emit
  auto emit = [&](int u) {
    if (eP) {  // the stage optimum under the launch's cap level: min_k D[k][ecap] (a kernel parameter)
      const int rc = args.ecap / B;
      if (rank == rc) {
        const int lc = args.ecap - rc * B, jc = lc / T, tc = lc - jc * T;
        if (t == tc) {
          int32_t v = INF;
#pragma unroll
          for (int j = 0; j < V; ++j)
            if (j == jc)
#pragma unroll
              for (int k = 0; k < NS; ++k) v = min(v, d[k][j]);
          sProw[u] = v;  // written to global after the sweep (no global store
                         // outstanding at the per-layer cluster barrier)
          if constexpr (TM) {  // NEXT-1: every strategy's state at ecap, flushed after the sweep
            int32_t* row = sProw + MAXL + u * NSP;
#pragma unroll
            for (int j = 0; j < V; ++j)
              if (j == jc)
#pragma unroll
                for (int k = 0; k < NS; ++k) row[k] = d[k][j];
          }
        }
      }
    }
    if (eG) {
      const int lo = in.a - in.n + 1;
      int32_t* g = args.G + in.gofs + (int64_t)(u - lo) * NSP * Q;
#pragma unroll
      for (int k = 0; k < NS; ++k)
#pragma unroll
        for (int j = 0; j < V; ++j) {
          const int q = rank * B + j * T + t;
          if (q < Q) g[(int64_t)k * Q + q] = d[k][j];
        }
    }
  };

  // ---- first layer ----
  int u = in.a;
  {
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      int32_t a = __ldg(gA + (int64_t)u * NSP + k);
      int32_t m = min(__ldg(gM + (int64_t)u * NSP + k), MBIG);
      if (ks >= 0) {
        if (u >= skip + 2) a += __ldg(gRs + ((int64_t)u * NSP + ks) * NSP + k);
        if (u == skip && k != ks) m = MBIG;
      }
      if (in.kf >= 0 && k != in.kf) m = MBIG;  // NEXT-1: the first layer on strategy kf
#pragma unroll
      for (int j = 0; j < V; ++j) d[k][j] = (rank * B + j * T + t >= m) ? a : INF;
    }
  }
  fetch_stage(1, u + in.dir);
  store_stage(1);
  if (in.n > 2) fetch_stage(2, u + 2 * in.dir);
  __syncthreads();
  emit(u);

  for (int step = 1; step < in.n; ++step) {
    u += in.dir;
    int32_t* Eb = sE + (DB ? (step & 1) * NS * ROW : 0) + 4;  // row 0, bucket 0
    const int32_t* Tb = sT + (step % 3) * SW;
    // ---- E-step: registers only; R broadcast from shared memory ----
    // RR destination rows per pass: RR*V independent VIADDMNMX chains.
    {
      int32_t* Et = Eb + t;
      auto rows = [&](auto rrc, int k) {
        constexpr int RR = decltype(rrc)::value;
        int32_t acc[RR][V];
#pragma unroll
        for (int r = 0; r < RR; ++r)
#pragma unroll
          for (int j = 0; j < V; ++j) acc[r][j] = INF;
#pragma unroll
        for (int c = 0; c < NSP / 4; ++c) {
          int4 x[RR];
#pragma unroll
          for (int r = 0; r < RR; ++r) x[r] = reinterpret_cast<const int4*>(Tb + (k + r) * NSP)[c];
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (4 * c + i < NS)
#pragma unroll
              for (int r = 0; r < RR; ++r)
#pragma unroll
                for (int j = 0; j < V; ++j) acc[r][j] = addmin(d[4 * c + i][j], comp(x[r], i), acc[r][j]);
        }
#pragma unroll
        for (int r = 0; r < RR; ++r)
#pragma unroll
          for (int j = 0; j < V; ++j) Et[(k + r) * ROW + j * T] = acc[r][j];
      };
      constexpr int RR = (V >= 8) ? 2 : (V >= 4 ? 2 : 4);
      constexpr int RRC = RR < NS ? RR : NS;
      constexpr int NFULL = NS / RRC * RRC;
      if constexpr (NS <= KUNROLL) {
#pragma unroll
        for (int k = 0; k < NFULL; k += RRC) rows(std::integral_constant<int, RRC>{}, k);
      } else {
#pragma unroll 1
        for (int k = 0; k < NFULL; k += RRC) rows(std::integral_constant<int, RRC>{}, k);
      }
      if constexpr (NS - NFULL > 0) rows(std::integral_constant<int, NS - NFULL>{}, NFULL);
    }
    // Split-phase: arrive on the cluster barrier (release E; before staging
    // the next tables, which only this CTA reads, so the release does not
    // wait for those stores), stage the tables of the step after next, issue
    // the next table fetch, sync the CTA, shift from the local E while the
    // other CTAs catch up, then wait (acquire) before the few reads from a
    // lower CTA's range.
    if constexpr (CL) cl_arrive();
    if (step + 1 < in.n) store_stage(step + 1);
    if (step + 2 < in.n) fetch_stage(step + 2, u + 2 * in.dir);
    __syncthreads();
    // ---- shift by the layer's memory, add A' ----
    // Byte addresses in the shared window: row k's bucket x sits at
    // rowb_k + 4x; x < 0 is clamped onto the guard word at rowb_k - 4 by one
    // VIADDMNMX (max form), so a cell costs VIADDMNMX + LDS + VIADDMNMX.
    const char* Ec = reinterpret_cast<const char*>(Eb);
    int32_t mmax = 0;  // largest shift of this layer (for the DSMEM fix-up test)
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      const int2 am = *reinterpret_cast<const int2*>(Tb + NS * NSP + 2 * k);
      if constexpr (CL) mmax = max(mmax, am.y <= cap ? am.y : 0);  // forbidden rows are all INF
      const int32_t bk = (k * ROW + t - am.y) * 4;  // byte offset of bucket t - M in row k
      const int32_t gk = k * ROW * 4 - 4;          // the row's guard word
      if (V > 1 && am.y <= T) {
        // (warp-uniform) only j = 0 can fall below the row start: the other
        // buckets read at constant offsets from one clamped base
        const char* base = Ec + bk;
        d[k][0] = *reinterpret_cast<const int32_t*>(Ec + max(bk, gk));
#pragma unroll
        for (int j = 1; j < V; ++j) d[k][j] = *reinterpret_cast<const int32_t*>(base + j * T * 4);
      } else {
#pragma unroll
        for (int j = 0; j < V; ++j)
          d[k][j] = *reinterpret_cast<const int32_t*>(Ec + __viaddmax_s32(bk, j * T * 4, gk));
      }
    }
    if constexpr (CL) {
      // buckets whose shifted source q - M lies in a lower CTA's range: the
      // local read above returned the guard (INF); fetch the value over DSMEM
      const uint32_t tok = cl_wait_tok();
      const int wbase = t & ~31;
      if (rank > 0 && wbase < mmax && mmax <= T) {
        // common case (every shift <= T): only bucket j = 0 of threads t < M_k
        // needs a fix-up, and its source is bucket B + t - M_k of CTA rank-1:
        // one mapped base per layer, one predicated load per row
        // (generic loads: ordered after the wait by its memory clobber)
        const int32_t* rb = map_rank(Eb + B + t, (uint32_t)rank - 1);
#pragma unroll
        for (int k = 0; k < NS; ++k) {
          const int mk = Tb[NS * NSP + 2 * k + 1];  // > cap >= T when forbidden
          if (t < mk && mk <= T) d[k][0] = rb[k * ROW - mk];
        }
      } else if (rank > 0 && wbase < mmax) {  // warp-uniform: only the low warps of a CTA
        // predicated loads, all in flight together: a cell that needs no
        // fix-up reads its own E word (shared::cluster window, own rank)
        const uint32_t ebase = (uint32_t)__cvta_generic_to_shared(Eb) + tok;
#pragma unroll
        for (int k = 0; k < NS; ++k) {
          const int mk = Tb[NS * NSP + 2 * k + 1];
#pragma unroll
          for (int j = 0; j < V; ++j) {
            const int lx = j * T + t - mk;
            const int x = lx + rank * B;
            const bool need = lx < 0 && x >= 0;
            const int xc = need ? x : rank * B + j * T + t;  // own word when no fix-up
            const uint32_t la = ebase + (uint32_t)((k * ROW + (xc & (B - 1))) * 4);
            const int32_t v = ld_cluster(mapa32(la, (uint32_t)(xc / B)));
            d[k][j] = need ? v : d[k][j];
          }
        }
      }
    }
    if constexpr (!DB) __syncthreads();  // E is rewritten by the next layer
    emit(u);
  }
  // the forward sweep's stage optima P[a][a..a+n-1], from its owner thread
  if (eP && rank == args.ecap / B && t == (args.ecap - (args.ecap / B) * B) % T) {
    int32_t* Pc = args.P + cf.offP + (int64_t)args.inst[ii].lev * L * L;  // (read here: not live in the loop)
    for (int uu = in.elo; uu <= in.ehi; ++uu) {  // (the trim keeps [elo, ehi] inside the layers swept)
      int32_t* dst = in.dir > 0 ? Pc + (int64_t)in.a * L + uu : Pc + (int64_t)uu * L + in.a;
      if ((in.emit & 3) == 2) atomicMin(dst, sProw[uu]);
      else *dst = sProw[uu];
    }
    if constexpr (TM) {  // NEXT-1: T[a][b][kf'][kl'] of the config, index NSP = that end free
      constexpr int W = NSP + 1;
      int32_t* Tc = args.T + cf.offT;
      const int kf = args.inst[ii].kf;
      for (int uu = in.elo; uu <= in.ehi; ++uu)
        for (int k = 0; k < NS; ++k) {
          // forward from a: first = kf (or free), last = k; backward (suffix) from
          // L-1: first = k, last free
          const int64_t i = in.dir > 0 ? (((int64_t)in.a * L + uu) * W + (kf < 0 ? NSP : kf)) * W + k
                                       : (((int64_t)uu * L + in.a) * W + k) * W + NSP;
          const int32_t v = sProw[MAXL + uu * NSP + k];
          if ((in.emit & 3) == 2) atomicMin(Tc + i, v);
          else Tc[i] = v;
        }
    }
  }
  if constexpr (CL) cl_sync();  // keep this CTA's E alive for remote readers
  if (args.trace && t == 0) trace_put(args.trace, args.tag, t_start, rank, ii, in.n);
  if (args.tim && t == 0) {  // the forward phase's device time (uniap_fetch: ms_gpu_dp)
    atomicMax(args.tim, ~t_start);
    atomicMax(args.tim + 1, gtimer());
  }
}

template <int NS>
constexpr size_t k2_smem(int B, int ne = 2) {
  return (size_t)(ne * NS * (B + 4) + 3 * Stage<NS>::WORDS + MAXL) * sizeof(int32_t);
}
// + the per-strategy rows of a NEXT-1 (tmode) launch
template <int NS>
constexpr size_t k2_smem_t() {
  return (size_t)MAXL * Stage<NS>::NSP * sizeof(int32_t);
}

// Instantiation helper used by the per-NS translation units: only the shapes
// the class chooser (chain_dp.cu, k2_pick_class) can return are instantiated.
typedef void (*k2_fn)(const K2Args);

template <int NS>
k2_fn k2_get(int V, int T, bool CL, bool DB, bool TM) {
  if (TM) {  // NEXT-1 launches: one CTA per sweep, double-buffered (k2_pick_class_t)
    if (CL || !DB) return nullptr;
#define UNIAP_TSHAPE(VV, TT)                                                                   \
  if (V == VV && T == TT) {                                                                    \
    if constexpr (k2_smem<NS>(VV * TT) + k2_smem_t<NS>() <= 200 * 1024)                       \
      return k2_chain<NS, VV, TT, false, true, true>;                                          \
    return nullptr;                                                                            \
  }
    UNIAP_TSHAPE(1, 32)
    UNIAP_TSHAPE(2, 32)
    UNIAP_TSHAPE(2, 64)
    UNIAP_TSHAPE(2, 128)
    UNIAP_TSHAPE(2, 256)
    UNIAP_TSHAPE(2, 512)
    if constexpr (NS <= 12) { UNIAP_TSHAPE(4, 512) }
#undef UNIAP_TSHAPE
    return nullptr;
  }
  if (!DB) {  // single-buffered E, one CTA per instance (large B without a cluster)
    if (CL) return nullptr;
    if constexpr (NS > 24 && k2_smem<NS>(1024, 1) <= 200 * 1024) if (V == 2 && T == 512) return k2_chain<NS, 2, 512, false, false>;
    if constexpr (NS > 12 && NS <= 24 && k2_smem<NS>(2048, 1) <= 200 * 1024) if (V == 4 && T == 512) return k2_chain<NS, 4, 512, false, false>;
    if constexpr (NS > 6 && NS <= 10) if (V == 8 && T == 512) return k2_chain<NS, 8, 512, false, false>;
    return nullptr;
  }
#define UNIAP_SHAPE(VV, TT)                                                 \
  if (V == VV && T == TT) {                                                 \
    if constexpr (k2_smem<NS>(VV * TT) <= 200 * 1024)                       \
      return CL ? k2_chain<NS, VV, TT, true> : k2_chain<NS, VV, TT, false>; \
    return nullptr;                                                         \
  }
  if (V == 1 && T == 32) return CL ? nullptr : k2_chain<NS, 1, 32, false>;
  UNIAP_SHAPE(2, 32)
  UNIAP_SHAPE(2, 64)
  UNIAP_SHAPE(2, 128)
  UNIAP_SHAPE(1, 128)
  UNIAP_SHAPE(1, 256)
  UNIAP_SHAPE(1, 512)
  UNIAP_SHAPE(2, 256)
  UNIAP_SHAPE(2, 512)
  if constexpr (NS <= 16) { UNIAP_SHAPE(4, 256) }
  if constexpr (NS <= 12) { UNIAP_SHAPE(4, 512) }
  if constexpr (NS <= 6) { UNIAP_SHAPE(8, 512) }
#undef UNIAP_SHAPE
  return nullptr;
}

}  // namespace uniap
