// chain_dp.cuh -- K2: the batched tropical chain DP (the hot kernel).
//
// One "instance" sweeps a chain of layers for one candidate config, starting
// at layer a (forward: a, a+1, ...; backward: b, b-1, ... for the traceback).
// The state D[k][q] is the minimum of Eq. (3)'s stage cost over the layers
// swept so far, with the current layer on strategy k and the memory sum of
// Eq. (5) at most q buckets.  Each step is
//   E[k][x] = min_k' ( D[k'][x] + R[k'][k] )        (min-plus mat-vec per bucket;
//                                                    R = the resharding term of Eq. 3)
//   D[k][q] = min( INF, A'[u][k] + E[k][q - M[u][k]] )  (shift by the layer's memory,
//                                                    INF where q < M)
// and a forward instance emits P[a][u] = min_k D[k][cap] (the stage optimum of
// [a,u]).  The transposed order of the two updates (E first, then the shift)
// keeps the |S|^2 work of a bucket inside one thread.
//
// Mapping (sm_100a): a CTA (or a thread-block cluster of C CTAs splitting the
// bucket axis) owns one instance.  Thread t of CTA r owns buckets
// q = r*B + j*T + t (j < V): D lives in REGISTERS, the E-step is
// register-only with one DPX VIADDMNMX per relaxation (__viaddmin_s32), R is a
// warp-uniform broadcast load reused across the V buckets, E goes to shared
// memory (double-buffered: one barrier per layer) so the shifted read
// E[k][q-M] -- a warp-uniform shift -- is bank-conflict-free.  A guard word
// (INF) before every row turns q < M into a clamped read.  In a cluster the
// shifted read may cross to the previous CTA's bucket range: DSMEM
// (ld.shared::cluster) on that path only.
#pragma once
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
__device__ __forceinline__ int32_t ld_dsmem(const int32_t* p, uint32_t rank) {
  uint32_t la = (uint32_t)__cvta_generic_to_shared(p), ra;
  int32_t v;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(rank));
  asm volatile("ld.shared::cluster.s32 %0, [%1];" : "=r"(v) : "r"(ra) : "memory");
  return v;
}

template <int NSP>
__device__ __forceinline__ void load_row(int32_t (&r)[NSP], const int32_t* __restrict__ p) {
  const int4* p4 = reinterpret_cast<const int4*>(p);
#pragma unroll
  for (int i = 0; i < NSP / 4; ++i) {
    int4 x = __ldg(p4 + i);
    r[4 * i] = x.x;
    r[4 * i + 1] = x.y;
    r[4 * i + 2] = x.z;
    r[4 * i + 3] = x.w;
  }
}

// E[k][.] for one destination strategy k: V independent VIADDMNMX chains of length NS.
template <int NS, int V, int T, int NSP, int ROW>
__device__ __forceinline__ void estep_k(const int32_t (&d)[NS][V], const int32_t (&r)[NSP], int32_t* E, int k) {
  int32_t acc[V];
#pragma unroll
  for (int j = 0; j < V; ++j) acc[j] = INF;
#pragma unroll
  for (int kp = 0; kp < NS; ++kp)
#pragma unroll
    for (int j = 0; j < V; ++j) acc[j] = addmin(d[kp][j], r[kp], acc[j]);
  int32_t* e = E + k * ROW;
#pragma unroll
  for (int j = 0; j < V; ++j) e[j * T] = acc[j];
}

template <int NS, int V, int T, bool CL, bool DB>
__global__ void __launch_bounds__(T) k2_chain(const K2Args args) {
  constexpr int B = T * V;          // buckets per CTA
  constexpr int ROW = B + 4;        // 4 guard words + B buckets
  constexpr int NSP = (NS + 3) & ~3;
  constexpr int NB = DB ? 2 : 1;
  constexpr int KUNROLL = 8;
  constexpr int MBIG = UNIAP_MAX_Q * 2 + 1;  // > every bucket index: "never fits"
  extern __shared__ int4 smem4[];
  int32_t* sE = reinterpret_cast<int32_t*>(smem4);
  const int t = threadIdx.x;
  int rank = 0, ii = blockIdx.x;
  if constexpr (CL) {
    rank = (int)cl_rank();
    ii = blockIdx.x / (int)cl_size();
  }
  const Inst in = args.inst[ii];
  const CfgDev cf = args.cfg[in.cfg];
  const int32_t* __restrict__ gA = args.arena + cf.offA;
  const int32_t* __restrict__ gM = args.arena + cf.offM;
  const int32_t* __restrict__ gR = args.arena + (in.dir > 0 ? cf.offRt : cf.offRf);
  const int32_t* __restrict__ gRs = args.arena + cf.offRs;
  const int skip = cf.skip, ks = in.ks, cap = args.cap;

  for (int r = t; r < NB * NS; r += T) *reinterpret_cast<int4*>(sE + r * ROW) = make_int4(INF, INF, INF, INF);

  // A'[u][k] (execution cost + skip-edge term when conditioned) and M[u][k];
  // a strategy excluded by the conditioning gets an unreachable memory.
  int32_t Ak[NSP], Mk[NSP];
  auto load_layer = [&](int u) {
    load_row<NSP>(Ak, gA + (int64_t)u * NSP);
    load_row<NSP>(Mk, gM + (int64_t)u * NSP);
#pragma unroll
    for (int k = 0; k < NSP; ++k) Mk[k] = min(Mk[k], MBIG);
    if (ks >= 0) {
      if (u >= skip + 2) {
        int32_t rs[NSP];
        load_row<NSP>(rs, gRs + ((int64_t)u * NSP + ks) * NSP);
#pragma unroll
        for (int k = 0; k < NSP; ++k) Ak[k] += rs[k];
      } else if (u == skip) {
#pragma unroll
        for (int k = 0; k < NSP; ++k)
          if (k != ks) Mk[k] = MBIG;
      }
    }
  };

  const int Q = cap + 1;
  const int L = args.L;
  int32_t d[NS][V];
  auto emit = [&](int u) {
    if (in.dir > 0) {
      const int rc = cap / B;
      if (rank == rc) {
        const int lc = cap - rc * B, jc = lc / T, tc = lc - jc * T;
        if (t == tc) {
          int32_t v = INF;
#pragma unroll
          for (int j = 0; j < V; ++j)
            if (j == jc)
#pragma unroll
              for (int k = 0; k < NS; ++k) v = min(v, d[k][j]);
          int32_t* dst = args.P + cf.offP + (int64_t)in.a * L + u;
          if (in.emit == 2) atomicMin(dst, v);
          else *dst = v;
        }
      }
    } else {
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

  int u = in.a;
  load_layer(u);
#pragma unroll
  for (int k = 0; k < NS; ++k)
#pragma unroll
    for (int j = 0; j < V; ++j) d[k][j] = (rank * B + j * T + t >= Mk[k]) ? Ak[k] : INF;
  emit(u);

  for (int step = 1; step < in.n; ++step) {
    const int up = u;
    u += in.dir;
    const int e = in.dir > 0 ? up : u;  // chain edge between the two layers
    const int32_t* __restrict__ Rm = gR + (int64_t)e * NSP * NSP;
    int32_t* Eb = sE + (DB ? (step & 1) * NS * ROW : 0) + 4;
    // ---- E-step: registers only ----
    {
      int32_t* Et = Eb + t;
      if constexpr (NS <= KUNROLL) {
#pragma unroll
        for (int k = 0; k < NS; ++k) {
          int32_t r[NSP];
          load_row<NSP>(r, Rm + k * NSP);
          estep_k<NS, V, T, NSP, ROW>(d, r, Et, k);
        }
      } else {
        int32_t ra[NSP], rb[NSP];
        load_row<NSP>(ra, Rm);
#pragma unroll 1
        for (int k = 0; k < NS; k += 2) {
          if (k + 1 < NS) load_row<NSP>(rb, Rm + (k + 1) * NSP);
          estep_k<NS, V, T, NSP, ROW>(d, ra, Et, k);
          if (k + 1 < NS) {
            if (k + 2 < NS) load_row<NSP>(ra, Rm + (k + 2) * NSP);
            estep_k<NS, V, T, NSP, ROW>(d, rb, Et, k + 1);
          }
        }
      }
    }
    load_layer(u);
    if constexpr (CL) cl_sync();
    else __syncthreads();
    // ---- shift by the layer's memory, add A' ----
    // Byte addresses in the shared window: row k's bucket x sits at
    // rowb_k + 4x; x < 0 is clamped onto the guard word at rowb_k - 4 by one
    // VIADDMNMX (max form), so a cell costs VIADDMNMX + LDS + VIADDMNMX.
    {
      const int32_t sb = (int32_t)__cvta_generic_to_shared(Eb);
#pragma unroll
      for (int k = 0; k < NS; ++k) {
        const int32_t rowb = sb + k * ROW * 4;
        const int32_t bk = rowb + (t - Mk[k]) * 4;
        const int32_t gk = rowb - 4;
#pragma unroll
        for (int j = 0; j < V; ++j) {
          const int32_t addr = __viaddmax_s32(bk, j * T * 4, gk);
          int32_t ev;
          asm volatile("ld.shared.s32 %0, [%1];" : "=r"(ev) : "r"(addr) : "memory");
          if constexpr (CL) {
            const int lx = j * T + t - Mk[k];
            if (lx < 0) {
              const int x = lx + rank * B;
              if (x >= 0) ev = ld_dsmem(Eb + k * ROW + (x & (B - 1)), (uint32_t)(x / B));
            }
          }
          d[k][j] = addmin(ev, Ak[k], INF);
        }
      }
    }
    if constexpr (!DB) {
      if constexpr (CL) cl_sync();
      else __syncthreads();
    }
    emit(u);
  }
  if constexpr (CL) cl_sync();  // keep this CTA's E alive for remote readers
}

// Instantiation helper used by the per-NS translation units: only the shapes
// the class chooser (chain_dp.cu, k2_pick_class) can return are instantiated.
typedef void (*k2_fn)(const K2Args);

template <int NS>
k2_fn k2_get(int V, int T, bool CL, bool DB) {
  if (!CL && DB) {
    if (V == 1 && T == 32) return k2_chain<NS, 1, 32, false, true>;
    if (V == 2 && T == 32) return k2_chain<NS, 2, 32, false, true>;
    if (V == 4 && T == 32) return k2_chain<NS, 4, 32, false, true>;
    if (V == 4 && T == 64) return k2_chain<NS, 4, 64, false, true>;
    if (V == 4 && T == 128) return k2_chain<NS, 4, 128, false, true>;
  }
  if (V == 4 && T == 256) {
    if constexpr (NS <= 24) {
      if (DB) return CL ? k2_chain<NS, 4, 256, true, true> : k2_chain<NS, 4, 256, false, true>;
    } else {
      if (!DB) return CL ? k2_chain<NS, 4, 256, true, false> : k2_chain<NS, 4, 256, false, false>;
    }
  }
  if constexpr (NS <= 6) {
    if (V == 8 && T == 512 && DB) return CL ? k2_chain<NS, 8, 512, true, true> : k2_chain<NS, 8, 512, false, true>;
  }
  return nullptr;
}

}  // namespace uniap
