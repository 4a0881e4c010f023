// combine.cu -- K3 (theta candidates), K4 (stage combine, Eq. 2), K5a
// (per-config and global argmin + stage ends), K5c (strategy walk).
//
// Combine (Eq. 2).  For a config with interval optima
// P[a][b] (K2) and cut costs O[e], the optimum over ordered placements of
//     tpi = sum_i p_i + sum_j o_j + (c-1) * max(P u O)
// is  min over theta of  Val(theta) = F_theta + (c-1) * theta,  where
// F_theta = min sum_i P[a_i][b_i] + sum_j O[b_j] over placements whose every
// P and O is <= theta, and theta ranges over the distinct P / O values (K3).
// Proof: for an optimal placement pi* with max X*, F_{X*} <= sum(pi*) so
// Val(X*) <= OPT; conversely the placement attaining F_theta has tpi <=
// Val(theta).  The optimal placements are exactly the argmin sets of F_theta
// over theta with Val(theta) = OPT.  For c = 1, Val =
// F_theta and the largest theta (no constraint) contains every argmin.
#include <cub/block/block_scan.cuh>

#include "uniap_impl.h"

namespace uniap {



__global__ void k_fill(int32_t* p, int64_t n, int32_t v) {
  TraceScope tr(TR_FILL);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

// Publish: copy the run's results (record, builder flags, phase clock,
// per-config optima) into the handle's mapped pinned host block with plain
// (zero-copy) stores, so a fetch is one stream sync and no DMA round trips.
__global__ void k_publish(int32_t* __restrict__ d_rec, const int32_t* __restrict__ rec, int rec_words,
                          int64_t* __restrict__ d_qg, const int64_t* __restrict__ qg,
                          unsigned long long* __restrict__ d_tm, const unsigned long long* __restrict__ tm,
                          int64_t* __restrict__ d_cfg, const int64_t* __restrict__ cfgopt, int ncfg) {
  pdl_wait();  // K5c's record (PDL)
  const int t = threadIdx.x;
  for (int i = t; i < rec_words; i += blockDim.x) d_rec[i] = rec[i];
  if (t < 2) {
    d_qg[t] = qg ? qg[t] : 0;
    d_tm[t] = tm ? tm[t] : 0ull;
  }
  for (int i = t; i < ncfg; i += blockDim.x) d_cfg[i] = cfgopt[i];
}

cudaError_t launch_publish(int32_t* d_rec, const uniap_record* rec, int64_t* d_qg, const int64_t* qg,
                           unsigned long long* d_tm, const unsigned long long* tm, int64_t* d_cfg,
                           const int64_t* cfgopt, int ncfg, cudaStream_t st) {
  static_assert(sizeof(uniap_record) % 4 == 0, "record words");
  cudaError_t e = pdl_launch(k_publish, dim3(1), dim3(256), 0, st, d_rec, reinterpret_cast<const int32_t*>(rec),
                             (int)(sizeof(uniap_record) / 4), d_qg, qg, d_tm, tm, d_cfg, cfgopt, ncfg);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_fill(int32_t* p, int64_t n, int32_t v, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
  k_fill<<<blocks, 256, 0, st>>>(p, n, v);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// K3: sorted distinct theta candidates per config (one CTA per config).
// ---------------------------------------------------------------------------
constexpr int K3T = 1024;
typedef cub::BlockScan<int, K3T> K3Scan;
// Sorted distinct theta candidates of config `cf` into v[0..n) (returns n):
// valid P[a][b] < INF and every O[e].  The values are first de-duplicated in
// an open-addressing hash set in v (identical layers make most of them
// equal), compacted with a block scan, then sorted: by rank counting when
// few (<= 64), else bitonic.  The config's P block and O row are copied to
// sP / sO on the way (K4 reads them from shared memory).
constexpr int32_t EMPTY = 0x7fffffff;
__device__ __forceinline__ void hset_insert(int32_t* v, int32_t x) {
  uint32_t h = ((uint32_t)x * 2654435761u) >> (32 - 12);  // SORTN = 4096 slots
  for (;;) {
    const int32_t old = atomicCAS(v + h, EMPTY, x);
    if (old == EMPTY || old == x) return;
    h = (h + 1) & (SORTN - 1);
  }
}
__device__ int sort_thetas(const CfgDev& cf, const int32_t* __restrict__ arena, const int32_t* __restrict__ P, int L,
                           int32_t* v, int32_t* sP, int32_t* sO, typename K3Scan::TempStorage& scan_tmp) {
  static_assert(SORTN == 4 * K3T, "4 hash slots per thread");
  const int t = threadIdx.x;
  for (int i = t; i < SORTN; i += K3T) v[i] = EMPTY;
  __syncthreads();
  const int32_t* Pc = P + cf.offP;  // one L*L table per cap level (NEXT-2)
  for (int idx = t; idx < cf.nlev * L * L; idx += K3T) {
    const int r = idx % (L * L), a = r / L, b = r - a * L;
    const int32_t x = Pc[idx];
    sP[idx] = x;
    if (a <= b && x < INF) hset_insert(v, x);
  }
  const int32_t* O = arena + cf.offO;
  for (int e = t; e < L - 1; e += K3T) {
    const int32_t x = O[e];
    sO[e] = x;
    hset_insert(v, x);
  }
  __syncthreads();
  int flags[4], c = 0;
  int32_t vals[4];
  for (int r = 0; r < 4; ++r) {
    vals[r] = v[4 * t + r];
    flags[r] = vals[r] != EMPTY;
    c += flags[r];
  }
  int pos, n;
  K3Scan(scan_tmp).ExclusiveSum(c, pos, n);
  __syncthreads();  // every read of v above is done before the compaction writes
  for (int r = 0; r < 4; ++r)
    if (flags[r]) v[pos++] = vals[r];
  __syncthreads();
  if (n <= 64) {  // rank counting (values are distinct)
    int32_t x = EMPTY;
    int rank = 0;
    if (t < n) {
      x = v[t];
      for (int j = 0; j < n; ++j) rank += v[j] < x;
    }
    __syncthreads();
    if (t < n) v[rank] = x;
    __syncthreads();
    return n;
  }
  int N = 2;
  while (N < n) N <<= 1;
  for (int i = n + t; i < N; i += K3T) v[i] = EMPTY;
  __syncthreads();
  for (int k = 2; k <= N; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = t; i < N; i += K3T) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const bool up = (i & k) == 0;
          const int32_t x = v[i], y = v[ixj];
          if ((x > y) == up) {
            v[i] = y;
            v[ixj] = x;
          }
        }
      }
      __syncthreads();
    }
  return n;
}

// ---------------------------------------------------------------------------
// Placement DPs by one warp over (stage i, end b); lanes own b (b = lane,
// lane + 32).  Stage i = [a, b] with i-1 <= a <= b <= L-1-(deg-i); the last
// stage ends at L-1.  sP: the config's P[L][L] in shared memory (INF for
// a > b and for intervals no placement uses), sO: O[L-1], g: 128 words of
// warp-private scratch holding w[a] = (best placement of stages < i ending
// at a-1) (+) O[a-1], double-buffered by stage parity.
//  F:          F_theta = min sum P + sum O over placements with every P, O <=
//              theta (theta = INF: no limit)   -- (min, +) semiring
//  BOTTLENECK: the bottleneck min over placements of max(P u O), i.e. the
//              smallest theta with a feasible placement -- (min, max) semiring
// The a-loop reads one broadcast w and one conflict-free P word per lane
// and accumulates with one DPX op (unsigned: INF + INF = 2^31 fits), two
// accumulators per column for ILP.
// ---------------------------------------------------------------------------
// slev[i]: the cap level of stage i (0-based; NEXT-2): stage i reads the
// interval table sP + slev[i] * L * L.
template <bool BOTTLENECK, bool MASK>
__device__ int32_t warp_dp(const int32_t* sPall, const int32_t* slev, const int32_t* sO, int32_t* g, int L, int deg,
                           int32_t theta) {
  const int lane = threadIdx.x & 31;
  const int b0 = lane, b1 = lane + 32;
  auto mask = [&](int32_t p) { return (MASK && p > theta) ? INF : p; };
  // w of the next stage from this stage's value c at column b (stage ends at b)
  auto put_w = [&](int32_t* w, int b, int32_t c) {
    if (b + 1 < L) {
      const int32_t o = sO[b];
      int32_t x;
      if (BOTTLENECK) x = max(c, o);
      else x = (c < INF && !(MASK && o > theta)) ? c + o : INF;
      w[b + 1] = x;
    }
  };
  int32_t c0 = INF, c1 = INF;
  {  // stage 1 = [0, b], b <= L - deg
    const int32_t* sP = sPall + slev[0] * L * L;
    if (b0 < L && b0 <= L - deg) c0 = mask(sP[b0]);
    if (b1 < L && b1 <= L - deg) c1 = mask(sP[b1]);
    if (deg > 1) {
      if (b0 < L) put_w(g, b0, c0);
      if (b1 < L) put_w(g, b1, c1);
    }
  }
  for (int i = 2; i <= deg; ++i) {
    __syncwarp();
    const int32_t* sP = sPall + slev[i - 1] * L * L;
    const int32_t* w = g + ((i & 1) ? 64 : 0);  // written by stage i-1
    int32_t* wn = g + ((i & 1) ? 0 : 64);
    const int blo = (i == deg) ? L - 1 : i - 1, bhi = L - 1 - (deg - i);
    uint32_t x0 = INF, y0 = INF, x1 = INF, y1 = INF;  // two accumulators per column
    const bool two = L > 32;
    int a = i - 1;
    for (; a + 1 <= bhi; a += 2) {
      const uint32_t wa = (uint32_t)w[a], wb = (uint32_t)w[a + 1];
      const uint32_t pa0 = (uint32_t)mask(sP[a * L + b0]), pb0 = (uint32_t)mask(sP[(a + 1) * L + b0]);
      if (BOTTLENECK) {
        x0 = min(x0, max(wa, pa0));
        y0 = min(y0, max(wb, pb0));
      } else {
        x0 = __viaddmin_u32(wa, pa0, x0);
        y0 = __viaddmin_u32(wb, pb0, y0);
      }
      if (two) {
        const uint32_t pa1 = (uint32_t)mask(sP[a * L + b1]), pb1 = (uint32_t)mask(sP[(a + 1) * L + b1]);
        if (BOTTLENECK) {
          x1 = min(x1, max(wa, pa1));
          y1 = min(y1, max(wb, pb1));
        } else {
          x1 = __viaddmin_u32(wa, pa1, x1);
          y1 = __viaddmin_u32(wb, pb1, y1);
        }
      }
    }
    if (a <= bhi) {
      const uint32_t wa = (uint32_t)w[a];
      const uint32_t pa0 = (uint32_t)mask(sP[a * L + b0]);
      x0 = BOTTLENECK ? min(x0, max(wa, pa0)) : __viaddmin_u32(wa, pa0, x0);
      if (two) {
        const uint32_t pa1 = (uint32_t)mask(sP[a * L + b1]);
        x1 = BOTTLENECK ? min(x1, max(wa, pa1)) : __viaddmin_u32(wa, pa1, x1);
      }
    }
    c0 = (b0 >= blo && b0 <= bhi) ? (int32_t)min(min(x0, y0), (uint32_t)INF) : INF;
    c1 = (b1 < L && b1 >= blo && b1 <= bhi) ? (int32_t)min(min(x1, y1), (uint32_t)INF) : INF;
    if (i < deg) {
      if (b0 < L) put_w(wn, b0, c0);
      if (b1 < L) put_w(wn, b1, c1);
    }
  }
  const int32_t F = __shfl_sync(0xffffffffu, (L - 1) < 32 ? c0 : c1, (L - 1) & 31);
  __syncwarp();
  return F;
}
__device__ __forceinline__ int32_t warp_F(const int32_t* sP, const int32_t* slev, const int32_t* sO, int32_t* g, int L,
                                          int deg, int32_t theta) {
  return theta >= INF ? warp_dp<false, false>(sP, slev, sO, g, L, deg, INF)
                      : warp_dp<false, true>(sP, slev, sO, g, L, deg, theta);
}

// ---------------------------------------------------------------------------
// K4: Val(theta) of one config per CTA (32 warps), and the config's optimum.
//  1. F_inf = F at the largest theta (no limit).  c = 1: OPT = F_inf.
//  2. theta_min, the smallest theta with a feasible placement (F is finite
//     exactly for theta >= theta_min): one bottleneck (min, max) DP.
//  3. U = Val(theta_min) bounds OPT, so only theta <= (U - F_inf)/(c-1)
//     can reach it (Val(theta) >= F_inf + (c-1) theta); those are evaluated
//     in ascending order by the 32 warps, skipping theta once
//     F_inf + (c-1) theta > best-so-far (strict: ties stay for the tie-break).
// Unevaluated entries keep Val = INT64_MAX (> OPT, so never in Theta*).
// ---------------------------------------------------------------------------
constexpr int K4W = 32;
struct K4Smem {
  int32_t v[SORTN];  // sorted distinct thetas (K3)
  int32_t sP[MAXLEV * MAXL * MAXL];  // the config's interval tables, one per cap level
  int32_t slev[MAXL];                // cap level of each stage
  int32_t sO[MAXL];
  int32_t g[K4W][128];
  int32_t probeF[K4W];
  int32_t cnt, s_hi;
  unsigned long long s_best;
  typename K3Scan::TempStorage scan_tmp;
};

__global__ void __launch_bounds__(K4W * 32) k4_vals(const CfgDev* __restrict__ cfgs, const int32_t* __restrict__ arena,
                                                   const int32_t* __restrict__ P, const int32_t* __restrict__ cfg_list,
                                                   int li0, int L, int32_t* __restrict__ thetas,
                                                   int32_t* __restrict__ ntheta, int64_t* __restrict__ vals,
                                                   int64_t* __restrict__ cfg_opt) {
  TraceScope tr(TR_K4 | (uint32_t)li0 << 8);
  extern __shared__ __align__(16) unsigned char k4raw[];
  K4Smem& S = *reinterpret_cast<K4Smem*>(k4raw);
  int32_t* sP = S.sP;
  int32_t* sO = S.sO;
  int32_t* probeF = S.probeF;
  int& s_hi = S.s_hi;
  unsigned long long& s_best = S.s_best;
  auto g = S.g;
  const int li = li0 + blockIdx.x;
  const CfgDev cf = cfgs[cfg_list[li]];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // K3 fused: the sorted distinct theta candidates (also kept for K5a)
  for (int i = threadIdx.x; i < MAXL; i += blockDim.x)  // (from global: no local copy of cf; visible after
    S.slev[i] = cfgs[cfg_list[li]].lev_of[i];           //  sort_thetas' first barrier)
  const int nt = sort_thetas(cf, arena, P, L, S.v, sP, sO, S.scan_tmp);
  const int32_t* slev = S.slev;
  for (int i = threadIdx.x; i < nt; i += blockDim.x) thetas[(int64_t)li * TMAX + i] = S.v[i];
  if (threadIdx.x == 0) ntheta[li] = nt;
  int64_t* V = vals + (int64_t)li * (TMAX + 2);  // [0..nt) Val, [TMAX] F_inf, [TMAX+1] opt
  const int32_t* th = S.v;
  for (int i = threadIdx.x; i < nt; i += blockDim.x) V[i] = INT64_MAX;
  if (cf.deg > L || nt == 0) {  // Eq. 7b cannot hold (reading A-22)
    if (threadIdx.x == 0) { V[TMAX] = INT64_MAX; cfg_opt[cfg_list[li]] = INT64_MAX; }
    return;
  }
  const int64_t cm1 = cf.c - 1;
  if (nt <= K4W && cf.c > 1) {
    // few candidates: every F_theta in one round, one warp each (the
    // largest theta bounds every P and O, so F of it is F_inf)
    if (w < nt) {
      const int32_t F = warp_F(sP, slev, sO, g[w], L, cf.deg, w == nt - 1 ? INF : S.v[w]);
      if (lane == 0) probeF[w] = F;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      const int32_t Finf = probeF[nt - 1];
      int64_t best = INT64_MAX;
      for (int i = 0; i < nt; ++i)
        if (Finf < INF && probeF[i] < INF) {
          const int64_t val = (int64_t)probeF[i] + cm1 * S.v[i];
          V[i] = val;
          best = min(best, val);
        }
      V[TMAX] = Finf >= INF ? INT64_MAX : (int64_t)Finf;
      cfg_opt[cfg_list[li]] = Finf >= INF ? INT64_MAX : best;
      tr.extra = (uint32_t)nt | (uint32_t)nt << 12;
    }
    return;
  }
  // 1. F_inf (warp 0) and the bottleneck theta_min (warp 1)
  if (w == 0) {
    const int32_t F = warp_F(sP, slev, sO, g[0], L, cf.deg, INF);
    if (lane == 0) probeF[0] = F;
  } else if (w == 1) {
    const int32_t Bm = warp_dp<true, false>(sP, slev, sO, g[1], L, cf.deg, INF);
    if (lane == 0) probeF[1] = Bm;
  }
  __syncthreads();
  const int32_t Finf = probeF[0];
  if (Finf >= INF || cf.c == 1) {
    if (threadIdx.x == 0) {
      V[TMAX] = Finf >= INF ? INT64_MAX : (int64_t)Finf;
      cfg_opt[cfg_list[li]] = V[TMAX];
    }
    return;
  }
  // 2. the index of theta_min in the sorted candidates (it is one of them)
  if (threadIdx.x == 0) {
    const int32_t tm = probeF[1];
    int lo = 0, hi = nt - 1;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (th[mid] < tm) lo = mid + 1;
      else hi = mid;
    }
    s_hi = lo;
  }
  __syncthreads();
  const int imin = s_hi;
  // 3. U = Val(theta_min); evaluate theta_min .. theta_hi
  if (w == 0) {
    const int32_t F = warp_F(sP, slev, sO, g[0], L, cf.deg, th[imin]);
    if (lane == 0) {
      const int64_t U = (int64_t)F + cm1 * th[imin];
      V[imin] = U;
      s_best = (unsigned long long)U;
    }
  }
  __syncthreads();
  const int64_t U = (int64_t)s_best;
  if (threadIdx.x == 0) S.cnt = 0;
  __syncthreads();
  for (int i = imin + 1 + w; i < nt; i += K4W) {
    const int32_t theta = th[i];
    const int64_t lb = (int64_t)Finf + cm1 * theta;
    if (lb > U) break;  // ascending thetas: every later one is worse too
    if ((unsigned long long)lb > *(volatile unsigned long long*)&s_best) continue;
    const int32_t F = warp_F(sP, slev, sO, g[w], L, cf.deg, theta);
    if (g_trace && lane == 0) atomicAdd(&S.cnt, 1);  // diagnostics: thetas evaluated
    if (F < INF && lane == 0) {
      const int64_t val = (int64_t)F + cm1 * theta;
      V[i] = val;
      atomicMin(&s_best, (unsigned long long)val);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    V[TMAX] = Finf;
    cfg_opt[cfg_list[li]] = (int64_t)s_best;
    tr.extra = (uint32_t)S.cnt | (uint32_t)nt << 12 | (uint32_t)(nt - imin) << 24;
  }
}

cudaError_t launch_k4(const CfgDev* cfg, const int32_t* arena, const int32_t* P, const int32_t* cfg_list, int li0,
                      int n_local, int L, int32_t* thetas, int32_t* ntheta, int64_t* vals, int64_t* cfg_opt,
                      cudaStream_t st) {
  if (n_local <= 0) return cudaSuccess;
  k4_vals<<<n_local, K4W * 32, sizeof(K4Smem), st>>>(cfg, arena, P, cfg_list, li0, L, thetas, ntheta, vals, cfg_opt);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// K5a: per-config optimum, global (objective, deg, c) argmin, and the
// lexicographically largest stage-end vector over the optimal placements
// (= lexicographically smallest stage_of, reading A-11).  One CTA.
// ---------------------------------------------------------------------------
constexpr int K5T = 1024;
constexpr int K5PP = MAXL + 1;  // odd pitch of K5a's interval tables
// K5a's dynamic shared memory: the suffix table H, then the winner's interval
// tables (one per cap level)
constexpr int K5A_DYN = (MAXL + 1) * (MAXL + 1) * 4 + MAXLEV * MAXL * K5PP * 4;
__global__ void __launch_bounds__(K5T) k5a_winner(const CfgDev* __restrict__ cfgs, const int32_t* __restrict__ arena,
                                                  const int32_t* __restrict__ P, const int32_t* __restrict__ cfg_list,
                                                  int n_local, int L, const int32_t* __restrict__ thetas,
                                                  const int32_t* __restrict__ ntheta, const int64_t* __restrict__ vals,
                                                  const int64_t* __restrict__ cfg_opt, int32_t* __restrict__ scratch,
                                                  Winner* __restrict__ win, RecordArgs ra) {
  TraceScope tr(TR_K5A);
  __shared__ int32_t sO[MAXL];
  __shared__ int32_t stars[TMAX];
  __shared__ int32_t nstar;
  __shared__ int32_t ends[32][MAXL];
  __shared__ int32_t okw[32];
  __shared__ int64_t s_opt[1];
  __shared__ int32_t s_win;
  const int t = threadIdx.x, w = t >> 5, lane = t & 31;
  // 2. winner by (objective, deg, c): warp 0, lanes over the local configs,
  //    then a shuffle argmin on the key tuple
  if (w == 0) {
    int wi = -1, bd = 0, bc = 0;
    int64_t best = INT64_MAX;
    for (int li = lane; li < n_local; li += 32) {
      const int ci = cfg_list[li];
      const int64_t v = cfg_opt[ci];
      const int dg = cfgs[ci].deg, cc = cfgs[ci].c;
      if (v != INT64_MAX && (wi < 0 || v < best || (v == best && (dg < bd || (dg == bd && cc < bc))))) {
        wi = li; best = v; bd = dg; bc = cc;
      }
    }
    for (int off = 16; off > 0; off >>= 1) {
      const int owi = __shfl_down_sync(0xffffffffu, wi, off), obd = __shfl_down_sync(0xffffffffu, bd, off),
                obc = __shfl_down_sync(0xffffffffu, bc, off);
      const int64_t ob = __shfl_down_sync(0xffffffffu, best, off);
      if (owi >= 0 && (wi < 0 || ob < best || (ob == best && (obd < bd || (obd == bd && obc < bc))))) {
        wi = owi; best = ob; bd = obd; bc = obc;
      }
    }
    if (lane == 0) {
      s_win = wi;
      s_opt[0] = best;
      nstar = 0;
    }
  }
  __syncthreads();
  const int wl = s_win;
  // the record header: every field K5c does not write (assignment arrays zeroed)
  if (t < UNIAP_MAX_LAYERS) {
    uniap_record* r = ra.rec;
    r->stage_of[t] = 0;
    r->strategy_of[t] = 0;
    r->stage_cost[t] = 0;
    r->cut_cost[t] = 0;
    r->stage_mem[t] = 0;
  }
  if (t < MAXCLS) ra.bw->count[t] = 0;
  if (t == 0) {
    uniap_record* r = ra.rec;
    r->objective = INT64_MAX;
    r->cfg_index = -1;
    r->deg = r->c = 0;
    r->L = ra.L;
    r->status = (ra.qglob && ra.qglob[1] != 0) ? UNIAP_ERR_RANGE : 0;
    r->n_cfg_local = ra.n_local;
    r->dp_cells = ra.cells;
    r->dp_relax = ra.relax;
    if (ra.work) {  // level 2: the counts K1f made where it trimmed the sweeps
      unsigned long long c = 0, x = 0;
      for (int li = 0; li < ra.n_local; ++li) {
        c += ra.work[2 * cfg_list[li]];
        x += ra.work[2 * cfg_list[li] + 1];
      }
      r->dp_cells = c;
      r->dp_relax = x;
    }
    r->dp_cells_canonical = ra.cells_canon;
  }
  if (wl < 0) {
    if (t == 0) { win->objective = INT64_MAX; win->cfg = -1; win->status = 0; }
    return;
  }
  const int ci = cfg_list[wl];
  if (cfgs[ci].cut) {
    // NEXT-1 winner: K4c found its stage ends and boundary strategies; the
    // traceback sweeps start at each stage's last layer restricted to its
    // last strategy, and K5c starts each walk on the stage's first strategy
    if (t == 0) {
      const CfgDev* cp = cfgs + ci;
      const CutRes& X = ra.cutres[wl];
      const int deg = cp->deg;
      const bool have = X.status == 1;
      win->objective = s_opt[0];
      win->cfg = ci;
      win->deg = deg;
      win->c = cp->c;
      win->S = cp->S;
      win->NSP = cp->NSP;
      win->n_theta_star = 0;
      win->status = have ? 0 : 99;
      uniap_record* r = ra.rec;
      if (!have) r->status = X.status == UNIAP_ERR_RANGE ? UNIAP_ERR_RANGE : UNIAP_ERR_INTERNAL;
      r->objective = s_opt[0];
      r->cfg_index = ci;
      r->deg = deg;
      r->c = cp->c;
      int n = 0, a = 0;
      int64_t goff = 0;
      for (int i = 0; i < deg && have; ++i) {
        const int b = X.ends[i], len = b - a + 1;
        win->end[i] = b;
        win->p[i] = X.p[i];
        win->o[i] = X.o[i];
        win->kfirst[i] = X.kfirst[i];
        win->klast[i] = X.klast[i];
        const bool cond = cp->skip >= 0 && a <= cp->skip && cp->skip + 2 <= b;
        for (int ks = cond ? 0 : -1; ks < (cond ? cp->S : 0); ++ks) {
          ra.bw->gofs[i * 33 + ks + 1] = goff;
          ra.bw_inst[n++] = Inst{ci, b, len, ks, -1, 0, goff, 0, -1, len, 0, 0, X.klast[i]};
          goff += (int64_t)len * cp->NSP * (ra.cap + 1);
        }
        a = b + 1;
      }
      ra.bw->count[ra.cls_of_cfg[ci]] = n;
    }
    return;
  }
  const CfgDev cf = cfgs[ci];
  const int64_t OPT = s_opt[0];
  const int64_t* V = vals + (int64_t)wl * (TMAX + 2);
  const int32_t* th = thetas + (int64_t)wl * TMAX;
  const int nt = ntheta[wl];
  // the winner's interval tables P_lev[a][b] at lev * L * PP + a * PP + b
  // (odd pitch: lanes over a or b conflict-free), in dynamic shared memory
  // after the suffix table sH
  extern __shared__ int32_t k5dyn[];
  int32_t* sPl = k5dyn + (MAXL + 1) * (MAXL + 1);
  const int PP = L | 1;
  for (int i = t; i < cf.nlev * L * L; i += K5T) {
    const int lv = i / (L * L), r = i - lv * L * L;
    sPl[lv * L * PP + (r / L) * PP + r % L] = P[cf.offP + i];
  }
  // stage i (1-based) reads the table of its cap level
  const int8_t* lev_of = cfgs[ci].lev_of;  // (global: no local copy of cf)
  auto SPs = [&](int i) { return sPl + lev_of[i - 1] * L * PP; };
  for (int i = t; i < L - 1; i += K5T) sO[i] = arena[cf.offO + i];
  // 3. Theta*: every theta with Val = OPT (c > 1); the unconstrained one (c = 1)
  if (cf.c == 1) {
    if (t == 0) { stars[0] = -1; nstar = 1; }
  } else {
    for (int i = t; i < nt; i += K5T)
      if (V[i] == OPT) stars[atomicAdd(&nstar, 1)] = i;
  }
  __syncthreads();
  const int ns = nstar;
  const int deg = cf.deg;
  // 4. per theta in Theta*: suffix DP H_i[a] (cover [a, L-1] with stages i..deg)
  //    then the greedy largest end per stage.
  int32_t* H = scratch + (int64_t)w * (MAXL + 1) * (MAXL + 1);  // [i][a], i = 1..deg, a = 0..L
  int32_t* mine = ends[w];
  int32_t best_end[MAXL];
  bool have = false;
  // Few theta* (the usual case: one): the whole CTA per theta, H in shared
  // memory -- stages sequential (one barrier each), warps over the start a,
  // lanes over the end b with a warp min.  Many: one warp per theta below.
  constexpr int HP = MAXL + 1;
  int32_t* sH = k5dyn;  // [i][a], i = 1..deg, a = 0..L
  for (int si = 0; si < ns && ns <= 4; ++si) {
    const int32_t theta = stars[si] < 0 ? INF : th[stars[si]];
    const int64_t F_target = stars[si] < 0 ? OPT : OPT - (int64_t)(cf.c - 1) * theta;
    for (int a = t; a <= L; a += K5T) {
      int32_t v = INF;
      if (a < L) { const int32_t p = SPs(deg)[a * PP + L - 1]; v = p <= theta ? p : INF; }
      sH[deg * HP + a] = v;
    }
    __syncthreads();
    for (int i = deg - 1; i >= 1; --i) {
      // H_i[a] = min_b P_i[a][b] + O[b] + H_{i+1}[b+1], b <= L-1-(deg-i)
      const int bhi = L - 1 - (deg - i);
      const int32_t* sP = SPs(i);
      for (int a = w; a <= L; a += K5T / 32) {
        uint32_t v = INF;
        for (int b = a + lane; b <= bhi && a < L; b += 32) {
          const int32_t p = sP[a * PP + b], o = sO[b], hh = sH[(i + 1) * HP + b + 1];
          if (p <= theta && o <= theta && hh < INF) v = min(v, (uint32_t)p + (uint32_t)o + (uint32_t)hh);
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, off));
        if (lane == 0) sH[i * HP + a] = (int32_t)min(v, (uint32_t)INF);
      }
      __syncthreads();
    }
    bool ok = (int64_t)sH[1 * HP + 0] == F_target;
    if (w == 0) {  // greedy: the largest feasible end of each stage
      int64_t pre = 0;
      int a = 0;
      for (int i = 1; i < deg && ok; ++i) {
        const int32_t* sP = SPs(i);
        int found = -1;
        for (int b0 = L - 1 - (deg - i); b0 >= a && found < 0; b0 -= 32) {
          const int b = b0 - lane;
          bool c = false;
          if (b >= a) {
            const int32_t p = sP[a * PP + b], o = sO[b], hh = sH[(i + 1) * HP + b + 1];
            c = p <= theta && o <= theta && hh < INF && pre + p + o + hh == F_target;
          }
          const unsigned m = __ballot_sync(0xffffffffu, c);
          if (m) found = b0 - (__ffs(m) - 1);
        }
        if (found < 0) { ok = false; break; }
        if (lane == 0) ends[0][i - 1] = found;
        pre += sP[a * PP + found] + sO[found];
        a = found + 1;
      }
      if (lane == 0) {
        ends[0][deg - 1] = L - 1;
        okw[0] = ok;
      }
    }
    __syncthreads();
    if (t == 0 && okw[0]) {  // lexicographically largest end vector over theta*
      bool better = !have;
      for (int i = 0; i < deg && !better; ++i) {
        if (ends[0][i] != best_end[i]) { better = ends[0][i] > best_end[i]; break; }
      }
      if (better) {
        for (int i = 0; i < deg; ++i) best_end[i] = ends[0][i];
        have = true;
      }
    }
    __syncthreads();
  }
  for (int base = 0; base < ns && ns > 4; base += 32) {
    const int si = base + w;
    bool ok = false;
    if (si < ns) {
      const int32_t theta = stars[si] < 0 ? INF : th[stars[si]];
      const int64_t F_target = stars[si] < 0 ? OPT : OPT - (int64_t)(cf.c - 1) * theta;
      // H_deg[a] = P[a][L-1]
      for (int a = lane; a <= L; a += 32) {
        int32_t v = INF;
        if (a < L) { const int32_t p = SPs(deg)[a * PP + L - 1]; v = p <= theta ? p : INF; }
        H[deg * (MAXL + 1) + a] = v;
      }
      __syncwarp();
      for (int i = deg - 1; i >= 1; --i) {
        // H_i[a] = min_b P[a][b] + (O[b] + H_{i+1}[b+1]); the bracket is
        // lane-independent (broadcast), P[a][b] read transposed
        const int bhi = L - 1 - (deg - i);
        const int32_t* Hn = H + (i + 1) * (MAXL + 1);
        const int32_t* sP = SPs(i);
        for (int a = lane; a <= L; a += 32) {
          uint32_t x = INF, y = INF;
          if (a < L) {
            int b = a;
            for (; b + 1 <= bhi; b += 2) {
              const int32_t p0 = sP[a * PP + b], p1 = sP[a * PP + b + 1];
              const int32_t o0 = sO[b], o1 = sO[b + 1], h0 = Hn[b + 1], h1 = Hn[b + 2];
              const uint32_t w0 = (o0 <= theta && h0 < INF) ? (uint32_t)(o0 + h0) : INF;
              const uint32_t w1 = (o1 <= theta && h1 < INF) ? (uint32_t)(o1 + h1) : INF;
              x = __viaddmin_u32(w0, p0 <= theta ? (uint32_t)p0 : INF, x);
              y = __viaddmin_u32(w1, p1 <= theta ? (uint32_t)p1 : INF, y);
            }
            if (b <= bhi) {
              const int32_t p0 = sP[a * PP + b], o0 = sO[b], h0 = Hn[b + 1];
              const uint32_t w0 = (o0 <= theta && h0 < INF) ? (uint32_t)(o0 + h0) : INF;
              x = __viaddmin_u32(w0, p0 <= theta ? (uint32_t)p0 : INF, x);
            }
          }
          H[i * (MAXL + 1) + a] = (int32_t)min(min(x, y), (uint32_t)INF);
        }
        __syncwarp();
      }
      ok = (int64_t)H[1 * (MAXL + 1) + 0] == F_target;
      // greedy: the largest feasible end of each stage
      int64_t pre = 0;
      int a = 0;
      for (int i = 1; i < deg && ok; ++i) {
        const int32_t* sP = SPs(i);
        int found = -1;
        for (int b0 = L - 1 - (deg - i); b0 >= a && found < 0; b0 -= 32) {
          const int b = b0 - lane;
          bool c = false;
          if (b >= a) {
            const int32_t p = sP[a * PP + b], o = sO[b], h = H[(i + 1) * (MAXL + 1) + b + 1];
            c = p <= theta && o <= theta && h < INF && pre + p + o + h == F_target;
          }
          const unsigned m = __ballot_sync(0xffffffffu, c);
          if (m) found = b0 - (__ffs(m) - 1);
        }
        if (found < 0) { ok = false; break; }
        if (lane == 0) mine[i - 1] = found;
        pre += sP[a * PP + found] + sO[found];
        a = found + 1;
      }
      if (lane == 0) mine[deg - 1] = L - 1;
      __syncwarp();
    }
    if (lane == 0) okw[w] = ok;
    __syncthreads();
    // lexicographically largest end vector (theta order is deterministic)
    if (t == 0) {
      for (int j = 0; j < 32 && base + j < ns; ++j) {
        if (!okw[j]) continue;
        bool better = !have;
        for (int i = 0; i < deg && !better; ++i) {
          if (ends[j][i] != best_end[i]) { better = ends[j][i] > best_end[i]; break; }
        }
        if (better) {
          for (int i = 0; i < deg; ++i) best_end[i] = ends[j][i];
          have = true;
        }
      }
    }
    __syncthreads();
  }
  if (t == 0) {
    for (int i = 0; i < MAXL; ++i) win->kfirst[i] = win->klast[i] = -1;
    win->objective = OPT;
    win->cfg = ci;
    win->deg = deg;
    win->c = cf.c;
    win->S = cf.S;
    win->NSP = cf.NSP;
    win->n_theta_star = ns;
    win->status = have ? 0 : 99;
    int a = 0;
    for (int i = 0; i < deg; ++i) {
      const int b = have ? best_end[i] : L - 1;
      win->end[i] = b;
      win->p[i] = SPs(i + 1)[a * PP + b];
      win->o[i] = (i + 1 < deg) ? sO[b] : 0;
      a = b + 1;
    }
    uniap_record* r = ra.rec;
    if (!have) r->status = UNIAP_ERR_INTERNAL;
    r->objective = OPT;
    r->cfg_index = ci;
    r->deg = deg;
    r->c = cf.c;
    // the backward sweeps of the traceback: one per stage, one per skip
    // conditioning ks when the stage contains the skip source and an edge of it
    int n = 0;
    int64_t goff = 0;
    a = 0;
    for (int i = 0; i < deg && have && r->status == 0; ++i) {
      const int b = best_end[i], len = b - a + 1;
      const bool cond = cf.skip >= 0 && a <= cf.skip && cf.skip + 2 <= b;
      const int64_t kept = ra.gstore[ci];  // deg = 1: the forward phase's sweep kept its tables
      for (int ks = cond ? 0 : -1; ks < (cond ? cf.S : 0); ++ks) {
        if (kept >= 0) {
          ra.bw->gofs[i * 33 + ks + 1] = kept + (int64_t)(ks < 0 ? 0 : ks) * L * cf.NSP * (ra.cap + 1);
          continue;
        }
        ra.bw->gofs[i * 33 + ks + 1] = goff;
        ra.bw_inst[n++] = Inst{ci, b, len, ks, -1, 0, goff, 0, -1, len};
        goff += (int64_t)len * cf.NSP * (ra.cap + 1);
      }
      a = b + 1;
    }
    ra.bw->count[ra.cls_of_cfg[ci]] = n;
  }
}

cudaError_t launch_k5a(const CfgDev* cfg, const int32_t* arena, const int32_t* P, const int32_t* cfg_list, int n_local,
                       int L, const int32_t* thetas, const int32_t* ntheta, const int64_t* vals, const int64_t* cfg_opt,
                       int32_t* scratch, Winner* win, const RecordArgs& ra, cudaStream_t st) {
  k5a_winner<<<1, K5T, K5A_DYN, st>>>(cfg, arena, P, cfg_list, n_local, L, thetas, ntheta, vals, cfg_opt, scratch,
                                      win, ra);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// K5c: per stage, the lexicographically smallest strategy vector reaching the
// stage optimum, walking the backward tables G (K2 backward sweeps):
// at layer u take the smallest k with  R[u-1][k_{u-1}][k] + G[u][k][q] = rest.
// One CTA per stage; warp w walks the conditioning ks = w (or none).
// Also writes the record (objective, placement, costs, memory).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) k5c_walk(const CfgDev* __restrict__ cfgs, const int32_t* __restrict__ arena,
                                                 const int32_t* __restrict__ G, const BwPlan* __restrict__ bw,
                                                 const Winner* __restrict__ win, int L, int cap,
                                                 uniap_record* __restrict__ rec) {
  pdl_wait();  // the backward sweeps' tables (PDL when one launch precedes on the stream)
  TraceScope tr(TR_K5C);
  __shared__ int32_t vec[32][MAXL];
  __shared__ int32_t mem[32];
  __shared__ int32_t okw[32];
  const int stage = blockIdx.x;
  const Winner& W = *win;  // by reference: fields are read on demand, no per-thread copy
  if (W.cfg < 0 || W.objective == INT64_MAX || W.status != 0 || stage >= W.deg || rec->status != 0) return;
  const CfgDev cf = cfgs[W.cfg];
  int skip;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int a = stage == 0 ? 0 : W.end[stage - 1] + 1, b = W.end[stage];
  skip = cf.skip;
  const bool cond = skip >= 0 && a <= skip && skip + 2 <= b;
  const int nks = cond ? cf.S : 1;
  const int NSP = cf.NSP, Q = cap + 1, S = cf.S;
  const int32_t* A = arena + cf.offA;
  const int32_t* M = arena + cf.offM;
  const int32_t* Rf = arena + cf.offRf;
  const int32_t* Rs = arena + cf.offRs;
  bool ok = false;
  if (w < nks) {
    const int ks = cond ? w : -1;
    const int32_t* g = G + bw->gofs[stage * 33 + (ks + 1)];
    int64_t rest = W.p[stage];
    int q = cfgs[W.cfg].lcap[cfgs[W.cfg].lev_of[stage]], kprev = -1;  // the stage's own memory cap (NEXT-2)
    const int kf0 = W.kfirst[stage];
    int32_t msum = 0;
    ok = true;
    for (int u = a; u <= b && ok; ++u) {
      const int k = lane;
      bool c = false;
      int32_t edge = 0, ap = 0, mk = 0;
      if (k < S && (u != a || kf0 < 0 || k == kf0)) {  // (NEXT-1: the stage's first strategy forced)
        mk = M[u * NSP + k];  // per lane, with the other loads: one global round trip per layer
        const int32_t gv = g[((int64_t)(u - a) * NSP + k) * Q + q];
        edge = (u > a) ? Rf[((int64_t)(u - 1) * NSP + kprev) * NSP + k] : 0;
        ap = A[u * NSP + k] + ((ks >= 0 && u >= skip + 2) ? Rs[((int64_t)u * NSP + ks) * NSP + k] : 0);
        c = gv < INF && (int64_t)edge + gv == rest;
      }
      const unsigned m = __ballot_sync(0xffffffffu, c);
      if (!m) { ok = false; break; }
      const int kk = __ffs(m) - 1;
      const int32_t e2 = __shfl_sync(0xffffffffu, edge, kk);
      const int32_t a2 = __shfl_sync(0xffffffffu, ap, kk);
      const int32_t m2 = __shfl_sync(0xffffffffu, mk, kk);
      rest -= (int64_t)e2 + a2;
      q -= m2;
      msum += m2;
      kprev = kk;
      if (lane == 0) vec[w][u] = kk;
    }
    if (lane == 0) mem[w] = msum;
  }
  if (lane == 0) okw[w] = ok;
  __syncthreads();
  if (threadIdx.x == 0) {
    int bw = -1;
    for (int j = 0; j < nks; ++j) {
      if (!okw[j]) continue;
      bool better = bw < 0;
      for (int u = a; u <= b && !better; ++u)
        if (vec[j][u] != vec[bw][u]) { better = vec[j][u] < vec[bw][u]; break; }
      if (better) bw = j;
    }
    if (bw < 0) {
      rec->status = UNIAP_ERR_INTERNAL;
    } else {
      for (int u = a; u <= b; ++u) {
        rec->strategy_of[u] = cfgs[W.cfg].orig[vec[bw][u]];  // caller's strategy index
        rec->stage_of[u] = stage;
      }
      rec->stage_mem[stage] = mem[bw];
      rec->stage_cost[stage] = W.p[stage];
      rec->cut_cost[stage] = W.o[stage];
    }
  }
}

cudaError_t launch_k5c_grid(int max_deg, const CfgDev* cfg, const int32_t* arena, const int32_t* G,
                            const BwPlan* bw, const Winner* win, int L, int cap, uniap_record* rec,
                            cudaStream_t st) {
  if (max_deg <= 0) return cudaSuccess;
  cudaError_t e = pdl_launch(k5c_walk, dim3(max_deg), dim3(1024), 0, st, cfg, arena, G, bw, win, L, cap, rec);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t combine_trace(unsigned long long* p) { return cudaMemcpyToSymbol(g_trace, &p, sizeof p); }

// Kernel attributes of this translation unit on the CURRENT device (function
// attributes are per device; uniap_create calls this once per device).
// Every kernel of the step prefers the maximum shared-memory carveout, as K2
// needs it: no L1/shared reconfiguration between the kernels of the step.
cudaError_t combine_init() {
  for (const void* f : {(const void*)k_fill, (const void*)k4_vals, (const void*)k5a_winner, (const void*)k5c_walk}) {
    cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
  }
  cudaError_t e = cudaFuncSetAttribute((const void*)k4_vals, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(K4Smem));
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute((const void*)k5a_winner, cudaFuncAttributeMaxDynamicSharedMemorySize, K5A_DYN);
}

}  // namespace uniap
