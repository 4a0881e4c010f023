// cutcombine.cu -- K4c, NEXT-1: the stage combine (Eq. 2) when the
// cross-stage cost depends on the strategies at the cut (Eq. 4 with R' per
// strategy pair): o_j = O[e_j] + Rcut[e_j][k_{e_j}][k_{e_j+1}].
//
// K2's tmode launches leave, per config, T[a][b][kf][kl] = the minimum of
// Eq. (3) over [a,b] under Eq. (5) with layer a on kf and layer b on kl
// (index NSP = that end free).  K4c, one CTA per such config:
//   F_theta = min over placements and boundary strategies of sum p + sum o
//             with every p, o <= theta: a DP over (stage, end b, strategy at
//             the end); Val(theta) = F_theta + (c-1) theta; OPT = min over
//             theta in the distinct p / o values (the argument of
//             combine.cu); c = 1: OPT = F_inf.
//   Then per theta in Theta* (Val = OPT) the tie-break of reading A-31: the
//   largest feasible end of each stage in turn (lexicographically smallest
//   stage_of), then the boundary strategies (k_{e_1}, k_{e_1+1}, k_{e_2},
//   ...) smallest first.  With theta fixed, the optimal solutions are exactly
//   the min-sum ones under the masks, so prefix and suffix minima decide
//   every existence test.  The lexicographic best over Theta* goes to K5a.
#include "uniap_impl.h"

namespace uniap {

constexpr int KCT = 1024;
constexpr int KC_SORT = 4096;  // distinct theta candidates above theta_min (more: UNIAP_ERR_RANGE)
constexpr int KW = UNIAP_MAX_STRAT + 1;

struct KcSmem {
  int32_t v[KC_SORT];        // theta candidates (hash set, then sorted)
  int64_t val[KC_SORT];      // Val(theta) of the evaluated candidates (INT64_MAX: not evaluated)
  int32_t W[MAXL * KW];      // per (end b, strategy at b)
  int32_t W2[MAXL * KW];
  int32_t U[MAXL * KW];      // per (end b, first strategy of the next stage)
  int32_t pre[KW], in[KW], he[KW], ze[KW];
  int32_t ends[MAXL], kfs[MAXL], kls[MAXL];
  int32_t bends[MAXL], bkfs[MAXL], bkls[MAXL];
  int32_t red[32];
  int32_t nv, flag, have, pick;
};

struct KcCtx {
  const int32_t* T;  // the config's T block
  const int32_t* O;
  const int32_t* Rc;
  int L, S, NSP, deg;
  __device__ int32_t t(int a, int b, int kf, int kl) const {  // kf / kl == NSP: that end free
    return T[(((int64_t)a * L + b) * (NSP + 1) + kf) * (NSP + 1) + kl];
  }
  __device__ int32_t o(int e, int kl, int kf) const { return O[e] + Rc[((int64_t)e * NSP + kl) * NSP + kf]; }
};

__device__ __forceinline__ int32_t msk(int32_t x, int32_t theta) { return x <= theta ? x : INF; }
__device__ __forceinline__ int32_t add2(int32_t a, int32_t b) { return (a >= INF || b >= INF) ? INF : min(a + b, INF); }

// CTA-wide reductions (every thread calls; uniform)
__device__ int32_t cta_min(int32_t x, int32_t* red) {
  for (int off = 16; off > 0; off >>= 1) x = min(x, __shfl_xor_sync(0xffffffffu, x, off));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = x;
  __syncthreads();
  int32_t y = INF;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) y = min(y, red[i]);
  __syncthreads();
  return y;
}
__device__ int32_t cta_max(int32_t x, int32_t* red) { return -cta_min(-x, red); }

// F_theta (MAXMODE: the bottleneck -- the smallest max term over placements,
// i.e. the smallest theta with a feasible placement).  Stage i (1-based)
// ends at b in [i-1, L-1-(deg-i)], the last stage at L-1.
template <bool MAXMODE>
__device__ int32_t kc_F(const KcCtx& X, KcSmem& S, int32_t theta) {
  const int L = X.L, Sn = X.S, deg = X.deg, NS1 = X.NSP + 1;
  auto comb = [&](int32_t a, int32_t b) { return MAXMODE ? max(a, b) : add2(a, b); };
  auto tv = [&](int a, int b, int kf, int kl) { return MAXMODE ? X.t(a, b, kf, kl) : msk(X.t(a, b, kf, kl), theta); };
  auto ov = [&](int e, int kl, int kf) { return MAXMODE ? X.o(e, kl, kf) : msk(X.o(e, kl, kf), theta); };
  for (int i = threadIdx.x; i < L * Sn; i += blockDim.x) {  // stage 1 = [0, b], first strategy free
    const int b = i / Sn, kl = i - b * Sn;
    S.W[b * NS1 + kl] = b <= L - deg ? tv(0, b, X.NSP, kl) : INF;
  }
  __syncthreads();
  int32_t F = INF;
  for (int st = 2; st <= deg; ++st) {
    const int blo = st - 2, bhi = L - 1 - (deg - st + 1);  // ends of stage st-1
    for (int i = threadIdx.x; i < L * Sn; i += blockDim.x) {  // into stage st at b+1 on kf
      const int b = i / Sn, kf = i - b * Sn;
      int32_t u = INF;
      if (b >= blo && b <= bhi)
        for (int kl = 0; kl < Sn; ++kl) {
          const int32_t w = S.W[b * NS1 + kl];
          if (w < INF) u = min(u, comb(w, ov(b, kl, kf)));
        }
      S.U[b * NS1 + kf] = u;
    }
    __syncthreads();
    const bool last = st == deg;
    const int clo = last ? L - 1 : st - 1, chi = L - 1 - (deg - st), nkl = last ? 1 : Sn;
    for (int i = threadIdx.x; i < L * nkl; i += blockDim.x) {
      const int b2 = i / nkl, kl2 = last ? X.NSP : i - b2 * nkl;
      int32_t wv = INF;
      if (b2 >= clo && b2 <= chi)
        for (int b = blo; b < b2 && b <= bhi; ++b)
          for (int kf = 0; kf < Sn; ++kf) {
            const int32_t u = S.U[b * NS1 + kf];
            if (u < INF) wv = min(wv, comb(u, tv(b + 1, b2, kf, kl2)));
          }
      S.W2[b2 * NS1 + (last ? 0 : kl2)] = wv;
    }
    __syncthreads();
    if (last) {
      F = S.W2[(L - 1) * NS1];
    } else {
      for (int i = threadIdx.x; i < L * NS1; i += blockDim.x) S.W[i] = S.W2[i];
    }
    __syncthreads();
  }
  return F;
}

// The tie-break search under one theta (masked): stage ends, then boundary
// strategies; false if none reaches F (a bug).  Z tables in global scratch:
// Z[i][b][kl] = min over stages i..deg covering [b+1, L-1] after a cut at b
// with strategy kl at b.
__device__ bool kc_trace(const KcCtx& X, KcSmem& S, int32_t theta, int32_t F, int32_t* Z) {
  const int L = X.L, Sn = X.S, deg = X.deg, NSP = X.NSP, NS1 = NSP + 1;
  auto tv = [&](int a, int b, int kf, int kl) { return msk(X.t(a, b, kf, kl), theta); };
  auto ov = [&](int e, int kl, int kf) { return msk(X.o(e, kl, kf), theta); };
  auto Zi = [&](int i, int b, int kl) -> int32_t& { return Z[((int64_t)i * L + b) * NS1 + kl]; };
  // suffix: H_i[a][kf] in S.U (rolling), Z_i from it
  for (int i = deg; i >= 2; --i) {
    for (int x = threadIdx.x; x < L * Sn; x += blockDim.x) {  // H_i[a][kf]
      const int a = x / Sn, kf = x - a * Sn;
      int32_t h = INF;
      if (a >= i - 1) {
        if (i == deg) h = tv(a, L - 1, kf, NSP);
        else
          for (int b = a; b <= L - 1 - (deg - i); ++b)
            for (int kl = 0; kl < Sn; ++kl) h = min(h, add2(tv(a, b, kf, kl), Zi(i + 1, b, kl)));
      }
      S.U[a * NS1 + kf] = h;
    }
    __syncthreads();
    for (int x = threadIdx.x; x < L * Sn; x += blockDim.x) {  // Z_i[b][kl]: a cut after b into stage i
      const int b = x / Sn, kl = x - b * Sn;
      int32_t z = INF;
      if (b + 1 < L)
        for (int kf = 0; kf < Sn; ++kf) z = min(z, add2(ov(b, kl, kf), S.U[(b + 1) * NS1 + kf]));
      Zi(i, b, kl) = z;
    }
    __syncthreads();
  }
  // ends: the largest feasible end of each stage in turn, prefix minima per
  // the strategy at the end
  int a = 0;
  for (int i = 1; i < deg; ++i) {
    if (i > 1)  // into stage i at a, first on kf: min_kp pre[kp] + o(a-1, kp, kf)
      for (int kf = threadIdx.x; kf < Sn; kf += blockDim.x) {
        int32_t x = INF;
        for (int kp = 0; kp < Sn; ++kp) x = min(x, add2(S.pre[kp], ov(a - 1, kp, kf)));
        S.in[kf] = x;
      }
    __syncthreads();
    const int bhi = L - 1 - (deg - i);
    int32_t best_b = -1;
    const int nk = i == 1 ? 1 : Sn;
    for (int x = threadIdx.x; x < (bhi - a + 1) * nk * Sn; x += blockDim.x) {
      const int b = a + x / (nk * Sn), r = x % (nk * Sn), kf = r / Sn, kl = r - kf * Sn;
      const int32_t p = i == 1 ? tv(0, b, NSP, kl) : add2(S.in[kf], tv(a, b, kf, kl));
      if (add2(p, Zi(i + 1, b, kl)) == F) best_b = max(best_b, b);
    }
    best_b = cta_max(best_b, S.red);
    if (best_b < 0) return false;
    S.ends[i - 1] = best_b;
    __syncthreads();
    for (int kl = threadIdx.x; kl < Sn; kl += blockDim.x) {  // prefix minima through stage i
      int32_t x = INF;
      if (i == 1) x = tv(0, best_b, NSP, kl);
      else
        for (int kf = 0; kf < Sn; ++kf) x = min(x, add2(S.in[kf], tv(a, best_b, kf, kl)));
      S.W2[kl] = x;
    }
    __syncthreads();
    for (int kl = threadIdx.x; kl < Sn; kl += blockDim.x) S.pre[kl] = S.W2[kl];
    __syncthreads();
    a = best_b + 1;
  }
  S.ends[deg - 1] = L - 1;
  __syncthreads();
  // boundary strategies with the ends fixed (small: one thread)
  if (threadIdx.x == 0) {
    int st[MAXL + 1];
    st[0] = 0;
    for (int i = 1; i < deg; ++i) st[i] = S.ends[i - 1] + 1;
    // suffix with fixed ends: he[kf] of stages i..deg, stage i first on kf
    // (rolling from the last stage); ZE[i][kl] kept in Z row 0 of stage i
    for (int kf = 0; kf < Sn; ++kf) S.he[kf] = tv(st[deg - 1], L - 1, kf, NSP);
    for (int i = deg - 1; i >= 1; --i) {
      const int e = S.ends[i - 1];
      for (int kl = 0; kl < Sn; ++kl) {  // ZE_{i+1}[kl] = min_kf o(e, kl, kf) + he[kf]
        int32_t z = INF;
        for (int kf = 0; kf < Sn; ++kf) z = min(z, add2(ov(e, kl, kf), S.he[kf]));
        Zi(i + 1, 0, kl) = z;  // (row b = 0 of Z_{i+1}: the fixed-end suffix, no longer needed as Z)
      }
      if (i > 1)
        for (int kf = 0; kf < Sn; ++kf) {
          int32_t h = INF;
          for (int kl = 0; kl < Sn; ++kl) h = min(h, add2(tv(st[i - 1], e, kf, kl), Zi(i + 1, 0, kl)));
          S.in[kf] = h;
        }
      for (int kf = 0; kf < Sn && i > 1; ++kf) S.he[kf] = S.in[kf];
    }
    // greedy: kl_1, kf_2, kl_2, kf_3, ... smallest first
    int32_t cur = 0;
    bool ok = true;
    for (int j = 1; j < deg && ok; ++j) {
      const int a0 = st[j - 1], e = S.ends[j - 1];
      const int kfj = j == 1 ? NSP : S.kfs[j - 1];
      int kl = -1;
      for (int k = 0; k < Sn && kl < 0; ++k)
        if (add2(add2(cur, tv(a0, e, kfj, k)), Zi(j + 1, 0, k)) == F) kl = k;
      if (kl < 0) { ok = false; break; }
      const int32_t pj = add2(cur, tv(a0, e, kfj, kl));
      // he of stage j+1 (first on kf) with the fixed ends: recompute forward-free
      int kf2 = -1;
      for (int k = 0; k < Sn && kf2 < 0; ++k) {
        // suffix from stage j+1 on k: T[st[j]][ends[j]][k][kl'] + ZE_{j+2}[kl'] (last stage: free end)
        int32_t h = INF;
        if (j + 1 == deg) h = tv(st[j], L - 1, k, NSP);
        else
          for (int k2 = 0; k2 < Sn; ++k2) h = min(h, add2(tv(st[j], S.ends[j], k, k2), Zi(j + 2, 0, k2)));
        if (add2(add2(pj, ov(e, kl, k)), h) == F) kf2 = k;
      }
      if (kf2 < 0) { ok = false; break; }
      S.kls[j - 1] = kl;
      S.kfs[j] = kf2;
      cur = add2(pj, ov(e, kl, kf2));
    }
    S.flag = ok;
  }
  __syncthreads();
  return S.flag != 0;
}

__global__ void __launch_bounds__(KCT) k4c_cut(const CfgDev* __restrict__ cfgs, const int32_t* __restrict__ arena,
                                               const int32_t* __restrict__ Tall, const int32_t* __restrict__ cfg_list,
                                               int li0, int L, int64_t* __restrict__ cfg_opt, CutRes* __restrict__ res,
                                               int32_t* __restrict__ zscratch, int64_t zstride) {
  extern __shared__ __align__(16) unsigned char kcraw[];
  KcSmem& S = *reinterpret_cast<KcSmem*>(kcraw);
  const int li = li0 + blockIdx.x, ci = cfg_list[li];
  const CfgDev* cf = cfgs + ci;
  KcCtx X{Tall + cf->offT, arena + cf->offO, arena + cf->offRc, L, cf->S, cf->NSP, cf->deg};
  CutRes* R = res + li;
  int32_t* Z = zscratch + (int64_t)li * zstride;
  const int c = cf->c;
  const int32_t Finf = kc_F<false>(X, S, INF);
  if (Finf >= INF) {
    if (threadIdx.x == 0) { cfg_opt[ci] = INT64_MAX; R->status = 0; }
    return;
  }
  int64_t OPT = Finf;
  int32_t tmin = INF;
  int nv = 0;
  if (c > 1) {
    tmin = kc_F<true>(X, S, INF);
    const int32_t Fmin = kc_F<false>(X, S, tmin);
    const int64_t Uv = (int64_t)Fmin + (int64_t)(c - 1) * tmin;
    const int64_t thi = (Uv - Finf) / (c - 1);  // Val(theta) >= F_inf + (c-1) theta
    // the distinct p / o values in (tmin, thi]: a hash set, then sorted
    for (int i = threadIdx.x; i < KC_SORT; i += blockDim.x) S.v[i] = 0x7fffffff;
    if (threadIdx.x == 0) S.flag = 0;
    __syncthreads();
    auto put = [&](int32_t x) {
      if (x <= tmin || (int64_t)x > thi) return;
      uint32_t hh = ((uint32_t)x * 2654435761u) >> 20;  // 4096 slots
      for (int probe = 0; probe < KC_SORT; ++probe) {
        const int32_t old = atomicCAS(&S.v[hh], 0x7fffffff, x);
        if (old == 0x7fffffff || old == x) return;
        hh = (hh + 1) & (KC_SORT - 1);
      }
      S.flag = 1;  // full
    };
    const int NS1 = X.NSP + 1;
    const int64_t nT = (int64_t)L * L * NS1 * NS1;
    for (int64_t i = threadIdx.x; i < nT; i += blockDim.x) {
      const int32_t x = X.T[i];
      if (x < INF) put(x);
    }
    for (int i = threadIdx.x; i < (L - 1) * X.S * X.S; i += blockDim.x) {
      const int e = i / (X.S * X.S), r = i % (X.S * X.S);
      put(X.o(e, r / X.S, r % X.S));
    }
    __syncthreads();
    if (S.flag) {  // more than KC_SORT candidates: not supported
      if (threadIdx.x == 0) { cfg_opt[ci] = INT64_MAX; R->status = UNIAP_ERR_RANGE; }
      return;
    }
    // compact + sort ascending (rank counting: values are distinct)
    if (threadIdx.x == 0) S.nv = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < KC_SORT; i += blockDim.x) {
      const int32_t x = S.v[i];
      if (x != 0x7fffffff) S.val[atomicAdd(&S.nv, 1)] = x;  // (val as scratch)
    }
    __syncthreads();
    nv = S.nv;
    for (int i = threadIdx.x; i < nv; i += blockDim.x) {
      const int32_t x = (int32_t)S.val[i];
      int rank = 0;
      for (int j = 0; j < nv; ++j) rank += (int32_t)S.val[j] < x;
      S.v[rank] = x;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nv; i += blockDim.x) S.val[i] = INT64_MAX;
    __syncthreads();
    // ascending thetas above theta_min, pruned once F_inf + (c-1) theta > best
    int64_t best = Uv;
    for (int i = 0; i < nv; ++i) {
      const int32_t th = S.v[i];
      if ((int64_t)Finf + (int64_t)(c - 1) * th > best) break;
      const int32_t F = kc_F<false>(X, S, th);
      if (F < INF) {
        const int64_t v = (int64_t)F + (int64_t)(c - 1) * th;
        if (threadIdx.x == 0) S.val[i] = v;
        best = min(best, v);
      }
      __syncthreads();
    }
    OPT = min(best, Uv);
  }
  // Theta* and the tie-break
  if (threadIdx.x == 0) S.have = 0;
  __syncthreads();
  const int nstar = c > 1 ? nv + 1 : 1;
  for (int si = 0; si < nstar; ++si) {
    int32_t th;
    if (c == 1) th = INF;
    else if (si == 0) {
      const int32_t Fmin = kc_F<false>(X, S, tmin);
      if ((int64_t)Fmin + (int64_t)(c - 1) * tmin != OPT) continue;
      th = tmin;
    } else {
      if (S.val[si - 1] != OPT) continue;
      th = S.v[si - 1];
    }
    const int32_t F = c == 1 ? Finf : (int32_t)(OPT - (int64_t)(c - 1) * th);
    if (!kc_trace(X, S, th, F, Z)) continue;
    if (threadIdx.x == 0) {  // keep the lexicographic best: ends largest, then boundaries smallest
      bool better = !S.have;
      const int deg = X.deg;
      for (int i = 0; i < deg && !better; ++i)
        if (S.ends[i] != S.bends[i]) { better = S.ends[i] > S.bends[i]; goto decided; }
      for (int j = 1; j < deg && !better; ++j) {
        if (S.kls[j - 1] != S.bkls[j - 1]) { better = S.kls[j - 1] < S.bkls[j - 1]; break; }
        if (S.kfs[j] != S.bkfs[j]) { better = S.kfs[j] < S.bkfs[j]; break; }
      }
    decided:
      if (better) {
        for (int i = 0; i < deg; ++i) { S.bends[i] = S.ends[i]; S.bkls[i] = S.kls[i]; S.bkfs[i] = S.kfs[i]; }
        S.have = 1;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    cfg_opt[ci] = S.have ? OPT : INT64_MAX;
    R->status = S.have ? 1 : UNIAP_ERR_INTERNAL;
    const int deg = X.deg;
    int a = 0;
    for (int i = 0; i < deg && S.have; ++i) {
      const int b = S.bends[i];
      const int kf = i > 0 ? S.bkfs[i] : -1, kl = i + 1 < deg ? S.bkls[i] : -1;
      R->ends[i] = b;
      R->kfirst[i] = kf;
      R->klast[i] = kl;
      R->p[i] = X.t(a, b, kf < 0 ? X.NSP : kf, kl < 0 ? X.NSP : kl);
      R->o[i] = i + 1 < deg ? X.o(b, kl, S.bkfs[i + 1]) : 0;
      a = b + 1;
    }
  }
}

cudaError_t launch_k4c(const CfgDev* cfg, const int32_t* arena, const int32_t* T, const int32_t* cfg_list, int li0,
                       int n, int L, int64_t* cfg_opt, void* res, int32_t* zscratch, int64_t zstride,
                       cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  k4c_cut<<<n, KCT, sizeof(KcSmem), st>>>(cfg, arena, T, cfg_list, li0, L, cfg_opt, reinterpret_cast<CutRes*>(res),
                                          zscratch, zstride);
  return cudaGetLastError();
}

size_t cut_result_bytes() { return sizeof(CutRes); }

cudaError_t cutcombine_init() {
  return cudaFuncSetAttribute((const void*)k4c_cut, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(KcSmem));
}

}  // namespace uniap
