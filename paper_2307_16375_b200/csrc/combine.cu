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
// K4's placement DPs, CTA-wide.  Placements of deg stages over [0, L-1]:
// stage i = [a, b] with i-1 <= a <= b <= bhi(i) = L-1-(deg-i), the last
// stage ends at L-1.  Every stage has n = L - deg + 1 candidate ends (and
// starts), so a stage is one small min-plus product: thread groups of g
// lanes own one target (an end b, or a start a), split its sources over the
// g lanes and reduce with shuffles; one barrier per stage.  (A warp-serial
// DP measured ~1000 cycles per stage on B200 -- tools/k4_micro.cu -- being
// bound by the latency of its source loop; here a stage is a few loads and
// log2(g) shuffles.)  The interval tables are in shared memory, pitch PP =
// L | 1, one table per cap level (slev[i]: the level of stage i, NEXT-2).
//  cta_lex: under "every P and O <= theta", the lexicographic minimum of
//           (sum P + sum O, max(P u O)) over placements: F_theta and the
//           smallest bottleneck m among its argmin placements.  (sum, max)
//           pairs under (+, max) with the lexicographic min form a semiring
//           (x <= y implies x (x) z <= y (x) z), so the stage DP is exact; a
//           pair is one 64-bit key sum << 32 | max.  With BN it also returns
//           theta_min = min over placements of max(P u O) (the (min, max)
//           semiring, unconstrained), the smallest theta with a feasible
//           placement.
//  cta_suffix: H_i[a] = min cost of covering [a, L-1] with stages i..deg
//           under theta (for the greedy of the stage ends).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t lex_key(uint32_t sum, uint32_t mx) { return (uint64_t)sum << 32 | mx; }
struct K4Geom {
  int n, g, q, j;  // candidates per stage, lanes per target, this thread's target and lane in its group
  __device__ K4Geom(int L, int deg) {
    // as many lanes per target as the CTA allows (a stage is latency-bound:
    // fewer sources per lane, a few more shuffle rounds); measured against
    // an unrolled 8-source loop with 512 threads (issue-bound, 1.6x slower)
    n = L - deg + 1;
    g = 32;
    while (g > 1 && g * n > (int)blockDim.x) g >>= 1;
    q = threadIdx.x / g;
    j = threadIdx.x % g;
  }
};
template <typename T>
__device__ __forceinline__ T group_min(T v, int g) {
  for (int o = 1; o < g; o <<= 1) {
    const T x = __shfl_xor_sync(0xffffffffu, v, o);
    v = x < v ? x : v;
  }
  return v;
}
__device__ __forceinline__ int32_t group_max(int32_t v, int g) {
  for (int o = 1; o < g; o <<= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// W: [2][MAXL + 1] keys (w of a stage: the best placement of the stages
// before it ending at a - 1, plus O[a - 1]); Wb: [2][MAXL + 1] bottleneck
// values (BN).  Returns (F, m), or (INF, INF) when infeasible; *tmin (BN).
template <bool BN>
__device__ int2 cta_lex(const int32_t* sPall, const int32_t* slev, const int32_t* sO, uint64_t* W, int32_t* Wb, int L,
                        int PP, int deg, int32_t theta, int32_t* tmin) {
  const K4Geom G(L, deg);
  const uint32_t lim = (uint32_t)min(theta, INF - 1);  // P = INF: no interval
  // An unusable w or P enters as sum INF: every key with sum >= INF (INF +
  // INF < 2^32) is larger than every valid key and is dropped at the stage
  // end, so the source loop is branch-free.
  const uint64_t KBAD = lex_key(INF, 0);
  __shared__ uint64_t s_res;
  __shared__ int32_t s_bn;
  auto put = [&](uint64_t* wn, int32_t* wbn, int b, uint64_t c, int32_t cb) {
    // w of the next stage at b + 1 from this stage's key c at end b
    const uint32_t o = (uint32_t)sO[b];
    const uint32_t sum = (uint32_t)(c >> 32) + o;
    wn[b + 1] = (o <= (uint32_t)theta && sum < (uint32_t)INF) ? lex_key(sum, max((uint32_t)c, o)) : KBAD;
    if (BN) wbn[b + 1] = max(cb, sO[b]);
  };
  // stage 1 = [0, b], b <= L - deg
  {
    const int32_t* sP = sPall + slev[0] * L * PP;
    for (int b = threadIdx.x; b <= L - deg; b += blockDim.x) {
      const uint32_t p = (uint32_t)sP[b];
      const uint64_t c = p <= lim ? lex_key(p, p) : KBAD;
      if (deg > 1) put(W, Wb, b, c, sP[b]);
      else if (b == L - 1) { s_res = c; if (BN) s_bn = sP[b]; }
    }
  }
  __syncthreads();
  for (int i = 2; i <= deg; ++i) {
    const int32_t* sP = sPall + slev[i - 1] * L * PP;
    const uint64_t* w = W + ((i & 1) ? MAXL + 1 : 0);  // written by stage i-1
    uint64_t* wn = W + ((i & 1) ? 0 : MAXL + 1);
    const int32_t* wb = Wb + ((i & 1) ? MAXL + 1 : 0);
    int32_t* wbn = Wb + ((i & 1) ? 0 : MAXL + 1);
    const int lo = i - 1;
    // this group's end (the last stage ends at L-1: group 0 writes it); a
    // thread of no group runs an empty source loop but joins the shuffles
    const bool mine = G.q < G.n && (i < deg || G.q == 0);
    const int b = (i == deg) ? L - 1 : lo + G.q;
    const int aend = mine ? b : lo - 1;
    uint64_t acc = KBAD;
    int32_t accb = INF;
    for (int a = lo + G.j; a <= aend; a += G.g) {
      const uint64_t wa = w[a];
      const int32_t p = sP[a * PP + b];
      const uint32_t pe = (uint32_t)p <= lim ? (uint32_t)p : (uint32_t)INF;
      acc = min(acc, lex_key((uint32_t)(wa >> 32) + pe, max((uint32_t)wa, pe)));
      if (BN) accb = min(accb, max(wb[a], p));
    }
    acc = group_min(acc, G.g);
    if (BN) accb = group_min(accb, G.g);
    if (mine && G.j == 0) {
      if ((acc >> 32) >= (uint64_t)INF) acc = KBAD;
      if (i < deg) put(wn, wbn, b, acc, accb);
      else { s_res = acc; if (BN) s_bn = accb; }
    }
    __syncthreads();
  }
  const uint64_t F = s_res;
  if (BN) *tmin = s_bn;
  __syncthreads();  // (s_res reused by the next call)
  // sums reaching INF are infeasible (the builder's quantum keeps every
  // placement sum of a valid input below it)
  return (F >> 32) >= (uint64_t)INF ? make_int2(INF, INF) : make_int2((int32_t)(F >> 32), (int32_t)(uint32_t)F);
}

// H: [deg + 1][L + 1]; entries of stage i are written for a in [i-1, bhi(i)],
// exactly the ones the greedy reads.
__device__ void cta_suffix(const int32_t* sPall, const int32_t* slev, const int32_t* sO, int32_t* H, int L, int PP,
                           int deg, int32_t theta) {
  const K4Geom G(L, deg);
  {
    const int32_t* Pd = sPall + slev[deg - 1] * L * PP;
    for (int a = deg - 1 + (int)threadIdx.x; a < L; a += blockDim.x) {
      const int32_t p = Pd[a * PP + L - 1];
      H[deg * (L + 1) + a] = p <= theta ? p : INF;
    }
  }
  __syncthreads();
  for (int i = deg - 1; i >= 1; --i) {
    // H_i[a] = min_b P_i[a][b] + O[b] + H_{i+1}[b+1], a <= b <= bhi
    const int bhi = L - 1 - (deg - i);
    const int32_t* Pi = sPall + slev[i - 1] * L * PP;
    const int32_t* Hn = H + (i + 1) * (L + 1);
    const int a = i - 1 + G.q;  // (a > bhi for a thread of no group: empty loop, joins the shuffles)
    uint32_t x = INF;
    for (int b = a + G.j; b <= bhi; b += G.g) {
      const int32_t p = Pi[a * PP + b], o = sO[b], h = Hn[b + 1];
      const uint32_t wv = (o <= theta && h < INF) ? (uint32_t)(o + h) : INF;
      x = __viaddmin_u32(wv, p <= theta ? (uint32_t)p : INF, x);
    }
    x = group_min(x, G.g);
    if (G.q < G.n && G.j == 0) H[i * (L + 1) + a] = (int32_t)min(x, (uint32_t)INF);
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// K4 (with K3): the config's optimum OPT = min over theta of Val(theta) =
// F_theta + (c-1) theta, and its lexicographically largest stage-end vector
// over the optimal placements (= smallest stage_of, reading A-11).  One CTA
// per config, on the stream of the config's forward group, so every config's
// ends are ready when K5a picks the winner.
//
// 1. Descent over the bottlenecks: theta_0 = INF; at theta_j, cta_lex gives
//    F_j = F_{theta_j} and m_j <= theta_j, the smallest max(P u O) of a
//    placement attaining F_j.  For theta in [m_j, theta_j] that placement is
//    feasible and optimal, so F_theta = F_j and Val(theta) = F_j + (c-1)
//    theta is smallest at theta = m_j (strictly, c > 1): record (m_j,
//    Val(m_j)), then continue at theta_{j+1} = m_j - 1 (integer costs).
//    Below theta_{j+1}, F_theta >= F_j and theta >= theta_min, so once
//    F_j + (c-1) theta_min > best no theta below can reach OPT (strict: ties
//    are kept for the tie-break).  The recorded m_j therefore include every
//    theta with Val(theta) = OPT (Theta*) and each Val(m_j) is exact; no
//    candidate list, sort or scan.  The number of steps is the number of
//    (sum, max) Pareto points visited: 2 for every Llama-like config, <= 9 on
//    the T5-like profile.  c = 1: Val = F_theta, OPT = F_INF, Theta* = {INF}.
// 2. Per theta in Theta*: the suffix DP H (cta_suffix), then the greedy
//    largest end of each stage (warp 0, a ballot over the ends) that still
//    reaches F_theta = OPT - (c-1) theta; the lexicographically largest end
//    vector over Theta* wins.
// Out: cfg_opt[config]; ends[li] = {ok, end of stage 1, ..., end of stage deg};
// thetas / vals: the descent's (m_j, Val(m_j)) (scratch).
// Dynamic shared memory: the interval tables (one per cap level, odd pitch
// L | 1), then H.
// ---------------------------------------------------------------------------
constexpr int K4T = 256;  // threads per K4 CTA
constexpr int K4EW = MAXL + 1;  // words per config in `ends`
// (+ 64 words of slack after H)
size_t k4_smem(int L, int nlev) { return (size_t)(nlev * L * (L | 1) + (L + 1) * (L + 1) + 64) * sizeof(int32_t); }
// dynamic shared memory K4 may take (its static arrays are ~3 KB); beyond it
// the interval tables stay in global memory (k4_vals: tabs_smem = 0)
constexpr size_t K4_SMEM_MAX = 200 * 1024;
__device__ __forceinline__ void cp_async4(int32_t* dst, const int32_t* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

template <bool TABS_SMEM>
__global__ void __launch_bounds__(K4T) k4_vals(const CfgDev* __restrict__ cfgs, const int32_t* __restrict__ arena,
                                               const int32_t* __restrict__ P, const int32_t* __restrict__ cfg_list,
                                               int li0, int L, int32_t* __restrict__ thetas,
                                               int64_t* __restrict__ vals, int32_t* __restrict__ ends,
                                               int64_t* __restrict__ cfg_opt, long long* __restrict__ best_obj) {
  TraceScope tr(TR_K4 | (uint32_t)li0 << 8);
  extern __shared__ __align__(16) int32_t k4dyn[];
  __shared__ int32_t slev[MAXL], sO[MAXL], cur[MAXL];
  __shared__ uint64_t W[2 * (MAXL + 1)];
  __shared__ int32_t Wb[2 * (MAXL + 1)];
  const int li = li0 + blockIdx.x;
  const int ci = cfg_list[li];
  const CfgDev& cf = cfgs[ci];
  const int deg = cf.deg;
  const int64_t cm1 = cf.c - 1;
  const int t = threadIdx.x, w = t >> 5, lane = t & 31;
  int32_t* E = ends + (int64_t)li * K4EW;
  int64_t* V = vals + (int64_t)li * TMAX;
  int32_t* th = thetas + (int64_t)li * TMAX;
  if (deg > L) {  // Eq. 7b cannot hold (reading A-22)
    if (t == 0) { E[0] = 0; cfg_opt[ci] = INT64_MAX; }
    return;
  }
  if (deg == 1) {  // one placement [0, L-1]: tpi = p + (c-1) p
    if (t == 0) {
      const int32_t p = P[cf.offP + (int64_t)cf.lev_of[0] * L * L + (L - 1)];
      E[0] = p < INF;
      E[1] = L - 1;
      cfg_opt[ci] = p < INF ? (int64_t)p + cm1 * p : INT64_MAX;
      tr.extra = 1;
    }
    return;
  }
  if (deg == L) {  // one placement, every layer a stage: tpi = sum P + sum O + (c-1) max(P u O)
    if (w == 0) {
      int64_t sum = 0;
      int32_t mx = 0;
      bool ok = true;
      for (int a = lane; a < L; a += 32) {
        const int32_t p = P[cf.offP + (int64_t)cf.lev_of[a] * L * L + (int64_t)a * L + a];
        const int32_t o = a < L - 1 ? arena[cf.offO + a] : 0;
        ok = ok && p < INF;
        sum += (int64_t)p + o;
        mx = max(mx, max(p, o));
      }
      for (int o = 16; o > 0; o >>= 1) {
        sum += __shfl_xor_sync(0xffffffffu, sum, o);
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      }
      ok = __all_sync(0xffffffffu, ok) && sum < INF;  // (a sum reaching INF is infeasible, as in cta_lex)
      for (int a = lane; a < L; a += 32) E[1 + a] = a;
      if (lane == 0) {
        E[0] = ok;
        cfg_opt[ci] = ok ? sum + cm1 * mx : INT64_MAX;
        tr.extra = 1;
      }
    }
    return;
  }
  // the interval tables in shared memory (odd pitch), or -- when a launch's
  // levels do not fit (1F1B: up to one level per stage) -- read in place
  // from global memory (L2) with pitch L
  // (two instantiations: the compiler sees a shared-memory pointer in the first)
  const int PP = TABS_SMEM ? (L | 1) : L;
  const int nlev = cf.nlev;
  const int32_t* sP = TABS_SMEM ? k4dyn : P + cf.offP;  // [nlev][L][PP]
  int32_t* H = k4dyn + (TABS_SMEM ? nlev * L * PP : 0);  // [deg + 1][L + 1]
  {  // asynchronous copies (LDGSTS): every load of the tables in flight at once
    const int32_t* Pc = P + cf.offP;
    for (int r = w; TABS_SMEM && r < nlev * L; r += K4T / 32)  // row r = level * L + a
      for (int b = lane; b < L; b += 32) cp_async4(k4dyn + r * PP + b, Pc + (int64_t)r * L + b);
    for (int i = t; i < L - 1; i += K4T) cp_async4(sO + i, arena + cf.offO + i);
  }
  for (int i = t; i < MAXL; i += K4T) slev[i] = cf.lev_of[i];
  cp_async_wait_all();
  __syncthreads();
  // diagnostics (UNIAP_TRACE): a record per phase, from the kernel's start
  auto phase = [&](uint32_t kind) {
    if (g_trace && t == 0) trace_put(g_trace, 0x80000000u | kind | (uint32_t)li0 << 8, tr.t0, 0, blockIdx.x, 0);
  };
  phase(9);  // tables loaded
  // ---- 1. OPT and the candidates of Theta* ----
  int32_t tmin = 0;
  int2 fm = cm1 > 0 ? cta_lex<true>(sP, slev, sO, W, Wb, L, PP, deg, INF, &tmin)
                    : cta_lex<false>(sP, slev, sO, W, Wb, L, PP, deg, INF, nullptr);
  const int32_t Finf = fm.x;
  int64_t best = Finf < INF ? (int64_t)Finf : INT64_MAX;
  int n = 0;
  if (Finf < INF && cm1 > 0) {
    best = INT64_MAX;
    for (;;) {  // (uniform: every thread holds the same fm)
      const int64_t val = (int64_t)fm.x + cm1 * fm.y;
      if (t == 0) { th[n] = fm.y; V[n] = val; }
      ++n;
      best = min(best, val);
      if ((int64_t)fm.x + cm1 * tmin > best || fm.y <= tmin || n == TMAX) break;
      fm = cta_lex<false>(sP, slev, sO, W, Wb, L, PP, deg, fm.y - 1, nullptr);
      if (fm.x >= INF) break;
    }
  }
  const int64_t OPT = best;
  __shared__ int s_skip;
  if (t == 0) {
    cfg_opt[ci] = OPT;
    tr.extra = (uint32_t)n;
    // the running minimum over the configs whose K4 got here first: a config
    // strictly worse than one of them cannot be the winner (K5a's key is
    // (objective, deg, c)), so its stage ends are not needed.  The winner
    // always finds the minimum >= its own objective and computes them.
    s_skip = OPT == INT64_MAX || (long long)OPT > atomicMin(best_obj, (long long)OPT);
  }
  __syncthreads();
  phase(10);  // OPT and Theta* known
  if (s_skip) {
    if (t == 0) E[0] = 0;
    return;
  }
  // ---- 2. the lexicographically largest stage ends over Theta* ----
  const int nst = cm1 > 0 ? n : 1;
  bool have = false;  // (thread 0: the best vector so far is E[1..deg])
  for (int j = 0; j < nst; ++j) {
    __syncthreads();  // th / V of the descent (thread 0) visible; H free
    if (cm1 > 0 && V[j] != OPT) continue;  // (uniform)
    const int32_t theta = cm1 > 0 ? th[j] : INF;
    const int64_t F_target = OPT - cm1 * (cm1 > 0 ? theta : 0);
    cta_suffix(sP, slev, sO, H, L, PP, deg, theta);
    phase(14);  // H of this theta
    if (w == 0) {
      bool ok = (int64_t)H[1 * (L + 1) + 0] == F_target;
      // greedy: the largest end of each stage that still reaches F_target
      int64_t pre = 0;
      int a = 0;
      for (int i = 1; i < deg && ok; ++i) {
        const int32_t* Pi = sP + slev[i - 1] * L * PP;
        const int32_t* Hn = H + (i + 1) * (L + 1);
        int found = -1;
        for (int b0 = L - 1 - (deg - i); b0 >= a && found < 0; b0 -= 32) {
          const int b = b0 - lane;
          bool c = false;
          if (b >= a) {
            const int32_t p = Pi[a * PP + b], o = sO[b], hh = Hn[b + 1];
            c = p <= theta && o <= theta && hh < INF && pre + p + o + hh == F_target;
          }
          const unsigned m = __ballot_sync(0xffffffffu, c);
          if (m) found = b0 - (__ffs(m) - 1);
        }
        if (found < 0) { ok = false; break; }
        if (lane == 0) cur[i - 1] = found;
        pre += Pi[a * PP + found] + sO[found];
        a = found + 1;
      }
      __syncwarp();
      if (lane == 0 && ok) {  // keep the lexicographically largest end vector
        cur[deg - 1] = L - 1;
        bool better = !have;
        for (int i = 0; i < deg && !better; ++i)
          if (cur[i] != E[1 + i]) { better = cur[i] > E[1 + i]; break; }
        if (better)
          for (int i = 0; i < deg; ++i) E[1 + i] = cur[i];
        have = true;
      }
    }
    phase(15);  // ends of this theta
  }
  if (t == 0) E[0] = have;
}

cudaError_t launch_k4(const CfgDev* cfg, const int32_t* arena, const int32_t* P, const int32_t* cfg_list, int li0,
                      int n_local, int L, int nlev, int32_t* thetas, int64_t* vals, int32_t* ends, int64_t* cfg_opt,
                      long long* best_obj, cudaStream_t st) {
  if (n_local <= 0) return cudaSuccess;
  if (k4_smem(L, nlev) <= K4_SMEM_MAX)
    k4_vals<true><<<n_local, K4T, k4_smem(L, nlev), st>>>(cfg, arena, P, cfg_list, li0, L, thetas, vals, ends,
                                                         cfg_opt, best_obj);
  else
    k4_vals<false><<<n_local, K4T, k4_smem(L, 0), st>>>(cfg, arena, P, cfg_list, li0, L, thetas, vals, ends,
                                                          cfg_opt, best_obj);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// K5a: global (objective, deg, c) argmin over the local configs, the record
// header, the winner's stages (its ends from K4 / K4c) and the device-side
// plan of the traceback's backward sweeps.  One CTA.
// ---------------------------------------------------------------------------
constexpr int K5T = 256;
__global__ void __launch_bounds__(K5T) k5a_winner(const CfgDev* __restrict__ cfgs, const int32_t* __restrict__ arena,
                                                  const int32_t* __restrict__ P, const int32_t* __restrict__ cfg_list,
                                                  int n_local, int L, const int32_t* __restrict__ ends,
                                                  const int64_t* __restrict__ cfg_opt, Winner* __restrict__ win,
                                                  long long* __restrict__ best_obj, RecordArgs ra) {
  TraceScope tr(TR_K5A);
  if (threadIdx.x == 0) *best_obj = LLONG_MAX;  // K4's running minimum, ready for the next run (every K4 is done)
  __shared__ int64_t s_opt[1];
  __shared__ int32_t s_win, s_ci;
  const int t = threadIdx.x, w = t >> 5, lane = t & 31;
  uniap_record* r = ra.rec;
  // winner by (objective, deg, c): warp 0, lanes over the local configs,
  // then a shuffle argmin on the key tuple
  if (w == 0) {
    int wi = -1, bd = 0, bc = 0, bci = -1;
    int64_t best = INT64_MAX;
    for (int li = lane; li < n_local; li += 32) {
      const int ci = cfg_list[li];
      const int64_t v = cfg_opt[ci];
      const int dg = cfgs[ci].deg, cc = cfgs[ci].c;
      if (v != INT64_MAX && (wi < 0 || v < best || (v == best && (dg < bd || (dg == bd && cc < bc))))) {
        wi = li; best = v; bd = dg; bc = cc; bci = ci;
      }
    }
    for (int off = 16; off > 0; off >>= 1) {
      const int owi = __shfl_down_sync(0xffffffffu, wi, off), obd = __shfl_down_sync(0xffffffffu, bd, off),
                obc = __shfl_down_sync(0xffffffffu, bc, off), oci = __shfl_down_sync(0xffffffffu, bci, off);
      const int64_t ob = __shfl_down_sync(0xffffffffu, best, off);
      if (owi >= 0 && (wi < 0 || ob < best || (ob == best && (obd < bd || (obd == bd && obc < bc))))) {
        wi = owi; best = ob; bd = obd; bc = obc; bci = oci;
      }
    }
    if (lane == 0) {
      s_win = wi;
      s_ci = bci;
      s_opt[0] = best;
    }
  } else if (w == 1) {  // the record's work counts (level 2: K1f's, where it trimmed the sweeps)
    unsigned long long c = 0, x = 0;
    if (ra.work)
      for (int li = lane; li < ra.n_local; li += 32) {
        c += ra.work[2 * cfg_list[li]];
        x += ra.work[2 * cfg_list[li] + 1];
      }
    for (int off = 16; off > 0; off >>= 1) {
      c += __shfl_xor_sync(0xffffffffu, c, off);
      x += __shfl_xor_sync(0xffffffffu, x, off);
    }
    if (lane == 0) {
      r->n_cfg_local = ra.n_local;
      r->L = ra.L;
      r->dp_cells = ra.work ? c : ra.cells;
      r->dp_relax = ra.work ? x : ra.relax;
      r->dp_cells_canonical = ra.cells_canon;
    }
  } else if (t == 64) {
    r->status = (ra.qglob && ra.qglob[1] != 0) ? UNIAP_ERR_RANGE : 0;
  }
  // the record header: every field K5c does not write (assignment arrays zeroed)
  for (int i = t; i < UNIAP_MAX_LAYERS; i += K5T) {
    r->stage_of[i] = 0;
    r->strategy_of[i] = 0;
    r->stage_cost[i] = 0;
    r->cut_cost[i] = 0;
    r->stage_mem[i] = 0;
  }
  if (t < MAXCLS) ra.bw->count[t] = 0;
  if (t < MAXL) win->kfirst[t] = win->klast[t] = -1;
  __syncthreads();
  const int wl = s_win;
  if (t == 0) {
    r->objective = INT64_MAX;
    r->cfg_index = -1;
    r->deg = r->c = 0;
    if (wl < 0) { win->objective = INT64_MAX; win->cfg = -1; win->status = 0; }
  }
  if (wl < 0) return;
  const int ci = s_ci;
  __syncthreads();  // the header is written before the winner's fields
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
  // the winner's stages from K4: stage i = [end[i-1] + 1, end[i]]
  const CfgDev& cf = cfgs[ci];
  const int deg = cf.deg;
  const int32_t* E = ends + (int64_t)wl * (MAXL + 1);
  const bool have = E[0] != 0;
  if (t < deg) {
    const int b = have ? E[1 + t] : L - 1;
    const int a = t == 0 ? 0 : (have ? E[t] + 1 : L - 1);
    win->end[t] = b;
    win->p[t] = P[cf.offP + (int64_t)cf.lev_of[t] * L * L + (int64_t)a * L + b];
    win->o[t] = (t + 1 < deg) ? arena[cf.offO + b] : 0;
  }
  const int64_t kept = ra.gstore[ci];  // deg = 1: the forward phase's sweep kept its tables
  const int cls = ra.cls_of_cfg[ci];
  const bool st_ok = have && r->status == 0;  // (r->status: written before the barrier above)
  __syncthreads();  // every thread has read r->status before thread 0 may overwrite it
  if (t == 0) {
    const int64_t OPT = s_opt[0];
    win->objective = OPT;
    win->cfg = ci;
    win->deg = deg;
    win->c = cf.c;
    win->S = cf.S;
    win->NSP = cf.NSP;
    win->n_theta_star = 0;
    win->status = have ? 0 : 99;
    if (!have) r->status = UNIAP_ERR_INTERNAL;
    r->objective = OPT;
    r->cfg_index = ci;
    r->deg = deg;
    r->c = cf.c;
  }
  // the backward sweeps of the traceback: one per stage, one per skip
  // conditioning ks when the stage contains the skip source and an edge of it
  // (NEXT-4: one per copy of the stage's run of skip sources), in stage order
  if (cf.nsk >= 2) {
    if (t != 0) return;
    int n = 0;
    int64_t goff = 0;
    int a = 0;
    for (int i = 0; i < deg && st_ok; ++i) {
      const int b = E[1 + i], len = b - a + 1;
      int jlo;
      const int nr = skip_run(cf, a, b, &jlo);
      int ncp = 1;
      for (int j = 0; j < nr; ++j) ncp *= cf.S;
      ra.bw->gofs[i * 33] = goff;  // copy kappa at goff + kappa * len * NSP * Q (k5c_walk)
      for (int kp = 0; kp < ncp; ++kp) {
        const int64_t ar = copy_rel(cf, jlo, nr, kp, L);
        ra.bw_inst[n++] = Inst{ci, b, len, -1, -1, 0, goff, 0, -1, len, cf.lev_of[i], 0, -1,
                               (int32_t)copy_mrel(cf, nr, ar, cf.lev_of[i], L), (int32_t)ar};
        goff += (int64_t)len * cf.NSP * (ra.cap + 1);
      }
      a = b + 1;
    }
    ra.bw->count[cls] = n;
    return;
  }
  // warp 0, lane l: stages 2l and 2l + 1 (deg <= 64); a scan of the sweep
  // counts and G sizes gives each stage its first instance and G offset
  if (w != 0) return;
  const int64_t row = (int64_t)cf.NSP * (ra.cap + 1);
  int cnt[2], a2[2], b2[2];
  bool cond2[2];
  int64_t sz[2];
  for (int h = 0; h < 2; ++h) {
    const int i = 2 * lane + h;
    cnt[h] = 0;
    sz[h] = 0;
    if (i < deg && st_ok) {
      b2[h] = E[1 + i];
      a2[h] = i == 0 ? 0 : E[i] + 1;
      cond2[h] = cf.skip >= 0 && a2[h] <= cf.skip && cf.skip + 2 <= b2[h];
      cnt[h] = kept >= 0 ? 0 : (cond2[h] ? cf.S : 1);
      sz[h] = (int64_t)cnt[h] * (b2[h] - a2[h] + 1) * row;
    }
  }
  int n_in = cnt[0] + cnt[1];
  int64_t g_in = sz[0] + sz[1];
  for (int o = 1; o < 32; o <<= 1) {  // inclusive scan over the lanes
    const int nn = __shfl_up_sync(0xffffffffu, n_in, o);
    const int64_t gg = __shfl_up_sync(0xffffffffu, g_in, o);
    if (lane >= o) { n_in += nn; g_in += gg; }
  }
  int n = n_in - cnt[0] - cnt[1];
  int64_t goff = g_in - sz[0] - sz[1];
  for (int h = 0; h < 2; ++h) {
    const int i = 2 * lane + h;
    if (i >= deg || !st_ok) break;
    const int b = b2[h], len = b - a2[h] + 1;
    const bool cond = cond2[h];
    for (int ks = cond ? 0 : -1; ks < (cond ? cf.S : 0); ++ks) {
      if (kept >= 0) {
        ra.bw->gofs[i * 33 + ks + 1] = kept + (int64_t)(ks < 0 ? 0 : ks) * L * row;
        continue;
      }
      ra.bw->gofs[i * 33 + ks + 1] = goff;
      ra.bw_inst[n++] = Inst{ci, b, len, ks, -1, 0, goff, 0, -1, len, cf.lev_of[i], 0, -1,
                             (int32_t)(cfg_moff(cf, cf.lev_of[i], L) - cf.offM)};  // (its stage's memory table)
      goff += (int64_t)len * row;
    }
  }
  if (lane == 31) ra.bw->count[cls] = st_ok ? n_in : 0;
}

// Phase 2 of a split multi-GPU run (uniap_run_phase): the global winner
// among the gathered phase-1 records, by uniap_pick's key (objective, deg, c);
// a rank whose local winner is not it skips its traceback (no backward
// sweeps, K5c idle), so only the winner's owner pays for one.
__global__ void k_decide(const uniap_record* __restrict__ recs, int world, int rank, BwPlan* bw, Winner* win) {
  if (threadIdx.x != 0) return;
  int best = -1;
  for (int r = 0; r < world; ++r) {
    const uniap_record& x = recs[r];
    if (x.status != 0 || x.objective == INT64_MAX) continue;
    if (best < 0) { best = r; continue; }
    const uniap_record& b = recs[best];
    if (x.objective < b.objective || (x.objective == b.objective && (x.deg < b.deg || (x.deg == b.deg && x.c < b.c))))
      best = r;
  }
  if (best != rank) {
    for (int c = 0; c < MAXCLS; ++c) bw->count[c] = 0;
    win->status = 97;  // (k5c_walk: nothing to walk)
  }
}

cudaError_t launch_decide(const uniap_record* recs, int world, int rank, BwPlan* bw, Winner* win, cudaStream_t st) {
  k_decide<<<1, 32, 0, st>>>(recs, world, rank, bw, win);
  return cudaGetLastError();
}

cudaError_t launch_k5a(const CfgDev* cfg, const int32_t* arena, const int32_t* P, const int32_t* cfg_list, int n_local,
                       int L, const int32_t* ends, const int64_t* cfg_opt, Winner* win, long long* best_obj,
                       const RecordArgs& ra, cudaStream_t st) {
  k5a_winner<<<1, K5T, 0, st>>>(cfg, arena, P, cfg_list, n_local, L, ends, cfg_opt, win, best_obj, ra);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// K5c: per stage, the lexicographically smallest strategy vector reaching the
// stage optimum, walking the backward tables G (K2 backward sweeps):
// at layer u take the smallest k with  R[u-1][k_{u-1}][k] + G[u][k][q] = rest.
// One CTA per stage; warp w walks the conditioning ks = w (or none).
// Also writes the record (objective, placement, costs, memory).
// ---------------------------------------------------------------------------
// NEXT-4 part of k5c_walk (a separate function, so the one-source walk's
// code is unchanged): the stage's conditioning copies, 32 at a time (one per
// warp), each walked on its own A' / M' tables; the lexicographically
// smallest vector over the copies.
__device__ __noinline__ void k5c_walk_copies(const CfgDev& cf, const CfgDev* __restrict__ cfgs,
                                             const int32_t* __restrict__ arena, const int32_t* __restrict__ G,
                                             const BwPlan* __restrict__ bw, const Winner& W, int L, int cap,
                                             uniap_record* __restrict__ rec, int stage, int a, int b,
                                             int32_t (*vec)[MAXL], int32_t* mem, int32_t* okw) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int NSP = cf.NSP, Q = cap + 1, S = cf.S;
  __shared__ int32_t best[MAXL];
  __shared__ int32_t best_mem, have;
  int jlo;
  const int nr = skip_run(cf, a, b, &jlo);
  int ncp = 1;
  for (int j = 0; j < nr; ++j) ncp *= S;
  const int len = b - a + 1;
  if (threadIdx.x == 0) have = 0;
  for (int c0 = 0; c0 < ncp; c0 += 32) {
    const int cp = c0 + w;
    bool ok = false;
    if (cp < ncp) {
      const int64_t ar = copy_rel(cf, jlo, nr, cp, L);
      const int32_t* Ac = arena + cf.offA + ar;  // A' (skip-edge terms folded in)
      const int32_t* Mc = arena + cf.offM + copy_mrel(cf, nr, ar, cf.lev_of[stage], L);  // M' (run sources held)
      const int32_t* Rfc = arena + cf.offRf;
      const int32_t* g = G + bw->gofs[stage * 33] + (int64_t)cp * len * NSP * Q;
      int64_t rest = W.p[stage];
      int q = cfgs[W.cfg].lcap[cfgs[W.cfg].lev_of[stage]], kprev = -1;
      int32_t msum = 0;
      ok = true;
      for (int u = a; u <= b && ok; ++u) {
        const int k = lane;
        bool c = false;
        int32_t edge = 0, ap = 0, mk = 0;
        if (k < S) {
          mk = Mc[u * NSP + k];
          const int32_t gv = g[((int64_t)(u - a) * NSP + k) * Q + q];
          edge = (u > a) ? Rfc[((int64_t)(u - 1) * NSP + kprev) * NSP + k] : 0;
          ap = Ac[u * NSP + k];
          c = gv < INF && (int64_t)edge + gv == rest;
        }
        const unsigned m = __ballot_sync(0xffffffffu, c);
        if (!m) { ok = false; break; }
        const int kk = __ffs(m) - 1;
        rest -= (int64_t)__shfl_sync(0xffffffffu, edge, kk) + __shfl_sync(0xffffffffu, ap, kk);
        const int32_t m2 = __shfl_sync(0xffffffffu, mk, kk);
        q -= m2;
        msum += m2;
        kprev = kk;
        if (lane == 0) vec[w][u] = kk;
      }
      if (lane == 0) mem[w] = msum;
    }
    if (lane == 0) okw[w] = ok;
    __syncthreads();
    if (threadIdx.x == 0)  // the lexicographically smallest vector over the copies so far
      for (int j = 0; j < 32 && c0 + j < ncp; ++j) {
        if (!okw[j]) continue;
        bool better = !have;
        for (int u = a; u <= b && !better; ++u)
          if (vec[j][u] != best[u]) { better = vec[j][u] < best[u]; break; }
        if (better) {
          for (int u = a; u <= b; ++u) best[u] = vec[j][u];
          best_mem = mem[j];
          have = 1;
        }
      }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (!have) {
      rec->status = UNIAP_ERR_INTERNAL;
    } else {
      for (int u = a; u <= b; ++u) {
        rec->strategy_of[u] = cfgs[W.cfg].orig[best[u]];
        rec->stage_of[u] = stage;
      }
      rec->stage_mem[stage] = best_mem;
      rec->stage_cost[stage] = W.p[stage];
      rec->cut_cost[stage] = W.o[stage];
    }
  }
  }

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
  const CfgDev& cf = cfgs[W.cfg];  // (by reference: the NEXT-4 path indexes its arrays)
  int skip;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int a = stage == 0 ? 0 : W.end[stage - 1] + 1, b = W.end[stage];
  skip = cf.skip;
  const bool cond = skip >= 0 && a <= skip && skip + 2 <= b;
  const int nks = cond ? cf.S : 1;
  const int NSP = cf.NSP, Q = cap + 1, S = cf.S;
  if (cf.nsk >= 2) {  // NEXT-4: the conditioning copies (k5c_walk_copies)
    k5c_walk_copies(cf, cfgs, arena, G, bw, W, L, cap, rec, stage, a, b, vec, mem, okw);
    return;
  }
  const int32_t* A = arena + cf.offA;
  const int32_t* M = arena + cfg_moff(cfgs[W.cfg], cfgs[W.cfg].lev_of[stage], L);  // the stage's memory table
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
  for (const void* f : {(const void*)k_fill, (const void*)k4_vals<true>, (const void*)k4_vals<false>,
                        (const void*)k5a_winner, (const void*)k5c_walk}) {
    cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
  }
  for (const void* f : {(const void*)k4_vals<true>, (const void*)k4_vals<false>}) {
    cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K4_SMEM_MAX);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace uniap
