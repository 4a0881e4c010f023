/* oracle.c -- UniAP CPU ORACLE: plain, slow, obviously correct.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Every function cites the passage
 * of /root/reference/PAPER.md it follows; readings of silent or ambiguous
 * passages are the A-n items of DESIGN.md Sec. 2.
 *
 * Pins (tests/test_oracle_*.py, all "not gpu"):
 *   - whole objective + argmin: brute force over every stage-and-strategy
 *     assignment (oracle/brute.py) on the toy and >= 2000 random instances;
 *   - interval table: textbook tropical matrix-chain product when memory is
 *     slack; multiple-choice-knapsack brute force when costs vanish;
 *   - deg=1 path == Appendix C QIP (an independent chain DP);
 *   - closed forms (R=0, |S|=1, c=1 & O=0 tie-break, large-c min-max);
 *   - builder': the SPEC.md worked examples and Eq. (1) anchors.
 */
#include "oracle.h"

#include <limits.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

typedef unsigned __int128 u128;

#define INF ((int64_t)1 << 60) /* "infeasible" inside the oracle (int64) */
#define ENTRY_MAX (1 << 22)    /* reading A-10: table entries in [0, 2^22]   */
#define SUM_MAX (1 << 28)      /* reading A-9: per-config sum bound          */

static int64_t add_sat(int64_t x, int64_t y) { return (x >= INF || y >= INF) ? INF : (x + y >= INF ? INF : x + y); }
static int64_t min64(int64_t x, int64_t y) { return x < y ? x : y; }
static int64_t max64(int64_t x, int64_t y) { return x > y ? x : y; }

/* ======================================================================== */
/* Validation of level-1 tables                                             */
/* ======================================================================== */
static int validate_tables(const orc_tables* t) {
  if (!t || t->L < 1 || t->L > ORC_MAX_L || t->cap < 0 || t->n_cfg < 1 || !t->cfg) return ORC_ERR_ARG;
  if (t->skip_src < -1 || t->skip_src >= t->L) return ORC_ERR_ARG;
  if (t->n_skip < 0 || t->n_skip > ORC_MAX_SKIP || (t->n_skip > 0 && (!t->skip_srcs || t->skip_src >= 0)))
    return ORC_ERR_ARG;
  for (int j = 0; j < t->n_skip; ++j) /* distinct, ascending (reading A-33) */
    if (t->skip_srcs[j] < 0 || t->skip_srcs[j] >= t->L || (j > 0 && t->skip_srcs[j] <= t->skip_srcs[j - 1]))
      return ORC_ERR_ARG;
  int L = t->L;
  for (int i = 0; i < t->n_cfg; ++i) {
    const orc_cfg* c = &t->cfg[i];
    if (c->deg < 1 || c->c < 1 || c->n_strat < 1 || c->n_strat > ORC_MAX_S) return ORC_ERR_ARG;
    if (!c->A || (!c->M && !c->M_stage) || (L > 1 && !c->R)) return ORC_ERR_ARG;
    for (int j = 0; j < i; ++j)
      if (t->cfg[j].deg == c->deg && t->cfg[j].c == c->c) return ORC_ERR_ARG;
    int S = c->n_strat;
    int64_t sum = 0, osum = 0;
    for (int u = 0; u < L; ++u) {
      int64_t ma = 0, mr = 0, ms = 0;
      for (int k = 0; k < S; ++k) {
        int32_t a = c->A[u * S + k], m = c->M ? c->M[u * S + k] : 0;
        if (a < 0 || a > ENTRY_MAX || m < 0) return ORC_ERR_RANGE;
        ma = max64(ma, a);
      }
      if (u >= 1)
        for (int k = 0; k < S * S; ++k) {
          int32_t r = c->R[(size_t)(u - 1) * S * S + k];
          if (r < 0 || r > ENTRY_MAX) return ORC_ERR_RANGE;
          mr = max64(mr, r);
        }
      if (c->Rskip && t->skip_src >= 0 && u >= t->skip_src + 2)
        for (int k = 0; k < S * S; ++k) {
          int32_t r = c->Rskip[(size_t)u * S * S + k];
          if (r < 0 || r > ENTRY_MAX) return ORC_ERR_RANGE;
          ms = max64(ms, r);
        }
      for (int j = 0; c->Rskips && j < t->n_skip; ++j) /* every source's edge into u */
        if (u >= t->skip_srcs[j] + 2) {
          int64_t mj = 0;
          for (int k = 0; k < S * S; ++k) {
            int32_t r = c->Rskips[((size_t)j * L + u) * S * S + k];
            if (r < 0 || r > ENTRY_MAX) return ORC_ERR_RANGE;
            mj = max64(mj, r);
          }
          ms += mj;
        }
      sum += ma + mr + ms;
    }
    if (c->O)
      for (int e = 0; e < L - 1; ++e) {
        if (c->O[e] < 0 || c->O[e] > ENTRY_MAX) return ORC_ERR_RANGE;
        osum += c->O[e];
      }
    if (c->stage_cap)
      for (int i = 0; i < c->deg; ++i)
        if (c->stage_cap[i] < 0 || c->stage_cap[i] > t->cap) return ORC_ERR_ARG;
    if (c->M_stage) { /* stage-indexed memory (1F1B, reading A-32): entries >= 0, not with Rcut */
      if (c->Rcut) return ORC_ERR_ARG;
      for (int64_t j = 0; j < (int64_t)c->deg * L * S; ++j)
        if (c->M_stage[j] < 0) return ORC_ERR_RANGE;
    }
    if (c->Rcut) {
      if (c->stage_cap) /* NEXT-1 and NEXT-2 are not combined: caps must all be the common cap */
        for (int i = 0; i < c->deg; ++i)
          if (c->stage_cap[i] != t->cap) return ORC_ERR_ARG;
      int64_t csum = 0;
      for (int e = 0; e < L - 1; ++e) {
        int64_t mx = 0;
        for (int k = 0; k < S * S; ++k) {
          int32_t r = c->Rcut[(size_t)e * S * S + k];
          if (r < 0 || r > ENTRY_MAX) return ORC_ERR_RANGE;
          mx = max64(mx, r);
        }
        csum += mx + (c->O ? c->O[e] : 0);
      }
      if (csum > SUM_MAX) return ORC_ERR_RANGE; /* every cut's o_j <= O[e] + max Rcut[e] */
    }
    if (sum > SUM_MAX || osum > SUM_MAX) return ORC_ERR_RANGE;
  }
  return ORC_OK;
}

/* ======================================================================== */
/* Per-layer cost terms of Eq. (3) with the skip-edge conditioning          */
/* ======================================================================== */
/* A'_uk: the execution cost A_uk plus, when the skip source s of the graph
 * lies in the same stage with strategy ks, the resharding term of the skip
 * edge <s,u> (Eq. 3's quadratic term; readings A-16, A-17). */
/* Skip edges (one source: T5's cross-attention; several sources: NEXT-4,
 * reading A-33).  A stage conditions on the strategy of every skip source it
 * holds together with one of that source's edges; a "copy" fixes those
 * strategies (kv[j] = -1: source j not conditioned in this copy). */
typedef struct {
  int n;                          /* skip sources of the graph with tables in this config */
  int src[ORC_MAX_SKIP];
  const int32_t* R[ORC_MAX_SKIP]; /* [L][S][S] per source: R[v][k_src][k_v] for v >= src + 2 */
  int kv[ORC_MAX_SKIP];
} cond_t;

static void skip_sources(const orc_tables* t, const orc_cfg* c, cond_t* cd) {
  cd->n = 0;
  if (t->n_skip > 0) {
    for (int j = 0; c->Rskips && j < t->n_skip; ++j) {
      cd->src[cd->n] = t->skip_srcs[j];
      cd->R[cd->n] = c->Rskips + (size_t)j * t->L * c->n_strat * c->n_strat;
      cd->kv[cd->n++] = -1;
    }
  } else if (t->skip_src >= 0 && c->Rskip) {
    cd->src[0] = t->skip_src;
    cd->R[0] = c->Rskip;
    cd->kv[0] = -1;
    cd->n = 1;
  }
}
/* number of copies of a stage [a, b]: |S| per source inside it with an edge inside it */
static int n_copies(const cond_t* base, int a, int b, int S) {
  int n = 1;
  for (int j = 0; j < base->n; ++j)
    if (a <= base->src[j] && base->src[j] + 2 <= b) n *= S;
  return n;
}
/* copy ci of the stage [a, b] (mixed radix over its conditioned sources) */
static cond_t copy_of(const cond_t* base, int a, int b, int S, int ci) {
  cond_t cd = *base;
  for (int j = 0; j < base->n; ++j) {
    cd.kv[j] = -1;
    if (a <= base->src[j] && base->src[j] + 2 <= b) {
      cd.kv[j] = ci % S;
      ci /= S;
    }
  }
  return cd;
}

static int64_t A_cond(const orc_tables* t, const orc_cfg* c, int u, int k, const cond_t* ks) {
  int S = c->n_strat;
  int64_t a = c->A[u * S + k];
  for (int j = 0; j < ks->n; ++j)
    if (ks->kv[j] >= 0 && u >= ks->src[j] + 2) a += ks->R[j][((size_t)u * S + ks->kv[j]) * S + k];
  (void)t;
  return a;
}
/* Strategy k of layer u is allowed: memory entry within the cap (Eq. 5 with
 * the forbidden sentinel), and layer s fixed to ks when conditioning. */
static int allowed(const orc_tables* t, const orc_cfg* c, int u, int k, const cond_t* ks) {
  if (c->M[u * c->n_strat + k] > t->cap) return 0;
  for (int j = 0; j < ks->n; ++j)
    if (ks->kv[j] >= 0 && u == ks->src[j] && k != ks->kv[j]) return 0;
  return 1;
}
static int32_t Rchain(const orc_cfg* c, int u, int k, int l) { /* edge u -> u+1 */
  int S = c->n_strat;
  return c->R[((size_t)u * S + k) * S + l];
}
static int64_t Ocut(const orc_cfg* c, int e) { return c->O ? c->O[e] : 0; }

/* ======================================================================== */
/* Interval table: the stage optimum of Eq. (3) under Eq. (5)               */
/* ======================================================================== */
/* For a fixed start layer a and skip conditioning ks (-1 = none), the
 * textbook forward chain DP over (layer, strategy, memory):
 *   D[a][k][q] = A'_ak                                   if M_ak <= q
 *   D[u][k][q] = A'_uk + min_k' ( D[u-1][k'][q-M_uk] + R_{u-1,u}[k'][k] )
 *                                                         if M_uk <= q
 * (INF otherwise), so D[u][k][q] is the minimum of Eq. (3)'s p over layers
 * a..u with layer u on strategy k and memory sum (Eq. 5) at most q.
 * Row b of the result is  min_k D[b][k][cap]. */
static void interval_row(const orc_tables* t, const orc_cfg* c, int a, const cond_t* ks, int64_t* row) {
  int L = t->L, S = c->n_strat, Q = t->cap + 1;
  int64_t* Dp = (int64_t*)malloc(sizeof(int64_t) * (size_t)S * Q);
  int64_t* Dc = (int64_t*)malloc(sizeof(int64_t) * (size_t)S * Q);
  for (int k = 0; k < S; ++k)
    for (int q = 0; q < Q; ++q)
      Dc[(size_t)k * Q + q] = (allowed(t, c, a, k, ks) && c->M[a * S + k] <= q) ? A_cond(t, c, a, k, ks) : INF;
  for (int u = a;; ++u) {
    int64_t best = INF;
    for (int k = 0; k < S; ++k) best = min64(best, Dc[(size_t)k * Q + t->cap]);
    row[u] = best;
    if (u + 1 >= L) break;
    int64_t* tmp = Dp; Dp = Dc; Dc = tmp;
    int v = u + 1;
    for (int k = 0; k < S; ++k) {
      int64_t* out = Dc + (size_t)k * Q;
      for (int q = 0; q < Q; ++q) out[q] = INF;
      if (!allowed(t, c, v, k, ks)) continue;
      int m = c->M[v * S + k];
      int64_t av = A_cond(t, c, v, k, ks);
      /* min over k' of D[u][k'][q-m] + R[k'][k]  (same min, k' outermost) */
      for (int kp = 0; kp < S; ++kp) {
        int64_t r = Rchain(c, u, kp, k);
        const int64_t* in = Dp + (size_t)kp * Q;
        for (int q = m; q < Q; ++q) {
          int64_t x = in[q - m] + r;
          if (x < out[q]) out[q] = x;
        }
      }
      for (int q = m; q < Q; ++q) out[q] = out[q] >= INF ? INF : out[q] + av;
    }
  }
  free(Dp);
  free(Dc);
}

/* P[a][b] for all a <= b.  When the skip source s lies in [a, b) the stage
 * also pays the skip edges <s,v> with v <= b (Eq. 3 sums every edge with both
 * ends in the stage), which couples layer s's strategy with later layers: the
 * minimum is taken over the conditioning ks of layer s (SURVEY.md Sec. 8c C-2
 * step 2). */
static void interval_table(const orc_tables* t, const orc_cfg* c, int64_t* P) {
  int L = t->L, S = c->n_strat;
  cond_t base;
  skip_sources(t, c, &base);
  int64_t* row = (int64_t*)malloc(sizeof(int64_t) * L);
  for (int i = 0; i < L * L; ++i) P[i] = INF;
  for (int a = 0; a < L; ++a) {
    /* the copies of the longest row: every source in [a, L-1] with an edge in it */
    const int nc = n_copies(&base, a, L - 1, S);
    for (int ci = 0; ci < nc; ++ci) {
      const cond_t ks = copy_of(&base, a, L - 1, S, ci);
      interval_row(t, c, a, &ks, row);
      for (int b = a; b < L; ++b) P[a * L + b] = min64(P[a * L + b], row[b]);
    }
  }
  free(row);
}

/* ======================================================================== */
/* Combine: Eq. (2) over ordered contiguous placements (Pareto-suffix DP)   */
/* ======================================================================== */
/* Set(i, a) = the non-dominated pairs (Sigma, mx) over ways to cover layers
 * [a, L-1] with stages i..deg, where Sigma = sum of their p and of the o of
 * their cuts and mx = max of those p and o.  Eq. (2) is
 *   tpi = Sigma + (c-1) * mx,
 * non-decreasing in both, so dominated pairs never matter. */
typedef struct { int64_t sig, mx; } pair_t;
typedef struct { pair_t* v; int n; } pset;

static int pair_cmp(const void* x, const void* y) {
  const pair_t *p = (const pair_t*)x, *q = (const pair_t*)y;
  if (p->sig != q->sig) return p->sig < q->sig ? -1 : 1;
  if (p->mx != q->mx) return p->mx < q->mx ? -1 : 1;
  return 0;
}
static void pareto(pset* s) {
  qsort(s->v, s->n, sizeof(pair_t), pair_cmp);
  int w = 0;
  for (int r = 0; r < s->n; ++r)
    if (w == 0 || s->v[r].mx < s->v[w - 1].mx) s->v[w++] = s->v[r];
  s->n = w;
}

typedef struct {
  int64_t obj;             /* INF if infeasible */
  int32_t end[ORC_MAX_L];  /* last layer of stage i */
  int32_t strat[ORC_MAX_L];
  int64_t p[ORC_MAX_L], o[ORC_MAX_L];
  int32_t mem[ORC_MAX_L];
  int status;
} cfg_sol;

/* value of Eq. (2) for a prefix (sig0,mx0) + stage (pa,ob) + suffix pair */
static int64_t tpi(int64_t sig, int64_t mx, int c) { return sig + (int64_t)(c - 1) * mx; }

/* ======================================================================== */
/* Strategies of one stage: lexicographically smallest optimal vector      */
/* ======================================================================== */
/* Backward DP G[u][k][q] = min cost of layers u..b given layer u on k and
 * memory at most q for u..b; then walk forward taking the smallest k that
 * still reaches the stage optimum (reading A-11). Returns 1 if found. */
static int stage_walk(const orc_tables* t, const orc_cfg* c, int a, int b, const cond_t* ks, int64_t target,
                      int32_t* out) {
  int S = c->n_strat, Q = t->cap + 1, n = b - a + 1;
  int64_t* G = (int64_t*)malloc(sizeof(int64_t) * (size_t)n * S * Q);
#define GI(u, k, q) G[(((size_t)((u) - a) * S) + (k)) * Q + (q)]
  for (int u = b; u >= a; --u)
    for (int k = 0; k < S; ++k)
      for (int q = 0; q < Q; ++q) {
        int m = c->M[u * S + k];
        int64_t v = INF;
        if (allowed(t, c, u, k, ks) && m <= q) {
          if (u == b) v = A_cond(t, c, u, k, ks);
          else {
            int64_t best = INF;
            for (int k2 = 0; k2 < S; ++k2) best = min64(best, add_sat(Rchain(c, u, k, k2), GI(u + 1, k2, q - m)));
            v = add_sat(best, A_cond(t, c, u, k, ks));
          }
        }
        GI(u, k, q) = v;
      }
  int64_t rem = target;
  int q = t->cap, found = 1, kprev = -1;
  for (int u = a; u <= b && found; ++u) {
    found = 0;
    for (int k = 0; k < S; ++k) {
      int64_t edge = (u > a) ? Rchain(c, u - 1, kprev, k) : 0;
      if (GI(u, k, q) < INF && edge + GI(u, k, q) == rem) {
        out[u] = k;
        rem -= edge + A_cond(t, c, u, k, ks);
        q -= c->M[u * S + k];
        kprev = k;
        found = 1;
        break;
      }
    }
  }
#undef GI
  free(G);
  return found;
}

static void stage_strategies(const orc_tables* t, const orc_cfg* c, int a, int b, int64_t target,
                             int32_t* strat) {
  int S = c->n_strat;
  cond_t base;
  skip_sources(t, c, &base);
  const int nc = n_copies(&base, a, b, S);
  if (nc == 1) {
    const cond_t ks = copy_of(&base, a, b, S, 0);
    stage_walk(t, c, a, b, &ks, target, strat);
    return;
  }
  int32_t best[ORC_MAX_L], cur[ORC_MAX_L];
  int have = 0;
  for (int ci = 0; ci < nc; ++ci) {
    const cond_t ks = copy_of(&base, a, b, S, ci);
    if (!stage_walk(t, c, a, b, &ks, target, cur)) continue;
    int less = !have;
    for (int u = a; u <= b && !less; ++u) {
      if (cur[u] != best[u]) { less = cur[u] < best[u]; break; }
    }
    if (less) { memcpy(best + a, cur + a, sizeof(int32_t) * (b - a + 1)); have = 1; }
  }
  memcpy(strat + a, best + a, sizeof(int32_t) * (b - a + 1));
}

/* ======================================================================== */
/* One candidate config: the MIQP of Sec. 3.3 solved exactly                */
/* ======================================================================== */
/* Memory cap of stage i (0-based): Eq. (5) with the stage's own m_i when the
 * devices are heterogeneous, else the common cap. */
static int stage_cap(const orc_tables* t, const orc_cfg* c, int i) { return c->stage_cap ? c->stage_cap[i] : t->cap; }
/* Memory table of stage i (0-based): the schedule's own table when the
 * memory of a layer depends on its stage (synchronous 1F1B: stage i holds
 * min(c, deg - i) micro-batches in flight, the footnote of PAPER.md:122;
 * reading A-32), else M. */
static const int32_t* stage_M(const orc_tables* t, const orc_cfg* c, int i) {
  return c->M_stage ? c->M_stage + (size_t)i * t->L * c->n_strat : c->M;
}
/* stage i's view of the config: the tables with M = its memory table */
static orc_cfg stage_view(const orc_tables* t, const orc_cfg* c, int i) {
  orc_cfg ci = *c;
  ci.M = stage_M(t, c, i);
  return ci;
}

static void solve_cfg(const orc_tables* t, const orc_cfg* c, cfg_sol* sol) {
  int L = t->L, deg = c->deg;
  sol->obj = INF;
  sol->status = ORC_OK;
  if (deg > L) return; /* Eq. (7b) cannot hold (reading A-22) */
  /* P_i[a][b]: the stage optimum of [a,b] under stage i's cap -- the
   * interval table of the same tables with cap = cap_i, per stage index */
  int64_t* Pall = (int64_t*)malloc(sizeof(int64_t) * (size_t)deg * L * L);
  const size_t mw = sizeof(int32_t) * (size_t)L * c->n_strat;
  for (int i = 0; i < deg; ++i) {
    int j = 0;
    while (j < i && (stage_cap(t, c, j) != stage_cap(t, c, i) || memcmp(stage_M(t, c, j), stage_M(t, c, i), mw))) ++j;
    if (j < i) { memcpy(Pall + (size_t)i * L * L, Pall + (size_t)j * L * L, sizeof(int64_t) * L * L); continue; }
    orc_tables ti = *t;
    ti.cap = stage_cap(t, c, i);
    orc_cfg ci = stage_view(t, c, i);
    interval_table(&ti, &ci, Pall + (size_t)i * L * L);
  }
#define PI(i, a, b) Pall[((size_t)((i) - 1) * L + (a)) * L + (b)] /* stage i = 1..deg */
  /* Set(i,a), i = 1..deg (index i-1), a = 0..L-1 */
  pset* sets = (pset*)calloc((size_t)deg * L, sizeof(pset));
#define SET(i, a) sets[(size_t)((i) - 1) * L + (a)]
  for (int a = 0; a < L; ++a) {
    pset* s = &SET(deg, a);
    if (PI(deg, a, L - 1) < INF) {
      s->v = (pair_t*)malloc(sizeof(pair_t));
      s->v[0].sig = PI(deg, a, L - 1);
      s->v[0].mx = PI(deg, a, L - 1);
      s->n = 1;
    }
  }
  for (int i = deg - 1; i >= 1; --i)
    for (int a = 0; a < L; ++a) {
      int cnt = 0;
      for (int b = a; b + 1 < L; ++b) if (PI(i, a, b) < INF) cnt += SET(i + 1, b + 1).n;
      pset* s = &SET(i, a);
      if (!cnt) continue;
      s->v = (pair_t*)malloc(sizeof(pair_t) * cnt);
      for (int b = a; b + 1 < L; ++b) {
        int64_t p = PI(i, a, b);
        if (p >= INF) continue;
        int64_t o = Ocut(c, b);
        const pset* nx = &SET(i + 1, b + 1);
        for (int j = 0; j < nx->n; ++j) {
          s->v[s->n].sig = p + o + nx->v[j].sig;
          s->v[s->n].mx = max64(max64(p, o), nx->v[j].mx);
          s->n++;
        }
      }
      pareto(s);
    }
  int64_t opt = INF;
  for (int j = 0; j < SET(1, 0).n; ++j) opt = min64(opt, tpi(SET(1, 0).v[j].sig, SET(1, 0).v[j].mx, c->c));
  sol->obj = opt;
  if (opt < INF) {
    /* Stage ends: the lexicographically smallest stage_of is the largest
     * feasible end for each stage in turn (reading A-11). */
    int64_t sig = 0, mx = 0;
    int a = 0;
    for (int i = 1; i < deg; ++i) {
      int chosen = -1;
      for (int b = L - 2; b >= a && chosen < 0; --b) {
        int64_t p = PI(i, a, b);
        if (p >= INF) continue;
        int64_t o = Ocut(c, b);
        const pset* nx = &SET(i + 1, b + 1);
        for (int j = 0; j < nx->n; ++j)
          if (tpi(sig + p + o + nx->v[j].sig, max64(max64(mx, max64(p, o)), nx->v[j].mx), c->c) == opt) {
            chosen = b;
            break;
          }
      }
      if (chosen < 0) { sol->status = ORC_ERR_INTERNAL; break; }
      int64_t p = PI(i, a, chosen), o = Ocut(c, chosen);
      sig += p + o;
      mx = max64(mx, max64(p, o));
      sol->end[i - 1] = chosen;
      sol->p[i - 1] = p;
      sol->o[i - 1] = o;
      a = chosen + 1;
    }
    sol->end[deg - 1] = L - 1;
    sol->p[deg - 1] = PI(deg, a, L - 1);
    /* strategies per stage, under the stage's own cap and memory table */
    int start = 0;
    for (int i = 0; i < deg && sol->status == ORC_OK; ++i) {
      orc_tables ti = *t;
      ti.cap = stage_cap(t, c, i);
      orc_cfg ci = stage_view(t, c, i);
      stage_strategies(&ti, &ci, start, sol->end[i], sol->p[i], sol->strat);
      start = sol->end[i] + 1;
    }
  }
  for (int i = 0; i < deg * L; ++i) free(sets[i].v);
#undef SET
#undef PI
  free(sets);
  free(Pall);
}

/* Literal re-evaluation of Eqs. (2), (3), (5) from (stage_of, strategy_of). */
static int check_solution(const orc_tables* t, const orc_cfg* c, cfg_sol* sol) {
  int L = t->L, S = c->n_strat, deg = c->deg;
  cond_t sk;
  skip_sources(t, c, &sk);
  int start = 0;
  int64_t sum = 0, mx = 0;
  for (int i = 0; i < deg; ++i) {
    int b = sol->end[i];
    if (b < start) return ORC_ERR_INTERNAL;
    int64_t p = 0, mem = 0;
    for (int u = start; u <= b; ++u) {
      int k = sol->strat[u];
      if (k < 0 || k >= S) return ORC_ERR_INTERNAL;
      p += c->A[u * S + k];
      mem += stage_M(t, c, i)[u * S + k];
      if (u < b) p += Rchain(c, u, k, sol->strat[u + 1]);
      for (int j = 0; j < sk.n; ++j) /* every skip edge <s_j, u> with both ends in the stage (Eq. 3) */
        if (start <= sk.src[j] && u >= sk.src[j] + 2) p += sk.R[j][((size_t)u * S + sol->strat[sk.src[j]]) * S + k];
    }
    if (mem > stage_cap(t, c, i) || p != sol->p[i]) return ORC_ERR_INTERNAL;
    sol->mem[i] = (int32_t)mem;
    sum += p;
    mx = max64(mx, p);
    if (i + 1 < deg) {
      int64_t o = Ocut(c, b) + (c->Rcut ? c->Rcut[((size_t)b * S + sol->strat[b]) * S + sol->strat[b + 1]] : 0);
      if (o != sol->o[i]) return ORC_ERR_INTERNAL;
      sum += o;
      mx = max64(mx, o);
    }
    start = b + 1;
  }
  if (start != L) return ORC_ERR_INTERNAL;
  if (tpi(sum, mx, c->c) != sol->obj) return ORC_ERR_INTERNAL;
  return ORC_OK;
}

/* ======================================================================== */
/* NEXT-1: strategy-dependent cross-stage cost (Eq. 4 with R' per strategy) */
/* ======================================================================== */
/* o_j = O[e_j] + Rcut[e_j][k_{e_j}][k_{e_j + 1}]: Eq. (4) sums S_u^T R'_uv S_v
 * over the edges from stage j to stage j+1; for the chain
 * edge e_j -> e_j + 1 that is Rcut, the edges skipping past the cut keep the
 * scalar part O (reading A-16).  The stage optimum now depends on the
 * strategies at the stage's two ends, so the interval table grows to
 * T[a][b][kf][kl]: the minimum of Eq. (3) over [a,b] under Eq. (5) with layer
 * a on kf and layer b on kl. */
static int32_t Rc(const orc_cfg* c, int e, int k, int l) {
  int S = c->n_strat;
  return c->Rcut[((size_t)e * S + k) * S + l];
}
static int64_t ocut(const orc_cfg* c, int e, int kl, int kf) { return Ocut(c, e) + Rc(c, e, kl, kf); }

/* Strategy k allowed at layer u with the start layer a restricted to kf. */
static int allowed_f(const orc_tables* t, const orc_cfg* c, int u, int k, const cond_t* ks, int a, int kf) {
  if (!allowed(t, c, u, k, ks)) return 0;
  if (kf >= 0 && u == a && k != kf) return 0;
  return 1;
}

/* The textbook forward DP of interval_row with the start layer on kf:
 * rowk[b][kl] = min cost of [a,b] with layer b on kl (INF if infeasible). */
static void interval_row_k(const orc_tables* t, const orc_cfg* c, int a, const cond_t* ks, int kf, int64_t* rowk) {
  int L = t->L, S = c->n_strat, Q = t->cap + 1;
  int64_t* Dp = (int64_t*)malloc(sizeof(int64_t) * (size_t)S * Q);
  int64_t* Dc = (int64_t*)malloc(sizeof(int64_t) * (size_t)S * Q);
  for (int k = 0; k < S; ++k)
    for (int q = 0; q < Q; ++q)
      Dc[(size_t)k * Q + q] = (allowed_f(t, c, a, k, ks, a, kf) && c->M[a * S + k] <= q) ? A_cond(t, c, a, k, ks) : INF;
  for (int u = a;; ++u) {
    for (int k = 0; k < S; ++k) rowk[(size_t)u * S + k] = Dc[(size_t)k * Q + t->cap];
    if (u + 1 >= L) break;
    int64_t* tmp = Dp; Dp = Dc; Dc = tmp;
    int v = u + 1;
    for (int k = 0; k < S; ++k) {
      int64_t* out = Dc + (size_t)k * Q;
      for (int q = 0; q < Q; ++q) out[q] = INF;
      if (!allowed_f(t, c, v, k, ks, a, kf)) continue;
      int m = c->M[v * S + k];
      int64_t av = A_cond(t, c, v, k, ks);
      for (int kp = 0; kp < S; ++kp) {
        int64_t r = Rchain(c, u, kp, k);
        const int64_t* in = Dp + (size_t)kp * Q;
        for (int q = m; q < Q; ++q) {
          int64_t x = in[q - m] + r;
          if (x < out[q]) out[q] = x;
        }
      }
      for (int q = m; q < Q; ++q) out[q] = out[q] >= INF ? INF : out[q] + av;
    }
  }
  free(Dp);
  free(Dc);
}

/* T[((a*L + b)*S + kf)*S + kl] for every a <= b (min over the skip
 * conditioning ks when the stage holds the skip source and one of its edges). */
static void cut_tables(const orc_tables* t, const orc_cfg* c, int64_t* T) {
  int L = t->L, S = c->n_strat;
  cond_t base;
  skip_sources(t, c, &base);
  size_t n = (size_t)L * L * S * S;
  for (size_t i = 0; i < n; ++i) T[i] = INF;
  int64_t* rowk = (int64_t*)malloc(sizeof(int64_t) * (size_t)L * S);
  for (int a = 0; a < L; ++a)
    for (int kf = 0; kf < S; ++kf) {
      const int nc = n_copies(&base, a, L - 1, S);
      for (int ci = 0; ci < nc; ++ci) {
        const cond_t ks = copy_of(&base, a, L - 1, S, ci);
        interval_row_k(t, c, a, &ks, kf, rowk);
        for (int b = a; b < L; ++b)
          for (int kl = 0; kl < S; ++kl) {
            int64_t* d = &T[(((size_t)a * L + b) * S + kf) * S + kl];
            *d = min64(*d, rowk[(size_t)b * S + kl]);
          }
      }
    }
  free(rowk);
}
#define TT(a, b, kf, kl) T[((((size_t)(a)) * L + (b)) * S + (kf)) * S + (kl)]

static void pset_add(pset* p, int64_t sig, int64_t mx, int* cap) {
  if (p->n == *cap) {
    *cap = *cap ? 2 * *cap : 16;
    p->v = (pair_t*)realloc(p->v, sizeof(pair_t) * (size_t)*cap);
  }
  p->v[p->n].sig = sig;
  p->v[p->n].mx = mx;
  p->n++;
}
/* exists (s2, m2) in set with sig + s2 + (c-1) max(mx, m2) == opt */
static int pset_hits(const pset* p, int64_t sig, int64_t mx, int c, int64_t opt) {
  for (int j = 0; j < p->n; ++j)
    if (tpi(sig + p->v[j].sig, max64(mx, p->v[j].mx), c) == opt) return 1;
  return 0;
}

/* Backward DP of stage_walk with the first layer restricted to kf and the
 * last to kl (-1: free): the lexicographically smallest strategy vector of
 * [a,b] reaching `target` (reading A-11 within the stage). */
static int stage_walk_fl(const orc_tables* t, const orc_cfg* c, int a, int b, const cond_t* ks, int kf, int kl, int64_t target,
                         int32_t* out) {
  int S = c->n_strat, Q = t->cap + 1, n = b - a + 1;
  int64_t* G = (int64_t*)malloc(sizeof(int64_t) * (size_t)n * S * Q);
#define GI(u, k, q) G[(((size_t)((u) - a) * S) + (k)) * Q + (q)]
  for (int u = b; u >= a; --u)
    for (int k = 0; k < S; ++k)
      for (int q = 0; q < Q; ++q) {
        int m = c->M[u * S + k];
        int64_t v = INF;
        int ok = allowed_f(t, c, u, k, ks, a, kf) && !(kl >= 0 && u == b && k != kl);
        if (ok && m <= q) {
          if (u == b) v = A_cond(t, c, u, k, ks);
          else {
            int64_t best = INF;
            for (int k2 = 0; k2 < S; ++k2) best = min64(best, add_sat(Rchain(c, u, k, k2), GI(u + 1, k2, q - m)));
            v = add_sat(best, A_cond(t, c, u, k, ks));
          }
        }
        GI(u, k, q) = v;
      }
  int64_t rem = target;
  int q = t->cap, found = 1, kprev = -1;
  for (int u = a; u <= b && found; ++u) {
    found = 0;
    for (int k = 0; k < S; ++k) {
      int64_t edge = (u > a) ? Rchain(c, u - 1, kprev, k) : 0;
      if (GI(u, k, q) < INF && edge + GI(u, k, q) == rem) {
        out[u] = k;
        rem -= edge + A_cond(t, c, u, k, ks);
        q -= c->M[u * S + k];
        kprev = k;
        found = 1;
        break;
      }
    }
  }
#undef GI
  free(G);
  return found;
}

static int stage_strategies_fl(const orc_tables* t, const orc_cfg* c, int a, int b, int kf, int kl, int64_t target,
                               int32_t* strat) {
  int S = c->n_strat;
  cond_t base;
  skip_sources(t, c, &base);
  const int nc = n_copies(&base, a, b, S);
  int32_t best[ORC_MAX_L], cur[ORC_MAX_L];
  int have = 0;
  for (int ci = 0; ci < nc; ++ci) {
    const cond_t ks = copy_of(&base, a, b, S, ci);
    if (!stage_walk_fl(t, c, a, b, &ks, kf, kl, target, cur)) continue;
    int less = !have;
    for (int u = a; u <= b && !less; ++u)
      if (cur[u] != best[u]) { less = cur[u] < best[u]; break; }
    if (less) { memcpy(best + a, cur + a, sizeof(int32_t) * (b - a + 1)); have = 1; }
  }
  if (have) memcpy(strat + a, best + a, sizeof(int32_t) * (b - a + 1));
  return have;
}

/* One candidate config with strategy-dependent cut costs, solved exactly:
 * Pareto sets Set(i, a, kf) of (sigma, mx) over ways to cover [a, L-1] with
 * stages i..deg when stage i starts at a on strategy kf; Eq. (2) from
 * Set(1, 0, *).  Then the tie-break of reading A-31: the largest feasible end
 * of each stage in turn (lexicographically smallest stage_of), then the
 * boundary strategies (k_{e_1}, k_{e_1 + 1}, ...) smallest first, then the
 * lexicographically smallest strategies inside each stage. */
static void solve_cfg_cut(const orc_tables* t, const orc_cfg* c, cfg_sol* sol) {
  int L = t->L, deg = c->deg, S = c->n_strat, cc = c->c;
  sol->obj = INF;
  sol->status = ORC_OK;
  if (deg > L) return;
  int64_t* T = (int64_t*)malloc(sizeof(int64_t) * (size_t)L * L * S * S);
  cut_tables(t, c, T);
  /* Set(i, a, kf): index ((i-1)*L + a)*S + kf */
  size_t nsets = (size_t)deg * L * S;
  pset* sets = (pset*)calloc(nsets, sizeof(pset));
#define SETF(i, a, kf) sets[(((size_t)((i) - 1) * L) + (a)) * S + (kf)]
  for (int a = 0; a < L; ++a)
    for (int kf = 0; kf < S; ++kf) {
      int64_t v = INF;
      for (int kl = 0; kl < S; ++kl) v = min64(v, TT(a, L - 1, kf, kl));
      if (v < INF) {
        int capn = 0;
        pset_add(&SETF(deg, a, kf), v, v, &capn);
      }
    }
  for (int i = deg - 1; i >= 1; --i)
    for (int a = 0; a < L; ++a)
      for (int kf = 0; kf < S; ++kf) {
        pset* ps = &SETF(i, a, kf);
        int capn = 0;
        for (int b = a; b + 1 < L; ++b)
          for (int kl = 0; kl < S; ++kl) {
            int64_t p = TT(a, b, kf, kl);
            if (p >= INF) continue;
            for (int kf2 = 0; kf2 < S; ++kf2) {
              const pset* nx = &SETF(i + 1, b + 1, kf2);
              int64_t o = ocut(c, b, kl, kf2);
              for (int j = 0; j < nx->n; ++j)
                pset_add(ps, p + o + nx->v[j].sig, max64(max64(p, o), nx->v[j].mx), &capn);
            }
          }
        if (ps->n) pareto(ps);
      }
  int64_t opt = INF;
  for (int kf = 0; kf < S; ++kf)
    for (int j = 0; j < SETF(1, 0, kf).n; ++j) opt = min64(opt, tpi(SETF(1, 0, kf).v[j].sig, SETF(1, 0, kf).v[j].mx, cc));
  sol->obj = opt;
  if (opt < INF) {
    /* (a) stage ends: prefix Pareto sets per last strategy of the fixed stages */
    pset pre[ORC_MAX_S], nxt[ORC_MAX_S];
    int precap[ORC_MAX_S], nxtcap[ORC_MAX_S];
    memset(pre, 0, sizeof pre);
    memset(nxt, 0, sizeof nxt);
    memset(precap, 0, sizeof precap);
    memset(nxtcap, 0, sizeof nxtcap);
    int a = 0;
    for (int i = 1; i <= deg && sol->status == ORC_OK; ++i) {
      int chosen = -1;
      int blo = (i == deg) ? L - 1 : a, bhi = (i == deg) ? L - 1 : L - 2;
      for (int b = bhi; b >= blo && chosen < 0; --b) {
        int hit = 0;
        for (int kf = 0; kf < S && !hit; ++kf)
          for (int kl = 0; kl < S && !hit; ++kl) {
            int64_t p = TT(a, b, kf, kl);
            if (p >= INF) continue;
            /* prefix pairs with the incoming cut (stage 1: none) */
            for (int kp = 0; kp < (i == 1 ? 1 : S) && !hit; ++kp) {
              const pset* pp = (i == 1) ? NULL : &pre[kp];
              int np = (i == 1) ? 1 : pp->n;
              for (int x = 0; x < np && !hit; ++x) {
                int64_t s0 = (i == 1) ? 0 : pp->v[x].sig, m0 = (i == 1) ? 0 : pp->v[x].mx;
                int64_t oin = (i == 1) ? 0 : ocut(c, a - 1, kp, kf);
                int64_t sg = s0 + oin + p, mx = max64(max64(m0, oin), p);
                if (i == deg) hit = tpi(sg, mx, cc) == opt;
                else
                  for (int kf2 = 0; kf2 < S && !hit; ++kf2) {
                    int64_t o = ocut(c, b, kl, kf2);
                    hit = pset_hits(&SETF(i + 1, b + 1, kf2), sg + o, max64(mx, o), cc, opt);
                  }
              }
            }
          }
        if (hit) chosen = b;
      }
      if (chosen < 0) { sol->status = ORC_ERR_INTERNAL; break; }
      sol->end[i - 1] = chosen;
      /* the prefix sets through stage i, per its last strategy */
      for (int kl = 0; kl < S; ++kl) nxt[kl].n = 0;
      for (int kf = 0; kf < S; ++kf)
        for (int kl = 0; kl < S; ++kl) {
          int64_t p = TT(a, chosen, kf, kl);
          if (p >= INF) continue;
          for (int kp = 0; kp < (i == 1 ? 1 : S); ++kp) {
            int np = (i == 1) ? 1 : pre[kp].n;
            for (int x = 0; x < np; ++x) {
              int64_t s0 = (i == 1) ? 0 : pre[kp].v[x].sig, m0 = (i == 1) ? 0 : pre[kp].v[x].mx;
              int64_t oin = (i == 1) ? 0 : ocut(c, a - 1, kp, kf);
              pset_add(&nxt[kl], s0 + oin + p, max64(max64(m0, oin), p), &nxtcap[kl]);
            }
          }
        }
      for (int kl = 0; kl < S; ++kl) {
        if (nxt[kl].n) pareto(&nxt[kl]);
        pset tmp = pre[kl]; pre[kl] = nxt[kl]; nxt[kl] = tmp;
        int tc = precap[kl]; precap[kl] = nxtcap[kl]; nxtcap[kl] = tc;
      }
      a = chosen + 1;
    }
    for (int k = 0; k < S; ++k) { free(pre[k].v); free(nxt[k].v); }
    /* (b) boundary strategies with the ends fixed: suffix sets SE(i, kf) of
     * stages i..deg (stage i first on kf, later boundaries free), then the
     * greedy (kl_1, kf_2, kl_2, ...) smallest first */
    int32_t kfs[ORC_MAX_L], kls[ORC_MAX_L];
    int st[ORC_MAX_L + 1];
    st[0] = 0;
    for (int i = 1; i < deg; ++i) st[i] = sol->end[i - 1] + 1;
    pset* SE = (pset*)calloc((size_t)(deg + 1) * S, sizeof(pset));
#define SEF(i, kf) SE[(size_t)(i) * S + (kf)]
    for (int i = deg; i >= 1 && sol->status == ORC_OK; --i) {
      int a0 = st[i - 1], b0 = sol->end[i - 1];
      for (int kf = 0; kf < S; ++kf) {
        pset* ps = &SEF(i, kf);
        int capn = 0;
        if (i == deg) {
          int64_t v = INF;
          for (int kl = 0; kl < S; ++kl) v = min64(v, TT(a0, b0, kf, kl));
          if (v < INF) pset_add(ps, v, v, &capn);
        } else {
          for (int kl = 0; kl < S; ++kl) {
            int64_t p = TT(a0, b0, kf, kl);
            if (p >= INF) continue;
            for (int kf2 = 0; kf2 < S; ++kf2) {
              int64_t o = ocut(c, b0, kl, kf2);
              const pset* nx = &SEF(i + 1, kf2);
              for (int j = 0; j < nx->n; ++j)
                pset_add(ps, p + o + nx->v[j].sig, max64(max64(p, o), nx->v[j].mx), &capn);
            }
          }
          if (ps->n) pareto(ps);
        }
      }
    }
    /* prefix state: Pareto set of the fixed stages 1..j (stage 1's first
     * strategy free), ending on kls[j-1] */
    pset cur = {0}, nw = {0};
    int curcap = 0, nwcap = 0;
    for (int j = 1; j < deg && sol->status == ORC_OK; ++j) {
      int a0 = st[j - 1], b0 = sol->end[j - 1];
      /* candidates of stage j's pairs given its first strategy (fixed for j > 1) */
      int chosen_kl = -1, chosen_kf = -1;
      for (int kl = 0; kl < S && chosen_kl < 0; ++kl) {
        nw.n = 0;
        for (int kf = 0; kf < S; ++kf) {
          if (j > 1 && kf != kfs[j - 1]) continue;
          int64_t p = TT(a0, b0, kf, kl);
          if (p >= INF) continue;
          int np = (j == 1) ? 1 : cur.n;
          for (int x = 0; x < np; ++x) {
            int64_t s0 = (j == 1) ? 0 : cur.v[x].sig, m0 = (j == 1) ? 0 : cur.v[x].mx;
            pset_add(&nw, s0 + p, max64(m0, p), &nwcap);
          }
        }
        for (int x = 0; x < nw.n && chosen_kl < 0; ++x)
          for (int kf2 = 0; kf2 < S && chosen_kl < 0; ++kf2) {
            int64_t o = ocut(c, b0, kl, kf2);
            if (pset_hits(&SEF(j + 1, kf2), nw.v[x].sig + o, max64(nw.v[x].mx, o), cc, opt)) chosen_kl = kl;
          }
      }
      if (chosen_kl < 0) { sol->status = ORC_ERR_INTERNAL; break; }
      /* nw holds stage j's prefix pairs ending on chosen_kl (the loop broke on it) */
      for (int kf2 = 0; kf2 < S && chosen_kf < 0; ++kf2) {
        int64_t o = ocut(c, b0, chosen_kl, kf2);
        for (int x = 0; x < nw.n && chosen_kf < 0; ++x)
          if (pset_hits(&SEF(j + 1, kf2), nw.v[x].sig + o, max64(nw.v[x].mx, o), cc, opt)) chosen_kf = kf2;
      }
      if (chosen_kf < 0) { sol->status = ORC_ERR_INTERNAL; break; }
      kls[j - 1] = chosen_kl;
      kfs[j] = chosen_kf;
      /* prefix through the cut into stage j+1 (its own cost added next round) */
      int64_t o = ocut(c, b0, chosen_kl, chosen_kf);
      cur.n = 0;
      for (int x = 0; x < nw.n; ++x) pset_add(&cur, nw.v[x].sig + o, max64(nw.v[x].mx, o), &curcap);
      pareto(&cur);
    }
    free(cur.v);
    free(nw.v);
    for (size_t i = 0; i < (size_t)(deg + 1) * S; ++i) free(SE[i].v);
    free(SE);
#undef SEF
    /* (c) strategies inside each stage, with the boundary strategies fixed;
     * p_i = T for fixed ends strategies (minimised over a free first / last) */
    for (int i = 0; i < deg && sol->status == ORC_OK; ++i) {
      int a0 = st[i], b0 = sol->end[i];
      int kf = i > 0 ? kfs[i] : -1, kl = i + 1 < deg ? kls[i] : -1;
      int64_t v = INF;
      for (int x = 0; x < S; ++x)
        for (int y = 0; y < S; ++y)
          if ((kf < 0 || x == kf) && (kl < 0 || y == kl)) v = min64(v, TT(a0, b0, x, y));
      sol->p[i] = v;
      if (i + 1 < deg) sol->o[i] = ocut(c, b0, kls[i], kfs[i + 1]);
      if (v >= INF || !stage_strategies_fl(t, c, a0, b0, kf, kl, v, sol->strat)) sol->status = ORC_ERR_INTERNAL;
    }
  }
  for (size_t i = 0; i < nsets; ++i) free(sets[i].v);
#undef SETF
  free(sets);
  free(T);
}
#undef TT

/* ======================================================================== */
/* Algorithm 1 outer loop over candidates, optionally on host threads       */
/* ======================================================================== */
typedef struct {
  const orc_tables* t;
  cfg_sol* sols;
  int next;
  pthread_mutex_t mu;
} pool_t;

static void* worker(void* arg) {
  pool_t* p = (pool_t*)arg;
  for (;;) {
    pthread_mutex_lock(&p->mu);
    int i = p->next++;
    pthread_mutex_unlock(&p->mu);
    if (i >= p->t->n_cfg) break;
    if (p->t->cfg[i].Rcut) solve_cfg_cut(p->t, &p->t->cfg[i], &p->sols[i]);
    else solve_cfg(p->t, &p->t->cfg[i], &p->sols[i]);
    if (p->sols[i].status == ORC_OK && p->sols[i].obj < INF)
      p->sols[i].status = check_solution(p->t, &p->t->cfg[i], &p->sols[i]);
  }
  return NULL;
}

int orc_solve(const orc_tables* t, int n_threads, orc_result* res, int64_t* cfg_obj) {
  int st = validate_tables(t);
  if (st != ORC_OK) return st;
  cfg_sol* sols = (cfg_sol*)calloc(t->n_cfg, sizeof(cfg_sol));
  pool_t pool = {t, sols, 0, PTHREAD_MUTEX_INITIALIZER};
  if (n_threads <= 0) n_threads = (int)sysconf(_SC_NPROCESSORS_ONLN);
  if (n_threads > t->n_cfg) n_threads = t->n_cfg;
  if (n_threads <= 1) {
    worker(&pool);
  } else {
    pthread_t th[256];
    if (n_threads > 256) n_threads = 256;
    for (int i = 0; i < n_threads; ++i) pthread_create(&th[i], NULL, worker, &pool);
    for (int i = 0; i < n_threads; ++i) pthread_join(th[i], NULL);
  }
  /* ordered minimum by (tpi, deg, c)  (PAPER.md:221 strict '<' over the
   * ascending enumeration; reading A-11) */
  int win = -1;
  for (int i = 0; i < t->n_cfg; ++i) {
    if (sols[i].status != ORC_OK) { st = sols[i].status; break; }
    if (cfg_obj) cfg_obj[i] = sols[i].obj < INF ? sols[i].obj : INT64_MAX;
    if (sols[i].obj >= INF) continue;
    if (win < 0) { win = i; continue; }
    const orc_cfg *x = &t->cfg[i], *w = &t->cfg[win];
    if (sols[i].obj < sols[win].obj ||
        (sols[i].obj == sols[win].obj && (x->deg < w->deg || (x->deg == w->deg && x->c < w->c))))
      win = i;
  }
  memset(res, 0, sizeof(*res));
  res->L = t->L;
  res->objective = INT64_MAX;
  res->cfg_index = -1;
  if (st == ORC_OK && win < 0) st = ORC_ERR_INFEASIBLE;
  if (st == ORC_OK) {
    const cfg_sol* s = &sols[win];
    const orc_cfg* c = &t->cfg[win];
    res->objective = s->obj;
    res->cfg_index = win;
    res->deg = c->deg;
    res->c = c->c;
    int stage = 0;
    for (int u = 0; u < t->L; ++u) {
      while (u > s->end[stage]) ++stage;
      res->stage_of[u] = stage;
      res->strategy_of[u] = s->strat[u];
    }
    for (int i = 0; i < c->deg; ++i) {
      res->stage_cost[i] = s->p[i];
      res->stage_mem[i] = s->mem[i];
      if (i + 1 < c->deg) res->cut_cost[i] = s->o[i];
    }
  }
  free(sols);
  return st;
}

int orc_interval_table(const orc_tables* t, int cfg, int64_t* P) {
  int st = validate_tables(t);
  if (st != ORC_OK) return st;
  if (cfg < 0 || cfg >= t->n_cfg) return ORC_ERR_ARG;
  orc_cfg c0 = stage_view(t, &t->cfg[cfg], 0); /* (stage 1's memory table when stage-indexed) */
  interval_table(t, &c0, P);
  for (int i = 0; i < t->L * t->L; ++i)
    if (P[i] >= INF) P[i] = INT64_MAX;
  return ORC_OK;
}

/* ======================================================================== */
/* Level 2: builder' -- the cost model of Sec. 3.2 in integers              */
/* ======================================================================== */
/* Strategy dictionary SD[deg]: every (TP, FSDP, DP)
 * degree triple (t,f,d) with t*f*d = g, t a profiled TP size (power of two);
 * ordered t ascending then f ascending, so index 0 is pure DP, as in
 * Appendix D's S_{l0}.  Reading A-6. */
int orc_catalogue(int32_t g, int32_t space, int32_t* tfd, int32_t cap) {
  int n = 0;
  if (g < 1) return 0;
  for (int t = 1; t <= g; t *= 2) {
    if (g % t) break;
    for (int f = 1; f <= g / t; ++f) {
      if ((g / t) % f) continue;
      int d = g / t / f;
      /* SPEC's space (StrategySpace): a (dp, tp) pair with the
       * dp axis either plain DP (f = 1) or fully FSDP-sharded (d = 1) */
      if (space == 1 && f != 1 && d != 1) continue;
      if (n < cap) { tfd[3 * n] = t; tfd[3 * n + 1] = f; tfd[3 * n + 2] = d; }
      ++n;
    }
  }
  return n;
}

/* Algorithm 1: first deg = 1 (the QIP of App. C, modelled
 * at batch B, reported as c = 1 -- reading A-4), then every factor deg > 1 of
 * n and every factor c > 1 of B, deg ascending then c ascending. */
int orc_candidates(int32_t n, int32_t B, int32_t* pairs, int32_t cap) {
  int k = 0;
  if (cap > 0) { pairs[0] = 1; pairs[1] = 1; }
  k = 1;
  for (int deg = 2; deg <= n; ++deg) {
    if (n % deg) continue;
    for (int c = 2; c <= B; ++c) {
      if (B % c) continue;
      if (k < cap) { pairs[2 * k] = deg; pairs[2 * k + 1] = c; }
      ++k;
    }
  }
  return k;
}

#define NS_LIMIT ((u128)1 << 62) /* any modelled time / byte count must stay below */

static u128 cdiv(u128 x, u128 y) { return (x + y - 1) / y; }

/* "dividing the size of transmitting tensors by the profiled communication
 * efficiency" with the ring model of SPEC.md:146; the link is
 * the inter-node one when the group's device span (stride * G) exceeds a
 * node (reading: collective bandwidth). */
static int64_t bw_for(const orc_cluster* cl, int64_t G, int64_t stride) {
  return (stride * G > cl->node_size) ? cl->bw_inter : cl->bw_intra;
}
static u128 t_allreduce(const orc_cluster* cl, u128 V, int64_t G, int64_t stride) {
  if (G <= 1) return 0;
  return cdiv((u128)2 * (G - 1) * V * 1000000000u, (u128)G * bw_for(cl, G, stride)) +
         (u128)2 * (G - 1) * cl->lat_ns;
}
static u128 t_allgather(const orc_cluster* cl, u128 V, int64_t G, int64_t stride) {
  if (G <= 1) return 0;
  return cdiv((u128)(G - 1) * V * 1000000000u, (u128)G * bw_for(cl, G, stride)) + (u128)(G - 1) * cl->lat_ns;
}
static u128 t_p2p(const orc_cluster* cl, u128 V) {
  return cdiv(V * 1000000000u, (u128)cl->p2p_bw) + (u128)cl->lat_ns;
}
/* "multiplies the profiled CCOC by the overlapping interval of computation
 * and communication": hidden = floor(ccoc * min / 1000)
 * (reading A-23). */
static u128 t_overlap(u128 comp, u128 comm, int32_t ccoc_permille) {
  u128 mn = comp < comm ? comp : comm;
  return comp + comm - (u128)ccoc_permille * mn / 1000;
}
static int ilog2(int x) { int r = 0; while ((1 << (r + 1)) <= x) ++r; return r; }

/* Resharding between the output layout of strategy (t1,f1,d1) and the input
 * layout of (t2,f2,d2) on a tensor of V bytes: free if the (TP, replica)
 * layouts match, else an all-reduce-shaped exchange over the
 * largest ratio of a differing axis, forward + backward (reading A-15). */
static u128 t_reshard(const orc_cluster* cl, const int32_t* s1, const int32_t* s2, u128 V) {
  int64_t t1 = s1[0], r1 = (int64_t)s1[1] * s1[2], t2 = s2[0], r2 = (int64_t)s2[1] * s2[2];
  if (t1 == t2 && r1 == r2) return 0;
  int64_t G = 1; /* ratio max/min of each differing axis, rounded up */
  if (t1 != t2) G = max64(G, t1 > t2 ? (t1 + t2 - 1) / t2 : (t2 + t1 - 1) / t1);
  if (r1 != r2) G = max64(G, r1 > r2 ? (r1 + r2 - 1) / r2 : (r2 + r1 - 1) / r1);
  return 2 * t_allreduce(cl, V, G, 1);
}

/* Offset of S(g) in the concatenation of S(g') over the divisors g' of n in
 * ascending order (g = n + 1: the total length |Cat|). */
static int64_t cat_offset(int n, int g, int space) {
  int64_t off = 0;
  for (int x = 1; x < g && x <= n; ++x)
    if (n % x == 0) off += orc_catalogue(x, space, NULL, 0);
  return off;
}

int orc_build(const orc_model* m, const orc_cluster* cl, const orc_options* o, int32_t* buf,
              int64_t buf_len, int32_t* n_cfg_out, int32_t* skip_out, int64_t* quantum_out,
              int64_t* words_out, int32_t* n_skip_out, int32_t* skip_srcs_out) {
  if (!m || !cl || !o || m->L < 1 || m->L > ORC_MAX_L || !m->layers) return ORC_ERR_ARG;
  if (cl->n_dev < 1 || cl->node_size < 1 || cl->bw_intra < 1 || cl->bw_inter < 1 || cl->p2p_bw < 1 ||
      cl->lat_ns < 0 || cl->ccoc_permille < 0 || cl->ccoc_permille > 1000)
    return ORC_ERR_ARG;
  if (o->B < 1 || o->B > 65536 || o->Q < 2 || o->Q > 8192 || (o->precision != 0 && o->precision != 1) ||
      o->quantum_ns < 0 || o->quantum_ns > ((int64_t)1 << 61))
    return ORC_ERR_ARG;
  int L = m->L, n = cl->n_dev, cap = o->Q - 1;
  if (cl->mem_bytes <= cl->mem_reserve || cl->mem_reserve < 0) return ORC_ERR_ARG;
  int64_t unit = (cl->mem_bytes - cl->mem_reserve) / cap; /* reading A-8 */
  if (unit < 1) return ORC_ERR_ARG;
  if (cl->dev_mem)
    for (int d = 0; d < cl->n_dev; ++d)
      if (cl->dev_mem[d] <= cl->mem_reserve || cl->dev_mem[d] > cl->mem_bytes) return ORC_ERR_ARG;
  int maxtp = 1;
  while (n % (maxtp * 2) == 0) maxtp *= 2;
  const int64_t LIM = (int64_t)1 << 46;
  for (int u = 0; u < L; ++u) {
    const orc_layer* ly = &m->layers[u];
    if (ly->param_bytes < 0 || ly->param_bytes > LIM || ly->ctx_bytes < 0 || ly->ctx_bytes > LIM ||
        ly->tpcomm_bytes < 0 || ly->tpcomm_bytes > LIM || !ly->fwd_ns || !ly->act_bytes)
      return ORC_ERR_ARG;
    for (int i = 0; i <= ilog2(maxtp); ++i)
      if (ly->fwd_ns[i] < 0 || ly->fwd_ns[i] > ((int64_t)1 << 40) || ly->act_bytes[i] < 0 ||
          ly->act_bytes[i] > LIM)
        return ORC_ERR_ARG;
  }
  /* edges: chain edges u->u+1, plus skip edges from up to ORC_MAX_SKIP
   * sources s to v >= s+2 (one source: T5's cross-attention; several: NEXT-4,
   * reading A-33), sources ascending */
  int nsrc = 0, srcs[ORC_MAX_SKIP];
  int64_t chain_tb[ORC_MAX_L];
  int has_chain[ORC_MAX_L];
  int64_t skip_tb[ORC_MAX_SKIP][ORC_MAX_L];
  int has_skip[ORC_MAX_SKIP][ORC_MAX_L];
  memset(has_chain, 0, sizeof has_chain);
  memset(has_skip, 0, sizeof has_skip);
  for (int e = 0; e < m->n_edges; ++e) {
    const orc_edge* ed = &m->edges[e];
    if (ed->src < 0 || ed->dst >= L || ed->src >= ed->dst || ed->tensor_bytes < 0 || ed->tensor_bytes > LIM)
      return ORC_ERR_ARG;
    if (ed->dst != ed->src + 1) {
      int j = 0;
      while (j < nsrc && srcs[j] != ed->src) ++j;
      if (j == nsrc) {
        if (nsrc == ORC_MAX_SKIP) return ORC_ERR_ARG;
        srcs[nsrc++] = ed->src;
      }
    }
  }
  for (int a = 0; a < nsrc; ++a) /* ascending */
    for (int b = a + 1; b < nsrc; ++b)
      if (srcs[b] < srcs[a]) { int x = srcs[a]; srcs[a] = srcs[b]; srcs[b] = x; }
  for (int e = 0; e < m->n_edges; ++e) {
    const orc_edge* ed = &m->edges[e];
    if (ed->dst == ed->src + 1) {
      if (has_chain[ed->src]) return ORC_ERR_ARG;
      has_chain[ed->src] = 1;
      chain_tb[ed->src] = ed->tensor_bytes;
    } else {
      int j = 0;
      while (srcs[j] != ed->src) ++j;
      if (has_skip[j][ed->dst]) return ORC_ERR_ARG;
      has_skip[j][ed->dst] = 1;
      skip_tb[j][ed->dst] = ed->tensor_bytes;
    }
  }
  const int skip = nsrc == 1 ? srcs[0] : -1;
  if (o->strategy_space != 0 && o->strategy_space != 1) return ORC_ERR_ARG;
  if (o->schedule != 0 && o->schedule != 1) return ORC_ERR_ARG;
  /* the concatenated catalogue Cat of the per-edge resharding matrices:
   * S(g) of every divisor g of n, ascending */
  const int64_t ncat = cat_offset(n, n + 1, o->strategy_space);
  const int64_t* chain_mat[ORC_MAX_L];
  const int64_t* skip_mat[ORC_MAX_SKIP][ORC_MAX_L];
  const int64_t* cut_mat[ORC_MAX_L];
  int any_cut = 0;
  for (int u = 0; u < L; ++u) {
    chain_mat[u] = cut_mat[u] = NULL;
    for (int j = 0; j < ORC_MAX_SKIP; ++j) skip_mat[j][u] = NULL;
  }
  for (int e = 0; e < m->n_edges; ++e) {
    const orc_edge* ed = &m->edges[e];
    if (ed->cut_ns) {
      if (ed->dst != ed->src + 1) return ORC_ERR_ARG; /* a cut follows a chain edge */
      for (int64_t j = 0; j < (int64_t)ncat * ncat; ++j)
        if (ed->cut_ns[j] < 0 || ed->cut_ns[j] > LIM) return ORC_ERR_ARG;
      cut_mat[ed->src] = ed->cut_ns;
      any_cut = 1;
    }
    if (!ed->reshard_ns) continue;
    for (int64_t j = 0; j < (int64_t)ncat * ncat; ++j)
      if (ed->reshard_ns[j] < 0 || ed->reshard_ns[j] > LIM) return ORC_ERR_ARG;
    if (ed->dst == ed->src + 1) chain_mat[ed->src] = ed->reshard_ns;
    else {
      int j = 0;
      while (srcs[j] != ed->src) ++j;
      skip_mat[j][ed->dst] = ed->reshard_ns;
    }
  }
  int32_t cand_buf[2 * 4096];
  int n_cand;
  const int32_t* cand;
  if (o->cand) {
    n_cand = o->n_cand;
    cand = o->cand;
    if (n_cand < 1) return ORC_ERR_ARG;
    for (int i = 0; i < n_cand; ++i) {
      int deg = cand[2 * i], c = cand[2 * i + 1];
      if (deg < 1 || c < 1 || n % deg || o->B % c) return ORC_ERR_ARG;
      for (int j = 0; j < i; ++j)
        if (cand[2 * j] == deg && cand[2 * j + 1] == c) return ORC_ERR_ARG;
    }
  } else {
    n_cand = orc_candidates(n, o->B, cand_buf, 4096);
    if (n_cand > 4096) return ORC_ERR_ARG;
    cand = cand_buf;
  }
  /* NEXT-1: a config carries Rcut when some chain edge has a cut matrix and it has cuts */
#define CUTS(i) (any_cut && cand[2 * (i)] >= 2 && cand[2 * (i)] <= L)
  /* words of config i's block (S = its strategy count) */
#define BLKW(i, S)                                                                                              \
  (4 + 2 * (int64_t)L * (S) + (int64_t)(L - 1) * (S) * (S) + (int64_t)L * (S) * (S) + (L - 1) + cand[2 * (i)] + \
   1 + (CUTS(i) ? (int64_t)(L - 1) * (S) * (S) : 0) + 1 + (o->schedule ? (int64_t)cand[2 * (i)] * L * (S) : 0) + \
   (nsrc >= 2 ? (int64_t)nsrc * L * (S) * (S) : 0))
  /* pass 1: sizes and the int64 ns/byte values */
  int64_t words = 0;
  int Ss[4096];
  for (int i = 0; i < n_cand; ++i) {
    int g = n / cand[2 * i];
    Ss[i] = orc_catalogue(g, o->strategy_space, NULL, 0);
    if (Ss[i] > ORC_MAX_S) return ORC_ERR_RANGE;
    int S = Ss[i];
    words += BLKW(i, S);
  }
  *words_out = words;
  *n_cfg_out = n_cand;
  *skip_out = skip;
  if (n_skip_out) *n_skip_out = nsrc >= 2 ? nsrc : 0;
  for (int j = 0; skip_srcs_out && j < nsrc; ++j) skip_srcs_out[j] = srcs[j];
  if (!buf || buf_len < words) return ORC_OK; /* size query */
  /* int64 tables (ns / bytes), then quantised into buf */
  int64_t* ns = (int64_t*)calloc((size_t)words, sizeof(int64_t));
  int64_t off = 0;
  int cdt = o->precision ? 8 : 4; /* c_dtype */
  int st = ORC_OK;
  for (int i = 0; i < n_cand && st == ORC_OK; ++i) {
    int deg = cand[2 * i], c = cand[2 * i + 1], g = n / deg, S = Ss[i];
    int64_t b = o->B / c; /* micro-batch size b = B / c (Algorithm 1) */
    int32_t cat[3 * ORC_MAX_S];
    orc_catalogue(g, o->strategy_space, cat, ORC_MAX_S);
    const int64_t co = cat_offset(n, g, o->strategy_space); /* this stage size's block of the edge matrices */
    int64_t* blk = ns + off;
    blk[0] = deg; blk[1] = c; blk[2] = S; blk[3] = g;
    int64_t* A = blk + 4;
    int64_t* M = A + (int64_t)L * S;
    int64_t* R = M + (int64_t)L * S;
    int64_t* Rs = R + (int64_t)(L - 1) * S * S;
    int64_t* O = Rs + (int64_t)L * S * S;
    for (int u = 0; u < L; ++u) {
      const orc_layer* ly = &m->layers[u];
      for (int k = 0; k < S; ++k) {
        int64_t t = cat[3 * k], f = cat[3 * k + 1], d = cat[3 * k + 2], r = f * d;
        if (b % r) { A[u * S + k] = 0; M[u * S + k] = -1; continue; } /* reading A-7 */
        int64_t bl = b / r;
        int lt = ilog2((int)t);
        /* time cost model: fwd = batch x per-sample time,
         * bp = 2 fp, TP comm overlapped with computation via CCOC */
        u128 fp = (u128)bl * ly->fwd_ns[lt];
        u128 comp = 3 * fp;
        u128 tpc = 3 * t_allreduce(cl, (u128)bl * ly->tpcomm_bytes, t, 1);
        u128 ov = t_overlap(comp, tpc, cl->ccoc_permille);
        u128 ps_t = cdiv((u128)ly->param_bytes, (u128)t);
        u128 ps_tf = cdiv((u128)ly->param_bytes, (u128)(t * f));
        u128 fsdp = f > 1 ? 2 * t_allgather(cl, ps_t, f, t) : 0;
        u128 sync = t_allreduce(cl, ps_tf, d, t * f) + (f > 1 ? t_allgather(cl, ps_t, f, t) : 0);
        u128 a = ov + fsdp + cdiv(sync, (u128)c);
        /* memory cost model, Eq. (1) + activations + context */
        u128 mem = cdiv((u128)cdt * ly->param_bytes, (u128)(t * f)) + (u128)c * bl * ly->act_bytes[lt] +
                   (u128)ly->ctx_bytes;
        if (a >= NS_LIMIT || mem >= NS_LIMIT) { st = ORC_ERR_RANGE; break; }
        A[u * S + k] = (int64_t)a;
        M[u * S + k] = (int64_t)mem;
      }
    }
    /* same-stage resharding R_uv (the quadratic term of Eq. 3): the caller's
     * per-edge matrix (per sample, times b) when given, else reading A-15 */
    for (int u = 0; u + 1 < L && st == ORC_OK; ++u)
      for (int k = 0; k < S; ++k)
        for (int l = 0; l < S; ++l) {
          u128 v = !has_chain[u] ? 0
                   : chain_mat[u] ? (u128)b * (u128)chain_mat[u][(co + k) * ncat + co + l]
                                  : t_reshard(cl, &cat[3 * k], &cat[3 * l], (u128)b * chain_tb[u]);
          if (v >= NS_LIMIT) st = ORC_ERR_RANGE;
          R[((int64_t)u * S + k) * S + l] = (int64_t)v;
        }
    /* skip edges (same formula per source): the single source's table in
     * Rs; several sources' tables at the block's tail (after M_stage), Rs 0 */
    int64_t* RSS = nsrc >= 2 ? blk + BLKW(i, S) - (int64_t)nsrc * L * S * S : Rs;
    for (int j = 0; j < (nsrc ? nsrc : 1) && st == ORC_OK; ++j)
      for (int v = 0; v < L && st == ORC_OK; ++v)
        for (int k = 0; k < S; ++k)
          for (int l = 0; l < S; ++l) {
            u128 x = (nsrc == 0 || !has_skip[j][v]) ? 0
                     : skip_mat[j][v] ? (u128)b * (u128)skip_mat[j][v][(co + k) * ncat + co + l]
                                      : t_reshard(cl, &cat[3 * k], &cat[3 * l], (u128)b * skip_tb[j][v]);
            if (x >= NS_LIMIT) st = ORC_ERR_RANGE;
            RSS[(((int64_t)j * L + v) * S + k) * S + l] = (int64_t)x;
          }
    /* cut cost o_j: the P2P of every edge crossing the cut, forward and
     * backward (o_j = fo_j + bo_j; readings A-1, A-16) */
    for (int e = 0; e + 1 < L && st == ORC_OK; ++e) {
      u128 sum = 0;
      for (int j = 0; j < m->n_edges; ++j) {
        const orc_edge* ed = &m->edges[j];
        if (ed->src <= e && e < ed->dst) sum += 2 * t_p2p(cl, (u128)b * ed->tensor_bytes);
      }
      if (sum >= NS_LIMIT) st = ORC_ERR_RANGE;
      O[e] = (int64_t)sum;
    }
    /* per-stage memory caps in buckets (Eq. 5 with m_i): the
     * smallest device memory among the stage's g devices */
    int64_t* SC = O + (L - 1);
    for (int st = 0; st < deg; ++st) {
      int64_t m = cl->mem_bytes;
      if (cl->dev_mem)
        for (int d = st * g; d < (st + 1) * g; ++d) m = cl->dev_mem[d] < m ? cl->dev_mem[d] : m;
      int64_t cp = (m - cl->mem_reserve) / unit;
      SC[st] = cp > cap ? cap : cp;
    }
    /* NEXT-1: the strategy-dependent cross-stage cost of each chain edge's
     * cut, b * the caller's per-sample value (Eq. 4) */
    int64_t* HR = SC + deg;
    HR[0] = CUTS(i);
    int64_t* RC = HR + 1;
    if (CUTS(i))
      for (int e = 0; e + 1 < L && st == ORC_OK; ++e)
        for (int k = 0; k < S; ++k)
          for (int l = 0; l < S; ++l) {
            u128 v = cut_mat[e] ? (u128)b * (u128)cut_mat[e][(co + k) * ncat + co + l] : 0;
            if (v >= NS_LIMIT) st = ORC_ERR_RANGE;
            RC[((int64_t)e * S + k) * S + l] = (int64_t)v;
          }
    /* synchronous 1F1B (reading A-32): stage sg keeps the activations of
     * n = min(c, deg - sg) micro-batches in flight instead of GPipe's c
     * (footnote of PAPER.md:122: only the memory constraint changes), so Eq. (1)
     * + activations + context is evaluated per stage with that n */
    int64_t* HM = RC + (CUTS(i) ? (int64_t)(L - 1) * S * S : 0);
    HM[0] = o->schedule;
    for (int sg = 0; o->schedule && sg < deg && st == ORC_OK; ++sg) {
      /* (deg > L: no placement exists, reading A-22; its stage tables are GPipe's) */
      const int64_t nf = deg > L ? c : (c < deg - sg ? c : deg - sg);
      for (int u = 0; u < L; ++u) {
        const orc_layer* ly = &m->layers[u];
        for (int k = 0; k < S; ++k) {
          int64_t t = cat[3 * k], f = cat[3 * k + 1], d = cat[3 * k + 2], r = f * d;
          int64_t* dst = &HM[1 + ((int64_t)sg * L + u) * S + k];
          if (b % r) { *dst = -1; continue; } /* reading A-7 */
          int64_t bl = b / r;
          u128 mem = cdiv((u128)cdt * ly->param_bytes, (u128)(t * f)) + (u128)nf * bl * ly->act_bytes[ilog2((int)t)] +
                     (u128)ly->ctx_bytes;
          if (mem >= NS_LIMIT) { st = ORC_ERR_RANGE; break; }
          *dst = (int64_t)mem;
        }
      }
    }
    off += BLKW(i, S);
  }
  /* time quantum (reading A-9): smallest power of two such that every entry
   * fits 2^22 and every config's sums fit 2^28 (or the caller's quantum). */
  int64_t qn = o->quantum_ns ? o->quantum_ns : 1;
  for (; st == ORC_OK; qn *= 2) {
    int ok = 1;
    off = 0;
    for (int i = 0; i < n_cand && ok; ++i) {
      int S = Ss[i];
      int64_t* A = ns + off + 4;
      int64_t* R = A + 2 * (int64_t)L * S;
      int64_t* Rs = R + (int64_t)(L - 1) * S * S;
      int64_t* O = Rs + (int64_t)L * S * S;
      int64_t sum = 0, osum = 0;
      for (int u = 0; u < L; ++u) {
        int64_t ma = 0, mr = 0, ms = 0;
        for (int k = 0; k < S; ++k) ma = max64(ma, (A[u * S + k] + qn - 1) / qn);
        if (u >= 1)
          for (int k = 0; k < S * S; ++k) mr = max64(mr, (R[(int64_t)(u - 1) * S * S + k] + qn - 1) / qn);
        if (skip >= 0 && u >= skip + 2)
          for (int k = 0; k < S * S; ++k) ms = max64(ms, (Rs[(int64_t)u * S * S + k] + qn - 1) / qn);
        if (nsrc >= 2) { /* every source's edge into u (the sum bound of reading A-9) */
          const int64_t* RSS = ns + off + BLKW(i, S) - (int64_t)nsrc * L * S * S;
          for (int j = 0; j < nsrc; ++j) {
            int64_t mj = 0;
            if (u >= srcs[j] + 2)
              for (int k = 0; k < S * S; ++k) mj = max64(mj, (RSS[((int64_t)j * L + u) * S * S + k] + qn - 1) / qn);
            if (mj > ENTRY_MAX) ok = 0;
            ms += mj;
          }
        }
        if (ma > ENTRY_MAX || mr > ENTRY_MAX || (nsrc < 2 && ms > ENTRY_MAX)) ok = 0;
        sum += ma + mr + ms;
      }
      const int64_t* RC = O + (L - 1) + cand[2 * i] + 1;
      for (int e = 0; e + 1 < L; ++e) {
        int64_t x = (O[e] + qn - 1) / qn, xr = 0;
        if (CUTS(i))
          for (int k = 0; k < S * S; ++k) xr = max64(xr, (RC[(int64_t)e * S * S + k] + qn - 1) / qn);
        if (x > ENTRY_MAX || xr > ENTRY_MAX) ok = 0;
        osum += x + xr; /* every o_j <= O + max Rcut (reading A-9 with NEXT-1) */
      }
      if (sum > SUM_MAX || osum > SUM_MAX) ok = 0;
      off += BLKW(i, S);
    }
    if (ok) break;
    if (o->quantum_ns) { st = ORC_ERR_RANGE; break; }
    if (qn >= ((int64_t)1 << 61)) { st = ORC_ERR_RANGE; break; }
  }
  if (st == ORC_OK) {
    *quantum_out = qn;
    off = 0;
    for (int i = 0; i < n_cand; ++i) {
      int S = Ss[i];
      int64_t* blk = ns + off;
      int32_t* out = buf + off;
      for (int j = 0; j < 4; ++j) out[j] = (int32_t)blk[j];
      int64_t nA = (int64_t)L * S;
      for (int64_t j = 0; j < nA; ++j) out[4 + j] = (int32_t)((blk[4 + j] + qn - 1) / qn);
      for (int64_t j = 0; j < nA; ++j) { /* memory buckets (reading A-8) */
        int64_t byt = blk[4 + nA + j];
        int64_t bk = byt < 0 ? (int64_t)cap + 1 : (byt + unit - 1) / unit;
        out[4 + nA + j] = (int32_t)(bk > cap ? cap + 1 : bk);
      }
      int64_t rest = (int64_t)(L - 1) * S * S + (int64_t)L * S * S + (L - 1);
      for (int64_t j = 0; j < rest; ++j) out[4 + 2 * nA + j] = (int32_t)((blk[4 + 2 * nA + j] + qn - 1) / qn);
      for (int st = 0; st < cand[2 * i]; ++st) out[4 + 2 * nA + rest + st] = (int32_t)blk[4 + 2 * nA + rest + st];
      int64_t x0 = 4 + 2 * nA + rest + cand[2 * i];
      out[x0] = (int32_t)blk[x0]; /* has_rcut */
      int64_t nrc = CUTS(i) ? (int64_t)(L - 1) * S * S : 0;
      for (int64_t j = 0; j < nrc; ++j) out[x0 + 1 + j] = (int32_t)((blk[x0 + 1 + j] + qn - 1) / qn);
      int64_t x1 = x0 + 1 + nrc;
      out[x1] = (int32_t)blk[x1]; /* has_mstage */
      int64_t nms = o->schedule ? (int64_t)cand[2 * i] * nA : 0;
      for (int64_t j = 0; j < nms; ++j) { /* memory buckets (reading A-8) */
        int64_t byt = blk[x1 + 1 + j];
        int64_t bk = byt < 0 ? (int64_t)cap + 1 : (byt + unit - 1) / unit;
        out[x1 + 1 + j] = (int32_t)(bk > cap ? cap + 1 : bk);
      }
      int64_t nrs = nsrc >= 2 ? (int64_t)nsrc * L * S * S : 0; /* several sources' skip tables */
      for (int64_t j = 0; j < nrs; ++j) out[x1 + 1 + nms + j] = (int32_t)((blk[x1 + 1 + nms + j] + qn - 1) / qn);
      off += x1 + 1 + nms + nrs;
    }
  }
  free(ns);
#undef CUTS
#undef BLKW
  return st;
}

/* ---- exported primitives (pinned by tests against SPEC.md's examples) ---- */
static int64_t clamp62(u128 x) { return x >= NS_LIMIT ? -1 : (int64_t)x; }
int64_t orc_allreduce_ns(int64_t V, int64_t G, int64_t bw, int64_t lat) {
  orc_cluster cl = {0};
  cl.node_size = 1 << 30; cl.bw_intra = cl.bw_inter = bw; cl.lat_ns = lat;
  return clamp62(t_allreduce(&cl, (u128)V, G, 1));
}
int64_t orc_allgather_ns(int64_t V, int64_t G, int64_t bw, int64_t lat) {
  orc_cluster cl = {0};
  cl.node_size = 1 << 30; cl.bw_intra = cl.bw_inter = bw; cl.lat_ns = lat;
  return clamp62(t_allgather(&cl, (u128)V, G, 1));
}
int64_t orc_p2p_ns(int64_t V, int64_t bw, int64_t lat) {
  orc_cluster cl = {0};
  cl.p2p_bw = bw; cl.lat_ns = lat;
  return clamp62(t_p2p(&cl, (u128)V));
}
int64_t orc_overlap_ns(int64_t comp, int64_t comm, int32_t ccoc_permille) {
  return clamp62(t_overlap((u128)comp, (u128)comm, ccoc_permille));
}
