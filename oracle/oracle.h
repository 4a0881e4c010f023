/* oracle.h -- UniAP CPU ORACLE (arXiv 2307.16375).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or constant with the CUDA product path
 * (paper_2307_16375_b200/); neither side includes or imports the other.
 *
 * What it computes (Sec. 3.3-3.4):
 *   for every candidate (deg, c) of Algorithm 1 the
 *   minimum over ordered contiguous layer->stage placements (Eqs. 6-7,
 *   PAPER.md:164-192) and per-layer strategies (Eq. 8)
 *   of the GPipe time per iteration (Eq. 2)
 *       tpi = sum_i p_i + sum_j o_j + (c-1) * max(P u O)
 *   with p_i from Eq. 3, o_j the scalar cut cost
 *   (Eq. 4 with a constant R', reading A-1), subject to the per-stage memory
 *   constraint Eq. 5; then the global minimum under the
 *   total key (tpi, deg, c, stage_of, strategy_of) (reading A-11).
 *
 * All arithmetic is integer (int64 / unsigned __int128); see DESIGN.md Sec. 2
 * for every reading of the paper this follows.
 */
#ifndef UNIAP_ORACLE_H
#define UNIAP_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define ORC_MAX_L 64
#define ORC_MAX_S 32
#define ORC_MAX_SKIP 4 /* skip sources of a graph (NEXT-4, reading A-33) */

enum { ORC_OK = 0, ORC_ERR_ARG = 1, ORC_ERR_INFEASIBLE = 2, ORC_ERR_RANGE = 3,
       ORC_ERR_INTERNAL = 99 };

/* ---- level 1: integer tables of one candidate config -------------------- */
typedef struct {
  int32_t deg, c, n_strat;
  const int32_t* A;      /* [L][S]      A_uk                          */
  const int32_t* M;      /* [L][S]      M_uk in buckets; > cap = forbidden             */
  const int32_t* R;      /* [L-1][S][S] R_{u,u+1}[k][l]  (Eq. 3)         */
  const int32_t* Rskip;  /* [L][S][S]   R_{s,v}[k_s][k_v] for v >= s+2, or NULL        */
  const int32_t* O;      /* [L-1]       cut cost after layer e, or NULL (=0)           */
  const int32_t* stage_cap; /* [deg] memory cap of stage i (0..cap), or NULL (= cap):
                               heterogeneous devices, PAPER.md:161 ("the value of m varies
                               in the case of heterogeneous computing devices")          */
  const int32_t* Rcut;   /* [L-1][S][S] or NULL: the strategy-dependent cross-stage cost of
                            the chain edge e -> e+1 when a cut follows layer e (Eq. 4,
                            S_u^T R'_uv S_v): o_j = O[e] + Rcut[e][k_e][k_e+1].
                            Not combined with stage_cap.  Tie-break key (reading A-31):
                            (tpi, deg, c, stage_of, boundary vector, strategy_of) with the
                            boundary vector (k_{e_1}, k_{e_1+1}, k_{e_2}, k_{e_2+1}, ...)    */
  const int32_t* M_stage; /* [deg][L][S] or NULL: the memory table of each pipeline stage
                            (a schedule whose memory depends on the stage: synchronous 1F1B
                            keeps min(c, deg - i) micro-batches of stage i in flight, footnote
                            of PAPER.md:122; reading A-32).  When given, stage i uses
                            M_stage[i] in Eq. 5 and M is ignored (may be NULL).  Not with Rcut. */
  const int32_t* Rskips;  /* [n_skip][L][S][S] or NULL, with orc_tables.n_skip > 0 (NEXT-4,
                            reading A-33): Rskips[j][v][k_s][k_v] for the skip edge
                            skip_srcs[j] -> v, v >= skip_srcs[j] + 2 (other rows ignored) */
} orc_cfg;

typedef struct {
  int32_t L, cap, skip_src, n_cfg;
  const orc_cfg* cfg;
  int32_t n_skip;            /* 0, or 1..ORC_MAX_SKIP skip sources (skip_src must be -1): a DAG
                                whose layers are in topological order with the chain edges and
                                further edges from these sources (NEXT-4, reading A-33)      */
  const int32_t* skip_srcs;  /* [n_skip] ascending                                           */
} orc_tables;

typedef struct {
  int64_t objective;     /* INT64_MAX if every config is infeasible */
  int32_t cfg_index, deg, c, L;
  int32_t stage_of[ORC_MAX_L], strategy_of[ORC_MAX_L];
  int64_t stage_cost[ORC_MAX_L], cut_cost[ORC_MAX_L];
  int32_t stage_mem[ORC_MAX_L];
} orc_result;

/* Solve: n_threads <= 0 means one thread per host core.  cfg_obj may be NULL
 * (else [n_cfg], INT64_MAX for an infeasible config). */
int orc_solve(const orc_tables* t, int n_threads, orc_result* res, int64_t* cfg_obj);

/* Interval table of one config: P[a*L+b] = min cost of the stage [a,b]
 * (Eq. 3 under Eq. 5), INT64_MAX if infeasible, for every a <= b. */
int orc_interval_table(const orc_tables* t, int cfg, int64_t* P);

/* ---- level 2: profiles -> tables (the cost model) ------ */
typedef struct {
  const int64_t* fwd_ns;     /* [1+log2(maxTP)] forward ns per sample by TP size 1,2,4.. */
  int64_t param_bytes;       /* ps, bytes at training dtype                          */
  const int64_t* act_bytes;  /* [1+log2(maxTP)] activation bytes per sample by TP size */
  int64_t ctx_bytes;         /* m_c                                                  */
  int64_t tpcomm_bytes;      /* TP collective bytes per sample per forward           */
} orc_layer;
typedef struct {
  int32_t src, dst;
  int64_t tensor_bytes;      /* activation bytes per sample crossing the edge            */
  const int64_t* reshard_ns; /* NULL, or the edge's resharding matrix R_uv per sample
                                (PAPER.md:134): [|Cat|][|Cat|] ns, Cat = S(g) of every
                                divisor g of n ascending, concatenated; R = b * value   */
  const int64_t* cut_ns;     /* NULL, or (chain edges only) the edge's strategy-dependent
                                cross-stage cost R'_uv per sample (Eq. 4),
                                same indexing: a config gets Rcut = b * value (NEXT-1)      */
} orc_edge;
typedef struct {
  int32_t n_dev, node_size;
  int64_t mem_bytes, mem_reserve, bw_intra, bw_inter, p2p_bw, lat_ns;
  int32_t ccoc_permille;
  const int64_t* dev_mem;    /* NULL, or [n_dev] memory of each device (heterogeneous):
                                stage i of a (deg, g) config runs on devices i*g .. i*g+g-1 and
                                its cap is floor((min of their memory - reserve) / unit);
                                each in (reserve, mem_bytes] (mem_bytes sets the unit)   */
} orc_cluster;
typedef struct { int32_t L; const orc_layer* layers; int32_t n_edges; const orc_edge* edges; } orc_model;
typedef struct {
  int32_t B, precision, Q;
  int64_t quantum_ns;        /* 0 = auto (reading A-9) */
  const int32_t* cand;       /* NULL = Algorithm 1; else n_cand (deg,c) pairs */
  int32_t n_cand;
  int32_t strategy_space;    /* 0 = (t,f,d) triples, 1 = SPEC's (dp,tp)+FSDP-flag pairs */
  int32_t schedule;          /* 0 = GPipe, 1 = synchronous 1F1B (footnote of
                                PAPER.md:122): stage i of deg keeps the activations of
                                min(c, deg - i) micro-batches instead of c (reading A-32) */
} orc_options;

/* Builder': writes, per candidate config in order, the block
 *   [deg, c, S, g, A[L][S], M[L][S], R[L-1][S][S], Rskip[L][S][S], O[L-1], stage_cap[deg],
 *    has_rcut, Rcut[L-1][S][S] if has_rcut, has_mstage, M_stage[deg][L][S] if has_mstage]
 * (has_rcut: some chain edge carries cut_ns and 2 <= deg <= L; has_mstage:
 * schedule = 1, M_stage[i] the memory buckets of stage i under 1F1B); with
 * several skip sources (NEXT-4) *skip_src = -1, *n_skip = their count,
 * skip_srcs[0..n_skip) ascending (ORC_MAX_SKIP entries), Rskip is 0 and the
 * block ends with Rskips[n_skip][L][S][S]; else *n_skip = 0.
 * into buf (int32).  *n_cfg, *skip_src, *quantum_ns, *words are outputs. */
int orc_build(const orc_model* m, const orc_cluster* cl, const orc_options* o,
              int32_t* buf, int64_t buf_len, int32_t* n_cfg, int32_t* skip_src,
              int64_t* quantum_ns, int64_t* words, int32_t* n_skip, int32_t* skip_srcs);

/* Strategy catalogue S(g) (reading A-6): writes (t,f,d) triples, returns count.
 * space 0: every (t,f,d) with t*f*d = g, t a power of two; space 1:
 * only f = 1 (DP) or d = 1 (FSDP over the whole replica axis).  (t, f) ascending. */
int orc_catalogue(int32_t g, int32_t space, int32_t* tfd, int32_t cap);

/* Candidate list of Algorithm 1: writes (deg,c) pairs. */
int orc_candidates(int32_t n, int32_t B, int32_t* pairs, int32_t cap);

/* Cost-model primitives (ns; -1 if >= 2^62), exported for the pins. */
int64_t orc_allreduce_ns(int64_t V, int64_t G, int64_t bw, int64_t lat);
int64_t orc_allgather_ns(int64_t V, int64_t G, int64_t bw, int64_t lat);
int64_t orc_p2p_ns(int64_t V, int64_t bw, int64_t lat);
int64_t orc_overlap_ns(int64_t comp, int64_t comm, int32_t ccoc_permille);

#ifdef __cplusplus
}
#endif
#endif
