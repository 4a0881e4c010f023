/* uniap.h -- C ABI of libuniap.so: exact UniAP strategy search on B200 (sm_100a).
 *
 * UniAP (arXiv 2307.16375), /root/reference/PAPER.md.  The library evaluates
 * exactly the paper's joint inter-/intra-layer objective: for every candidate
 * pipeline degree deg and micro-batch count c (Algorithm 1)
 * and every ordered contiguous layer->stage placement (Eqs. 6-7,
 * PAPER.md:164-192), the optimum of each stage (Eq. 3, PAPER.md:137-145,
 * under the memory constraint Eq. 5, one strategy per layer
 * Eq. 8) by a memory-constrained min-plus chain DP over
 * layer x strategy x memory bucket; the stage optima combined into the GPipe
 * time per iteration (Eq. 2)
 *        tpi = sum_i p_i + sum_j o_j + (c-1) * max(P u O)
 * and the global minimum under the key (tpi, deg, c, stage_of, strategy_of).
 * Readings of silent passages are DESIGN.md Sec. 2 (A-1 .. A-24).
 *
 * Conventions
 *   - Pointers are HOST pointers unless the name ends in _dev.
 *   - Inputs are borrowed for the duration of the call; outputs go to
 *     caller-owned memory.  A handle owns all its device buffers (grown on
 *     demand, reused across calls) and runs on one CUDA stream; one call at a
 *     time per handle; handles are independent (one per GPU / thread).
 *   - Every entry point returns a uniap_status; no exception crosses the ABI.
 *     uniap_last_error(h) gives a message valid until the next call on h.
 *   - All costs are integers: time entries in quanta (reading A-9), memory in
 *     buckets (reading A-8).  The objective is int64.
 *   - Determinism: results are identical for any world size, run and schedule.
 *   - There is no CPU fallback: without a usable sm_100 device, uniap_create
 *     fails with UNIAP_ERR_CUDA.
 */
#ifndef UNIAP_H
#define UNIAP_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define UNIAP_INF 0x40000000        /* 2^30: DP "infeasible"; never a table entry (A-10)    */
#define UNIAP_MAX_ENTRY 0x00400000  /* 2^22: largest A, R, Rskip, O entry (A-10)             */
#define UNIAP_MAX_SUM 0x10000000    /* 2^28: per-config bound on sum_u (max A + max R into u + max Rskip into u) and on sum O (A-9) */
#define UNIAP_MAX_LAYERS 64
#define UNIAP_MAX_STRAT 32
#define UNIAP_MAX_Q 8192            /* memory buckets (cap + 1) */
#define UNIAP_MAX_CFG 4096
#define UNIAP_MAX_LEVELS 4          /* distinct per-stage memory caps per config (NEXT-2)   */
#define UNIAP_MAX_SKIP 4            /* skip sources of a DAG (NEXT-4, uniap_tables.skip_srcs) */
#define UNIAP_MAX_COPIES 4096       /* per config: conditioning copies over every contiguous run of
                                       its skip sources, sum of |S|^run length (NEXT-4)         */

typedef enum {
  UNIAP_OK = 0,
  UNIAP_ERR_ARG = 1,         /* shape / argument violation                                  */
  UNIAP_ERR_INFEASIBLE = 2,  /* every candidate infeasible (objective = INT64_MAX)          */
  UNIAP_ERR_RANGE = 3,       /* an entry > 2^22, a sum bound > 2^28, or a modelled value >= 2^62 */
  UNIAP_ERR_CUDA = 4,        /* CUDA runtime / launch failure, or no sm_100 device          */
  UNIAP_ERR_COMM = 5,        /* record exchange failure (reported by the binding)           */
  UNIAP_ERR_OOM = 6,         /* device allocation failed                                    */
  UNIAP_ERR_INTERNAL = 99    /* self-check of the answer failed (a bug)                      */
} uniap_status;

typedef struct uniap_handle uniap_handle;

/* Create a handle on CUDA device `device`, issuing work on `cuda_stream`
 * (a cudaStream_t; NULL = the handle creates and owns its own stream).
 * Fails with UNIAP_ERR_CUDA if the device is not compute capability 10.x. */
uniap_status uniap_create(uniap_handle** h, int device, void* cuda_stream);
void uniap_destroy(uniap_handle* h);
const char* uniap_last_error(const uniap_handle* h);
const char* uniap_status_string(uniap_status s);
const char* uniap_version(void);

/* ---- result ---------------------------------------------------------- */
/* = SPEC's Assignment + ParallelPlan; the
 * Algorithm 1 output (cost*, deg*, c*, P*, S*) of PAPER.md:209: stage_of is P
 * (App. D: P[u][stage_of[u]] = 1), strategy_of is S. */
typedef struct {
  int64_t objective;                          /* Eq. 2 in quanta; INT64_MAX if infeasible        */
  int32_t cfg_index;                          /* winner's index in the candidate list, -1 none   */
  int32_t deg, c, L;
  int32_t stage_of[UNIAP_MAX_LAYERS];         /* non-decreasing 0..deg-1                          */
  int32_t strategy_of[UNIAP_MAX_LAYERS];      /* index into the config's strategy set             */
  int64_t stage_cost[UNIAP_MAX_LAYERS];       /* p_1..p_deg (Eq. 3)                               */
  int64_t cut_cost[UNIAP_MAX_LAYERS];         /* o_1..o_{deg-1}                                   */
  int32_t stage_mem[UNIAP_MAX_LAYERS];        /* buckets used per stage (Eq. 5 left side)         */
  int64_t* cfg_objective;                     /* IN: caller array [n_cfg] or NULL; OUT: per-config
                                                 optimum (INT64_MAX = infeasible)                 */
  int64_t quantum_ns;                         /* time quantum used (level 2), 0 for level 1       */
  uint64_t dp_cells;                          /* chain-DP cells executed (instance, layer, strategy, bucket) */
  uint64_t dp_relax;                          /* min-plus relaxations executed by the chain DP      */
  uint64_t dp_cells_canonical;                /* cells of the canonical plan (one forward sweep per
                                                 start layer): the workload size */
  double ms_gpu_dp;                           /* device time of the chain-DP kernels (ms)          */
  double ms_gpu_total;                        /* device time of the whole path (ms)                */
  uint64_t h2d_bytes, d2h_bytes;              /* host<->device bytes since the last prepare        */
  uint32_t n_launches;                        /* kernels this library launched since the last prepare */
  uint32_t n_k2_launches;                     /* of which chain-DP (K2) launches                    */
} uniap_result;

/* ---- level 1: integer tables (the parity-test entry) -- */
typedef struct {
  int32_t deg, c, n_strat;   /* 1 <= deg, 1 <= c, 1 <= n_strat <= 32                         */
  const int32_t* A;          /* [L][n_strat]  A_uk, execution cost, 0..2^22   */
  const int32_t* M;          /* [L][n_strat]  M_uk in buckets, >= 0; > cap => forbidden       */
  const int32_t* R;          /* [L-1][n_strat][n_strat]  R[u][k][l]: edge u->u+1 with layer u
                                on k and u+1 on l, 0..2^22 (the quadratic term of Eq. 3)      */
  const int32_t* Rskip;      /* [L][n_strat][n_strat] or NULL: Rskip[v][k_s][k_v] for the skip
                                edge skip_src->v, v >= skip_src+2 (other rows ignored)        */
  const int32_t* O;          /* [L-1] or NULL (= 0): cost of a cut after layer e (Eq. 4 with a
                                constant R', reading A-1)                                     */
  const int32_t* stage_cap;  /* [deg] or NULL (= cap): the memory cap of pipeline stage i,
                                0..cap -- heterogeneous devices, Eq. 5 with a per-stage m_i
                                ("the value of m varies in the case of
                                heterogeneous computing devices").  At most
                                UNIAP_MAX_LEVELS distinct values per config (else _RANGE)    */
  const int32_t* Rcut;       /* [L-1][n_strat][n_strat] or NULL: the strategy-dependent cross-stage
                                cost of the chain edge e -> e+1 when a cut follows layer e
                                (Eq. 4, S_u^T R'_uv S_v): o_j = O[e_j] +
                                Rcut[e_j][k_{e_j}][k_{e_j + 1}], entries 0..2^22, sum over e of
                                (O[e] + max Rcut[e]) <= 2^28.  Ties are then broken by
                                (tpi, deg, c, stage_of, boundary vector, strategy_of), the
                                boundary vector (k_{e_1}, k_{e_1+1}, k_{e_2}, k_{e_2+1}, ...)
                                (reading A-31).  Not combined with per-stage caps other than
                                cap (_ARG); its configs need Q <= 2048 (Q <= 1024 for |S| > 12),
                                else _RANGE                                                    */
  const int32_t* M_stage;    /* [deg][L][n_strat] or NULL: the memory table of each pipeline stage,
                                for a schedule whose memory depends on the stage -- synchronous
                                1F1B keeps min(c, deg - i) micro-batches of stage i in flight
                                instead of GPipe's c ("modify only the memory constraint",
                                footnote of PAPER.md:122; reading A-32).  Stage i then uses
                                M_stage[i] in Eq. 5 (entries >= 0, > its cap = forbidden) and M is
                                ignored (may be NULL).  Not with Rcut (_ARG).  Each distinct
                                (table, stage cap) pair is one interval table (<= deg per config) */
  const int32_t* Rskips;     /* [n_skip][L][n_strat][n_strat] or NULL, with uniap_tables.n_skip > 0
                                (NEXT-4): Rskips[j][v][k_s][k_v], the resharding cost of the skip
                                edge skip_srcs[j] -> v for v >= skip_srcs[j] + 2 (other rows
                                ignored), 0..2^22; NULL = this config has no skip edges.  Not with
                                Rcut (_ARG)                                                     */
} uniap_config;

typedef struct {
  int32_t L;                 /* 1..64 layers in topological order                              */
  int32_t cap;               /* memory capacity in buckets: Q = cap+1 DP columns, Q <= 8192    */
  int32_t skip_src;          /* -1, or the one layer whose edges skip ahead (T5 cross-attn)    */
  int32_t n_cfg;             /* 1..4096 candidate configs, any order; ties broken by the (deg,c)
                                VALUES; a duplicate (deg,c) is UNIAP_ERR_ARG                   */
  const uniap_config* cfg;
  int32_t n_skip;            /* 0, or 1..UNIAP_MAX_SKIP skip sources (then skip_src must be -1):
                                a DAG whose layers are given in topological order with every
                                chain edge u -> u+1 plus edges from these sources to later layers
                                (NEXT-4, general DAGs; reading A-33: with the
                                chain edges Def. 1's contiguous sets are exactly the intervals of
                                that order).  A stage pays every edge with both ends in it (Eq. 3)
                                and conditions on the strategy of each source it holds together
                                with an edge of it: sum over the contiguous runs of sources of
                                |S|^run length at most UNIAP_MAX_COPIES per config (_RANGE)     */
  const int32_t* skip_srcs;  /* [n_skip], strictly ascending layer indices                      */
} uniap_tables;

/* Solve level-1 tables: UNIAP_OK, UNIAP_ERR_INFEASIBLE (objective INT64_MAX,
 * cfg_objective filled), UNIAP_ERR_ARG / _RANGE on bad tables, _CUDA. */
uniap_status uniap_solve_tables(uniap_handle* h, const uniap_tables* t, uniap_result* out);

/* Interval table of one config, for parity tests: P_out[a*L+b] = the stage
 * optimum of [a,b] (Eq. 3 under Eq. 5), UNIAP_INF if infeasible, for EVERY
 * a <= b (the solver itself only evaluates the intervals a deg-stage
 * placement can use).  P_out has L*L int32; entries a > b are UNIAP_INF. */
uniap_status uniap_interval_table(uniap_handle* h, const uniap_tables* t, int32_t cfg, int32_t* P_out);

/* The interval optima the LAST run computed (for parity tests of the plan
 * that actually runs: prefix / middle / suffix sweeps, skip-conditioned
 * copies, the feasible-prefix trim): per config i in candidate order, one
 * L*L block per distinct stage cap of the config (levels in order of first
 * appearance over the stages; one block without per-stage caps):
 * P_out[off_i + (lev*L + a)*L + b], off_i = L*L * (levels of configs < i),
 * UNIAP_INF where infeasible OR not needed by any placement of config i (and
 * for configs another rank owns).  *P_words (if not NULL) receives the
 * total; P_out == NULL only queries it; else P_len must cover every block.
 * Synchronises the handle's stream. */
uniap_status uniap_fetch_intervals(uniap_handle* h, int32_t* P_out, int64_t P_len, int64_t* P_words);

/* ---- level 2: profiles (the paper's problem statement) -- */
typedef struct {
  const int64_t* fwd_ns_per_sample;   /* [1+log2(maxTP)] forward ns per sample, TP size 1,2,4,..
                                         (maxTP = largest power of two dividing n_dev)          */
  int64_t param_bytes;                /* ps, bytes at the training dtype          */
  const int64_t* act_bytes_per_sample;/* [1+log2(maxTP)] activation bytes per sample by TP size  */
  int64_t ctx_bytes;                  /* m_c                                                   */
  int64_t tp_comm_bytes_per_sample;   /* TP collective bytes per sample per forward pass        */
} uniap_layer;                        /* SPEC.md:22-27; each value in [0, 2^46], fwd <= 2^40  */

typedef struct {
  int32_t src, dst;                   /* src < dst; dst == src+1 (chain) or a skip edge from
                                         one of at most UNIAP_MAX_SKIP skip sources to dst >=
                                         src+2 (several sources: NEXT-4, see uniap_tables.n_skip;
                                         the builder emits per-source skip tables)             */
  int64_t tensor_bytes_per_sample;    /* activation bytes crossing the edge per sample (the
                                         cut cost o_j, Eq. 4 with a constant R', reading A-1)  */
  const int64_t* reshard_ns_per_sample; /* NULL, or the edge's resharding matrix R_uv
                                         (the quadratic term of Eq. 3) in ns per
                                         sample, row-major [|Cat|][|Cat|]: row = the strategy of
                                         src, column = the strategy of dst, both indices into
                                         Cat = S(g) of every divisor g of n_dev in ascending
                                         order, concatenated (uniap_catalogue order, the
                                         options' strategy space).  A stage of g devices with
                                         micro-batch b pays b * value.  Entries in [0, 2^46];
                                         borrowed for the call.  NULL: the built-in resharding
                                         formula (reading A-15)                              */
  const int64_t* cut_ns_per_sample;   /* NULL, or (chain edges only) the strategy-dependent
                                         cross-stage cost R'_uv of a cut after src (Eq. 4,
                                         PAPER.md:147-154), ns per sample, same indexing; a
                                         config with cuts gets Rcut = b * value (NEXT-1, see
                                         uniap_config.Rcut); not with dev_mem_bytes            */
} uniap_edge;

typedef struct {
  int32_t n_dev, node_size;           /* devices n, devices per node                           */
  int64_t mem_bytes, mem_reserve_bytes;  /* m and the reserve kept off it (reading A-8)       */
  int64_t bw_intra_Bps, bw_inter_Bps, p2p_Bps;  /* collective / P2P bandwidths, >= 1         */
  int64_t lat_ns;                     /* per-hop latency                                       */
  int32_t ccoc_permille;              /* CCOC in 0..1000                          */
  const int64_t* dev_mem_bytes;       /* NULL, or [n_dev] memory of each device (heterogeneous,
                                         PAPER.md:161): stage i of a (deg, g = n/deg) config runs
                                         on devices i*g .. i*g+g-1 and its cap is
                                         floor((their smallest memory - reserve) / unit), unit
                                         from mem_bytes (reading A-8); each entry in
                                         (mem_reserve_bytes, mem_bytes]                        */
} uniap_cluster;                      /* SPEC.md:115-120 as an alpha-beta record               */

typedef struct {
  int32_t L;
  const uniap_layer* layers;
  int32_t n_edges;
  const uniap_edge* edges;
} uniap_model;                        /* the computation graph G(V,E)           */

typedef struct {
  int32_t B;                          /* mini-batch size, 1..65536                             */
  int32_t precision;                  /* 0 = FP32 (c_dtype 4), 1 = FP16 mixed (c_dtype 8) */
  int32_t Q;                          /* memory buckets, 2..8192 (cap = Q-1)                   */
  int64_t quantum_ns;                 /* 0 = auto (smallest feasible power of two, A-9)        */
  const int32_t* cand;                /* NULL = Algorithm 1's list; else n_cand (deg,c) pairs   */
  int32_t n_cand;
  int32_t strategy_space;             /* 0 = every (t,f,d) triple (reading A-6); 1 = SPEC's
                                         (dp, tp) pairs with an FSDP flag: the
                                         triples with f = 1 or d = 1                            */
  int32_t schedule;                   /* 0 = GPipe (every stage keeps c micro-
                                         batches of activations); 1 = synchronous 1F1B (footnote
                                         of PAPER.md:122): stage i of deg keeps min(c, deg - i),
                                         so the builder emits per-stage memory tables
                                         (uniap_config.M_stage; reading A-32).  Time unchanged */
} uniap_options;

/* Algorithm 1 end to end: cost model on the GPU (K1), then the solve. */
uniap_status uniap_plan(uniap_handle* h, const uniap_model* m, const uniap_cluster* cl,
                        const uniap_options* o, uniap_result* out);

/* The builder's tables (for builder parity tests), per candidate config in
 * order, as int32 blocks
 *    [deg, c, S, g, A[L][S], M[L][S], R[L-1][S][S], Rskip[L][S][S], O[L-1], stage_cap[deg],
 *     has_rcut, Rcut[L-1][S][S] if has_rcut, has_mstage, M_stage[deg][L][S] if has_mstage]
 * (has_mstage = options.schedule; M is GPipe's table either way); with several
 * skip sources (NEXT-4) *skip_src = -1, Rskip is 0 and the block ends with
 * Rskips[n_src][L][S][S] (sources ascending, the model's skip-edge sources)
 * Call with buf == NULL to get *words; then with buf_len >= *words. */
uniap_status uniap_build_tables(uniap_handle* h, const uniap_model* m, const uniap_cluster* cl,
                                const uniap_options* o, int32_t* buf, int64_t buf_len, int64_t* words,
                                int32_t* n_cfg, int32_t* skip_src, int64_t* quantum_ns);

/* ---- split pipeline (device-resident timing, multi-GPU) --------------- */
/* prepare: validate + upload the profile (host->device) and plan the launch.
 * run:     everything on the device for this rank's share of the candidates
 *          (LPT over configs, uniap_shard_assign); writes this rank's best
 *          record into rec_dev (device pointer to one uniap_record; the NCCL
 *          send buffer of the exchange) or, if NULL, into the handle.
 * fetch:   device->host of the last run's record (the handle's, or rec_dev,
 *          which must still be allocated) into *out, plus cfg_objective and
 *          the counters (bytes copied, kernels launched, device times).      */
uniap_status uniap_prepare(uniap_handle* h, const uniap_model* m, const uniap_cluster* cl,
                           const uniap_options* o);
uniap_status uniap_prepare_tables(uniap_handle* h, const uniap_tables* t);
uniap_status uniap_run(uniap_handle* h, int32_t rank, int32_t world, void* rec_dev);
/* Algorithm 1 for this rank's share in one call:
 * uniap_prepare(m, cl, o) + uniap_run(rank, world, rec_dev); rec_dev is the
 * device buffer of one uniap_record, the send buffer of the exchange (one
 * all_gather over ranks), after which uniap_pick gives every rank the plan.
 * The stream-ordered result is in rec_dev when the handle's stream is. */
uniap_status uniap_plan_shard(uniap_handle* h, const uniap_model* m, const uniap_cluster* cl, const uniap_options* o,
                              int32_t rank, int32_t world, void* rec_dev);
/* The same run in two halves, so that across ranks only the owner of the
 * global winner runs a traceback (the stage strategies of Algorithm 1's
 * output): phase 1 runs everything up to this rank's local
 * winner and writes its record HEADER (objective, cfg_index, deg, c, status,
 * counters) into rec_dev; the caller gathers the `world` records (e.g. one
 * NCCL all_gather) into a device array recs_dev; phase 2 picks the global
 * winner on the device by uniap_pick's key and, on the rank holding it only,
 * runs the traceback into rec_dev; then one more gather and uniap_pick.  Both
 * phases are enqueued on the handle's stream without host synchronisation;
 * phase 2 must follow phase 1 of the same (rank, world, rec_dev). */
uniap_status uniap_run_phase(uniap_handle* h, int32_t rank, int32_t world, void* rec_dev, int32_t phase,
                             const void* recs_dev);
uniap_status uniap_fetch(uniap_handle* h, uniap_result* out);

typedef struct {                      /* fixed-size record exchanged between ranks            */
  int64_t objective;                  /* INT64_MAX if this rank holds no feasible config       */
  int32_t cfg_index, deg, c, L, status, n_cfg_local;
  int32_t stage_of[UNIAP_MAX_LAYERS], strategy_of[UNIAP_MAX_LAYERS];
  int64_t stage_cost[UNIAP_MAX_LAYERS], cut_cost[UNIAP_MAX_LAYERS];
  int32_t stage_mem[UNIAP_MAX_LAYERS];
  uint64_t dp_cells, dp_relax, dp_cells_canonical;
} uniap_record;

/* Deterministic LPT assignment of the n_cfg candidates of the prepared
 * problem to `world` ranks: owner_out[i] = rank of candidate i.  Host only. */
uniap_status uniap_shard_assign(uniap_handle* h, int32_t world, int32_t* owner_out);
/* The same assignment computed from the shapes of level-1 tables alone
 * (host only, no handle or device). */
uniap_status uniap_shard_tables(const uniap_tables* t, int32_t world, int32_t* owner_out);

/* Pick the winner among `world` host records by (objective, deg, c); fills
 * *out (cfg_objective untouched).  Host only (no device needed). */
uniap_status uniap_pick(const uniap_record* recs, int32_t world, uniap_result* out);

/* Host-only self check: every chain-DP kernel shape the planner can choose
 * for 1 <= |S| <= 32 and 1 <= Q <= 8192 is compiled into the library.
 * Returns 0, or 1 with the first failing (S, Q, single-chain flag). */
int32_t uniap_selftest(int32_t* S, int32_t* Q, int32_t* single);

/* Candidate list of Algorithm 1 and the strategy catalogue S(g) of a
 * strategy space (0 / 1, see uniap_options) as (t,f,d) triples (host only). */
int32_t uniap_candidates(int32_t n, int32_t B, int32_t* pairs_out, int32_t cap);
int32_t uniap_catalogue(int32_t g, int32_t space, int32_t* tfd_out, int32_t cap);

#ifdef __cplusplus
}
#endif
#endif /* UNIAP_H */
