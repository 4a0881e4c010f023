// uniap_impl.h -- internal declarations of libuniap.so (not part of the ABI).
//
// Device data layout (one "arena" of int32 words per handle, 16-byte aligned
// blocks; NSP = the padded strategy count of the config's kernel class):
//   A  [L][NSP]        execution cost A_uk (pad: 0)
//   M  [L][NSP]        memory buckets M_uk (pad / forbidden: cap+1)
//   Rt [L-1][NSP][NSP] Rt[e][k][k'] = R[e][k'][k]   (forward sweep: for a
//                      destination k the sources k' are contiguous)
//   Rf [L-1][NSP][NSP] Rf[e][k][l]  = R[e][k][l]    (backward sweep)
//   Rs [L][NSP][NSP]   Rs[v][ks][k] = Rskip[v][ks][k] (0 where no skip edge)
//   O  [L-1 (pad 4)]   cut cost
// P arena: [cfg][L][L] int32 interval optima (UNIAP_INF = not computed /
// infeasible).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "uniap.h"

namespace uniap {

constexpr int32_t INF = UNIAP_INF;
constexpr int MAXL = UNIAP_MAX_LAYERS;
constexpr int TMAX = 2176;   // >= L(L+1)/2 + L - 1 theta candidates for L <= 64
constexpr int SORTN = 4096;  // bitonic size (power of two >= TMAX)
// Interval-table levels of a config: its distinct (memory cap, memory table)
// pairs over the stages -- at most UNIAP_MAX_LEVELS distinct caps (NEXT-2),
// and with stage-indexed memory tables (1F1B) up to one level per stage.
constexpr int MAXLEV = UNIAP_MAX_LAYERS;

struct CfgDev {
  int32_t deg, c, S, NSP, g, skip;        // skip: skip source of this config's tables (-1 none)
  int64_t offA, offM, offRt, offRf, offRs, offO;  // word offsets into the arena
  int64_t offP;                            // word offset into the P arena
  // Strategy compaction: the tables hold only the S strategies that can be
  // feasible; orig[k] is the catalogue / caller index of
  // table strategy k, comp[j] the table index of catalogue strategy j (-1:
  // dropped), Sfull the catalogue size (the canonical work counts use it).
  int32_t Sfull, nlev;
  int8_t orig[UNIAP_MAX_STRAT], comp[UNIAP_MAX_STRAT];
  // Per-stage memory caps (NEXT-2): the config's distinct caps
  // lcap[0..nlev), stage i uses level lev_of[i]; the P block of the config
  // holds one L*L table per level (P_lev[a][b] = optimum of [a,b] under lcap).
  int16_t lcap[MAXLEV];  // (caps <= UNIAP_MAX_Q - 1)
  int8_t lev_of[MAXL];
  // Memory tables (1F1B, reading A-32): nmt tables [nmt][L][NSP] at offM;
  // level l reads table lmt[l]; level 2: table j holds mtn[j] micro-batches
  // of activations in flight (0 = the config's c, GPipe)
  int32_t nmt, pad3_;
  int8_t lmt[MAXLEV];
  int8_t mtn[MAXLEV];
  // NEXT-4 (several skip sources, level 1): the sources sk[0..nsk) ascending
  // (nsk >= 2; one source uses `skip`), and per contiguous run of them
  // (index jlo * UNIAP_MAX_SKIP + jhi) the word offset from offA of its
  // conditioning copies: |S|^(jhi - jlo + 1) table pairs [A'][M'] of L*NSP
  // words each, copy kappa = mixed radix over the run's strategies (-1: none)
  int32_t nsk;
  int16_t sk[UNIAP_MAX_SKIP];
  int32_t cprel[UNIAP_MAX_SKIP * UNIAP_MAX_SKIP];
  // NEXT-1 (strategy-dependent cut cost, Eq. 4): cut = 1 when the config has
  // Rcut [L-1][NSP][NSP] at offRc; its stage tables are then
  // T[a][b][kf][kl] ((NSP+1)^2 per interval, index NSP = that end free) at
  // offT in the T arena instead of P
  int32_t cut, pad2_;
  int64_t offRc, offT;
};

// Word offset of the memory table of level `lev` of a config.
__host__ __device__ inline int64_t cfg_moff(const CfgDev& cf, int lev, int L) {
  return cf.offM + (int64_t)cf.lmt[lev] * L * cf.NSP;
}

// NEXT-4: the contiguous run of skip sources a stage [a, b] conditions on
// (every source s with a <= s and s + 2 <= b: it holds s and an edge of s);
// returns its length, *jlo its first source (sources ascending).
__host__ __device__ inline int skip_run(const CfgDev& cf, int a, int b, int* jlo) {
  int n = 0;
  *jlo = -1;
  for (int j = 0; j < cf.nsk; ++j)
    if (a <= cf.sk[j] && cf.sk[j] + 2 <= b) {
      if (*jlo < 0) *jlo = j;
      ++n;
    }
  return n;
}
// Word offset from offA of copy kappa's tables of the run [jlo, jlo + n):
// A', then one M' per memory table of the config (1F1B: per in-flight
// count), L*NSP words each (0: the plain tables, n = 0).
__host__ __device__ inline int64_t copy_words(const CfgDev& cf, int L) { return (int64_t)(1 + cf.nmt) * L * cf.NSP; }
__host__ __device__ inline int64_t copy_rel(const CfgDev& cf, int jlo, int n, int kappa, int L) {
  return n == 0 ? 0 : cf.cprel[jlo * UNIAP_MAX_SKIP + jlo + n - 1] + (int64_t)kappa * copy_words(cf, L);
}
// The memory table a sweep of level `lev` reads, relative to offM: the
// copy's M' of the level's table (n > 0), else the level's table itself.
__host__ __device__ inline int64_t copy_mrel(const CfgDev& cf, int n, int64_t arel, int lev, int L) {
  const int64_t mt = cf.lmt[lev];
  return n ? cf.offA + arel + (1 + mt) * L * cf.NSP - cf.offM : mt * L * cf.NSP;
}

// One chain sweep of K2.
struct Inst {
  int32_t cfg;   // config index
  int32_t a;     // first layer swept
  int32_t n;     // number of layers swept (>= 1): a P-emitting sweep's feasible prefix of n0
                 // (Eq. 5: past it every state is INF), set by the host (level 1) or K1f (level 2),
                 // which also shrink [elo, ehi] to the layers swept
  int32_t ks;    // skip-source conditioning (-1 = none)
  int32_t dir;   // +1 forward (emit P[a][u]), -1 backward (store G[u])
  int32_t emit;  // 1: P plain store, 2: P atomicMin (several copies), 0: store G (traceback);
                 // 5 / 6: as 1 / 2 and store G too (the whole-chain sweep of a deg = 1 config,
                 // kept for its traceback)
  int64_t gofs;  // G stores: word offset of this sweep's G block (layers a-n+1..a)
  // emit 1/2: P entries of the layers u in [elo, ehi] only -- P[a][u] for a
  // forward sweep (intervals starting at a), P[u][a] for a backward sweep
  // (intervals ending at a: the suffix sweep of the last stage)
  int32_t elo, ehi;
  int32_t n0;    // the planned length (the layers a placement can use)
  int32_t lev;   // the config's cap level this sweep emits (P block lev, column ecap)
  int32_t ecap;  // = lcap[lev]: the bucket whose state min_k D[k][ecap] is the stage optimum
  int32_t kf = -1;  // NEXT-1: the first layer swept restricted to strategy kf (-1: free)
  int32_t mrel = 0;  // the sweep's memory table: word offset from CfgDev::offM (lmt[lev] * L * NSP, 1F1B)
  int32_t arel = 0;  // the sweep's execution-cost table: word offset from CfgDev::offA (NEXT-4 copies)
};

struct K2Args {
  const Inst* inst;
  const int32_t* n_inst;  // device count of valid instances (backward), or nullptr
  const CfgDev* cfg;
  const int32_t* arena;
  int32_t* P;
  int32_t* G;
  int32_t L, cap, skip;
  int32_t ecap;  // emission bucket of this launch's sweeps (their cap level's cap; Inst::ecap)
  // NEXT-1 launches (tmode = 1): emit every strategy's state at ecap into the
  // config's T table (CfgDev::offT) instead of the minimum into P
  int32_t tmode = 0;
  int32_t* T = nullptr;
  // diagnostics (UNIAP_TRACE): per-CTA timeline records, or nullptr
  unsigned long long* trace = nullptr;
  uint32_t tag = 0;
  // forward-phase clock (%globaltimer, ns): tim[0] = max of ~start, tim[1] =
  // max of end over the launch's CTAs (both reset to 0 per run), or nullptr
  unsigned long long* tim = nullptr;
};

// Timeline record of one CTA (UNIAP_TRACE): trace[0] = record count, trace[1]
// = capacity, records of 4 words from trace[4]:
//   {tag, %globaltimer at start, at end, smid | ctarank << 8 | inst << 16 | n << 40}
constexpr int TRACE_CAP = 1 << 15;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void trace_put(unsigned long long* tr, uint32_t tag, unsigned long long t0, uint32_t rank,
                                          uint32_t inst, uint32_t n) {
  uint32_t sm;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
  const unsigned long long i = atomicAdd(tr, 1ull);
  if (i < tr[1]) {
    unsigned long long* r = tr + 4 + 4 * i;
    r[0] = tag;
    r[1] = t0;
    r[2] = gtimer();
    r[3] = sm | (rank << 8) | ((unsigned long long)inst << 16) | ((unsigned long long)n << 40);
  }
}
// Programmatic dependent launch (PDL): a kernel launched with pdl_launch may
// start while its same-stream predecessor finishes; it waits here before it
// reads anything the predecessor wrote (griddepcontrol, sm_90+).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
template <typename... KArgs, typename... Args>
inline cudaError_t pdl_launch(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

// The non-K2 kernels record through a per-translation-unit pointer (set by
// combine_trace / builder_trace); tag bit 31 marks them, bits 0-7 the kernel.
enum TraceKind : uint32_t { TR_K1 = 1, TR_K1D = 2, TR_K1F = 3, TR_FILL = 4, TR_K4 = 5, TR_K5A = 6, TR_K5C = 7 };
static __device__ unsigned long long* g_trace = nullptr;
struct TraceScope {  // one record per CTA, written by thread 0 when the kernel returns
  uint32_t tag, extra;  // extra: a kernel-defined count (default blockIdx.y)
  unsigned long long t0 = 0;
  __device__ explicit TraceScope(uint32_t k) : tag(0x80000000u | k), extra(blockIdx.y) {
    if (g_trace && threadIdx.x == 0) t0 = gtimer();
  }
  __device__ ~TraceScope() {
    if (g_trace && threadIdx.x == 0) trace_put(g_trace, tag, t0, 0, blockIdx.x, extra);
  }
};
cudaError_t combine_trace(unsigned long long* p);
cudaError_t builder_trace(unsigned long long* p);
cudaError_t combine_init();  // kernel attributes on the current device (once per device)
cudaError_t builder_init();

// Kernel class: template shape of K2.
struct K2Class {
  int NS;      // strategies (padded)
  int V;       // buckets per thread
  int T;       // threads per CTA
  int C;       // CTAs per cluster
  bool DB;     // double-buffered E (one barrier per layer); single: two
  bool TM = false;  // NEXT-1 launch (per-strategy emission into T)
};

// chain_dp.cu
// single = the config has one long chain (deg = 1): spread its buckets over
// more SMs (a wider cluster) to shorten the critical path.
// few = the config has only a few sweeps (deg = 2: prefix + suffix): each is
// a critical path, so a bucket range that needs a cluster keeps it rather
// than folding into one single-buffered CTA (which halves the SMs per sweep).
// single: a long chain on a cluster, at least single_b buckets per CTA (a
// power of two >= 32)
bool k2_pick_class(int S, int Q, bool single, K2Class* out, bool few = false, int single_b = 256);
// The class of a NEXT-1 (tmode) sweep: one CTA of B = pow2ceil(Q) buckets;
// false when that does not fit (|S| > 12 needs Q <= 1024, else Q <= 2048).
bool k2_pick_class_t(int S, int Q, K2Class* out);
int k2_ns_round(int S);
size_t k2_smem_bytes(const K2Class& c);
// priority: launch priority (0 = default; lower = served first, see
// cudaDeviceGetStreamPriorityRange)
cudaError_t k2_launch(const K2Class& c, const K2Args& args, int n_inst, cudaStream_t st, int priority = 0);
int k2_selftest(int* S_out, int* Q_out, int* single_out);

// Winner of the combine step (written by K5a, read by the host and K5c).
struct Winner {
  int64_t objective;  // INT64_MAX if none
  int32_t cfg, deg, c, S, NSP, n_theta_star, status;
  int32_t end[MAXL];
  int64_t p[MAXL], o[MAXL];
  int32_t kfirst[MAXL], klast[MAXL];  // NEXT-1: each stage's boundary strategies (-1: free)
};

// cutcombine.cu (K4c, NEXT-1): per local config the winner data K5a reads
struct CutRes {
  int32_t status;  // 1 found, 0 infeasible, UNIAP_ERR_RANGE / UNIAP_ERR_INTERNAL
  int32_t ends[MAXL], kfirst[MAXL], klast[MAXL];  // stage ends, boundary strategies (-1: free end)
  int64_t p[MAXL], o[MAXL];
};

// Backward-sweep plan written on the device by K5a for the winner config.
constexpr int MAXCLS = 32;
struct BwPlan {
  int32_t count[MAXCLS];     // backward instances per kernel class (0 but the winner's)
  int64_t gofs[MAXL * 33];   // G word offset per (stage, ks + 1)
};
struct RecordArgs {          // what K5a writes into the record besides the winner
  uniap_record* rec;
  uint64_t cells, relax;           // executed forward-phase work (level 1: the host plan), or
  const unsigned long long* work;  // level 2: per config {cells, relax} written by K1f (k1f_trim)
  uint64_t cells_canon;
  int32_t n_local, L, cap;
  const int64_t* qglob;      // builder flags (level 2) or nullptr
  const int32_t* cls_of_cfg; // kernel class id per config
  Inst* bw_inst;             // out: backward instances of the winner
  BwPlan* bw;                // out
  const CutRes* cutres;      // NEXT-1: per local config its K4c result, or nullptr
  // per config: word offset in G of the whole-chain backward sweep's tables
  // kept from the forward phase (deg = 1; per skip conditioning ks consecutive
  // blocks of L * NSP * Q words), or -1 (the traceback runs its own sweep)
  const int64_t* gstore;
};

// combine.cu
cudaError_t launch_fill(int32_t* p, int64_t n, int32_t v, cudaStream_t st);
struct BwPlan;
struct Winner;
cudaError_t launch_decide(const uniap_record* recs, int world, int rank, BwPlan* bw, Winner* win, cudaStream_t st);
cudaError_t launch_publish(int32_t* d_rec, const uniap_record* rec, int64_t* d_qg, const int64_t* qg,
                           unsigned long long* d_tm, const unsigned long long* tm, int64_t* d_cfg,
                           const int64_t* cfgopt, int ncfg, cudaStream_t st);
// K3 (theta candidates) is fused into K4; K4 also finds each config's stage
// ends (ends[li] = {ok, end_1, ..., end_deg}, MAXL + 1 words per config).
size_t k4_smem(int L, int nlev);
cudaError_t launch_k4(const CfgDev* cfg, const int32_t* arena, const int32_t* P, const int32_t* cfg_list, int li0,
                      int n_local, int L, int nlev, int32_t* thetas, int64_t* vals, int32_t* ends,
                      int64_t* cfg_opt, long long* best_obj, cudaStream_t st);
cudaError_t launch_k5a(const CfgDev* cfg, const int32_t* arena, const int32_t* P, const int32_t* cfg_list,
                       int n_local, int L, const int32_t* ends, const int64_t* cfg_opt, Winner* win,
                       long long* best_obj, const RecordArgs& ra, cudaStream_t st);
cudaError_t launch_k5c_grid(int max_deg, const CfgDev* cfg, const int32_t* arena, const int32_t* G,
                            const BwPlan* bw, const Winner* win, int L, int cap, uniap_record* rec,
                            cudaStream_t st);

// cutcombine.cu (K4c, NEXT-1): CutRes (above) per local config
cudaError_t launch_k4c(const CfgDev* cfg, const int32_t* arena, const int32_t* T, const int32_t* cfg_list, int li0,
                       int n, int L, int64_t* cfg_opt, void* res, int32_t* zscratch, int64_t zstride,
                       cudaStream_t st);
size_t cut_result_bytes();
cudaError_t cutcombine_init();

// builder.cu (K1)
struct ClusterDev {
  int32_t n_dev, node_size, ccoc, B, prec, Q, NT, pad;  // no implicit padding (hashed bytewise)
  int64_t mem_bytes, mem_reserve, bw_intra, bw_inter, p2p, lat, quantum;
};
struct CatDev {  // per config: catalogue (t,f,d) of its strategies
  int32_t tfd[UNIAP_MAX_STRAT * 3];
  int32_t co, ncat;  // block offset of S(g) in the per-edge resharding matrices, their order |Cat|
};
struct BuildBufs {
  const int64_t* fwd;     // [L][NT]
  const int64_t* act;     // [L][NT]
  const int64_t* ps;      // [L]
  const int64_t* ctx;     // [L]
  const int64_t* tpc;     // [L]
  const int64_t* chain;   // [L] tensor bytes of edge u->u+1, -1 none
  const int64_t* skipb;   // [L] tensor bytes of edge skip->v, -1 none
  const int64_t* esrc_dst_bytes;  // [E][3]
  int32_t n_edges;
  const int64_t* rmat;    // caller resharding matrices (ns per sample), concatenated
  const int64_t* chain_mat;  // [L] word offset into rmat of edge u->u+1's matrix, -1 none
  const int64_t* skip_mat;   // [L] word offset of edge skip->v's matrix, -1 none
  const int64_t* cut_mat;    // [L] word offset of edge u->u+1's cut matrix (NEXT-1), -1 none; null: none at all
  const CatDev* cat;      // [ncfg]
  Inst* inst;             // the forward instances of the run (K1f writes each P sweep's feasible length)
  const int32_t* inst_off;  // [ncfg + 1] CSR: config i's instances are inst[inst_idx[inst_off[i] ..]]
  const int32_t* inst_idx;
  int32_t n_trim;           // K1f trim blocks per config (0 when inst is null)
  unsigned long long* work;  // [ncfg][2] executed cells, relaxations of each config's forward sweeps
  int64_t* ns;            // int64 scratch arena, same offsets as the int32 arena
  int64_t* qcfg;          // [ncfg] smallest passing quantum per config
  int64_t* qmax;          // [ncfg][MAXL][5] per layer: max A, max R into u, max Rskip into u, O[u], max Rcut[u]
  int64_t* qglob;         // [3]: quantum, error flags, completion counter of K1d
  int32_t max_nmt = 1;    // the largest memory-table count of a config (K1a's grid)
  int32_t n_src = 1;      // rows of skipb / skip_mat (skip sources, at least 1; NEXT-4: several)
};
cudaError_t launch_k1(const ClusterDev& cl, const BuildBufs& bb, const CfgDev* cfg, int ncfg, int L, int skip,
                      int32_t* arena, cudaStream_t st);

}  // namespace uniap
