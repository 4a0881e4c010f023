// abi.cu -- the C ABI of libuniap.so (include/uniap.h): validation, the
// candidate enumerator (K0, Algorithm 1), the strategy catalogue, device
// layout, launch plan (instances, LPT sharding) and the pipeline
//   K1 builder -> K2 chain DP -> K3 thetas -> K4 combine -> K5a argmin/ends
//   -> K2 backward sweeps -> K5c strategy walk -> record.
// Host code does shapes, bookkeeping and launches only; every step of the
// method's arithmetic runs in the kernels.
#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

#include "uniap_impl.h"

using namespace uniap;

namespace {

template <class T>
struct View {  // non-owning device pointer
  T* p = nullptr;
};

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaError_t ensure(size_t count) {
    if (count <= n && p) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    cudaError_t e = cudaMalloc((void**)&p, std::max<size_t>(count, 1) * sizeof(T));
    if (e == cudaSuccess) n = std::max<size_t>(count, 1);
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
};

int round4(int x) { return (x + 3) & ~3; }

// Buckets per CTA of the traceback's backward sweeps (k2_pick_class single
// mode: the bucket axis over a cluster of up to 16 CTAs).  Measured (A/B on
// the five workloads): up to 1024 buckets one CTA without a cluster is
// fastest (T5 / Swin / ViT -1.2 to -2.4 % per plan against 4 x 256), at
// 4096 buckets 16 x 256 beats 4 x 1024 (Llama +1.2 % with the latter).
static int tb_buckets(int Q) { return Q <= 1024 ? 1024 : 256; }

bool env_flag(const char* name) {
  const char* v = getenv(name);
  return v && *v && *v != '0';
}

}  // namespace

// Interval-table levels of one config: the distinct (memory cap, memory
// table) pairs over the stages in order of first appearance -- per-stage
// caps (NEXT-2) and per-stage memory tables (1F1B, reading A-32) -- and each
// stage's level.
struct Levels {
  int nlev = 1;
  int32_t lcap[MAXLEV] = {};
  int8_t lmt[MAXLEV] = {};
  std::vector<int8_t> lev_of;  // [deg]
};
// caps: [deg] per-stage caps (empty = every stage at cap); mts: [deg] each
// stage's memory table (empty = table 0).  false if more than
// UNIAP_MAX_LEVELS distinct caps.
static bool make_levels(int deg, int cap, const std::vector<int32_t>& caps, const std::vector<int>& mts, Levels& lv) {
  lv.nlev = 0;
  lv.lev_of.assign(std::max(deg, 1), 0);
  int32_t dc[UNIAP_MAX_LEVELS];
  int ndc = 0;
  for (int i = 0; i < std::max(deg, 1); ++i) {
    const int32_t c = caps.empty() ? cap : caps[i];
    const int mt = i < (int)mts.size() ? mts[i] : 0;
    int j = 0;
    while (j < ndc && dc[j] != c) ++j;
    if (j == ndc) {
      if (ndc == UNIAP_MAX_LEVELS) return false;
      dc[ndc++] = c;
    }
    int l = 0;
    while (l < lv.nlev && (lv.lcap[l] != c || lv.lmt[l] != mt)) ++l;
    if (l == lv.nlev) {
      if (lv.nlev == MAXLEV) return false;
      lv.lcap[lv.nlev] = c;
      lv.lmt[lv.nlev++] = (int8_t)mt;
    }
    lv.lev_of[i] = (int8_t)l;
  }
  return true;
}

// The memory tables of a level-1 config: with M_stage, its distinct stage
// tables (by content) in order of first appearance and each stage's table;
// else the one table M (mts empty).
static void stage_tables(const uniap_config& x, int L, std::vector<const int32_t*>& tabs, std::vector<int>& mts) {
  tabs.clear();
  mts.clear();
  if (!x.M_stage) {
    tabs.push_back(x.M);
    return;
  }
  const size_t w = (size_t)L * x.n_strat;
  for (int i = 0; i < std::min(x.deg, L); ++i) {  // (deg > L: infeasible, reading A-22)
    const int32_t* m = x.M_stage + (size_t)i * w;
    size_t j = 0;
    while (j < tabs.size() && memcmp(tabs[j], m, w * sizeof(int32_t))) ++j;
    if (j == tabs.size()) tabs.push_back(m);
    mts.push_back((int)j);
  }
}

// one K2 launch: instances of one kernel class
struct K2Group {
  size_t s, e;  // [s, e) in the uploaded instance array
  K2Class cls;
  double crit;
  int max_inst;  // device-sized launches (backward): grid bound
  int priority = 0;  // launch priority (cluster classes and long critical paths first)
  int ecap = -1;     // emission bucket of every sweep of the launch (K2Args::ecap; -1: the cap)
  int max_deg = 0;   // largest pipeline degree of the group's configs (its K4's stage count)
};

struct RunPlan {
  bool valid = false;
  int rank = 0, world = 1;
  const uniap_record* rec = nullptr;
  std::vector<int32_t> local;
  std::vector<K2Group> fgrp, bgrp;
  std::vector<std::pair<int, int>> k4range;  // per forward group: its configs in `local`
  std::pair<int, int> k4rest{0, 0};          // configs without chain-DP work (deg > L)
  int n_trim = 1;                            // K1f trim blocks per config (8 sweeps per block and pass)
  int max_deg = 0;
};

struct uniap_handle {
  int device = 0;
  cudaStream_t st = nullptr;
  bool own_stream = false;
  std::string err;
  // prepared problem
  bool ready = false, level2 = false;
  int L = 0, cap = 0, Q = 0, skip = -1, ncfg = 0;
  std::vector<CfgDev> cfg;
  std::vector<K2Class> cls;
  std::vector<K2Class> bcls;  // class of the traceback sweeps: spread over a cluster (few instances)
  std::vector<CatDev> cat;
  int64_t arena_words = 0;
  ClusterDev cl{};
  int n_edges = 0;
  // device buffers
  DevBuf<int32_t> arena, P, thetas, ends, cfglist, G;
  DevBuf<int64_t> ns, vals, cfgopt, qcfg, gofs, qmax, gstore;
  View<int64_t> qglob;  // [3] builder quantum / flags / counter: zeroed by each prepare's upload
  // the level-2 profile, config and catalogue arrays: views into ONE device
  // blob filled by one DMA per prepare
  DevBuf<char> upb;
  View<int64_t> fwd, act, ps, ctx, tpc, chain, skipb, edges, rmat, chain_mat, skip_mat, cut_mat;
  View<CfgDev> dcfg;
  View<CatDev> dcat;
  DevBuf<CfgDev> dcfg1;  // level 1: the config array (the arena is its own buffer)
  DevBuf<Inst> inst, binst;
  DevBuf<Inst> iinst;                      // uniap_interval_table's own instance list (not in any graph)
  DevBuf<int32_t> iP;                      // uniap_interval_table's own P block
  DevBuf<Winner> win;
  DevBuf<uniap_record> rec;
  // last run
  uniap_record rec_host{};
  uint64_t cells = 0, relax = 0, cells_canon = 0;
  float ms_dp = 0.f, ms_total = 0.f;
  int64_t quantum = 0;
  cudaEvent_t ev[4] = {};
  uint64_t h2d = 0, d2h = 0;
  uint32_t launches = 0, k2_launches = 0;
  const uniap_record* last_rec = nullptr;  // where the last run wrote its record
  std::vector<cudaStream_t> side;          // K2 classes run concurrently
  std::vector<cudaEvent_t> side_ev;
  cudaEvent_t fork_ev = nullptr;
  RunPlan plan;                            // launch plan of the last (rank, world)
  DevBuf<int32_t> clsid;
  DevBuf<BwPlan> bwp;
  DevBuf<long long> k4best;  // K4's running minimum objective of the run (k4_vals)
  DevBuf<unsigned long long> trace;        // UNIAP_TRACE: K2 per-CTA timeline (diagnostics)
  DevBuf<unsigned long long> tim;          // forward K2 phase clock (see K2Args::tim)
  DevBuf<unsigned long long> work;         // level 2: per config executed {cells, relax} (k1f_trim)
  DevBuf<int32_t> inst_csr;                // per config: its forward instances (offsets [ncfg+1], indices)
  cudaGraphExec_t graph_exec = nullptr;    // the captured pipeline of `plan`
  cudaGraphExec_t graph_ph[2] = {nullptr, nullptr};  // its two halves (uniap_run_phase 1 / 2)
  const void* ph2_recs = nullptr;          // the gathered records phase 2's graph reads
  uint32_t graph_launches = 0, graph_k2 = 0;
  bool capturing = false, timed = false;
  bool no_compact = false;  // uniap_build_tables: keep every strategy in the tables
  // pinned host staging of the uploads of one prepare (one DMA each, no
  // stream sync; stage_ev: the previous prepare's copies have read it) and
  // of the reads of one fetch
  char* stage = nullptr;
  size_t stage_n = 0, stage_off = 0;
  cudaEvent_t stage_ev = nullptr;
  struct FetchBlock {
    uniap_record rec;
    int64_t qg[2];
    unsigned long long tm[2];
    int64_t cfgopt[UNIAP_MAX_CFG];
  }* fb = nullptr, *fb_dev = nullptr;  // mapped pinned block (host / device address), written by k_publish
  std::vector<int64_t> sig;                // what the captured graph depends on
  // level 1 only: per (config, layer) the smallest M of the caller's tables
  // over the config's strategies (cap + 1 = none fits); the plan stops each
  // forward P sweep at its feasible prefix (Eq. 5).  Level 2: K1f does it on
  // the device from the builder's M (k1f_trim).
  std::vector<int32_t> minM;
  std::vector<size_t> minMoff;  // per config: its block of minM, [memory table][layer]
  std::vector<int64_t> layout_key;  // level 2: the inputs of the last layout (reused while equal)
  bool layout_l2 = false;           // the current layout is a level-2 one built from layout_key
  int max_nmt = 1;              // level 2: the largest memory-table count of a config (K1a's grid)
  int n_src = 0;                // level 2: skip sources of the model (NEXT-4: several)
  // per-stage memory caps (NEXT-2): per config its levels and stage caps
  std::vector<Levels> lev;
  std::vector<std::vector<int32_t>> scap;
  int64_t P_words = 0;  // interval tables of every config and cap level
  // NEXT-1: configs with a strategy-dependent cut cost (cut[i]), their
  // boundary-strategy tables T and the K4c results / scratch
  std::vector<char> cut;
  int64_t T_words = 0;
  bool any_cut = false;  // level 2: some edge carries a cut matrix
  DevBuf<int32_t> T, zscr;
  DevBuf<char> cutres;
  int64_t zstride = 0;
};

static void drop_graphs(uniap_handle* h) {
  if (h->graph_exec) { cudaGraphExecDestroy(h->graph_exec); h->graph_exec = nullptr; }
  for (auto& g : h->graph_ph)
    if (g) { cudaGraphExecDestroy(g); g = nullptr; }
}

// A prepared problem keeps the launch plan and the captured graph when
// nothing they depend on changed (shapes, classes, offsets, buffers, and the
// kernel-parameter values of the builder); otherwise both are rebuilt.
static void update_signature(uniap_handle* h) {
  std::vector<int64_t> sg = {h->L, h->Q, h->ncfg, h->skip, h->level2, h->n_edges, h->arena_words, h->n_src};
  for (int32_t m : h->minM) sg.push_back(m);  // level 1: the plan's sweep lengths depend on them
  for (int i = 0; i < h->ncfg; ++i) {
    const CfgDev& d = h->cfg[i];
    const K2Class& k = h->cls[i];
    for (int64_t x : {(int64_t)d.deg, (int64_t)d.c, (int64_t)d.S, (int64_t)d.NSP, (int64_t)d.skip, d.offA, d.offP,
                      (int64_t)k.NS, (int64_t)k.V, (int64_t)k.T, (int64_t)k.C, (int64_t)k.DB, (int64_t)k.TM,
                      (int64_t)d.cut, d.offT, (int64_t)d.nlev, (int64_t)d.nmt})
      sg.push_back(x);
    for (int l = 0; l < d.nlev; ++l) sg.push_back((int64_t)d.lcap[l] << 8 | (uint8_t)d.lmt[l]);
    for (int j = 0; j < d.nsk; ++j) sg.push_back(d.sk[j]);
    for (int st = 0; st < std::min(d.deg, MAXL); ++st) sg.push_back(d.lev_of[st]);
  }
  if (h->level2) {
    const int64_t* c = reinterpret_cast<const int64_t*>(&h->cl);
    for (size_t i = 0; i < sizeof(ClusterDev) / 8; ++i) sg.push_back(c[i]);
  }
  for (const void* p : {(const void*)h->arena.p, (const void*)h->ns.p, (const void*)h->dcfg.p, (const void*)h->dcat.p,
                        (const void*)h->fwd.p, (const void*)h->act.p, (const void*)h->ps.p, (const void*)h->ctx.p,
                        (const void*)h->tpc.p, (const void*)h->chain.p, (const void*)h->skipb.p,
                        (const void*)h->edges.p, (const void*)h->qcfg.p, (const void*)h->qmax.p,
                        (const void*)h->qglob.p, (const void*)h->rmat.p, (const void*)h->chain_mat.p,
                        (const void*)h->skip_mat.p, (const void*)h->cut_mat.p, (const void*)(intptr_t)h->any_cut})
    sg.push_back(reinterpret_cast<int64_t>(p));
  if (sg != h->sig) {
    h->sig.swap(sg);
    h->plan.valid = false;
    drop_graphs(h);
  }
}

// every host<->device copy goes through these (counted for the e2e report)
static cudaError_t h2d(uniap_handle* h, void* dst, const void* src, size_t bytes) {
  h->h2d += bytes;
  return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, h->st);
}
static cudaError_t stage_begin(uniap_handle* h, size_t bytes) {
  if (h->stage_ev) {
    cudaError_t e = cudaEventSynchronize(h->stage_ev);
    if (e != cudaSuccess) return e;
  }
  if (bytes > h->stage_n) {
    if (h->stage) cudaFreeHost(h->stage);
    h->stage = nullptr;
    h->stage_n = 0;
    cudaError_t e = cudaMallocHost((void**)&h->stage, bytes);
    if (e != cudaSuccess) return e;
    h->stage_n = bytes;
  }
  h->stage_off = 0;
  return cudaSuccess;
}
static cudaError_t stage_put(uniap_handle* h, void* dst, const void* src, size_t bytes) {
  if (h->stage_off + bytes > h->stage_n) return cudaErrorInvalidValue;
  memcpy(h->stage + h->stage_off, src, bytes);
  h->h2d += bytes;
  cudaError_t e = cudaMemcpyAsync(dst, h->stage + h->stage_off, bytes, cudaMemcpyHostToDevice, h->st);
  h->stage_off += (bytes + 15) & ~(size_t)15;
  return e;
}
static size_t staged(size_t bytes) { return (bytes + 15) & ~(size_t)15; }
static cudaError_t stage_end(uniap_handle* h) {
  if (!h->stage_ev) {
    cudaError_t e = cudaEventCreateWithFlags(&h->stage_ev, cudaEventDisableTiming);
    if (e != cudaSuccess) return e;
  }
  return cudaEventRecord(h->stage_ev, h->st);
}
static cudaError_t d2h(uniap_handle* h, void* dst, const void* src, size_t bytes) {
  h->d2h += bytes;
  return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, h->st);
}

#define FAIL(h, code, ...)                                   \
  do {                                                       \
    char _b[512];                                            \
    snprintf(_b, sizeof _b, __VA_ARGS__);                    \
    (h)->err = _b;                                           \
    return (code);                                           \
  } while (0)

#define CK(h, x)                                                                                       \
  do {                                                                                                 \
    cudaError_t _e = (x);                                                                              \
    if (_e != cudaSuccess) {                                                                           \
      (h)->err = std::string("CUDA: ") + cudaGetErrorString(_e) + " at " #x;                           \
      return _e == cudaErrorMemoryAllocation ? UNIAP_ERR_OOM : UNIAP_ERR_CUDA;                         \
    }                                                                                                  \
  } while (0)

// ---------------------------------------------------------------------------
// K0 / a-2: candidate enumeration and the strategy catalogue (host).
// ---------------------------------------------------------------------------
extern "C" int32_t uniap_candidates(int32_t n, int32_t B, int32_t* pairs, int32_t cap) {
  // Algorithm 1: the QIP (deg = 1, modelled at batch B,
  // reported c = 1, reading A-4), then deg in factors(n)\{1} x c in
  // factors(B)\{1}, deg ascending then c ascending.
  int32_t k = 0;
  auto put = [&](int32_t d, int32_t c) {
    if (k < cap && pairs) { pairs[2 * k] = d; pairs[2 * k + 1] = c; }
    ++k;
  };
  if (n < 1 || B < 1) return 0;
  put(1, 1);
  for (int32_t d = 2; d <= n; ++d)
    if (n % d == 0)
      for (int32_t c = 2; c <= B; ++c)
        if (B % c == 0) put(d, c);
  return k;
}

extern "C" int32_t uniap_catalogue(int32_t g, int32_t space, int32_t* tfd, int32_t cap) {
  // SD[deg] (reading A-6): (t,f,d) with t*f*d = g, t a
  // power of two; t ascending then f ascending (index 0 = pure DP).  Space 1
  // (SPEC.md:42-64): a (dp, tp) pair whose dp axis is plain DP (f = 1) or
  // fully FSDP-sharded (d = 1).
  int32_t k = 0;
  if (g < 1 || space < 0 || space > 1) return 0;
  for (int32_t t = 1; t <= g && g % t == 0; t *= 2)
    for (int32_t f = 1; f <= g / t; ++f)
      if ((g / t) % f == 0 && (space == 0 || f == 1 || f == g / t)) {
        if (k < cap && tfd) { tfd[3 * k] = t; tfd[3 * k + 1] = f; tfd[3 * k + 2] = g / t / f; }
        ++k;
      }
  return k;
}

extern "C" int32_t uniap_selftest(int32_t* S, int32_t* Q, int32_t* single) { return k2_selftest(S, Q, single); }

extern "C" const char* uniap_version(void) { return "uniap-b200 0.1 (sm_100a)"; }

extern "C" const char* uniap_status_string(uniap_status s) {
  switch (s) {
    case UNIAP_OK: return "ok";
    case UNIAP_ERR_ARG: return "invalid argument";
    case UNIAP_ERR_INFEASIBLE: return "infeasible";
    case UNIAP_ERR_RANGE: return "value out of range";
    case UNIAP_ERR_CUDA: return "CUDA error";
    case UNIAP_ERR_COMM: return "communication error";
    case UNIAP_ERR_OOM: return "out of device memory";
    case UNIAP_ERR_INTERNAL: return "internal self-check failed";
  }
  return "unknown";
}

extern "C" const char* uniap_last_error(const uniap_handle* h) { return h ? h->err.c_str() : "null handle"; }

extern "C" uniap_status uniap_create(uniap_handle** out, int device, void* stream) {
  if (!out) return UNIAP_ERR_ARG;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) return UNIAP_ERR_CUDA;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess || prop.major != 10) return UNIAP_ERR_CUDA;
  if (cudaSetDevice(device) != cudaSuccess) return UNIAP_ERR_CUDA;
  {
    // kernel attributes are per device: set them once for every device used
    static std::mutex mu;
    static std::vector<int> done;
    std::lock_guard<std::mutex> g(mu);
    if (std::find(done.begin(), done.end(), device) == done.end()) {
      if (combine_init() != cudaSuccess || builder_init() != cudaSuccess || cutcombine_init() != cudaSuccess)
        return UNIAP_ERR_CUDA;
      done.push_back(device);
    }
  }
  uniap_handle* h = new uniap_handle();
  h->device = device;
  if (stream) {
    h->st = (cudaStream_t)stream;
  } else {
    if (cudaStreamCreateWithFlags(&h->st, cudaStreamNonBlocking) != cudaSuccess) { delete h; return UNIAP_ERR_CUDA; }
    h->own_stream = true;
  }
  for (auto& e : h->ev)
    if (cudaEventCreate(&e) != cudaSuccess) { delete h; return UNIAP_ERR_CUDA; }
  if (cudaEventCreateWithFlags(&h->fork_ev, cudaEventDisableTiming) != cudaSuccess) { delete h; return UNIAP_ERR_CUDA; }
  *out = h;
  return UNIAP_OK;
}

extern "C" void uniap_destroy(uniap_handle* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  cudaStreamSynchronize(h->st);
  for (auto* b : {&h->arena, &h->P, &h->thetas, &h->ends, &h->cfglist, &h->G}) b->release();
  for (auto* b : {&h->ns, &h->vals, &h->cfgopt, &h->qcfg, &h->gofs, &h->qmax, &h->gstore}) b->release();
  h->upb.release();
  h->dcfg1.release();
  drop_graphs(h);
  h->clsid.release();
  h->bwp.release();
  h->k4best.release();
  h->inst.release();
  h->binst.release();
  h->T.release();
  h->zscr.release();
  h->cutres.release();
  h->iinst.release();
  h->iP.release();
  h->win.release();
  h->rec.release();
  h->tim.release();
  h->work.release();
  h->inst_csr.release();
  h->trace.release();
  for (auto e : h->ev)
    if (e) cudaEventDestroy(e);
  for (auto e : h->side_ev) cudaEventDestroy(e);
  if (h->stage_ev) cudaEventDestroy(h->stage_ev);
  if (h->stage) cudaFreeHost(h->stage);
  if (h->fb) cudaFreeHost(h->fb);
  for (auto x : h->side) cudaStreamDestroy(x);
  if (h->fork_ev) cudaEventDestroy(h->fork_ev);
  if (h->own_stream) cudaStreamDestroy(h->st);
  delete h;
}

static void plan_instances(int L, int i, int deg, int S, int skip, bool all_intervals, int ecap, std::vector<Inst>& out);
static void plan_fast(int L, int i, int deg, int S, int skip, const Levels& lv, bool cut, std::vector<Inst>& out);
static void plan_multi(int L, int i, const CfgDev& d, const Levels& lv, bool all_intervals, std::vector<Inst>& out);

// ---------------------------------------------------------------------------
// Layout of the configs in the device arena.
// ---------------------------------------------------------------------------
// keep[i]: the strategies of config i that can be feasible (ascending caller
// indices); the tables, kernels and plan use only these (S = keep size).
// caps[i]: the per-stage caps of config i ([deg], or empty = all at cap).
// mts[i]: each stage's memory table ([deg], or empty = one table); mtn[i]:
// per memory table its micro-batches in flight (level 2; 0 = c) -- its size
// is the config's table count.
static uniap_status layout_configs(uniap_handle* h, const std::vector<std::vector<int>>& keep,
                                   const std::vector<int>& Sfull, const std::vector<int>& deg,
                                   const std::vector<int>& c, const std::vector<int>& g, const std::vector<int>& skipc,
                                   const std::vector<std::vector<int32_t>>& caps,
                                   const std::vector<std::vector<int>>& mts,
                                   const std::vector<std::vector<int8_t>>& mtn,
                                   const std::vector<std::vector<int>>* msrc = nullptr) {
  const int L = h->L;
  std::vector<int> S(h->ncfg);
  for (int i = 0; i < h->ncfg; ++i) S[i] = (int)keep[i].size();
  h->cfg.assign(h->ncfg, CfgDev{});
  h->cls.assign(h->ncfg, K2Class{});
  h->bcls.assign(h->ncfg, K2Class{});
  h->lev.assign(h->ncfg, Levels{});
  h->scap = caps;
  if ((int)h->cut.size() != h->ncfg) h->cut.assign(h->ncfg, 0);
  h->T_words = 0;
  int64_t off = 0, poff = 0;
  for (int i = 0; i < h->ncfg; ++i)
    if (!make_levels(deg[i], h->cap, caps[i], mts[i], h->lev[i]))
      FAIL(h, UNIAP_ERR_RANGE, "config %d: more than %d distinct per-stage caps", i, UNIAP_MAX_LEVELS);
  for (int i = 0; i < h->ncfg; ++i) {
    // a config with only a few (long) chains spreads each over more SMs
    // (deg = 1: the whole chain, or its |S| skip-conditioned copies, is the
    // critical path of the step; measured: giving deg = 2's prefix + suffix
    // sweeps the same treatment starves the many-sweep classes of SMs)
    static thread_local std::vector<Inst> v;  // (only counted: no allocation per config)
    v.clear();
    const bool multi = msrc && (*msrc)[i].size() >= 2;  // NEXT-4: several skip sources
    if (multi) {
      CfgDev tmp{};
      tmp.deg = deg[i]; tmp.S = S[i]; tmp.NSP = round4(S[i]); tmp.nsk = (int)(*msrc)[i].size();
      for (int j = 0; j < tmp.nsk; ++j) tmp.sk[j] = (int16_t)(*msrc)[i][j];
      plan_multi(L, i, tmp, h->lev[i], false, v);
    } else {
      plan_fast(L, i, deg[i], S[i], skipc[i], h->lev[i], h->cut[i], v);
    }
    const bool single = !v.empty() && ((deg[i] == 1 && !multi) || v.size() <= 1);
    const bool few = !v.empty() && v.size() <= 4;  // deg = 2 (prefix + suffix): keep clusters
    K2Class k;
    if (h->cut[i]) {  // NEXT-1: one-CTA per-strategy emission
      if (!k2_pick_class_t(S[i], h->Q, &k))
        FAIL(h, UNIAP_ERR_RANGE, "config %d: a strategy-dependent cut cost needs Q <= %d at |S| = %d", i,
             S[i] > 12 ? 1024 : 2048, S[i]);
    } else if (!k2_pick_class(S[i], h->Q, single, &k, few,
                              (v.size() == 1 && h->Q <= 1024 && S[i] > 10) ? 128 : 256)) {  // (a lone chain)
      FAIL(h, UNIAP_ERR_ARG, "no kernel class for |S|=%d Q=%d", S[i], h->Q);
    }
    h->cls[i] = k;
    if (!k2_pick_class(S[i], h->Q, true, &h->bcls[i], false, tb_buckets(h->Q)) || h->bcls[i].NS != k.NS)
      FAIL(h, UNIAP_ERR_ARG, "no traceback class for |S|=%d Q=%d", S[i], h->Q);
    CfgDev& d = h->cfg[i];
    const int NSP = round4(k.NS);
    d.deg = deg[i]; d.c = c[i]; d.S = S[i]; d.NSP = NSP; d.g = g[i]; d.skip = skipc[i];
    d.Sfull = Sfull[i];
    for (int j = 0; j < UNIAP_MAX_STRAT; ++j) d.orig[j] = d.comp[j] = -1;
    for (int k = 0; k < S[i]; ++k) {
      d.orig[k] = (int8_t)keep[i][k];
      d.comp[keep[i][k]] = (int8_t)k;
    }
    d.offA = off; off += (int64_t)L * NSP;
    const int nmt = std::max<int>(1, (int)mtn[i].size());  // (empty: one table, GPipe)
    d.offM = off; off += (int64_t)nmt * L * NSP;  // the memory tables [nmt][L][NSP]
    d.offRt = off; off += (int64_t)(L - 1) * NSP * NSP;
    d.offRf = off; off += (int64_t)(L - 1) * NSP * NSP;
    d.offRs = off; off += (int64_t)(multi ? (*msrc)[i].size() : 1) * L * NSP * NSP;  // (NEXT-4: per source)
    d.offO = off; off += std::max(4, round4(L - 1));
    d.cut = h->cut[i];
    d.offRc = off; off += h->cut[i] ? (int64_t)(L - 1) * NSP * NSP : 0;
    d.offT = h->T_words; h->T_words += h->cut[i] ? (int64_t)L * L * (NSP + 1) * (NSP + 1) : 0;
    const Levels& lv = h->lev[i];
    d.nlev = lv.nlev;  // (d is zero-initialised: lmt / mtn of unused levels / tables stay 0)
    for (int l = 0; l < lv.nlev; ++l) {
      d.lcap[l] = (int16_t)lv.lcap[l];
      d.lmt[l] = lv.lmt[l];
    }
    d.nmt = nmt;
    for (size_t j = 0; j < mtn[i].size(); ++j) d.mtn[j] = mtn[i][j];
    for (int st = 0; st < std::min<int>(MAXL, (int)lv.lev_of.size()); ++st) d.lev_of[st] = lv.lev_of[st];
    d.offP = poff; poff += (int64_t)lv.nlev * L * L;  // one L*L interval table per level
    // NEXT-4: the conditioning copies of every contiguous run of skip sources
    d.nsk = multi ? (int)(*msrc)[i].size() : 0;
    for (int j = 0; j < d.nsk; ++j) d.sk[j] = (int16_t)(*msrc)[i][j];
    int64_t ncopies = 0;
    for (int jlo = 0; jlo < d.nsk; ++jlo)
      for (int jhi = jlo; jhi < d.nsk; ++jhi) {
        int64_t ncp = 1;
        for (int j = jlo; j <= jhi; ++j) ncp *= S[i];
        ncopies += ncp;
        if (ncopies > UNIAP_MAX_COPIES)
          FAIL(h, UNIAP_ERR_RANGE, "config %d: more than %d skip-conditioning copies", i, UNIAP_MAX_COPIES);
        d.cprel[jlo * UNIAP_MAX_SKIP + jhi] = (int32_t)(off - d.offA);
        off += ncp * (int64_t)(1 + nmt) * L * NSP;  // A' + one M' per memory table
      }
    if (off - d.offA > INT32_MAX) FAIL(h, UNIAP_ERR_RANGE, "config %d: tables too large", i);
  }
  h->arena_words = off;
  h->P_words = poff;
  return UNIAP_OK;
}

// ---------------------------------------------------------------------------
// Level-1 tables: validation and upload.
// ---------------------------------------------------------------------------
static void reset_counters(uniap_handle* h) { h->h2d = h->d2h = 0; h->launches = h->k2_launches = 0; }

extern "C" uniap_status uniap_prepare_tables(uniap_handle* h, const uniap_tables* tin) {
  if (!h) return UNIAP_ERR_ARG;
  h->ready = false;
  reset_counters(h);
  if (!tin || !tin->cfg) FAIL(h, UNIAP_ERR_ARG, "null tables");
  const uniap_tables* t = tin;
  // NEXT-4: skip sources given as a list (one source: the single-source path)
  uniap_tables t1;
  std::vector<uniap_config> c1;
  std::vector<int> srcs;
  if (tin->n_skip != 0) {
    if (tin->n_skip < 0 || tin->n_skip > UNIAP_MAX_SKIP || !tin->skip_srcs || tin->skip_src != -1 || tin->n_cfg < 1 ||
        tin->n_cfg > UNIAP_MAX_CFG)
      FAIL(h, UNIAP_ERR_ARG, "n_skip=%d (1..%d sources with skip_src = -1)", tin->n_skip, UNIAP_MAX_SKIP);
    for (int j = 0; j < tin->n_skip; ++j) {
      if (tin->skip_srcs[j] < 0 || tin->skip_srcs[j] >= tin->L || (j > 0 && tin->skip_srcs[j] <= tin->skip_srcs[j - 1]))
        FAIL(h, UNIAP_ERR_ARG, "skip_srcs must be ascending layer indices");
      srcs.push_back(tin->skip_srcs[j]);
    }
    t1 = *tin;
    c1.assign(tin->cfg, tin->cfg + tin->n_cfg);
    if (tin->n_skip == 1) {
      t1.skip_src = srcs[0];
      for (auto& x : c1) { x.Rskip = x.Rskips; x.Rskips = nullptr; }
      srcs.clear();
    } else {
      for (auto& x : c1) x.Rskip = nullptr;
    }
    t1.n_skip = 0;
    t1.cfg = c1.data();
    t = &t1;
  }
  const int L = t->L;
  if (L < 1 || L > UNIAP_MAX_LAYERS) FAIL(h, UNIAP_ERR_ARG, "L=%d out of 1..64", L);
  if (t->cap < 0 || t->cap + 1 > UNIAP_MAX_Q) FAIL(h, UNIAP_ERR_ARG, "cap=%d out of 0..%d", t->cap, UNIAP_MAX_Q - 1);
  if (t->skip_src < -1 || t->skip_src >= L) FAIL(h, UNIAP_ERR_ARG, "skip_src=%d", t->skip_src);
  if (t->n_cfg < 1 || t->n_cfg > UNIAP_MAX_CFG) FAIL(h, UNIAP_ERR_ARG, "n_cfg=%d", t->n_cfg);
  h->L = L; h->cap = t->cap; h->Q = t->cap + 1; h->skip = t->skip_src; h->ncfg = t->n_cfg; h->level2 = false;
  h->n_src = 0;
  h->layout_l2 = false;  // (level-1 layouts are rebuilt every time: they depend on the tables' values)
  std::vector<int> S(h->ncfg), deg(h->ncfg), c(h->ncfg), g(h->ncfg, 0), skc(h->ncfg);
  std::vector<std::vector<int>> keep(h->ncfg), mts(h->ncfg);
  std::vector<std::vector<const int32_t*>> tabs(h->ncfg);
  std::vector<std::vector<int8_t>> mtn(h->ncfg);
  for (int i = 0; i < h->ncfg; ++i) {
    const uniap_config& x = t->cfg[i];
    if (x.deg < 1 || x.c < 1 || x.n_strat < 1 || x.n_strat > UNIAP_MAX_STRAT)
      FAIL(h, UNIAP_ERR_ARG, "config %d: deg=%d c=%d n_strat=%d", i, x.deg, x.c, x.n_strat);
    if (!x.A || (!x.M && !x.M_stage) || (L > 1 && !x.R)) FAIL(h, UNIAP_ERR_ARG, "config %d: null table", i);
    for (int j = 0; j < i; ++j)
      if (t->cfg[j].deg == x.deg && t->cfg[j].c == x.c) FAIL(h, UNIAP_ERR_ARG, "duplicate (deg,c)=(%d,%d)", x.deg, x.c);
    const int s = x.n_strat;
    int64_t sum = 0, osum = 0;
    for (int u = 0; u < L; ++u) {
      int64_t ma = 0, mr = 0, ms = 0;
      for (int k = 0; k < s; ++k) {
        const int32_t a = x.A[u * s + k], m = x.M_stage ? 0 : x.M[u * s + k];
        if (a < 0 || a > UNIAP_MAX_ENTRY || m < 0) FAIL(h, UNIAP_ERR_RANGE, "config %d: A/M out of range at layer %d", i, u);
        ma = std::max<int64_t>(ma, a);
      }
      if (u >= 1)
        for (int k = 0; k < s * s; ++k) {
          const int32_t r = x.R[(int64_t)(u - 1) * s * s + k];
          if (r < 0 || r > UNIAP_MAX_ENTRY) FAIL(h, UNIAP_ERR_RANGE, "config %d: R out of range at edge %d", i, u - 1);
          mr = std::max<int64_t>(mr, r);
        }
      if (x.Rskip && t->skip_src >= 0 && u >= t->skip_src + 2)
        for (int k = 0; k < s * s; ++k) {
          const int32_t r = x.Rskip[(int64_t)u * s * s + k];
          if (r < 0 || r > UNIAP_MAX_ENTRY) FAIL(h, UNIAP_ERR_RANGE, "config %d: Rskip out of range at %d", i, u);
          ms = std::max<int64_t>(ms, r);
        }
      for (size_t j = 0; x.Rskips && j < srcs.size(); ++j)  // NEXT-4: every source's edge into u
        if (u >= srcs[j] + 2) {
          int64_t mj = 0;
          for (int k = 0; k < s * s; ++k) {
            const int32_t r = x.Rskips[((int64_t)j * L + u) * s * s + k];
            if (r < 0 || r > UNIAP_MAX_ENTRY) FAIL(h, UNIAP_ERR_RANGE, "config %d: Rskips out of range at %d", i, u);
            mj = std::max<int64_t>(mj, r);
          }
          ms += mj;
        }
      sum += ma + mr + ms;
    }
    if (x.Rskips && !srcs.empty() && x.Rcut)
      FAIL(h, UNIAP_ERR_ARG, "config %d: several skip sources with Rcut are not supported", i);
    if (x.O)
      for (int e = 0; e < L - 1; ++e) {
        if (x.O[e] < 0 || x.O[e] > UNIAP_MAX_ENTRY) FAIL(h, UNIAP_ERR_RANGE, "config %d: O out of range", i);
        osum += x.O[e];
      }
    if (sum > UNIAP_MAX_SUM || osum > UNIAP_MAX_SUM) FAIL(h, UNIAP_ERR_RANGE, "config %d: sum bound exceeds 2^28", i);
    if (x.M_stage) {  // per-stage memory tables (1F1B, reading A-32)
      if (x.Rcut) FAIL(h, UNIAP_ERR_ARG, "config %d: M_stage with Rcut is not supported", i);
      for (int64_t j = 0; j < (int64_t)x.deg * L * s; ++j)
        if (x.M_stage[j] < 0) FAIL(h, UNIAP_ERR_RANGE, "config %d: M_stage entry < 0", i);
    }
    if (x.Rcut && L > 1) {  // NEXT-1: every o_j <= O[e] + max Rcut[e]; the sum of those bounded like O's
      for (int st = 0; x.stage_cap && st < x.deg; ++st)  // (per-stage caps other than cap: not combined)
        if (x.stage_cap[st] != t->cap) FAIL(h, UNIAP_ERR_ARG, "config %d: Rcut with per-stage caps is not supported", i);
      int64_t csum = 0;
      for (int e = 0; e < L - 1; ++e) {
        int64_t mx = 0;
        for (int k = 0; k < s * s; ++k) {
          const int32_t r = x.Rcut[(int64_t)e * s * s + k];
          if (r < 0 || r > UNIAP_MAX_ENTRY) FAIL(h, UNIAP_ERR_RANGE, "config %d: Rcut out of range at edge %d", i, e);
          mx = std::max<int64_t>(mx, r);
        }
        csum += mx + (x.O ? x.O[e] : 0);
      }
      if (csum > UNIAP_MAX_SUM) FAIL(h, UNIAP_ERR_RANGE, "config %d: cut-cost sum bound exceeds 2^28", i);
    }
    S[i] = s; deg[i] = x.deg; c[i] = x.c;
    skc[i] = (x.Rskip && t->skip_src >= 0) ? t->skip_src : -1;
    // strategies with M > cap at every layer (of every stage table) can
    // never be part of a solution
    stage_tables(x, L, tabs[i], mts[i]);
    for (int k = 0; k < s; ++k) {
      bool ok = false;
      for (const int32_t* M : tabs[i])
        for (int u = 0; u < L && !ok; ++u) ok = M[u * s + k] <= t->cap;
      if (ok || h->no_compact) keep[i].push_back(k);
    }
    mtn[i].assign(tabs[i].size(), 0);
    if (keep[i].empty()) keep[i].push_back(0);  // all forbidden: the config is infeasible
  }
  // per (config, memory table, layer) the smallest M over the config's
  // strategies (min over given integers: no cost model)
  h->minMoff.assign(h->ncfg, 0);
  size_t nmin = 0;
  for (int i = 0; i < h->ncfg; ++i) { h->minMoff[i] = nmin; nmin += tabs[i].size() * L; }
  h->minM.assign(nmin, t->cap + 1);
  for (int i = 0; i < h->ncfg; ++i) {
    const uniap_config& x = t->cfg[i];
    for (size_t j = 0; j < tabs[i].size(); ++j)
      for (int u = 0; u < L; ++u) {
        int32_t& mn = h->minM[h->minMoff[i] + j * L + u];
        for (int k : keep[i]) mn = std::min(mn, tabs[i][j][u * x.n_strat + k]);
      }
  }
  std::vector<std::vector<int32_t>> caps(h->ncfg);
  for (int i = 0; i < h->ncfg; ++i)
    if (t->cfg[i].stage_cap) {
      for (int st = 0; st < t->cfg[i].deg; ++st) {
        const int32_t v = t->cfg[i].stage_cap[st];
        if (v < 0 || v > t->cap) FAIL(h, UNIAP_ERR_ARG, "config %d: stage_cap[%d] = %d out of 0..cap", i, st, v);
        caps[i].push_back(v);
      }
    }
  h->any_cut = false;
  h->cut.assign(h->ncfg, 0);  // NEXT-1: a strategy-dependent cut cost matters only with cuts
  for (int i = 0; i < h->ncfg; ++i) h->cut[i] = t->cfg[i].Rcut && L > 1 && deg[i] >= 2 && deg[i] <= L;
  std::vector<std::vector<int>> msrc(h->ncfg);  // NEXT-4: the sources of configs with skip edges
  for (int i = 0; i < h->ncfg; ++i)
    if (t->cfg[i].Rskips && srcs.size() >= 2) msrc[i] = srcs;
  uniap_status st = layout_configs(h, keep, S, deg, c, g, skc, caps, mts, mtn, &msrc);
  if (st != UNIAP_OK) return st;
  // pack the host tables into the device layout (pads: A 0, M cap+1, R 0)
  std::vector<int32_t> a(h->arena_words, 0);
  for (int i = 0; i < h->ncfg; ++i) {
    const uniap_config& x = t->cfg[i];
    const CfgDev& d = h->cfg[i];
    const int s = x.n_strat, N = d.NSP, sc = d.S;
    const std::vector<int>& kp = keep[i];
    for (int u = 0; u < L; ++u)
      for (int k = 0; k < N; ++k) a[d.offA + u * N + k] = k < sc ? x.A[u * s + kp[k]] : 0;
    for (size_t j = 0; j < tabs[i].size(); ++j)
      for (int u = 0; u < L; ++u)
        for (int k = 0; k < N; ++k)
          a[d.offM + ((int64_t)j * L + u) * N + k] = k < sc ? std::min(tabs[i][j][u * s + kp[k]], h->cap + 1) : h->cap + 1;
    for (int e = 0; e + 1 < L; ++e)
      for (int k = 0; k < sc; ++k)
        for (int l = 0; l < sc; ++l) {
          const int32_t r = x.R[((int64_t)e * s + kp[k]) * s + kp[l]];
          a[d.offRf + ((int64_t)e * N + k) * N + l] = r;
          a[d.offRt + ((int64_t)e * N + l) * N + k] = r;
        }
    if (d.skip >= 0)
      for (int v = d.skip + 2; v < L; ++v)
        for (int k = 0; k < sc; ++k)
          for (int l = 0; l < sc; ++l)
            a[d.offRs + ((int64_t)v * N + k) * N + l] = x.Rskip[((int64_t)v * s + kp[k]) * s + kp[l]];
    if (x.O)
      for (int e = 0; e + 1 < L; ++e) a[d.offO + e] = x.O[e];
    if (d.cut)
      for (int e = 0; e + 1 < L; ++e)
        for (int k = 0; k < sc; ++k)
          for (int l = 0; l < sc; ++l)
            a[d.offRc + ((int64_t)e * N + k) * N + l] = x.Rcut[((int64_t)e * s + kp[k]) * s + kp[l]];
    // NEXT-4: per run of skip sources and strategy vector kappa of the run,
    // A' = A + the run's skip-edge terms into every later layer, M' = M with
    // each run source held on its strategy (the others forbidden)
    for (int jlo = 0; jlo < d.nsk; ++jlo)
      for (int jhi = jlo; jhi < d.nsk; ++jhi) {
        int ncp = 1;
        for (int j = jlo; j <= jhi; ++j) ncp *= sc;
        for (int kap = 0; kap < ncp; ++kap) {
          int kv[UNIAP_MAX_SKIP];
          for (int j = jlo, r = kap; j <= jhi; ++j, r /= sc) kv[j] = r % sc;
          const int64_t o = d.offA + copy_rel(d, jlo, jhi - jlo + 1, kap, L);
          for (int u = 0; u < L; ++u)
            for (int k = 0; k < N; ++k) {
              int64_t av = 0;
              bool held = false;  // a run source on another strategy than the copy's
              if (k < sc) {
                av = x.A[u * s + kp[k]];
                for (int j = jlo; j <= jhi; ++j) {
                  if (u >= srcs[j] + 2) av += x.Rskips[(((int64_t)j * L + u) * s + kp[kv[j]]) * s + kp[k]];
                  if (u == srcs[j] && k != kv[j]) held = true;
                }
              }
              a[o + (int64_t)u * N + k] = (int32_t)av;
              for (size_t mt = 0; mt < tabs[i].size(); ++mt)  // M' of every memory table
                a[o + ((int64_t)(1 + mt) * L + u) * N + k] =
                    (k < sc && !held) ? std::min(tabs[i][mt][u * s + kp[k]], h->cap + 1) : h->cap + 1;
            }
        }
      }
  }
  CK(h, cudaSetDevice(h->device));
  CK(h, h->arena.ensure(h->arena_words));
  CK(h, h->dcfg1.ensure(h->ncfg));
  h->dcfg.p = h->dcfg1.p;
  h->dcat.p = nullptr;
  CK(h, stage_begin(h, staged(a.size() * 4) + staged(h->ncfg * sizeof(CfgDev))));
  CK(h, stage_put(h, h->arena.p, a.data(), a.size() * 4));
  CK(h, stage_put(h, h->dcfg.p, h->cfg.data(), h->ncfg * sizeof(CfgDev)));
  CK(h, stage_end(h));
  update_signature(h);
  h->ready = true;
  return UNIAP_OK;
}

// ---------------------------------------------------------------------------
// Level-2 profiles: validation and upload (the builder K1 runs in run()).
// ---------------------------------------------------------------------------
extern "C" uniap_status uniap_prepare(uniap_handle* h, const uniap_model* m, const uniap_cluster* cl,
                                      const uniap_options* o) {
  if (!h) return UNIAP_ERR_ARG;
  h->ready = false;
  reset_counters(h);
  if (!m || !cl || !o || !m->layers) FAIL(h, UNIAP_ERR_ARG, "null argument");
  const int L = m->L;
  if (L < 1 || L > UNIAP_MAX_LAYERS) FAIL(h, UNIAP_ERR_ARG, "L=%d", L);
  if (cl->n_dev < 1 || cl->node_size < 1 || cl->bw_intra_Bps < 1 || cl->bw_inter_Bps < 1 || cl->p2p_Bps < 1 ||
      cl->lat_ns < 0 || cl->ccoc_permille < 0 || cl->ccoc_permille > 1000)
    FAIL(h, UNIAP_ERR_ARG, "bad cluster record");
  if (o->B < 1 || o->B > 65536 || o->Q < 2 || o->Q > UNIAP_MAX_Q || (o->precision != 0 && o->precision != 1) ||
      o->quantum_ns < 0 || o->quantum_ns > ((int64_t)1 << 61) || (o->strategy_space != 0 && o->strategy_space != 1) ||
      (o->schedule != 0 && o->schedule != 1))
    FAIL(h, UNIAP_ERR_ARG, "bad options");
  if (cl->mem_reserve_bytes < 0 || cl->mem_bytes <= cl->mem_reserve_bytes) FAIL(h, UNIAP_ERR_ARG, "memory <= reserve");
  if ((cl->mem_bytes - cl->mem_reserve_bytes) / (o->Q - 1) < 1) FAIL(h, UNIAP_ERR_ARG, "memory unit < 1 byte");
  const int n = cl->n_dev;
  int maxtp = 1;
  while (n % (maxtp * 2) == 0) maxtp *= 2;
  int NT = 1;
  while ((1 << (NT - 1)) < maxtp) ++NT;
  const int64_t LIM = (int64_t)1 << 46;
  std::vector<int64_t> fwd(L * NT), act(L * NT), ps(L), ctx(L), tpc(L), chain(L, -1), skipb(L, -1);
  for (int u = 0; u < L; ++u) {
    const uniap_layer& y = m->layers[u];
    if (!y.fwd_ns_per_sample || !y.act_bytes_per_sample) FAIL(h, UNIAP_ERR_ARG, "layer %d: null profile", u);
    if (y.param_bytes < 0 || y.param_bytes > LIM || y.ctx_bytes < 0 || y.ctx_bytes > LIM ||
        y.tp_comm_bytes_per_sample < 0 || y.tp_comm_bytes_per_sample > LIM)
      FAIL(h, UNIAP_ERR_ARG, "layer %d: value out of range", u);
    for (int i = 0; i < NT; ++i) {
      if (y.fwd_ns_per_sample[i] < 0 || y.fwd_ns_per_sample[i] > ((int64_t)1 << 40) || y.act_bytes_per_sample[i] < 0 ||
          y.act_bytes_per_sample[i] > LIM)
        FAIL(h, UNIAP_ERR_ARG, "layer %d: profile out of range", u);
      fwd[u * NT + i] = y.fwd_ns_per_sample[i];
      act[u * NT + i] = y.act_bytes_per_sample[i];
    }
    ps[u] = y.param_bytes; ctx[u] = y.ctx_bytes; tpc[u] = y.tp_comm_bytes_per_sample;
  }
  // Cat = S(g) of every divisor g of n ascending: the index space of the
  // caller's per-edge resharding matrices (uniap_edge)
  std::vector<int32_t> cat_off(n + 2, 0);
  for (int g = 1; g <= n; ++g)
    cat_off[g + 1] = cat_off[g] + (n % g == 0 ? uniap_catalogue(g, o->strategy_space, nullptr, 0) : 0);
  const int64_t ncat = cat_off[n + 1];
  int skip = -1;
  std::vector<int64_t> ed, rmat, chain_mat(L, -1), skip_mat(L, -1), cut_mat(L, -1);
  // skip sources (one: T5's path; several: NEXT-4, reading A-33), ascending;
  // skipb / skip_mat hold one row of L per source
  std::vector<int> srcs;
  for (int i = 0; i < m->n_edges; ++i) {
    const uniap_edge& e = m->edges[i];
    if (e.dst != e.src + 1 && std::find(srcs.begin(), srcs.end(), e.src) == srcs.end()) srcs.push_back(e.src);
  }
  if ((int)srcs.size() > UNIAP_MAX_SKIP) FAIL(h, UNIAP_ERR_ARG, "more than %d skip sources", UNIAP_MAX_SKIP);
  std::sort(srcs.begin(), srcs.end());
  const int nsrc_rows = std::max<int>(1, (int)srcs.size());
  skipb.assign((size_t)nsrc_rows * L, -1);
  skip_mat.assign((size_t)nsrc_rows * L, -1);
  bool any_cut = false;
  for (int i = 0; i < m->n_edges; ++i) {
    const uniap_edge& e = m->edges[i];
    if (e.src < 0 || e.dst >= L || e.src >= e.dst || e.tensor_bytes_per_sample < 0 || e.tensor_bytes_per_sample > LIM)
      FAIL(h, UNIAP_ERR_ARG, "edge %d invalid", i);
    if (e.dst == e.src + 1) {
      if (chain[e.src] >= 0) FAIL(h, UNIAP_ERR_ARG, "duplicate edge %d->%d", e.src, e.dst);
      chain[e.src] = e.tensor_bytes_per_sample;
    } else {
      const int j = (int)(std::find(srcs.begin(), srcs.end(), e.src) - srcs.begin());
      if (srcs.size() == 1) skip = e.src;
      if (skipb[(size_t)j * L + e.dst] >= 0) FAIL(h, UNIAP_ERR_ARG, "duplicate edge %d->%d", e.src, e.dst);
      skipb[(size_t)j * L + e.dst] = e.tensor_bytes_per_sample;
    }
    ed.push_back(e.src); ed.push_back(e.dst); ed.push_back(e.tensor_bytes_per_sample);
    if (e.cut_ns_per_sample) {  // NEXT-1: a cut after a chain edge only
      if (e.dst != e.src + 1) FAIL(h, UNIAP_ERR_ARG, "edge %d: a cut matrix on a skip edge", i);
      if (ncat * ncat > ((int64_t)1 << 24)) FAIL(h, UNIAP_ERR_ARG, "cut matrix too large (|Cat| = %lld)", (long long)ncat);
      cut_mat[e.src] = (int64_t)rmat.size();
      any_cut = true;
      for (int64_t j = 0; j < ncat * ncat; ++j) {
        const int64_t v = e.cut_ns_per_sample[j];
        if (v < 0 || v > LIM) FAIL(h, UNIAP_ERR_ARG, "edge %d: cut matrix entry out of [0, 2^46]", i);
        rmat.push_back(v);
      }
    }
    if (e.reshard_ns_per_sample) {
      if (ncat * ncat > ((int64_t)1 << 24)) FAIL(h, UNIAP_ERR_ARG, "resharding matrix too large (|Cat| = %lld)", (long long)ncat);
      if (e.dst == e.src + 1) chain_mat[e.src] = (int64_t)rmat.size();
      else skip_mat[(size_t)(std::find(srcs.begin(), srcs.end(), e.src) - srcs.begin()) * L + e.dst] = (int64_t)rmat.size();
      for (int64_t j = 0; j < ncat * ncat; ++j) {
        const int64_t v = e.reshard_ns_per_sample[j];
        if (v < 0 || v > LIM) FAIL(h, UNIAP_ERR_ARG, "edge %d: resharding matrix entry out of [0, 2^46]", i);
        rmat.push_back(v);
      }
    }
  }
  // candidate list (Algorithm 1 or explicit)
  std::vector<int32_t> cand;
  if (o->cand) {
    if (o->n_cand < 1 || o->n_cand > UNIAP_MAX_CFG) FAIL(h, UNIAP_ERR_ARG, "n_cand=%d", o->n_cand);
    for (int i = 0; i < o->n_cand; ++i) {
      const int d = o->cand[2 * i], c = o->cand[2 * i + 1];
      if (d < 1 || c < 1 || n % d || o->B % c) FAIL(h, UNIAP_ERR_ARG, "candidate (%d,%d) does not divide (n,B)", d, c);
      for (int j = 0; j < i; ++j)
        if (o->cand[2 * j] == d && o->cand[2 * j + 1] == c) FAIL(h, UNIAP_ERR_ARG, "duplicate candidate");
      cand.push_back(d); cand.push_back(c);
    }
  } else {
    const int k = uniap_candidates(n, o->B, nullptr, 0);
    if (k > UNIAP_MAX_CFG) FAIL(h, UNIAP_ERR_ARG, "too many candidates");
    cand.resize(2 * k);
    uniap_candidates(n, o->B, cand.data(), k);
  }
  h->L = L; h->Q = o->Q; h->cap = o->Q - 1; h->skip = skip; h->ncfg = (int)cand.size() / 2; h->level2 = true;
  std::vector<int> S(h->ncfg), deg(h->ncfg), c(h->ncfg), g(h->ncfg), skc(h->ncfg, skip);
  h->cat.assign(h->ncfg, CatDev{});
  std::vector<std::vector<int>> keep(h->ncfg);
  for (int i = 0; i < h->ncfg; ++i) {
    deg[i] = cand[2 * i]; c[i] = cand[2 * i + 1]; g[i] = n / deg[i];
    S[i] = uniap_catalogue(g[i], o->strategy_space, nullptr, 0);
    if (S[i] > UNIAP_MAX_STRAT) FAIL(h, UNIAP_ERR_RANGE, "|S(%d)| = %d > 32", g[i], S[i]);
    uniap_catalogue(g[i], o->strategy_space, h->cat[i].tfd, UNIAP_MAX_STRAT);
    h->cat[i].co = cat_off[g[i]];
    h->cat[i].ncat = (int32_t)ncat;
    // b mod (f d) != 0 forbids a strategy at every layer (reading A-7)
    const int b = o->B / c[i];
    for (int k = 0; k < S[i]; ++k)
      if (h->no_compact || b % (h->cat[i].tfd[3 * k + 1] * h->cat[i].tfd[3 * k + 2]) == 0) keep[i].push_back(k);
    if (keep[i].empty()) keep[i].push_back(0);
  }
  // per-stage caps from the per-device memory (NEXT-2): stage
  // i of (deg, g) runs on devices i*g .. i*g+g-1; its cap in buckets is
  // floor((their smallest memory - reserve) / unit), the capacity side of
  // reading A-8 (bucket-feasible => byte-feasible on every device)
  std::vector<std::vector<int32_t>> caps(h->ncfg);
  if (cl->dev_mem_bytes) {
    for (int d = 0; d < n; ++d)
      if (cl->dev_mem_bytes[d] <= cl->mem_reserve_bytes || cl->dev_mem_bytes[d] > cl->mem_bytes)
        FAIL(h, UNIAP_ERR_ARG, "dev_mem_bytes[%d] outside (reserve, mem_bytes]", d);
    const int64_t unit = (cl->mem_bytes - cl->mem_reserve_bytes) / (o->Q - 1);
    for (int i = 0; i < h->ncfg; ++i)
      for (int stg = 0; stg < deg[i]; ++stg) {
        int64_t m = cl->mem_bytes;
        for (int d = stg * g[i]; d < (stg + 1) * g[i]; ++d) m = std::min(m, cl->dev_mem_bytes[d]);
        caps[i].push_back((int32_t)std::min<int64_t>((m - cl->mem_reserve_bytes) / unit, o->Q - 1));
      }
  }
  // NEXT-1 at level 2: configs with cuts get Rcut from the edges' cut matrices
  if (any_cut && srcs.size() >= 2) FAIL(h, UNIAP_ERR_ARG, "cut matrices with several skip sources are not supported");
  h->cut.assign(h->ncfg, 0);
  for (int i = 0; i < h->ncfg && any_cut; ++i) {
    h->cut[i] = deg[i] >= 2 && deg[i] <= L;
    for (size_t st = 0; h->cut[i] && st < caps[i].size(); ++st)
      if (caps[i][st] != o->Q - 1) FAIL(h, UNIAP_ERR_ARG, "cut matrices with per-stage memory caps are not supported");
  }
  h->any_cut = any_cut;
  // memory tables: GPipe keeps c micro-batches in flight on every stage
  // (table 0); synchronous 1F1B keeps min(c, deg - i) on stage i (footnote of
  // PAPER.md:122, reading A-32): one more table per distinct count below c
  std::vector<std::vector<int>> mts(h->ncfg);
  std::vector<std::vector<int8_t>> mtn(h->ncfg);
  for (int i = 0; i < h->ncfg && o->schedule == 1; ++i) {
    mtn[i].assign(1, 0);
    if (deg[i] > L) continue;  // (deg > L: infeasible, reading A-22: GPipe's table)
    if (h->cut[i]) FAIL(h, UNIAP_ERR_ARG, "cut matrices with the 1F1B schedule are not supported");
    for (int stg = 0; stg < deg[i]; ++stg) {
      const int nf = std::min(c[i], deg[i] - stg);
      int j = 0;
      if (nf != c[i]) {
        j = 1;
        while (j < (int)mtn[i].size() && mtn[i][j] != nf) ++j;
        if (j == (int)mtn[i].size()) mtn[i].push_back((int8_t)nf);
      }
      mts[i].push_back(j);
    }
  }
  std::vector<std::vector<int>> msrc(h->ncfg);  // NEXT-4: several skip sources (every config)
  if (srcs.size() >= 2)
    for (int i = 0; i < h->ncfg; ++i) msrc[i] = srcs;
  h->n_src = (int)srcs.size();
  // The layout (arena offsets, kernel classes, levels) depends on shapes
  // only: a profile of the same shapes as the last level-2 prepare (new cost
  // values, e.g. re-profiled layers) keeps it.  Key: every layout input.
  std::vector<int64_t> key = {L, o->Q, o->strategy_space, o->schedule, h->no_compact, h->ncfg, (int64_t)srcs.size(),
                              (int64_t)h->any_cut};
  for (int x : srcs) key.push_back(x);
  for (int i = 0; i < h->ncfg; ++i) {
    for (int64_t x : {(int64_t)deg[i], (int64_t)c[i], (int64_t)g[i], (int64_t)S[i], (int64_t)skc[i],
                      (int64_t)keep[i].size(), (int64_t)caps[i].size(), (int64_t)mts[i].size(), (int64_t)mtn[i].size(),
                      (int64_t)h->cut[i]})
      key.push_back(x);
    for (int x : keep[i]) key.push_back(x);
    for (int32_t x : caps[i]) key.push_back(x);
    for (int x : mts[i]) key.push_back(x);
    for (int8_t x : mtn[i]) key.push_back(x);
  }
  if (!(h->layout_l2 && key == h->layout_key)) {
    h->layout_l2 = false;
    uniap_status st = layout_configs(h, keep, S, deg, c, g, skc, caps, mts, mtn, &msrc);
    if (st != UNIAP_OK) return st;
    h->layout_key.swap(key);
    h->layout_l2 = true;
  }
  h->max_nmt = 1;
  for (int i = 0; i < h->ncfg; ++i) h->max_nmt = std::max(h->max_nmt, std::max(1, (int)mtn[i].size()));
  h->minM.clear();  // the sweep trim runs on the device (k1f_trim)
  h->minMoff.clear();
  h->cl = ClusterDev{cl->n_dev, cl->node_size, cl->ccoc_permille, o->B, o->precision, o->Q, NT, 0,
                     cl->mem_bytes, cl->mem_reserve_bytes, cl->bw_intra_Bps, cl->bw_inter_Bps, cl->p2p_Bps,
                     cl->lat_ns, o->quantum_ns};
  h->n_edges = m->n_edges;
  CK(h, cudaSetDevice(h->device));
  CK(h, h->arena.ensure(h->arena_words));
  CK(h, h->ns.ensure(h->arena_words));
  CK(h, h->qcfg.ensure(h->ncfg));
  {  // per-layer maxima of K1 (zeroed again by K1d after each use): zero when (re)allocated
    const size_t nbefore = h->qmax.n;  // (a reallocation may return the same address)
    CK(h, h->qmax.ensure((size_t)h->ncfg * MAXL * 5));
    if (h->qmax.n != nbefore) CK(h, cudaMemsetAsync(h->qmax.p, 0, h->qmax.n * sizeof(int64_t), h->st));
  }
  {  // one pinned staging block -> one device blob, one DMA
    constexpr int NB = 15;  // ... qglob, zeroed by the same copy (no memset node), then the cut offsets
    const size_t sz[NB] = {fwd.size() * 8, act.size() * 8, (size_t)L * 8, (size_t)L * 8, (size_t)L * 8, (size_t)L * 8,
                           skipb.size() * 8, std::max<size_t>(ed.size(), 3) * 8, h->ncfg * sizeof(CfgDev),
                           h->ncfg * sizeof(CatDev), std::max<size_t>(rmat.size(), 1) * 8, (size_t)L * 8,
                           skip_mat.size() * 8, 3 * 8, (size_t)L * 8};
    const size_t used[NB] = {sz[0], sz[1], sz[2], sz[3], sz[4], sz[5], sz[6], ed.size() * 8, sz[8], sz[9],
                             rmat.size() * 8, sz[11], sz[12], 0, sz[14]};
    const void* src[NB] = {fwd.data(), act.data(), ps.data(), ctx.data(), tpc.data(), chain.data(), skipb.data(),
                           ed.data(), h->cfg.data(), h->cat.data(), rmat.data(), chain_mat.data(), skip_mat.data(),
                           nullptr, cut_mat.data()};
    size_t off[NB], tot = 0;
    for (int i = 0; i < NB; ++i) { off[i] = tot; tot += staged(sz[i]); }
    CK(h, h->upb.ensure(tot));
    CK(h, stage_begin(h, tot));
    memset(h->stage, 0, tot);
    for (int i = 0; i < NB; ++i)
      if (src[i] && used[i]) memcpy(h->stage + off[i], src[i], used[i]);
    h->h2d += tot;
    CK(h, cudaMemcpyAsync(h->upb.p, h->stage, tot, cudaMemcpyHostToDevice, h->st));
    char* b = h->upb.p;
    h->fwd.p = (int64_t*)(b + off[0]); h->act.p = (int64_t*)(b + off[1]); h->ps.p = (int64_t*)(b + off[2]);
    h->ctx.p = (int64_t*)(b + off[3]); h->tpc.p = (int64_t*)(b + off[4]); h->chain.p = (int64_t*)(b + off[5]);
    h->skipb.p = (int64_t*)(b + off[6]); h->edges.p = (int64_t*)(b + off[7]);
    h->dcfg.p = (CfgDev*)(b + off[8]); h->dcat.p = (CatDev*)(b + off[9]);
    h->rmat.p = (int64_t*)(b + off[10]); h->chain_mat.p = (int64_t*)(b + off[11]);
    h->skip_mat.p = (int64_t*)(b + off[12]); h->qglob.p = (int64_t*)(b + off[13]);
    h->cut_mat.p = (int64_t*)(b + off[14]);
  }
  CK(h, stage_end(h));
  update_signature(h);
  h->ready = true;
  return UNIAP_OK;
}

// ---------------------------------------------------------------------------
// Launch plan
// ---------------------------------------------------------------------------
// Forward instances of config i: every start layer a whose interval [a,b] can
// be a stage of a deg-stage ordered placement (a >= stages before it, enough
// layers after it); with the skip source inside the sweep, one copy per
// strategy ks of the skip source (Eq. 3 couples it with later layers).
// Canonical plan (the survey's work definition; also the all-intervals mode
// of uniap_interval_table): one forward sweep per start layer a, over every
// interval [a, b] a deg-stage ordered placement can use.
static void plan_instances(int L, int i, int deg, int S, int skip, bool all_intervals, int ecap, std::vector<Inst>& out) {
  if (!all_intervals && deg > L) return;
  for (int a = 0; a < L; ++a) {
    int bmax;
    if (all_intervals) bmax = L - 1;
    else if (deg == 1) { if (a > 0) break; bmax = L - 1; }
    else bmax = L - 1 - deg + std::min(a + 1, deg);
    if (bmax < a) continue;
    const int n = bmax - a + 1;
    if (skip >= 0 && a <= skip && bmax >= skip + 2) {
      for (int ks = 0; ks < S; ++ks) out.push_back(Inst{i, a, n, ks, +1, 2, 0, a, bmax, n, 0, ecap});
    } else {
      out.push_back(Inst{i, a, n, -1, +1, 1, 0, a, bmax, n, 0, ecap});
    }
  }
}

// The plan the solver runs.  Stage 1 of a placement is a prefix [0, b]
// (b <= L - deg), the last stage a suffix [a, L-1] (a >= deg - 1), the
// middle stages (deg >= 3) intervals [a, b] with 1 <= a, b <= L - 2.  Every
// prefix comes from the forward sweep started at 0 and every suffix from ONE
// backward sweep started at L-1 (the backward DP's min over strategies at
// layer a is the optimum of [a, L-1]), so only the middle stages need a sweep
// per start layer: deg = 2 costs 2 sweeps instead of L.  With the skip
// source s inside a sweep, one copy per strategy ks of s (Eq. 3 couples it
// with later layers); a suffix sweep emits the conditioned copies for a <= s
// and an unconditioned sweep for a > s.
// With per-stage caps (NEXT-2) a sweep emits the optima under ONE cap level
// (column ecap of its state): the prefix sweep under stage 1's, the suffix
// sweep under the last stage's, and the middle sweeps once per distinct
// level among the middle stages, starting where a stage of that level can.
// NEXT-1 (cut): every middle sweep once per first strategy kf (T[a][b][kf][*]),
// the prefix and suffix sweeps emit per strategy at their open end.
static void plan_fast(int L, int i, int deg, int S, int skip, const Levels& lv, bool cut, std::vector<Inst>& out) {
  if (deg > L) return;
  auto fwd = [&](int a, int bmax, int lev, int kf = -1) {
    if (bmax < a) return;
    const int n = bmax - a + 1, ec = lv.lcap[lev];
    if (skip >= 0 && a <= skip && bmax >= skip + 2) {
      for (int ks = 0; ks < S; ++ks)
        if (kf < 0 || a != skip || ks == kf)  // (the first layer is the skip source: one strategy)
          out.push_back(Inst{i, a, n, ks, +1, 2, 0, a, bmax, n, lev, ec, kf});
    } else {
      out.push_back(Inst{i, a, n, -1, +1, 1, 0, a, bmax, n, lev, ec, kf});
    }
  };
  if (deg == 1) {
    // the whole chain as ONE backward sweep from L-1 that also keeps its G
    // tables: the traceback of a deg = 1 winner then needs no sweep of its
    // own (gofs assigned by make_plan).  With the skip source inside, the
    // |S| conditioned copies would keep |S| tables: plain forward sweep.
    const int l0 = lv.lev_of[0];
    if ((skip >= 0 && skip + 2 <= L - 1) || S == 1) fwd(0, L - 1, l0);  // |S| = 1: closed form, no G
    else out.push_back(Inst{i, L - 1, L, -1, -1, 5, -1, 0, 0, L, l0, lv.lcap[l0]});
    return;
  }
  fwd(0, L - deg, lv.lev_of[0]);                                 // stage 1: prefixes
  for (int l = 0; l < lv.nlev && deg >= 3; ++l)                  // middle stages, per cap level:
    for (int a = 1; a <= L - 2; ++a) {                           // stage i (0-based 1..deg-2) can
      int im = -1;                                               // start at a >= i and end at
      for (int st = 1; st <= std::min(a, deg - 2); ++st)         // b <= L - deg + i
        if (lv.lev_of[st] == l) im = st;
      if (im >= 0)
        for (int kf = cut ? 0 : -1; kf < (cut ? S : 0); ++kf) fwd(a, L - deg + im, l, kf);
    }
  const int amin = deg - 1, b = L - 1;                           // last stage: suffixes
  const int ll = lv.lev_of[deg - 1], ec = lv.lcap[ll];
  if (skip >= 0 && amin <= skip && b >= skip + 2) {
    for (int ks = 0; ks < S; ++ks) out.push_back(Inst{i, b, b - amin + 1, ks, -1, 2, 0, amin, skip, b - amin + 1, ll, ec});
    if (skip + 1 <= b) out.push_back(Inst{i, b, b - skip, -1, -1, 1, 0, skip + 1, b, b - skip, ll, ec});
  } else {
    out.push_back(Inst{i, b, b - amin + 1, -1, -1, 1, 0, amin, b, b - amin + 1, ll, ec});
  }
}

// NEXT-4 (several skip sources, reading A-33): the sweeps of plan_fast (or
// of the canonical all-intervals plan), each conditioned on the run of skip
// sources it holds with an edge (skip_run over its longest interval), one
// copy per strategy vector of the run, reading the copy's own A' (skip-edge
// terms folded in) and M' (each conditioned source on its strategy) through
// Inst::arel / Inst::mrel, so K2 runs them as plain sweeps; several copies
// combine by atomicMin.  Extra conditioning of a shorter interval is
// harmless (the minimum over the copies).  The suffix sweep runs once per
// segment of start layers with the same run.
static void plan_multi(int L, int i, const CfgDev& d, const Levels& lv, bool all_intervals, std::vector<Inst>& out) {
  const int deg = d.deg, S = d.S;
  if (!all_intervals && deg > L) return;
  auto put = [&](Inst x, int a, int b) {  // one Inst per copy of the run of [a, b]
    int jlo;
    const int n = skip_run(d, a, b, &jlo);
    int ncp = 1;
    for (int j = 0; j < n; ++j) ncp *= S;
    for (int kp = 0; kp < ncp; ++kp) {
      const int64_t ar = copy_rel(d, jlo, n, kp, L);
      x.emit = ncp > 1 ? 2 : 1;
      x.arel = (int32_t)ar;
      x.mrel = (int32_t)copy_mrel(d, n, ar, x.lev, L);
      out.push_back(x);
    }
  };
  auto fwd = [&](int a, int bmax, int lev) {
    if (bmax < a) return;
    const int n = bmax - a + 1;
    put(Inst{i, a, n, -1, +1, 1, 0, a, bmax, n, lev, lv.lcap[lev]}, a, bmax);
  };
  if (all_intervals) {
    for (int a = 0; a < L; ++a) fwd(a, L - 1, 0);
    return;
  }
  if (deg == 1) {
    fwd(0, L - 1, lv.lev_of[0]);
    return;
  }
  fwd(0, L - deg, lv.lev_of[0]);
  for (int l = 0; l < lv.nlev && deg >= 3; ++l)
    for (int a = 1; a <= L - 2; ++a) {
      int im = -1;
      for (int st = 1; st <= std::min(a, deg - 2); ++st)
        if (lv.lev_of[st] == l) im = st;
      if (im >= 0) fwd(a, L - deg + im, l);
    }
  const int amin = deg - 1, b = L - 1, ll = lv.lev_of[deg - 1];
  for (int a = amin; a <= b;) {  // suffixes [a, L-1], per segment of equal runs
    int j0, j1;
    const int n0 = skip_run(d, a, b, &j0);
    int a2 = a;
    while (a2 + 1 <= b && skip_run(d, a2 + 1, b, &j1) == n0 && j1 == j0) ++a2;
    put(Inst{i, b, b - a + 1, -1, -1, 1, 0, a, a2, b - a + 1, ll, lv.lcap[ll]}, a, b);
    a = a2 + 1;
  }
}

static void forward_instances(const uniap_handle* h, int i, bool all_intervals, std::vector<Inst>& out) {
  const CfgDev& d = h->cfg[i];
  const size_t first = out.size();
  if (d.nsk >= 2) plan_multi(h->L, i, d, h->lev[i], all_intervals, out);  // NEXT-4
  else if (all_intervals) plan_instances(h->L, i, d.deg, d.S, d.skip, all_intervals, h->cap, out);
  else plan_fast(h->L, i, d.deg, d.S, d.skip, h->lev[i], h->cut[i], out);
  if (d.nsk < 2)  // (NEXT-4 copies carry their own M' offsets)
    for (size_t j = first; j < out.size(); ++j) out[j].mrel = (int32_t)(cfg_moff(d, out[j].lev, h->L) - d.offM);
  // Level 1: stop each forward P sweep where it becomes infeasible -- the
  // memory sum of Eq. 5 over the layers swept is at least the running sum of
  // the per-layer minima of the caller's M, so past the first layer where
  // that exceeds cap every state is INF and the interval optima stay INF
  // from the fill (exact; K2 clamps its emitted range to the n it sweeps).
  // G-storing sweeps (deg = 1's kept tables) run in full.  Level 2: K1f.
  if (all_intervals || h->minM.empty()) return;
  const int L = h->L;
  for (size_t j = first; j < out.size(); ++j) {
    Inst& x = out[j];
    if (x.emit != 1 && x.emit != 2) continue;
    int64_t sum = 0;
    int n = 0;
    for (; n < x.n; ++n) {
      sum += h->minM[h->minMoff[i] + (size_t)d.lmt[x.lev] * L + x.a + x.dir * n];  // (a lower bound also at a conditioned skip layer)
      if (sum > x.ecap) break;
    }
    x.n = std::max(n, 1);
    if (x.dir > 0) x.ehi = std::min(x.ehi, x.a + x.n - 1);  // emit only the layers swept
    else x.elo = std::max(x.elo, x.a - x.n + 1);
  }
}

// LPT over configs by executed chain-DP work (sum over the sweeps of n |S|^2 Q); ties
// keep the candidate order, the least-loaded (then lowest) rank takes the next.
static void lpt_shapes(int L, int Q, const std::vector<int>& deg, const std::vector<int>& S,
                       const std::vector<int>& skip, const std::vector<Levels>& lev, const std::vector<char>& cut,
                       int world, std::vector<int>& owner, const std::vector<CfgDev>* multi = nullptr) {
  const int n = (int)deg.size();
  std::vector<int> order(n);
  std::vector<double> w(n);
  for (int i = 0; i < n; ++i) {
    std::vector<Inst> v;
    if (multi && (*multi)[i].nsk >= 2) plan_multi(L, i, (*multi)[i], lev[i], false, v);  // NEXT-4
    else plan_fast(L, i, deg[i], S[i], skip[i], lev[i], cut[i], v);  // the executed sweeps
    double x = 1.0;  // + the combine
    for (auto& e : v) x += (double)e.n * S[i] * S[i] * Q;
    order[i] = i;
    w[i] = x;
  }
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return w[a] > w[b]; });
  std::vector<double> load(world, 0.0);
  owner.assign(n, 0);
  for (int i : order) {
    int r = 0;
    for (int k = 1; k < world; ++k)
      if (load[k] < load[r]) r = k;
    owner[i] = r;
    load[r] += w[i];
  }
}

static void lpt(const uniap_handle* h, int world, std::vector<int>& owner) {
  std::vector<int> deg(h->ncfg), S(h->ncfg), sk(h->ncfg);
  for (int i = 0; i < h->ncfg; ++i) { deg[i] = h->cfg[i].deg; S[i] = h->cfg[i].S; sk[i] = h->cfg[i].skip; }
  lpt_shapes(h->L, h->Q, deg, S, sk, h->lev, h->cut, world, owner, &h->cfg);
}

extern "C" uniap_status uniap_shard_tables(const uniap_tables* t, int32_t world, int32_t* owner_out) {
  if (!t || !t->cfg || !owner_out || world < 1 || t->n_cfg < 1 || t->L < 1) return UNIAP_ERR_ARG;
  if (t->n_skip < 0 || t->n_skip > UNIAP_MAX_SKIP || (t->n_skip > 0 && !t->skip_srcs)) return UNIAP_ERR_ARG;
  std::vector<CfgDev> mc(t->n_cfg, CfgDev{});  // NEXT-4: the shapes plan_multi needs
  std::vector<int> deg(t->n_cfg), S(t->n_cfg), sk(t->n_cfg), owner;
  std::vector<Levels> lev(t->n_cfg);
  std::vector<char> cut(t->n_cfg);
  for (int i = 0; i < t->n_cfg; ++i) {
    deg[i] = t->cfg[i].deg;
    std::vector<int32_t> caps;
    if (t->cfg[i].stage_cap) caps.assign(t->cfg[i].stage_cap, t->cfg[i].stage_cap + deg[i]);
    std::vector<const int32_t*> tabs;
    std::vector<int> mts;
    if (!t->cfg[i].M && !t->cfg[i].M_stage) return UNIAP_ERR_ARG;
    stage_tables(t->cfg[i], t->L, tabs, mts);
    if (!make_levels(deg[i], t->cap, caps, mts, lev[i])) return UNIAP_ERR_RANGE;
    cut[i] = t->cfg[i].Rcut && deg[i] >= 2 && deg[i] <= t->L;
    // the strategy count the prepared tables hold (strategies feasible at some layer)
    const uniap_config& x = t->cfg[i];
    if (x.n_strat < 1) return UNIAP_ERR_ARG;
    S[i] = 0;
    for (int k = 0; k < x.n_strat; ++k) {
      bool ok = false;
      for (const int32_t* M : tabs)
        for (int u = 0; u < t->L && !ok; ++u) ok = M[u * x.n_strat + k] <= t->cap;
      S[i] += ok;
    }
    S[i] = std::max(S[i], 1);
    sk[i] = (x.Rskip && t->skip_src >= 0) ? t->skip_src : -1;
    if (t->n_skip == 1 && x.Rskips) sk[i] = t->skip_srcs[0];
    if (t->n_skip >= 2 && x.Rskips) {
      mc[i].deg = deg[i]; mc[i].S = S[i]; mc[i].NSP = round4(S[i]); mc[i].nsk = t->n_skip;
      for (int j = 0; j < t->n_skip; ++j) mc[i].sk[j] = (int16_t)t->skip_srcs[j];
    }
  }
  lpt_shapes(t->L, t->cap + 1, deg, S, sk, lev, cut, world, owner, &mc);
  for (int i = 0; i < t->n_cfg; ++i) owner_out[i] = owner[i];
  return UNIAP_OK;
}

extern "C" uniap_status uniap_shard_assign(uniap_handle* h, int32_t world, int32_t* owner_out) {
  if (!h || !owner_out || world < 1) return UNIAP_ERR_ARG;
  if (!h->ready) FAIL(h, UNIAP_ERR_ARG, "nothing prepared");
  std::vector<int> owner;
  lpt(h, world, owner);
  for (int i = 0; i < h->ncfg; ++i) owner_out[i] = owner[i];
  return UNIAP_OK;
}

// ---------------------------------------------------------------------------
// K2 launch groups: instances grouped by kernel class (one launch each),
// sorted longest sweep first (LPT within the launch); classes run
// concurrently on side streams (fork / join with events), longest critical
// path first -- the serial chain of one instance: layers x a model of one
// layer's time (its relaxations at the CTA's share of the ALU rate plus the
// per-layer synchronisation) -- so it starts on free SMs.
// ---------------------------------------------------------------------------

static int class_key(const K2Class& k) {
  return k.NS * 1000000 + k.V * 100000 + k.T * 10 + k.C + (k.DB ? 0 : 50000) + (k.TM ? 25000 : 0);
}

// launches group sweeps by kernel class and emission bucket (per-stage caps:
// a launch emits one cap level's column, a kernel parameter)
static int64_t group_key(const uniap_handle* h, const Inst& x) {
  return (int64_t)class_key(h->cls[x.cfg]) * 16384 + x.ecap;
}

static void group_instances(const uniap_handle* h, std::vector<Inst>& all, std::vector<K2Group>& grp) {
  std::vector<int64_t> key(all.size());
  for (size_t j = 0; j < all.size(); ++j) key[j] = group_key(h, all[j]);
  std::vector<size_t> idx(all.size());
  std::iota(idx.begin(), idx.end(), 0);
  std::stable_sort(idx.begin(), idx.end(), [&](size_t a, size_t b) {
    if (key[a] != key[b]) return key[a] < key[b];
    return all[a].n > all[b].n;
  });
  std::vector<Inst> sorted(all.size());
  for (size_t j = 0; j < idx.size(); ++j) sorted[j] = all[idx[j]];
  grp.clear();
  for (size_t s = 0; s < sorted.size();) {
    size_t e = s;
    const int64_t id = group_key(h, sorted[s]);
    double c = 0;
    while (e < sorted.size() && group_key(h, sorted[e]) == id) {
      const K2Class& k = h->cls[sorted[e].cfg];
      const double step = (double)k.NS * k.NS * k.T * k.V / (64.0 * std::min(1.0, k.T / 512.0)) + 3000.0 +
                          (k.C > 1 ? 3000.0 : 0.0);
      c = std::max(c, (double)sorted[e].n * step);
      ++e;
    }
    grp.push_back(K2Group{s, e, h->cls[sorted[s].cfg], c, 0, 0, sorted[s].ecap});
    for (size_t x = s; x < e; ++x) grp.back().max_deg = std::max(grp.back().max_deg, h->cfg[sorted[x].cfg].deg);
    s = e;
  }
  std::stable_sort(grp.begin(), grp.end(), [](const K2Group& a, const K2Group& b) { return a.crit > b.crit; });
  // Launch priorities: a cluster launch needs C free SMs of one GPC at once,
  // so once one-CTA classes hold the SMs it starves until they drain; cluster
  // classes therefore get the highest priority, then the longest critical
  // paths.  (Running the group with the longest K4 -- the largest deg --
  // first instead was measured: the bulk class then starts 36 us late and
  // ends after the chain, Llama +11 %.)
  int least = 0, greatest = 0;
  if (cudaDeviceGetStreamPriorityRange(&least, &greatest) == cudaSuccess && greatest < least) {
    std::vector<size_t> ord(grp.size());
    std::iota(ord.begin(), ord.end(), 0);
    std::stable_sort(ord.begin(), ord.end(), [&](size_t a, size_t b) {
      if ((grp[a].cls.C > 1) != (grp[b].cls.C > 1)) return grp[a].cls.C > 1;
      return grp[a].crit > grp[b].crit;
    });
    for (size_t r = 0; r < ord.size(); ++r) grp[ord[r]].priority = std::min(greatest + (int)r, least);
  }
  all.swap(sorted);
}

static uniap_status ensure_side_streams(uniap_handle* h, size_t n) {
  while (h->side.size() < n) {
    cudaStream_t x;
    cudaEvent_t ev;
    CK(h, cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
    CK(h, cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    h->side.push_back(x);
    h->side_ev.push_back(ev);
  }
  return UNIAP_OK;
}

// Enqueue K2 launches of `grp` (instances at `dinst`) on h->st with fork/join.
// Per-group follow-up on the group's stream (K4 of the group's configs).
struct GroupTail {
  const std::vector<std::pair<int, int>>* ranges;  // [group] -> (li0, count) in the local config list
};

static uniap_status enqueue_k4_range(uniap_handle* h, int li0, int cnt, cudaStream_t st);

static uniap_status enqueue_k2(uniap_handle* h, const std::vector<K2Group>& grp, const Inst* dinst,
                               const int32_t* dcount_per_class, int32_t* Pdev, const GroupTail* tail = nullptr) {
  const bool fork = grp.size() > 1 || tail;
  if (fork) {
    uniap_status s = ensure_side_streams(h, std::max<size_t>(grp.size(), 1));
    if (s != UNIAP_OK) return s;
    CK(h, cudaEventRecord(h->fork_ev, h->st));
  }
  for (size_t g = 0; g < grp.size(); ++g) {
    cudaStream_t st = fork ? h->side[g] : h->st;
    if (fork) CK(h, cudaStreamWaitEvent(st, h->fork_ev, 0));
    const int n = dcount_per_class ? grp[g].max_inst : (int)(grp[g].e - grp[g].s);
    K2Args args{dcount_per_class ? dinst : dinst + grp[g].s,
                dcount_per_class ? dcount_per_class + g : nullptr,
                h->dcfg.p, h->arena.p, Pdev, h->G.p, h->L, h->cap, h->skip,
                grp[g].ecap >= 0 ? grp[g].ecap : h->cap};
    args.tmode = grp[g].cls.TM;  // NEXT-1 launches emit into T
    args.T = h->T.p;
    if (!dcount_per_class) args.tim = h->tim.p;  // forward launches: phase clock
    if (h->trace.p) {  // diagnostics: tag = class shape | forward/backward | group
      const K2Class& k = grp[g].cls;
      args.trace = h->trace.p;
      args.tag = (uint32_t)k.NS | (uint32_t)k.V << 6 | (uint32_t)(k.T / 32) << 10 | (uint32_t)k.C << 16 |
                 (uint32_t)k.DB << 24 | (uint32_t)(dcount_per_class ? 1 : 0) << 25 |
                 (uint32_t)(g & 31) << 26;
    }
    CK(h, k2_launch(grp[g].cls, args, n, st, grp[g].priority));
    h->launches++;
    h->k2_launches++;
    if (tail) {
      const auto& r = (*tail->ranges)[g];
      uniap_status s = enqueue_k4_range(h, r.first, r.second, st);
      if (s != UNIAP_OK) return s;
    }
    if (fork) CK(h, cudaEventRecord(h->side_ev[g], st));
  }
  if (fork)
    for (size_t g = 0; g < grp.size(); ++g) CK(h, cudaStreamWaitEvent(h->st, h->side_ev[g], 0));
  return UNIAP_OK;
}

static uniap_status launch_k2_groups(uniap_handle* h, std::vector<Inst>& all, DevBuf<Inst>& buf, int32_t* Pdev) {
  std::vector<K2Group> grp;
  group_instances(h, all, grp);
  CK(h, buf.ensure(all.size()));
  if (!all.empty()) CK(h, h2d(h, buf.p, all.data(), all.size() * sizeof(Inst)));
  return enqueue_k2(h, grp, buf.p, nullptr, Pdev);
}

static BuildBufs build_bufs(uniap_handle* h) {
  return BuildBufs{h->fwd.p, h->act.p, h->ps.p, h->ctx.p, h->tpc.p, h->chain.p, h->skipb.p, h->edges.p,
                   h->n_edges, h->rmat.p, h->chain_mat.p, h->skip_mat.p, h->any_cut ? h->cut_mat.p : nullptr,
                   h->dcat.p, nullptr, nullptr, nullptr, 0, nullptr, h->ns.p, h->qcfg.p, h->qmax.p, h->qglob.p,
                   h->max_nmt, std::max(1, h->n_src)};
}

// ---------------------------------------------------------------------------
// The launch plan of one (rank, world): data-independent, uploaded once.
// ---------------------------------------------------------------------------
static uniap_status make_plan(uniap_handle* h, int rank, int world, const uniap_record* rec) {
  RunPlan& R = h->plan;
  R.valid = false;  // set again only when every field and upload below succeeded
  std::vector<int> owner;
  lpt(h, world, owner);
  R.local.clear();
  for (int i = 0; i < h->ncfg; ++i)
    if (owner[i] == rank) R.local.push_back(i);
  const int nl = (int)R.local.size();
  // forward instances
  std::vector<Inst> fw;
  for (int i : R.local) forward_instances(h, i, false, fw);
  // executed cells / relaxations: level 1 from the host-trimmed plan, level 2
  // counted by K1f where it trims (k1f_trim); the canonical count is the
  // workload size
  h->cells = h->relax = 0;
  for (auto& x : fw) {
    const uint64_t S = h->cfg[x.cfg].S;
    if (S == 1) continue;  // closed form (k2_closed_s1): no DP cells
    h->cells += (uint64_t)x.n * S * h->Q;
    h->relax += (uint64_t)(x.n - 1) * S * S * h->Q;
  }
  h->cells_canon = 0;
  for (int i : R.local) {
    std::vector<Inst> cv;
    plan_instances(h->L, i, h->cfg[i].deg, h->cfg[i].Sfull, h->cfg[i].skip, false, h->cap, cv);
    for (auto& x : cv) h->cells_canon += (uint64_t)x.n * h->cfg[i].Sfull * h->Q;
  }
  group_instances(h, fw, R.fgrp);
  // local configs ordered by forward group, so each group's K4 takes a range;
  // a config whose sweeps span several groups (several cap levels) runs its
  // K4 after the join (k4rest)
  {
    std::vector<int32_t> ordered, grp_of(h->ncfg, -1);
    std::vector<char> used(h->ncfg, 0);
    for (size_t g = 0; g < R.fgrp.size(); ++g)
      for (size_t j = R.fgrp[g].s; j < R.fgrp[g].e; ++j) {
        int32_t& x = grp_of[fw[j].cfg];
        x = (x == -1 || x == (int32_t)g) ? (int32_t)g : -2;
      }
    R.k4range.assign(R.fgrp.size(), {0, 0});
    for (size_t g = 0; g < R.fgrp.size(); ++g) {
      const int start = (int)ordered.size();
      for (int i : R.local)
        if (!used[i] && grp_of[i] == (int32_t)g) { ordered.push_back(i); used[i] = 1; }
      R.k4range[g] = {start, (int)ordered.size() - start};
    }
    const int rest0 = (int)ordered.size();
    for (int i : R.local)
      if (!used[i]) ordered.push_back(i);
    R.k4rest = {rest0, (int)ordered.size() - rest0};
    R.local.swap(ordered);
  }
  CK(h, h->tim.ensure(2));
  CK(h, h->work.ensure(2 * (size_t)h->ncfg));
  // backward: one device-sized launch per kernel class of the local configs
  std::vector<int32_t> cls_of_cfg(h->ncfg, 0);
  R.bgrp.clear();
  int64_t gmax = 1;
  R.max_deg = 0;
  for (int i : R.local) {
    const CfgDev& d = h->cfg[i];
    int copies = d.skip >= 0 ? d.S : 1;
    if (d.nsk >= 2) {  // NEXT-4: the copies of the run of all sources (bounds any stage's)
      copies = 1;
      for (int j = 0; j < d.nsk && copies <= UNIAP_MAX_COPIES; ++j) copies *= d.S;
      copies = std::min(copies, UNIAP_MAX_COPIES);
    }
    const int bound = d.deg + copies - 1;  // stages + extra skip copies of one stage
    gmax = std::max<int64_t>(gmax, (int64_t)copies * h->L * d.NSP * h->Q);
    R.max_deg = std::max(R.max_deg, std::min(d.deg, h->L));
    int g = -1;
    for (size_t j = 0; j < R.bgrp.size(); ++j)
      if (class_key(R.bgrp[j].cls) == class_key(h->bcls[i])) g = (int)j;
    if (g < 0) {
      g = (int)R.bgrp.size();
      R.bgrp.push_back(K2Group{0, 0, h->bcls[i], 0.0, 0});
    }
    R.bgrp[g].max_inst = std::max(R.bgrp[g].max_inst, bound);
    cls_of_cfg[i] = g;
  }
  if ((int)R.bgrp.size() > MAXCLS) FAIL(h, UNIAP_ERR_ARG, "too many kernel classes");
  // G blocks kept from the forward phase (deg = 1 whole-chain sweeps), after
  // the traceback's own blocks
  std::vector<int64_t> gstore(h->ncfg, -1);
  {
    int64_t off = gmax;
    for (auto& x : fw)
      if (x.emit & 4) {
        const CfgDev& d = h->cfg[x.cfg];
        if (gstore[x.cfg] < 0) {
          gstore[x.cfg] = off;
          off += (int64_t)(d.skip >= 0 && d.skip + 2 <= h->L - 1 ? d.S : 1) * h->L * d.NSP * h->Q;
        }
        x.gofs = gstore[x.cfg] + (int64_t)(x.ks < 0 ? 0 : x.ks) * h->L * d.NSP * h->Q;
      }
    gmax = off;
  }
  CK(h, h->gstore.ensure(h->ncfg));
  CK(h, h2d(h, h->gstore.p, gstore.data(), h->ncfg * 8));
  int max_bw = 1;
  for (auto& g : R.bgrp) max_bw = std::max(max_bw, g.max_inst);
  // device buffers + uploads (outside any graph)
  CK(h, h->P.ensure((size_t)h->P_words));
  if (h->T_words > 0) {  // NEXT-1: T tables, K4c results and suffix scratch
    int maxdeg = 1;
    for (int i = 0; i < h->ncfg; ++i)
      if (h->cut[i]) maxdeg = std::max(maxdeg, h->cfg[i].deg);
    h->zstride = (int64_t)(maxdeg + 2) * h->L * (UNIAP_MAX_STRAT + 1);
    CK(h, h->T.ensure((size_t)h->T_words));
    CK(h, h->zscr.ensure((size_t)std::max(nl, 1) * h->zstride));
    CK(h, h->cutres.ensure((size_t)std::max(nl, 1) * sizeof(CutRes)));
  }
  CK(h, h->inst.ensure(std::max<size_t>(fw.size(), 1)));
  CK(h, h->binst.ensure(max_bw));
  CK(h, h->G.ensure(gmax));
  CK(h, h->cfglist.ensure(std::max(nl, 1)));
  CK(h, h->clsid.ensure(h->ncfg));
  CK(h, h->thetas.ensure((size_t)std::max(nl, 1) * TMAX));
  CK(h, h->ends.ensure((size_t)std::max(nl, 1) * (MAXL + 1)));
  if (!h->k4best.p) {  // K4's running minimum objective (K5a resets it after every run)
    CK(h, h->k4best.ensure(1));
    const long long m = LLONG_MAX;
    CK(h, h2d(h, h->k4best.p, &m, sizeof m));
  }
  CK(h, h->vals.ensure((size_t)std::max(nl, 1) * TMAX));
  CK(h, h->cfgopt.ensure(h->ncfg));
  CK(h, h->win.ensure(1));
  CK(h, h->bwp.ensure(1));
  if (!fw.empty()) CK(h, h2d(h, h->inst.p, fw.data(), fw.size() * sizeof(Inst)));
  {  // per config: its forward instances in the uploaded (grouped) order, for K1f's trim
    std::vector<int32_t> csr(h->ncfg + 1 + fw.size(), 0);
    for (auto& x : fw) csr[x.cfg + 1]++;
    for (int i = 0; i < h->ncfg; ++i) csr[i + 1] += csr[i];
    std::vector<int32_t> fill(csr.begin(), csr.begin() + h->ncfg);
    for (size_t j = 0; j < fw.size(); ++j) csr[h->ncfg + 1 + fill[fw[j].cfg]++] = (int32_t)j;
    int most = 1;
    for (int i = 0; i < h->ncfg; ++i) most = std::max(most, csr[i + 1] - csr[i]);
    R.n_trim = std::min(64, (most + 7) / 8);  // about one sweep per warp
    CK(h, h->inst_csr.ensure(csr.size()));
    CK(h, h2d(h, h->inst_csr.p, csr.data(), csr.size() * 4));
  }
  if (nl > 0) CK(h, h2d(h, h->cfglist.p, R.local.data(), nl * 4));
  CK(h, h2d(h, h->clsid.p, cls_of_cfg.data(), h->ncfg * 4));
  std::vector<int64_t> big(h->ncfg, INT64_MAX);  // non-local configs stay "infeasible"
  CK(h, h2d(h, h->cfgopt.p, big.data(), h->ncfg * 8));
  CK(h, cudaStreamSynchronize(h->st));
  R.rank = rank;
  R.world = world;
  R.rec = rec;
  R.valid = true;
  return UNIAP_OK;
}

static uniap_status enqueue_k4_range(uniap_handle* h, int li0, int cnt, cudaStream_t st) {
  // runs of NEXT-1 configs (K4c over T) and of the others (K4 over P)
  for (int s = li0, e; s < li0 + cnt; s = e) {
    const bool cut = h->cut[h->plan.local[s]];
    int nlev = 1;
    for (e = s; e < li0 + cnt && (bool)h->cut[h->plan.local[e]] == cut; ++e)
      nlev = std::max(nlev, h->cfg[h->plan.local[e]].nlev);
    if (cut) {
      CK(h, launch_k4c(h->dcfg.p, h->arena.p, h->T.p, h->cfglist.p, s, e - s, h->L, h->cfgopt.p, h->cutres.p,
                       h->zscr.p, h->zstride, st));
    } else {
      CK(h, launch_k4(h->dcfg.p, h->arena.p, h->P.p, h->cfglist.p, s, e - s, h->L, nlev, h->thetas.p, h->vals.p,
                      h->ends.p, h->cfgopt.p, h->k4best.p, st));
    }
    h->launches++;
  }
  return UNIAP_OK;
}

// Builder, forward chain-DP classes with their K4, and K5a (the local winner
// and the record header), enqueued on h->st with no host synchronisation.
static uniap_status enqueue_forward(uniap_handle* h, uniap_record* rec) {
  const RunPlan& R = h->plan;
  const int L = h->L, nl = (int)R.local.size();
  if (h->trace.p) CK(h, cudaMemsetAsync(h->trace.p, 0, 8, h->st));
  if (h->level2) {
    // the P fill overlaps the builder (side stream, joined before K2)
    uniap_status s = ensure_side_streams(h, 1);
    if (s != UNIAP_OK) return s;
    CK(h, cudaEventRecord(h->fork_ev, h->st));
    CK(h, cudaStreamWaitEvent(h->side[0], h->fork_ev, 0));
    CK(h, cudaMemsetAsync(h->tim.p, 0, 2 * sizeof(unsigned long long), h->side[0]));  // forward phase clock
    CK(h, launch_fill(h->P.p, h->P_words, INF, h->side[0]));
    CK(h, cudaEventRecord(h->side_ev[0], h->side[0]));
    BuildBufs bb = build_bufs(h);
    bb.inst = h->inst.p;  // K1f trims the forward sweeps of this plan (k1f_trim)
    bb.inst_off = h->inst_csr.p;
    bb.inst_idx = h->inst_csr.p + h->ncfg + 1;
    bb.n_trim = R.n_trim;
    bb.work = h->work.p;
    CK(h, launch_k1(h->cl, bb, h->dcfg.p, h->ncfg, L, h->skip, h->arena.p, h->st));
    CK(h, cudaStreamWaitEvent(h->st, h->side_ev[0], 0));
    h->launches += 3 + (h->n_src >= 2);  // (K1g: NEXT-4 copies)
  } else {
    CK(h, cudaMemsetAsync(h->tim.p, 0, 2 * sizeof(unsigned long long), h->st));  // forward phase clock
    CK(h, launch_fill(h->P.p, h->P_words, INF, h->st));
  }
  h->launches++;
  if (h->T_words > 0) {  // NEXT-1 boundary-strategy tables
    CK(h, launch_fill(h->T.p, h->T_words, INF, h->st));
    h->launches++;
  }

  {
    // K2 per class on side streams, each followed by the K4 of its configs
    GroupTail tail{&R.k4range};
    uniap_status s = enqueue_k2(h, R.fgrp, h->inst.p, nullptr, h->P.p, R.fgrp.empty() ? nullptr : &tail);
    if (s != UNIAP_OK) return s;
    s = enqueue_k4_range(h, R.k4rest.first, R.k4rest.second, h->st);
    if (s != UNIAP_OK) return s;
  }

  RecordArgs ra{rec, h->cells, h->relax, h->level2 ? h->work.p : nullptr, h->cells_canon, nl, L, h->cap,
                h->level2 ? h->qglob.p : nullptr, h->clsid.p, h->binst.p, h->bwp.p,
                h->T_words > 0 ? reinterpret_cast<const CutRes*>(h->cutres.p) : nullptr, h->gstore.p};
  CK(h, launch_k5a(h->dcfg.p, h->arena.p, h->P.p, h->cfglist.p, nl, L, h->ends.p, h->cfgopt.p, h->win.p,
                   h->k4best.p, ra, h->st));
  h->launches += 1;
  return UNIAP_OK;
}

// The winner's traceback: backward sweeps sized on the device (K5a's plan),
// then the strategy walk.
static uniap_status enqueue_traceback(uniap_handle* h, uniap_record* rec) {
  const RunPlan& R = h->plan;
  const int L = h->L;
  {
    uniap_status s = enqueue_k2(h, R.bgrp, h->binst.p, h->bwp.p->count, h->P.p);
    if (s != UNIAP_OK) return s;
  }
  CK(h, launch_k5c_grid(R.max_deg, h->dcfg.p, h->arena.p, h->G.p, h->bwp.p, h->win.p, L, h->cap, rec, h->st));
  if (R.max_deg > 0) h->launches++;
  return UNIAP_OK;
}

// The results into the mapped host block (uniap_fetch: one sync, no copies).
static uniap_status enqueue_publish(uniap_handle* h, uniap_record* rec) {
  auto* fd = h->fb_dev;
  CK(h, launch_publish(reinterpret_cast<int32_t*>(&fd->rec), rec, fd->qg, h->level2 ? h->qglob.p : nullptr, fd->tm,
                       h->tim.p, fd->cfgopt, h->cfgopt.p, h->ncfg, h->st));
  h->launches++;
  return UNIAP_OK;
}

// The whole path for this rank (phase 0), or one half of the split run
// (uniap_run_phase): 1 = up to the local winner, 2 = k_decide against the
// gathered phase-1 records `recs` (the traceback runs only on the rank that
// holds the global winner) and the traceback.  Captured as one CUDA graph.
static uniap_status enqueue_pipeline(uniap_handle* h, uniap_record* rec, int phase = 0,
                                     const uniap_record* recs = nullptr) {
  uniap_status s = UNIAP_OK;
  if (phase == 2) {
    CK(h, launch_decide(recs, h->plan.world, h->plan.rank, h->bwp.p, h->win.p, h->st));
    h->launches++;
  } else if ((s = enqueue_forward(h, rec)) != UNIAP_OK) {
    return s;
  }
  if (phase != 1 && (s = enqueue_traceback(h, rec)) != UNIAP_OK) return s;
  return enqueue_publish(h, rec);
}


static uniap_status run_phase(uniap_handle* h, int32_t rank, int32_t world, void* rec_dev, int phase, const void* recs) {
  if (!h) return UNIAP_ERR_ARG;
  if (!h->ready) FAIL(h, UNIAP_ERR_ARG, "nothing prepared");
  if (world < 1 || rank < 0 || rank >= world) FAIL(h, UNIAP_ERR_ARG, "rank %d / world %d", rank, world);
  CK(h, cudaSetDevice(h->device));
  uniap_record* rec = rec_dev ? (uniap_record*)rec_dev : nullptr;
  if (!rec) {
    CK(h, h->rec.ensure(1));
    rec = h->rec.p;
  }
  h->last_rec = rec;
  if (!h->fb) {  // before any capture: the graph's k_publish writes here
    CK(h, cudaHostAlloc((void**)&h->fb, sizeof(*h->fb), cudaHostAllocMapped));
    CK(h, cudaHostGetDevicePointer((void**)&h->fb_dev, h->fb, 0));
  }
  if (!h->plan.valid || h->plan.rank != rank || h->plan.world != world || h->plan.rec != rec) {
    drop_graphs(h);
    uniap_status s = make_plan(h, rank, world, rec);
    if (s != UNIAP_OK) return s;
  }
  if (phase == 2 && h->ph2_recs != recs && h->graph_ph[1]) {  // its graph reads the gathered records
    cudaGraphExecDestroy(h->graph_ph[1]);
    h->graph_ph[1] = nullptr;
  }
  if (phase == 2) h->ph2_recs = recs;
  cudaGraphExec_t& gx = phase == 0 ? h->graph_exec : h->graph_ph[phase - 1];
  if (getenv("UNIAP_TRACE") && !h->trace.p) {  // diagnostics: allocated before any capture
    CK(h, h->trace.ensure(4 + 4 * (size_t)TRACE_CAP));
    const unsigned long long hdr[2] = {0ull, (unsigned long long)TRACE_CAP};
    CK(h, cudaMemcpy(h->trace.p, hdr, sizeof hdr, cudaMemcpyHostToDevice));
    CK(h, combine_trace(h->trace.p));
    CK(h, builder_trace(h->trace.p));
  }
  const bool use_graph = !env_flag("UNIAP_NO_GRAPH");
  CK(h, cudaEventRecord(h->ev[0], h->st));
  if (use_graph) {
    if (!gx) {
      // capture the pipeline once; replay it on every later run of this plan
      const uint32_t l0 = h->launches, k0 = h->k2_launches;
      CK(h, cudaStreamBeginCapture(h->st, cudaStreamCaptureModeThreadLocal));
      h->capturing = true;
      uniap_status s = enqueue_pipeline(h, rec, phase, (const uniap_record*)recs);
      h->capturing = false;
      cudaGraph_t g = nullptr;
      cudaError_t e = cudaStreamEndCapture(h->st, &g);
      if (s != UNIAP_OK) { if (g) cudaGraphDestroy(g); return s; }
      CK(h, e);
      e = cudaGraphInstantiate(&gx, g, cudaGraphInstantiateFlagUseNodePriority);  // K2 launch priorities
      cudaGraphDestroy(g);
      CK(h, e);
      h->graph_launches = h->launches - l0;
      h->graph_k2 = h->k2_launches - k0;
      h->launches = l0;
      h->k2_launches = k0;
    }
    CK(h, cudaGraphLaunch(gx, h->st));
    h->launches += h->graph_launches;
    h->k2_launches += h->graph_k2;
  } else {
    uniap_status s = enqueue_pipeline(h, rec, phase, (const uniap_record*)recs);
    if (s != UNIAP_OK) return s;
  }
  CK(h, cudaEventRecord(h->ev[3], h->st));
  CK(h, cudaGetLastError());
  h->timed = true;
  return UNIAP_OK;
}

extern "C" uniap_status uniap_run(uniap_handle* h, int32_t rank, int32_t world, void* rec_dev) {
  return run_phase(h, rank, world, rec_dev, 0, nullptr);
}

extern "C" uniap_status uniap_plan_shard(uniap_handle* h, const uniap_model* m, const uniap_cluster* cl,
                                         const uniap_options* o, int32_t rank, int32_t world, void* rec_dev) {
  if (!h) return UNIAP_ERR_ARG;
  if (!rec_dev) FAIL(h, UNIAP_ERR_ARG, "uniap_plan_shard needs the record device buffer");
  uniap_status s = uniap_prepare(h, m, cl, o);
  if (s != UNIAP_OK) return s;
  return uniap_run(h, rank, world, rec_dev);
}

extern "C" uniap_status uniap_run_phase(uniap_handle* h, int32_t rank, int32_t world, void* rec_dev, int32_t phase,
                                        const void* recs_dev) {
  if (!h) return UNIAP_ERR_ARG;
  if (phase != 1 && phase != 2) FAIL(h, UNIAP_ERR_ARG, "phase %d (1 or 2)", phase);
  if (!rec_dev) FAIL(h, UNIAP_ERR_ARG, "a split run needs the record device buffer");
  if (phase == 2 && !recs_dev) FAIL(h, UNIAP_ERR_ARG, "phase 2 needs the gathered phase-1 records");
  if (phase == 2 && (!h->plan.valid || h->plan.rank != rank || h->plan.world != world || h->plan.rec != rec_dev))
    FAIL(h, UNIAP_ERR_ARG, "phase 2 without the phase 1 of the same (rank, world, record)");
  return run_phase(h, rank, world, rec_dev, phase, recs_dev);
}

extern "C" uniap_status uniap_fetch(uniap_handle* h, uniap_result* out) {
  if (!h || !out) return UNIAP_ERR_ARG;
  CK(h, cudaSetDevice(h->device));
  const uniap_record* src = h->last_rec;
  if (!src) FAIL(h, UNIAP_ERR_ARG, "nothing has run on this handle");
  // every result of the run is already on its way into the mapped block
  // (k_publish, the last kernel of the run): one sync, no copies
  (void)src;
  auto* fb = h->fb;
  int64_t* keep = out->cfg_objective;
  CK(h, cudaStreamSynchronize(h->st));
  h->d2h += sizeof fb->rec + (h->level2 ? 16 : 0) + (keep ? h->ncfg * 8 : 0);  // device -> host bytes
  const uniap_record& R = fb->rec;
  h->quantum = h->level2 ? fb->qg[0] : 0;
  if (h->timed) {
    h->ms_dp = 0.f;
    const unsigned long long* tm = fb->tm;
    if (h->tim.p && tm[0] && tm[1] >= ~tm[0]) h->ms_dp = (float)((double)(tm[1] - ~tm[0]) * 1e-6);
    cudaEventElapsedTime(&h->ms_total, h->ev[0], h->ev[3]);
    h->timed = false;
  }
  if (h->trace.p) {  // diagnostics: append this run's K2 timeline to $UNIAP_TRACE
    CK(h, cudaStreamSynchronize(h->st));
    unsigned long long n = 0;
    CK(h, cudaMemcpy(&n, h->trace.p, 8, cudaMemcpyDeviceToHost));
    n = std::min<unsigned long long>(n, TRACE_CAP);
    std::vector<unsigned long long> r(4 * n);
    if (n) CK(h, cudaMemcpy(r.data(), h->trace.p + 4, 32 * n, cudaMemcpyDeviceToHost));
    if (FILE* f = fopen(getenv("UNIAP_TRACE"), "a")) {
      fprintf(f, "run %llu\n", n);
      for (unsigned long long i = 0; i < n; ++i)
        fprintf(f, "%llu %llu %llu %llu\n", r[4 * i], r[4 * i + 1], r[4 * i + 2], r[4 * i + 3]);
      fclose(f);
    }
  }
  memset(out, 0, sizeof *out);
  out->cfg_objective = keep;
  if (keep) memcpy(keep, fb->cfgopt, h->ncfg * 8);
  out->objective = R.objective;
  out->cfg_index = R.cfg_index;
  out->deg = R.deg;
  out->c = R.c;
  out->L = h->L;
  for (int i = 0; i < UNIAP_MAX_LAYERS; ++i) {
    out->stage_of[i] = R.stage_of[i];
    out->strategy_of[i] = R.strategy_of[i];
    out->stage_cost[i] = R.stage_cost[i];
    out->cut_cost[i] = R.cut_cost[i];
    out->stage_mem[i] = R.stage_mem[i];
  }
  out->quantum_ns = h->quantum;
  out->dp_cells = R.dp_cells;
  out->dp_relax = R.dp_relax;
  out->dp_cells_canonical = R.dp_cells_canonical;
  out->ms_gpu_dp = h->ms_dp;
  out->ms_gpu_total = h->ms_total;
  out->h2d_bytes = h->h2d;
  out->d2h_bytes = h->d2h;
  out->n_launches = h->launches;
  out->n_k2_launches = h->k2_launches;
  if (R.status != 0) FAIL(h, (uniap_status)R.status, "device pipeline reported status %d", R.status);
  if (R.objective == INT64_MAX) FAIL(h, UNIAP_ERR_INFEASIBLE, "every candidate config is infeasible");
  return UNIAP_OK;
}

extern "C" uniap_status uniap_solve_tables(uniap_handle* h, const uniap_tables* t, uniap_result* out) {
  uniap_status s = uniap_prepare_tables(h, t);
  if (s != UNIAP_OK) return s;
  s = uniap_run(h, 0, 1, nullptr);
  if (s != UNIAP_OK) return s;
  return uniap_fetch(h, out);
}

extern "C" uniap_status uniap_plan(uniap_handle* h, const uniap_model* m, const uniap_cluster* cl,
                                   const uniap_options* o, uniap_result* out) {
  uniap_status s = uniap_prepare(h, m, cl, o);
  if (s != UNIAP_OK) return s;
  s = uniap_run(h, 0, 1, nullptr);
  if (s != UNIAP_OK) return s;
  return uniap_fetch(h, out);
}

extern "C" uniap_status uniap_interval_table(uniap_handle* h, const uniap_tables* t, int32_t cfg, int32_t* P_out) {
  uniap_status s = uniap_prepare_tables(h, t);
  if (s != UNIAP_OK) return s;
  if (cfg < 0 || cfg >= h->ncfg || !P_out) FAIL(h, UNIAP_ERR_ARG, "cfg index %d", cfg);
  // Own buffers: the captured pipeline graph of the prepared tables bakes in
  // the addresses of h->inst / h->P / h->G, so this call must not reallocate
  // them (a later solve on the same tables replays that graph).  Only the
  // emitted P entries are written (K2 does not store G for emit 1 / 2).
  const int L = h->L;
  std::vector<Inst> fw;
  forward_instances(h, cfg, true, fw);
  CK(h, h->iP.ensure((size_t)h->P_words));
  CK(h, launch_fill(h->iP.p, h->P_words, INF, h->st));
  s = launch_k2_groups(h, fw, h->iinst, h->iP.p);
  if (s != UNIAP_OK) return s;
  CK(h, d2h(h, P_out, h->iP.p + h->cfg[cfg].offP, (size_t)L * L * 4));
  CK(h, cudaStreamSynchronize(h->st));
  CK(h, cudaGetLastError());
  return UNIAP_OK;
}

extern "C" uniap_status uniap_fetch_intervals(uniap_handle* h, int32_t* P_out, int64_t P_len, int64_t* P_words) {
  if (!h) return UNIAP_ERR_ARG;
  if (!h->last_rec || !h->plan.valid || !h->P.p) FAIL(h, UNIAP_ERR_ARG, "nothing has run on this handle");
  const int64_t n = h->P_words;
  if (P_words) *P_words = n;
  if (!P_out) return UNIAP_OK;
  if (P_len < n) FAIL(h, UNIAP_ERR_ARG, "P_len %lld < %lld", (long long)P_len, (long long)n);
  CK(h, cudaSetDevice(h->device));
  CK(h, d2h(h, P_out, h->P.p, (size_t)n * 4));
  CK(h, cudaStreamSynchronize(h->st));
  return UNIAP_OK;
}

extern "C" uniap_status uniap_build_tables(uniap_handle* h, const uniap_model* m, const uniap_cluster* cl,
                                           const uniap_options* o, int32_t* buf, int64_t buf_len, int64_t* words,
                                           int32_t* n_cfg, int32_t* skip_src, int64_t* quantum_ns) {
  h->no_compact = true;  // the documented layout holds every catalogue strategy
  uniap_status s = uniap_prepare(h, m, cl, o);
  h->no_compact = false;
  if (s != UNIAP_OK) return s;
  const int L = h->L;
  int64_t need = 0;
  for (auto& d : h->cfg)
    need += 4 + 2 * (int64_t)L * d.S + (int64_t)(L - 1) * d.S * d.S + (int64_t)L * d.S * d.S + (L - 1) + d.deg + 1 +
            (d.cut ? (int64_t)(L - 1) * d.S * d.S : 0) + 1 + (o->schedule ? (int64_t)d.deg * L * d.S : 0) +
            (d.nsk >= 2 ? (int64_t)d.nsk * L * d.S * d.S : 0);
  if (words) *words = need;
  if (n_cfg) *n_cfg = h->ncfg;
  if (skip_src) *skip_src = h->skip;
  if (!buf) return UNIAP_OK;
  if (buf_len < need) FAIL(h, UNIAP_ERR_ARG, "buffer too small (%lld < %lld)", (long long)buf_len, (long long)need);
  CK(h, launch_k1(h->cl, build_bufs(h), h->dcfg.p, h->ncfg, L, h->skip, h->arena.p, h->st));
  std::vector<int32_t> a(h->arena_words);
  int64_t qg[2];
  CK(h, d2h(h, a.data(), h->arena.p, a.size() * 4));
  CK(h, d2h(h, qg, h->qglob.p, 16));
  CK(h, cudaStreamSynchronize(h->st));
  if (qg[1] != 0) FAIL(h, UNIAP_ERR_RANGE, "modelled value out of range (flags %lld)", (long long)qg[1]);
  if (quantum_ns) *quantum_ns = qg[0];
  // unpack the device layout into the documented block layout
  int64_t w = 0;
  for (int i = 0; i < h->ncfg; ++i) {
    const CfgDev& d = h->cfg[i];
    const int S = d.S, N = d.NSP;
    buf[w++] = d.deg; buf[w++] = d.c; buf[w++] = S; buf[w++] = d.g;
    for (int u = 0; u < L; ++u)
      for (int k = 0; k < S; ++k) buf[w++] = a[d.offA + u * N + k];
    for (int u = 0; u < L; ++u)
      for (int k = 0; k < S; ++k) buf[w++] = a[d.offM + u * N + k];
    for (int e = 0; e + 1 < L; ++e)
      for (int k = 0; k < S; ++k)
        for (int l = 0; l < S; ++l) buf[w++] = a[d.offRf + ((int64_t)e * N + k) * N + l];
    for (int v = 0; v < L; ++v)  // (several sources: 0 here, their tables at the block's tail)
      for (int k = 0; k < S; ++k)
        for (int l = 0; l < S; ++l) buf[w++] = d.nsk >= 2 ? 0 : a[d.offRs + ((int64_t)v * N + k) * N + l];
    for (int e = 0; e + 1 < L; ++e) buf[w++] = a[d.offO + e];
    for (int st = 0; st < d.deg; ++st) buf[w++] = h->scap[i].empty() ? h->cap : h->scap[i][st];
    buf[w++] = d.cut;  // NEXT-1: has_rcut, then Rcut
    for (int e = 0; d.cut && e + 1 < L; ++e)
      for (int k = 0; k < S; ++k)
        for (int l = 0; l < S; ++l) buf[w++] = a[d.offRc + ((int64_t)e * N + k) * N + l];
    buf[w++] = o->schedule;  // 1F1B: has_mstage, then each stage's memory table
    for (int st = 0; o->schedule && st < d.deg; ++st) {
      const int64_t mo = d.deg <= L ? cfg_moff(d, d.lev_of[st], L) : d.offM;  // (deg > L: GPipe's, A-32)
      for (int u = 0; u < L; ++u)
        for (int k = 0; k < S; ++k) buf[w++] = a[mo + u * N + k];
    }
    for (int j = 0; j < (d.nsk >= 2 ? d.nsk : 0); ++j)  // NEXT-4: each source's skip table
      for (int v = 0; v < L; ++v)
        for (int k = 0; k < S; ++k)
          for (int l = 0; l < S; ++l) buf[w++] = a[d.offRs + (((int64_t)j * L + v) * N + k) * N + l];
  }
  return UNIAP_OK;
}

extern "C" uniap_status uniap_pick(const uniap_record* recs, int32_t world, uniap_result* out) {
  if (!recs || world < 1 || !out) return UNIAP_ERR_ARG;
  int best = -1;
  uint64_t cells = 0, relax = 0, canon = 0;
  for (int r = 0; r < world; ++r) {
    const uniap_record& x = recs[r];
    if (x.status != 0) return (uniap_status)x.status;
    cells += x.dp_cells;
    relax += x.dp_relax;
    canon += x.dp_cells_canonical;
    if (x.objective == INT64_MAX) continue;
    if (best < 0) { best = r; continue; }
    const uniap_record& b = recs[best];
    if (x.objective < b.objective || (x.objective == b.objective && (x.deg < b.deg || (x.deg == b.deg && x.c < b.c))))
      best = r;
  }
  int64_t* keep = out->cfg_objective;
  memset(out, 0, sizeof *out);
  out->cfg_objective = keep;
  out->dp_cells = cells;
  out->dp_relax = relax;
  out->dp_cells_canonical = canon;
  out->objective = INT64_MAX;
  out->cfg_index = -1;
  if (best < 0) return UNIAP_ERR_INFEASIBLE;
  const uniap_record& b = recs[best];
  out->objective = b.objective;
  out->cfg_index = b.cfg_index;
  out->deg = b.deg;
  out->c = b.c;
  out->L = b.L;
  for (int i = 0; i < UNIAP_MAX_LAYERS; ++i) {
    out->stage_of[i] = b.stage_of[i];
    out->strategy_of[i] = b.strategy_of[i];
    out->stage_cost[i] = b.stage_cost[i];
    out->cut_cost[i] = b.cut_cost[i];
    out->stage_mem[i] = b.stage_mem[i];
  }
  return UNIAP_OK;
}
