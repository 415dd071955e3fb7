// libclimber C ABI (include/climber.h): context, arena carving, K/V page pool,
// handles, and the per-request orchestration of the SUMI hot path
// (SURVEY §3 call stacks 1-2; PAPER.md L257 serving steps).
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <chrono>
#include <mutex>
#include <thread>
#include <string>
#include <vector>

#include <dlfcn.h>
#include <nccl.h>

#include "../../include/climber.h"
#include "kernels.cuh"

using namespace climber;

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
static thread_local std::string g_last_error;

// NCCL, resolved at run time from the process's libnccl.so.2 (the one torch
// already loaded, else the system one): only multi-GPU contexts need it.
struct NcclApi {
  decltype(&ncclGetUniqueId) get_uid = nullptr;
  decltype(&ncclCommInitRank) init = nullptr;
  decltype(&ncclBroadcast) bcast = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclGetErrorString) err = nullptr;
  decltype(&ncclCommAbort) abort = nullptr;
  decltype(&ncclCommGetAsyncError) async_err = nullptr;
  bool ok = false;
};
static NcclApi& nccl_api() {
  static NcclApi a = [] {
    NcclApi x;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return x;
    x.get_uid = (decltype(x.get_uid))dlsym(h, "ncclGetUniqueId");
    x.init = (decltype(x.init))dlsym(h, "ncclCommInitRank");
    x.bcast = (decltype(x.bcast))dlsym(h, "ncclBroadcast");
    x.destroy = (decltype(x.destroy))dlsym(h, "ncclCommDestroy");
    x.err = (decltype(x.err))dlsym(h, "ncclGetErrorString");
    x.abort = (decltype(x.abort))dlsym(h, "ncclCommAbort");
    x.async_err = (decltype(x.async_err))dlsym(h, "ncclCommGetAsyncError");
    x.ok = x.get_uid && x.init && x.bcast && x.destroy && x.err && x.abort && x.async_err;
    return x;
  }();
  return a;
}

static climber_status fail(climber_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return st;
}

#define CU(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) return fail(CLIMBER_E_CUDA, "%s: %s", #x, cudaGetErrorString(e_)); \
  } while (0)

// ---------------------------------------------------------------------------
// context
// ---------------------------------------------------------------------------
struct Carver {
  char* base;  // nullptr: dry run (size only)
  size_t off = 0;
  template <typename P>
  void take(P*& p, size_t bytes) {
    off = (off + 255) & ~size_t(255);
    p = base ? reinterpret_cast<P*>(base + off) : nullptr;
    off += bytes;
  }
};

struct SlotState {
  uint32_t gen = 1;
  bool live = false;
  int r = 0;
  int kb0 = 0, kb1 = 0;  // blocks whose K/V this handle holds (all, unless encoded block-parallel)
  std::vector<int> pages;
};

struct ProfRec;
struct climber_ctx_s {
  climber_config cfg;
  Dims D;
  size_t esz;           // bytes per stored element (2 bf16, 4 fp32)
  uint16_t ctx_id;
  std::vector<climber_strategy> strat;
  // weights (device)
  void *e_item, *e_act, *e_scn;
  float *g1, *g2, *tau, *fg1, *fg2, *tau_f, *b_se1, *b_se2, *w_head;
  float *bpos = nullptr, *btime = nullptr, *cbias = nullptr;  // relative bias (rel_bias = 1)
  int* hage = nullptr;
  void *w_qkv, *w_o, *w1, *w2, *fw_qkv, *fw_o, *fw1, *fw2, *w_se1, *w_se2;
  float b_head;
  unsigned long long *amask, *smask;
  // K/V pool + per-slot tables (device)
  void* pool;
  long long n_pages;
  int per_slot;  // pages per handle = Nb * L * ppb
  int max_slots;
  int *ptab, *vlen_all, *idx_all, *bad_all, *err;
  // per-call metadata (device) and its pinned host staging
  int64_t *d_ev_off, *d_cand_off;
  int *d_slots, *d_r, *d_ptab_stage;
  char* h_stage;
  size_t stage_bytes;
  cudaEvent_t stage_evt;
  // scratch (device)
  long long rows_cap;
  float* X;
  void *H, *QKV, *O, *Fh;
  // fused-norm bf16 path: bf16 copy of the residual stream and per-row partial
  // sums of squares (pld = d / 128 partials per row, one per GEMM column tile)
  bool fused = false;
  int pld = 1;
  void* Xb;
  float* part;
  // host bookkeeping
  std::mutex mu;
  std::vector<int> free_pages;
  std::vector<int> free_slots;
  std::vector<SlotState> slots;
  long long launches = 0;
  bool use_tc = true;
  int attn_mode = 2;  // bf16 attention: 2 tcgen05 (where supported), 1 mma.sync, 0 SIMT
  bool sync_check = false;
  // profiler
  bool prof = false;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_next = 0;
  std::vector<struct ProfRec> recs;
  // rank_host staging (device, lazily allocated)
  void* io = nullptr;
  size_t io_bytes = 0;
  // latency mode (rank_host with B = 1): the encode + score kernel sequence
  // captured once per (events, candidates) shape and replayed as one CUDA graph
  cudaGraphExec_t g_exec = nullptr;
  long long g_E = -1, g_P = -1;
  void* g_io = nullptr;
  long long g_launches = 0;
  long long g_seen_E = -1, g_seen_P = -1;  // last shape run eagerly
  // serving cache store (NEXT-4): (user_key, r) -> entry; LRU by tick
  struct CacheEntry {
    climber_kv_t kv;
    uint64_t digest;
    int pins;
    unsigned long long tick;
    bool dropped;  // stale while pinned: released on the last unpin
    long long n_s;  // events the cached K/V was built from
  };
  int* d_flags = nullptr;  // incremental append: per-block "a new event matches a_k"
  std::mutex store_mu;
  std::map<std::pair<uint64_t, int>, CacheEntry> store;
  std::vector<CacheEntry> orphans;  // uncached (stale-while-pinned) handles still held by callers
  unsigned long long store_tick = 0;
  long long st_hits = 0, st_miss = 0, st_evict = 0;
  cudaStream_t g_stream = nullptr;          // capture stream
  // latency graph: score layer l starts its attention as soon as the encode
  // wrote layer l's K/V (encode and score on two captured streams)
  cudaStream_t g_stream2 = nullptr;
  // multi-GPU: this rank's NCCL communicator (climber_kv_broadcast)
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
  void* bslab = nullptr;  // broadcast slab (device, slab_bytes)
  std::vector<cudaEvent_t> ov_evt;          // [L + 2]: per-layer K/V ready, fork, join
  bool ov_record = false, ov_wait = false;
  // pipelined replication (climber_encode_user_bcast): [0] extraction done,
  // [1 + l] layer l's pages written, [L + 1] broadcasts done; the root's side stream
  std::vector<cudaEvent_t> bc_evt;
  bool bc_record = false;
  cudaStream_t bc_stream = nullptr;
  bool graphs = true;
};

static uint16_t g_next_ctx_id = 1;
static std::mutex g_ctx_mu;

static climber_kv_t make_handle(const climber_ctx_s* c, int slot, uint32_t gen) {
  uint64_t v = (uint64_t(c->ctx_id) << 48) | (uint64_t(gen & 0xFFFFFF) << 24) | uint64_t(slot + 1);
  return reinterpret_cast<climber_kv_t>(v);
}

static climber_status resolve(climber_ctx_s* c, climber_kv_t kv, int* slot_out) {
  uint64_t v = reinterpret_cast<uint64_t>(kv);
  if (!kv) return fail(CLIMBER_E_INVALID_ARG, "null kv handle");
  if ((v >> 48) != c->ctx_id) return fail(CLIMBER_E_STALE, "kv handle belongs to another ctx");
  int slot = int(v & 0xFFFFFF) - 1;
  uint32_t gen = uint32_t((v >> 24) & 0xFFFFFF);
  if (slot < 0 || slot >= c->max_slots) return fail(CLIMBER_E_STALE, "kv handle slot out of range");
  const SlotState& s = c->slots[slot];
  if (!s.live || (s.gen & 0xFFFFFF) != gen) return fail(CLIMBER_E_STALE, "kv handle released or stale");
  *slot_out = slot;
  return CLIMBER_OK;
}

static bool dims_from(const climber_config* cfg, Dims* D, std::string* why) {
  if (cfg->abi_version != CLIMBER_ABI_VERSION) { *why = "abi_version mismatch"; return false; }
  if (cfg->d <= 0 || cfg->n_heads <= 0 || cfg->d % cfg->n_heads) { *why = "d % n_heads != 0"; return false; }
  int dh = cfg->d / cfg->n_heads;
  if (dh != 16 && dh != 32 && dh != 64) { *why = "d_h must be 16, 32 or 64"; return false; }
  if (cfg->d % 32) { *why = "d must be a multiple of 32"; return false; }
  // the row kernels (k_rmsnorm's per-lane buffer, the embedding kernels' norm
  // partials) cover rows of at most 1024 columns
  if (cfg->d > 1024) { *why = "d must be <= 1024"; return false; }
  if (cfg->n_layers < 1 || cfg->n_blocks < 1 || cfg->n_blocks > 8) { *why = "need L >= 1, 1 <= N_b <= 8"; return false; }
  if (cfg->n_k < 32 || cfg->n_k % 32 || cfg->n_k > 1024) { *why = "n_k must be a multiple of 32 in [32, 1024]"; return false; }
  if (cfg->ffn_mult < 1 || cfg->se_reduction < 1 || (cfg->n_blocks * cfg->d) % cfg->se_reduction ||
      ((cfg->n_blocks * cfg->d) / cfg->se_reduction) % 16) { *why = "bad ffn_mult / se_reduction"; return false; }
  if (cfg->vocab < 1 || cfg->n_actions < 1 || cfg->n_actions > 64 || cfg->n_scenarios < 1 || cfg->n_scenarios > 64) {
    *why = "bad vocabulary sizes"; return false; }
  if (cfg->max_candidates < 1) { *why = "max_candidates < 1"; return false; }
  if (cfg->dtype != CLIMBER_BF16 && cfg->dtype != CLIMBER_FP32) { *why = "bad dtype"; return false; }
  if (cfg->page_tokens != PAGE) { *why = "page_tokens must be 64"; return false; }
  if (!(cfg->rms_eps >= 0.f)) { *why = "rms_eps < 0"; return false; }
  if (cfg->max_batch_users < 1 || cfg->max_wave_users < 1 || cfg->max_wave_pairs < cfg->max_candidates ||
      cfg->kv_pages < 1) { *why = "bad capacity fields (max_wave_pairs must be >= max_candidates)"; return false; }
  D->d = cfg->d; D->h = cfg->n_heads; D->dh = dh; D->L = cfg->n_layers; D->Nb = cfg->n_blocks; D->nk = cfg->n_k;
  D->F = cfg->ffn_mult * cfg->d; D->Dse = cfg->n_blocks * cfg->d; D->Hse = D->Dse / cfg->se_reduction;
  D->V = cfg->vocab; D->A = cfg->n_actions; D->R = cfg->n_scenarios; D->Mmax = cfg->max_candidates;
  D->causal = cfg->hist_causal ? 1 : 0; D->ppb = (cfg->n_k + PAGE - 1) / PAGE; D->eps = cfg->rms_eps;
  D->bpos = D->btime = nullptr; D->hage = nullptr; D->cbias = nullptr;
  if (cfg->rel_bias != 0 && cfg->rel_bias != 1) { *why = "rel_bias must be 0 or 1"; return false; }
  if (cfg->rel_bias && cfg->dtype == CLIMBER_BF16 && !((dh == 32 || dh == 64) && cfg->n_k % PAGE == 0)) {
    *why = "rel_bias on the bf16 path needs d_h in {32, 64} and n_k % 64 == 0 (tcgen05 attention)";
    return false;
  }
  return true;
}

static void carve(climber_ctx_s* c, Carver& cv) {
  const Dims& D = c->D;
  const size_t e = c->esz;
  const size_t d = D.d, L = D.L, Nb = D.Nb, F = D.F;
  cv.take(c->e_item, (size_t)D.V * d * e);
  cv.take(c->e_act, (size_t)D.A * d * e);
  cv.take(c->e_scn, (size_t)D.R * d * e);
  cv.take(c->g1, Nb * L * d * 4);
  cv.take(c->g2, Nb * L * d * 4);
  cv.take(c->w_qkv, Nb * L * 3 * d * d * e);
  cv.take(c->w_o, Nb * L * d * d * e);
  cv.take(c->w1, Nb * L * F * d * e);
  cv.take(c->w2, Nb * L * d * F * e);
  cv.take(c->tau, L * Nb * D.R * D.h * 4);
  cv.take(c->fg1, d * 4);
  cv.take(c->fg2, d * 4);
  cv.take(c->fw_qkv, 3 * d * d * e);
  cv.take(c->fw_o, d * d * e);
  cv.take(c->fw1, F * d * e);
  cv.take(c->fw2, d * F * e);
  cv.take(c->tau_f, (size_t)D.R * D.h * 4);
  cv.take(c->w_se1, (size_t)D.Hse * D.Dse * e);
  cv.take(c->b_se1, (size_t)D.Hse * 4);
  cv.take(c->w_se2, (size_t)D.Dse * D.Hse * e);
  cv.take(c->b_se2, (size_t)D.Dse * 4);
  cv.take(c->w_head, (size_t)D.Dse * 4);
  cv.take(c->amask, Nb * 8);
  cv.take(c->smask, Nb * 8);
  if (c->cfg.rel_bias) {
    cv.take(c->bpos, L * Nb * D.R * D.h * NB_POS * 4);
    cv.take(c->btime, L * Nb * D.R * D.h * NB_TIME * 4);
  }
  // K/V pool: page = [2][h][64][dh]
  c->per_slot = D.Nb * D.L * D.ppb;
  c->n_pages = c->cfg.kv_pages;
  c->max_slots = (int)(c->n_pages / c->per_slot);
  cv.take(c->pool, (size_t)c->n_pages * 2 * PAGE * d * e);
  size_t S = (size_t)(c->max_slots > 0 ? c->max_slots : 1);
  cv.take(c->ptab, S * c->per_slot * 4);
  cv.take(c->vlen_all, S * Nb * 4);
  cv.take(c->idx_all, S * Nb * D.nk * 4);
  cv.take(c->bad_all, S * 4);
  cv.take(c->err, 256);
  if (c->cfg.rel_bias) {  // per handle: history token ages at the request time, candidate bias rows
    cv.take(c->hage, S * Nb * D.nk * 4);
    cv.take(c->cbias, S * L * Nb * D.h * D.nk * 4);
  }
  // per-call metadata
  size_t Bm = c->cfg.max_batch_users;
  cv.take(c->d_ev_off, (Bm + 1) * 8);
  cv.take(c->d_cand_off, (2 * Bm + 1) * 8);
  cv.take(c->d_slots, Bm * 4);
  cv.take(c->d_r, Bm * 4);
  cv.take(c->d_ptab_stage, Bm * c->per_slot * 4);
  // scratch
  long long rows_h = (long long)c->cfg.max_wave_users * D.nk * D.Nb;  // grouped encode: all blocks at once
  long long rows_c = (long long)c->cfg.max_wave_pairs * D.Nb;
  c->rows_cap = rows_h > rows_c ? rows_h : rows_c;
  size_t R = (size_t)c->rows_cap;
  cv.take(c->X, R * d * 4);
  cv.take(c->H, R * d * e);
  cv.take(c->QKV, R * 3 * d * e);
  cv.take(c->O, R * d * e);
  cv.take(c->Fh, R * F * e);
  c->pld = D.d >= 128 ? D.d / 128 : 1;  // one partial per 128 columns of the RESID_NORM GEMMs
  cv.take(c->Xb, R * d * 2);
  cv.take(c->part, R * c->pld * 4);
}

// ---------------------------------------------------------------------------
// weight upload (host fp32 [in][out] -> device T, GEMM B operands K-major)
// ---------------------------------------------------------------------------
static uint16_t bf16_rne(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return 0x7fc0;
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

struct Uploader {
  climber_ctx_s* c;
  std::vector<char> buf;
  climber_status st = CLIMBER_OK;
  // copy `n` values, optionally transposing each of `batch` [rows][cols] matrices
  void put(void* dst, const float* src, size_t batch, size_t rows, size_t cols, bool transpose, bool as_T) {
    if (st != CLIMBER_OK) return;
    size_t n = batch * rows * cols, es = as_T ? c->esz : 4;
    buf.resize(n * es);
    for (size_t b = 0; b < batch; ++b)
      for (size_t i = 0; i < rows; ++i)
        for (size_t j = 0; j < cols; ++j) {
          size_t si = b * rows * cols + i * cols + j;
          size_t di = transpose ? b * rows * cols + j * rows + i : si;
          float v = src[si];
          if (es == 2) {
            uint16_t h = bf16_rne(v);
            memcpy(&buf[di * 2], &h, 2);
          } else {
            memcpy(&buf[di * 4], &v, 4);
          }
        }
    cudaError_t e = cudaMemcpy(dst, buf.data(), n * es, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) st = fail(CLIMBER_E_CUDA, "weight upload: %s", cudaGetErrorString(e));
  }
};

extern "C" size_t climber_arena_bytes(const climber_config* cfg) {
  if (!cfg) return 0;
  climber_ctx_s c;
  std::string why;
  if (!dims_from(cfg, &c.D, &why)) return 0;
  c.cfg = *cfg;
  c.esz = cfg->dtype == CLIMBER_BF16 ? 2 : 4;
  Carver cv{nullptr};
  carve(&c, cv);
  return cv.off + 256;
}

extern "C" climber_status climber_create(const climber_config* cfg, const climber_strategy* strategies,
                                         const climber_weights* w, void* arena, size_t arena_bytes, int32_t rank,
                                         int32_t world, const void* nccl_uid, climber_ctx_t* out) {
  try {
    if (!cfg || !strategies || !w || !arena || !out) return fail(CLIMBER_E_INVALID_ARG, "null argument");
    if (world < 1 || rank < 0 || rank >= world) return fail(CLIMBER_E_INVALID_ARG, "rank/world out of range");
    if (world > 1 && !nccl_uid) return fail(CLIMBER_E_INVALID_ARG, "world > 1 needs an NCCL unique id");
    if (nccl_uid && !nccl_api().ok) return fail(CLIMBER_E_UNSUPPORTED, "libnccl.so.2 not loadable");
    if (reinterpret_cast<uintptr_t>(arena) % 256) return fail(CLIMBER_E_INVALID_ARG, "arena must be 256-byte aligned");
    std::string why;
    Dims D;
    if (!dims_from(cfg, &D, &why)) return fail(CLIMBER_E_CONFIG, "config: %s", why.c_str());
    for (int k = 0; k < cfg->n_blocks; ++k)
      if (!strategies[k].action_mask || !strategies[k].scenario_mask)
        return fail(CLIMBER_E_CONFIG, "strategy %d has an empty filter", k);
    const float* need[] = {w->emb_item, w->emb_act, w->emb_scn, w->g1, w->w_qkv, w->w_o, w->g2, w->w1, w->w2,
                           w->tau, w->f_g1, w->f_w_qkv, w->f_w_o, w->f_g2, w->f_w1, w->f_w2, w->tau_f,
                           w->w_se1, w->b_se1, w->w_se2, w->b_se2, w->w_head};
    for (const float* p : need)
      if (!p) return fail(CLIMBER_E_INVALID_ARG, "null weight pointer");
    if (cfg->rel_bias && (!w->b_pos || !w->b_time))
      return fail(CLIMBER_E_INVALID_ARG, "rel_bias = 1 needs the b_pos and b_time tables");
    size_t ntau = (size_t)D.L * D.Nb * D.R * D.h;
    for (size_t i = 0; i < ntau; ++i)
      if (!(w->tau[i] > 0.f) || !std::isfinite(w->tau[i])) return fail(CLIMBER_E_CONFIG, "tau[%zu] <= 0 or non-finite", i);
    for (size_t i = 0; i < (size_t)D.R * D.h; ++i)
      if (!(w->tau_f[i] > 0.f) || !std::isfinite(w->tau_f[i])) return fail(CLIMBER_E_CONFIG, "tau_f[%zu] <= 0 or non-finite", i);

    auto* c = new climber_ctx_s();
    c->cfg = *cfg;
    c->D = D;
    c->esz = cfg->dtype == CLIMBER_BF16 ? 2 : 4;
    {
      std::lock_guard<std::mutex> g(g_ctx_mu);
      c->ctx_id = g_next_ctx_id++;
      if (g_next_ctx_id == 0) g_next_ctx_id = 1;
    }
    c->strat.assign(strategies, strategies + cfg->n_blocks);
    Carver dry{nullptr};
    carve(c, dry);
    if (dry.off + 256 > arena_bytes) {
      delete c;
      return fail(CLIMBER_E_CAPACITY, "arena too small: need %zu bytes", dry.off + 256);
    }
    if (c->max_slots < 1) {
      delete c;
      return fail(CLIMBER_E_CAPACITY, "kv_pages %lld < pages per handle", (long long)cfg->kv_pages);
    }
    Carver cv{reinterpret_cast<char*>(arena)};
    carve(c, cv);
    // bf16: tcgen05 GEMMs and attention wherever supported (d_h 32 / 64),
    // mma.sync attention for d_h = 16; fp32: the SIMT verification kernels
    c->use_tc = true;
    c->attn_mode = 2;
    const char* sc = getenv("CLIMBER_SYNC_CHECK");
    c->sync_check = sc && atoi(sc) != 0;
    c->graphs = true;

    const size_t d = D.d, L = D.L, Nb = D.Nb, F = D.F;
    // Fused-norm bf16 path: every RMSNorm gain is folded into the rows (input
    // dimension) of the weight matrix that consumes the normalised activations,
    // W' = diag(g) W (rounded to bf16 once), and 1/rms is applied per row in
    // that GEMM's epilogue from the producer's partial sums of squares.
    c->fused = cfg->dtype == CLIMBER_BF16 && c->use_tc && gemm_tc_available() && D.d % 128 == 0 &&
               (D.dh == 32 || D.dh == 64) && D.Hse % 128 == 0;
    std::vector<float> wqkv_f, w1_f, fwqkv_f, fw1_f;
    const float *w_qkv = w->w_qkv, *w1 = w->w1, *f_w_qkv = w->f_w_qkv, *f_w1 = w->f_w1;
    if (c->fused) {
      auto fold = [](std::vector<float>& dst, const float* W, const float* g, size_t batch, size_t rows, size_t cols) {
        dst.resize(batch * rows * cols);
        for (size_t b = 0; b < batch; ++b)
          for (size_t i = 0; i < rows; ++i)
            for (size_t j = 0; j < cols; ++j)
              dst[(b * rows + i) * cols + j] = g[b * rows + i] * W[(b * rows + i) * cols + j];
      };
      fold(wqkv_f, w->w_qkv, w->g1, Nb * L, d, 3 * d);
      fold(w1_f, w->w1, w->g2, Nb * L, d, F);
      fold(fwqkv_f, w->f_w_qkv, w->f_g1, 1, d, 3 * d);
      fold(fw1_f, w->f_w1, w->f_g2, 1, d, F);
      w_qkv = wqkv_f.data();
      w1 = w1_f.data();
      f_w_qkv = fwqkv_f.data();
      f_w1 = fw1_f.data();
    }
    Uploader up{c};
    up.put(c->e_item, w->emb_item, 1, D.V, d, false, true);
    up.put(c->e_act, w->emb_act, 1, D.A, d, false, true);
    up.put(c->e_scn, w->emb_scn, 1, D.R, d, false, true);
    up.put(c->g1, w->g1, 1, Nb * L, d, false, false);
    up.put(c->g2, w->g2, 1, Nb * L, d, false, false);
    up.put(c->w_qkv, w_qkv, Nb * L, d, 3 * d, true, true);
    up.put(c->w_o, w->w_o, Nb * L, d, d, true, true);
    up.put(c->w1, w1, Nb * L, d, F, true, true);
    up.put(c->w2, w->w2, Nb * L, F, d, true, true);
    up.put(c->tau, w->tau, 1, 1, ntau, false, false);
    up.put(c->fg1, w->f_g1, 1, 1, d, false, false);
    up.put(c->fg2, w->f_g2, 1, 1, d, false, false);
    up.put(c->fw_qkv, f_w_qkv, 1, d, 3 * d, true, true);
    up.put(c->fw_o, w->f_w_o, 1, d, d, true, true);
    up.put(c->fw1, f_w1, 1, d, F, true, true);
    up.put(c->fw2, w->f_w2, 1, F, d, true, true);
    up.put(c->tau_f, w->tau_f, 1, 1, (size_t)D.R * D.h, false, false);
    up.put(c->w_se1, w->w_se1, 1, D.Dse, D.Hse, true, true);
    up.put(c->b_se1, w->b_se1, 1, 1, D.Hse, false, false);
    up.put(c->w_se2, w->w_se2, 1, D.Hse, D.Dse, true, true);
    up.put(c->b_se2, w->b_se2, 1, 1, D.Dse, false, false);
    up.put(c->w_head, w->w_head, 1, 1, D.Dse, false, false);
    if (cfg->rel_bias) {  // fp32 tables, as given
      up.put(c->bpos, w->b_pos, 1, 1, (size_t)L * Nb * D.R * D.h * NB_POS, false, false);
      up.put(c->btime, w->b_time, 1, 1, (size_t)L * Nb * D.R * D.h * NB_TIME, false, false);
      c->D.bpos = c->bpos;
      c->D.btime = c->btime;
      c->D.hage = c->hage;
      c->D.cbias = c->cbias;
    }
    if (up.st != CLIMBER_OK) {
      delete c;
      return up.st;
    }
    c->b_head = w->b_head;
    std::vector<unsigned long long> am(Nb), sm(Nb);
    for (size_t k = 0; k < Nb; ++k) {
      am[k] = strategies[k].action_mask;
      sm[k] = strategies[k].scenario_mask;
    }
    CU(cudaMemcpy(c->amask, am.data(), Nb * 8, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(c->smask, sm.data(), Nb * 8, cudaMemcpyHostToDevice));
    CU(cudaMemset(c->err, 0, 256));
    // host state
    c->free_pages.resize(c->n_pages);
    for (long long i = 0; i < c->n_pages; ++i) c->free_pages[i] = (int)(c->n_pages - 1 - i);
    c->slots.resize(c->max_slots);
    c->free_slots.resize(c->max_slots);
    for (int i = 0; i < c->max_slots; ++i) c->free_slots[i] = c->max_slots - 1 - i;
    size_t Bm = cfg->max_batch_users;
    c->stage_bytes = (Bm + 1) * 8 + (2 * Bm + 1) * 8 + Bm * 8 + Bm * (size_t)c->per_slot * 4 + 1024;
    CU(cudaMallocHost(&c->h_stage, c->stage_bytes));
    CU(cudaEventCreateWithFlags(&c->stage_evt, cudaEventDisableTiming));
    CU(cudaEventRecord(c->stage_evt, 0));
    CU(cudaDeviceSynchronize());
    c->rank = rank;
    c->world = world;
    if (nccl_uid) {  // collective: every rank of the group creates its ctx concurrently
      ncclUniqueId id;
      memcpy(&id, nccl_uid, sizeof(id));
      ncclResult_t nr = nccl_api().init(&c->comm, world, id, rank);
      if (nr != ncclSuccess) {
        c->comm = nullptr;
        const char* m = nccl_api().err(nr);
        delete c;
        return fail(CLIMBER_E_NCCL, "ncclCommInitRank: %s", m);
      }
    }
    *out = c;
    return CLIMBER_OK;
  } catch (const std::exception& ex) {
    return fail(CLIMBER_E_CUDA, "create: %s", ex.what());
  } catch (...) {
    return fail(CLIMBER_E_CUDA, "create: unknown exception");
  }
}

extern "C" climber_status climber_destroy(climber_ctx_t c) {
  if (!c) return fail(CLIMBER_E_INVALID_ARG, "null ctx");
  cudaDeviceSynchronize();
  if (c->h_stage) cudaFreeHost(c->h_stage);
  if (c->io) cudaFree(c->io);
  if (c->g_exec) cudaGraphExecDestroy(c->g_exec);
  if (c->comm) nccl_api().destroy(c->comm);
  if (c->bslab) cudaFree(c->bslab);
  if (c->g_stream) cudaStreamDestroy(c->g_stream);
  if (c->g_stream2) cudaStreamDestroy(c->g_stream2);
  for (cudaEvent_t ev : c->ov_evt) cudaEventDestroy(ev);
  if (c->bc_stream) cudaStreamDestroy(c->bc_stream);
  for (cudaEvent_t ev : c->bc_evt) cudaEventDestroy(ev);
  if (c->d_flags) cudaFree(c->d_flags);
  cudaEventDestroy(c->stage_evt);
  for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
  delete c;
  return CLIMBER_OK;
}

// ---------------------------------------------------------------------------
// GEMM dispatch: tcgen05 tensor cores for bf16, SIMT for the fp32 build
// ---------------------------------------------------------------------------
// Profiler: CUDA events on the launching stream around each launch, per class.
struct ProfRec {
  int cls;
  cudaEvent_t e0, e1;
  double flops, bytes;
};

static cudaEvent_t prof_event(climber_ctx_s* c) {
  if (c->ev_next == c->ev_pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    c->ev_pool.push_back(e);
  }
  return c->ev_pool[c->ev_next++];
}

struct Prof {
  climber_ctx_s* c;
  int cls;
  cudaStream_t s;
  double flops, bytes;
  cudaEvent_t e0 = nullptr;
  Prof(climber_ctx_s* c_, int cls_, cudaStream_t s_, double flops_ = 0, double bytes_ = 0)
      : c(c_), cls(cls_), s(s_), flops(flops_), bytes(bytes_) {
    c->launches++;
    if (c->prof) {
      e0 = prof_event(c);
      cudaEventRecord(e0, s);
    }
  }
  ~Prof() {
    if (e0) {
      cudaEvent_t e1 = prof_event(c);
      cudaEventRecord(e1, s);
      c->recs.push_back({cls, e0, e1, flops, bytes});
    }
  }
};

// GEMM dispatch: tcgen05 tensor cores for bf16, SIMT for the fp32 build
template <typename T>
static void gemm(climber_ctx_s* c, int cls, const T* A, long long lda, const T* B, long long ldb, long long M, int N,
                 int K, const Epilogue& e, cudaStream_t s) {
  Prof p(c, cls, s, 2.0 * M * N * K);
  if constexpr (std::is_same<T, bf16>::value) {
    if (c->use_tc && gemm_tc_supported(M, N, K, lda, ldb)) {
      launch_gemm_tc(A, lda, B, ldb, M, N, K, e, s);
      return;
    }
  }
  launch_gemm_simt<T>(A, lda, B, ldb, M, N, K, e, s);
}

static Epilogue epi_store(void* out, long long ldo, int act = ACT_NONE, const float* bias = nullptr) {
  Epilogue e{};
  e.kind = EPI_STORE; e.act = act; e.out = out; e.ldo = ldo; e.bias = bias;
  return e;
}
static Epilogue epi_resid(float* out, long long ldo) {
  Epilogue e{};
  e.kind = EPI_RESID; e.out = out; e.ldo = ldo;
  return e;
}

// ---------------------------------------------------------------------------
// encode: one wave of U users (SURVEY §3 call stack 1)
// ---------------------------------------------------------------------------
template <typename T>
static void encode_wave(climber_ctx_s* c, const EventsDev& ev, int u0, int U, long long n_events, cudaStream_t s) {
  const Dims& D = c->D;
  const long long rows = (long long)U * D.nk;
  const long long d = D.d, F = D.F;
  const double es = (double)c->esz;
  const int* wslot = c->d_slots + u0;
  const int* wr = c->d_r + u0;
  {
    Prof p(c, CLIMBER_K_EXTRACT, s, 0, (double)n_events * 14 + (double)U * D.Nb * D.nk * 4);
    launch_extract(ev, c->d_ev_off + u0, wslot, U, c->amask, c->smask, c->idx_all, c->vlen_all, c->bad_all, c->err,
                   D, s);
  }
  if (c->cfg.rel_bias) {
    Prof p(c, CLIMBER_K_OTHER, s, 0, (double)U * D.L * D.Nb * D.h * D.nk * 12);
    launch_cand_bias(wslot, c->d_r + u0, U, c->vlen_all, D, s);
  }
  T* H = (T*)c->H;
  T* Qb = (T*)c->QKV;
  T* O = (T*)c->O;
  T* Fh = (T*)c->Fh;
  const double norm_bytes = (double)rows * d * (4 + es);
  const double causal_pairs = D.causal ? (double)D.nk * (D.nk + 1) / 2 : (double)D.nk * D.nk;
  for (int k = 0; k < D.Nb; ++k) {
    {
      Prof p(c, CLIMBER_K_EMBED, s, 0, (double)rows * d * (3 * es + 4));
      launch_embed_hist<T>(ev, c->d_ev_off + u0, wslot, U, c->idx_all, c->vlen_all, c->bad_all, (const T*)c->e_item,
                           (const T*)c->e_act, (const T*)c->e_scn, c->X, (T*)nullptr, nullptr, 0, k, D, s);
    }
    for (int l = 0; l < D.L; ++l) {
      const size_t kl = (size_t)k * D.L + l;
      {
        Prof p(c, CLIMBER_K_RMSNORM, s, 0, norm_bytes);
        launch_rmsnorm<T>(c->X, d, c->g1 + kl * d, H, d, rows, D.d, D.eps, s);
      }
      Epilogue e{};
      e.kind = EPI_QKV_PAGES; e.out = Qb; e.ldo = d; e.pool = c->pool; e.ptab = c->ptab; e.wave_slot = wslot;
      e.pool_rows = c->n_pages * 2 * PAGE;
      e.blk = k; e.layer = l; e.d = D.d; e.h = D.h; e.dh = D.dh; e.nk = D.nk; e.Nb = D.Nb; e.L = D.L; e.ppb = D.ppb;
      const T* Wqkv = (const T*)c->w_qkv + kl * 3 * d * d;
      if (l < D.L - 1) {
        e.col_off = 0;
        gemm<T>(c, CLIMBER_K_GEMM_QKV, H, d, Wqkv, d, rows, 3 * D.d, D.d, e, s);
        {
          Prof p(c, CLIMBER_K_ATTN_HIST, s, 4.0 * U * causal_pairs * d, (double)rows * d * es * 4);
          if constexpr (std::is_same<T, bf16>::value) {
            if (c->attn_mode == 2 && attn_tc_supported(D.dh, D.nk, true)) {
              launch_attn_hist_tc(Qb, wslot, wr, U, (const T*)c->pool, c->n_pages * 2 * PAGE, c->ptab, c->vlen_all,
                                  c->tau, O, k, l, D, s);
            } else if (c->attn_mode >= 1) {
              launch_attn_hist_mma(Qb, wslot, wr, U, (const T*)c->pool, c->ptab, c->vlen_all, c->tau, O, k, l, D, s);
            } else {
              launch_attn_hist<T>(Qb, wslot, wr, U, (const T*)c->pool, c->ptab, c->vlen_all, c->tau, O, k, l, D, s);
            }
          } else {
            launch_attn_hist<T>(Qb, wslot, wr, U, (const T*)c->pool, c->ptab, c->vlen_all, c->tau, O, k, l, D, s);
          }
        }
        gemm<T>(c, CLIMBER_K_GEMM_O, O, d, (const T*)c->w_o + kl * d * d, d, rows, D.d, D.d, epi_resid(c->X, d), s);
        {
          Prof p(c, CLIMBER_K_RMSNORM, s, 0, norm_bytes);
          launch_rmsnorm<T>(c->X, d, c->g2 + kl * d, H, d, rows, D.d, D.eps, s);
        }
        gemm<T>(c, CLIMBER_K_GEMM_FFN_UP, H, d, (const T*)c->w1 + kl * F * d, d, rows, D.F, D.d,
                epi_store(Fh, F, ACT_SILU), s);
        gemm<T>(c, CLIMBER_K_GEMM_FFN_DOWN, Fh, F, (const T*)c->w2 + kl * d * F, F, rows, D.d, D.F,
                epi_resid(c->X, d), s);
      } else {
        // last layer: only K/V of the history are ever read -> N = 2d
        e.col_off = D.d;
        gemm<T>(c, CLIMBER_K_GEMM_QKV, H, d, Wqkv + d * d, d, rows, 2 * D.d, D.d, e, s);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// score: one wave of U users / P pairs (SURVEY §3 call stack 2)
// ---------------------------------------------------------------------------
template <typename T>
static void score_wave(climber_ctx_s* c, const int32_t* items, const int64_t* wcand, int u0, int U, long long P,
                       int Mmax_wave, float* scores, cudaStream_t s) {
  const Dims& D = c->D;
  const long long d = D.d, F = D.F, Nb = D.Nb, ldC = Nb * d;
  const double es = (double)c->esz;
  const int* wslot = c->d_slots + u0;
  const int* wr = c->d_r + u0;
  T* H = (T*)c->H;
  T* QKV = (T*)c->QKV;
  T* O = (T*)c->O;
  T* Fh = (T*)c->Fh;
  float* X = c->X;  // C[p][k][d]
  {
    Prof p(c, CLIMBER_K_EMBED, s, 0, (double)P * d * (2 * es + 4 * Nb));
    launch_embed_cand<T>(items, wcand, wr, U, P, (const T*)c->e_item, (const T*)c->e_scn, X, (T*)nullptr, nullptr, 0,
                         c->err, D, s);
  }
  const double norm_bytes = (double)P * d * (4 + es);
  for (int k = 0; k < D.Nb; ++k) {
    float* Ck = X + k * d;
    for (int l = 0; l < D.L; ++l) {
      const size_t kl = (size_t)k * D.L + l;
      {
        Prof p(c, CLIMBER_K_RMSNORM, s, 0, norm_bytes);
        launch_rmsnorm<T>(Ck, ldC, c->g1 + kl * d, H, d, P, D.d, D.eps, s);
      }
      gemm<T>(c, CLIMBER_K_GEMM_QKV, H, d, (const T*)c->w_qkv + kl * 3 * d * d, d, P, 3 * D.d, D.d,
              epi_store(QKV, 3 * d), s);
      {
        Prof p(c, CLIMBER_K_ATTN_SUMI, s, 4.0 * P * (D.nk + 1) * d,
               (double)P * d * es * 4 + (double)U * D.nk * d * 2 * es);
        if constexpr (std::is_same<T, bf16>::value) {
          if (c->attn_mode == 2 && attn_tc_supported(D.dh, D.nk, false)) {
            launch_attn_sumi_tc(QKV, P, wcand, wslot, wr, U, Mmax_wave, (const T*)c->pool, c->n_pages * 2 * PAGE,
                                c->ptab, c->vlen_all, c->tau, O, k, l, D, s);
          } else if (c->attn_mode >= 1) {
            launch_attn_sumi_mma(QKV, wcand, wslot, wr, U, Mmax_wave, (const T*)c->pool, c->ptab, c->vlen_all, c->tau,
                                 O, k, l, D, s);
          } else {
            launch_attn_sumi<T>(QKV, wcand, wslot, wr, U, Mmax_wave, (const T*)c->pool, c->ptab, c->vlen_all, c->tau,
                                O, k, l, D, s);
          }
        } else {
          launch_attn_sumi<T>(QKV, wcand, wslot, wr, U, Mmax_wave, (const T*)c->pool, c->ptab, c->vlen_all, c->tau, O,
                              k, l, D, s);
        }
      }
      gemm<T>(c, CLIMBER_K_GEMM_O, O, d, (const T*)c->w_o + kl * d * d, d, P, D.d, D.d, epi_resid(Ck, ldC), s);
      {
        Prof p(c, CLIMBER_K_RMSNORM, s, 0, norm_bytes);
        launch_rmsnorm<T>(Ck, ldC, c->g2 + kl * d, H, d, P, D.d, D.eps, s);
      }
      gemm<T>(c, CLIMBER_K_GEMM_FFN_UP, H, d, (const T*)c->w1 + kl * F * d, d, P, D.F, D.d,
              epi_store(Fh, F, ACT_SILU), s);
      gemm<T>(c, CLIMBER_K_GEMM_FFN_DOWN, Fh, F, (const T*)c->w2 + kl * d * F, F, P, D.d, D.F, epi_resid(Ck, ldC),
              s);
    }
  }
  // ---- BGF (Eq. 4): fusion ATL over the N_b tokens of every pair, rows = P*N_b
  const long long R = P * Nb;
  {
    Prof p(c, CLIMBER_K_RMSNORM, s, 0, (double)R * d * (4 + es));
    launch_rmsnorm<T>(X, d, c->fg1, H, d, R, D.d, D.eps, s);
  }
  gemm<T>(c, CLIMBER_K_GEMM_QKV, H, d, (const T*)c->fw_qkv, d, R, 3 * D.d, D.d, epi_store(QKV, 3 * d), s);
  {
    Prof p(c, CLIMBER_K_ATTN_FUSION, s, 4.0 * P * Nb * Nb * d, (double)R * d * es * 4);
    launch_attn_fusion<T>(QKV, wcand, wr, U, P, c->tau_f, O, D, s);
  }
  gemm<T>(c, CLIMBER_K_GEMM_O, O, d, (const T*)c->fw_o, d, R, D.d, D.d, epi_resid(X, d), s);
  {
    Prof p(c, CLIMBER_K_RMSNORM, s, 0, (double)R * d * (4 + es));
    launch_rmsnorm<T>(X, d, c->fg2, H, d, R, D.d, D.eps, s);
  }
  gemm<T>(c, CLIMBER_K_GEMM_FFN_UP, H, d, (const T*)c->fw1, d, R, D.F, D.d, epi_store(Fh, F, ACT_SILU), s);
  gemm<T>(c, CLIMBER_K_GEMM_FFN_DOWN, Fh, F, (const T*)c->fw2, F, R, D.d, D.F, epi_resid(X, d), s);
  // ---- squeeze-and-excitation gate on vec(G) = X viewed as [P][N_b d]
  const T* G = nullptr;
  if constexpr (std::is_same<T, float>::value) {
    G = X;
  } else {
    Prof p(c, CLIMBER_K_OTHER, s, 0, (double)P * D.Dse * (4 + es));
    launch_convert<T>(X, H, P * D.Dse, s);
    G = H;
  }
  T* Z1 = O;  // [P][Hse]
  gemm<T>(c, CLIMBER_K_GEMM_SE, G, D.Dse, (const T*)c->w_se1, D.Dse, P, D.Hse, D.Dse,
          epi_store(Z1, D.Hse, ACT_RELU, c->b_se1), s);
  float* gate = reinterpret_cast<float*>(c->Fh);  // [P][Dse] fp32 (fits: rows_cap * F * esz >= P * Dse * 4)
  Epilogue eg{};
  eg.kind = EPI_STORE_F32; eg.act = ACT_SIGMOID; eg.out = gate; eg.ldo = D.Dse; eg.bias = c->b_se2;
  gemm<T>(c, CLIMBER_K_GEMM_SE, Z1, D.Hse, (const T*)c->w_se2, D.Hse, P, D.Dse, D.Hse, eg, s);
  // ---- Y = G . gate (Eq. 4) fused with the head (G18)
  {
    Prof p(c, CLIMBER_K_HEAD, s, 3.0 * P * D.Dse, (double)P * D.Dse * 8 + P * 4);
    launch_head(X, gate, c->w_head, c->b_head, scores, P, D.Dse, s);
  }
}

// ---------------------------------------------------------------------------
// fused-norm bf16 path (tcgen05 GEMMs): no RMSNorm kernels.  Residual-add GEMMs
// (EPI_RESID_NORM) write the fp32 residual, its bf16 copy and per-row partial
// sums of squares; the GEMM that consumes the normalised rows reads the bf16
// copy with the gain folded into its weights and scales each row by 1/rms.
// ---------------------------------------------------------------------------
static Epilogue epi_resid_norm(float* X, long long ldo, void* Xb, float* part, long long part_rs) {
  Epilogue e{};
  e.kind = EPI_RESID_NORM; e.out = X; e.ldo = ldo; e.out_b16 = Xb; e.part = part; e.part_rs = part_rs;
  return e;
}
static Epilogue with_rs(Epilogue e, const climber_ctx_s* c, const float* part, long long rs_rs) {
  e.rs_part = part; e.rs_rs = rs_rs; e.rs_n = c->pld; e.rs_inv_d = 1.0f / (float)c->D.d; e.rs_eps = c->D.eps;
  return e;
}

static void attn_hist_bf16(climber_ctx_s* c, const bf16* Q, const int* wslot, const int* wr, int U, bf16* O, int k,
                           int l, cudaStream_t s) {
  const Dims& D = c->D;
  if (c->attn_mode == 2 && attn_tc_supported(D.dh, D.nk, true))
    launch_attn_hist_tc(Q, wslot, wr, U, (const bf16*)c->pool, c->n_pages * 2 * PAGE, c->ptab, c->vlen_all, c->tau,
                        O, k, l, D, s);
  else if (c->attn_mode >= 1)
    launch_attn_hist_mma(Q, wslot, wr, U, (const bf16*)c->pool, c->ptab, c->vlen_all, c->tau, O, k, l, D, s);
  else
    launch_attn_hist<bf16>(Q, wslot, wr, U, (const bf16*)c->pool, c->ptab, c->vlen_all, c->tau, O, k, l, D, s);
}

static void attn_sumi_bf16(climber_ctx_s* c, const bf16* QKV, long long P, const int64_t* wcand, const int* wslot,
                           const int* wr, int U, int Mmax, bf16* O, int k, int l, cudaStream_t s) {
  const Dims& D = c->D;
  if (c->attn_mode == 2 && attn_tc_supported(D.dh, D.nk, false))
    launch_attn_sumi_tc(QKV, P, wcand, wslot, wr, U, Mmax, (const bf16*)c->pool, c->n_pages * 2 * PAGE, c->ptab,
                        c->vlen_all, c->tau, O, k, l, D, s);
  else if (c->attn_mode >= 1)
    launch_attn_sumi_mma(QKV, wcand, wslot, wr, U, Mmax, (const bf16*)c->pool, c->ptab, c->vlen_all, c->tau, O, k, l,
                         D, s);
  else
    launch_attn_sumi<bf16>(QKV, wcand, wslot, wr, U, Mmax, (const bf16*)c->pool, c->ptab, c->vlen_all, c->tau, O, k,
                           l, D, s);
}

static void encode_wave_fused(climber_ctx_s* c, const EventsDev& ev, int u0, int U, long long n_events,
                              cudaStream_t s) {
  const Dims& D = c->D;
  const long long rows = (long long)U * D.nk;
  const long long d = D.d, F = D.F, pld = c->pld;
  const int* wslot = c->d_slots + u0;
  const int* wr = c->d_r + u0;
  {
    Prof p(c, CLIMBER_K_EXTRACT, s, 0, (double)n_events * 14 + (double)U * D.Nb * D.nk * 4);
    launch_extract(ev, c->d_ev_off + u0, wslot, U, c->amask, c->smask, c->idx_all, c->vlen_all, c->bad_all, c->err,
                   D, s);
  }
  if (c->cfg.rel_bias) {
    Prof p(c, CLIMBER_K_OTHER, s, 0, (double)U * D.L * D.Nb * D.h * D.nk * 12);
    launch_cand_bias(wslot, c->d_r + u0, U, c->vlen_all, D, s);
  }
  bf16* Xb = (bf16*)c->Xb;
  bf16* Qb = (bf16*)c->QKV;
  bf16* O = (bf16*)c->O;
  bf16* Fh = (bf16*)c->Fh;
  float* X = c->X;
  const double causal_pairs = D.causal ? (double)D.nk * (D.nk + 1) / 2 : (double)D.nk * D.nk;
  for (int k = 0; k < D.Nb; ++k) {
    {
      Prof p(c, CLIMBER_K_EMBED, s, 0, (double)rows * d * (3 * 2 + 4 + 2));
      launch_embed_hist<bf16>(ev, c->d_ev_off + u0, wslot, U, c->idx_all, c->vlen_all, c->bad_all,
                              (const bf16*)c->e_item, (const bf16*)c->e_act, (const bf16*)c->e_scn, X, Xb, c->part,
                              c->pld, k, D, s);
    }
    for (int l = 0; l < D.L; ++l) {
      const size_t kl = (size_t)k * D.L + l;
      Epilogue e{};
      e.kind = EPI_QKV_PAGES; e.out = Qb; e.ldo = d; e.pool = c->pool; e.ptab = c->ptab; e.wave_slot = wslot;
      e.pool_rows = c->n_pages * 2 * PAGE;
      e.blk = k; e.layer = l; e.d = D.d; e.h = D.h; e.dh = D.dh; e.nk = D.nk; e.Nb = D.Nb; e.L = D.L; e.ppb = D.ppb;
      e = with_rs(e, c, c->part, pld);
      const bf16* Wqkv = (const bf16*)c->w_qkv + kl * 3 * d * d;
      if (l < D.L - 1) {
        e.col_off = 0;
        gemm<bf16>(c, CLIMBER_K_GEMM_QKV, Xb, d, Wqkv, d, rows, 3 * D.d, D.d, e, s);
        {
          Prof p(c, CLIMBER_K_ATTN_HIST, s, 4.0 * U * causal_pairs * d, (double)rows * d * 2 * 4);
          attn_hist_bf16(c, Qb, wslot, wr, U, O, k, l, s);
        }
        gemm<bf16>(c, CLIMBER_K_GEMM_O, O, d, (const bf16*)c->w_o + kl * d * d, d, rows, D.d, D.d,
                   epi_resid_norm(X, d, Xb, c->part, pld), s);
        gemm<bf16>(c, CLIMBER_K_GEMM_FFN_UP, Xb, d, (const bf16*)c->w1 + kl * F * d, d, rows, D.F, D.d,
                   with_rs(epi_store(Fh, F, ACT_SILU), c, c->part, pld), s);
        gemm<bf16>(c, CLIMBER_K_GEMM_FFN_DOWN, Fh, F, (const bf16*)c->w2 + kl * d * F, F, rows, D.d, D.F,
                   epi_resid_norm(X, d, Xb, c->part, pld), s);
      } else {
        e.col_off = D.d;  // last layer: only K/V of the history are ever read
        gemm<bf16>(c, CLIMBER_K_GEMM_QKV, Xb, d, Wqkv + d * d, d, rows, 2 * D.d, D.d, e, s);
      }
    }
  }
}

static void score_wave_fused(climber_ctx_s* c, const int32_t* items, const int64_t* wcand, int u0, int U, long long P,
                             int Mmax_wave, float* scores, cudaStream_t s) {
  const Dims& D = c->D;
  const long long d = D.d, F = D.F, Nb = D.Nb, ldC = Nb * d, pld = c->pld;
  const int* wslot = c->d_slots + u0;
  const int* wr = c->d_r + u0;
  bf16* Cb = (bf16*)c->Xb;  // [p][k][d] bf16 copy of the residual
  bf16* QKV = (bf16*)c->QKV;
  bf16* O = (bf16*)c->O;
  bf16* Fh = (bf16*)c->Fh;
  float* C = c->X;  // [p][k][d]
  {
    Prof p(c, CLIMBER_K_EMBED, s, 0, (double)P * d * (2 * 2 + 6 * Nb));
    launch_embed_cand<bf16>(items, wcand, wr, U, P, (const bf16*)c->e_item, (const bf16*)c->e_scn, C, Cb, c->part,
                            c->pld, c->err, D, s);
  }
  for (int k = 0; k < D.Nb; ++k) {
    float* Ck = C + k * d;
    bf16* Cbk = Cb + k * d;
    float* pk = c->part + k * pld;
    const long long prs = Nb * pld;
    for (int l = 0; l < D.L; ++l) {
      const size_t kl = (size_t)k * D.L + l;
      gemm<bf16>(c, CLIMBER_K_GEMM_QKV, Cbk, ldC, (const bf16*)c->w_qkv + kl * 3 * d * d, d, P, 3 * D.d, D.d,
                 with_rs(epi_store(QKV, 3 * d), c, pk, prs), s);
      {
        Prof p(c, CLIMBER_K_ATTN_SUMI, s, 4.0 * P * (D.nk + 1) * d, (double)P * d * 2 * 4 + (double)U * D.nk * d * 4);
        attn_sumi_bf16(c, QKV, P, wcand, wslot, wr, U, Mmax_wave, O, k, l, s);
      }
      gemm<bf16>(c, CLIMBER_K_GEMM_O, O, d, (const bf16*)c->w_o + kl * d * d, d, P, D.d, D.d,
                 epi_resid_norm(Ck, ldC, Cbk, pk, prs), s);
      gemm<bf16>(c, CLIMBER_K_GEMM_FFN_UP, Cbk, ldC, (const bf16*)c->w1 + kl * F * d, d, P, D.F, D.d,
                 with_rs(epi_store(Fh, F, ACT_SILU), c, pk, prs), s);
      gemm<bf16>(c, CLIMBER_K_GEMM_FFN_DOWN, Fh, F, (const bf16*)c->w2 + kl * d * F, F, P, D.d, D.F,
                 epi_resid_norm(Ck, ldC, Cbk, pk, prs), s);
    }
  }
  // ---- BGF (Eq. 4): the N_b block outputs of a pair are contiguous rows of C
  const long long R = P * Nb;
  gemm<bf16>(c, CLIMBER_K_GEMM_QKV, Cb, d, (const bf16*)c->fw_qkv, d, R, 3 * D.d, D.d,
             with_rs(epi_store(QKV, 3 * d), c, c->part, pld), s);
  {
    Prof p(c, CLIMBER_K_ATTN_FUSION, s, 4.0 * P * Nb * Nb * d, (double)R * d * 2 * 4);
    launch_attn_fusion<bf16>(QKV, wcand, wr, U, P, c->tau_f, O, D, s);
  }
  gemm<bf16>(c, CLIMBER_K_GEMM_O, O, d, (const bf16*)c->fw_o, d, R, D.d, D.d,
             epi_resid_norm(C, d, Cb, c->part, pld), s);
  gemm<bf16>(c, CLIMBER_K_GEMM_FFN_UP, Cb, d, (const bf16*)c->fw1, d, R, D.F, D.d,
             with_rs(epi_store(Fh, F, ACT_SILU), c, c->part, pld), s);
  gemm<bf16>(c, CLIMBER_K_GEMM_FFN_DOWN, Fh, F, (const bf16*)c->fw2, F, R, D.d, D.F,
             epi_resid_norm(C, d, Cb, c->part, pld), s);
  // ---- squeeze-and-excitation on vec(G): the bf16 copy Cb viewed as [P][N_b d]
  bf16* Z1 = O;  // [P][Hse]
  gemm<bf16>(c, CLIMBER_K_GEMM_SE, Cb, D.Dse, (const bf16*)c->w_se1, D.Dse, P, D.Hse, D.Dse,
             epi_store(Z1, D.Hse, ACT_RELU, c->b_se1), s);
  float* gate = reinterpret_cast<float*>(c->Fh);
  Epilogue eg{};
  eg.kind = EPI_STORE_F32; eg.act = ACT_SIGMOID; eg.out = gate; eg.ldo = D.Dse; eg.bias = c->b_se2;
  gemm<bf16>(c, CLIMBER_K_GEMM_SE, Z1, D.Hse, (const bf16*)c->w_se2, D.Hse, P, D.Dse, D.Hse, eg, s);
  {
    Prof p(c, CLIMBER_K_HEAD, s, 3.0 * P * D.Dse, (double)P * D.Dse * 8 + P * 4);
    launch_head(C, gate, c->w_head, c->b_head, scores, P, D.Dse, s);
  }
}

// ---------------------------------------------------------------------------
// grouped fused path: each GEMM / attention launch covers all N_b blocks of a
// layer (3-D TMA maps, block = batch index), so small waves and single
// requests fill the GPU with 8x fewer launches (SURVEY K5 "grouped over k").
// ---------------------------------------------------------------------------
static void gemm_g(climber_ctx_s* c, int cls, const bf16* A, long long lda, long long a_bs, const bf16* B,
                   long long ldb, long long b_bs, long long M, int N, int K, int batch, const Epilogue& e,
                   cudaStream_t s) {
  Prof p(c, cls, s, 2.0 * M * N * K * batch);
  launch_gemm_tc_batched(A, lda, a_bs, B, ldb, b_bs, M, N, K, batch, e, s);
}

static void gemm_stage(climber_ctx_s* c, int /*stage*/, int cls, const bf16* A, long long lda, long long a_bs,
                       const bf16* B, long long ldb, long long b_bs, long long M, int N, int K, int batch,
                       const Epilogue& e, cudaStream_t s) {
  gemm_g(c, cls, A, lda, a_bs, B, ldb, b_bs, M, N, K, batch, e, s);
}

static bool grouped_ok(const climber_ctx_s* c) {
  return c->fused && c->attn_mode == 2 && attn_tc_supported(c->D.dh, c->D.nk, false);
}

// blocks [k0, k0 + nbk) only (block-parallel serving, NEXT-2); the layouts
// keep absolute block indices, so a partial encode writes the same bytes as
// the corresponding part of a full one
static void encode_wave_grouped(climber_ctx_s* c, const EventsDev& ev, int u0, int U, long long n_events,
                                cudaStream_t s, int k0 = 0, int nbk = -1) {
  if (nbk < 0) nbk = c->D.Nb;
  const Dims& D = c->D;
  const long long rows = (long long)U * D.nk;  // per block
  const long long d = D.d, F = D.F, pld = c->pld, Lk = D.L;
  const int* wslot = c->d_slots + u0;
  const int* wr = c->d_r + u0;
  {
    Prof p(c, CLIMBER_K_EXTRACT, s, 0, (double)n_events * 14 + (double)U * D.Nb * D.nk * 4);
    launch_extract(ev, c->d_ev_off + u0, wslot, U, c->amask, c->smask, c->idx_all, c->vlen_all, c->bad_all, c->err,
                   D, s);
  }
  if (c->cfg.rel_bias) {
    Prof p(c, CLIMBER_K_OTHER, s, 0, (double)U * D.L * D.Nb * D.h * D.nk * 12);
    launch_cand_bias(wslot, c->d_r + u0, U, c->vlen_all, D, s);
  }
  if (c->bc_record) cudaEventRecord(c->bc_evt[0], s);  // v_k (and the bias state) final
  if (nbk == 0) return;  // extraction (and the candidate bias rows) only: incremental append
  bf16* Xb = (bf16*)c->Xb;   // [Nb][rows][d]
  bf16* Qb = (bf16*)c->QKV;  // [Nb][rows][d]
  bf16* O = (bf16*)c->O;     // [Nb][rows][d]
  bf16* Fh = (bf16*)c->Fh;   // [Nb][rows][F]
  float* X = c->X;           // [Nb][rows][d]
  // the grouped launches below see blocks k0 .. k0 + nbk - 1 as batch 0 .. nbk - 1
  bf16 *gXb = Xb + k0 * rows * d, *gQb = Qb + k0 * rows * d, *gO = O + k0 * rows * d, *gFh = Fh + k0 * rows * F;
  float* gX = X + k0 * rows * d;
  float* gpart = c->part + k0 * rows * pld;
  const size_t wk = (size_t)k0 * Lk;  // first weight slice of block k0
  const double causal_pairs = D.causal ? (double)D.nk * (D.nk + 1) / 2 : (double)D.nk * D.nk;
  for (int k = k0; k < k0 + nbk; ++k) {
    Prof p(c, CLIMBER_K_EMBED, s, 0, (double)rows * d * (3 * 2 + 4 + 2));
    launch_embed_hist<bf16>(ev, c->d_ev_off + u0, wslot, U, c->idx_all, c->vlen_all, c->bad_all,
                            (const bf16*)c->e_item, (const bf16*)c->e_act, (const bf16*)c->e_scn, X + k * rows * d,
                            Xb + k * rows * d, c->part + k * rows * pld, c->pld, k, D, s);
  }
  for (int l = 0; l < D.L; ++l) {
    Epilogue e{};
    e.kind = EPI_QKV_PAGES; e.out = gQb; e.ldo = d; e.out_bs = rows * d; e.pool = c->pool; e.ptab = c->ptab;
    e.wave_slot = wslot; e.pool_rows = c->n_pages * 2 * PAGE; e.blk_from_batch = 1;
    e.blk = k0; e.layer = l; e.d = D.d; e.h = D.h; e.dh = D.dh; e.nk = D.nk; e.Nb = D.Nb; e.L = D.L; e.ppb = D.ppb;
    e = with_rs(e, c, gpart, pld);
    e.rs_bs = rows * pld;
    const bf16* Wqkv = (const bf16*)c->w_qkv + (wk + l) * 3 * d * d;  // block k at + k * L * 3d * d
    if (l < D.L - 1) {
      e.col_off = 0;
      gemm_g(c, CLIMBER_K_GEMM_QKV, gXb, d, rows * d, Wqkv, d, Lk * 3 * d * d, rows, 3 * D.d, D.d, nbk, e, s);
      if (c->ov_record) cudaEventRecord(c->ov_evt[l], s);  // layer l's K/V pages written
      if (c->bc_record) cudaEventRecord(c->bc_evt[1 + l], s);
      {
        Prof p(c, CLIMBER_K_ATTN_HIST, s, 4.0 * U * causal_pairs * d * nbk, (double)rows * d * 2 * 4 * nbk);
        launch_attn_hist_tc(gQb, wslot, wr, U, (const bf16*)c->pool, c->n_pages * 2 * PAGE, c->ptab, c->vlen_all,
                            c->tau, gO, k0, l, D, s, nbk);
      }
      Epilogue eo = epi_resid_norm(gX, d, gXb, gpart, pld);
      eo.out_bs = rows * d; eo.out_b16_bs = rows * d; eo.part_bs = rows * pld;
      gemm_g(c, CLIMBER_K_GEMM_O, gO, d, rows * d, (const bf16*)c->w_o + (wk + l) * d * d, d, Lk * d * d, rows,
             D.d, D.d, nbk, eo, s);
      Epilogue eu = with_rs(epi_store(gFh, F, ACT_SILU), c, gpart, pld);
      eu.out_bs = rows * F; eu.rs_bs = rows * pld;
      gemm_g(c, CLIMBER_K_GEMM_FFN_UP, gXb, d, rows * d, (const bf16*)c->w1 + (wk + l) * F * d, d, Lk * F * d, rows,
             D.F, D.d, nbk, eu, s);
      gemm_g(c, CLIMBER_K_GEMM_FFN_DOWN, gFh, F, rows * F, (const bf16*)c->w2 + (wk + l) * d * F, F, Lk * d * F,
             rows, D.d, D.F, nbk, eo, s);
    } else {
      e.col_off = D.d;  // last layer: only K/V of the history are ever read
      gemm_g(c, CLIMBER_K_GEMM_QKV, gXb, d, rows * d, Wqkv + d * d, d, Lk * 3 * d * d, rows, 2 * D.d, D.d, nbk, e,
             s);
      if (c->ov_record) cudaEventRecord(c->ov_evt[l], s);
      if (c->bc_record) cudaEventRecord(c->bc_evt[1 + l], s);
    }
  }
}

// blocks [k0, k0 + nbk) of the candidate stacks (all of them for a full
// score; a slice for block-parallel serving, NEXT-2): candidate rows
// C [p][N_b][d] hold every block's residual, the launches see the slice
static void score_blocks_grouped(climber_ctx_s* c, const int32_t* items, const int64_t* wcand, int u0, int U,
                                 long long P, int Mmax_wave, cudaStream_t s, int k0, int nbk) {
  const Dims& D = c->D;
  const long long d = D.d, F = D.F, Nb = D.Nb, ldC = Nb * d, pld = c->pld, Lk = D.L;
  const int* wslot = c->d_slots + u0;
  const int* wr = c->d_r + u0;
  bf16* Cb = (bf16*)c->Xb;   // [p][k][d] (interleaved blocks)
  bf16* QKV = (bf16*)c->QKV; // [k - k0][p][3d]
  bf16* O = (bf16*)c->O;     // [k - k0][p][d]
  bf16* Fh = (bf16*)c->Fh;   // [k - k0][p][F]
  float* C = c->X;           // [p][k][d]
  {
    Prof p(c, CLIMBER_K_EMBED, s, 0, (double)P * d * (2 * 2 + 6 * Nb));
    launch_embed_cand<bf16>(items, wcand, wr, U, P, (const bf16*)c->e_item, (const bf16*)c->e_scn, C, Cb, c->part,
                            c->pld, c->err, D, s);
  }
  bf16* gCb = Cb + k0 * d;
  float* gC = C + k0 * d;
  float* gpart = c->part + k0 * pld;
  const size_t wk = (size_t)k0 * Lk;
  // candidate rows of block k: row p at (p * Nb + k) -> batch stride d (elements), partials stride pld
  for (int l = 0; l < D.L; ++l) {
    Epilogue eq = with_rs(epi_store(QKV, 3 * d), c, gpart, Nb * pld);
    eq.out_bs = P * 3 * d; eq.rs_bs = pld;
    gemm_stage(c, 1, CLIMBER_K_GEMM_QKV, gCb, ldC, d, (const bf16*)c->w_qkv + (wk + l) * 3 * d * d, d, Lk * 3 * d * d,
               P, 3 * D.d, D.d, nbk, eq, s);
    if (c->ov_wait) cudaStreamWaitEvent(s, c->ov_evt[l], 0);  // the user's layer-l K/V
    {
      Prof p(c, CLIMBER_K_ATTN_SUMI, s, 4.0 * P * (D.nk + 1) * d * nbk,
             ((double)P * d * 2 * 4 + (double)U * D.nk * d * 4) * nbk);
      launch_attn_sumi_tc(QKV, P, wcand, wslot, wr, U, Mmax_wave, (const bf16*)c->pool, c->n_pages * 2 * PAGE,
                          c->ptab, c->vlen_all, c->tau, O, k0, l, D, s, nbk);
    }
    Epilogue eo = epi_resid_norm(gC, ldC, gCb, gpart, Nb * pld);
    eo.out_bs = d; eo.out_b16_bs = d; eo.part_bs = pld;
    gemm_stage(c, 4, CLIMBER_K_GEMM_O, O, d, P * d, (const bf16*)c->w_o + (wk + l) * d * d, d, Lk * d * d, P, D.d,
               D.d, nbk, eo, s);
    Epilogue eu = with_rs(epi_store(Fh, F, ACT_SILU), c, gpart, Nb * pld);
    eu.out_bs = P * F; eu.rs_bs = pld;
    gemm_stage(c, 8, CLIMBER_K_GEMM_FFN_UP, gCb, ldC, d, (const bf16*)c->w1 + (wk + l) * F * d, d, Lk * F * d, P,
               D.F, D.d, nbk, eu, s);
    gemm_stage(c, 16, CLIMBER_K_GEMM_FFN_DOWN, Fh, F, P * F, (const bf16*)c->w2 + (wk + l) * d * F, F, Lk * d * F, P,
               D.d, D.F, nbk, eo, s);
  }
}

// a5/a6 on the candidate rows C [p][N_b][d] (fp32 residual, bf16 copy and
// per-128-column partial sums of squares already in place)
static void fuse_grouped(climber_ctx_s* c, const int64_t* wcand, int u0, int U, long long P, float* scores,
                         cudaStream_t s) {
  const Dims& D = c->D;
  const long long d = D.d, F = D.F, Nb = D.Nb, pld = c->pld;
  const int* wr = c->d_r + u0;
  bf16* Cb = (bf16*)c->Xb;
  bf16* QKV = (bf16*)c->QKV;
  bf16* O = (bf16*)c->O;
  bf16* Fh = (bf16*)c->Fh;
  float* C = c->X;
  // ---- BGF (Eq. 4) + SE gate + head: identical to the per-block fused path
  const long long R = P * Nb;
  gemm<bf16>(c, CLIMBER_K_GEMM_QKV, Cb, d, (const bf16*)c->fw_qkv, d, R, 3 * D.d, D.d,
             with_rs(epi_store(QKV, 3 * d), c, c->part, pld), s);
  {
    Prof p(c, CLIMBER_K_ATTN_FUSION, s, 4.0 * P * Nb * Nb * d, (double)R * d * 2 * 4);
    launch_attn_fusion<bf16>(QKV, wcand, wr, U, P, c->tau_f, O, D, s);
  }
  gemm<bf16>(c, CLIMBER_K_GEMM_O, O, d, (const bf16*)c->fw_o, d, R, D.d, D.d, epi_resid_norm(C, d, Cb, c->part, pld),
             s);
  gemm<bf16>(c, CLIMBER_K_GEMM_FFN_UP, Cb, d, (const bf16*)c->fw1, d, R, D.F, D.d,
             with_rs(epi_store(Fh, F, ACT_SILU), c, c->part, pld), s);
  gemm<bf16>(c, CLIMBER_K_GEMM_FFN_DOWN, Fh, F, (const bf16*)c->fw2, F, R, D.d, D.F,
             epi_resid_norm(C, d, Cb, c->part, pld), s);
  bf16* Z1 = O;
  gemm<bf16>(c, CLIMBER_K_GEMM_SE, Cb, D.Dse, (const bf16*)c->w_se1, D.Dse, P, D.Hse, D.Dse,
             epi_store(Z1, D.Hse, ACT_RELU, c->b_se1), s);
  float* gate = reinterpret_cast<float*>(c->Fh);
  Epilogue eg{};
  eg.kind = EPI_STORE_F32; eg.act = ACT_SIGMOID; eg.out = gate; eg.ldo = D.Dse; eg.bias = c->b_se2;
  gemm<bf16>(c, CLIMBER_K_GEMM_SE, Z1, D.Hse, (const bf16*)c->w_se2, D.Hse, P, D.Dse, D.Hse, eg, s);
  {
    Prof p(c, CLIMBER_K_HEAD, s, 3.0 * P * D.Dse, (double)P * D.Dse * 8 + P * 4);
    launch_head(C, gate, c->w_head, c->b_head, scores, P, D.Dse, s);
  }
}

static void score_wave_grouped(climber_ctx_s* c, const int32_t* items, const int64_t* wcand, int u0, int U,
                               long long P, int Mmax_wave, float* scores, cudaStream_t s) {
  score_blocks_grouped(c, items, wcand, u0, U, P, Mmax_wave, s, 0, c->D.Nb);
  fuse_grouped(c, wcand, u0, U, P, scores, s);
}

// ---------------------------------------------------------------------------
// staging of per-call metadata (one H2D copy per call, pinned buffer reused
// only after the previous call's copy completed)
// ---------------------------------------------------------------------------
struct Stage {
  int64_t* ev_off;
  int64_t* cand_off;
  int* slots;
  int* r;
  int* ptab;
};

static Stage stage_layout(climber_ctx_s* c, char* base) {
  size_t Bm = c->cfg.max_batch_users;
  Stage st;
  st.ev_off = reinterpret_cast<int64_t*>(base);
  st.cand_off = st.ev_off + (Bm + 1);
  st.slots = reinterpret_cast<int*>(st.cand_off + (2 * Bm + 1));
  st.r = st.slots + Bm;
  st.ptab = st.r + Bm;
  return st;
}

static climber_status stage_upload(climber_ctx_s* c, int B, bool with_ptab, cudaStream_t s) {
  size_t Bm = c->cfg.max_batch_users;
  Stage h = stage_layout(c, c->h_stage);
  CU(cudaMemcpyAsync(c->d_ev_off, h.ev_off, (B + 1) * 8, cudaMemcpyHostToDevice, s));
  CU(cudaMemcpyAsync(c->d_cand_off, h.cand_off, (2 * Bm + 1) * 8, cudaMemcpyHostToDevice, s));
  CU(cudaMemcpyAsync(c->d_slots, h.slots, B * 4, cudaMemcpyHostToDevice, s));
  CU(cudaMemcpyAsync(c->d_r, h.r, B * 4, cudaMemcpyHostToDevice, s));
  if (with_ptab) {
    CU(cudaMemcpyAsync(c->d_ptab_stage, h.ptab, (size_t)B * c->per_slot * 4, cudaMemcpyHostToDevice, s));
    Prof p(c, CLIMBER_K_OTHER, s, 0, (double)B * c->per_slot * 8);
    launch_scatter_ptab(c->d_ptab_stage, c->d_slots, B, c->per_slot, c->ptab, s);
  }
  CU(cudaEventRecord(c->stage_evt, s));
  return CLIMBER_OK;
}

static climber_status check_launch(climber_ctx_s* c, cudaStream_t s) {
  char msg[256];
  if (take_launch_error(msg, sizeof msg)) return fail(CLIMBER_E_CUDA, "launch setup: %s", msg);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(CLIMBER_E_CUDA, "kernel launch: %s", cudaGetErrorString(e));
  if (c->sync_check) {
    e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return fail(CLIMBER_E_CUDA, "sync check: %s", cudaGetErrorString(e));
  }
  return CLIMBER_OK;
}

// ---------------------------------------------------------------------------
// encode
// ---------------------------------------------------------------------------
static climber_status encode_users_range(climber_ctx_t c, int32_t B, const int64_t* ev_offsets,
                                         const climber_events* events, const int32_t* scenario_r,
                                         climber_stream_t stream, climber_kv_t* out, int k0, int k1) {
  try {
    if (!c || !ev_offsets || !events || !scenario_r || !out) return fail(CLIMBER_E_INVALID_ARG, "null argument");
    if (B < 1 || B > c->cfg.max_batch_users) return fail(CLIMBER_E_INVALID_ARG, "B=%d outside [1, max_batch_users]", B);
    for (int b = 0; b < B; ++b) {
      if (ev_offsets[b + 1] < ev_offsets[b]) return fail(CLIMBER_E_INVALID_ARG, "ev_offsets decreasing at %d", b);
      if (scenario_r[b] < 0 || scenario_r[b] >= c->D.R) return fail(CLIMBER_E_OUT_OF_RANGE, "scenario_r[%d] out of range", b);
    }
    if (ev_offsets[B] > ev_offsets[0] &&
        (!events->item || !events->action || !events->scenario || !events->ts))
      return fail(CLIMBER_E_INVALID_ARG, "null event array");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    std::vector<int> slots(B);
    {
      std::lock_guard<std::mutex> g(c->mu);
      if ((int)c->free_slots.size() < B || (long long)c->free_pages.size() < (long long)B * c->per_slot)
        return fail(CLIMBER_E_CAPACITY, "K/V page pool exhausted (%zu free slots)", c->free_slots.size());
      CU(cudaEventSynchronize(c->stage_evt));
      Stage h = stage_layout(c, c->h_stage);
      for (int b = 0; b < B; ++b) {
        int slot = c->free_slots.back();
        c->free_slots.pop_back();
        SlotState& st = c->slots[slot];
        st.live = true;
        st.r = scenario_r[b];
        st.kb0 = k0;
        st.kb1 = k1;
        st.pages.resize(c->per_slot);
        for (int i = 0; i < c->per_slot; ++i) {
          st.pages[i] = c->free_pages.back();
          c->free_pages.pop_back();
          h.ptab[(size_t)b * c->per_slot + i] = st.pages[i];
        }
        slots[b] = slot;
        h.slots[b] = slot;
        h.r[b] = scenario_r[b];
        h.ev_off[b] = ev_offsets[b];
        out[b] = make_handle(c, slot, st.gen);
      }
      h.ev_off[B] = ev_offsets[B];
      climber_status rs = stage_upload(c, B, true, s);
      if (rs != CLIMBER_OK) return rs;
    }
    EventsDev ev{events->item, events->action, events->scenario, events->ts};
    for (int u0 = 0; u0 < B; u0 += c->cfg.max_wave_users) {
      int U = B - u0 < c->cfg.max_wave_users ? B - u0 : c->cfg.max_wave_users;
      long long nev = ev_offsets[u0 + U] - ev_offsets[u0];
      if (c->fused && grouped_ok(c) && attn_tc_supported(c->D.dh, c->D.nk, true))
        encode_wave_grouped(c, ev, u0, U, nev, s, k0, k1 - k0);
      else if (c->fused) encode_wave_fused(c, ev, u0, U, nev, s);
      else if (c->cfg.dtype == CLIMBER_BF16) encode_wave<bf16>(c, ev, u0, U, nev, s);
      else encode_wave<float>(c, ev, u0, U, nev, s);
      climber_status rs = check_launch(c, s);
      if (rs != CLIMBER_OK) return rs;
    }
    return CLIMBER_OK;
  } catch (...) {
    return fail(CLIMBER_E_CUDA, "encode: exception");
  }
}

extern "C" climber_status climber_encode_users(climber_ctx_t c, int32_t B, const int64_t* ev_offsets,
                                               const climber_events* events, const int32_t* scenario_r,
                                               climber_stream_t stream, climber_kv_t* out) {
  return encode_users_range(c, B, ev_offsets, events, scenario_r, stream, out, 0, c ? c->D.Nb : 0);
}

static bool block_parallel_ok(const climber_ctx_s* c) {
  return c->fused && grouped_ok(c) && attn_tc_supported(c->D.dh, c->D.nk, true);
}

extern "C" climber_status climber_encode_users_blocks(climber_ctx_t c, int32_t B, const int64_t* ev_offsets,
                                                      const climber_events* events, const int32_t* scenario_r,
                                                      int32_t k0, int32_t k1, climber_stream_t stream,
                                                      climber_kv_t* out) {
  if (!c) return fail(CLIMBER_E_INVALID_ARG, "null ctx");
  if (k0 < 0 || k1 > c->D.Nb || k0 >= k1) return fail(CLIMBER_E_INVALID_ARG, "block range [%d, %d) invalid", k0, k1);
  if (!block_parallel_ok(c)) return fail(CLIMBER_E_UNSUPPORTED, "block ranges need the bf16 grouped tcgen05 path");
  return encode_users_range(c, B, ev_offsets, events, scenario_r, stream, out, k0, k1);
}

extern "C" climber_status climber_encode_user(climber_ctx_t c, const climber_events* events, int64_t n_s,
                                              int32_t scenario_r, climber_stream_t stream, climber_kv_t* out) {
  if (n_s < 0) return fail(CLIMBER_E_INVALID_ARG, "n_s < 0");
  int64_t off[2] = {0, n_s};
  return climber_encode_users(c, 1, off, events, &scenario_r, stream, out);
}

// ---------------------------------------------------------------------------
// score
// ---------------------------------------------------------------------------
// mode 0: full score (blocks + BGF + head) -> scores; mode 1: blocks [k0, k1)
// only -> E [P][k1 - k0][d]; mode 2: BGF + head from E ([n_slices][P][N_b /
// n_slices][d]) with the per-user scenarios given (no handles) -> scores
static climber_status score_common(climber_ctx_t c, int32_t B, const climber_kv_t* kvs, const int64_t* cand_offsets,
                                   const int32_t* items, const int32_t* scen, int mode, int k0, int k1,
                                   int n_slices, float* E, float* scores, climber_stream_t stream) {
  try {
    if (!c || !cand_offsets || (mode != 2 && (!kvs || !items)) || (mode == 2 && (!scen || !E)) ||
        (mode != 1 && !scores) || (mode == 1 && !E))
      return fail(CLIMBER_E_INVALID_ARG, "null argument");
    if (B < 1 || B > c->cfg.max_batch_users) return fail(CLIMBER_E_INVALID_ARG, "B=%d outside [1, max_batch_users]", B);
    for (int b = 0; b < B; ++b) {
      long long m = cand_offsets[b + 1] - cand_offsets[b];
      if (m < 1 || m > c->cfg.max_candidates)
        return fail(CLIMBER_E_INVALID_ARG, "user %d has M=%lld outside [1, max_candidates]", b, m);
    }
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    // waves: consecutive users while pairs <= max_wave_pairs and users <= max_wave_users
    struct Wave { int u0, U, Mmax; long long P; int coff; };
    std::vector<Wave> waves;
    {
      std::lock_guard<std::mutex> g(c->mu);
      std::vector<int> slots(B, 0);
      if (mode != 2) {
        for (int b = 0; b < B; ++b) {
          climber_status rs = resolve(c, kvs[b], &slots[b]);
          if (rs != CLIMBER_OK) return rs;
          const SlotState& ss = c->slots[slots[b]];
          if (k0 < ss.kb0 || k1 > ss.kb1)
            return fail(CLIMBER_E_INVALID_ARG, "handle %d holds blocks [%d, %d), not [%d, %d)", b, ss.kb0, ss.kb1, k0, k1);
        }
      }
      CU(cudaEventSynchronize(c->stage_evt));
      Stage h = stage_layout(c, c->h_stage);
      int coff = 0;
      for (int u0 = 0; u0 < B;) {
        Wave w{u0, 0, 0, 0, coff};
        while (u0 + w.U < B && w.U < c->cfg.max_wave_users) {
          long long m = cand_offsets[u0 + w.U + 1] - cand_offsets[u0 + w.U];
          if (w.P + m > c->cfg.max_wave_pairs) break;
          w.P += m;
          w.Mmax = w.Mmax > m ? w.Mmax : (int)m;
          w.U++;
        }
        for (int i = 0; i <= w.U; ++i) h.cand_off[coff + i] = cand_offsets[u0 + i] - cand_offsets[u0];
        coff += w.U + 1;
        waves.push_back(w);
        u0 += w.U;
      }
      for (int b = 0; b < B; ++b) {
        h.slots[b] = slots[b];
        h.r[b] = mode == 2 ? scen[b] : c->slots[slots[b]].r;
        if (h.r[b] < 0 || h.r[b] >= c->D.R) return fail(CLIMBER_E_OUT_OF_RANGE, "scenario_r[%d] out of range", b);
      }
      h.ev_off[0] = 0;
      climber_status rs = stage_upload(c, B, false, s);
      if (rs != CLIMBER_OK) return rs;
    }
    const long long d = c->D.d, Nb = c->D.Nb;
    for (const Wave& w : waves) {
      const int32_t* it = items ? items + cand_offsets[w.u0] : nullptr;
      float* sc = scores ? scores + cand_offsets[w.u0] : nullptr;
      const int64_t* wc = c->d_cand_off + w.coff;
      const long long q0 = cand_offsets[w.u0] - cand_offsets[0];  // first pair of the wave
      if (mode == 1) {  // block stacks of [k0, k1), then E = C[:, k0:k1, :]
        score_blocks_grouped(c, it, wc, w.u0, w.U, w.P, w.Mmax, s, k0, k1 - k0);
        CU(cudaMemcpy2DAsync(E + q0 * (k1 - k0) * d, (k1 - k0) * d * 4, c->X + k0 * d, Nb * d * 4, (k1 - k0) * d * 4,
                             w.P, cudaMemcpyDeviceToDevice, s));
      } else if (mode == 2) {  // C = E (slices rank-major), recompute the bf16 copy + norm partials, fuse
        const long long ns = Nb / n_slices, Ptot = cand_offsets[B] - cand_offsets[0];
        for (int g = 0; g < n_slices; ++g)
          CU(cudaMemcpy2DAsync(c->X + g * ns * d, Nb * d * 4, E + ((long long)g * Ptot + q0) * ns * d, ns * d * 4,
                               ns * d * 4, w.P, cudaMemcpyDeviceToDevice, s));
        {
          Prof p(c, CLIMBER_K_OTHER, s, 0, (double)w.P * Nb * d * 6);
          launch_row_prep(c->X, (bf16*)c->Xb, c->part, w.P * Nb, c->D.d, c->pld, s);
        }
        fuse_grouped(c, wc, w.u0, w.U, w.P, sc, s);
      } else if (c->fused && grouped_ok(c)) score_wave_grouped(c, it, wc, w.u0, w.U, w.P, w.Mmax, sc, s);
      else if (c->fused) score_wave_fused(c, it, wc, w.u0, w.U, w.P, w.Mmax, sc, s);
      else if (c->cfg.dtype == CLIMBER_BF16) score_wave<bf16>(c, it, wc, w.u0, w.U, w.P, w.Mmax, sc, s);
      else score_wave<float>(c, it, wc, w.u0, w.U, w.P, w.Mmax, sc, s);
      if (c->sync_check && sc) launch_check_finite(sc, w.P, c->err, s);
      climber_status rs = check_launch(c, s);
      if (rs != CLIMBER_OK) return rs;
      if (c->sync_check && sc) {  // synchronous numeric check (the header's E_NUMERIC contract)
        int err = 0;
        CU(cudaMemcpy(&err, c->err, 4, cudaMemcpyDeviceToHost));
        if (err & ERR_NUMERIC) {
          const int keep = err & ~ERR_NUMERIC;
          CU(cudaMemcpy(c->err, &keep, 4, cudaMemcpyHostToDevice));
          return fail(CLIMBER_E_NUMERIC, "non-finite score in users [%d, %d)", w.u0, w.u0 + w.U);
        }
      }
    }
    return CLIMBER_OK;
  } catch (...) {
    return fail(CLIMBER_E_CUDA, "score: exception");
  }
}

extern "C" climber_status climber_score_items_batched(climber_ctx_t c, int32_t B, const climber_kv_t* kvs,
                                                      const int64_t* cand_offsets, const int32_t* items,
                                                      float* scores, climber_stream_t stream) {
  return score_common(c, B, kvs, cand_offsets, items, nullptr, 0, 0, c ? c->D.Nb : 0, 1, nullptr, scores, stream);
}

extern "C" climber_status climber_score_blocks(climber_ctx_t c, int32_t B, const climber_kv_t* kvs,
                                               const int64_t* cand_offsets, const int32_t* items, int32_t k0,
                                               int32_t k1, float* E, climber_stream_t stream) {
  if (!c) return fail(CLIMBER_E_INVALID_ARG, "null ctx");
  if (k0 < 0 || k1 > c->D.Nb || k0 >= k1) return fail(CLIMBER_E_INVALID_ARG, "block range [%d, %d) invalid", k0, k1);
  if (!block_parallel_ok(c)) return fail(CLIMBER_E_UNSUPPORTED, "block ranges need the bf16 grouped tcgen05 path");
  return score_common(c, B, kvs, cand_offsets, items, nullptr, 1, k0, k1, 1, E, nullptr, stream);
}

extern "C" climber_status climber_fuse_scores(climber_ctx_t c, int32_t B, const int64_t* cand_offsets,
                                              const int32_t* scenario_r, int32_t n_slices, const float* E,
                                              float* scores, climber_stream_t stream) {
  if (!c) return fail(CLIMBER_E_INVALID_ARG, "null ctx");
  if (n_slices < 1 || c->D.Nb % n_slices) return fail(CLIMBER_E_INVALID_ARG, "n_slices must divide N_b");
  if (!block_parallel_ok(c)) return fail(CLIMBER_E_UNSUPPORTED, "block ranges need the bf16 grouped tcgen05 path");
  return score_common(c, B, nullptr, cand_offsets, nullptr, scenario_r, 2, 0, c->D.Nb, n_slices,
                      const_cast<float*>(E), scores, stream);
}

extern "C" climber_status climber_score_items(climber_ctx_t c, climber_kv_t kv, const int32_t* items, int32_t M,
                                              float* scores, climber_stream_t stream) {
  int64_t off[2] = {0, M};
  return climber_score_items_batched(c, 1, &kv, off, items, scores, stream);
}

extern "C" climber_status climber_kv_release(climber_ctx_t c, climber_kv_t kv) {
  if (!c) return fail(CLIMBER_E_INVALID_ARG, "null ctx");
  std::lock_guard<std::mutex> g(c->mu);
  int slot;
  climber_status rs = resolve(c, kv, &slot);
  if (rs != CLIMBER_OK) return rs;
  SlotState& st = c->slots[slot];
  for (int p : st.pages) c->free_pages.push_back(p);
  st.pages.clear();
  st.live = false;
  st.gen = (st.gen + 1) & 0xFFFFFF;
  if (st.gen == 0) st.gen = 1;
  c->free_slots.push_back(slot);
  return CLIMBER_OK;
}

static size_t page_bytes(const climber_ctx_s* c);
static size_t bias_state_bytes(const climber_ctx_s* c);
static climber_status copy_bias_state_at(climber_ctx_s* c, int slot, char* sec, bool to_slab, cudaStream_t s);

// replicate one user's K/V to every rank of the ctx's NCCL
// group.  The root exports its handle into one slab (256 B header: config
// fingerprint, v_k per block, scenario r; then the pages and, with rel_bias,
// the handle's bias state), one ncclBroadcast over NVLink/NVSwitch
// replicates it, every other rank imports it into its own page pool and
// receives a new handle in *kv.  Collective: every rank reaches the
// broadcast, also when the root's export fails (it then sends an invalid
// header and every receiver fails with E_STALE); the receivers wait for the
// header with a deadline (CLIMBER_NCCL_TIMEOUT_MS, default 120 s) and abort
// the communicator on timeout or on an asynchronous NCCL error.
static climber_status nccl_abort(climber_ctx_s* c, const char* why) {
  if (c->comm) nccl_api().abort(c->comm);
  c->comm = nullptr;
  return fail(CLIMBER_E_NCCL, "%s; communicator aborted", why);
}

// wait for `stream` with a deadline, watching the communicator's async error
static climber_status nccl_wait(climber_ctx_s* c, cudaStream_t s) {
  static const long long timeout_ms = [] {
    const char* e = getenv("CLIMBER_NCCL_TIMEOUT_MS");
    return e ? atoll(e) : 120000LL;
  }();
  cudaEvent_t ev;
  CU(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  CU(cudaEventRecord(ev, s));
  const auto t0 = std::chrono::steady_clock::now();
  climber_status st = CLIMBER_OK;
  for (;;) {
    cudaError_t q = cudaEventQuery(ev);
    if (q == cudaSuccess) break;
    if (q != cudaErrorNotReady) { st = fail(CLIMBER_E_CUDA, "broadcast wait: %s", cudaGetErrorString(q)); break; }
    ncclResult_t ae = ncclSuccess;
    nccl_api().async_err(c->comm, &ae);
    if (ae != ncclSuccess && ae != ncclInProgress) { st = nccl_abort(c, nccl_api().err(ae)); break; }
    if (std::chrono::duration_cast<std::chrono::milliseconds>(std::chrono::steady_clock::now() - t0).count() >
        timeout_ms) {
      st = nccl_abort(c, "K/V broadcast timed out");
      break;
    }
    std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
  cudaEventDestroy(ev);
  return st;
}

extern "C" climber_status climber_kv_broadcast(climber_ctx_t c, climber_kv_t* kv, int32_t root,
                                               climber_stream_t stream) {
  // checks that depend only on arguments every rank passes alike, so every
  // rank returns before the collective or none does
  if (!c || !kv) return fail(CLIMBER_E_INVALID_ARG, "null argument");
  if (root < 0 || root >= c->world) return fail(CLIMBER_E_INVALID_ARG, "root out of range");
  if (c->world == 1 && !c->comm) return CLIMBER_OK;  // a single rank already holds it
  if (!c->comm) return fail(CLIMBER_E_UNSUPPORTED, "ctx has no NCCL communicator (aborted or never created)");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const size_t bytes = climber_kv_slab_bytes(c);
  if (!c->bslab) CU(cudaMalloc(&c->bslab, bytes + 16));  // + 16: the pipelined layout's padded header
  climber_status root_st = CLIMBER_OK;
  if (c->rank == root) {
    root_st = climber_kv_export(c, *kv, c->bslab, stream);
    // still join the collective: an invalid header tells the receivers
    if (root_st != CLIMBER_OK) CU(cudaMemsetAsync(c->bslab, 0, 256, s));
  }
  ncclResult_t nr = nccl_api().bcast(c->bslab, c->bslab, bytes, ncclUint8, root, c->comm, s);
  if (nr != ncclSuccess) return nccl_abort(c, nccl_api().err(nr));
  // CLIMBER_DEBUG_BCAST_SELF=1: the root also takes the receiver path (tests
  // the whole export -> broadcast -> import chain on one GPU)
  static const bool self_import = getenv("CLIMBER_DEBUG_BCAST_SELF") != nullptr;
  if (c->rank == root && (!self_import || root_st != CLIMBER_OK)) return root_st;
  climber_status ws = nccl_wait(c, s);
  if (ws != CLIMBER_OK) return ws;
  int32_t hdr[8];
  CU(cudaMemcpy(hdr, c->bslab, sizeof hdr, cudaMemcpyDeviceToHost));
  if (hdr[0] != 0x4B56534C) return fail(CLIMBER_E_STALE, "kv_broadcast: the root's export failed (no handle sent)");
  return climber_kv_import(c, c->bslab, hdr[7], stream, kv);
}

// Pipelined replication of one user's K/V while it is encoded (SURVEY §8(e):
// "pipelined per layer, overlapping encode of layer l+1 with the broadcast of
// layer l").  Slab sections: [header 256 B + bias state][layer 0 pages]...
// [layer L-1 pages]; L + 1 ncclBroadcasts on every rank in that order.  The
// root posts its broadcasts on a side stream, each behind the event its
// encode records when that section is final; receivers post theirs on
// `stream` and unpack each section right behind it -- no host sync anywhere.
// A rank whose own preparation fails still posts all L + 1 broadcasts (the
// root with a zeroed header, so the receivers' imports fail on the device
// with E_CONFIG) and returns its error.
extern "C" climber_status climber_encode_user_bcast(climber_ctx_t c, const climber_events* events, int64_t n_s,
                                                    int32_t scenario_r, int32_t root, climber_stream_t stream,
                                                    climber_kv_t* out) {
  if (!c || !out) return fail(CLIMBER_E_INVALID_ARG, "null argument");
  if (root < 0 || root >= c->world) return fail(CLIMBER_E_INVALID_ARG, "root out of range");
  if (scenario_r < 0 || scenario_r >= c->D.R) return fail(CLIMBER_E_OUT_OF_RANGE, "scenario_r out of range");
  if (!c->comm) return fail(CLIMBER_E_UNSUPPORTED, "ctx has no NCCL communicator (aborted or never created)");
  if (!(c->fused && grouped_ok(c) && attn_tc_supported(c->D.dh, c->D.nk, true)))
    return fail(CLIMBER_E_UNSUPPORTED, "encode_user_bcast needs the grouped bf16 tcgen05 path");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const Dims& D = c->D;
  const size_t hdr_bytes = (256 + bias_state_bytes(c) + 15) / 16 * 16;
  const size_t layer_bytes = (size_t)D.Nb * D.ppb * page_bytes(c);
  const size_t bytes = hdr_bytes + (size_t)D.L * layer_bytes;
  if (!c->bslab) CU(cudaMalloc(&c->bslab, climber_kv_slab_bytes(c) + 16));
  char* slab = reinterpret_cast<char*>(c->bslab);
  static_assert(sizeof(int) == 4, "");
  if ((size_t)bytes > climber_kv_slab_bytes(c) + 16) return fail(CLIMBER_E_CUDA, "slab layout");
  if ((int)c->bc_evt.size() < D.L + 2) {
    while ((int)c->bc_evt.size() < D.L + 2) {
      cudaEvent_t ev;
      CU(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      c->bc_evt.push_back(ev);
    }
  }
  static const bool self_import = getenv("CLIMBER_DEBUG_BCAST_SELF") != nullptr;
  climber_status local = CLIMBER_OK;
  ncclResult_t nr = ncclSuccess;
  auto bcast = [&](size_t off, size_t n, cudaStream_t st) {
    if (nr == ncclSuccess) nr = nccl_api().bcast(slab + off, slab + off, n, ncclUint8, root, c->comm, st);
  };
  // receiver side: allocate the handle, then (broadcast +) unpack section by section
  auto receive = [&](bool do_bcast) -> climber_status {
    int slot = -1;
    climber_status mine = CLIMBER_OK;
    {
      std::lock_guard<std::mutex> g(c->mu);
      if (c->free_slots.empty() || (long long)c->free_pages.size() < c->per_slot) {
        mine = fail(CLIMBER_E_CAPACITY, "K/V page pool exhausted");
      } else {
        cudaError_t e = cudaEventSynchronize(c->stage_evt);
        if (e != cudaSuccess) return fail(CLIMBER_E_CUDA, "stage: %s", cudaGetErrorString(e));
        Stage h = stage_layout(c, c->h_stage);
        slot = c->free_slots.back();
        c->free_slots.pop_back();
        SlotState& st = c->slots[slot];
        st.live = true;
        st.r = scenario_r;
        st.kb0 = 0;
        st.kb1 = D.Nb;
        st.pages.resize(c->per_slot);
        for (int i = 0; i < c->per_slot; ++i) {
          st.pages[i] = c->free_pages.back();
          c->free_pages.pop_back();
          h.ptab[i] = st.pages[i];
        }
        h.slots[0] = slot;
        h.r[0] = scenario_r;
        h.ev_off[0] = h.ev_off[1] = 0;
        climber_status rs = stage_upload(c, 1, true, s);
        if (rs != CLIMBER_OK) return rs;
        *out = make_handle(c, slot, st.gen);
      }
    }
    if (do_bcast) bcast(0, hdr_bytes, s);
    if (mine == CLIMBER_OK) {
      launch_kv_import(c->pool, c->ptab, c->vlen_all, slot, 0, (long long)page_bytes(c), slab, c->err, D,
                       c->cfg.dtype, s);
      climber_status st = copy_bias_state_at(c, slot, slab + 256, false, s);
      if (st != CLIMBER_OK) return st;
    }
    for (int l = 0; l < D.L; ++l) {
      if (do_bcast) bcast(hdr_bytes + l * layer_bytes, layer_bytes, s);
      if (mine == CLIMBER_OK)
        launch_kv_layer_copy(c->pool, c->ptab, slot, l, (long long)page_bytes(c),
                             slab + hdr_bytes + l * layer_bytes, true, D, s);
    }
    if (nr != ncclSuccess) return nccl_abort(c, nccl_api().err(nr));
    if (mine != CLIMBER_OK) return mine;
    return check_launch(c, s);
  };
  if (c->rank == root) {
    if (!c->bc_stream) CU(cudaStreamCreateWithFlags(&c->bc_stream, cudaStreamNonBlocking));
    cudaStream_t bs = c->bc_stream;
    int slot = -1;
    if (!events) {
      local = fail(CLIMBER_E_INVALID_ARG, "root needs the events");
    } else {
      const int64_t off[2] = {0, n_s};
      c->bc_record = true;
      local = encode_users_range(c, 1, off, events, &scenario_r, stream, out, 0, D.Nb);
      c->bc_record = false;
      if (local == CLIMBER_OK) {
        std::lock_guard<std::mutex> g(c->mu);
        if (resolve(c, *out, &slot) != CLIMBER_OK) local = fail(CLIMBER_E_STALE, "fresh handle");
      }
    }
    CU(cudaStreamWaitEvent(bs, c->bc_evt[0], 0));  // also orders behind earlier work on the ctx
    if (local == CLIMBER_OK) {
      launch_kv_export(c->pool, c->ptab, c->vlen_all, slot, 0, (long long)page_bytes(c), slab, D, c->cfg.dtype,
                       scenario_r, bs);
      climber_status st = copy_bias_state_at(c, slot, slab + 256, true, bs);
      if (st != CLIMBER_OK) return st;
    } else {
      CU(cudaMemsetAsync(slab, 0, 256, bs));
    }
    bcast(0, hdr_bytes, bs);
    for (int l = 0; l < D.L; ++l) {
      if (local == CLIMBER_OK) {
        CU(cudaStreamWaitEvent(bs, c->bc_evt[1 + l], 0));
        launch_kv_layer_copy(c->pool, c->ptab, slot, l, (long long)page_bytes(c), slab + hdr_bytes + l * layer_bytes,
                             false, D, bs);
      }
      bcast(hdr_bytes + l * layer_bytes, layer_bytes, bs);
    }
    CU(cudaEventRecord(c->bc_evt[D.L + 1], bs));
    CU(cudaStreamWaitEvent(s, c->bc_evt[D.L + 1], 0));  // the slab and the pages are reused in stream order
    if (nr != ncclSuccess) return nccl_abort(c, nccl_api().err(nr));
    if (local != CLIMBER_OK || !self_import) return local;
    // CLIMBER_DEBUG_BCAST_SELF (world-1 tests): the root also takes the receiver
    // path (allocation, header and per-layer unpack) from its own slab into a
    // second handle, which it returns
    const climber_kv_t sent = *out;
    climber_status st = receive(false);
    CU(cudaStreamSynchronize(s));
    climber_kv_release(c, sent);
    return st;
  }
  return receive(true);
}

extern "C" climber_status climber_nccl_unique_id(void* out) {
  if (!out) return fail(CLIMBER_E_INVALID_ARG, "null argument");
  if (!nccl_api().ok) return fail(CLIMBER_E_UNSUPPORTED, "libnccl.so.2 not loadable");
  ncclUniqueId id;
  ncclResult_t nr = nccl_api().get_uid(&id);
  if (nr != ncclSuccess) return fail(CLIMBER_E_NCCL, "ncclGetUniqueId: %s", nccl_api().err(nr));
  memcpy(out, &id, sizeof(id));
  return CLIMBER_OK;
}

static size_t page_bytes(const climber_ctx_s* c) { return (size_t)2 * PAGE * c->D.d * c->esz; }

// relative-bias state of one handle (rel_bias = 1): hage [N_b][n_k] int32 and
// cbias [L][N_b][h][n_k] fp32, both contiguous per slot
static size_t bias_state_bytes(const climber_ctx_s* c) {
  if (!c->cfg.rel_bias) return 0;
  const Dims& D = c->D;
  return (size_t)D.Nb * D.nk * 4 + (size_t)D.L * D.Nb * D.h * D.nk * 4;
}

extern "C" size_t climber_kv_slab_bytes(climber_ctx_t c) {
  return c ? 256 + (size_t)c->per_slot * page_bytes(c) + bias_state_bytes(c) : 0;
}

static climber_status copy_bias_state(climber_ctx_s* c, int slot, char* slab, bool to_slab, cudaStream_t s) {
  return copy_bias_state_at(c, slot, slab + 256 + (size_t)c->per_slot * page_bytes(c), to_slab, s);
}
// the bias state of `slot` to / from `sec` (hage rows, then cbias rows)
static climber_status copy_bias_state_at(climber_ctx_s* c, int slot, char* sec, bool to_slab, cudaStream_t s) {
  if (!c->cfg.rel_bias) return CLIMBER_OK;
  const Dims& D = c->D;
  const size_t hb = (size_t)D.Nb * D.nk * 4, cb = (size_t)D.L * D.Nb * D.h * D.nk * 4;
  char* h = reinterpret_cast<char*>(c->hage) + slot * hb;
  char* cbs = reinterpret_cast<char*>(c->cbias) + slot * cb;
  if (to_slab) {
    CU(cudaMemcpyAsync(sec, h, hb, cudaMemcpyDeviceToDevice, s));
    CU(cudaMemcpyAsync(sec + hb, cbs, cb, cudaMemcpyDeviceToDevice, s));
  } else {
    CU(cudaMemcpyAsync(h, sec, hb, cudaMemcpyDeviceToDevice, s));
    CU(cudaMemcpyAsync(cbs, sec + hb, cb, cudaMemcpyDeviceToDevice, s));
  }
  return CLIMBER_OK;
}

extern "C" climber_status climber_kv_export(climber_ctx_t c, climber_kv_t kv, void* slab, climber_stream_t stream) {
  if (!c || !slab) return fail(CLIMBER_E_INVALID_ARG, "null argument");
  if (reinterpret_cast<uintptr_t>(slab) % 16) return fail(CLIMBER_E_INVALID_ARG, "slab must be 16-byte aligned");
  int slot, r;
  {
    std::lock_guard<std::mutex> g(c->mu);
    climber_status rs = resolve(c, kv, &slot);
    if (rs != CLIMBER_OK) return rs;
    r = c->slots[slot].r;
    if (c->slots[slot].kb0 != 0 || c->slots[slot].kb1 != c->D.Nb)
      return fail(CLIMBER_E_INVALID_ARG, "kv_export: the handle holds blocks [%d, %d) only (block-parallel encode)",
                  c->slots[slot].kb0, c->slots[slot].kb1);
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  {
    Prof p(c, CLIMBER_K_OTHER, s, 0, 2.0 * c->per_slot * page_bytes(c));
    launch_kv_export(c->pool, c->ptab, c->vlen_all, slot, c->per_slot, (long long)page_bytes(c), slab, c->D,
                     c->cfg.dtype, r, s);
  }
  climber_status bs = copy_bias_state(c, slot, (char*)slab, true, s);
  if (bs != CLIMBER_OK) return bs;
  return check_launch(c, s);
}

extern "C" climber_status climber_kv_import(climber_ctx_t c, const void* slab, int32_t scenario_r,
                                            climber_stream_t stream, climber_kv_t* out) {
  if (!c || !slab || !out) return fail(CLIMBER_E_INVALID_ARG, "null argument");
  if (reinterpret_cast<uintptr_t>(slab) % 16) return fail(CLIMBER_E_INVALID_ARG, "slab must be 16-byte aligned");
  if (scenario_r < 0 || scenario_r >= c->D.R) return fail(CLIMBER_E_OUT_OF_RANGE, "scenario_r out of range");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int slot;
  {
    std::lock_guard<std::mutex> g(c->mu);
    if (c->free_slots.empty() || (long long)c->free_pages.size() < c->per_slot)
      return fail(CLIMBER_E_CAPACITY, "K/V page pool exhausted");
    CU(cudaEventSynchronize(c->stage_evt));
    Stage h = stage_layout(c, c->h_stage);
    slot = c->free_slots.back();
    c->free_slots.pop_back();
    SlotState& st = c->slots[slot];
    st.live = true;
    st.r = scenario_r;
    st.kb0 = 0;
    st.kb1 = c->D.Nb;
    st.pages.resize(c->per_slot);
    for (int i = 0; i < c->per_slot; ++i) {
      st.pages[i] = c->free_pages.back();
      c->free_pages.pop_back();
      h.ptab[i] = st.pages[i];
    }
    h.slots[0] = slot;
    h.r[0] = scenario_r;
    h.ev_off[0] = h.ev_off[1] = 0;
    climber_status rs = stage_upload(c, 1, true, s);
    if (rs != CLIMBER_OK) return rs;
    *out = make_handle(c, slot, st.gen);
  }
  {
    Prof p(c, CLIMBER_K_OTHER, s, 0, 2.0 * c->per_slot * page_bytes(c));
    launch_kv_import(c->pool, c->ptab, c->vlen_all, slot, c->per_slot, (long long)page_bytes(c), slab, c->err, c->D,
                     c->cfg.dtype, s);
  }
  climber_status bs = copy_bias_state(c, slot, (char*)const_cast<void*>(slab), false, s);
  if (bs != CLIMBER_OK) return bs;
  return check_launch(c, s);
}

extern "C" climber_status climber_stream_status(climber_ctx_t c, climber_stream_t stream) {
  if (!c) return fail(CLIMBER_E_INVALID_ARG, "null ctx");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  CU(cudaStreamSynchronize(s));
  int err = 0;
  CU(cudaMemcpy(&err, c->err, 4, cudaMemcpyDeviceToHost));
  CU(cudaMemset(c->err, 0, 4));
  if (err & ERR_RANGE) return fail(CLIMBER_E_OUT_OF_RANGE, "an item/action/scenario id was out of range");
  if (err & ERR_UNSORTED) return fail(CLIMBER_E_UNSORTED, "a lifecycle sequence had decreasing timestamps");
  if (err & ERR_CONFIG) return fail(CLIMBER_E_CONFIG, "an imported K/V slab did not match this ctx's config");
  if (err & ERR_NUMERIC) return fail(CLIMBER_E_NUMERIC, "a score was not finite");
  return CLIMBER_OK;
}

// ---------------------------------------------------------------------------
// latency mode: one request (B = 1) as one CUDA graph.  The host bookkeeping
// (slot / page allocation) and ONE metadata upload (event and candidate
// offsets, slot, scenario, page table) run eagerly; every kernel reads the
// request's slot from device memory, so the encode + score launch sequence
// depends only on (E, P) and is captured once per shape, then replayed.
// ---------------------------------------------------------------------------
static climber_status rank_one_graph(climber_ctx_s* c, long long E, long long P, const climber_events& ev,
                                     int32_t r, const int32_t* d_items, float* d_scores, float* h_scores,
                                     cudaStream_t s) {
  if (r < 0 || r >= c->D.R) return fail(CLIMBER_E_OUT_OF_RANGE, "scenario_r out of range");
  if (E < 0) return fail(CLIMBER_E_INVALID_ARG, "ev_offsets decreasing");
  if (P < 1 || P > c->cfg.max_candidates) return fail(CLIMBER_E_INVALID_ARG, "M=%lld outside [1, max_candidates]", P);
  if (P > c->cfg.max_wave_pairs) return fail(CLIMBER_E_INVALID_ARG, "M exceeds max_wave_pairs");
  climber_kv_t kv;
  {
    std::lock_guard<std::mutex> g(c->mu);
    if (c->free_slots.empty() || (long long)c->free_pages.size() < c->per_slot)
      return fail(CLIMBER_E_CAPACITY, "K/V page pool exhausted");
    CU(cudaEventSynchronize(c->stage_evt));
    Stage h = stage_layout(c, c->h_stage);
    const int slot = c->free_slots.back();
    c->free_slots.pop_back();
    SlotState& st = c->slots[slot];
    st.live = true;
    st.r = r;
    st.kb0 = 0;
    st.kb1 = c->D.Nb;
    st.pages.resize(c->per_slot);
    for (int i = 0; i < c->per_slot; ++i) {
      st.pages[i] = c->free_pages.back();
      c->free_pages.pop_back();
      h.ptab[i] = st.pages[i];
    }
    h.slots[0] = slot;
    h.r[0] = r;
    h.ev_off[0] = 0;
    h.ev_off[1] = E;
    h.cand_off[0] = 0;
    h.cand_off[1] = P;
    kv = make_handle(c, slot, st.gen);
    climber_status rs = stage_upload(c, 1, true, s);
    if (rs != CLIMBER_OK) return rs;
  }
  EventsDev evd{ev.item, ev.action, ev.scenario, ev.ts};
  climber_status st = CLIMBER_OK;
  const bool have = c->g_exec && c->g_E == E && c->g_P == P && c->g_io == c->io;
  if (!have && !(c->g_seen_E == E && c->g_seen_P == P)) {
    // first request of this shape: run eagerly (loads every kernel it needs;
    // lazy module loading is not permitted inside a capture); a repeat of
    // the shape is captured
    c->g_seen_E = E;
    c->g_seen_P = P;
    encode_wave_grouped(c, evd, 0, 1, E, s);
    score_wave_grouped(c, d_items, c->d_cand_off, 0, 1, P, (int)P, d_scores, s);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(h_scores, d_scores, P * 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) st = fail(CLIMBER_E_CUDA, "rank_host: %s", cudaGetErrorString(e));
    climber_kv_release(c, kv);
    return st;
  }
  if (!have) {
    if (c->g_exec) cudaGraphExecDestroy(c->g_exec);
    c->g_exec = nullptr;
    cudaGraph_t graph = nullptr;
    const long long l0 = c->launches;
    // capture on a private stream (the caller's may be the legacy default
    // stream, which cannot capture); nothing executes during capture
    cudaError_t e = cudaSuccess;
    if (!c->g_stream) e = cudaStreamCreateWithFlags(&c->g_stream, cudaStreamNonBlocking);
    if (e == cudaSuccess && !c->g_stream2) e = cudaStreamCreateWithFlags(&c->g_stream2, cudaStreamNonBlocking);
    const int L = c->D.L;
    while (e == cudaSuccess && (int)c->ov_evt.size() < L + 2) {
      cudaEvent_t ev;
      e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
      if (e == cudaSuccess) c->ov_evt.push_back(ev);
    }
    // the score runs in its own scratch rows (after the encode's) so the two
    // streams never share a buffer; without room, one stream
    const long long enc_rows = (long long)c->D.nk * c->D.Nb;
    const bool overlap = enc_rows + P * c->D.Nb <= c->rows_cap;
    if (e == cudaSuccess) e = cudaStreamBeginCapture(c->g_stream, cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess && overlap) {
      const long long d = c->D.d;
      float* X0 = c->X;
      void *Xb0 = c->Xb, *QKV0 = c->QKV, *O0 = c->O, *Fh0 = c->Fh;
      float* part0 = c->part;
      cudaEventRecord(c->ov_evt[L], c->g_stream);  // fork
      cudaStreamWaitEvent(c->g_stream2, c->ov_evt[L], 0);
      c->ov_record = true;
      encode_wave_grouped(c, evd, 0, 1, E, c->g_stream);
      c->ov_record = false;
      c->X = X0 + enc_rows * d;
      c->Xb = (bf16*)Xb0 + enc_rows * d;
      c->QKV = (bf16*)QKV0 + enc_rows * 3 * d;
      c->O = (bf16*)O0 + enc_rows * d;
      c->Fh = (bf16*)Fh0 + enc_rows * c->D.F;
      c->part = part0 + enc_rows * c->pld;
      c->ov_wait = true;
      score_wave_grouped(c, d_items, c->d_cand_off, 0, 1, P, (int)P, d_scores, c->g_stream2);
      c->ov_wait = false;
      c->X = X0; c->Xb = Xb0; c->QKV = QKV0; c->O = O0; c->Fh = Fh0; c->part = part0;
      cudaEventRecord(c->ov_evt[L + 1], c->g_stream2);  // join
      cudaStreamWaitEvent(c->g_stream, c->ov_evt[L + 1], 0);
      e = cudaStreamEndCapture(c->g_stream, &graph);
    } else if (e == cudaSuccess) {
      encode_wave_grouped(c, evd, 0, 1, E, c->g_stream);
      score_wave_grouped(c, d_items, c->d_cand_off, 0, 1, P, (int)P, d_scores, c->g_stream);
      e = cudaStreamEndCapture(c->g_stream, &graph);
    }
    if (e == cudaSuccess) e = cudaGraphInstantiate(&c->g_exec, graph, 0);
    if (graph) cudaGraphDestroy(graph);
    if (e != cudaSuccess) {
      c->g_exec = nullptr;
      st = fail(CLIMBER_E_CUDA, "rank_host graph capture: %s", cudaGetErrorString(e));
    } else {
      c->g_E = E;
      c->g_P = P;
      c->g_io = c->io;
      c->g_launches = c->launches - l0;
      c->launches = l0;
    }
  }
  if (st == CLIMBER_OK) {
    cudaError_t e = cudaGraphLaunch(c->g_exec, s);
    c->launches += c->g_launches;
    if (e == cudaSuccess) e = cudaMemcpyAsync(h_scores, d_scores, P * 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) st = fail(CLIMBER_E_CUDA, "rank_host: %s", cudaGetErrorString(e));
  } else {
    cudaStreamSynchronize(s);
  }
  climber_kv_release(c, kv);
  return st;
}

// ---------------------------------------------------------------------------
// serving cache store (NEXT-4)
// ---------------------------------------------------------------------------
static bool pool_has_room(climber_ctx_s* c) {
  std::lock_guard<std::mutex> g(c->mu);
  return !c->free_slots.empty() && (long long)c->free_pages.size() >= c->per_slot;
}

// evict the least-recently-used unpinned entry; false if none
static bool store_evict_one(climber_ctx_s* c) {
  auto victim = c->store.end();
  for (auto it = c->store.begin(); it != c->store.end(); ++it)
    if (it->second.pins == 0 && (victim == c->store.end() || it->second.tick < victim->second.tick)) victim = it;
  if (victim == c->store.end()) return false;
  climber_kv_release(c, victim->second.kv);
  c->store.erase(victim);
  ++c->st_evict;
  return true;
}

extern "C" climber_status climber_cache_acquire(climber_ctx_t c, uint64_t user_key, int32_t scenario_r,
                                                uint64_t digest, const climber_events* events, int64_t n_s,
                                                climber_stream_t stream, climber_kv_t* out, int32_t* result) {
  if (!c || !events || !out || !result) return fail(CLIMBER_E_INVALID_ARG, "null argument");
  std::lock_guard<std::mutex> g(c->store_mu);
  const auto key = std::make_pair(user_key, (int)scenario_r);
  auto it = c->store.find(key);
  if (it != c->store.end() && it->second.digest == digest && !it->second.dropped) {
    it->second.pins++;
    it->second.tick = ++c->store_tick;
    ++c->st_hits;
    *out = it->second.kv;
    *result = CLIMBER_CACHE_HIT;
    return CLIMBER_OK;
  }
  ++c->st_miss;
  bool uncached = false;
  if (it != c->store.end()) {  // stale digest
    if (it->second.pins == 0) {
      climber_kv_release(c, it->second.kv);
      c->store.erase(it);
    } else {  // another caller still reads the old K/V: hand out an uncached build
      uncached = true;
    }
  }
  while (!pool_has_room(c))
    if (!store_evict_one(c)) return fail(CLIMBER_E_CAPACITY, "every cached handle is pinned");
  climber_kv_t kv;
  climber_status st = climber_encode_user(c, events, n_s, scenario_r, stream, &kv);
  if (st != CLIMBER_OK) return st;
  climber_ctx_s::CacheEntry e{kv, digest, 1, ++c->store_tick, uncached, n_s};
  if (uncached) c->orphans.push_back(e);
  else c->store[key] = e;
  *out = kv;
  *result = uncached ? CLIMBER_CACHE_UNCACHED : CLIMBER_CACHE_ENCODED;
  return CLIMBER_OK;
}

// Incremental update of a cached user whose event log grew by appending
// (PAPER.md L161's critique of static caches).  The
// blocks are independent (Eq. 2: S_k is a filter of S), so only the blocks
// whose strategy a_k matches an appended event change; their stacks are
// recomputed in place, the others keep their K/V (bit-identical to a full
// re-encode of the new log).  Extraction and the request-time bias rows are
// always redone (the request time moved).
extern "C" climber_status climber_cache_append(climber_ctx_t c, uint64_t user_key, int32_t scenario_r,
                                               uint64_t digest_prefix, uint64_t digest, const climber_events* events,
                                               int64_t n_s, climber_stream_t stream, climber_kv_t* out,
                                               int32_t* result, int32_t* blocks_recomputed) {
  if (!c || !events || !out || !result || !blocks_recomputed) return fail(CLIMBER_E_INVALID_ARG, "null argument");
  *blocks_recomputed = 0;
  {
    std::unique_lock<std::mutex> g(c->store_mu);
    auto it = c->store.find(std::make_pair(user_key, (int)scenario_r));
    const bool inplace = it != c->store.end() && it->second.digest == digest_prefix && !it->second.dropped &&
                         it->second.pins == 0 && n_s >= it->second.n_s && grouped_ok(c) &&
                         attn_tc_supported(c->D.dh, c->D.nk, true) && n_s > 0;
    if (inplace) {
      cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
      climber_ctx_s::CacheEntry& e = it->second;
      int slot;
      {
        std::lock_guard<std::mutex> gm(c->mu);
        climber_status rs = resolve(c, e.kv, &slot);
        if (rs != CLIMBER_OK) return rs;
      }
      const int Nb = c->D.Nb;
      if (!c->d_flags) CU(cudaMalloc(&c->d_flags, 64 * sizeof(int)));
      CU(cudaMemsetAsync(c->d_flags, 0, Nb * sizeof(int), s));
      if (n_s > e.n_s)
        launch_append_flags(events->action, events->scenario, e.n_s, n_s, c->amask, c->smask, c->d_flags, c->D, s);
      int flags[64];
      CU(cudaMemcpyAsync(flags, c->d_flags, Nb * sizeof(int), cudaMemcpyDeviceToHost, s));
      CU(cudaStreamSynchronize(s));
      {
        std::lock_guard<std::mutex> gm(c->mu);
        CU(cudaEventSynchronize(c->stage_evt));
        Stage h = stage_layout(c, c->h_stage);
        h.slots[0] = slot;
        h.r[0] = scenario_r;
        h.ev_off[0] = 0;
        h.ev_off[1] = n_s;
        climber_status rs = stage_upload(c, 1, false, s);
        if (rs != CLIMBER_OK) return rs;
      }
      EventsDev ev{events->item, events->action, events->scenario, events->ts};
      int done = 0;
      for (int k = 0; k < Nb;) {  // contiguous runs of changed blocks
        if (!flags[k]) { ++k; continue; }
        int k1 = k;
        while (k1 < Nb && flags[k1]) ++k1;
        encode_wave_grouped(c, ev, 0, 1, n_s, s, k, k1 - k);
        done += k1 - k;
        k = k1;
      }
      if (done == 0) encode_wave_grouped(c, ev, 0, 1, n_s, s, 0, 0);  // extraction + bias rows only
      climber_status rs = check_launch(c, s);
      if (rs != CLIMBER_OK) return rs;
      e.digest = digest;
      e.n_s = n_s;
      e.pins = 1;
      e.tick = ++c->store_tick;
      ++c->st_hits;
      *out = e.kv;
      *result = CLIMBER_CACHE_APPENDED;
      *blocks_recomputed = done;
      return CLIMBER_OK;
    }
  }
  // not incrementally updatable: a (re)build under the new digest
  *blocks_recomputed = c->D.Nb;
  return climber_cache_acquire(c, user_key, scenario_r, digest, events, n_s, stream, out, result);
}

extern "C" climber_status climber_cache_release(climber_ctx_t c, climber_kv_t kv) {
  if (!c) return fail(CLIMBER_E_INVALID_ARG, "null ctx");
  std::lock_guard<std::mutex> g(c->store_mu);
  for (auto& kvp : c->store)
    if (kvp.second.kv == kv) {
      if (kvp.second.pins <= 0) return fail(CLIMBER_E_STALE, "cache handle is not pinned");
      kvp.second.pins--;
      return CLIMBER_OK;
    }
  for (size_t i = 0; i < c->orphans.size(); ++i)
    if (c->orphans[i].kv == kv) {
      climber_kv_release(c, kv);
      c->orphans.erase(c->orphans.begin() + i);
      return CLIMBER_OK;
    }
  return fail(CLIMBER_E_STALE, "handle is not held by the cache store");
}

extern "C" climber_status climber_cache_stats(climber_ctx_t c, int64_t* stats) {
  if (!c || !stats) return fail(CLIMBER_E_INVALID_ARG, "null argument");
  std::lock_guard<std::mutex> g(c->store_mu);
  long long pinned = 0;
  for (auto& kvp : c->store) pinned += kvp.second.pins > 0;
  stats[0] = (int64_t)c->store.size();
  stats[1] = pinned + (int64_t)c->orphans.size();
  stats[2] = c->st_hits;
  stats[3] = c->st_miss;
  stats[4] = c->st_evict;
  return CLIMBER_OK;
}

// ---------------------------------------------------------------------------
// SUMI forward of compressed training records:
// one "single user, multiple items" record per user = history + its items in
// one pass (causal history, items full-visible to the history, diagonal among
// items), no cache kept: encode + score with transient handles.
// ---------------------------------------------------------------------------
extern "C" climber_status climber_forward(climber_ctx_t c, int32_t B, const int64_t* ev_offsets,
                                          const climber_events* events, const int32_t* scenario_r,
                                          const int64_t* cand_offsets, const int32_t* items, float* scores,
                                          climber_stream_t stream) {
  if (!c || !cand_offsets || !items || !scores) return fail(CLIMBER_E_INVALID_ARG, "null argument");
  if (B < 1 || B > c->cfg.max_batch_users) return fail(CLIMBER_E_INVALID_ARG, "B out of range");
  std::vector<climber_kv_t> kvs(B);
  climber_status st = climber_encode_users(c, B, ev_offsets, events, scenario_r, stream, kvs.data());
  if (st != CLIMBER_OK) return st;
  st = climber_score_items_batched(c, B, kvs.data(), cand_offsets, items, scores, stream);
  // the pages return to the pool now; later calls on this stream are ordered
  // after this one (other streams: synchronise first)
  for (int b = 0; b < B; ++b) climber_kv_release(c, kvs[b]);
  return st;
}

// ---------------------------------------------------------------------------
// end-to-end call with host buffers
// ---------------------------------------------------------------------------
extern "C" climber_status climber_rank_host(climber_ctx_t c, int32_t B, const int64_t* ev_offsets,
                                            const int32_t* item, const uint8_t* action, const uint8_t* scenario,
                                            const int64_t* ts, const int32_t* scenario_r,
                                            const int64_t* cand_offsets, const int32_t* items, float* scores,
                                            climber_stream_t stream) {
  if (!c || !ev_offsets || !scenario_r || !cand_offsets || !items || !scores)
    return fail(CLIMBER_E_INVALID_ARG, "null argument");
  if (B < 1 || B > c->cfg.max_batch_users) return fail(CLIMBER_E_INVALID_ARG, "B out of range");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int64_t E = ev_offsets[B] - ev_offsets[0], P = cand_offsets[B] - cand_offsets[0];
  if (E > 0 && (!item || !action || !scenario || !ts)) return fail(CLIMBER_E_INVALID_ARG, "null event array");
  size_t need = (size_t)E * (4 + 1 + 1 + 8) + (size_t)P * (4 + 4) + 4096;
  if (need > c->io_bytes) {
    if (c->io) cudaFree(c->io);
    c->io = nullptr;
    c->io_bytes = 0;
    CU(cudaMalloc(&c->io, need));
    c->io_bytes = need;
  }
  char* p = (char*)c->io;
  auto carve = [&](size_t bytes) { char* q = p; p += (bytes + 255) & ~size_t(255); return q; };
  int64_t* d_ts = (int64_t*)carve((size_t)E * 8);
  int32_t* d_item = (int32_t*)carve((size_t)E * 4);
  int32_t* d_items = (int32_t*)carve((size_t)P * 4);
  float* d_scores = (float*)carve((size_t)P * 4);
  uint8_t* d_act = (uint8_t*)carve((size_t)E);
  uint8_t* d_scn = (uint8_t*)carve((size_t)E);
  const int64_t e0 = ev_offsets[0], c0 = cand_offsets[0];
  if (E > 0) {
    CU(cudaMemcpyAsync(d_item, item + e0, E * 4, cudaMemcpyHostToDevice, s));
    CU(cudaMemcpyAsync(d_act, action + e0, E, cudaMemcpyHostToDevice, s));
    CU(cudaMemcpyAsync(d_scn, scenario + e0, E, cudaMemcpyHostToDevice, s));
    CU(cudaMemcpyAsync(d_ts, ts + e0, E * 8, cudaMemcpyHostToDevice, s));
  }
  CU(cudaMemcpyAsync(d_items, items + c0, P * 4, cudaMemcpyHostToDevice, s));
  std::vector<int64_t> eo(B + 1), co(B + 1);
  for (int b = 0; b <= B; ++b) {
    eo[b] = ev_offsets[b] - e0;
    co[b] = cand_offsets[b] - c0;
  }
  climber_events ev{d_item, d_act, d_scn, d_ts};
  if (B == 1 && c->graphs && !c->prof && !c->sync_check && grouped_ok(c) &&
      attn_tc_supported(c->D.dh, c->D.nk, true))
    return rank_one_graph(c, E, P, ev, scenario_r[0], d_items, d_scores, scores + c0, s);
  std::vector<climber_kv_t> kvs(B);
  climber_status st = climber_encode_users(c, B, eo.data(), &ev, scenario_r, stream, kvs.data());
  if (st != CLIMBER_OK) return st;
  st = climber_score_items_batched(c, B, kvs.data(), co.data(), d_items, d_scores, stream);
  if (st == CLIMBER_OK) {
    cudaError_t e = cudaMemcpyAsync(scores + c0, d_scores, P * 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) st = fail(CLIMBER_E_CUDA, "rank_host: %s", cudaGetErrorString(e));
  } else {
    cudaStreamSynchronize(s);
  }
  for (int b = 0; b < B; ++b) climber_kv_release(c, kvs[b]);
  return st;
}

// ---------------------------------------------------------------------------
// debug exports
// ---------------------------------------------------------------------------
extern "C" climber_status climber_debug_extract(climber_ctx_t c, climber_kv_t kv, int32_t* idx, int32_t* vlen) {
  if (!c || !idx || !vlen) return fail(CLIMBER_E_INVALID_ARG, "null argument");
  int slot;
  {
    std::lock_guard<std::mutex> g(c->mu);
    climber_status rs = resolve(c, kv, &slot);
    if (rs != CLIMBER_OK) return rs;
  }
  CU(cudaDeviceSynchronize());
  CU(cudaMemcpy(idx, c->idx_all + (size_t)slot * c->D.Nb * c->D.nk, (size_t)c->D.Nb * c->D.nk * 4,
                cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(vlen, c->vlen_all + (size_t)slot * c->D.Nb, (size_t)c->D.Nb * 4, cudaMemcpyDeviceToHost));
  return CLIMBER_OK;
}

extern "C" climber_status climber_debug_mask(climber_ctx_t c, climber_kv_t kv, int32_t M, uint8_t* mask) {
  if (!c || !mask || M < 1) return fail(CLIMBER_E_INVALID_ARG, "bad argument");
  int slot;
  {
    std::lock_guard<std::mutex> g(c->mu);
    climber_status rs = resolve(c, kv, &slot);
    if (rs != CLIMBER_OK) return rs;
  }
  size_t T = (size_t)c->D.nk + M, n = (size_t)c->D.Nb * T * T;
  uint8_t* d = nullptr;
  CU(cudaMalloc(&d, n));
  launch_debug_mask(c->vlen_all, slot, M, d, c->D, 0);
  c->launches++;
  cudaError_t e = cudaMemcpy(mask, d, n, cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) return fail(CLIMBER_E_CUDA, "debug_mask: %s", cudaGetErrorString(e));
  return CLIMBER_OK;
}

extern "C" climber_status climber_debug_kv(climber_ctx_t c, climber_kv_t kv, int32_t layer, int32_t block, void* K,
                                           void* V) {
  if (!c || !K || !V) return fail(CLIMBER_E_INVALID_ARG, "null argument");
  if (layer < 0 || layer >= c->D.L || block < 0 || block >= c->D.Nb) return fail(CLIMBER_E_INVALID_ARG, "layer/block");
  int slot;
  {
    std::lock_guard<std::mutex> g(c->mu);
    climber_status rs = resolve(c, kv, &slot);
    if (rs != CLIMBER_OK) return rs;
  }
  CU(cudaDeviceSynchronize());
  int v = 0;
  CU(cudaMemcpy(&v, c->vlen_all + (size_t)slot * c->D.Nb + block, 4, cudaMemcpyDeviceToHost));
  size_t bytes = (size_t)v * c->D.d * c->esz;
  if (bytes == 0) return CLIMBER_OK;
  void *dk = nullptr, *dv = nullptr;
  CU(cudaMalloc(&dk, bytes));
  CU(cudaMalloc(&dv, bytes));
  if (c->cfg.dtype == CLIMBER_BF16)
    launch_debug_kv<bf16>((const bf16*)c->pool, c->ptab, c->vlen_all, slot, block, layer, (bf16*)dk, (bf16*)dv, c->D, 0);
  else
    launch_debug_kv<float>((const float*)c->pool, c->ptab, c->vlen_all, slot, block, layer, (float*)dk, (float*)dv,
                           c->D, 0);
  c->launches++;
  cudaError_t e1 = cudaMemcpy(K, dk, bytes, cudaMemcpyDeviceToHost);
  cudaError_t e2 = cudaMemcpy(V, dv, bytes, cudaMemcpyDeviceToHost);
  cudaFree(dk);
  cudaFree(dv);
  if (e1 != cudaSuccess || e2 != cudaSuccess) return fail(CLIMBER_E_CUDA, "debug_kv copy failed");
  return CLIMBER_OK;
}

// Mask probe: the production attention kernel of `mode` run on the probe
// pattern of launch_probe_pages (see include/climber.h).  Synchronous; the
// handle's K/V of (layer, block) is overwritten.
extern "C" climber_status climber_debug_attn_probe(climber_ctx_t c, climber_kv_t kv, int32_t mode, int32_t layer,
                                                   int32_t block, int32_t M, int32_t key_off, float* out) {
  if (!c || !out) return fail(CLIMBER_E_INVALID_ARG, "null argument");
  const Dims& D = c->D;
  if ((mode != 0 && mode != 1) || layer < 0 || layer >= D.L || block < 0 || block >= D.Nb || key_off < 0)
    return fail(CLIMBER_E_INVALID_ARG, "mode/layer/block/key_off");
  if (mode == 1 && (M < 1 || M > D.Mmax)) return fail(CLIMBER_E_INVALID_ARG, "M out of [1, max_candidates]");
  if (c->cfg.rel_bias) return fail(CLIMBER_E_UNSUPPORTED, "attn probe: rel_bias contexts add f_b to the scores");
  int slot, r;
  {
    std::lock_guard<std::mutex> g(c->mu);
    climber_status rs = resolve(c, kv, &slot);
    if (rs != CLIMBER_OK) return rs;
    r = c->slots[slot].r;
    if (block < c->slots[slot].kb0 || block >= c->slots[slot].kb1)
      return fail(CLIMBER_E_INVALID_ARG, "block not held by this handle");
  }
  CU(cudaDeviceSynchronize());
  cudaStream_t s = 0;
  const int64_t coff[2] = {0, (int64_t)M};
  CU(cudaMemcpy(c->d_slots, &slot, 4, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(c->d_r, &r, 4, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(c->d_cand_off, coff, sizeof(coff), cudaMemcpyHostToDevice));
  const long long rows = mode == 0 ? D.nk : M;
  const bool b16 = c->cfg.dtype == CLIMBER_BF16;
  if (b16) launch_probe_pages<bf16>((bf16*)c->pool, c->ptab, slot, block, layer, key_off, D, s);
  else launch_probe_pages<float>((float*)c->pool, c->ptab, slot, block, layer, key_off, D, s);
  if (mode == 0) {
    CU(cudaMemsetAsync(c->QKV, 0, (size_t)rows * D.d * c->esz, s));
  } else if (b16) {
    launch_probe_qkv<bf16>((bf16*)c->QKV, rows, D, s);
  } else {
    launch_probe_qkv<float>((float*)c->QKV, rows, D, s);
  }
  CU(cudaMemsetAsync(c->O, 0, (size_t)rows * D.d * c->esz, s));
  if (b16) {
    if (mode == 0)
      attn_hist_bf16(c, (const bf16*)c->QKV, c->d_slots, c->d_r, 1, (bf16*)c->O, block, layer, s);
    else
      attn_sumi_bf16(c, (const bf16*)c->QKV, M, c->d_cand_off, c->d_slots, c->d_r, 1, M, (bf16*)c->O, block, layer,
                     s);
  } else {
    if (mode == 0)
      launch_attn_hist<float>((const float*)c->QKV, c->d_slots, c->d_r, 1, (const float*)c->pool, c->ptab,
                              c->vlen_all, c->tau, (float*)c->O, block, layer, D, s);
    else
      launch_attn_sumi<float>((const float*)c->QKV, c->d_cand_off, c->d_slots, c->d_r, 1, M, (const float*)c->pool,
                              c->ptab, c->vlen_all, c->tau, (float*)c->O, block, layer, D, s);
  }
  c->launches += 4;
  CU(cudaDeviceSynchronize());
  std::vector<uint8_t> h((size_t)rows * D.d * c->esz);
  CU(cudaMemcpy(h.data(), c->O, h.size(), cudaMemcpyDeviceToHost));
  for (long long i = 0; i < rows * D.d; ++i) {
    if (b16) {
      uint32_t u = (uint32_t)reinterpret_cast<const uint16_t*>(h.data())[i] << 16;
      memcpy(out + i, &u, 4);
    } else {
      out[i] = reinterpret_cast<const float*>(h.data())[i];
    }
  }
  return CLIMBER_OK;
}

extern "C" climber_status climber_debug_gemm(const void* A, const void* B, void* D, int64_t M, int32_t N, int32_t K,
                                             int32_t use_tc, int32_t epi, climber_stream_t stream) {
  if (!A || !B || !D || M < 1 || N < 1 || K < 1 || epi < 0 || epi > 3)
    return fail(CLIMBER_E_INVALID_ARG, "bad argument");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (epi == 3) {
    // grouped (2 interleaved blocks): A is [M][2][K] (block b = columns b*K..), B is [2][N][K],
    // D is fp32 [M][2][N] += A_b B_b^T -- the candidate-block layout of the batched path
    if (!use_tc || !gemm_tc_supported(M, N, K, 2 * K, K)) return fail(CLIMBER_E_UNSUPPORTED, "shape");
    Epilogue e = epi_resid(reinterpret_cast<float*>(D), 2LL * N);
    e.out_bs = N;
    launch_gemm_tc_batched((const bf16*)A, 2LL * K, K, (const bf16*)B, K, (long long)N * K, M, N, K, 2, e, s);
    CU(cudaGetLastError());
    return CLIMBER_OK;
  }
  Epilogue e = epi == 0 ? epi_resid(reinterpret_cast<float*>(D), N)
                        : epi_store(D, N, epi == 2 ? ACT_SILU : ACT_NONE);
  if (use_tc) {
    if (!gemm_tc_supported(M, N, K, K, K)) return fail(CLIMBER_E_UNSUPPORTED, "shape not supported by tcgen05 GEMM");
    launch_gemm_tc((const bf16*)A, K, (const bf16*)B, K, M, N, K, e, s);
  } else {
    if (K % 16 || N % 4) return fail(CLIMBER_E_UNSUPPORTED, "shape not supported by SIMT GEMM");
    launch_gemm_simt<bf16>((const bf16*)A, K, (const bf16*)B, K, M, N, K, e, s);
  }
  CU(cudaGetLastError());
  return CLIMBER_OK;
}

extern "C" climber_status climber_profile(climber_ctx_t c, int32_t enable) {
  if (!c) return fail(CLIMBER_E_INVALID_ARG, "null ctx");
  c->prof = enable != 0;
  return CLIMBER_OK;
}

extern "C" climber_status climber_profile_read(climber_ctx_t c, double* out) {
  if (!c || !out) return fail(CLIMBER_E_INVALID_ARG, "null argument");
  for (int i = 0; i < 4 * CLIMBER_K_NUM; ++i) out[i] = 0;
  for (const ProfRec& r : c->recs) {
    CU(cudaEventSynchronize(r.e1));
    float ms = 0.f;
    CU(cudaEventElapsedTime(&ms, r.e0, r.e1));
    double* o = out + 4 * r.cls;
    o[0] += 1;
    o[1] += ms;
    o[2] += r.flops;
    o[3] += r.bytes;
  }
  c->recs.clear();
  c->ev_next = 0;
  return CLIMBER_OK;
}

extern "C" int64_t climber_launch_count(climber_ctx_t c) { return c ? c->launches : -1; }

extern "C" const char* climber_last_error(void) { return g_last_error.c_str(); }
