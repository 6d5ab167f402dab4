// C-ABI layer of libleanattn.so (include/la.h): argument validation, plan ownership of
// device state, launch configuration.  Every step of the decode path runs in the kernels
// of decode.cu; this file only plans (integer work, planner.cpp) and marshals.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "la_internal.h"

using la::DevUnit;

struct la_plan_s {
  la::Problem prob;
  la::Schedule sched;
  la::KernelInfo kinfo;
  int stage_tokens = 0;
  bool host_only = true;
  int split = 0;             // LA_SCHED_FIXED_SPLIT: chunks per unit actually used
  int pt_stride = 0;         // LA_KV_PAGED: padded block-table row stride
  int device = -1;
  int engine = -1;           // la_engine of the T_m > 1 tiles (-1: CUDA cores / FP8 engine)
  // planning options, kept for la_plan_update
  int opt_grid = 0, opt_dyn_first = 750, opt_dyn_min = 2, opt_split = 0;
  int max_ctas = 0;          // co-resident CTAs (device) / num_sms x ctas_per_sm (host-only)
  int slot_cap = 0;          // (virtual) CTA capacity of the range table, partial slots, flags
  int64_t updates = 0;       // la_plan_update calls
  std::vector<int32_t> weights;  // la_plan_set_weights: per-CTA stream-K weights (empty: Eq. 2's equal ranges)
  // ---- device state, ONE allocation ---------------------------------------------------
  // upload region (rewritten by la_plan_update with one async copy):
  //   [hdr 256 B][units U x 48 B][cta_begin cap + 1][cta_first cap][claim cap][block table B x pt_stride]
  // then kernel state: partials [2][cap][rows][d] + [2][cap][rows][4], flags [cap],
  //   counters [kNumCounters] + unit_count [U], trace, engine fold scratch
  void* d_tables = nullptr;
  size_t up_bytes = 0, off_units = 0, off_begin = 0, off_first = 0, off_claim = 0, off_bt = 0;
  int32_t* d_hdr = nullptr;
  DevUnit* d_units = nullptr;
  int32_t* d_cta_begin = nullptr;
  int32_t* d_cta_first = nullptr;
  int32_t* d_claim = nullptr;
  int32_t* d_block_table = nullptr;
  float* d_part_o = nullptr;
  float* d_part_ml = nullptr;
  uint32_t* d_flags = nullptr;
  int* d_counters = nullptr;
  int* d_unit_count = nullptr;
  unsigned long long* d_trace = nullptr;
  float* d_gfold = nullptr;
  unsigned char* h_stage = nullptr;   // pinned host copy of the upload region
  cudaEvent_t up_done = nullptr;      // the last upload's copy has left h_stage
  bool up_pending = false;
  int64_t workspace = 0;
  la::TmapCache tmaps;                // K / V tensor maps of the last (k, v, rows)
  // la_decode_host staging
  void* d_stage = nullptr;
  size_t stage_bytes = 0;
  // NEXT-2 cross-GPU exchange (xw > 1)
  int xw = 0, xr = 0;
  void* d_xchg = nullptr;           // own buffer (separate allocation: it is IPC-exported)
  size_t xflag_off = 0;
  float* xpeer[la::kMaxXchgWorld] = {};
  bool xpeer_ipc[la::kMaxXchgWorld] = {};
};

namespace {

thread_local std::string g_err;

la_status fail(la_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

la_status cuda_fail(cudaError_t e, const char* what) {
  g_err = std::string(what) + ": " + cudaGetErrorString(e);
  cudaGetLastError();  // clear sticky-less errors
  return LA_ERR_CUDA;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

int auto_tile_n(const la::Problem& p) {
  // 64 KiB of K+V per LeanTile: 128 tokens at d=128 and 256 at d=64 for 16-bit inputs,
  // the sizes the paper's sweep found, whatever the problem size.  Smaller tiles
  // for problems with fewer LeanTiles than SMs were measured never faster on B200 and up to
  // 18% slower (a single-unit problem split over more CTAs has its host fold more peers; the
  // load is latency-, not bandwidth-bound at that size).
  const int row_bytes = p.head_dim * p.elem_bytes();
  return std::max(32, std::min(512, 65536 / (2 * row_bytes)));
}

void release_device(la_plan_s* p) {
  for (int r = 0; r < la::kMaxXchgWorld; ++r)
    if (p->xpeer_ipc[r] && p->xpeer[r]) cudaIpcCloseMemHandle(p->xpeer[r]);
  if (p->d_xchg) cudaFree(p->d_xchg);
  if (p->d_tables) cudaFree(p->d_tables);
  if (p->d_stage) cudaFree(p->d_stage);
  if (p->h_stage) cudaFreeHost(p->h_stage);
  if (p->up_done) cudaEventDestroy(p->up_done);
  p->d_tables = nullptr;
  p->d_stage = nullptr;
  p->d_xchg = nullptr;
  p->h_stage = nullptr;
  p->up_done = nullptr;
}

// Exchange buffer layout: a 256-B head -- the error word at +0 and the owner's shape header
// at +64, at a fixed offset so a peer can read it before it knows the shape (checked by
// la_plan_xchg_open) -- then the data DecodeArgs::xpeer points at: [2][P][rows][d + 4] fp32
// and, at xflag_off from there, [P][units] uint32 flags.
constexpr size_t kXchgHead = 256;
size_t xchg_flag_off(const la::Problem& p, int P) {
  return align256(size_t(2) * P * p.q_rows() * (p.head_dim + 4) * sizeof(float));
}
size_t xchg_bytes(const la::Problem& p, int P) {
  return kXchgHead + xchg_flag_off(p, P) + align256(size_t(P) * p.num_units() * sizeof(uint32_t));
}
constexpr int kXchgHdrInts = 12;
void xchg_header(const la_plan_s* pl, int32_t (&h)[kXchgHdrInts]) {
  const la::Problem& p = pl->prob;
  const int64_t rows = p.q_rows(), units = p.num_units();
  const int32_t v[kXchgHdrInts] = {0x4c415848 /* "LAXH" */, p.batch, p.heads_q, p.heads_kv, p.head_dim, p.dtype,
                                   int32_t(rows), int32_t(units), pl->xw, pl->xr, p.tile_rows, 0};
  std::memcpy(h, v, sizeof(v));
}

// I if every request had its capacity length: BHSD with an explicit max_ctx, paged pools
// (pages_per_seq x page_size).  Sizes the launch grid so that a plan updated to longer
// contexts keeps one CTA per SM.  Else the current I.
int64_t capacity_iters(const la::Problem& p, int tile_n, bool explicit_max_ctx, int64_t cur) {
  int64_t cap_len = 0;
  if (p.layout == LA_KV_BHSD && explicit_max_ctx) cap_len = p.max_ctx;
  if (p.layout == LA_KV_PAGED) cap_len = int64_t(p.pages_per_seq) * p.page_size;
  if (cap_len <= 0) return cur;
  const int64_t per = (cap_len + tile_n - 1) / tile_n;
  return std::max(cur, per * (p.num_units()));
}

// Alg2§4-18 for the plan's current ctx_lens: units in memory order, the (virtual) CTA
// ranges of the plan's schedule, host / last CTA per unit.  `launch` (CTAs launched) is
// chosen on the first call and kept: a CUDA graph captured on the plan keeps its grid, and
// CTAs without a range exit at once.
la_status plan_schedule(la_plan_s* plan, bool first, int64_t icap_hint) {
  const la::Problem& p = plan->prob;
  la::Schedule& s = plan->sched;
  const int M = plan->max_ctas;
  la::build_units(p, s.tile_n, s.units, s.total_iters);
  if (s.total_iters >= (int64_t(1) << 31)) return fail(LA_ERR_INVALID, "too many LeanTiles");
  const int64_t I = s.total_iters;
  if (first) {
    const int64_t icap = std::max(I, icap_hint);
    int launch;
    if (p.schedule == LA_SCHED_SEQUENTIAL)
      launch = int(s.units.size());
    else if (plan->opt_grid)
      launch = (plan->host_only && p.schedule == LA_SCHED_STREAMK) ? plan->opt_grid : std::min(plan->opt_grid, M);
    else
      launch = int(std::max<int64_t>(1, std::min<int64_t>(M, icap)));
    s.phys_grid = std::max(1, launch);
  }
  const int launch = s.phys_grid;
  plan->split = 0;
  if (p.schedule == LA_SCHED_SEQUENTIAL) {
    la::sequential_ranges(s.units, s.cta_begin);
  } else if (p.schedule == LA_SCHED_DYNAMIC) {
    const int G = plan->opt_grid ? launch : int(std::max<int64_t>(1, std::min<int64_t>(launch, I)));
    la::balanced_ranges(I, G, plan->opt_dyn_first, plan->opt_dyn_min, la::kMaxTailChunks, s.cta_begin, s.claim);
  } else if (p.schedule == LA_SCHED_FIXED_SPLIT) {
    int64_t max_cn = 1;
    for (const DevUnit& u : s.units) max_cn = std::max<int64_t>(max_cn, u.iter_end - u.iter_begin);
    plan->split = plan->opt_split ? plan->opt_split : la::fa2_num_splits(int64_t(s.units.size()), max_cn, M);
    la::fixed_split_ranges(s.units, plan->split, s.cta_begin);
  } else {
    // stream-K (Eq. 2): G = forced grid, else min(launch, I) equal ranges (reading C15)
    const int G = plan->opt_grid ? launch : int(std::max<int64_t>(1, std::min<int64_t>(launch, I)));
    if (plan->weights.empty()) {
      la::streamk_ranges(I, G, s.cta_begin);
    } else {  // SM-rate-weighted ranges (la_plan_set_weights): CTA g keeps weight g
      const std::vector<int32_t> w(plan->weights.begin(), plan->weights.begin() + G);
      la::weighted_ranges(I, w, s.cta_begin);
    }
  }
  if (p.schedule != LA_SCHED_DYNAMIC) {  // ranges are claimed in order
    s.claim.resize(s.cta_begin.size() - 1);
    for (size_t v = 0; v < s.claim.size(); ++v) s.claim[v] = int32_t(v);
  }
  la::finish_schedule(s);
  return LA_OK;
}

// Quantization efficiency: I / (W x max_w load_w).  Static schedules:
// W = the ranges (one CTA each); dynamic / fixed split: W = the persistent CTAs, the c-th
// claimed range on CTA c mod W (the launch-order wave model, as oracle.fixed_split_segments
// deals chunks; the run-time claims of the dynamic schedule are faster than this model).
double quant_eff(const la_plan_s* plan) {
  const la::Schedule& s = plan->sched;
  const bool waves = plan->prob.schedule == LA_SCHED_DYNAMIC || plan->prob.schedule == LA_SCHED_FIXED_SPLIT;
  const int W = waves ? s.phys_grid : s.grid;
  if (W < 1 || s.total_iters < 1) return 0.0;
  std::vector<int64_t> load(size_t(W), 0);
  for (int c = 0; c < s.grid; ++c) {
    const int v = waves ? s.claim[size_t(c)] : c;
    load[size_t(waves ? c % W : c)] += s.cta_begin[v + 1] - s.cta_begin[v];
  }
  const int64_t mx = *std::max_element(load.begin(), load.end());
  return mx > 0 ? double(s.total_iters) / (double(W) * double(mx)) : 0.0;
}

// Copy the current schedule (and block table) into the pinned staging buffer and upload it
// with ONE async H2D on `stream`.  sync: also wait for it (la_plan without a stream).
la_status upload_tables(la_plan_s* plan, cudaStream_t stream, bool sync) {
  const la::Schedule& s = plan->sched;
  if (plan->up_pending) {  // the previous upload may still be reading the staging buffer
    cudaError_t e = cudaEventSynchronize(plan->up_done);
    if (e != cudaSuccess) return cuda_fail(e, "la_plan_update: previous upload");
    plan->up_pending = false;
  }
  unsigned char* h = plan->h_stage;
  const int32_t hdr[4] = {s.grid, 0, 0, 0};
  std::memcpy(h, hdr, sizeof(hdr));
  std::memcpy(h + plan->off_units, s.units.data(), s.units.size() * sizeof(DevUnit));
  // the kernel reads no range count: the tables are padded to the plan's capacity with empty
  // ranges [I, I) (static CTAs past the schedule idle) and claims of -1 (a dynamic CTA that
  // draws one has no more work; every CTA draws exactly one, so cap + launch entries)
  const int CAP = plan->slot_cap;
  int32_t* cb = reinterpret_cast<int32_t*>(h + plan->off_begin);
  int32_t* cf = reinterpret_cast<int32_t*>(h + plan->off_first);
  int32_t* cl = reinterpret_cast<int32_t*>(h + plan->off_claim);
  std::memcpy(cb, s.cta_begin.data(), size_t(s.grid + 1) * sizeof(int32_t));
  std::fill(cb + s.grid + 1, cb + CAP + 1, int32_t(s.total_iters));
  std::memcpy(cf, s.cta_first_unit.data(), size_t(s.grid) * sizeof(int32_t));
  std::fill(cf + s.grid, cf + CAP, int32_t(s.units.empty() ? 0 : s.units.size() - 1));
  std::memcpy(cl, s.claim.data(), size_t(s.grid) * sizeof(int32_t));
  std::fill(cl + s.grid, cl + CAP + s.phys_grid, int32_t(-1));
  const la::Problem& p = plan->prob;
  if (plan->pt_stride) {  // block table, rows padded to pt_stride (the producer reads 32-entry windows)
    int32_t* bt = reinterpret_cast<int32_t*>(h + plan->off_bt);
    for (int b = 0; b < p.batch; ++b) {
      std::copy(p.block_table.begin() + size_t(b) * p.pages_per_seq,
                p.block_table.begin() + size_t(b + 1) * p.pages_per_seq, bt + size_t(b) * plan->pt_stride);
      std::fill(bt + size_t(b) * plan->pt_stride + p.pages_per_seq, bt + size_t(b + 1) * plan->pt_stride, 0);
    }
  }
  cudaError_t e = cudaMemcpyAsync(plan->d_tables, h, plan->up_bytes, cudaMemcpyHostToDevice, stream);
  if (e == cudaSuccess) e = cudaEventRecord(plan->up_done, stream);
  if (e == cudaSuccess && sync) e = cudaEventSynchronize(plan->up_done);
  if (e != cudaSuccess) return cuda_fail(e, "schedule upload");
  plan->up_pending = !sync;
  return LA_OK;
}

la_status check_lens(const la::Problem& p, const int32_t* ctx_lens, int64_t* maxn_out) {
  int64_t maxn = 0;
  for (int b = 0; b < p.batch; ++b) {
    if (ctx_lens[b] < 1) return fail(LA_ERR_INVALID, "every ctx_lens[b] must be >= 1 (reading C6)");
    if (ctx_lens[b] < p.q_lens[b])
      return fail(LA_ERR_INVALID, "ctx_lens[b] must be >= q_lens[b] (the queries are cached tokens)");
    maxn = std::max<int64_t>(maxn, ctx_lens[b]);
  }
  *maxn_out = maxn;
  return LA_OK;
}

la_status check_block_table(const la::Problem& p, const int32_t* bt) {
  for (int b = 0; b < p.batch; ++b)
    for (int i = 0; i < (p.ctx_lens[b] + p.page_size - 1) / p.page_size; ++i) {
      const int32_t pg = bt[size_t(b) * p.pages_per_seq + i];
      if (pg < 0 || pg >= p.num_pages) return fail(LA_ERR_INVALID, "block_table entry out of range");
    }
  return LA_OK;
}

}  // namespace

extern "C" {

int la_version(void) { return LA_VERSION; }

const char* la_last_error(void) { return g_err.c_str(); }

const char* la_status_string(la_status s) {
  switch (s) {
    case LA_OK: return "LA_OK";
    case LA_ERR_INVALID: return "LA_ERR_INVALID";
    case LA_ERR_UNSUPPORTED: return "LA_ERR_UNSUPPORTED";
    case LA_ERR_CUDA: return "LA_ERR_CUDA";
    case LA_ERR_NOMEM: return "LA_ERR_NOMEM";
    case LA_ERR_STATE: return "LA_ERR_STATE";
    case LA_ERR_TIMEOUT: return "LA_ERR_TIMEOUT";
  }
  return "LA_ERR_UNKNOWN";
}

int64_t la_launch_count(void) { return la::launch_count(); }

la_status la_plan_opts_init(la_plan_opts* o) {
  if (!o) return fail(LA_ERR_INVALID, "opts is NULL");
  std::memset(o, 0, sizeof(*o));
  o->layout = LA_KV_BHSD;
  o->num_sms = 148;
  o->ctas_per_sm = 1;
  o->schedule = LA_SCHED_AUTO;
  o->dyn_first_permille = 940;
  o->dyn_min_chunk = 2;
  o->q_len = 1;
  o->causal = 1;
  o->engine = LA_ENGINE_AUTO;
  return LA_OK;
}

la_status la_plan(int batch, int heads_q, int heads_kv, int head_dim, const int32_t* ctx_lens,
                  int tile_n, la_dtype dtype, const la_plan_opts* opts_in, la_plan_t* out) {
  if (!out) return fail(LA_ERR_INVALID, "out is NULL");
  *out = nullptr;
  la_plan_opts opts;
  la_plan_opts_init(&opts);
  if (opts_in) opts = *opts_in;
  if (batch < 1 || heads_q < 1 || heads_kv < 1) return fail(LA_ERR_INVALID, "batch/heads must be >= 1");
  if (heads_q % heads_kv) return fail(LA_ERR_INVALID, "heads_q must be a multiple of heads_kv (reading C3)");
  if (!ctx_lens) return fail(LA_ERR_INVALID, "ctx_lens is NULL");
  if (head_dim != 64 && head_dim != 128) return fail(LA_ERR_UNSUPPORTED, "head_dim must be 64 or 128");
  if (dtype != LA_BF16 && dtype != LA_FP16 && dtype != LA_FP32 && dtype != LA_FP8_E4M3)
    return fail(LA_ERR_INVALID, "bad dtype");
  if (dtype == LA_FP8_E4M3 && head_dim != 128) return fail(LA_ERR_UNSUPPORTED, "FP8 KV needs head_dim 128");
  if (opts.layout != LA_KV_BHSD && opts.layout != LA_KV_PACKED && opts.layout != LA_KV_PAGED)
    return fail(LA_ERR_INVALID, "bad layout");
  if (opts.schedule != LA_SCHED_STREAMK && opts.schedule != LA_SCHED_SEQUENTIAL &&
      opts.schedule != LA_SCHED_DYNAMIC && opts.schedule != LA_SCHED_FIXED_SPLIT && opts.schedule != LA_SCHED_AUTO)
    return fail(LA_ERR_INVALID, "bad schedule");
  if (opts.split < 0) return fail(LA_ERR_INVALID, "split must be >= 0");
  if (opts.dyn_first_permille < 0 || opts.dyn_first_permille > 1000 || opts.dyn_min_chunk < 1)
    return fail(LA_ERR_INVALID, "dyn_first_permille must be in [0, 1000] and dyn_min_chunk >= 1");
  if (tile_n != 0 && tile_n != 16 && tile_n != 32 && tile_n != 64 && tile_n != 128 && tile_n != 256 &&
      tile_n != 512)
    return fail(LA_ERR_INVALID, "tile_n must be 0 or one of 16..512 (powers of two)");
  if (opts.grid < 0) return fail(LA_ERR_INVALID, "grid must be >= 0");
  const int xw = opts.xchg_world > 1 ? opts.xchg_world : 0;
  if (opts.xchg_world < 0 || xw > la::kMaxXchgWorld)
    return fail(LA_ERR_INVALID, "xchg_world must be in 0..8");
  if (xw && (opts.xchg_rank < 0 || opts.xchg_rank >= xw)) return fail(LA_ERR_INVALID, "xchg_rank out of range");

  la::Problem p;
  p.batch = batch;
  p.heads_q = heads_q;
  p.heads_kv = heads_kv;
  p.head_dim = head_dim;
  p.group = heads_q / heads_kv;
  if (opts.q_len < 1) return fail(LA_ERR_INVALID, "q_len must be >= 1");
  p.causal = opts.causal ? 1 : 0;
  if (opts.q_lens) {
    p.q_lens.assign(opts.q_lens, opts.q_lens + batch);
    for (int32_t n : p.q_lens)
      if (n < 1) return fail(LA_ERR_INVALID, "every q_lens[b] must be >= 1");
  } else {
    p.q_lens.assign(batch, opts.q_len);
  }
  int max_rows = 0;
  bool uniform = true;
  for (int32_t n : p.q_lens) {
    max_rows = std::max(max_rows, p.group * n);
    uniform = uniform && n == p.q_lens[0];
  }
  p.q_len = uniform ? p.q_lens[0] : 0;
  // Engine for T_m > 1 tiles.  AUTO takes tcgen05 (measured): more than 8 rows per
  // KV head (g * N_q > 8), which its N = 16 / 32 MMAs cover in one pass over the cache where
  // mma.sync tiles need two / four, and the 8-row tiles of a BHSD / packed cache.
  if (opts.engine != LA_ENGINE_MMA_SYNC && opts.engine != LA_ENGINE_TCGEN05 && opts.engine != LA_ENGINE_AUTO)
    return fail(LA_ERR_INVALID, "engine must be LA_ENGINE_AUTO, LA_ENGINE_MMA_SYNC or LA_ENGINE_TCGEN05");
  const bool tc5_ok = head_dim == 128 && (dtype == LA_BF16 || dtype == LA_FP16);
  // AUTO resolves to stream-K for multi-row tiles (below), so it admits the wide tcgen05 tiles
  const bool static_sched = opts.schedule == LA_SCHED_STREAMK || opts.schedule == LA_SCHED_SEQUENTIAL ||
                            opts.schedule == LA_SCHED_AUTO;
  // (r02: 8-row tiles too -- c3 at parity after the round-2 engine work, tcgen05 ahead in the
  // last two same-box series: 304.5 vs 305.1 us over 5 alternating runs, 305.1 vs 305.5 us --
  // except on paged pools, where it measured box-dependent: 323 vs 331 us on one box, 338 vs
  // 332 us on two others; 16/32-row tiles need a static schedule)
  const bool tc5_wins = max_rows > 8 ? static_sched : opts.layout != LA_KV_PAGED;
  const int engine = opts.engine != LA_ENGINE_AUTO ? opts.engine
                     : (tc5_wins && tc5_ok ? LA_ENGINE_TCGEN05 : LA_ENGINE_MMA_SYNC);
  // T_m: 1 -> CUDA-core engine, else tensor-core tiles of <= 8 rows (mma.sync: N = 8), or
  // <= 32 on the tcgen05 engine (N = 16 / 32 per MMA at no extra cost: one KV pass per 32 rows)
  const bool wide = engine == LA_ENGINE_TCGEN05 && tc5_ok;
  p.tile_rows = std::min(wide ? 32 : 8, max_rows);
  if (xw && p.causal)
    for (int32_t n : p.q_lens)
      if (n > 1) return fail(LA_ERR_UNSUPPORTED, "sequence-shard exchange needs N_b == 1 or causal == 0");
  if (p.q_rows() >= (int64_t(1) << 31)) return fail(LA_ERR_INVALID, "too many query rows");
  p.dtype = dtype;
  p.layout = opts.layout;
  p.schedule = opts.schedule;
  p.ctx_lens.assign(ctx_lens, ctx_lens + batch);
  int64_t maxn = 0, total = 0;
  for (int32_t n : p.ctx_lens) {
    if (n < 1) return fail(LA_ERR_INVALID, "every ctx_lens[b] must be >= 1 (reading C6)");
    maxn = std::max<int64_t>(maxn, n);
    total += n;
  }
  for (int b = 0; b < batch; ++b)
    if (p.ctx_lens[b] < p.q_lens[b])
      return fail(LA_ERR_INVALID, "ctx_lens[b] must be >= q_lens[b] (the queries are cached tokens)");
  p.max_ctx = opts.max_ctx ? opts.max_ctx : maxn;
  if (p.layout == LA_KV_BHSD && p.max_ctx < maxn) return fail(LA_ERR_INVALID, "max_ctx < max(ctx_lens)");
  p.scale = opts.scale != 0.f ? opts.scale : float(1.0 / std::sqrt(double(head_dim)));
  if (!(p.scale > 0.f) || !std::isfinite(p.scale)) return fail(LA_ERR_INVALID, "scale must be finite and > 0");
  if (dtype == LA_FP8_E4M3) {
    p.k_scale = opts.k_scale != 0.f ? opts.k_scale : 1.f;
    p.v_scale = opts.v_scale != 0.f ? opts.v_scale : 1.f;
    if (!(p.k_scale > 0.f) || !std::isfinite(p.k_scale) || !(p.v_scale > 0.f) || !std::isfinite(p.v_scale))
      return fail(LA_ERR_INVALID, "k_scale / v_scale must be finite and > 0");
  }
  if (opts.block_table && p.layout != LA_KV_PAGED)
    return fail(LA_ERR_INVALID, "block_table given for a non-paged layout");
  if (p.layout == LA_KV_PAGED) {
    const int ps = opts.page_size;
    if (ps != 16 && ps != 32 && ps != 64 && ps != 128 && ps != 256)
      return fail(LA_ERR_INVALID, "page_size must be 16, 32, 64, 128 or 256");
    if (!opts.block_table) return fail(LA_ERR_INVALID, "paged layout needs a block_table");
    if (opts.num_pages < 1) return fail(LA_ERR_INVALID, "num_pages must be >= 1");
    if (int64_t(opts.pages_per_seq) * ps < maxn)
      return fail(LA_ERR_INVALID, "pages_per_seq * page_size < max(ctx_lens)");
    p.page_size = ps;
    p.pages_per_seq = opts.pages_per_seq;
    p.num_pages = opts.num_pages;
    p.block_table.assign(opts.block_table, opts.block_table + size_t(batch) * opts.pages_per_seq);
    la_status st = check_block_table(p, p.block_table.data());
    if (st != LA_OK) return st;
  }

  auto* plan = new (std::nothrow) la_plan_s();
  if (!plan) return fail(LA_ERR_NOMEM, "host allocation failed");
  plan->prob = p;
  plan->host_only = opts.host_only != 0;
  plan->xw = xw;
  plan->xr = xw ? opts.xchg_rank : 0;
  plan->opt_grid = opts.grid;
  // exchange plans claim the dynamic schedule's ranges in iteration order (no tail chunks):
  // the cross-GPU deadlock-freedom argument needs every CTA to visit units in increasing order
  plan->opt_dyn_first = xw ? 1000 : opts.dyn_first_permille;
  plan->opt_dyn_min = opts.dyn_min_chunk;
  plan->opt_split = opts.split;

  // ---- co-resident CTA budget (reading C15) -----------------------------------------
  if (plan->host_only) {
    plan->max_ctas = std::max(1, opts.num_sms) * std::max(1, opts.ctas_per_sm);
  } else {
    if (engine == LA_ENGINE_TCGEN05 && p.rows() > 1 && dtype == LA_FP8_E4M3) {
      delete plan;
      return fail(LA_ERR_UNSUPPORTED, "LA_ENGINE_TCGEN05 covers T_m > 1 tiles of a bf16 / fp16 cache");
    }
    plan->kinfo = la::decode_kernel_info(dtype, head_dim, p.rows(), p.rows() > 1 ? engine : 0);
    plan->engine = p.rows() > 1 && dtype != LA_FP8_E4M3 ? engine : -1;
    if (plan->kinfo.global_fold_floats > 0 && (p.schedule == LA_SCHED_DYNAMIC || p.schedule == LA_SCHED_FIXED_SPLIT)) {
      delete plan;  // their fold tree stages peers in the (shared-memory) fold buffer
      return fail(LA_ERR_UNSUPPORTED, "16-row tcgen05 tiles run the static schedules (streamk, sequential)");
    }
    if (!plan->kinfo.supported) {
      delete plan;
      return fail(LA_ERR_UNSUPPORTED, "no decode kernel for this (dtype, head_dim, group) in this build");
    }
    cudaError_t e = cudaGetDevice(&plan->device);
    if (e != cudaSuccess) { delete plan; return cuda_fail(e, "cudaGetDevice"); }
    int sms = 0, occ = 0;
    e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, plan->device);
    if (e != cudaSuccess) { delete plan; return cuda_fail(e, "cudaDeviceGetAttribute"); }
    e = cudaFuncSetAttribute(plan->kinfo.fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             plan->kinfo.smem_bytes);
    if (e != cudaSuccess) { delete plan; return cuda_fail(e, "cudaFuncSetAttribute"); }
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, plan->kinfo.fn, plan->kinfo.threads,
                                                      plan->kinfo.smem_bytes);
    if (e != cudaSuccess) { delete plan; return cuda_fail(e, "cudaOccupancyMaxActiveBlocksPerMultiprocessor"); }
    if (occ < 1) { delete plan; return fail(LA_ERR_UNSUPPORTED, "decode kernel does not fit on an SM"); }
    if (plan->kinfo.uses_tma_tensor && p.kv_rows() >= (int64_t(1) << 31)) {
      delete plan;
      return fail(LA_ERR_UNSUPPORTED, "KV cache rows exceed the TMA int32 coordinate range");
    }
    plan->max_ctas = sms * occ;
  }

  // ---- schedule (Alg2§4-18) -----------------------------------------------------------
  plan->sched.tile_n = tile_n ? tile_n : auto_tile_n(p);
  if (p.schedule == LA_SCHED_AUTO) {
    // the balanced dynamic schedule for one-row tiles whose Eq. 2 ranges are long enough for a
    // tail to matter (measured faster on B200: c2 -1%, c4 -1%, c5 -1%); stream-K for multi-row
    // tiles (whose 8-32-row folds cost more per piece than the balance gains) and exchange plans
    std::vector<DevUnit> tmp;
    int64_t I = 0;
    la::build_units(p, plan->sched.tile_n, tmp, I);
    const int64_t G = std::max<int64_t>(1, std::min<int64_t>(plan->opt_grid ? plan->opt_grid : plan->max_ctas, I));
    // (measured slower with dynamic, r02: the FP8 engine -- c2 314 vs 309 us -- and paged pools,
    // whose producer refills a page window at every piece -- c2 page 16: 650 vs 622 us)
    p.schedule = (p.rows() == 1 && !xw && I / G >= 64 && p.dtype != LA_FP8_E4M3 && p.layout != LA_KV_PAGED)
                     ? LA_SCHED_DYNAMIC : LA_SCHED_STREAMK;
    plan->prob.schedule = p.schedule;
  }
  {
    const int64_t icap = capacity_iters(p, plan->sched.tile_n, opts.max_ctx > 0, 0);
    la_status st = plan_schedule(plan, true, icap);
    if (st != LA_OK) { delete plan; return st; }
  }
  la::Schedule& s = plan->sched;
  if (!plan->host_only && p.schedule == LA_SCHED_STREAMK && s.phys_grid > plan->max_ctas) {
    delete plan;
    return fail(LA_ERR_INVALID, "grid exceeds the co-resident CTA count");
  }
  plan->stage_tokens = plan->host_only ? std::min(s.tile_n, 64) : std::min(s.tile_n, plan->kinfo.stage_tokens_max);
  // capacity of (virtual) CTAs: static schedules never exceed the launch grid (stream-K) or the
  // unit count (sequential), the dynamic one (1 + kMaxTailChunks) pieces per range; the
  // fixed-split chunk count varies with ctx_lens, so leave room
  if (p.schedule == LA_SCHED_DYNAMIC)
    plan->slot_cap = std::max(s.grid, s.phys_grid * (1 + la::kMaxTailChunks));
  else if (p.schedule == LA_SCHED_FIXED_SPLIT)
    plan->slot_cap = 2 * s.grid + s.phys_grid;
  else
    plan->slot_cap = std::max(s.grid, s.phys_grid);

  // ---- device state -------------------------------------------------------------------
  if (!plan->host_only) {
    const int CAP = plan->slot_cap, GP = s.phys_grid;
    const size_t U = s.units.size();
    plan->pt_stride = p.layout == LA_KV_PAGED ? (p.pages_per_seq + 31) / 32 * 32 : 0;
    plan->off_units = 256;
    plan->off_begin = plan->off_units + align256(U * sizeof(DevUnit));
    plan->off_first = plan->off_begin + align256(size_t(CAP + 1) * sizeof(int32_t));
    plan->off_claim = plan->off_first + align256(size_t(CAP) * sizeof(int32_t));
    plan->off_bt = plan->off_claim + align256(size_t(CAP + GP) * sizeof(int32_t));
    plan->up_bytes = plan->off_bt + align256(size_t(p.batch) * plan->pt_stride * sizeof(int32_t));
    const size_t b_po = align256(size_t(CAP) * 2 * p.rows() * head_dim * sizeof(float));
    const size_t b_pml = align256(size_t(CAP) * 2 * p.rows() * 4 * sizeof(float));
    const size_t b_flags = align256(size_t(CAP) * sizeof(uint32_t));
    const size_t b_cnt = align256((la::kNumCounters + U) * sizeof(int));
    const size_t b_trace = opts.trace ? align256(size_t(GP) * LA_TRACE_FIELDS * sizeof(uint64_t)) : 0;
    const size_t b_gf = align256(size_t(GP) * plan->kinfo.global_fold_floats * sizeof(float));
    const size_t o_po = plan->up_bytes, o_pml = o_po + b_po, o_flags = o_pml + b_pml, o_cnt = o_flags + b_flags;
    const size_t o_trace = o_cnt + b_cnt, o_gf = o_trace + b_trace, bytes = o_gf + b_gf;
    cudaError_t e = cudaMalloc(&plan->d_tables, bytes);
    if (e != cudaSuccess) { delete plan; return cuda_fail(e, "cudaMalloc(plan tables)"); }
    e = cudaMallocHost(&plan->h_stage, plan->up_bytes);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&plan->up_done, cudaEventDisableTiming);
    if (e != cudaSuccess) {
      release_device(plan);
      delete plan;
      return cuda_fail(e, "plan staging");
    }
    std::memset(plan->h_stage, 0, plan->up_bytes);
    char* base = static_cast<char*>(plan->d_tables);
    plan->d_hdr = reinterpret_cast<int32_t*>(base);
    plan->d_units = reinterpret_cast<DevUnit*>(base + plan->off_units);
    plan->d_cta_begin = reinterpret_cast<int32_t*>(base + plan->off_begin);
    plan->d_cta_first = reinterpret_cast<int32_t*>(base + plan->off_first);
    plan->d_claim = reinterpret_cast<int32_t*>(base + plan->off_claim);
    plan->d_block_table = plan->pt_stride ? reinterpret_cast<int32_t*>(base + plan->off_bt) : nullptr;
    plan->d_part_o = reinterpret_cast<float*>(base + o_po);
    plan->d_part_ml = reinterpret_cast<float*>(base + o_pml);
    plan->d_flags = reinterpret_cast<uint32_t*>(base + o_flags);
    plan->d_counters = reinterpret_cast<int*>(base + o_cnt);
    plan->d_unit_count = plan->d_counters + la::kNumCounters;
    if (opts.trace) plan->d_trace = reinterpret_cast<unsigned long long*>(base + o_trace);
    if (b_gf) plan->d_gfold = reinterpret_cast<float*>(base + o_gf);
    plan->workspace = int64_t(bytes);
    // kernel state (flags, counters, trace) starts at zero; then the tables, one async copy
    cudaStream_t st = static_cast<cudaStream_t>(opts.stream);
    e = cudaMemsetAsync(base + o_flags, 0, o_gf - o_flags, st);
    if (e != cudaSuccess) {
      release_device(plan);
      delete plan;
      return cuda_fail(e, "plan state init");
    }
    la_status us = upload_tables(plan, st, /*sync=*/opts.stream == nullptr);
    if (us != LA_OK) {
      release_device(plan);
      delete plan;
      return us;
    }
    if (plan->xw) {
      const size_t xb = xchg_bytes(p, plan->xw);
      plan->xflag_off = xchg_flag_off(p, plan->xw);
      e = cudaMalloc(&plan->d_xchg, xb);
      if (e == cudaSuccess) e = cudaMemset(plan->d_xchg, 0, xb);
      int32_t hdr[kXchgHdrInts];
      xchg_header(plan, hdr);
      if (e == cudaSuccess) e = cudaMemcpy(static_cast<char*>(plan->d_xchg) + 64, hdr, sizeof(hdr),
                                           cudaMemcpyHostToDevice);
      if (e != cudaSuccess) {
        release_device(plan);
        delete plan;
        return cuda_fail(e, "exchange buffer");
      }
      plan->xpeer[plan->xr] = static_cast<float*>(plan->d_xchg);
      plan->workspace += int64_t(xb);
    }
  }
  *out = plan;
  return LA_OK;
}

la_status la_plan_update(la_plan_t plan, const int32_t* ctx_lens, const int32_t* block_table, void* stream) {
  if (!plan || !ctx_lens) return fail(LA_ERR_INVALID, "NULL argument");
  la::Problem& p = plan->prob;
  if (block_table && p.layout != LA_KV_PAGED) return fail(LA_ERR_INVALID, "block_table given for a non-paged plan");
  int64_t maxn = 0;
  la_status st = check_lens(p, ctx_lens, &maxn);
  if (st != LA_OK) return st;
  if (p.layout == LA_KV_BHSD && maxn > p.max_ctx)
    return fail(LA_ERR_INVALID, "ctx_lens exceed the plan's max_ctx (the BHSD slab stride)");
  if (p.layout == LA_KV_PAGED && maxn > int64_t(p.pages_per_seq) * p.page_size)
    return fail(LA_ERR_INVALID, "ctx_lens exceed pages_per_seq * page_size");
  la::Problem np = p;
  np.ctx_lens.assign(ctx_lens, ctx_lens + p.batch);
  if (block_table) np.block_table.assign(block_table, block_table + size_t(p.batch) * p.pages_per_seq);
  if (p.layout == LA_KV_PAGED) {
    st = check_block_table(np, np.block_table.data());
    if (st != LA_OK) return st;
  }
  if (!plan->host_only && p.layout == LA_KV_PACKED && plan->kinfo.uses_tma_tensor && np.kv_rows() >= (int64_t(1) << 31))
    return fail(LA_ERR_UNSUPPORTED, "KV cache rows exceed the TMA int32 coordinate range");
  const la::Problem old_p = p;
  const la::Schedule old_s = plan->sched;
  const int old_split = plan->split;
  p = np;
  st = plan_schedule(plan, false, 0);
  if (st == LA_OK && !plan->host_only && plan->sched.grid > plan->slot_cap)
    st = fail(LA_ERR_STATE, "the new schedule has more (virtual) CTA ranges than the plan allocated: re-plan");
  if (st == LA_OK && !plan->host_only) st = upload_tables(plan, static_cast<cudaStream_t>(stream), false);
  if (st != LA_OK) {  // the plan is left as it was
    p = old_p;
    plan->sched = old_s;
    plan->split = old_split;
    return st;
  }
  ++plan->updates;
  return LA_OK;
}

la_status la_plan_set_weights(la_plan_t plan, const int32_t* weights, int n, void* stream) {
  if (!plan) return fail(LA_ERR_INVALID, "plan is NULL");
  if (plan->prob.schedule != LA_SCHED_STREAMK) return fail(LA_ERR_STATE, "weights apply to LA_SCHED_STREAMK plans");
  if (weights) {
    if (n != plan->sched.phys_grid) return fail(LA_ERR_INVALID, "n must equal la_plan_info.grid");
    for (int g = 0; g < n; ++g)
      if (weights[g] < 1 || weights[g] > (1 << 20)) return fail(LA_ERR_INVALID, "weights must be in [1, 2^20]");
  }
  std::vector<int32_t> old_w = plan->weights;
  const la::Schedule old_s = plan->sched;
  if (weights)
    plan->weights.assign(weights, weights + n);
  else
    plan->weights.clear();
  la_status st = plan_schedule(plan, false, 0);
  if (st == LA_OK && !plan->host_only) st = upload_tables(plan, static_cast<cudaStream_t>(stream), false);
  if (st != LA_OK) {
    plan->weights = old_w;
    plan->sched = old_s;
  }
  return st;
}

static la_status decode_impl(la_plan_t plan, const void* q, const void* k, const void* v, float* out,
                             float* lse, void* stream, bool xchg = true);

la_status la_plan_calibrate(la_plan_t plan, const void* q, const void* k_cache, const void* v_cache, float* out,
                            float* lse, int launches, int rounds, void* stream) {
  if (!plan) return fail(LA_ERR_INVALID, "plan is NULL");
  if (plan->host_only) return fail(LA_ERR_STATE, "host-only plan cannot decode");
  if (plan->prob.schedule != LA_SCHED_STREAMK) return fail(LA_ERR_STATE, "calibration applies to LA_SCHED_STREAMK plans");
  if (launches < 1 || rounds < 1) return fail(LA_ERR_INVALID, "launches and rounds must be >= 1");
  if (plan->xw > 1)  // its launches would wait for the peers' exchange launches
    return fail(LA_ERR_STATE, "la_plan_calibrate on a cross-GPU exchange plan: use la_plan_set_weights");
  const int GP = plan->sched.phys_grid;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  unsigned long long* own_trace = plan->d_trace;
  unsigned long long* tmp = nullptr;
  if (!own_trace) {
    cudaError_t e = cudaMalloc(&tmp, size_t(GP) * LA_TRACE_FIELDS * sizeof(uint64_t));
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(calibration trace)");
    plan->d_trace = tmp;
  }
  std::vector<int32_t> w = plan->weights.empty() ? std::vector<int32_t>(size_t(GP), 1 << 16) : plan->weights;
  std::vector<uint64_t> tr(size_t(GP) * LA_TRACE_FIELDS);
  la_status rs = LA_OK;
  for (int r = 0; r < rounds && rs == LA_OK; ++r) {
    rs = la_plan_set_weights(plan, w.data(), GP, stream);
    std::vector<double> t(size_t(GP), 0.0);
    for (int i = 0; i <= launches && rs == LA_OK; ++i) {  // sample 0 warms the new tables up
      // each sample: kSteady launches back to back, the trace is the last one's -- a launch
      // that starts on an idle GPU (after a host sync) streams differently from the steady
      // state a decode loop runs in
      constexpr int kSteady = 3;
      for (int j = 0; j < kSteady && rs == LA_OK; ++j) rs = decode_impl(plan, q, k_cache, v_cache, out, lse, stream);
      if (rs != LA_OK) break;
      cudaError_t e = cudaStreamSynchronize(st);
      if (e == cudaSuccess)
        e = cudaMemcpy(tr.data(), plan->d_trace, tr.size() * sizeof(uint64_t), cudaMemcpyDeviceToHost);
      if (e != cudaSuccess) { rs = cuda_fail(e, "la_plan_calibrate"); break; }
      if (i == 0) continue;
      for (int g = 0; g < GP; ++g) {
        const uint64_t* x = &tr[size_t(g) * LA_TRACE_FIELDS];
        if (x[6] > x[1]) t[size_t(g)] += double(x[6] - x[1]);
      }
    }
    if (rs != LA_OK) break;
    // rate-proportional shares: w_g <- w_g * mean(t) / t_g over the CTAs that streamed
    const la::Schedule& s = plan->sched;
    double tsum = 0.0;
    int cnt = 0;
    for (int g = 0; g < s.grid; ++g)
      if (s.cta_begin[g + 1] > s.cta_begin[g] && t[size_t(g)] > 0.0) {
        tsum += t[size_t(g)];
        ++cnt;
      }
    if (cnt == 0) break;
    const double tm = tsum / cnt;
    for (int g = 0; g < s.grid; ++g)
      if (s.cta_begin[g + 1] > s.cta_begin[g] && t[size_t(g)] > 0.0) {
        const double nw = std::round(double(w[size_t(g)]) * tm / t[size_t(g)]);
        w[size_t(g)] = int32_t(std::min(double(1 << 20), std::max(1.0, nw)));
      }
  }
  if (rs == LA_OK) rs = la_plan_set_weights(plan, w.data(), GP, stream);
  if (rs == LA_OK) {
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) rs = cuda_fail(e, "la_plan_calibrate");
  }
  if (tmp) {
    plan->d_trace = own_trace;
    cudaFree(tmp);
  }
  return rs;
}

la_status la_plan_info_get(la_plan_t plan, la_plan_info* info) {
  if (!plan || !info) return fail(LA_ERR_INVALID, "NULL argument");
  const la::Problem& p = plan->prob;
  const la::Schedule& s = plan->sched;
  std::memset(info, 0, sizeof(*info));
  info->batch = p.batch;
  info->heads_q = p.heads_q;
  info->heads_kv = p.heads_kv;
  info->head_dim = p.head_dim;
  info->group = p.group;
  info->dtype = p.dtype;
  info->layout = p.layout;
  info->schedule = p.schedule;
  info->tile_n = s.tile_n;
  info->stage_tokens = plan->stage_tokens;
  info->grid = s.phys_grid;
  info->num_vctas = s.grid;
  info->split = plan->split;
  info->q_len = p.q_len;
  info->tile_rows = p.tile_rows;
  info->engine = plan->engine;
  info->q_rows = p.q_rows();
  info->quantization_efficiency = quant_eff(plan);
  info->slot_capacity = plan->slot_cap;
  info->updates = plan->updates;
  info->sm_weighted = plan->weights.empty() ? 0 : 1;
  info->num_units = int(s.units.size());
  info->total_iters = s.total_iters;
  info->num_segments = s.num_segments;
  info->num_partials = s.num_partials;
  info->workspace_bytes = plan->workspace;
  int64_t tokens = 0;
  for (int32_t n : p.ctx_lens) tokens += n;
  info->kv_bytes = 2 * int64_t(p.heads_kv) * tokens * p.head_dim * p.elem_bytes();
  info->scale = p.scale;
  return LA_OK;
}

la_status la_plan_export_claims(la_plan_t plan, int32_t* claims, size_t cap, size_t* n) {
  if (!plan || !n) return fail(LA_ERR_INVALID, "NULL argument");
  const std::vector<int32_t>& c = plan->sched.claim;
  *n = c.size();
  if (cap == 0) return LA_OK;
  if (!claims || cap < c.size()) return fail(LA_ERR_INVALID, "claims buffer too small");
  std::memcpy(claims, c.data(), c.size() * sizeof(int32_t));
  return LA_OK;
}

la_status la_plan_export(la_plan_t plan, int32_t* rows, size_t cap_rows, size_t* n_rows) {
  if (!plan || !n_rows) return fail(LA_ERR_INVALID, "NULL argument");
  std::vector<int32_t> r;
  la::export_segments(plan->sched, r);
  *n_rows = r.size() / 7;
  if (cap_rows == 0) return LA_OK;
  if (!rows || cap_rows < *n_rows) return fail(LA_ERR_INVALID, "rows buffer too small");
  std::memcpy(rows, r.data(), r.size() * sizeof(int32_t));
  return LA_OK;
}

static la_status decode_impl(la_plan_t plan, const void* q, const void* k, const void* v, float* out,
                             float* lse, void* stream, bool xchg) {
  if (!plan) return fail(LA_ERR_INVALID, "plan is NULL");
  if (plan->host_only) return fail(LA_ERR_STATE, "host-only plan cannot decode");
  if (!q || !k || !v || !out) return fail(LA_ERR_INVALID, "NULL tensor pointer");
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(out))
    return fail(LA_ERR_INVALID, "tensor pointers must be 16-byte aligned");
  la::DecodeArgs a{};
  a.q = q;
  a.k = k;
  a.v = v;
  a.out = out;
  a.lse = lse;
  a.units = plan->d_units;
  a.cta_begin = plan->d_cta_begin;
  a.cta_first_unit = plan->d_cta_first;
  a.claim = plan->d_claim;
  a.part_o = plan->d_part_o;
  a.part_ml = plan->d_part_ml;
  a.flags = plan->d_flags;
  a.trace = plan->d_trace;
  a.gfold = plan->d_gfold;
  a.counters = plan->d_counters;
  a.unit_count = plan->d_unit_count;
  a.slot_stride = plan->slot_cap;
  a.dynamic = (plan->prob.schedule == LA_SCHED_DYNAMIC || plan->prob.schedule == LA_SCHED_FIXED_SPLIT) ? 1 : 0;
  a.paged = plan->prob.layout == LA_KV_PAGED ? 1 : 0;
  a.block_table = plan->d_block_table;
  a.pt_stride = plan->pt_stride;
  a.heads_kv = plan->prob.heads_kv;
  a.page_shift = 0;
  while (a.paged && (1 << a.page_shift) < plan->prob.page_size) ++a.page_shift;
  const int box = plan->kinfo.stage_tokens_max;  // GQA / FP8 TMA box height = a full stage
  a.box_rows = a.paged ? std::min(box, plan->prob.page_size) : box;
  a.box_shift = 0;
  while ((1 << a.box_shift) < a.box_rows) ++a.box_shift;
  a.grid = plan->sched.phys_grid;
  a.tile_n = plan->sched.tile_n;
  a.stage_tokens = plan->stage_tokens;
  a.group = plan->prob.rows();
  a.q_len = plan->prob.q_len;
  a.causal = plan->prob.causal;
  a.scale_log2 = float(double(plan->prob.scale) * double(plan->prob.k_scale) * 1.4426950408889634);
  a.out_scale = plan->prob.v_scale;
  if (plan->xw && xchg) {
    for (int r = 0; r < plan->xw; ++r)
      if (!plan->xpeer[r]) return fail(LA_ERR_STATE, "exchange peer " + std::to_string(r) + " not opened/attached");
    a.xw = plan->xw;
    a.xr = plan->xr;
    a.xrows = int(plan->prob.q_rows());
    a.xunits = int(plan->sched.units.size());
    a.xflag_off = plan->xflag_off;
    for (int r = 0; r < plan->xw; ++r) a.xpeer[r] = reinterpret_cast<float*>(reinterpret_cast<char*>(plan->xpeer[r]) + kXchgHead);
    a.xerr = static_cast<int*>(plan->d_xchg);
  }
  std::string err;
  const la::Problem& p = plan->prob;
  // stream-K hosts may wait on peers (Alg2§28): co-residency by a cooperative launch (the launch
  // grid never exceeds the co-resident count; measured no cost vs a plain launch)
  const bool coop = p.schedule == LA_SCHED_STREAMK;

  const int rc = la::launch_decode(plan->kinfo, a, p.kv_rows(), p.head_dim, p.dtype, coop, stream, &plan->tmaps, err);
  if (rc != 0) return fail(LA_ERR_CUDA, err);
  return LA_OK;
}

la_status la_decode(la_plan_t plan, const void* q, const void* k_cache, const void* v_cache, float* out,
                    float* lse, void* stream) {
  return decode_impl(plan, q, k_cache, v_cache, out, lse, stream, true);
}

la_status la_decode_partial(la_plan_t plan, const void* q, const void* k_shard, const void* v_shard,
                            float* o_part, float* lse_part, void* stream) {
  if (!lse_part) return fail(LA_ERR_INVALID, "la_decode_partial needs lse_part");
  return decode_impl(plan, q, k_shard, v_shard, o_part, lse_part, stream, /*xchg=*/false);
}

la_status la_combine_strided(const float* o_parts, int64_t o_part_stride, const float* lse_parts,
                             int64_t lse_part_stride, int parts, int rows, int head_dim, float* out, float* lse,
                             void* stream) {
  if (!o_parts || !lse_parts || !out) return fail(LA_ERR_INVALID, "NULL tensor pointer");
  if (parts < 1 || rows < 1) return fail(LA_ERR_INVALID, "parts and rows must be >= 1");
  if (head_dim != 64 && head_dim != 128) return fail(LA_ERR_UNSUPPORTED, "head_dim must be 64 or 128");
  if (o_part_stride < int64_t(rows) * head_dim || lse_part_stride < rows)
    return fail(LA_ERR_INVALID, "part strides smaller than one part");
  std::string err;
  if (la::launch_combine(o_parts, size_t(o_part_stride), lse_parts, size_t(lse_part_stride), parts, rows, head_dim,
                         out, lse, stream, err) != 0)
    return fail(LA_ERR_CUDA, err);
  return LA_OK;
}

la_status la_combine(const float* o_parts, const float* lse_parts, int parts, int rows, int head_dim,
                     float* out, float* lse, void* stream) {
  return la_combine_strided(o_parts, int64_t(rows) * head_dim, lse_parts, rows, parts, rows, head_dim, out, lse,
                            stream);
}

la_status la_decode_host(la_plan_t plan, const void* q, const void* k_cache, const void* v_cache,
                         int64_t kv_rows, float* out, float* lse, void* stream) {
  if (!plan) return fail(LA_ERR_INVALID, "plan is NULL");
  if (plan->host_only) return fail(LA_ERR_STATE, "host-only plan cannot decode");
  if (!q || !k_cache || !v_cache || !out) return fail(LA_ERR_INVALID, "NULL host pointer");
  const la::Problem& p = plan->prob;
  if (kv_rows != p.kv_rows()) return fail(LA_ERR_INVALID, "kv_rows does not match the plan");
  const size_t eb = size_t(p.elem_bytes());
  const size_t q_bytes = size_t(p.q_rows()) * p.head_dim * p.q_elem_bytes();
  const size_t kv_bytes = size_t(kv_rows) * p.head_dim * eb;
  const size_t o_bytes = size_t(p.q_rows()) * p.head_dim * sizeof(float);
  const size_t l_bytes = size_t(p.q_rows()) * sizeof(float);
  auto align = [](size_t x) { return (x + 255) & ~size_t(255); };
  const size_t need = align(q_bytes) + 2 * align(kv_bytes) + align(o_bytes) + align(l_bytes);
  if (plan->stage_bytes < need) {
    if (plan->d_stage) cudaFree(plan->d_stage);
    plan->d_stage = nullptr;
    plan->stage_bytes = 0;
    cudaError_t e = cudaMalloc(&plan->d_stage, need);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(staging)");
    plan->stage_bytes = need;
  }
  char* base = static_cast<char*>(plan->d_stage);
  void* dq = base;
  void* dk = base + align(q_bytes);
  void* dv = base + align(q_bytes) + align(kv_bytes);
  float* dout = reinterpret_cast<float*>(base + align(q_bytes) + 2 * align(kv_bytes));
  float* dlse = reinterpret_cast<float*>(base + align(q_bytes) + 2 * align(kv_bytes) + align(o_bytes));
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaMemcpyAsync(dq, q, q_bytes, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dk, k_cache, kv_bytes, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dv, v_cache, kv_bytes, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return cuda_fail(e, "H2D");
  la_status s = decode_impl(plan, dq, dk, dv, dout, lse ? dlse : nullptr, stream, true);
  if (s != LA_OK) return s;
  e = cudaMemcpyAsync(out, dout, o_bytes, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess && lse) e = cudaMemcpyAsync(lse, dlse, l_bytes, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "D2H/sync");
  return LA_OK;
}

la_status la_plan_trace(la_plan_t plan, uint64_t* out, size_t cap_ctas, size_t* n_ctas) {
  if (!plan || !n_ctas) return fail(LA_ERR_INVALID, "NULL argument");
  if (!plan->d_trace) return fail(LA_ERR_STATE, "plan was created without opts.trace");
  const size_t G = size_t(plan->sched.phys_grid);
  *n_ctas = G;
  if (cap_ctas == 0) return LA_OK;
  if (!out || cap_ctas < G) return fail(LA_ERR_INVALID, "trace buffer too small");
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess)
    e = cudaMemcpy(out, plan->d_trace, G * LA_TRACE_FIELDS * sizeof(uint64_t), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(e, "la_plan_trace");
  return LA_OK;
}

la_status la_plan_xchg_handle(la_plan_t plan, void* handle) {
  if (!plan || !handle) return fail(LA_ERR_INVALID, "NULL argument");
  if (!plan->d_xchg) return fail(LA_ERR_STATE, "plan has no exchange buffer (xchg_world <= 1 or host-only)");
  static_assert(sizeof(cudaIpcMemHandle_t) == LA_XCHG_HANDLE_BYTES, "IPC handle size");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, plan->d_xchg);
  if (e != cudaSuccess) return cuda_fail(e, "cudaIpcGetMemHandle");
  std::memcpy(handle, &h, sizeof(h));
  return LA_OK;
}

la_status la_plan_xchg_open(la_plan_t plan, int peer, const void* handle) {
  if (!plan || !handle) return fail(LA_ERR_INVALID, "NULL argument");
  if (!plan->d_xchg) return fail(LA_ERR_STATE, "plan has no exchange buffer");
  if (peer < 0 || peer >= plan->xw || peer == plan->xr) return fail(LA_ERR_INVALID, "bad peer rank");
  if (plan->xpeer[peer]) return fail(LA_ERR_STATE, "peer already opened/attached");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  void* ptr = nullptr;
  cudaError_t e = cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return cuda_fail(e, "cudaIpcOpenMemHandle");
  // the peer's shape header (written at its la_plan) must describe the same problem
  int32_t mine[kXchgHdrInts], theirs[kXchgHdrInts];
  xchg_header(plan, mine);
  e = cudaMemcpy(theirs, static_cast<char*>(ptr) + 64, sizeof(theirs), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) {
    cudaIpcCloseMemHandle(ptr);
    return cuda_fail(e, "reading the peer's exchange header");
  }
  mine[9] = peer;  // the peer's rank
  if (std::memcmp(mine, theirs, sizeof(mine)) != 0) {
    cudaIpcCloseMemHandle(ptr);
    return fail(LA_ERR_INVALID, "peer plan has another shape, world or rank (exchange header mismatch)");
  }
  plan->xpeer[peer] = static_cast<float*>(ptr);
  plan->xpeer_ipc[peer] = true;
  return LA_OK;
}

la_status la_plan_xchg_attach(la_plan_t plan, int peer, la_plan_t peer_plan) {
  if (!plan || !peer_plan) return fail(LA_ERR_INVALID, "NULL argument");
  if (!plan->d_xchg || !peer_plan->d_xchg) return fail(LA_ERR_STATE, "plan has no exchange buffer");
  if (peer < 0 || peer >= plan->xw || peer == plan->xr) return fail(LA_ERR_INVALID, "bad peer rank");
  if (peer_plan->xw != plan->xw || peer_plan->xr != peer) return fail(LA_ERR_INVALID, "peer plan has another rank/world");
  const la::Problem &p = plan->prob, &q = peer_plan->prob;
  if (p.batch != q.batch || p.heads_q != q.heads_q || p.heads_kv != q.heads_kv || p.head_dim != q.head_dim ||
      p.q_lens != q.q_lens)
    return fail(LA_ERR_INVALID, "peer plan has another shape");
  if (plan->xpeer[peer]) return fail(LA_ERR_STATE, "peer already opened/attached");
  plan->xpeer[peer] = static_cast<float*>(peer_plan->d_xchg);
  return LA_OK;
}

la_status la_plan_status(la_plan_t plan) {
  if (!plan) return fail(LA_ERR_INVALID, "plan is NULL");
  if (plan->host_only) return fail(LA_ERR_STATE, "host-only plan");
  int err = 0, xerr = 0;
  cudaError_t e = cudaDeviceSynchronize();
  int* d_err = plan->d_counters + la::CTR_ERROR;
  int* d_xerr = plan->d_xchg ? static_cast<int*>(plan->d_xchg) : nullptr;
  if (e == cudaSuccess) e = cudaMemcpy(&err, d_err, sizeof(int), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && d_xerr) e = cudaMemcpy(&xerr, d_xerr, sizeof(int), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && err) e = cudaMemset(d_err, 0, sizeof(int));
  if (e == cudaSuccess && xerr) e = cudaMemset(d_xerr, 0, sizeof(int));
  if (e != cudaSuccess) return cuda_fail(e, "la_plan_status");
  if (xerr) return fail(LA_ERR_TIMEOUT, "a cross-GPU exchange wait timed out (a peer rank never arrived)");
  if (err) return fail(LA_ERR_TIMEOUT, "a host CTA's wait for a peer partial timed out (Alg2 Wait, reading C17)");
  return LA_OK;
}

la_status la_plan_xchg_status(la_plan_t plan) {
  if (!plan) return fail(LA_ERR_INVALID, "plan is NULL");
  if (!plan->d_xchg) return fail(LA_ERR_STATE, "plan has no exchange buffer");
  return la_plan_status(plan);
}

void la_plan_destroy(la_plan_t plan) {
  if (!plan) return;
  release_device(plan);
  delete plan;
}

}  // extern "C"
