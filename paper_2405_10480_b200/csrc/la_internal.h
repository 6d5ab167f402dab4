// Internal declarations shared by the planner, the C-ABI layer and the kernels.
// Nothing here is visible through include/la.h.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "la.h"

namespace la {

// A work unit = one output tile: (request b, KV head h_kv, query tile m).  Its rows are
// r0 .. r0 + rows - 1 of the g * N_b rows of (b, h_kv), row r = q-head j * N_b + query i
// (Alg2§4's C_m query tiles of T_m rows; C_m = 1 whenever g * N_b <= T_m).  48 bytes,
// uploaded as-is to the device.
struct DevUnit {
  int64_t row0;        // first K/V row of the unit (a row = head_dim elements)
  int32_t len;         // n_b
  int32_t iter_begin;  // tile_iter of Alg2§12: global index of the unit's first LeanTile
  int32_t iter_end;    // tile_iter_end of Alg2§13
  int32_t q_row;       // first query/output row of the unit (rows are contiguous)
  int32_t last_cta;    // owner(iter_end - 1): reading C9 of Alg2§26
  int32_t host_cta;    // owner(iter_begin): the host block of P:412 / Alg2§17
  int32_t rows;        // output rows of this unit (<= T_m)
  int32_t r0;          // index of its first row among the g * N_b rows of (b, h_kv)
  int32_t nq;          // N_b: query tokens of request b
  int32_t pad_;
};
static_assert(sizeof(DevUnit) == 48, "DevUnit layout");

// Host-side schedule: Alg2§4-18 for every (virtual) CTA.  Pure integer work, no CUDA.
struct Schedule {
  int tile_n = 0;
  int grid = 0;         // (virtual) CTAs = ranges of the iteration space (Alg. 2's G)
  int phys_grid = 0;    // CTAs launched (= grid for static schedules)
  int64_t total_iters = 0;
  std::vector<DevUnit> units;
  std::vector<int32_t> cta_begin;       // grid + 1 entries: CTA v owns [cta_begin[v], cta_begin[v+1])
  std::vector<int32_t> cta_first_unit;  // grid entries: unit containing cta_begin[v]
  std::vector<int32_t> claim;           // grid entries: the v taken by the c-th dynamic claim
  int64_t num_segments = 0;
  int64_t num_partials = 0;
};

struct Problem {
  int batch = 0, heads_q = 0, heads_kv = 0, head_dim = 0, group = 0;
  int q_len = 1, causal = 1;   // uniform N_q (0 if per-request q_lens differ) and the mask (NEXT-3)
  std::vector<int32_t> q_lens; // N_b per request
  int tile_rows = 1;           // T_m: output rows per unit (1: MHA engine; else <= 8)
  int rows() const { return tile_rows; }
  int64_t num_units() const {  // sum_b H_kv * C_m(b), C_m(b) = ceil(g N_b / T_m)
    int64_t u = 0;
    for (int32_t n : q_lens) u += int64_t(heads_kv) * ((int64_t(group) * n + tile_rows - 1) / tile_rows);
    return u;
  }
  int64_t q_rows() const {     // query/output rows: sum_b H_q * N_b
    int64_t r = 0;
    for (int32_t n : q_lens) r += int64_t(heads_q) * n;
    return r;
  }
  int dtype = LA_BF16, layout = LA_KV_BHSD, schedule = LA_SCHED_STREAMK;
  int64_t max_ctx = 0;
  float scale = 0.f;
  std::vector<int32_t> ctx_lens;
  // LA_KV_PAGED
  int page_size = 0, pages_per_seq = 0;
  int64_t num_pages = 0;
  std::vector<int32_t> block_table;  // [batch][pages_per_seq]
  int64_t kv_rows() const;   // rows of one K (or V) cache in its layout
  float k_scale = 1.f, v_scale = 1.f;  // LA_FP8_E4M3: K = codes x k_scale, V = codes x v_scale
  int elem_bytes() const { return dtype == LA_FP32 ? 4 : (dtype == LA_FP8_E4M3 ? 1 : 2); }  // K/V
  int q_elem_bytes() const { return dtype == LA_FP32 ? 4 : 2; }  // Q (bf16 with FP8 KV)
};

// Build units in memory order (reading C14) with their row bases and C_n = ceil(n/T_n).
void build_units(const Problem& p, int tile_n, std::vector<DevUnit>& units, int64_t& total_iters);
// Eq. 2 / Alg2§7-9 with the remainder rule (reading C8); grid >= 1.
void streamk_ranges(int64_t total_iters, int grid, std::vector<int32_t>& cta_begin);
// SM-rate-weighted Eq. 2 (la_plan_set_weights): cta_begin[g] = min(g, I) + floor((I - G)+ *
// sum_{i<g} w_i / sum w), w_i in [1, 2^20] (oracle.weighted_ranges).
void weighted_ranges(int64_t total_iters, const std::vector<int32_t>& w, std::vector<int32_t>& cta_begin);
// Sequential (FA2): one CTA per unit.
void sequential_ranges(const std::vector<DevUnit>& units, std::vector<int32_t>& cta_begin);
// LA_SCHED_DYNAMIC: every Eq. 2 range split into a head and k <= max_chunks tail chunks of
// s LeanTiles (oracle.balanced_ranges); `claim` = heads in range order, then tail chunks
// round by round over the ranges.
void balanced_ranges(int64_t total_iters, int grid, int head_permille, int min_chunk, int max_chunks,
                     std::vector<int32_t>& cta_begin, std::vector<int32_t>& claim);
// FlashDecoding's fixed split: unit u cut into min(split, C_n(u)) chunks, the
// first (C_n mod s) one LeanTile longer; ranges in unit order.
void fixed_split_ranges(const std::vector<DevUnit>& units, int split, std::vector<int32_t>& cta_begin);
// FlashAttention-2's split heuristic: 1 if units fill 80% of the SMs, else the smallest s
// whose wave efficiency units*s / (ceil(units*s/sms)*sms) is >= 85% of the best s <= 128.
int fa2_num_splits(int64_t units, int64_t max_cn, int sms);
// host_cta / last_cta per unit, first unit per CTA, segment & partial counts.
void finish_schedule(Schedule& s);
// Segment rows (7 int32 each, SPEC S:275 order) by the Alg2§10-18,§41 walk.
void export_segments(const Schedule& s, std::vector<int32_t>& rows);

// ---- device side (decode.cu) --------------------------------------------------------
struct DecodeArgs {
  const void* q;
  const void* k;
  const void* v;
  float* out;
  float* lse;
  // Schedule tables (device; rewritten by la_plan_update, so nothing that depends on ctx_lens
  // is passed by value -- a CUDA graph captured on the plan replays across updates; padded
  // to the plan's capacity so the kernel needs no range count):
  const DevUnit* units;
  const int32_t* cta_begin;       // [cap + 1]: ranges past the schedule's are empty [I, I)
  const int32_t* cta_first_unit;  // [cap]
  const int32_t* claim;           // [cap + grid] dynamic: claim c runs virtual CTA claim[c] (-1: no more)
  float* part_o;      // [2][slot_stride][group][d]  Op of Alg2§20 (slot 1: host partials that wait
                      //                              or are folded by the dynamic tree)
  float* part_ml;     // [2][slot_stride][group][4]  mp, lp, -, - of Alg2§21-22 (m in log2 units)
  uint32_t* flags;    // [slot_stride]               flags of Alg2§23/§28, epoch-valued (reading C17)
  int* counters;      // [kNumCounters] see CTR_* (device-side: a captured CUDA graph replays correctly)
  int* unit_count;    // [units] dynamic mode: segments of the unit published so far (the last
                      //   arriver folds them all; one counter per unit, reset by that arriver)
  int slot_stride;    // capacity of (virtual) CTAs: partial slot 1 of CTA v is slot_stride + v
  unsigned long long* trace;  // [phys_grid][LA_TRACE_FIELDS] or nullptr
  float* gfold;       // [phys_grid][KernelInfo::global_fold_floats] or nullptr
  int dynamic;        // 1: claim virtual CTAs dynamically, last-arriver fold
  int grid;           // CTAs launched (fixed for the plan's life)
  int tile_n;
  int stage_tokens;
  int group;          // T_m: rows of a partial slot (a unit's own row count is DevUnit::rows)
  int q_len;          // N_q (unused by the kernels: per-unit DevUnit::nq)
  int causal;         // N_q > 1: query i attends to unit-local keys [0, n - N_q + i]
  int uses_tmap;      // set by launch_decode for the TMA-tensor (GQA) engine
  float scale_log2;   // scale * log2(e) (* k_scale for FP8 KV): scores live in the exp2 domain
  float out_scale;    // finalize multiplies O by this: v_scale for FP8 KV, else 1
  // LA_KV_PAGED: DevUnit.row0 holds b * heads_kv + h; token t of the unit is row
  // (block_table[b * pt_stride + (t >> page_shift)] * heads_kv + h) * page + (t & (page - 1))
  const int32_t* block_table;
  int paged;
  int page_shift;
  int pt_stride;      // padded to a multiple of 32 entries (the producer reads 32-entry windows)
  int heads_kv;
  int box_rows;       // GQA TMA box height: min(64, page_size) when paged, else 64
  int box_shift;      // log2(box_rows)
  // NEXT-2 fused cross-GPU exchange (xw > 1).  Every rank's buffer holds
  // [2 launch parity][xw source ranks][xrows][d + 4] fp32 (normalised O_r, then L_r in log2
  // units) followed, at byte offset xflag_off, by [xw source ranks][xunits] uint32 flags.
  int xw;             // ranks P (0/1: off)
  int xr;             // this rank
  int xrows;          // output rows B * H_q * N_q
  int xunits;         // units B * H_kv
  size_t xflag_off;
  float* xpeer[8];    // every rank's buffer (xpeer[xr] = own), device-accessible addresses
  int* xerr;          // own buffer's error word: 1 after a wait timed out
  int win;            // > 0: at most this many ring stages in flight (else the engine's default)
};

// DecodeArgs::counters
enum {
  CTR_CLAIM = 0,   // dynamic: next virtual CTA to claim
  CTR_DONE = 1,    // dynamic: CTAs done (the last resets CTR_CLAIM)
  CTR_EXITED = 2,  // CTAs exited (the last one advances CTR_EPOCH / CTR_XEPOCH)
  CTR_EPOCH = 3,   // launch epoch: value of this launch's Signal flags (reading C17)
  CTR_XEPOCH = 4,  // cross-GPU exchange sequence: advanced only by exchange launches
  CTR_ERROR = 5,   // 1: an intra-GPU host wait (Alg2§28) gave up after kWaitTimeoutNs
  kNumCounters = 8
};
constexpr unsigned long long kWaitTimeoutNs = 10000000000ull;  // 10 s: intra-GPU host waits
constexpr unsigned long long kXchgTimeoutNs = 5000000000ull;   // 5 s: cross-GPU exchange waits

constexpr int kMaxXchgWorld = 8;
constexpr int kMaxTailChunks = 8;  // LA_SCHED_DYNAMIC: tail chunks per Eq. 2 range (balanced_ranges)

// Kernel configuration for (dtype, head_dim, group): threads, dynamic smem, max stage tokens.
struct KernelInfo {
  bool supported = false;
  int threads = 0;
  int smem_bytes = 0;
  int stage_tokens_max = 0;
  bool uses_tma_tensor = false;   // K/V TMA tensor maps (cached per (k, v, rows) in the plan)
  int box_halves = 2;             // d = 128 bf16/fp16 maps: 128-B row halves per TMA box
  int global_fold_floats = 0;     // > 0: consumer -> epilogue fold buffers live in plan-owned
                                  // global scratch (floats per CTA), not shared memory
  const void* fn = nullptr;
};
KernelInfo decode_kernel_info(int dtype, int head_dim, int group, int engine);
// The plan's encoded K / V tensor maps and the (k, v, rows) they were encoded for.
struct TmapCache {
  const void* k = nullptr;
  const void* v = nullptr;
  int64_t rows = -1;
  alignas(64) unsigned char maps[256];  // CUtensorMap k, v
};
// Launch the decode kernel (cooperative when a static-schedule CTA may wait on a peer).
int launch_decode(const KernelInfo& ki, const DecodeArgs& a, int64_t kv_rows, int head_dim, int dtype,
                  bool cooperative, void* stream, TmapCache* cache, std::string& err);
int launch_combine(const float* o_parts, size_t o_stride, const float* lse_parts, size_t l_stride, int parts,
                   int rows, int head_dim, float* out, float* lse, void* stream, std::string& err);
void note_launch();
int64_t launch_count();

}  // namespace la
