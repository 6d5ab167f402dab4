#pragma once
// sm_100a decode kernel of libleanattn.so: LeanAttention in ONE persistent launch.
// Included by one translation unit per engine family (decode_{mha,gqa,fp8,tc5_*}.cu, built in
// parallel); the host side (tensor maps, launch, the shard combine) is decode.cu.
//
//   la_decode<Engine>   stream-K segment walk (Alg2§10-18, §41) + LeanTile online softmax
//                       (Alg. 1) + in-kernel fixup with the softmax re-scaling operator
//                       (§4.1, Alg2§19-36) + finalize (Alg2§38-39).
//
// Structure of la_decode:
//  * the last warp (one elected lane) is the PRODUCER: it walks the iteration range of each
//    (virtual) CTA it is handed and streams every <= 64-token stage of K and V HBM -> SMEM
//    into an NST-deep ring guarded by full/empty mbarriers (L2 evict-first: KV is read
//    once).  MHA: two 1-D bulk copies (UBLKCP); GQA: TMA tensor loads in the 128-B
//    swizzled layout (UTMALDG).
//  * NCW = NST * WPS CONSUMER warps: WPS warps own each ring slot (fixed ownership keeps a
//    slot's consumers in stage order, so a parity wait cannot alias a completed phase) and
//    split its 32-token rounds.  Each warp keeps its own (m, l, O) -- a §4.1 partial -- and
//    at a segment end hands it to the EPILOGUE warp through one of two fold buffers
//    (mbarrier full/empty) and moves straight on to the next segment.
//  * the EPILOGUE warp folds the NCW warp partials with the re-scaling operator and runs the
//    whole fixup (partial stores, flags / counters, peer folds, finalize) off the consumers'
//    critical path.
//  * the Engine supplies the per-stage math:
//      MhaEngine (group 1, CUDA cores): FHFMA bf16 x bf16 -> fp32 dot products, XOR
//        transpose-butterfly, exp2-domain online softmax, FFMA2 PV.
//      GqaEngine (group 2..8, tensor cores): swap-AB mma.sync m16n8k16 (N = the GQA group),
//        movmatrix.trans from the S^T accumulator to the P^T operand, ldmatrix.trans V^T.
//  * SCHEDULES.  Static (LA_SCHED_STREAMK / SEQUENTIAL): CTA g runs Alg. 2's range g; a
//    non-host segment publishes its partial and a release flag, a non-finishing host spins
//    on its peers' flags and folds them in ascending order (needs co-residency ->
//    cooperative launch).  Dynamic (LA_SCHED_DYNAMIC): the planner cuts every Alg. 2 range
//    into a head and small tail chunks ("virtual CTAs"); persistent CTAs claim all heads,
//    then the chunks (atomic counter + claim table), so fast SMs take more work.  Every
//    non-trivial piece stores its partial and counts itself in; the unit's last arriving
//    piece folds them all in ascending order -- deterministic, and no CTA ever waits.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstring>
#include <string>
#include <type_traits>

#include "la_internal.h"
#include "ptx.cuh"
#include "tc5.cuh"

// Ring / warp configuration (build-time; the defaults are the measured best on B200).
#ifndef LA_MHA_NST
#define LA_MHA_NST 5  // MHA ring stages of 32 KiB
#endif
#ifndef LA_MHA_WPS
#define LA_MHA_WPS 2  // MHA consumer warps per ring slot
#endif
#ifndef LA_GQA_NST
#define LA_GQA_NST 4
#endif
#ifndef LA_GQA_WPS
#define LA_GQA_WPS 2
#endif
#ifndef LA_GQA_FB
#define LA_GQA_FB 2   // GQA consumer -> epilogue fold buffers (33 KB each at NCW = 8)
#endif
#ifndef LA_GQA_SPLITP
#define LA_GQA_SPLITP 1  // P = P_hi + P_lo on the tensor cores (0: single KV-type P)
#endif
#ifndef LA_FP8_NST
#define LA_FP8_NST 5   // FP8 engine (T_m up to 8) ring stages of 32 KiB (128 tokens)
#endif
#ifndef LA_FP8_WPS
#define LA_FP8_WPS 2
#endif
#ifndef LA_FP8_FB
#define LA_FP8_FB 1    // fold buffers: 1 x 41.6 KB (NCW = 10) leaves room for the 5-deep ring
#endif
#ifndef LA_FP8M_NST
#define LA_FP8M_NST 6  // FP8 engine, MHA (T_m = 1): 1-row fold buffers allow a 6-deep ring
#endif
#ifndef LA_FP8M_WPS
#define LA_FP8M_WPS 2
#endif
#ifndef LA_FP8M_FB
#define LA_FP8M_FB 2
#endif
#ifndef LA_TC5_NST
#define LA_TC5_NST 3   // tcgen05 engine: ring stages of 64 KiB (128 tokens), one warpgroup each
#endif
#ifndef LA_TC5_NST32
#define LA_TC5_NST32 3  // the same for 32-row query tiles
#endif
#ifndef LA_TC5_NWG32
#define LA_TC5_NWG32 2  // warpgroups for 32-row tiles (< NST32: the ring prefetches past the warpgroups)
#endif
#ifndef LA_TC5_NWG16
#define LA_TC5_NWG16 LA_TC5_NST  // the same for 16-row tiles
#endif
#ifndef LA_TC5_NWG8
#define LA_TC5_NWG8 LA_TC5_NST   // the same for 8-row tiles
#endif
#ifndef LA_TC5_FB8
#define LA_TC5_FB8 1             // 8-row tiles: consumer -> epilogue fold buffers (2 fit with NWG8 = 2)
#endif
#ifndef LA_TC5_BOXH
#define LA_TC5_BOXH 1  // tcgen05 engine: one 128-B half of 128 rows per TMA box (16 KiB)
#endif
#ifndef LA_TC5_WIN8
#define LA_TC5_WIN8 0   // tcgen05 engine, 8-row tiles: stages in flight (0: the whole ring; measured: the
                        // full ring scatters the CTAs' rates, 2 stages 311 -> 305 us, 3 with V at 2: 306 -> 304)
#endif
#ifndef LA_TC5_VWIN8
#define LA_TC5_VWIN8 2  // tcgen05 engine, 8-row tiles: V of stage j after stage j - VWIN8 is consumed (0: off;
                        // every tile size: K on the whole ring, V 2 stages ahead -- 32 rows 317.9 -> 317.2 us)
#endif
#ifndef LA_TC5_VWIN16
#define LA_TC5_VWIN16 2  // ... 16-row tiles (0: off)
#endif
#ifndef LA_TC5_VWIN32
#define LA_TC5_VWIN32 2  // ... 32-row tiles (0: off)
#endif
#ifndef LA_TC5_WIN16
#define LA_TC5_WIN16 0  // ... 16-row tiles (2 measured c3 N_q = 2 317 -> 313 us; V window 2 alone: 313.1 vs 313.7 us)
#endif
#ifndef LA_WIDE_NEP16
#define LA_WIDE_NEP16 2  // 16-row tcgen05 tiles: epilogue warps (each folds / writes its own 8-row groups)
#endif
#ifndef LA_WIDE_NEP32
#define LA_WIDE_NEP32 2  // 32-row tiles: epilogue warps (4 would cap the kernel at 152 registers)
#endif
#ifndef LA_TC5_WIN32
#define LA_TC5_WIN32 0  // ... 32-row tiles (compute-bound: 2 stages measured 314 -> 355 us)
#endif
#ifndef LA_MHA_WIN
#define LA_MHA_WIN 0    // MHA engine: stages in flight (0: the whole ring; 4 measured within noise for
                        // c2 stream-K, slower dynamic (582 -> 586 us) and paged (620 -> 649 us); 3: 630 us)
#endif
#ifndef LA_TC5_QSTAGE8
#define LA_TC5_QSTAGE8 1  // tcgen05 8-row tiles: Q rows staged per segment by the producer (2-deep queue)
#endif
#ifndef LA_TC5_LD32
#define LA_TC5_LD32 1  // tcgen05 16/32-row tiles: 32-column TMEM loads (fewer load round trips)
#endif
#ifndef LA_ELECT_PRODUCE
#define LA_ELECT_PRODUCE 1  // tcgen05 8-row tiles (BHSD / packed): stage loads issued by an elected lane of the
                            // warp (measured equal to lane-0 issue: 305.0 vs 305.0 us; kept for one issue path)
#endif
#ifndef LA_PAGED_ELECT
#define LA_PAGED_ELECT 1  // paged GQA / tcgen05 producers: loads issued by an elected lane of the converged warp
#endif
#ifndef LA_FP8_WIN
#define LA_FP8_WIN 0    // FP8 engine: stages in flight (0: the whole ring; 4 measured slower: c2 304 -> 319 us)
#endif
#ifndef LA_GQA_WIN
#define LA_GQA_WIN 0    // mma.sync GQA engine: stages in flight (0: the whole ring)
#endif
#ifndef LA_TC5_MMA8
#define LA_TC5_MMA8 1  // tcgen05 engine: each stage's 8 k-step MMAs of one product in one asm statement
#endif
#ifndef LA_TC5_SPLIT
#define LA_TC5_SPLIT 1  // tcgen05 engine: 1 or 2 independent accumulator chains per MMA (4 k-steps each)
#endif
#ifndef LA_FP8_SPLITP
#define LA_FP8_SPLITP 0  // one f16 P (2^-12 relative, 256x finer than the E4M3 data); 1: P_hi + P_lo
#endif

namespace la {

struct alignas(64) TmapPair {
  CUtensorMap k;
  CUtensorMap v;
};

namespace {

using namespace dev;

// =======================================================================================
// MHA arithmetic on one 16-byte chunk of a K / V row
//   dot : acc + sum_e q[e] k[e]    (fp32)          axpy: o[e] += p v[e]   (fp32)
// =======================================================================================
template <typename T>
struct Chunk;

template <>
struct Chunk<__nv_bfloat16> {
  static constexpr int EPL = 8;
  struct Q {
    unsigned short h[8];  // exact bf16 inputs
  };
  __device__ __forceinline__ static Q load_q(const void* p) {
    const uint4 w = *reinterpret_cast<const uint4*>(p);
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
    Q q;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      q.h[2 * i] = static_cast<unsigned short>(ws[i] & 0xffffu);
      q.h[2 * i + 1] = static_cast<unsigned short>(ws[i] >> 16);
    }
    return q;
  }
  // FHFMA.BF16: the bf16 x bf16 product is exact in fp32; one rounding on the add.
  __device__ __forceinline__ static float dot(const uint4 k, const Q& q, float acc) {
    asm("{\n\t.reg .b16 l0, h0, l1, h1, l2, h2, l3, h3;\n\t"
        "mov.b32 {l0, h0}, %1;\n\tmov.b32 {l1, h1}, %2;\n\t"
        "mov.b32 {l2, h2}, %3;\n\tmov.b32 {l3, h3}, %4;\n\t"
        "fma.rn.f32.bf16 %0, l0, %5, %0;\n\tfma.rn.f32.bf16 %0, h0, %6, %0;\n\t"
        "fma.rn.f32.bf16 %0, l1, %7, %0;\n\tfma.rn.f32.bf16 %0, h1, %8, %0;\n\t"
        "fma.rn.f32.bf16 %0, l2, %9, %0;\n\tfma.rn.f32.bf16 %0, h2, %10, %0;\n\t"
        "fma.rn.f32.bf16 %0, l3, %11, %0;\n\tfma.rn.f32.bf16 %0, h3, %12, %0;\n\t}"
        : "+f"(acc)
        : "r"(k.x), "r"(k.y), "r"(k.z), "r"(k.w), "h"(q.h[0]), "h"(q.h[1]), "h"(q.h[2]), "h"(q.h[3]),
          "h"(q.h[4]), "h"(q.h[5]), "h"(q.h[6]), "h"(q.h[7]));
    return acc;
  }
  __device__ __forceinline__ static void axpy(float p, const uint4 v, float2 (&o)[4]) {
    const float2 pp = make_float2(p, p);
    const uint32_t ws[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i)
      o[i] = __ffma2_rn(pp, make_float2(__uint_as_float(ws[i] << 16), __uint_as_float(ws[i] & 0xffff0000u)), o[i]);
  }
};

template <>
struct Chunk<__half> {
  static constexpr int EPL = 8;
  struct Q {
    unsigned short h[8];
  };
  __device__ __forceinline__ static Q load_q(const void* p) {
    const uint4 w = *reinterpret_cast<const uint4*>(p);
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
    Q q;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      q.h[2 * i] = static_cast<unsigned short>(ws[i] & 0xffffu);
      q.h[2 * i + 1] = static_cast<unsigned short>(ws[i] >> 16);
    }
    return q;
  }
  __device__ __forceinline__ static float dot(const uint4 k, const Q& q, float acc) {
    asm("{\n\t.reg .b16 l0, h0, l1, h1, l2, h2, l3, h3;\n\t"
        "mov.b32 {l0, h0}, %1;\n\tmov.b32 {l1, h1}, %2;\n\t"
        "mov.b32 {l2, h2}, %3;\n\tmov.b32 {l3, h3}, %4;\n\t"
        "fma.rn.f32.f16 %0, l0, %5, %0;\n\tfma.rn.f32.f16 %0, h0, %6, %0;\n\t"
        "fma.rn.f32.f16 %0, l1, %7, %0;\n\tfma.rn.f32.f16 %0, h1, %8, %0;\n\t"
        "fma.rn.f32.f16 %0, l2, %9, %0;\n\tfma.rn.f32.f16 %0, h2, %10, %0;\n\t"
        "fma.rn.f32.f16 %0, l3, %11, %0;\n\tfma.rn.f32.f16 %0, h3, %12, %0;\n\t}"
        : "+f"(acc)
        : "r"(k.x), "r"(k.y), "r"(k.z), "r"(k.w), "h"(q.h[0]), "h"(q.h[1]), "h"(q.h[2]), "h"(q.h[3]),
          "h"(q.h[4]), "h"(q.h[5]), "h"(q.h[6]), "h"(q.h[7]));
    return acc;
  }
  __device__ __forceinline__ static void axpy(float p, const uint4 v, float2 (&o)[4]) {
    const float2 pp = make_float2(p, p);
    const uint32_t ws[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) o[i] = __ffma2_rn(pp, __half22float2(*reinterpret_cast<const __half2*>(&ws[i])), o[i]);
  }
};

template <>
struct Chunk<float> {
  static constexpr int EPL = 4;
  struct Q {
    float f[4];
  };
  __device__ __forceinline__ static Q load_q(const void* p) {
    const float4 w = *reinterpret_cast<const float4*>(p);
    return Q{{w.x, w.y, w.z, w.w}};
  }
  __device__ __forceinline__ static float dot(const uint4 k, const Q& q, float acc) {
    acc = fmaf(__uint_as_float(k.x), q.f[0], acc);
    acc = fmaf(__uint_as_float(k.y), q.f[1], acc);
    acc = fmaf(__uint_as_float(k.z), q.f[2], acc);
    return fmaf(__uint_as_float(k.w), q.f[3], acc);
  }
  __device__ __forceinline__ static void axpy(float p, const uint4 v, float2 (&o)[2]) {
    const float2 pp = make_float2(p, p);
    o[0] = __ffma2_rn(pp, make_float2(__uint_as_float(v.x), __uint_as_float(v.y)), o[0]);
    o[1] = __ffma2_rn(pp, make_float2(__uint_as_float(v.z), __uint_as_float(v.w)), o[1]);
  }
};

// =======================================================================================
// Paged KV (LA_KV_PAGED): the producer's 32-entry window onto one request's block-table
// row, refilled with 8 independent 16-byte loads (one L2 round trip per 32 pages).
// =======================================================================================
struct PageWin {
  // A window of 64 consecutive block-table entries of the unit's request, held one per lane in
  // two registers (entries base + lane and base + 32 + lane): a lookup is a shuffle, a stage
  // (<= 8 pages) never straddles the window, and sliding by 32 entries reuses the upper half
  // and issues ONE coalesced 128-B load for the next (consumed only at the slide after, so its
  // latency is off the producer's path).  r01's per-lane local-memory table cost every stage
  // dependent local-memory round trips and every 32 pages a 32-entry spill per lane.
  const int32_t* row;
  int heads_kv, h, shift, base, n;
  int32_t e0, e1;
  __device__ __forceinline__ int32_t ld(int i) const { return i < n ? __ldg(row + i) : 0; }
  __device__ __forceinline__ void init(const DecodeArgs& a, int64_t unit_bh) {
    const int b = int(unit_bh / a.heads_kv);
    h = int(unit_bh % a.heads_kv);
    row = a.block_table + size_t(b) * a.pt_stride;
    n = a.pt_stride;
    heads_kv = a.heads_kv;
    shift = a.page_shift;
    base = -1;
  }
  // Whole warp (converged).  p0: the stage's first page (warp-uniform); t: this lane's token
  // (any value for an idle lane: its result is garbage but harmless).  Pool row of token t.
  __device__ __forceinline__ int64_t rows(int p0, int t, int lane) {
    if (base < 0 || p0 < base || p0 >= base + 64) {  // (re)load both halves around p0
      base = p0 & ~31;
      e0 = ld(base + lane);
      e1 = ld(base + 32 + lane);
    } else if (p0 >= base + 32) {                    // slide by 32: the next half is prefetched
      base += 32;
      e0 = e1;
      e1 = ld(base + 32 + lane);
    }
    const int pi = (t >> shift) - base;              // in [0, 64) for the stage's tokens
    const int32_t lo = __shfl_sync(0xffffffffu, e0, pi & 31), hi = __shfl_sync(0xffffffffu, e1, pi & 31);
    const int32_t pg = pi < 32 ? lo : hi;
    return (int64_t(pg) * heads_kv + h) * (int64_t(1) << shift) + (t & ((1 << shift) - 1));
  }
};

// =======================================================================================
// MHA engine (T_m = 1): CUDA-core fp32 arithmetic
// =======================================================================================
template <typename T, int D_, int NST_, int WPS_>
struct MhaEngine {
  static constexpr int D = D_, NST = NST_, WPS = WPS_, NWG = NST, NCW = NWG * WPS;  // NWG: consumer warp sets
  static constexpr int WIN = LA_MHA_WIN > 0 ? LA_MHA_WIN : NST;  // stages in flight
  static constexpr int ROWB = D * int(sizeof(T));          // bytes of one K (or V) row
  static constexpr int LPK = ROWB / 16;                     // lanes per key
  static constexpr int EPL = 16 / int(sizeof(T));           // elements per 16-byte chunk
  static constexpr int STAGE_TOK = 32768 / (2 * ROWB);      // 32 KiB of K+V per stage
  static constexpr int STAGE_BYTES = 2 * STAGE_TOK * ROWB;
  static constexpr int HEADS = 1;                           // q-heads per unit
  static constexpr int FOLD_FLOATS = NCW * (D + 4);         // per warp: O[D], m, l, pad (16-B rows)
  static constexpr int FOLD_BUFS = 2;                       // double-buffered hand-off
  static constexpr bool ZERO_RING = false;                  // tail V rows are zeroed per warp
  using QElem = T;                                          // Q storage type
  static constexpr bool QSTAGE = true;                      // Q rows staged in smem per segment
  static_assert(LPK >= 2 && LPK <= 32 && (LPK & (LPK - 1)) == 0, "lanes per key");
  static_assert(STAGE_TOK % 32 == 0, "stage holds whole 32-key rounds");

  struct State {
    typename Chunk<T>::Q qf;
    float m, l;
    float2 o[EPL / 2];
  };

  __device__ __forceinline__ static void produce(unsigned char* dst, const DecodeArgs& a, const TmapPair&, int64_t row,
                                                 int ntok, uint64_t* bar, uint64_t pol) {
    const uint32_t bytes = uint32_t(ntok) * ROWB;
    mbar_arrive_expect_tx(bar, 2 * bytes);
    const size_t goff = size_t(row) * ROWB;
    bulk_g2s(dst, static_cast<const unsigned char*>(a.k) + goff, bytes, bar, pol);
    bulk_g2s(dst + STAGE_TOK * ROWB, static_cast<const unsigned char*>(a.v) + goff, bytes, bar, pol);
  }

  // Paged KV: one bulk copy per page-contiguous run of the stage's tokens; lane r of the
  // producer warp issues run r (a stage spans at most 5 pages).
  __device__ __forceinline__ static void produce_paged(unsigned char* dst, const DecodeArgs& a, const TmapPair&,
                                                       PageWin& pw, int s0, int ntok, uint64_t* bar, uint64_t pol,
                                                       int lane) {
    if (lane == 0) mbar_arrive_expect_tx(bar, 2 * uint32_t(ntok) * ROWB);
    __syncwarp();
    const int page = 1 << a.page_shift;
    const int first = s0 & ~(page - 1);
    const int t = lane == 0 ? s0 : first + lane * page;
    const int64_t prow = pw.rows(s0 >> a.page_shift, t, lane);  // whole warp
    if constexpr (LA_PAGED_ELECT > 1) {  // (measured slower for 1-D bulk copies: c2 page 16 628 -> 672 us)
      const int nrun = ((s0 + ntok - 1) >> a.page_shift) - (s0 >> a.page_shift) + 1;  // pages in the stage
      #pragma unroll 1
      for (int r = 0; r < nrun; ++r) {  // converged warp, one elected lane copies run r
        const int tr = __shfl_sync(0xffffffffu, t, r);
        const int64_t pr = __shfl_sync(0xffffffffu, prow, r);
        const int run = min(first + (r + 1) * page, s0 + ntok) - tr;
        const size_t goff = size_t(pr) * ROWB;
        const int doff = (tr - s0) * ROWB;
        bulk_g2s_kv_elect(dst + doff, dst + STAGE_TOK * ROWB + doff, static_cast<const unsigned char*>(a.k) + goff,
                          static_cast<const unsigned char*>(a.v) + goff, uint32_t(run) * ROWB, bar, pol);
      }
    } else if (t < s0 + ntok) {
      const int run = min(first + (lane + 1) * page, s0 + ntok) - t;
      const size_t goff = size_t(prow) * ROWB;
      const int doff = (t - s0) * ROWB;
      bulk_g2s(dst + doff, static_cast<const unsigned char*>(a.k) + goff, uint32_t(run) * ROWB, bar, pol);
      bulk_g2s(dst + STAGE_TOK * ROWB + doff, static_cast<const unsigned char*>(a.v) + goff, uint32_t(run) * ROWB,
               bar, pol);
    }
  }

  __device__ __forceinline__ static void seg_begin(State& s, const DecodeArgs& a, const DevUnit& u, int lane,
                                                   const void* qsrc) {  // qsrc: the unit's Q row (smem)
    s.qf = Chunk<T>::load_q(static_cast<const T*>(qsrc) + (lane % LPK) * EPL);
    s.m = -INFINITY;  // Alg1§8-9
    s.l = 0.f;
#pragma unroll
    for (int e = 0; e < EPL / 2; ++e) s.o[e] = make_float2(0.f, 0.f);
  }

  // This warp's 32-key rounds (sub, sub + WPS, ...) of one stage of ntok keys.
  __device__ __forceinline__ static void stage(State& s, unsigned char* st, int sub, int ntok, int /*tok0*/,
                                               float scale_log2, int lane, int /*bs*/) {
    const int kg = lane / LPK, li = lane % LPK;
    const unsigned char* ks = st;
    const unsigned char* vs = st + STAGE_TOK * ROWB;
    for (int r = sub * 32; r < ntok; r += 32 * WPS) {
      if (r + 32 > ntok) {
        // keys ntok .. r + 31 of this round are past the stage (the next unit's rows, or stale
        // smem that may not be finite): their scores are masked, and their V rows zeroed so
        // that 0 * V stays 0 (reading C5) -- only a unit's short last stage gets here
        uint4* vz = reinterpret_cast<uint4*>(st + STAGE_TOK * ROWB + ntok * ROWB);
        for (int i = lane; i < (r + 32 - ntok) * (ROWB / 16); i += 32) vz[i] = make_uint4(0u, 0u, 0u, 0u);
        __syncwarp();
      }
      const int kb = r + kg * LPK;
      // S_f = Q_f K_f^T (Alg1§20): lane li accumulates key (jj ^ li) over its chunk li
      float acc[LPK];
#pragma unroll
      for (int jj = 0; jj < LPK; ++jj)
        acc[jj] = Chunk<T>::dot(*reinterpret_cast<const uint4*>(ks + (kb + (jj ^ li)) * ROWB + li * 16), s.qf, 0.f);
      // XOR transpose-butterfly: acc[0] of lane li ends up as the full dot of key kb + li
#pragma unroll
      for (int off = LPK / 2; off >= 1; off >>= 1) {
#pragma unroll
        for (int jj = 0; jj < off; ++jj) acc[jj] += __shfl_xor_sync(0xffffffffu, acc[jj + off], off);
      }
      const float sc = (kb + li < ntok) ? acc[0] * scale_log2 : -INFINITY;  // reading C5
      float mr = sc;                                                         // Alg1§21
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) mr = fmaxf(mr, __shfl_xor_sync(0xffffffffu, mr, off));
      if (mr > s.m) {  // warp-uniform: e^{m - m_new} rescale (Alg1§23-24)
        const float alpha = ex2(s.m - mr);
        s.l *= alpha;
        const float2 aa = make_float2(alpha, alpha);
#pragma unroll
        for (int e = 0; e < EPL / 2; ++e) s.o[e] = __fmul2_rn(aa, s.o[e]);
        s.m = mr;
      }
      const float p = ex2(sc - s.m);  // Alg1§22
      s.l += p;                       // Alg1§23
#pragma unroll
      for (int jj = 0; jj < LPK; ++jj)  // O_acc += P_f V_f (Alg1§24); lane li owns chunk li
        Chunk<T>::axpy(__shfl_sync(0xffffffffu, p, jj, LPK),
                       *reinterpret_cast<const uint4*>(vs + (kb + jj) * ROWB + li * 16), s.o);
      if (r + 32 > ntok) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic -> TMA WAR
    }
  }

  // Fold this warp's lane groups and write (O[D], m, l) to its fold-buffer row.
  __device__ __forceinline__ static void seg_end(State& s, float* fold, int warp, int lane) {
    const int kg = lane / LPK, li = lane % LPK;
#pragma unroll
    for (int off = LPK; off < 32; off <<= 1) {
#pragma unroll
      for (int e = 0; e < EPL / 2; ++e) {
        s.o[e].x += __shfl_xor_sync(0xffffffffu, s.o[e].x, off);
        s.o[e].y += __shfl_xor_sync(0xffffffffu, s.o[e].y, off);
      }
    }
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) s.l += __shfl_xor_sync(0xffffffffu, s.l, off);
    float* fb = fold + warp * (D + 4);
    if (kg == 0) {
#pragma unroll
      for (int e = 0; e < EPL / 2; ++e) {
        fb[li * EPL + 2 * e] = s.o[e].x;
        fb[li * EPL + 2 * e + 1] = s.o[e].y;
      }
    }
    if (lane == 0) {
      fb[D] = s.m;
      fb[D + 1] = s.l;
    }
  }
};

// =======================================================================================
// GQA engine (T_m = g q-heads of one KV head): tensor cores
// =======================================================================================
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}

__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}

__device__ __forceinline__ uint32_t movmatrix_t(uint32_t x) {
  uint32_t y;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}

template <typename T>
struct Mma;

template <>
struct Mma<__nv_bfloat16> {
  __device__ __forceinline__ static void run(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
        "{%0, %1, %2, %3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  }
  __device__ __forceinline__ static uint32_t pack(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
  }
  __device__ __forceinline__ static float2 unpack(uint32_t w) {
    return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w));
  }
};

template <>
struct Mma<__half> {
  __device__ __forceinline__ static void run(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
        "{%0, %1, %2, %3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  }
  __device__ __forceinline__ static uint32_t pack(float lo, float hi) {
    __half2 v = __floats2half2_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
  }
  __device__ __forceinline__ static float2 unpack(uint32_t w) {
    return __half22float2(*reinterpret_cast<const __half2*>(&w));
  }
};

// Whole (converged) warp: one elected lane issues the 3-D box loads of K and V at the same
// coordinates (paged producers: the operands are warp-uniform, so ptxas needs no per-lane
// waterfall loop around the instructions)
__device__ __forceinline__ void tma_load_3d_kv_elect(void* dk, void* dv, const CUtensorMap* tk, const CUtensorMap* tv,
                                                     int c1, int c2, uint64_t* bk, uint64_t* bv, uint64_t policy) {
  asm volatile(
      "{\n\t.reg .pred pe;\n\telect.sync _|pe, 0xffffffff;\n\t"
      "@pe cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%2, {0, %4, %5}], [%6], %8;\n\t"
      "@pe cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%1], [%3, {0, %4, %5}], [%7], %8;\n\t}" ::"r"(smem_u32(dk)),
      "r"(smem_u32(dv)), "l"(reinterpret_cast<uint64_t>(tk)), "l"(reinterpret_cast<uint64_t>(tv)), "r"(c1), "r"(c2),
      "r"(smem_u32(bk)), "r"(smem_u32(bv)), "l"(policy)
      : "memory");
}
// Whole (converged) warp: one elected lane loads both 128-B halves (coordinate 2 = 0, 1) of
// one tensor's rows into dst and dst + 16 KiB
__device__ __forceinline__ void tma_load_3d_halves_elect(void* dst, const CUtensorMap* tm, int c1, uint64_t* bar,
                                                         uint64_t policy) {
  asm volatile(
      "{\n\t.reg .pred pe;\n\telect.sync _|pe, 0xffffffff;\n\t"
      "@pe cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%2, {0, %3, 0}], [%4], %5;\n\t"
      "@pe cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%1], [%2, {0, %3, 1}], [%4], %5;\n\t}" ::"r"(smem_u32(dst)),
      "r"(smem_u32(dst) + 16384u), "l"(reinterpret_cast<uint64_t>(tm)), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d_kv_elect(void* dk, void* dv, const CUtensorMap* tk, const CUtensorMap* tv,
                                                     int c1, uint64_t* bar, uint64_t policy) {
  asm volatile(
      "{\n\t.reg .pred pe;\n\telect.sync _|pe, 0xffffffff;\n\t"
      "@pe cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%2, {0, %4}], [%5], %6;\n\t"
      "@pe cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%1], [%3, {0, %4}], [%5], %6;\n\t}" ::"r"(smem_u32(dk)),
      "r"(smem_u32(dv)), "l"(reinterpret_cast<uint64_t>(tk)), "l"(reinterpret_cast<uint64_t>(tv)), "r"(c1),
      "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tm, int c0, int c1, uint64_t* bar,
                                            uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// 3-D tile: coordinates {element, row, 64-element half}; the d = 128 K/V maps view a row as
// two 128-B halves so ONE box brings both halves of box_rows rows: smem [half][rows][128 B].
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* tm, int c0, int c1, int c2, uint64_t* bar,
                                            uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

template <typename T, int D_, int NST_, int WPS_>
struct GqaEngine {
  static constexpr int D = D_, NST = NST_, WPS = WPS_, NWG = NST, NCW = NWG * WPS;  // NWG: consumer warp sets
  static constexpr int WIN = LA_GQA_WIN > 0 ? LA_GQA_WIN : NST;  // stages in flight
  static constexpr int STAGE_TOK = 64;            // = TMA box rows
  static constexpr int NBOX = D / 64;             // 64-element (128-B) boxes per row
  static constexpr int BOX_BYTES = STAGE_TOK * 128;
  static constexpr int KV_BYTES = NBOX * BOX_BYTES;
  static constexpr int STAGE_BYTES = 2 * KV_BYTES;
  static constexpr int HEADS = 8;                 // MMA N: q-heads per unit (padded to 8)
  static constexpr int KS = D / 16;               // k-steps of QK^T = m-tiles of PV
  static constexpr int FOLD_FLOATS = NCW * HEADS * (D + 4);
  static constexpr int FOLD_BUFS = LA_GQA_FB;     // double-buffered hand-off (measured best)
  static constexpr bool ZERO_RING = false;        // tail V rows are zeroed per warp
  using QElem = T;
  static constexpr bool QSTAGE = true;

  struct State {
    uint32_t qb[KS][2];     // Q^T B-fragments (exact inputs)
    float m[2], l[2];       // tile rows 2tq, 2tq+1 (unit row r0 + r = head j * N_b + query i)
    float o[KS][4];         // O^T fragments: dims 16mm + gq (+8), rows 2tq, 2tq+1
    int lim[2];             // causal key limit of rows 2tq, 2tq+1 (unit-local, exclusive)
  };

  __device__ __forceinline__ static void produce(unsigned char* dst, const DecodeArgs&, const TmapPair& tm, int64_t row,
                                                 int, uint64_t* bar, uint64_t pol) {
    mbar_arrive_expect_tx(bar, STAGE_BYTES);  // full boxes (rows past the tensor are zero-filled)
    if (NBOX == 1) {
      tma_load_2d(dst, &tm.k, 0, int(row), bar, pol);
      tma_load_2d(dst + KV_BYTES, &tm.v, 0, int(row), bar, pol);
    } else {  // both 128-B halves of 64 rows per op: [half][64 rows][128 B]
      tma_load_3d(dst, &tm.k, 0, int(row), 0, bar, pol);
      tma_load_3d(dst + KV_BYTES, &tm.v, 0, int(row), 0, bar, pol);
    }
  }

  // Byte offset of the first 128-B line of stage row `tok` and the distance between the two
  // halves of a row: a stage is 64 / box_rows boxes of [half][box_rows][128 B] (box_rows =
  // 2^bs: 64 unpaged -- the plain [half][64][128 B] layout -- or min(64, page) paged).
  __device__ __forceinline__ static uint32_t row_off(int tok, int bs) {
    return NBOX == 1 ? uint32_t(tok) << 7
                     : (uint32_t(tok >> bs) << (bs + 8)) + (uint32_t(tok & ((1 << bs) - 1)) << 7);
  }
  __device__ __forceinline__ static uint32_t half_stride(int bs) { return NBOX == 1 ? 0u : (1u << (bs + 7)); }

  // Paged KV: boxes of box_rows = min(64, page) rows (both halves), each inside one page,
  // at 1024-B multiples so the 128-B swizzle phase is the row index (see row_off).  Lane r
  // of the producer warp issues load r = (box i, K or V): 2 ops per page, not 2 * NBOX.
  __device__ __forceinline__ static void produce_paged(unsigned char* dst, const DecodeArgs& a, const TmapPair& tm,
                                                       PageWin& pw, int s0, int ntok, uint64_t* bar, uint64_t pol,
                                                       int lane) {
    const int br = a.box_rows;
    const int nb = (ntok + br - 1) / br;
    if (lane == 0) mbar_arrive_expect_tx(bar, uint32_t(nb * br * 128 * NBOX * 2));
    __syncwarp();
    const int rowl = int(pw.rows(s0 >> a.page_shift, s0 + lane * br, lane));  // whole warp: lane i -> box i
    if constexpr (NBOX == 2 && LA_PAGED_ELECT) {
      #pragma unroll 1
      for (int i = 0; i < nb; ++i) {  // converged warp, one elected lane issues (warp-uniform operands)
        unsigned char* d = dst + i * br * 128 * NBOX;
        tma_load_3d_kv_elect(d, d + KV_BYTES, &tm.k, &tm.v, __shfl_sync(0xffffffffu, rowl, i), 0, bar, bar, pol);
      }
    } else if (lane < nb) {  // lane i: box i (<= 8), its K and V loads (one row coordinate for both)
      unsigned char* d = dst + lane * br * 128 * NBOX;
      if (NBOX == 1) {
        tma_load_2d(d, &tm.k, 0, rowl, bar, pol);
        tma_load_2d(d + KV_BYTES, &tm.v, 0, rowl, bar, pol);
      } else {
        tma_load_3d(d, &tm.k, 0, rowl, 0, bar, pol);
        tma_load_3d(d + KV_BYTES, &tm.v, 0, rowl, 0, bar, pol);
      }
    }
  }

  __device__ __forceinline__ static void seg_begin(State& s, const DecodeArgs& a, const DevUnit& u, int lane,
                                                   const void* qsrc) {  // qsrc: the unit's Q rows (smem)
    const int gq = lane >> 2, tq = lane & 3;
    const uint32_t* qrow = reinterpret_cast<const uint32_t*>(static_cast<const T*>(qsrc) + size_t(gq) * D);
    const bool ok = gq < u.rows;
#pragma unroll
    for (int kk = 0; kk < KS; ++kk) {  // b0 = Q[gq][16kk + 2tq, +1], b1 = Q[gq][16kk + 8 + 2tq, +1]
      s.qb[kk][0] = ok ? qrow[8 * kk + tq] : 0u;
      s.qb[kk][1] = ok ? qrow[8 * kk + 4 + tq] : 0u;
    }
    s.m[0] = s.m[1] = -INFINITY;
    s.l[0] = s.l[1] = 0.f;
#pragma unroll
    for (int mm = 0; mm < KS; ++mm) s.o[mm][0] = s.o[mm][1] = s.o[mm][2] = s.o[mm][3] = 0.f;
    // N_b > 1, causal: query i (row r0 + r = j * N_b + i) is the token at n - N_b + i (NEXT-3)
#pragma unroll
    for (int e = 0; e < 2; ++e)
      s.lim[e] = a.causal ? u.len - u.nq + ((u.r0 + 2 * tq + e) % u.nq) + 1 : u.len;
  }

  // This warp's 32-token rounds (sub, sub + WPS, ...) of one stage of ntok tokens starting
  // at unit-local token tok0.
  __device__ __forceinline__ static void stage(State& s, unsigned char* st, int sub, int ntok, int tok0,
                                               float scale_log2, int lane, int bs) {
    for (int rb = sub * 32; rb < ntok; rb += 32 * WPS) round(s, st, rb, ntok, tok0, scale_log2, lane, bs);
  }

  __device__ __forceinline__ static void round(State& s, unsigned char* st, int rb, int ntok, int tok0,
                                               float scale_log2, int lane, int bs) {
    const uint32_t hs = half_stride(bs);
    const int gq = lane >> 2, mi = lane >> 3, ri = lane & 7;
    if (rb + 32 > ntok) {
      // rows >= ntok of this round hold the next unit's rows or cache padding: zero this
      // warp's V rows so 0 * (non-finite) can never reach the accumulator
      for (int r = rb + (lane >> 3); r < rb + 32; r += 4)
        if (r >= ntok)
#pragma unroll
          for (int b = 0; b < NBOX; ++b)
            *reinterpret_cast<uint4*>(st + KV_BYTES + b * hs + row_off(r, bs) + (ri << 4)) = make_uint4(0u, 0u, 0u, 0u);
      __syncwarp();
    }
    const uint32_t kbase = smem_u32(st), vbase = smem_u32(st + KV_BYTES);
    // ---- S^T = K_f Q_f^T for two 16-token blocks (Alg1§20) ------------------------------
    float sc[2][4];
#pragma unroll
    for (int blk = 0; blk < 2; ++blk) {
      sc[blk][0] = sc[blk][1] = sc[blk][2] = sc[blk][3] = 0.f;
      const int tok = rb + blk * 16 + ri + ((mi & 1) << 3);
      const uint32_t ro = kbase + row_off(tok, bs);
#pragma unroll
      for (int kk = 0; kk < KS; ++kk) {
        const int chunk = 2 * kk + (mi >> 1);
        uint32_t af[4];
        ldsm_x4(ro + (chunk >> 3) * hs + (((chunk & 7) ^ (tok & 7)) << 4), af);
        Mma<T>::run(sc[blk], af, s.qb[kk][0], s.qb[kk][1]);
      }
    }
    // ---- scale, mask the tail (C5), running max per head (Alg1§21) ------------------------
    float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int blk = 0; blk < 2; ++blk) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int tok = rb + blk * 16 + gq + ((e >> 1) << 3);
        const bool ok = tok < ntok && tok0 + tok < s.lim[e & 1];  // tail (C5) and causal limit
        sc[blk][e] = ok ? sc[blk][e] * scale_log2 : -INFINITY;
        mx[e & 1] = fmaxf(mx[e & 1], sc[blk][e]);
      }
    }
#pragma unroll
    for (int off = 4; off <= 16; off <<= 1) {
      mx[0] = fmaxf(mx[0], __shfl_xor_sync(0xffffffffu, mx[0], off));
      mx[1] = fmaxf(mx[1], __shfl_xor_sync(0xffffffffu, mx[1], off));
    }
    if (__any_sync(0xffffffffu, (mx[0] > s.m[0]) || (mx[1] > s.m[1]))) {  // Alg1§23-24 rescale
      const float mn0 = fmaxf(s.m[0], mx[0]), mn1 = fmaxf(s.m[1], mx[1]);
      const float al0 = ex2_sub(s.m[0], mn0), al1 = ex2_sub(s.m[1], mn1);
      s.l[0] *= al0;
      s.l[1] *= al1;
#pragma unroll
      for (int mm = 0; mm < KS; ++mm) {
        s.o[mm][0] *= al0;
        s.o[mm][2] *= al0;
        s.o[mm][1] *= al1;
        s.o[mm][3] *= al1;
      }
      s.m[0] = mn0;
      s.m[1] = mn1;
    }
    // ---- P_f = exp(S_f - m) (Alg1§22); O^T += V^T P^T (Alg1§24) -----------------------------
#pragma unroll
    for (int blk = 0; blk < 2; ++blk) {
      // ex2_sub: a row that has seen no key yet (m = -inf, fully masked) gets p = 0, not NaN
      const float p0 = ex2_sub(sc[blk][0], s.m[0]), p1 = ex2_sub(sc[blk][1], s.m[1]);
      const float p2 = ex2_sub(sc[blk][2], s.m[0]), p3 = ex2_sub(sc[blk][3], s.m[1]);
      s.l[0] += p0 + p2;
      s.l[1] += p1 + p3;
      // P = P_hi + P_lo, both in the KV type (P_lo = round(p - P_hi), exact subtraction):
      // two MMAs on the same V^T fragments keep P to ~2^-16 relative instead of the KV
      // type's 2^-8 (reading C18; the tensor pipe is ~10% busy, so the extra MMA is free).
      const uint32_t h01 = Mma<T>::pack(p0, p1), h23 = Mma<T>::pack(p2, p3);
      const float2 r01 = Mma<T>::unpack(h01), r23 = Mma<T>::unpack(h23);
      const uint32_t b0 = movmatrix_t(h01);  // P_hi[tok 2tq..][head gq]
      const uint32_t b1 = movmatrix_t(h23);
      const uint32_t c0 = movmatrix_t(Mma<T>::pack(p0 - r01.x, p1 - r01.y));  // P_lo
      const uint32_t c1 = movmatrix_t(Mma<T>::pack(p2 - r23.x, p3 - r23.y));
      const int tok = rb + blk * 16 + ri + ((mi >> 1) << 3);
      const uint32_t ro = vbase + row_off(tok, bs);
#pragma unroll
      for (int mm = 0; mm < KS; ++mm) {
        const int chunk = 2 * mm + (mi & 1);
        uint32_t af[4];
        ldsm_x4_t(ro + (chunk >> 3) * hs + (((chunk & 7) ^ (tok & 7)) << 4), af);
        Mma<T>::run(s.o[mm], af, b0, b1);
        if (LA_GQA_SPLITP) Mma<T>::run(s.o[mm], af, c0, c1);
      }
    }
    if (rb + 32 > ntok) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic -> TMA WAR
  }

  __device__ __forceinline__ static void seg_end(State& s, float* fold, int warp, int lane) {
    const int gq = lane >> 2, tq = lane & 3;
#pragma unroll
    for (int off = 4; off <= 16; off <<= 1) {
      s.l[0] += __shfl_xor_sync(0xffffffffu, s.l[0], off);
      s.l[1] += __shfl_xor_sync(0xffffffffu, s.l[1], off);
    }
    float* fb = fold + warp * HEADS * (D + 4);  // [head][D + 4]
    const int h0 = 2 * tq, h1 = 2 * tq + 1;
#pragma unroll
    for (int mm = 0; mm < KS; ++mm) {
      const int c = 16 * mm + gq;
      fb[h0 * (D + 4) + c] = s.o[mm][0];
      fb[h1 * (D + 4) + c] = s.o[mm][1];
      fb[h0 * (D + 4) + c + 8] = s.o[mm][2];
      fb[h1 * (D + 4) + c + 8] = s.o[mm][3];
    }
    if (gq == 0) {
      fb[h0 * (D + 4) + D] = s.m[0];
      fb[h0 * (D + 4) + D + 1] = s.l[0];
      fb[h1 * (D + 4) + D] = s.m[1];
      fb[h1 * (D + 4) + D + 1] = s.l[1];
    }
  }
};

// =======================================================================================
// FP8 engine (NEXT-4: E4M3 KV cache, bf16 Q; any T_m <= 8 incl. MHA): tensor cores
// =======================================================================================
// The KV codes are widened to f16 in registers (cvt.rn.f16x2.e4m3x2: exact, every E4M3
// value is an f16 normal or zero) straight from ldmatrix fragments, and the GQA engine's
// swap-AB m16n8k16 MMAs run in f16 (Q rounded bf16 -> f16, reading C23).  The fragments
// come from ldmatrix on byte PAIRS, so their element order differs from a 16-bit tile:
//  * S^T = K_f Q_f^T: a plain ldmatrix of 8 tokens x 16 codes gives lane (gq, tq) the four
//    codes at dims 4tq .. 4tq+3 of one token -- the A fragment's k pairs (2tq, 2tq+1) and
//    (2tq+8, 2tq+9) take dims (4tq, 4tq+1) and (4tq+2, 4tq+3).  The contraction index may
//    be permuted freely, so Q's B fragment is built with the same permutation.
//  * O^T += V^T P^T: ldmatrix.trans of 8 tokens x 16 codes gives lane (gq, tq) the codes
//    of dims (2gq, 2gq+1) of tokens (2tq, 2tq+1); one byte permute regroups them per dim,
//    so A row gq holds dim 2gq and row gq + 8 dim 2gq + 1 of the 16-dim slice (an output-
//    row permutation, undone where the accumulator is written out).
__device__ __forceinline__ uint32_t e4m3x2_lo(uint32_t x) {  // codes in bits 0-15 -> f16x2
  uint32_t y;
  asm("{\n\t.reg .b16 lo, hi;\n\tmov.b32 {lo, hi}, %1;\n\tcvt.rn.f16x2.e4m3x2 %0, lo;\n\t}" : "=r"(y) : "r"(x));
  return y;
}
__device__ __forceinline__ uint32_t e4m3x2_hi(uint32_t x) {  // codes in bits 16-31 -> f16x2
  uint32_t y;
  asm("{\n\t.reg .b16 lo, hi;\n\tmov.b32 {lo, hi}, %1;\n\tcvt.rn.f16x2.e4m3x2 %0, hi;\n\t}" : "=r"(y) : "r"(x));
  return y;
}
__device__ __forceinline__ uint32_t prmt(uint32_t x, uint32_t sel) {
  uint32_t y;
  asm("prmt.b32 %0, %1, 0, %2;" : "=r"(y) : "r"(x), "r"(sel));
  return y;
}

// ROWS_: output rows a unit can have (T_m): 8, or 1 for MHA decode -- the MMA still spans
// 8 columns, but the fold buffer (and the epilogue's accumulator) only keep ROWS_ of them,
// which frees shared memory for a deeper ring.
template <int D_, int NST_, int WPS_, int ROWS_>
struct Fp8Engine {
  static constexpr int D = D_, NST = NST_, WPS = WPS_, NWG = NST, NCW = NWG * WPS;  // NWG: consumer warp sets
  static constexpr int WIN = LA_FP8_WIN > 0 ? LA_FP8_WIN : NST;  // stages in flight
  static_assert(ROWS_ == 1 || ROWS_ == 8, "fold rows");
  static_assert(D == 128, "an E4M3 row of d = 128 is exactly one 128-B swizzle span");
  static constexpr int STAGE_TOK = 128;           // = TMA box rows (32 KiB of K+V per stage)
  static constexpr int KV_BYTES = STAGE_TOK * 128;
  static constexpr int STAGE_BYTES = 2 * KV_BYTES;
  static constexpr int HEADS = ROWS_;             // fold-buffer rows (MMA N is 8 regardless)
  static constexpr int KS = D / 16;
  static constexpr int FOLD_FLOATS = NCW * HEADS * (D + 4);
  static constexpr int FOLD_BUFS = ROWS_ == 1 ? LA_FP8M_FB : LA_FP8_FB;
  static constexpr bool ZERO_RING = false;        // tail V rows are zeroed per warp
  using QElem = __nv_bfloat16;                    // bf16 q next to the E4M3 cache
  static constexpr bool QSTAGE = true;

  struct State {
    uint32_t qb[KS][2];  // Q^T B-fragments (f16, permuted contraction order, see above)
    float m[2], l[2];
    float o[KS][4];      // O^T: dims 16mm + 2gq (+1), rows 2tq, 2tq+1
    int lim[2];
  };

  __device__ __forceinline__ static void produce(unsigned char* dst, const DecodeArgs&, const TmapPair& tm, int64_t row,
                                                 int, uint64_t* bar, uint64_t pol) {
    mbar_arrive_expect_tx(bar, STAGE_BYTES);
    tma_load_2d(dst, &tm.k, 0, int(row), bar, pol);
    tma_load_2d(dst + KV_BYTES, &tm.v, 0, int(row), bar, pol);
  }

  // Paged: boxes of box_rows = min(128, page) rows inside one page; lane r issues load r.
  __device__ __forceinline__ static void produce_paged(unsigned char* dst, const DecodeArgs& a, const TmapPair& tm,
                                                       PageWin& pw, int s0, int ntok, uint64_t* bar, uint64_t pol,
                                                       int lane) {
    const int br = a.box_rows;
    const int nb = (ntok + br - 1) / br;
    if (lane == 0) mbar_arrive_expect_tx(bar, uint32_t(nb * br * 128 * 2));
    __syncwarp();
    const int rowl = int(pw.rows(s0 >> a.page_shift, s0 + lane * br, lane));  // whole warp: lane i -> box i
    if constexpr (LA_PAGED_ELECT) {
      #pragma unroll 1
      for (int i = 0; i < nb; ++i) {  // converged warp, one elected lane issues (warp-uniform operands)
        const int row = __shfl_sync(0xffffffffu, rowl, i);
        tma_load_2d_kv_elect(dst + i * br * 128, dst + KV_BYTES + i * br * 128, &tm.k, &tm.v, row, bar, pol);
      }
    } else if (lane < nb) {  // lane i: box i (<= 8), its K and V loads (one row coordinate for both)
      tma_load_2d(dst + lane * br * 128, &tm.k, 0, rowl, bar, pol);
      tma_load_2d(dst + KV_BYTES + lane * br * 128, &tm.v, 0, rowl, bar, pol);
    }
  }

  __device__ __forceinline__ static void seg_begin(State& s, const DecodeArgs& a, const DevUnit& u, int lane,
                                                   const void* qsrc) {  // qsrc: the unit's Q rows (smem)
    const int gq = lane >> 2, tq = lane & 3;
    const __nv_bfloat16* qrow = static_cast<const __nv_bfloat16*>(qsrc) + size_t(gq) * D;
    const bool ok = gq < u.rows;
#pragma unroll
    for (int kk = 0; kk < KS; ++kk) {  // b0 = Q[gq][16kk + 4tq, +1], b1 = Q[gq][16kk + 4tq + 2, +3]
      const uint2 w = ok ? *reinterpret_cast<const uint2*>(qrow + 16 * kk + 4 * tq) : make_uint2(0u, 0u);
      const float2 f01 = Mma<__nv_bfloat16>::unpack(w.x), f23 = Mma<__nv_bfloat16>::unpack(w.y);
      s.qb[kk][0] = Mma<__half>::pack(f01.x, f01.y);
      s.qb[kk][1] = Mma<__half>::pack(f23.x, f23.y);
    }
    s.m[0] = s.m[1] = -INFINITY;
    s.l[0] = s.l[1] = 0.f;
#pragma unroll
    for (int mm = 0; mm < KS; ++mm) s.o[mm][0] = s.o[mm][1] = s.o[mm][2] = s.o[mm][3] = 0.f;
#pragma unroll
    for (int e = 0; e < 2; ++e)
      s.lim[e] = a.causal ? u.len - u.nq + ((u.r0 + 2 * tq + e) % u.nq) + 1 : u.len;
  }

  __device__ __forceinline__ static void stage(State& s, unsigned char* st, int sub, int ntok, int tok0,
                                               float scale_log2, int lane, int /*bs*/) {
    for (int rb = sub * 32; rb < ntok; rb += 32 * WPS) round(s, st, rb, ntok, tok0, scale_log2, lane);
  }

  __device__ __forceinline__ static void round(State& s, unsigned char* st, int rb, int ntok, int tok0,
                                               float scale_log2, int lane) {
    const int gq = lane >> 2, mi = lane >> 3, ri = lane & 7;
    if (rb + 32 > ntok) {  // rows past the stage's tokens: zero this warp's V rows (codes may be NaN)
      for (int r = rb + (lane >> 3); r < rb + 32; r += 4)
        if (r >= ntok) *reinterpret_cast<uint4*>(st + KV_BYTES + r * 128 + (ri << 4)) = make_uint4(0u, 0u, 0u, 0u);
      __syncwarp();
    }
    const uint32_t kbase = smem_u32(st), vbase = smem_u32(st + KV_BYTES);
    // ---- S^T = K_f Q_f^T (Alg1§20): matrices (token half mi&1, 16-dim chunk 2kp + mi>>1) ---
    float sc[2][4];
#pragma unroll
    for (int blk = 0; blk < 2; ++blk) {
      sc[blk][0] = sc[blk][1] = sc[blk][2] = sc[blk][3] = 0.f;
      const int tok = rb + blk * 16 + ((mi & 1) << 3) + ri;
      const uint32_t ro = kbase + uint32_t(tok) * 128;
#pragma unroll
      for (int kp = 0; kp < KS / 2; ++kp) {
        uint32_t r[4];
        ldsm_x4(ro + (((2 * kp + (mi >> 1)) ^ (tok & 7)) << 4), r);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t af[4] = {e4m3x2_lo(r[2 * h]), e4m3x2_lo(r[2 * h + 1]), e4m3x2_hi(r[2 * h]),
                                  e4m3x2_hi(r[2 * h + 1])};
          Mma<__half>::run(sc[blk], af, s.qb[2 * kp + h][0], s.qb[2 * kp + h][1]);
        }
      }
    }
    // ---- scale, mask (C5, causal), running max per row (Alg1§21) ----------------------------
    float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int blk = 0; blk < 2; ++blk) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int tok = rb + blk * 16 + gq + ((e >> 1) << 3);
        const bool ok = tok < ntok && tok0 + tok < s.lim[e & 1];
        sc[blk][e] = ok ? sc[blk][e] * scale_log2 : -INFINITY;
        mx[e & 1] = fmaxf(mx[e & 1], sc[blk][e]);
      }
    }
#pragma unroll
    for (int off = 4; off <= 16; off <<= 1) {
      mx[0] = fmaxf(mx[0], __shfl_xor_sync(0xffffffffu, mx[0], off));
      mx[1] = fmaxf(mx[1], __shfl_xor_sync(0xffffffffu, mx[1], off));
    }
    if (__any_sync(0xffffffffu, (mx[0] > s.m[0]) || (mx[1] > s.m[1]))) {  // Alg1§23-24 rescale
      const float mn0 = fmaxf(s.m[0], mx[0]), mn1 = fmaxf(s.m[1], mx[1]);
      const float al0 = ex2_sub(s.m[0], mn0), al1 = ex2_sub(s.m[1], mn1);
      s.l[0] *= al0;
      s.l[1] *= al1;
#pragma unroll
      for (int mm = 0; mm < KS; ++mm) {
        s.o[mm][0] *= al0;
        s.o[mm][2] *= al0;
        s.o[mm][1] *= al1;
        s.o[mm][3] *= al1;
      }
      s.m[0] = mn0;
      s.m[1] = mn1;
    }
    // ---- P_f = exp(S_f - m) (Alg1§22); O^T += V^T P^T (Alg1§24) -----------------------------
#pragma unroll
    for (int blk = 0; blk < 2; ++blk) {
      const float p0 = ex2_sub(sc[blk][0], s.m[0]), p1 = ex2_sub(sc[blk][1], s.m[1]);
      const float p2 = ex2_sub(sc[blk][2], s.m[0]), p3 = ex2_sub(sc[blk][3], s.m[1]);
      s.l[0] += p0 + p2;
      s.l[1] += p1 + p3;
      // P in f16 (11-bit significand); P_lo carries the rest when LA_GQA_SPLITP (reading C18)
      const uint32_t h01 = Mma<__half>::pack(p0, p1), h23 = Mma<__half>::pack(p2, p3);
      const uint32_t b0 = movmatrix_t(h01), b1 = movmatrix_t(h23);
      uint32_t c0 = 0u, c1 = 0u;
      if (LA_FP8_SPLITP) {
        const float2 r01 = Mma<__half>::unpack(h01), r23 = Mma<__half>::unpack(h23);
        c0 = movmatrix_t(Mma<__half>::pack(p0 - r01.x, p1 - r01.y));
        c1 = movmatrix_t(Mma<__half>::pack(p2 - r23.x, p3 - r23.y));
      }
      const int tok = rb + blk * 16 + ((mi & 1) << 3) + ri;
      const uint32_t ro = vbase + uint32_t(tok) * 128;
#pragma unroll
      for (int mp = 0; mp < KS / 2; ++mp) {
        uint32_t r[4];
        ldsm_x4_t(ro + (((2 * mp + (mi >> 1)) ^ (tok & 7)) << 4), r);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          // bytes (t 2tq: dim 2gq, 2gq+1 | t 2tq+1: dim 2gq, 2gq+1) -> per dim: (t 2tq, t 2tq+1)
          const uint32_t x0 = prmt(r[2 * h], 0x3120u), x1 = prmt(r[2 * h + 1], 0x3120u);
          const uint32_t af[4] = {e4m3x2_lo(x0), e4m3x2_hi(x0), e4m3x2_lo(x1), e4m3x2_hi(x1)};
          Mma<__half>::run(s.o[2 * mp + h], af, b0, b1);
          if (LA_FP8_SPLITP) Mma<__half>::run(s.o[2 * mp + h], af, c0, c1);
        }
      }
    }
    if (rb + 32 > ntok) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic -> TMA WAR
  }

  __device__ __forceinline__ static void seg_end(State& s, float* fold, int warp, int lane) {
    const int gq = lane >> 2, tq = lane & 3;
#pragma unroll
    for (int off = 4; off <= 16; off <<= 1) {
      s.l[0] += __shfl_xor_sync(0xffffffffu, s.l[0], off);
      s.l[1] += __shfl_xor_sync(0xffffffffu, s.l[1], off);
    }
    float* fb = fold + warp * HEADS * (D + 4);  // [head][D + 4]
    const int h0 = 2 * tq, h1 = 2 * tq + 1;
    if (h0 < HEADS) {
#pragma unroll
      for (int mm = 0; mm < KS; ++mm)  // accumulator rows gq / gq + 8 = dims c / c + 1
        *reinterpret_cast<float2*>(fb + h0 * (D + 4) + 16 * mm + 2 * gq) = make_float2(s.o[mm][0], s.o[mm][2]);
      if (gq == 0) {
        fb[h0 * (D + 4) + D] = s.m[0];
        fb[h0 * (D + 4) + D + 1] = s.l[0];
      }
    }
    if (h1 < HEADS) {
#pragma unroll
      for (int mm = 0; mm < KS; ++mm)
        *reinterpret_cast<float2*>(fb + h1 * (D + 4) + 16 * mm + 2 * gq) = make_float2(s.o[mm][1], s.o[mm][3]);
      if (gq == 0) {
        fb[h1 * (D + 4) + D] = s.m[1];
        fb[h1 * (D + 4) + D + 1] = s.l[1];
      }
    }
  }
};

// =======================================================================================
// tcgen05 engine (T_m = 8, 16 or 32 q-rows of one KV head, bf16 / fp16, d = 128; BHSD, packed, paged): 5th-gen tensor
// cores with TMEM accumulators (option LA_ENGINE_TCGEN05)
// =======================================================================================
// One WARPGROUP per ring slot (WPS = 4: warp sub reads TMEM lanes 32 sub .. 32 sub + 31)
// takes every stage of 128 tokens that lands in its slot:
//   S^T[128 tok][16] = K_f Q_f^T      tcgen05.mma M=128 N=16 K=16 x 8, A = K (K-major, the
//                                     TMA 128-B swizzled box), B = Q (rows >= T_m zero)
//   thread t <- token t's 8 scores    tcgen05.ld 32x32b; mask (C5, causal), per-row max over
//                                     the warp (shuffles) and the warpgroup (smem, bar.sync)
//   P^T[16][128 tok] (bf16 / fp16)    rows 0-7 P_hi, rows 8-15 P_lo = p - P_hi (reading C18),
//                                     written MN-major SW128 over the stage's dead K tile
//   O^T[128 dim][16] = V_f^T P_f^T    tcgen05.mma M=128 N=16, A = V read MN-major from the
//                                     same TMA box (no transpose pass), B = P
//   thread t <- dim t's 16 columns    O_t[h] = alpha_h O_t[h] + O^T[t][h] + O^T[t][8 + h]
// Each slot owns 32 TMEM columns (S at +0, O-tile at +16), or 64 with LA_TC5_SPLIT = 2
// independent accumulator chains per contraction (summed after tcgen05.ld).  The per-tile O^T is a fresh
// accumulator that is re-scaled and summed in registers (Alg1§24-25), so the tensor core
// never needs the running max.
__device__ __forceinline__ float lds_f32(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
  return v;
}

__device__ __forceinline__ float4 lds_f32x4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a) : "memory");
  return v;
}

template <typename T>
__device__ __forceinline__ T to_kv(float x);
template <>
__device__ __forceinline__ __nv_bfloat16 to_kv<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }
template <>
__device__ __forceinline__ __half to_kv<__half>(float x) { return __float2half_rn(x); }
__device__ __forceinline__ float kv_to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
__device__ __forceinline__ float kv_to_f(__half x) { return __half2float(x); }

template <typename T, int NST_, int HEADS_, int NWG_ = NST_>
struct Tc5Engine {
  // NST ring slots of 128 tokens; NWG warpgroups take the stages round-robin (NWG < NST: a
  // warpgroup's next tile is already in flight while it computes)
  static constexpr int D = 128, NST = NST_, WPS = 4, NWG = NWG_, NCW = NWG * WPS;
  static constexpr int WIN_ = HEADS_ == 8 ? LA_TC5_WIN8 : HEADS_ == 16 ? LA_TC5_WIN16 : LA_TC5_WIN32;
  static constexpr int WIN = WIN_ > 0 ? WIN_ : NST;  // stages in flight
  // V of stage j waits until stage j - VWIN is consumed (VWIN < WIN: ~WIN - 1/2 stages in flight)
  static constexpr int VWIN_ = HEADS_ == 8 ? LA_TC5_VWIN8 : HEADS_ == 16 ? LA_TC5_VWIN16 : LA_TC5_VWIN32;
  static constexpr int VWIN = VWIN_ > 0 ? VWIN_ : WIN;
  static_assert(NWG <= NST && NST <= 8, "ring");
  static constexpr int STAGE_TOK = 128;             // = TMA box rows = MMA M
  static constexpr int BOX_HALVES = LA_TC5_BOXH;    // 128-B row halves per TMA box (16 or 32 KiB boxes)
  static constexpr int KV_BYTES = 2 * STAGE_TOK * 128;  // [half][128 rows][128 B]
  static constexpr int STAGE_BYTES = 2 * KV_BYTES;  // 64 KiB
  static constexpr int HEADS = HEADS_;              // T_m: 8, or 16 (the wider N of tcgen05: one KV pass
                                                    // for g * N_b <= 16 rows where mma.sync tiles need two)
  static_assert(HEADS == 8 || HEADS == 16 || HEADS == 32, "T_m");
  static constexpr int QR = HEADS < 16 ? 16 : HEADS;  // Q^T operand rows = S^T MMA N (>= 16)
  static constexpr int QHS = QR * 128;               // Q^T dim-half stride
  // 32 rows: the warp's running sum of row `lane` (a transpose-butterfly per stage); <= 16
  // rows: every thread keeps its token's share of each row's sum (r01 also tried per-thread
  // 32-row sums updated after the PV MMA: 1% slower, removed)
  // NWG < NST: a warpgroup's next stage sits in ANOTHER ring slot, so its PV MMA need not be
  // waited for at the end of a stage -- the warpgroup moves on, issues the next stage's S^T
  // MMA, and only then folds the previous O^T tile (both tensor-core round trips overlap the
  // other's work instead of adding up).  With NWG == NST the next stage's data cannot land
  // before this PV completes (same slot), so there is nothing to overlap.
  static constexpr bool OVERLAP = NWG < NST;
  static constexpr int LN = HEADS == 32 ? 1 : HEADS;
  static constexpr int NO = 2 * HEADS;              // O^T columns: P_hi rows, then P_lo rows
  static constexpr int FOLD_WPS = 1;                // one fold row set per slot (warpgroup)
  static constexpr int FOLD_FLOATS = NWG * HEADS * (D + 4);
  static constexpr int FOLD_BUFS = HEADS > 8 ? 1 : LA_TC5_FB8;
  static constexpr bool GLOBAL_FOLD = HEADS > 8;    // 16-row fold buffers (25 KB) do not fit next to the ring
  static constexpr bool ZERO_RING = false;          // tail V rows are zeroed per stage
  using QElem = T;
  // 8-row tiles: the producer stages each segment's Q rows in shared memory (2 KiB per queue
  // entry, a 2-deep queue fits next to the ring) so a warpgroup's segment start reads no global
  // memory; wider tiles read Q from global (no room next to their bigger per-warpgroup state)
  static constexpr bool QSTAGE = HEADS == 8 && LA_TC5_QSTAGE8;
  static constexpr int QD = QSTAGE ? 2 : 4;
  // accumulator chains per contraction (1 or 2).  LA_TC5_SPLIT = 2 applies to 8-row tiles only:
  // at 16 / 32 rows it fails a wide-tile parity test and measured slower (32 rows: 383 vs 368 us)
  static constexpr int SPLIT = HEADS == 8 ? LA_TC5_SPLIT : 1;
  static constexpr int OC = QR * SPLIT;             // first O^T column of a slot (S^T chains before it)
  static constexpr int COLS = (OC + NO * SPLIT) <= 32 ? 32 : (OC + NO * SPLIT) <= 64 ? 64 : 128;  // per slot
  static_assert(NWG * COLS <= 512, "TMEM columns");
  static constexpr int TMEM_COLS = NWG * COLS <= 32 ? 32 : NWG * COLS <= 64 ? 64 : NWG * COLS <= 128 ? 128 : NWG * COLS <= 256 ? 256 : 512;
  // extra smem per slot: Q^T operand [half][16 rows][128 B] (4 KiB, 1024-aligned), the
  // warpgroup's max exchange red[4][8] + l exchange red2[4][8], two MMA-completion barriers
  // per-slot extra: Q^T [2][QR][128 B], red [4][HEADS], red2 [4][HEADS], 3 barriers, mb [2][HEADS]
  static constexpr int RED_OFF = 2 * QHS, RED2_OFF = RED_OFF + 16 * HEADS, BAR_OFF = RED2_OFF + 16 * HEADS;
  static constexpr int MB_OFF = BAR_OFF + 32;
  static constexpr int AL_OFF = MB_OFF + 8 * HEADS;  // alpha_h = e^{m - m_new} of the current stage [HEADS]
  static constexpr int XS = (AL_OFF + 4 * HEADS + 1023) / 1024 * 1024;
  static constexpr int EXTRA_BYTES = NWG * XS + 1024;  // + the ring slots' V barriers [NST] and the TMEM base address
  static constexpr uint32_t IDESC_S = tc5::idesc_f16(std::is_same<T, __nv_bfloat16>::value, 128, QR, false, false);
  static constexpr uint32_t IDESC_O = tc5::idesc_f16(std::is_same<T, __nv_bfloat16>::value, 128, NO, true, true);

  struct State {
    float l[LN];               // HEADS <= 16: this token lane's share of every row's running sum;
                               // 32: the warp's running sum of row `lane` (transpose-butterfly)
    float o[HEADS];            // O~ of dim 32 sub + lane, every row
    int lbase, r0, nq;         // causal key limit of row h: lbase + (r0 + h) % nq (unit-local, exclusive)
    int mpar;                  // the running max m (uniform over the warpgroup) lives in shared memory,
                               // mb[mpar][row]; a stage writes the new m into mb[mpar ^ 1]
    int pend;                  // OVERLAP: barrier parity of this warpgroup's PV MMA still in flight (-1: none)
#ifdef LA_TC5_PROF
    long long pt[6];           // debug: cycles per stage phase, summed
    int pn;
#endif
  };

  __device__ __forceinline__ static unsigned char* extra() {
    extern __shared__ unsigned char smem_raw[];
    unsigned char* ring =
        reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    return ring + NST * STAGE_BYTES;
  }
  __device__ __forceinline__ static int slot_of_thread() { return int(threadIdx.x >> 5) / WPS; }
  __device__ __forceinline__ static uint32_t* tmem_base_ptr() { return reinterpret_cast<uint32_t*>(extra() + NWG * XS + 64); }
  __device__ __forceinline__ static uint64_t* vbar_of(int ring_slot) {  // V tile landed (expect_tx + TMA bytes)
    return reinterpret_cast<uint64_t*>(extra() + NWG * XS) + ring_slot;
  }
  __device__ __forceinline__ static void wg_bar(int slot) {  // the slot's 4 warps
    asm volatile("bar.sync %0, 128;" ::"r"(2 + slot) : "memory");
  }
  __device__ __forceinline__ static void init_barriers() {  // thread 0, before __syncthreads
    for (int s = 0; s < NWG; ++s) {
      uint64_t* b = reinterpret_cast<uint64_t*>(extra() + s * XS + BAR_OFF);
      mbar_init(&b[0], 1);  // S^T ready (tcgen05.commit)
      mbar_init(&b[1], 1);  // O^T tile ready (tcgen05.commit)
    }
    for (int s = 0; s < NST; ++s) mbar_init(vbar_of(s), 1);
  }

  // Whole producer warp: K on the full barrier, then (after stage j - VWIN is consumed: vwait)
  // V on the slot's barrier, each pair of half boxes issued by one elected lane.
  __device__ __forceinline__ static void produce_w(unsigned char* dst, const TmapPair& tm, int64_t row, uint64_t* bar,
                                                   uint64_t pol, int lane, uint64_t* vwait, uint32_t vpar) {
    static_assert(BOX_HALVES == 1, "half boxes");
    const int slot = int((dst - (extra() - NST * STAGE_BYTES)) / STAGE_BYTES);
    uint64_t* vbar = vbar_of(slot);
    if (lane == 0) mbar_arrive_expect_tx(bar, KV_BYTES);
    __syncwarp();
    tma_load_3d_halves_elect(dst, &tm.k, int(row), bar, pol);
    if (vwait) mbar_wait(vwait, vpar);
    if (lane == 0) mbar_arrive_expect_tx(vbar, KV_BYTES);
    __syncwarp();
    tma_load_3d_halves_elect(dst + KV_BYTES, &tm.v, int(row), vbar, pol);
  }
  __device__ __forceinline__ static void produce_k(unsigned char* dst, const TmapPair& tm, int64_t row, uint64_t* bar,
                                                   uint64_t pol) {
    mbar_arrive_expect_tx(bar, KV_BYTES);
#pragma unroll
    for (int h = 0; h < 2 / BOX_HALVES; ++h) tma_load_3d(dst + h * 16384, &tm.k, 0, int(row), h, bar, pol);
  }
  __device__ __forceinline__ static void produce_v(unsigned char* dst, const TmapPair& tm, int64_t row, uint64_t pol) {
    const int slot = int((dst - (extra() - NST * STAGE_BYTES)) / STAGE_BYTES);
    uint64_t* vbar = vbar_of(slot);
    mbar_arrive_expect_tx(vbar, KV_BYTES);
#pragma unroll
    for (int h = 0; h < 2 / BOX_HALVES; ++h) tma_load_3d(dst + KV_BYTES + h * 16384, &tm.v, 0, int(row), h, vbar, pol);
  }
  __device__ __forceinline__ static void produce(unsigned char* dst, const DecodeArgs&, const TmapPair& tm, int64_t row,
                                                 int, uint64_t* bar, uint64_t pol) {
    // K on the ring's full barrier, V on the slot's own barrier: S^T, the softmax and P
    // overlap the V transfer (full boxes; rows past the tensor are zero-filled)
    const int slot = int((dst - (extra() - NST * STAGE_BYTES)) / STAGE_BYTES);
    uint64_t* vbar = vbar_of(slot);
    mbar_arrive_expect_tx(bar, KV_BYTES);
    mbar_arrive_expect_tx(vbar, KV_BYTES);
#pragma unroll
    for (int h = 0; h < 2 / BOX_HALVES; ++h) tma_load_3d(dst + h * 16384, &tm.k, 0, int(row), h, bar, pol);
#pragma unroll
    for (int h = 0; h < 2 / BOX_HALVES; ++h) tma_load_3d(dst + KV_BYTES + h * 16384, &tm.v, 0, int(row), h, vbar, pol);
  }
  // Paged KV: boxes of box_rows = min(128, page) rows of ONE 128-B half, each inside one
  // page, placed so the stage keeps the [half][128 rows][128 B] operand layout; lane r issues
  // load r = (box i, half, K or V).
  __device__ __forceinline__ static void produce_paged(unsigned char* dst, const DecodeArgs& a, const TmapPair& tm,
                                                       PageWin& pw, int s0, int ntok, uint64_t* bar, uint64_t pol,
                                                       int lane) {
    const int br = a.box_rows;
    const int nb = (ntok + br - 1) / br;
    const int slot = int((dst - (extra() - NST * STAGE_BYTES)) / STAGE_BYTES);
    uint64_t* vbar = vbar_of(slot);
    if (lane == 0) {
      mbar_arrive_expect_tx(bar, uint32_t(nb * br * 128 * 2));
      mbar_arrive_expect_tx(vbar, uint32_t(nb * br * 128 * 2));
    }
    __syncwarp();
    const int rowl = int(pw.rows(s0 >> a.page_shift, s0 + lane * br, lane));  // whole warp: lane i -> box i
    if constexpr (LA_PAGED_ELECT) {
      #pragma unroll 1
      for (int i = 0; i < nb; ++i) {  // converged warp, one elected lane issues (warp-uniform operands)
        const int row = __shfl_sync(0xffffffffu, rowl, i);
#pragma unroll
        for (int half = 0; half < 2; ++half)
          tma_load_3d_kv_elect(dst + half * 16384 + i * br * 128, dst + KV_BYTES + half * 16384 + i * br * 128, &tm.k,
                               &tm.v, row, half, bar, vbar, pol);
      }
    } else if (lane < nb) {  // lane i: box i (<= 8), both halves of its K and V
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        tma_load_3d(dst + half * 16384 + lane * br * 128, &tm.k, 0, rowl, half, bar, pol);
        tma_load_3d(dst + KV_BYTES + half * 16384 + lane * br * 128, &tm.v, 0, rowl, half, vbar, pol);
      }
    }
  }

  __device__ __forceinline__ static void seg_begin(State& s, const DecodeArgs& a, const DevUnit& u, int lane,
                                                   const void* qsrc) {  // qsrc: the unit's Q rows (global)
    const int slot = slot_of_thread(), tid = (int(threadIdx.x >> 5) % WPS) * 32 + lane;
    unsigned char* qs = extra() + slot * XS;
    // Q^T operand, K-major 128-B swizzle: row r (q-row of the tile, zero past u.rows),
    // dims 64 half .. 64 half + 63 in the 128-B line (half * QHS + r * 128)
#pragma unroll
    for (int i = 0; i < QR / 8; ++i) {
      const int c = tid + 128 * i, r = c >> 4, ch = c & 15, half = ch >> 3, cc = ch & 7;
      uint4 w = make_uint4(0u, 0u, 0u, 0u);
      if (r < u.rows) w = *reinterpret_cast<const uint4*>(static_cast<const T*>(qsrc) + size_t(r) * D + 8 * ch);
      *reinterpret_cast<uint4*>(qs + half * QHS + r * 128 + ((cc ^ (r & 7)) << 4)) = w;
    }
#pragma unroll
    for (int h = 0; h < HEADS; ++h) s.o[h] = 0.f;
#pragma unroll
    for (int h = 0; h < LN; ++h) s.l[h] = 0.f;
    if (tid < 2 * HEADS) reinterpret_cast<float*>(qs + MB_OFF)[tid] = -INFINITY;
    s.mpar = 0;
    s.pend = -1;
#ifdef LA_TC5_PROF
    for (int i = 0; i < 6; ++i) s.pt[i] = 0;
    s.pn = 0;
#endif
    s.lbase = a.causal ? u.len - u.nq + 1 : u.len;  // N_q > 1, causal: query i is token n - N_b + i
    s.r0 = u.r0;
    s.nq = a.causal ? u.nq : 1;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // Q writes -> tensor core
    wg_bar(slot);
  }

  __device__ __forceinline__ static void stage(State& s, unsigned char* st, int sub, int ntok, int tok0,
                                               float scale_log2, int lane, int /*bs*/, uint32_t par, uint64_t* empty) {
    const int slot = slot_of_thread(), tid = sub * 32 + lane;
    unsigned char* xs = extra() + slot * XS;
    float* red = reinterpret_cast<float*>(xs + RED_OFF);  // [4][HEADS]
    uint64_t* bars = reinterpret_cast<uint64_t*>(xs + BAR_OFF);
    const uint32_t tbase = *tmem_base_ptr() + uint32_t(COLS * slot);
    const uint32_t tlane = uint32_t(32 * sub) << 16;
    const uint32_t kaddr = smem_u32(st), vaddr = smem_u32(st + KV_BYTES), qaddr = smem_u32(xs);
    const uint32_t rpar = par & 1u, wpar = par >> 1;  // ring slot's / warpgroup's barrier parity
    uint64_t* vbar = vbar_of(int((st - (extra() - NST * STAGE_BYTES)) / STAGE_BYTES));
#ifdef LA_TC5_PROF
    long long ck[6];
    ck[0] = clock64();
#define TC5_CK(i) ck[i] = clock64()
#else
#define TC5_CK(i)
#endif
    // ---- S^T = K_f Q_f^T (Alg1§20) -----------------------------------------------------------
    if (SPLIT == 1 && LA_TC5_MMA8) {
      if (sub == 0) {  // warp 0, converged: one elected lane issues (operands stay warp-uniform)
        tc5::fence_after();
        constexpr int Q = QHS / 16;  // k-step kk: K at (kk >> 2) 16 KiB + (kk & 3) 32 B, Q^T likewise
        tc5::mma8_f16<2, 4, 6, 1024, 1026, 1028, 1030, 2, 4, 6, Q, Q + 2, Q + 4, Q + 6>(
            tbase, tc5::sdesc(kaddr, 16, 1024), tc5::sdesc(qaddr, 16, 1024), IDESC_S);
        tc5::commit_elect(&bars[0]);
      }
    } else if (tid == 0) {
      tc5::fence_after();
      {
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {  // chain c = kk / (8 / SPLIT) accumulates in columns 16 c
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          const int c = kk / (8 / SPLIT);
          tc5::mma_f16(tbase + QR * c, tc5::sdesc(kaddr + off, 16, 1024),
                       tc5::sdesc(qaddr + (kk >> 2) * QHS + (kk & 3) * 32, 16, 1024), IDESC_S, kk % (8 / SPLIT) > 0);
        }
      }
      tc5::commit(&bars[0]);
    }
    if (ntok < STAGE_TOK) {  // rows past the stage's tokens: zero V once it landed (may be non-finite)
      mbar_wait(vbar, rpar);
      if (tid >= ntok)
#pragma unroll
        for (int hf = 0; hf < 2; ++hf)
#pragma unroll
          for (int c = 0; c < 8; ++c)
            *reinterpret_cast<uint4*>(st + KV_BYTES + hf * 16384 + tid * 128 + (c << 4)) = make_uint4(0u, 0u, 0u, 0u);
    }
    if constexpr (OVERLAP) {  // the previous stage's O^T tile, while this stage's S^T MMA runs
      if (s.pend >= 0) finish_o(s, sub, lane, uint32_t(s.pend));
    }
    TC5_CK(1);
    mbar_wait(&bars[0], wpar);
    tc5::fence_after();
    TC5_CK(2);
    float sc[QR];
    if constexpr (QR == 32 && SPLIT == 1 && LA_TC5_LD32) {  // one TMEM round trip for the 32 columns
      tc5::ld32(tbase + tlane, sc);
    } else
#pragma unroll
    for (int c = 0; c < QR; c += 16) {
      float t16[16];
      tc5::ld16(tbase + tlane + c, t16);
#pragma unroll
      for (int i = 0; i < 16; ++i) sc[c + i] = t16[i];
      if (SPLIT == 2) {
        tc5::ld16(tbase + tlane + QR + c, t16);
#pragma unroll
        for (int i = 0; i < 16; ++i) sc[c + i] += t16[i];
      }
    }
    // ---- scale, mask (C5, causal), running max per row (Alg1§21) ----------------------------
    float mx[HEADS];
    if (tid < ntok && tok0 + STAGE_TOK <= s.lbase) {  // the common stage: no key of it is masked
#pragma unroll
      for (int h = 0; h < HEADS; ++h) mx[h] = sc[h] = sc[h] * scale_log2;
    } else {  // the stage reaches past the smallest causal limit (or the context end): per-row test,
              // row h's limit lbase + (r0 + h) mod nq stepped without a division per row
      const int t = tok0 + tid;
      int r = s.r0 % s.nq;
#pragma unroll
      for (int h = 0; h < HEADS; ++h) {
        const bool ok = tid < ntok && t < s.lbase + r;
        mx[h] = sc[h] = ok ? sc[h] * scale_log2 : -INFINITY;
        r = r + 1 == s.nq ? 0 : r + 1;
      }
    }
#pragma unroll
    for (int h = 0; h < HEADS; ++h)  // warp max: one CREDUX per row (sm_100a f32 redux)
      asm volatile("redux.sync.max.f32 %0, %0, 0xffffffff;" : "+f"(mx[h]));
    if (lane == 0)  // every lane holds every row's warp max: one lane stores them, 16 B at a time
#pragma unroll
      for (int h = 0; h < HEADS; h += 4)
        *reinterpret_cast<float4*>(red + sub * HEADS + h) = make_float4(mx[h], mx[h + 1], mx[h + 2], mx[h + 3]);
    wg_bar(slot);
    TC5_CK(3);
    const uint32_t mcur = smem_u32(xs + MB_OFF) + 4 * HEADS * s.mpar, mnext = smem_u32(xs + MB_OFF) + 4 * HEADS * (s.mpar ^ 1);
    const uint32_t alp = smem_u32(xs + AL_OFF);
    // lane r < HEADS of every warp: row r's m_new (Alg1§21) and alpha = e^{m - m_new}; every
    // thread then takes them by shuffles (one lane's loads per row instead of every thread
    // re-reading all rows' maxima); warp 0 also stores them for the O update and the next stage
    float mrow_l = 0.f, al_l = 0.f;
    if (lane < HEADS) {
      const uint32_t rl = smem_u32(red) + 4 * lane;
      const float mo = lds_f32(mcur + 4 * lane);
      mrow_l = fmaxf(mo, fmaxf(fmaxf(lds_f32(rl), lds_f32(rl + 4 * HEADS)),
                               fmaxf(lds_f32(rl + 8 * HEADS), lds_f32(rl + 12 * HEADS))));
      al_l = ex2_sub(mo, mrow_l);
      if (sub == 0) {
        asm volatile("st.shared.f32 [%0], %1;" ::"r"(mnext + 4 * lane), "f"(mrow_l) : "memory");
        asm volatile("st.shared.f32 [%0], %1;" ::"r"(alp + 4 * lane), "f"(al_l) : "memory");
      }
    }
    // ---- P_f = exp(S_f - m_new) (Alg1§22) --------------------------------------------------
#pragma unroll
    for (int h = 0; h < HEADS; ++h) {
      const float p = ex2_sub(sc[h], __shfl_sync(0xffffffffu, mrow_l, h));
      if constexpr (HEADS < 32) s.l[h] = fmaf(__shfl_sync(0xffffffffu, al_l, h), s.l[h], p);  // Alg1§23
      sc[h] = p;
    }
    // P^T MN-major: token t's 2 HEADS columns (P_hi rows, then P_lo rows) in one 128-B swizzled
    // line over the dead K tile -> 2 HEADS / 8 16-B stores per thread (the B-operand layout
    // scripts/tc5_probe.cu checks exactly)
    {
      unsigned char* pl = st + tid * 128;
#pragma unroll
      for (int j = 0; j < HEADS / 8; ++j) {
        uint32_t hw[4], lw[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float p0 = sc[8 * j + 2 * e], p1 = sc[8 * j + 2 * e + 1];
          hw[e] = Mma<T>::pack(p0, p1);
          const float2 r = Mma<T>::unpack(hw[e]);
          lw[e] = Mma<T>::pack(p0 - r.x, p1 - r.y);
        }
        *reinterpret_cast<uint4*>(pl + ((j ^ (tid & 7)) << 4)) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
        *reinterpret_cast<uint4*>(pl + (((HEADS / 8 + j) ^ (tid & 7)) << 4)) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
      }
    }
    if constexpr (HEADS == 32) {  // Alg1§23 for 32 rows: XOR transpose-butterfly of the 32 p's
      // (31 shuffles) leaves the warp's sum of row `lane` in sc[0] of lane `lane`
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) {
        const bool up = (lane & off) != 0;
#pragma unroll
        for (int j = 0; j < off; ++j) {
          const float keep = up ? sc[j + off] : sc[j], send = up ? sc[j] : sc[j + off];
          sc[j] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
      }
      s.l[0] = fmaf(al_l, s.l[0], sc[0]);  // lane = row: its own alpha
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // P (+ zeroed V) -> tensor core
    tc5::fence_before();                                           // S loads done before reuse
    wg_bar(slot);
    TC5_CK(4);
    // ---- O^T_tile = V_f^T P_f^T (Alg1§24) ----------------------------------------------------
    if (SPLIT == 1 && LA_TC5_MMA8) {
      if (sub == 0) {  // warp 0, converged: one elected lane issues
        mbar_wait(vbar, rpar);  // V landed
        tc5::fence_after();     // k-step kk: 16 tokens = 2 KiB further in V and in P^T
        tc5::mma8_f16<128, 256, 384, 512, 640, 768, 896, 128, 256, 384, 512, 640, 768, 896>(
            tbase + OC, tc5::sdesc(vaddr, 16384, 1024), tc5::sdesc(kaddr, 8192, 1024), IDESC_O);
        tc5::commit_elect(empty);     // the slot is free the moment the tensor core is done with it
        tc5::commit_elect(&bars[1]);
      } else if (lane == 0) {
        mbar_arrive(empty);     // this warp no longer touches the slot's shared memory
      }
    } else if (tid == 0) {
      mbar_wait(vbar, rpar);  // V landed
      tc5::fence_after();
      {
#pragma unroll
        for (int kk = 0; kk < STAGE_TOK / 16; ++kk)
          tc5::mma_f16(tbase + OC + NO * (kk / (8 / SPLIT)), tc5::sdesc(vaddr + kk * 2048, 16384, 1024),
                       tc5::sdesc(kaddr + kk * 2048, 8192, 1024),  // MN-major P^T: 16 token lines per k-step
                       IDESC_O, kk % (8 / SPLIT) > 0);
      }
      tc5::commit(empty);     // the slot is free the moment the tensor core is done with it
      tc5::commit(&bars[1]);
    } else if (sub != 0 && lane == 0) {
      mbar_arrive(empty);     // this warp no longer touches the slot's shared memory
    }
    if constexpr (OVERLAP) {
      s.pend = int(wpar);     // folded by the next stage (or seg_end)
    } else {
      finish_o(s, sub, lane, wpar);
    }
    s.mpar ^= 1;
#ifdef LA_TC5_PROF
    ck[5] = clock64();
    for (int i = 0; i < 5; ++i) s.pt[i] += ck[i + 1] - ck[i];
    ++s.pn;
#endif
#undef TC5_CK
  }

  // O~ += the stage's O^T tile with the stage's alpha (Alg1§24-25): wait for its PV MMA (barrier
  // parity wpar), read the tile from TMEM, fold.  Must precede the next softmax's alpha writes.
  __device__ __forceinline__ static void finish_o(State& s, int sub, int lane, uint32_t wpar) {
    const int slot = slot_of_thread();
    unsigned char* xs = extra() + slot * XS;
    uint64_t* bars = reinterpret_cast<uint64_t*>(xs + BAR_OFF);
    const uint32_t tbase = *tmem_base_ptr() + uint32_t(COLS * slot);
    const uint32_t tlane = uint32_t(32 * sub) << 16;
    const uint32_t alp = smem_u32(xs + AL_OFF);
    mbar_wait(&bars[1], wpar);
    tc5::fence_after();
    // alpha from shared memory, 8 rows at a time (no registers held across the MMA)
    // O^T tile: column h = V^T P_hi row h, column HEADS + h = V^T P_lo row h (per chain)
    if constexpr (HEADS >= 16 && SPLIT == 1 && LA_TC5_LD32) {  // 32-column loads: 1 (16 rows) / 2 (32 rows)
      // TMEM round trips instead of 4 / 8; o[h] = alpha_h o[h] + (hi_h + lo_h) as below
#pragma unroll
      for (int c0 = 0; c0 < HEADS; c0 += 16) {
        float hl[32];
        if constexpr (HEADS == 16) {
          tc5::ld32(tbase + tlane + OC, hl);  // hi 0-15, lo 16-31
        } else {                            // rows c0 .. c0 + 15: hi columns c0.., lo columns 32 + c0..
          float t16[16];
          tc5::ld16(tbase + tlane + OC + c0, t16);
#pragma unroll
          for (int i = 0; i < 16; ++i) hl[i] = t16[i];
          tc5::ld16(tbase + tlane + OC + HEADS + c0, t16);
#pragma unroll
          for (int i = 0; i < 16; ++i) hl[16 + i] = t16[i];
        }
#pragma unroll
        for (int q = 0; q < 16; q += 4) {
          const float4 a = lds_f32x4(alp + 4 * (c0 + q));
          const float al[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
          for (int i = 0; i < 4; ++i) s.o[c0 + q + i] = fmaf(al[i], s.o[c0 + q + i], hl[q + i] + hl[16 + q + i]);
        }
      }
      tc5::fence_before();
      return;
    }
#pragma unroll
    for (int c0 = 0; c0 < HEADS; c0 += 8) {  // 8 rows at a time: hi columns c0.., lo columns HEADS + c0..
      float hv[8], lv[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) hv[i] = lv[i] = 0.f;
#pragma unroll
      for (int ch = 0; ch < SPLIT; ++ch) {
        float a16[16];
        if (HEADS == 8) {  // 16 columns: hi 0-7, lo 8-15
          tc5::ld16(tbase + tlane + OC + NO * ch, a16);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            hv[i] += a16[i];
            lv[i] += a16[8 + i];
          }
        } else {           // 32 columns: hi 0-15, lo 16-31; this pass takes rows c0 .. c0 + 7
          tc5::ld8(tbase + tlane + OC + NO * ch + c0, hv, ch > 0);
          tc5::ld8(tbase + tlane + OC + NO * ch + HEADS + c0, lv, ch > 0);
        }
      }
      const float4 a0 = lds_f32x4(alp + 4 * c0), a1 = lds_f32x4(alp + 4 * c0 + 16);
      const float al[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
#pragma unroll
      for (int i = 0; i < 8; ++i) s.o[c0 + i] = fmaf(al[i], s.o[c0 + i], hv[i] + lv[i]);  // Alg1§25
    }
    tc5::fence_before();
  }

  __device__ __forceinline__ static void seg_end(State& s, float* fold, int warp, int lane) {
    const int slot = warp / WPS, sub = warp % WPS;
    if constexpr (OVERLAP) {  // the segment's last O^T tile
      if (s.pend >= 0) finish_o(s, sub, lane, uint32_t(s.pend));
      s.pend = -1;
    }
#ifdef LA_TC5_PROF
    if (sub == 0 && lane == 0 && blockIdx.x % 37 == 0 && s.pn > 8)
      printf("TC5PROF cta %d wg %d H %d stages %d: [S-issue..finish_o] %lld [S wait] %lld [ld+mask+redux+bar] %lld "
             "[alpha+P+bar] %lld [PV issue..end] %lld cycles/stage\n", int(blockIdx.x), slot, HEADS, s.pn,
             s.pt[0] / s.pn, s.pt[1] / s.pn, s.pt[2] / s.pn, s.pt[3] / s.pn, s.pt[4] / s.pn);
#endif
    float* red2 = reinterpret_cast<float*>(extra() + slot * XS + RED2_OFF);  // [4][HEADS]
    float* fb = fold + slot * HEADS * (D + 4);                                  // [row][D + 4]
#pragma unroll
    for (int h = 0; h < HEADS; ++h) fb[h * (D + 4) + 32 * sub + lane] = s.o[h];
    if constexpr (HEADS == 32) {
      red2[sub * HEADS + lane] = s.l[0];  // lane = row
    } else {
#pragma unroll
      for (int h = 0; h < HEADS; ++h) {
        float l = s.l[h];
#pragma unroll
        for (int off = 16; off; off >>= 1) l += __shfl_xor_sync(0xffffffffu, l, off);
        if (lane == h) red2[sub * HEADS + h] = l;
      }
    }
    // read m before the barrier: past it, the next segment's seg_begin resets mb
    const float mv = lane < HEADS ? reinterpret_cast<const float*>(extra() + slot * XS + MB_OFF)[HEADS * s.mpar + lane]
                                  : 0.f;
    wg_bar(slot);
    if (sub == 0 && lane < HEADS) {
      const int h = lane;
      fb[h * (D + 4) + D] = mv;
      fb[h * (D + 4) + D + 1] = (red2[h] + red2[HEADS + h]) + (red2[2 * HEADS + h] + red2[3 * HEADS + h]);
    }
  }

};

// =======================================================================================
// The persistent decode kernel
// =======================================================================================
// depth of the producer -> consumer virtual-CTA queue: EngX<E>::QD (4; the tcgen05 8-row
// engine stages its segments' Q rows in shared memory with a 2-deep queue)
constexpr int kClaimAhead = 4;  // dynamic: LeanTiles before a piece's end at which the next claim is taken

// One segment (one LeanTile() call, Alg2§11-18) handed from the producer to the consumer
// warps through shared memory, with its unit record: the consumers never read the schedule
// tables or Q from global memory (those dependent loads stalled every segment start).
struct alignas(16) SegQ {
  DevUnit u;
  int v, unit, it, it_end, host, finishing, pad_[2];
};

struct SegInfo {
  int v, unit, host, finishing;
  int s0;    // ring slot of the segment's first stage
  int jend;  // stages consumed by the CTA once this segment is done
};

// Engines with tcgen05 state (Tc5Engine) declare TMEM columns, an extra smem region after
// the ring and fewer fold rows per slot; the others get the neutral values.
template <class E, class = void>
struct EngX {
  static constexpr int TMEM = 0, EXTRA = 0, FW = E::WPS, VWIN = 1 << 20, QD = 4, NEP = 1;
  static constexpr bool GF = false;  // fold buffers in global scratch (DecodeArgs::gfold)
};
template <class E>
struct EngX<E, std::void_t<decltype(E::TMEM_COLS)>> {
  static constexpr int TMEM = E::TMEM_COLS, EXTRA = E::EXTRA_BYTES, FW = E::FOLD_WPS, VWIN = E::VWIN, QD = E::QD;
  static constexpr bool GF = E::GLOBAL_FOLD;
  // epilogue warps: one for 8-row tiles, else the 8-row groups split over NEP warps
  static constexpr int NEP = E::HEADS == 8 ? 1 : E::HEADS == 16 ? LA_WIDE_NEP16 : LA_WIDE_NEP32;
  static_assert(E::HEADS % (8 * NEP) == 0, "whole row groups per epilogue warp");
};

template <class E>
struct Smem {
  static constexpr int RING = E::NST * E::STAGE_BYTES;
  static constexpr int EXTRA = EngX<E>::EXTRA;  // engine state right after the ring
  static constexpr int kFB = E::FOLD_BUFS;  // consumer -> epilogue fold buffers
  static constexpr int FOLD = EngX<E>::GF ? 0 : kFB * E::FOLD_FLOATS * 4;
  static constexpr int kQD = EngX<E>::QD;
  static constexpr int BARS = (2 * E::NST + 2 * kQD + 4 * kFB + 1) * 8;
  // segment queue, hand-off records, prod_j; then the segments' Q rows (TMA bulk copies)
  static constexpr int SQ_OFF = (RING + EXTRA + FOLD + BARS + 15) / 16 * 16;
  static constexpr int MISC = kQD * int(sizeof(SegQ)) + kFB * int(sizeof(SegInfo)) + 32 + 32 * 8 * 4;  // + prod_j, fold weights (16-B aligned)
  static constexpr int QB = E::QSTAGE ? (E::HEADS * E::D * int(sizeof(typename E::QElem)) + 127) / 128 * 128 : 0;
  static constexpr int QB_OFF = (SQ_OFF + MISC + 127) / 128 * 128;
  static constexpr int BYTES = 1024 + QB_OFF + kQD * QB;
};

// The epilogue warp's accumulator for one segment: lane owns dims J lane .. J lane + J - 1 of
// every head h (one 16-B / 8-B vector per row); the fold buffer layout is [warp][head][D + 4]
// = O[D], m, l, pad for every engine.
template <int J>
__device__ __forceinline__ void ldv(const float* p, float (&x)[J]) {
  if constexpr (J == 4) {
    const float4 t = *reinterpret_cast<const float4*>(p);
    x[0] = t.x; x[1] = t.y; x[2] = t.z; x[3] = t.w;
  } else {
    static_assert(J == 2, "J");
    const float2 t = *reinterpret_cast<const float2*>(p);
    x[0] = t.x; x[1] = t.y;
  }
}
template <int J>
__device__ __forceinline__ void ldv_cg(const float* p, float (&x)[J]) {  // L1-bypassing (acquired data)
  if constexpr (J == 4) {
    const float4 t = __ldcg(reinterpret_cast<const float4*>(p));
    x[0] = t.x; x[1] = t.y; x[2] = t.z; x[3] = t.w;
  } else {
    const float2 t = __ldcg(reinterpret_cast<const float2*>(p));
    x[0] = t.x; x[1] = t.y;
  }
}
template <int J>
__device__ __forceinline__ void stv(float* p, const float (&x)[J], float scale = 1.f) {
  if constexpr (J == 4)
    *reinterpret_cast<float4*>(p) = make_float4(x[0] * scale, x[1] * scale, x[2] * scale, x[3] * scale);
  else
    *reinterpret_cast<float2*>(p) = make_float2(x[0] * scale, x[1] * scale);
}
template <class E>
struct EpiAcc {
  static constexpr int H = E::HEADS, D = E::D, J = E::D / 32;
  float o[H][J], m[H], l[H];
};

// =======================================================================================
// Epilogue of the 16 / 32-row tcgen05 tiles (static schedules): the same fixup as the kernel's
// epilogue below, but every step runs in groups of 8 rows whose accumulator lives in
// registers.  A 32-row accumulator does not fit the register file; spilled to local memory it
// thrashes the L1 (nearly all carved out as shared memory), and the last segment's fold +
// write at a CTA's end took ~25 us (r02 trace).
// =======================================================================================
template <class E>
__device__ __forceinline__ void wide_epilogue(const DecodeArgs& a, const TmapPair&, unsigned char* ring, float* fold,
                                              uint64_t* fold_full, uint64_t* fold_empty, uint64_t* stage_bar,
                                              const SegInfo* seginfo, int* prod_j, uint32_t epoch,
                                              uint32_t xepoch, unsigned long long* tr, int lane, int e) {
  constexpr int NWG = E::NWG, D = E::D, H = E::HEADS, J = D / 32, RG = 8, RS = D + 4;
  constexpr int FW = EngX<E>::FW, kFB = E::FOLD_BUFS, FOLD_FLOATS = E::FOLD_FLOATS;
  // NEP epilogue warps: warp e owns rows [e RW, e RW + RW) of every segment (whole 8-row
  // groups, each folded in the same order as by one warp: the bits do not depend on NEP).
  // Warp 0 alone stages, waits on the peers' flags, signals, exchanges and counts out.
  constexpr int NEP = EngX<E>::NEP, RW = H / NEP;
  static_assert(H % RG == 0 && RW % RG == 0, "row groups");
  static_assert((FOLD_FLOATS * 4) % 16 == 0, "fold buffer: whole 16-B units for one bulk copy");
  auto epi_sync = [&]() {  // the NEP epilogue warps (named barrier 15; the consumers use 1 .. 2 + NST)
    if constexpr (NEP > 1) asm volatile("bar.sync 15, %0;" ::"n"(NEP * 32) : "memory");
  };
  volatile int* epi_flags = prod_j + 1;  // warp 0 -> warps 1 .. NEP-1: this segment's idle / stage_peers
  float o[RG][J], m[RG], l[RG];
  uint32_t stage_ph = 0;
  int nr = 0;
  #pragma unroll 1
  for (int seg = 0;; ++seg) {
    const int b = seg % kFB;
    mbar_wait(&fold_full[b], (seg / kFB) & 1);
    const SegInfo si = seginfo[b];
    if (si.unit < 0) break;
#ifndef LA_PROF
    if (e == 0 && tr && lane == 0) tr[TR_STREAM] = globaltimer();  // the consumers finished this segment
#endif
    const DevUnit u = a.units[si.unit];
    const int v = si.v;
    nr = u.rows;
    const bool out = si.host && si.finishing;  // one CTA computed the whole unit (Alg2§38-39)
    const bool host_wait = si.host && !si.finishing;
    // The CTA's last segment (its producer has issued every stage, all consumed): the ring is
    // idle, so the segment's warp partials (global fold buffer) and, for a waiting host, all
    // of its peers' partial rows and (m, l) are staged there by bulk copies -- ONE L2 round
    // trip each instead of three dependent ones per 8-row group (the 32-row host fold took
    // ~13 us that way, on the kernel's critical path).  The arithmetic is unchanged: only
    // where the operands are read from differs, so results stay bitwise identical.
    const int np = host_wait ? u.last_cta - v : 0;
    float* fstg = reinterpret_cast<float*>(ring);         // [FOLD_FLOATS]
    float* pml = fstg + FOLD_FLOATS;                       // [np][nr][4]  peers' (m, l, -, -)
    float* prow = pml + size_t(np) * nr * 4;               // [np][nr][D]  peers' O~ rows
    bool idle = false, stage_peers = false;
    if (e == 0) {
      idle = *reinterpret_cast<volatile const int*>(prod_j) == si.jend;
      stage_peers = idle && host_wait && FOLD_FLOATS * 4 + size_t(np) * nr * (D + 4) * 4 <= size_t(Smem<E>::RING);
      if (idle) {
        asm volatile("fence.proxy.async.global;" ::: "memory");      // consumers' fold-buffer stores -> TMA
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the ring's last generic reads
        __syncwarp();
        if (lane == 0) {
          mbar_arrive_expect_tx(stage_bar, uint32_t(FOLD_FLOATS) * 4);
          bulk_g2s_plain(fstg, fold + b * FOLD_FLOATS, uint32_t(FOLD_FLOATS) * 4, stage_bar);
        }
      }
      if (host_wait) {  // Wait(flags[cta]) for cta = g+1 .. last_cta (Alg2§26-28, reading C9)
        if (tr && lane == 0) tr[TR_WAIT0] = globaltimer();
        #pragma unroll 1
        for (int p = v + 1 + lane; p <= u.last_cta; p += 32) {
          const unsigned long long t0 = globaltimer();
          while (ld_acquire_gpu(&a.flags[p]) != epoch) {
            __nanosleep(20);
            if (globaltimer() - t0 > kWaitTimeoutNs || *reinterpret_cast<volatile int*>(&a.counters[CTR_ERROR])) {
              atomicExch(&a.counters[CTR_ERROR], 1);
              break;
            }
          }
        }
        __syncwarp();
        if (tr && lane == 0) tr[TR_WAIT1] = globaltimer();
        asm volatile("fence.proxy.async.global;" ::: "memory");  // acquired partials -> TMA
      }
      if (idle) {  // the fold buffer has landed (issued before the peer wait)
        mbar_wait(stage_bar, stage_ph);
        stage_ph ^= 1u;
      }
      if (stage_peers) {  // every peer's rows [0, nr) and (m, l): contiguous runs of its slot
        __syncwarp();
        if (lane == 0) mbar_arrive_expect_tx(stage_bar, uint32_t(np) * nr * (D + 4) * 4);
        __syncwarp();
        #pragma unroll 1
        for (int i = lane; i < np; i += 32) {
          const size_t row = size_t(v + 1 + i) * a.group;
          bulk_g2s_plain(prow + size_t(i) * nr * D, a.part_o + row * D, uint32_t(nr) * D * 4, stage_bar);
          bulk_g2s_plain(pml + size_t(i) * nr * 4, a.part_ml + row * 4, uint32_t(nr) * 16, stage_bar);
        }
        mbar_wait(stage_bar, stage_ph);
        stage_ph ^= 1u;
      }
      if (NEP > 1 && lane == 0) *epi_flags = int(idle) | int(stage_peers) << 1;
    }
    if constexpr (NEP > 1) {
      epi_sync();  // (A) staged operands, the acquired peers' partials and the flags word
      if (e != 0) {
        const int f = *epi_flags;
        idle = f & 1;
        stage_peers = f & 2;
      }
    }
    const float* fb = idle ? fstg : fold + b * FOLD_FLOATS;
#ifdef LA_WIDE_PRINT
    unsigned long long wt[8] = {globaltimer(), 0, 0, 0, 0, 0, 0, 0};
#endif
    const int rb = e * RW, re = min(nr, rb + RW);  // this warp's rows
    if (rb >= re && lane == 0) mbar_arrive(&fold_empty[b]);
    #pragma unroll 1
    for (int r0 = rb; r0 < re; r0 += RG) {
#ifdef LA_WIDE_PRINT
      if ((r0 - rb) / RG < 4) wt[1 + (r0 - rb) / RG] = globaltimer();
#endif
      // ---- rows r0 .. r0 + 7 of the NWG x FW warp partials (branch-free: loads issue together)
#pragma unroll
      for (int hh = 0; hh < RG; ++hh) {
        const int h = r0 + hh;
        float mw[NWG * FW], lw[NWG * FW], ow[NWG * FW][J], mx = -INFINITY, ls = 0.f;
#pragma unroll
        for (int cw = 0; cw < NWG * FW; ++cw) {  // warp sets relative to the segment's first stage (C16)
          const int w = ((si.s0 + cw / FW) % NWG) * FW + cw % FW;
          const float* r = fb + (w * H + h) * (D + 4);
          const float2 ml = *reinterpret_cast<const float2*>(r + D);
          mw[cw] = ml.x;
          lw[cw] = ml.y;
          ldv<J>(r + J * lane, ow[cw]);
        }
#pragma unroll
        for (int cw = 0; cw < NWG * FW; ++cw) mx = fmaxf(mx, mw[cw]);
#pragma unroll
        for (int jj = 0; jj < J; ++jj) o[hh][jj] = 0.f;
#pragma unroll
        for (int cw = 0; cw < NWG * FW; ++cw) {
          const float wt = ex2_sub(mw[cw], mx);
          ls = fmaf(wt, lw[cw], ls);
#pragma unroll
          for (int jj = 0; jj < J; ++jj) o[hh][jj] = fmaf(wt, ow[cw][jj], o[hh][jj]);
        }
        m[hh] = mx;
        l[hh] = ls;
      }
      __syncwarp();
      if (r0 + RG >= re && lane == 0) mbar_arrive(&fold_empty[b]);  // consumers may refill it
#ifdef LA_WIDE_PRINT
      if (r0 == rb) wt[5] = globaltimer();
#endif
      if (!out && !host_wait) {  // StorePartials (Alg2§20-22)
#pragma unroll
        for (int hh = 0; hh < RG; ++hh) {
          if (r0 + hh >= nr) continue;
          const size_t row = size_t(v) * a.group + r0 + hh;
          stv<J>(a.part_o + row * D + J * lane, o[hh]);
          if (lane == 0) *reinterpret_cast<float2*>(a.part_ml + row * 4) = make_float2(m[hh], l[hh]);
        }
        continue;
      }
      if (host_wait) {
        // ---- fold the peers v+1 .. last_cta (ascending, max-first, reading C22): staged above
        //      (stage_peers), else read from L2 (acquired by warp 0 before barrier A)
        const int p0 = v + 1, n = np;
        #pragma unroll 1
        for (int b0 = 0; b0 < n; b0 += 32) {  // (a 16 / 32-row unit spans few CTAs: one block)
          const int bn = min(32, n - b0);
          float2 ml[RG];
          if (!stage_peers) {
            const size_t mlrow = size_t(p0 + b0 + min(lane, bn - 1)) * a.group + r0;
#pragma unroll
            for (int hh = 0; hh < RG; ++hh) ml[hh] = __ldcg(reinterpret_cast<const float2*>(a.part_ml + (mlrow + hh) * 4));
          } else {
            const float* mls = pml + (size_t(b0 + min(lane, bn - 1)) * nr + r0) * 4;
#pragma unroll
            for (int hh = 0; hh < RG; ++hh)
              ml[hh] = r0 + hh < nr ? *reinterpret_cast<const float2*>(mls + hh * 4) : make_float2(-INFINITY, 0.f);
          }
          float w[RG];
#pragma unroll
          for (int hh = 0; hh < RG; ++hh) {
            float M = fmaxf(m[hh], lane < bn ? ml[hh].x : -INFINITY);
#pragma unroll
            for (int off = 16; off; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
            w[hh] = lane < bn ? ex2_sub(ml[hh].x, M) : 0.f;
            float lsum = w[hh] * (lane < bn ? ml[hh].y : 0.f);
#pragma unroll
            for (int off = 16; off; off >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, off);
            const float wa = ex2_sub(m[hh], M);
            l[hh] = fmaf(wa, l[hh], lsum);
            m[hh] = M;
#pragma unroll
            for (int jj = 0; jj < J; ++jj) o[hh][jj] *= wa;
          }
          #pragma unroll 1
          for (int i = 0; i < bn; ++i) {  // ascending peers
#pragma unroll
            for (int hh = 0; hh < RG; ++hh) {
              const float wk = __shfl_sync(0xffffffffu, w[hh], i);
              float rv[J];
              if (stage_peers)
                ldv<J>(prow + ((size_t(b0 + i) * nr + r0 + hh) * D + J * lane), rv);
              else
                ldv_cg<J>(a.part_o + (size_t(p0 + b0 + i) * a.group + r0 + hh) * D + J * lane, rv);
#pragma unroll
              for (int jj = 0; jj < J; ++jj) o[hh][jj] = fmaf(wk, rv[jj], o[hh][jj]);
            }
          }
          __syncwarp();
        }
      }
#ifdef LA_WIDE_PRINT
      if (r0 == rb) wt[6] = globaltimer();
#endif
      // ---- O = diag(l)^-1 O, L = m + log(l) (Alg2§38-39) -- or this rank's normalised shard
      //      partial pushed into every rank's exchange buffer (NEXT-2).  Lane hh computes row
      //      hh's 1 / l and log2 l (the same operations as a per-row loop, so the same bits):
      //      one division and one logarithm of latency instead of RG serial ones.
      float lsel = l[0], msel = m[0];
#pragma unroll
      for (int hh = 1; hh < RG; ++hh)
        if (lane == hh) {
          lsel = l[hh];
          msel = m[hh];
        }
      const float inv_lane = a.out_scale / lsel, l2_lane = msel + log2f(lsel);
      if (a.xw > 1) {
        const int P = a.xw, par = int(xepoch & 1u);
#pragma unroll
        for (int hh = 0; hh < RG; ++hh) {
          const float inv = __shfl_sync(0xffffffffu, inv_lane, hh), l2 = __shfl_sync(0xffffffffu, l2_lane, hh);
          if (r0 + hh >= nr) continue;
          #pragma unroll 1
          for (int d = 0; d < P; ++d) {
            float* dst = a.xpeer[d] + ((size_t(par) * P + a.xr) * a.xrows + u.q_row + r0 + hh) * RS;
            stv<J>(dst + J * lane, o[hh], inv);
            if (lane == 0) dst[D] = l2;
          }
        }
      } else {
        float* dst = a.out + size_t(u.q_row + r0) * D + J * lane;
#pragma unroll
        for (int hh = 0; hh < RG; ++hh) {
          const float inv = __shfl_sync(0xffffffffu, inv_lane, hh);
          if (r0 + hh < nr) stv<J>(dst + hh * D, o[hh], inv);
        }
        if (a.lse && lane < RG && r0 + lane < nr) a.lse[u.q_row + r0 + lane] = l2_lane * kLn2;
      }
    }
    if (!out && !host_wait) {  // Signal (Alg2§23)
      __threadfence();
      __syncwarp();
      epi_sync();  // (B) every epilogue warp's partial rows are out
      if (e == 0 && lane == 0) {
        st_release_gpu(&a.flags[v], epoch);
        if (tr && !tr[TR_PUBLISH]) tr[TR_PUBLISH] = globaltimer();
      }
    } else if (a.xw > 1) {  // NEXT-2: release, wait for the P ranks, fold their partials
      __threadfence_system();
      __syncwarp();
      epi_sync();  // (B) every epilogue warp's rows are in the exchange buffers
      if (e == 0) {
        const int P = a.xw, par = int(xepoch & 1u);
        if (lane < P) {
          uint32_t* f = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(a.xpeer[lane]) + a.xflag_off);
          st_release_sys(f + size_t(a.xr) * a.xunits + si.unit, xepoch);
          const uint32_t* mine = reinterpret_cast<const uint32_t*>(reinterpret_cast<const char*>(a.xpeer[a.xr]) +
                                                                   a.xflag_off) + size_t(lane) * a.xunits + si.unit;
          const unsigned long long t0 = globaltimer();
          while (int32_t(ld_acquire_sys(mine) - xepoch) < 0) {
            if (*reinterpret_cast<volatile int*>(a.xerr) || globaltimer() - t0 > kXchgTimeoutNs) {
              atomicExch(a.xerr, 1);
              break;
            }
            __nanosleep(64);
          }
        }
        __syncwarp();
        const float* xb = a.xpeer[a.xr] + size_t(par) * P * a.xrows * RS;
        #pragma unroll 1
        for (int h = 0; h < nr; ++h) {
          float M = -INFINITY, lsum = 0.f, acc[J];
          #pragma unroll 1
          for (int r = 0; r < P; ++r) M = fmaxf(M, ld_cg(xb + (size_t(r) * a.xrows + u.q_row + h) * RS + D));
#pragma unroll
          for (int jj = 0; jj < J; ++jj) acc[jj] = 0.f;
          #pragma unroll 1
          for (int r = 0; r < P; ++r) {
            const float* src = xb + (size_t(r) * a.xrows + u.q_row + h) * RS;
            const float w = ex2_sub(ld_cg(src + D), M);
            lsum += w;
            float rv[J];
            ldv_cg<J>(src + J * lane, rv);
#pragma unroll
            for (int jj = 0; jj < J; ++jj) acc[jj] = fmaf(w, rv[jj], acc[jj]);
          }
          stv<J>(a.out + size_t(u.q_row + h) * D + J * lane, acc, 1.f / lsum);
          if (lane == 0 && a.lse) a.lse[u.q_row + h] = (M + log2f(lsum)) * kLn2;
        }
      }
    } else {
      epi_sync();  // (B) the staged operands are read: the next segment may restage the ring
    }
    if (e == 0 && host_wait && tr && lane == 0) tr[TR_PUBLISH] = globaltimer();  // host: fold done
#ifdef LA_WIDE_PRINT
    if (lane == 0 && e == 0 && host_wait && blockIdx.x % 16 == 0)
      printf("WIDE cta %d np %d nr %d idle %d sp %d: w1->loop %llu, rg %llu %llu %llu %llu, end %llu ns; rg0: cfold %llu peers %llu write %llu\n",
             int(blockIdx.x), np, nr, int(idle), int(stage_peers), wt[0] - (tr ? tr[TR_WAIT1] : wt[0]), wt[1] - wt[0],
             wt[2] - wt[1], wt[3] - wt[2], wt[4] - wt[3], globaltimer() - wt[0], wt[5] - wt[1], wt[6] - wt[5],
             wt[2] - wt[6]);
#endif
  }
  if (e == 0 && lane == 0) {
    if (tr) tr[TR_END] = globaltimer();
    __threadfence();  // every flag wait of this CTA is over: the last one out advances the epoch
    if (atomicAdd(&a.counters[CTR_EXITED], 1) == int(gridDim.x) - 1) {
      a.counters[CTR_EXITED] = 0;
      *reinterpret_cast<volatile uint32_t*>(&a.counters[CTR_EPOCH]) = epoch;
      if (a.xw > 1) *reinterpret_cast<volatile uint32_t*>(&a.counters[CTR_XEPOCH]) = xepoch;
      __threadfence();
    }
  }
}

template <class E>
__global__ void __launch_bounds__((E::NCW + 1 + EngX<E>::NEP) * 32, 1) la_decode(const DecodeArgs a, const __grid_constant__ TmapPair tm) {
  constexpr int NST = E::NST, NWG = E::NWG, WPS = E::WPS, NCW = E::NCW, D = E::D, H = E::HEADS, J = D / 32;
  constexpr int FW = EngX<E>::FW;  // fold rows per ring slot (WPS, or 1 for a warpgroup engine)
  constexpr int FOLD_FLOATS = E::FOLD_FLOATS;
  constexpr int kFB = E::FOLD_BUFS;
  constexpr int kQD = EngX<E>::QD;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* ring =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* fold = EngX<E>::GF ? a.gfold + size_t(blockIdx.x) * kFB * E::FOLD_FLOATS
                            : reinterpret_cast<float*>(ring + Smem<E>::RING + Smem<E>::EXTRA);
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + Smem<E>::RING + Smem<E>::EXTRA + Smem<E>::FOLD);
  uint64_t* empty = full + NST;
  uint64_t* sq_full = empty + NST;         // segment queue entry written (+ its Q rows landed)
  uint64_t* sq_empty = sq_full + kQD;      // every consumer warp has read the entry
  uint64_t* fold_full = sq_empty + kQD;
  uint64_t* fold_empty = fold_full + kFB;
  uint64_t* stage_bar = fold_empty + kFB;  // peers' partials staged for a fold
  SegQ* squeue = reinterpret_cast<SegQ*>(ring + Smem<E>::SQ_OFF);
  SegInfo* seginfo = reinterpret_cast<SegInfo*>(squeue + kQD);
  int* prod_j = reinterpret_cast<int*>(seginfo + kFB);  // stages the producer issued in all, once done (-1 before)
  float* wscr = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(prod_j + 4) + 15) & ~uintptr_t(15));  // [32][<= 8] fold weights
  unsigned char* qbuf = ring + Smem<E>::QB_OFF;         // [kQD][QB]: Q rows of each queued segment

  const int warp = __shfl_sync(0xffffffffu, int(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int g = blockIdx.x;
  // This launch's epoch (reading C17): one more than the last launch's, kept ON THE DEVICE
  // (counters[3], advanced by the last CTA to exit) so a launch captured into a CUDA graph
  // publishes fresh flag values on every replay.  Launches on one stream never overlap, so
  // every CTA reads the same value.
  const uint32_t epoch_prev = *reinterpret_cast<volatile const uint32_t*>(&a.counters[CTR_EPOCH]);
  const uint32_t epoch = epoch_prev == 0xFFFFFFFFu ? 1u : epoch_prev + 1u;
  // The cross-GPU exchange has its own sequence number, advanced only by exchange launches
  // (la_decode_partial on the same plan must not shift it against the peers' sequence).
  const uint32_t xepoch_prev = *reinterpret_cast<volatile const uint32_t*>(&a.counters[CTR_XEPOCH]);
  const uint32_t xepoch = xepoch_prev == 0xFFFFFFFFu ? 1u : xepoch_prev + 1u;
  const bool dynamic = a.dynamic != 0;
  const int SS = a.slot_stride;     // partial slot 1 of (virtual) CTA v is SS + v
  unsigned long long* tr = a.trace ? a.trace + size_t(g) * TR_FIELDS : nullptr;
  if (tr && threadIdx.x == 0) {
    tr[TR_SMID] = smid();
    tr[TR_START] = globaltimer();
    tr[TR_PUBLISH] = tr[TR_WAIT0] = tr[TR_WAIT1] = tr[TR_STREAM] = 0;
  }
  if (E::ZERO_RING)  // rows past a short stage must be finite (masked p = 0; 0 * finite = 0)
    for (int i = threadIdx.x; i < Smem<E>::RING / 16; i += blockDim.x)
      reinterpret_cast<uint4*>(ring)[i] = make_uint4(0u, 0u, 0u, 0u);
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], WPS);
    }
    for (int q = 0; q < kQD; ++q) {
      mbar_init(&sq_full[q], 1);
      mbar_init(&sq_empty[q], NCW);
    }
    for (int b = 0; b < kFB; ++b) {
      mbar_init(&fold_full[b], NCW);
      mbar_init(&fold_empty[b], EngX<E>::NEP);
    }
    mbar_init(stage_bar, 1);
    *prod_j = -1;
    if constexpr (EngX<E>::TMEM > 0) E::init_barriers();
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if constexpr (EngX<E>::TMEM > 0) {
    if (warp == 0) tc5::tmem_alloc(E::tmem_base_ptr(), EngX<E>::TMEM);
    tc5::fence_before();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // zero-fill before TMA writes
  __syncthreads();
  if constexpr (EngX<E>::TMEM > 0) tc5::fence_after();

  if (warp == NCW + 1) {
    // ================================ producer ==========================================
    // The whole warp walks; lane 0 owns the barriers, the claim and the queue, and issues
    // the copies of contiguous stages.  For paged KV every lane issues one page run / TMA
    // box of the stage, so small pages do not serialise on one thread.
    const uint64_t pol = l2_evict_first_policy();
    if (lane == 0 && a.uses_tmap) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm.k)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm.v)) : "memory");
    }
    int j = 0, ks = 0;
    const int win = a.win > 0 ? min(a.win, E::WIN) : E::WIN;  // stages in flight
#ifdef LA_PROF
    long long prof_pwait = 0;  // producer cycles waiting for free slots -> trace field smid
    long long prof_issue = 0;  // paged: cycles in produce_paged -> trace field t_stream_end
#endif
    constexpr int QB = Smem<E>::QB;
    const int q_el = int(sizeof(typename E::QElem));
    // Hand segment (u, v, [it, it_end)) to the consumers: queue entry + its Q rows (lane 0).
    auto push_seg = [&](const DevUnit& u, int v, int unit, int it, int it_end, int host, int finishing) {
      const int qi = ks % kQD;
      if (ks >= kQD) mbar_wait(&sq_empty[qi], ((ks / kQD) - 1) & 1);
      SegQ& e = squeue[qi];
      e.u = u;
      e.v = v;
      e.unit = unit;
      e.it = it;
      e.it_end = it_end;
      e.host = host;
      e.finishing = finishing;
      if (QB > 0 && v >= 0) {
        const uint32_t bytes = uint32_t(u.rows) * D * q_el;
        mbar_arrive_expect_tx(&sq_full[qi], bytes);
        bulk_g2s_plain(qbuf + qi * QB, static_cast<const unsigned char*>(a.q) + size_t(u.q_row) * D * q_el, bytes,
                       &sq_full[qi]);
      } else {
        mbar_arrive(&sq_full[qi]);
      }
      ++ks;
    };
    // The current piece (virtual CTA v: iterations [it, it1), first unit `unit`) and, for the
    // dynamic schedule, the next one fetched AHEAD by lane 0 in steps spread over the piece's
    // last kClaimAhead LeanTiles (claim atomic -> claim table -> range -> unit record), so the
    // dependent round trips overlap the last stages instead of draining the ring at every
    // piece boundary.  The heads are the first G claims, so no CTA hoards two of them.
    int v = -1, it = 0, it1 = 0, unit = 0;
    int pst = 0, c_nx = -1, v_nx = -1, b_nx = 0, e_nx = 0, u_nx = 0;
    DevUnit du_nx{};
    auto fetch_ahead = [&](int rem, bool force) {  // lane 0, dynamic
      if (pst == 0 && (force || rem <= kClaimAhead)) {
        c_nx = atomicAdd(&a.counters[CTR_CLAIM], 1);
        pst = 1;
      }
      if (pst == 1 && (force || rem <= kClaimAhead - 1)) {
        v_nx = a.claim[c_nx];   // padded with -1 past the schedule's ranges: no more work
        pst = 2;
      }
      if (pst == 2 && (force || rem <= kClaimAhead - 2)) {
        if (v_nx >= 0) {
          b_nx = a.cta_begin[v_nx];
          e_nx = a.cta_begin[v_nx + 1];
          u_nx = a.cta_first_unit[v_nx];
        }
        pst = 3;
      }
      if (pst == 3 && (force || rem <= kClaimAhead - 3)) {
        if (v_nx >= 0) du_nx = a.units[u_nx];
        pst = 4;
      }
    };
    DevUnit u{};
    if (lane == 0) {
      if (dynamic) {
        fetch_ahead(0, true);
        v = v_nx;
        pst = 0;
#ifndef LA_EPI_TRACE
        if (tr) tr[TR_WAIT0] += 1;
#endif
      } else {
        v = g;   // static: CTA g runs range g (the range table is padded with empty ranges)
      }
      if (v >= 0) {
        it = dynamic ? b_nx : a.cta_begin[v];
        it1 = dynamic ? e_nx : a.cta_begin[v + 1];
        unit = dynamic ? u_nx : a.cta_first_unit[v];
        if (it >= it1) v = -1;   // an idle range (forced G > I: S:219; or a grid wider than the schedule)
        else u = dynamic ? du_nx : a.units[unit];
      }
    }
    while (__shfl_sync(0xffffffffu, v, 0) >= 0) {
      int seg_end = 0;
      DevUnit un{};  // the next unit of this piece, loaded ahead
      if (lane == 0) {
        while (u.iter_end <= it) u = a.units[++unit];      // (cta_first_unit makes this rare)
        seg_end = min(u.iter_end, it1);
        push_seg(u, v, unit, it, seg_end, it == u.iter_begin ? 1 : 0, it1 >= u.iter_end ? 1 : 0);  // Alg2§17-18
        if (it1 > u.iter_end) un = a.units[unit + 1];     // consumed at the next segment
      }
      // the whole warp walks the segment (paged: every lane issues page runs / TMA boxes)
      seg_end = __shfl_sync(0xffffffffu, seg_end, 0);
      it = __shfl_sync(0xffffffffu, it, 0);
      it1 = __shfl_sync(0xffffffffu, it1, 0);
      const int64_t row0 = __shfl_sync(0xffffffffu, u.row0, 0);
      const int ib = __shfl_sync(0xffffffffu, u.iter_begin, 0), ulen = __shfl_sync(0xffffffffu, u.len, 0);
      PageWin pw;
      if (a.paged) pw.init(a, row0);
      for (; it < seg_end; ++it) {                          // LeanTile iterations (Alg1§13)
        if (dynamic && lane == 0) fetch_ahead(it1 - it, false);
        const int t0 = (it - ib) * a.tile_n;                // kk = iter * T_n (Alg1§14)
        const int t1 = min(t0 + a.tile_n, ulen);
        for (int s0 = t0; s0 < t1; s0 += a.stage_tokens) {  // LoadFragment K, V (Alg1§17-18)
          const int slot = j % NST;
#ifdef LA_PROF
          const long long c0 = clock64();
#endif
          if (lane == 0 && j >= NST) mbar_wait(&empty[slot], ((j / NST) - 1) & 1);
          // at most `win` stages in flight: stage j - win must be consumed first (its slot's next
          // stage j - win + NST > j is not issued yet, so the phase cannot alias).  DESIGN §6: an
          // SM with more bytes in flight than the memory system serves it at its fair share only
          // adds queueing, and the CTAs' streaming rates then scatter (the kernel ends with the slowest)
          if (win < NST && lane == 0 && j >= win) mbar_wait(&empty[(j - win) % NST], ((j - win) / NST) & 1);
#ifdef LA_PROF
          if (lane == 0) prof_pwait += clock64() - c0;
#endif
          const int ntok = min(a.stage_tokens, t1 - s0);
          if (!a.paged) {
            if constexpr (EngX<E>::VWIN < E::WIN && LA_ELECT_PRODUCE) {  // (tcgen05) K now, V after stage j - VWIN;
              // the whole warp issues (one elected lane, warp-uniform operands)
              E::produce_w(ring + slot * E::STAGE_BYTES, tm, row0 + s0, &full[slot], pol, lane,
                           j >= E::VWIN ? &empty[(j - E::VWIN) % NST] : nullptr, ((j - E::VWIN) / NST) & 1);
            } else if constexpr (EngX<E>::VWIN < E::WIN) {
              if (lane == 0) {
                E::produce_k(ring + slot * E::STAGE_BYTES, tm, row0 + s0, &full[slot], pol);
                if (j >= E::VWIN) mbar_wait(&empty[(j - E::VWIN) % NST], ((j - E::VWIN) / NST) & 1);
                E::produce_v(ring + slot * E::STAGE_BYTES, tm, row0 + s0, pol);
              }
            } else {
              if (lane == 0) E::produce(ring + slot * E::STAGE_BYTES, a, tm, row0 + s0, ntok, &full[slot], pol);
            }
          } else {
#ifdef LA_PROF
            const long long ci = clock64();
#endif
            E::produce_paged(ring + slot * E::STAGE_BYTES, a, tm, pw, s0, ntok, &full[slot], pol, lane);
#ifdef LA_PROF
            __syncwarp();
            if (lane == 0) prof_issue += clock64() - ci;
#endif
          }
          ++j;
        }
      }
      if (lane == 0) {
        if (it < it1) {          // the piece continues in the next unit
          ++unit;
          u = un;
        } else if (dynamic) {    // next piece: finish the look-ahead (short pieces) and take it
          fetch_ahead(0, true);
          v = v_nx;
          pst = 0;
#ifndef LA_EPI_TRACE
          if (tr) tr[TR_WAIT0] += 1;
#endif
          if (v >= 0) {
            it = b_nx;
            it1 = e_nx;
            unit = u_nx;
            u = du_nx;
          }
        } else {
          v = -1;                // a static CTA runs exactly its range g
        }
      }
    }
    if (lane == 0) push_seg(DevUnit{}, -1, -1, 0, 0, 0, 0);   // terminator for the consumers
    // every stage this CTA will stream has been issued: once the consumers have used stage
    // j - 1, the ring is idle (a dynamic last arriver may stage its fold there)
    if (lane == 0) *reinterpret_cast<volatile int*>(prod_j) = j;
#ifdef LA_PROF
    if (tr && lane == 0) {
      tr[TR_SMID] = prof_pwait;
      tr[TR_STREAM] = prof_issue;
    }
#endif
    return;
  }

  if constexpr (H > 8) {
    if (warp == NCW || warp >= NCW + 2) {  // epilogue warps 0 .. NEP-1 (the producer is warp NCW + 1)
      wide_epilogue<E>(a, tm, ring, fold, fold_full, fold_empty, stage_bar, seginfo, prod_j, epoch, xepoch, tr, lane,
                       warp == NCW ? 0 : warp - NCW - 1);
      return;
    }
  }
  if constexpr (H <= 8) if (warp == NCW) {
    // ================================ epilogue ==========================================
    // Folds the NCW per-warp partials of each finished segment (§4.1 operator) and runs the
    // fixup -- partial stores, flags / counters, peer folds, finalize -- off the consumers'
    // critical path.
    EpiAcc<E> acc;
    auto reset = [&]() {
#pragma unroll
      for (int h = 0; h < H; ++h) {
        acc.m[h] = -INFINITY;
        acc.l[h] = 0.f;
#pragma unroll
        for (int jj = 0; jj < J; ++jj) acc.o[h][jj] = 0.f;
      }
    };
    int nr = 0;  // output rows of the current segment's unit (its query tile, <= H)
    uint32_t stage_ph = 0;  // phase of stage_bar (peers' partials staged for a fold)
    auto store_partial = [&](int slot) {  // StorePartials(Op, mp, lp) (Alg2§20-22)
#pragma unroll
      for (int h = 0; h < H; ++h) {
        if (h >= nr) continue;
        const size_t row = size_t(slot) * a.group + h;
        stv<J>(a.part_o + row * D + J * lane, acc.o[h]);
        if (lane == 0) {
          a.part_ml[row * 4] = acc.m[h];
          a.part_ml[row * 4 + 1] = acc.l[h];
        }
      }
      __threadfence();  // every lane: its stores are visible GPU-wide before the signal
      __syncwarp();
    };
    // Fold peers p0 .. p1 (ascending) into acc (Alg2§27-35, reading C22's max-first form): in
    // blocks of 32 peers (lane i <-> peer i of the block),
    //   A: every lane reads its peer's (m, l) of each row from L2; M = max(m_acc, m_p..) by a
    //      warp reduction, w_p = 2^(m_p - M), l = 2^(m_acc - M) l_acc + sum_p w_p l_p;
    //   B: the peers' O~ rows are staged in smem `stg` (stg_floats: the ring when idle, else a
    //      consumed fold buffer) by 1-D bulk copies -- ONE copy for a contiguous run of slot-0
    //      peers -- in as many rounds as the buffer needs, and O = 2^(m_acc - M) O_acc +
    //      sum_p w_p O~_p accumulates in NCH fixed chains (peer k of the block -> chain k % NCH).
    // The arithmetic depends only on the peers and their order -- never on the staging buffer
    // -- so the result is bitwise deterministic.  host_v's partial lives in slot 1 (SS + v).
    auto fold_smem = [&](int p0, int p1, int host_v, float* stg, int stg_floats) {
      constexpr int NCH = H == 1 ? 4 : 1;  // independent accumulator chains per row
      constexpr int RG = H < 8 ? H : 8;    // rows folded together (wide tcgen05 tiles: groups of 8)
      const int n = p1 < p0 ? 0 : p1 - p0 + 1;
      const int po = RG * D;               // staged per peer and row group: RG O~ rows
      const int cap = max(NCH, stg_floats / po / NCH * NCH);  // a multiple of NCH: peer k -> chain k % NCH
      auto slot_of = [&](int p) { return p + (p == host_v ? SS : 0); };
      // stage the O~ rows (row group r0) of peers q0 .. q0 + cs - 1 into stg, asynchronously
      auto stage = [&](int r0, int q0, int cs) {
        // one copy for a run of slot-0 peers whose RG rows are all of their rows
        const bool contiguous = RG == a.group && (host_v < q0 || host_v >= q0 + cs);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // earlier smem reads
        __syncwarp();
        const int rows = min(RG, a.group - r0);  // the slot's rows in this group
        if (lane == 0) mbar_arrive_expect_tx(stage_bar, uint32_t(cs) * rows * D * 4);
        __syncwarp();
        if (contiguous) {
          if (lane == 0) bulk_g2s_plain(stg, a.part_o + size_t(q0) * a.group * D, uint32_t(cs) * po * 4, stage_bar);
        } else {
          #pragma unroll 1
          for (int i = lane; i < cs; i += 32)
            bulk_g2s_plain(stg + i * po, a.part_o + (size_t(slot_of(q0 + i)) * a.group + r0) * D, uint32_t(rows) * D * 4,
                           stage_bar);
        }
      };
#ifdef LA_FOLD_PRINT
      const unsigned long long ft0 = globaltimer();
      unsigned long long ftA = 0, ftW = 0;
#endif
      asm volatile("fence.proxy.async.global;" ::: "memory");      // acquired partials -> TMA
      // this epilogue serves tiles of H <= 8 rows: ONE row group (RG = H), r0 a compile-time 0,
      // so every acc index below is static and the accumulator stays in registers (a runtime
      // row-group loop made them dynamic and put acc in local memory: every epilogue step
      // then paid dependent L1 round trips)
      static_assert(RG == H, "one row group");
      {
      constexpr int r0 = 0;
      #pragma unroll 1
      for (int b0 = 0; b0 < n; b0 += 32) {
        const int bn = min(32, n - b0);
        stage(r0, p0 + b0, min(cap, bn));  // the first round flies while A reads the (m, l)s
        // ---- A: max-first weights and l, every row at once (independent shuffle chains) --------
        const size_t mlrow = size_t(slot_of(p0 + b0 + min(lane, bn - 1))) * a.group + r0;
        float mp[RG], lp[RG], M[RG], wa[RG];
#pragma unroll
        for (int hh = 0; hh < RG; ++hh) {  // every row's (m, l) first: ONE L2 round trip
          const float2 ml = r0 + hh < nr ? __ldcg(reinterpret_cast<const float2*>(a.part_ml + (mlrow + hh) * 4))
                                         : make_float2(-INFINITY, 0.f);
          mp[hh] = lane < bn ? ml.x : -INFINITY;
          lp[hh] = lane < bn ? ml.y : 0.f;
          M[hh] = fmaxf(r0 + hh < nr ? acc.m[r0 + hh] : -INFINITY, mp[hh]);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1)
#pragma unroll
          for (int hh = 0; hh < RG; ++hh) M[hh] = fmaxf(M[hh], __shfl_xor_sync(0xffffffffu, M[hh], o));
#pragma unroll
        for (int hh = 0; hh < RG; ++hh) {
          mp[hh] = ex2_sub(mp[hh], M[hh]);  // w_p; 0 for lanes past the block / masked rows
          lp[hh] *= mp[hh];
        }
#pragma unroll
        for (int o = 16; o; o >>= 1)
#pragma unroll
          for (int hh = 0; hh < RG; ++hh) lp[hh] += __shfl_xor_sync(0xffffffffu, lp[hh], o);
        __syncwarp();  // the previous block's reads of wscr are done
#pragma unroll
        for (int hh = 0; hh < RG; ++hh) {
          wscr[lane * RG + hh] = mp[hh];  // peer lane's weights, read back as broadcasts in B
          const int h = r0 + hh;
          wa[hh] = 0.f;
          if (h >= nr) continue;
          wa[hh] = ex2_sub(acc.m[h], M[hh]);  // idle / masked accumulator: -inf -> 0
          acc.l[h] = fmaf(wa[hh], acc.l[h], lp[hh]);
          acc.m[h] = M[hh];
        }
        __syncwarp();
        // ---- B: O~ rows, round by round ----------------------------------------------------
#ifdef LA_FOLD_PRINT
        ftA += globaltimer() - ft0;
#endif
        float oc[NCH][RG][J];
#pragma unroll
        for (int c = 0; c < NCH; ++c)
#pragma unroll
          for (int hh = 0; hh < RG; ++hh)
#pragma unroll
            for (int jj = 0; jj < J; ++jj) oc[c][hh][jj] = c == 0 ? acc.o[r0 + hh][jj] * wa[hh] : 0.f;
        #pragma unroll 1
        for (int c0 = 0; c0 < bn; c0 += cap) {
          const int cs = min(cap, bn - c0);
          if (c0 > 0) stage(r0, p0 + b0 + c0, cs);
          mbar_wait(stage_bar, stage_ph);
          stage_ph ^= 1u;
#ifdef LA_FOLD_PRINT
          ftW += globaltimer() - ft0;
#endif
          #pragma unroll 1
          for (int i0 = 0; i0 < cs; i0 += NCH) {
#pragma unroll
            for (int c = 0; c < NCH; ++c) {
              const int i = i0 + c;  // block peer c0 + i is on chain c (c0 and i0 are multiples of NCH)
              if (i >= cs) break;
              float wk[RG];
#pragma unroll
              for (int hh = 0; hh < RG; hh += (RG % 4 == 0 ? 4 : 1)) {  // broadcast reads of the weights
                if constexpr (RG % 4 == 0) {
                  const float4 t = *reinterpret_cast<const float4*>(wscr + (c0 + i) * RG + hh);
                  wk[hh] = t.x; wk[hh + 1] = t.y; wk[hh + 2] = t.z; wk[hh + 3] = t.w;
                } else {
                  wk[hh] = wscr[(c0 + i) * RG + hh];
                }
              }
#pragma unroll
              for (int hh = 0; hh < RG; ++hh) {
                if (r0 + hh >= nr) continue;
                float rv[J];
                ldv<J>(stg + i * po + hh * D + J * lane, rv);
#pragma unroll
                for (int jj = 0; jj < J; ++jj) oc[c][hh][jj] = fmaf(wk[hh], rv[jj], oc[c][hh][jj]);
              }
            }
          }
          __syncwarp();  // the next round overwrites the stage
        }
#pragma unroll
        for (int hh = 0; hh < RG; ++hh)
#pragma unroll
          for (int jj = 0; jj < J; ++jj)
            acc.o[r0 + hh][jj] = NCH == 4 ? (oc[0][hh][jj] + oc[1 % NCH][hh][jj]) + (oc[2 % NCH][hh][jj] + oc[3 % NCH][hh][jj])
                                          : oc[0][hh][jj];
      }
      }
#ifdef LA_FOLD_PRINT
      if (lane == 0 && n > 1)
        printf("FOLD cta %d n %d nr %d cap %d ring %d: A-done %llu wait-done %llu total %llu ns\n", int(blockIdx.x), n, nr,
               cap, int(stg == reinterpret_cast<float*>(ring)), ftA, ftW, globaltimer() - ft0);
#endif
    };
    // NEXT-2: push this rank's normalised shard partial of unit `unit` into every rank's
    // exchange buffer, release flag [xr][unit] there, acquire the P flags of the unit here
    // and fold the P partials ascending (§4.1 operator; bitwise equal on every rank).
    // Deadlock freedom: every CTA (and the virtual-CTA claim order) visits units in
    // increasing order and pushes unit u before waiting on it.  Take the smallest unit m
    // anyone waits on: on every rank, all work of m precedes (in its CTA's order) any wait
    // on a unit > m, and no CTA is stuck on a unit < m, so every rank completes m's push.
    auto xchg_out = [&](int q_row, int unit) {
      constexpr int RS = D + 4;
      const int P = a.xw, par = int(xepoch & 1u);
#pragma unroll
      for (int h = 0; h < H; ++h) {
        if (h >= nr) continue;
        const float inv = a.out_scale / acc.l[h], l2 = acc.m[h] + log2f(acc.l[h]);
        #pragma unroll 1
        for (int d = 0; d < P; ++d) {
          float* dst = a.xpeer[d] + ((size_t(par) * P + a.xr) * a.xrows + q_row + h) * RS;
          stv<J>(dst + J * lane, acc.o[h], inv);
          if (lane == 0) dst[D] = l2;
        }
      }
      __threadfence_system();
      __syncwarp();
      if (lane < P) {
        uint32_t* f = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(a.xpeer[lane]) + a.xflag_off);
        st_release_sys(f + size_t(a.xr) * a.xunits + unit, xepoch);
        const uint32_t* mine = reinterpret_cast<const uint32_t*>(reinterpret_cast<const char*>(a.xpeer[a.xr]) +
                                                                 a.xflag_off) + size_t(lane) * a.xunits + unit;
        const unsigned long long t0 = globaltimer();
        // wrap-safe: a peer one launch ahead has already overwritten the flag with xepoch + 1
        // (its data for THIS launch sits untouched in parity xepoch & 1: it cannot finish
        // that next launch, let alone start another, before this rank pushes)
        while (int32_t(ld_acquire_sys(mine) - xepoch) < 0) {
          // a peer never arrived: flag it and move on (later waits then give up at once)
          if (*reinterpret_cast<volatile int*>(a.xerr) || globaltimer() - t0 > kXchgTimeoutNs) {
            atomicExch(a.xerr, 1);
            break;
          }
          __nanosleep(64);
        }
      }
      __syncwarp();
      const float* xb = a.xpeer[a.xr] + size_t(par) * P * a.xrows * RS;
#pragma unroll
      for (int h = 0; h < H; ++h) {
        if (h >= nr) continue;
        float M = -INFINITY;
        #pragma unroll 1
        for (int r = 0; r < P; ++r) M = fmaxf(M, ld_cg(xb + (size_t(r) * a.xrows + q_row + h) * RS + D));
        float l = 0.f, o[J];
#pragma unroll
        for (int jj = 0; jj < J; ++jj) o[jj] = 0.f;
        #pragma unroll 1
        for (int r = 0; r < P; ++r) {
          const float* src = xb + (size_t(r) * a.xrows + q_row + h) * RS;
          const float w = ex2_sub(ld_cg(src + D), M);
          l += w;
          float rv[J];
          ldv_cg<J>(src + J * lane, rv);
#pragma unroll
          for (int jj = 0; jj < J; ++jj) o[jj] = fmaf(w, rv[jj], o[jj]);
        }
        const float inv = 1.f / l;
        stv<J>(a.out + size_t(q_row + h) * D + J * lane, o, inv);
        if (lane == 0 && a.lse) a.lse[q_row + h] = (M + log2f(l)) * kLn2;
      }
    };
    auto write_out = [&](int q_row, int unit) {  // O = diag(l)^-1 O; L = m + log(l) (Alg2§38-39, C2)
      if (a.xw > 1) {
        xchg_out(q_row, unit);
        return;
      }
      // lane h computes row h's 1 / l and log2 l (the same operations as a per-row loop, so
      // the same bits): one division and one logarithm of latency instead of H serial ones
      float lsel = acc.l[0], msel = acc.m[0];
#pragma unroll
      for (int h = 1; h < H; ++h)
        if (lane == h) {
          lsel = acc.l[h];
          msel = acc.m[h];
        }
      const float inv_lane = a.out_scale / lsel;  // V = codes x v_scale (FP8 KV; 1 otherwise)
      const float l2_lane = msel + log2f(lsel);
      float* dst = a.out + size_t(q_row) * D + J * lane;
#pragma unroll
      for (int h = 0; h < H; ++h) {
        const float inv = H == 1 ? inv_lane : __shfl_sync(0xffffffffu, inv_lane, h);
        if (h < nr) stv<J>(dst + h * D, acc.o[h], inv);
      }
      if (a.lse && lane < H && lane < nr) a.lse[q_row + lane] = l2_lane * kLn2;
    };

    for (int seg = 0;; ++seg) {
      const int b = seg % kFB;
      mbar_wait(&fold_full[b], (seg / kFB) & 1);
      const SegInfo si = seginfo[b];
      if (si.unit < 0) break;
      if (tr && lane == 0) {
#ifndef LA_PROF
        tr[TR_STREAM] = globaltimer();                 // the consumers finished this segment
#endif
        if (dynamic) tr[TR_PUBLISH] = globaltimer();   // dynamic: the last segment taken
      }
      // ---- fold the consumer warps' partials of this segment ------------------------------
      const float* fb = fold + b * FOLD_FLOATS;
#pragma unroll
      for (int h = 0; h < H; ++h) {
        float mx = -INFINITY;
        float l = 0.f, o[J];
#pragma unroll
        for (int jj = 0; jj < J; ++jj) o[jj] = 0.f;
        // every load of the row first (with global fold buffers -- wide tiles -- a dependent
        // max -> weights -> rows chain cost two L2 round trips per row)
        float mw[NWG * FW], lw[NWG * FW], ow[NWG * FW][J];
#pragma unroll
        for (int cw = 0; cw < NWG * FW; ++cw) {
          // Summed in the order of the warp sets RELATIVE to the segment's first stage: warp
          // (set (s0 + c) % NWG, sub) holds the segment's stages c, c + NWG, ... whatever s0
          // is, so the rounding depends only on the segment, never on where the ring stood
          // when it began (dynamic claims need no ring alignment; reading C16).
          const int w = ((si.s0 + cw / FW) % NWG) * FW + cw % FW;
          const float* r = fb + (w * H + h) * (D + 4);
          const float2 ml = *reinterpret_cast<const float2*>(r + D);
          mw[cw] = ml.x;
          lw[cw] = ml.y;
          ldv<J>(r + J * lane, ow[cw]);
        }
#pragma unroll
        for (int cw = 0; cw < NWG * FW; ++cw) mx = fmaxf(mx, mw[cw]);
#pragma unroll
        for (int cw = 0; cw < NWG * FW; ++cw) {
          const float wt = ex2_sub(mw[cw], mx);  // idle warp / masked row: m = -inf -> 0
          l = fmaf(wt, lw[cw], l);
#pragma unroll
          for (int jj = 0; jj < J; ++jj) o[jj] = fmaf(wt, ow[cw][jj], o[jj]);
        }
        acc.m[h] = mx;
        acc.l[h] = l;
#pragma unroll
        for (int jj = 0; jj < J; ++jj) acc.o[h][jj] = o[jj];
      }
      __syncwarp();
      const DevUnit u = a.units[si.unit];
      const int v = si.v;
      nr = u.rows;
      // a dynamic last arriver may stage its peers in this (consumed) fold buffer: release later
      const bool keep_fb = dynamic && !(si.host && si.finishing);
      if (!keep_fb && lane == 0) mbar_arrive(&fold_empty[b]);  // consumers may refill it

      // Every path below ends in at most one fold loop and one write_out: ONE call site
      // each keeps the epilogue code small (it runs rarely; an inlined copy per path blew
      // the kernel up to 48k instructions and its folds ran from instruction-cache misses).
      bool out = si.host && si.finishing;  // one (virtual) CTA computed the whole unit (Alg2§38-39)
      int fp0 = 0, fp1 = -1, fhv = -1;
      float* fstg = nullptr;
      int fn = 0;
      if (out) {
      } else if (!dynamic) {
        if (!si.host) {
          // ---- static, non-host: StorePartials + Signal(flags[g]) (Alg2§19-23) -----------
          store_partial(v);
          if (lane == 0) {
            st_release_gpu(&a.flags[v], epoch);
            if (tr && !tr[TR_PUBLISH]) tr[TR_PUBLISH] = globaltimer();
          }
        } else {
          // ---- static host, not finishing: Wait(flags[cta]) for cta = g+1 .. last_cta
          //      (Alg2§26-28, reading C9), lanes poll peers in parallel; fold ascending -----
          if (tr && lane == 0) tr[TR_WAIT0] = globaltimer();
#pragma unroll 1
          for (int p = v + 1 + lane; p <= u.last_cta; p += 32) {
            const unsigned long long t0 = globaltimer();
            while (ld_acquire_gpu(&a.flags[p]) != epoch) {
              __nanosleep(20);
              // a protocol bug or a missing peer must not hang the device: give up after
              // kWaitTimeoutNs (or at once after another wait did), report via la_plan_status
              if (globaltimer() - t0 > kWaitTimeoutNs || *reinterpret_cast<volatile int*>(&a.counters[CTR_ERROR])) {
                atomicExch(&a.counters[CTR_ERROR], 1);
                break;
              }
            }
          }
          __syncwarp();
          if (tr && lane == 0) tr[TR_WAIT1] = globaltimer();
          fp0 = v + 1;
          fp1 = u.last_cta;
          fstg = reinterpret_cast<float*>(ring);  // idle: this is the CTA's last segment
          fn = Smem<E>::RING / 4;
        }
      } else {
        // ---- dynamic: publish, count in; the unit's LAST arriving piece folds all of the
        //      unit's pieces (virtual CTAs host_cta .. last_cta) in ascending order --
        //      deterministic (fixed pieces, fixed order), and nobody waits
        fhv = u.host_cta;
        store_partial(v + (si.host ? SS : 0));
        int last = 0;
        if (lane == 0) {
          if (atomicAdd(&a.unit_count[si.unit], 1) == u.last_cta - fhv) {
            __threadfence();
            a.unit_count[si.unit] = 0;  // ready for the next launch
            last = 1;
          }
#ifdef LA_EPI_TRACE  // debug builds: when the last segment's publish + count-in completed
          if (tr) tr[TR_WAIT0] = globaltimer();
#endif
        }
        if (__shfl_sync(0xffffffffu, last, 0)) {
          fp0 = fhv;
          fp1 = u.last_cta;
          // the ring is idle once this CTA has consumed every stage its producer will issue:
          // one staging round for all pieces; else this segment's consumed fold buffer
          const bool ring_free = *reinterpret_cast<volatile int*>(prod_j) == si.jend;
          fstg = ring_free ? reinterpret_cast<float*>(ring) : fold + b * FOLD_FLOATS;
          fn = ring_free ? Smem<E>::RING / 4 : FOLD_FLOATS;
        }
      }
      if (fstg) {
        if (dynamic) reset();
        fold_smem(fp0, fp1, fhv, fstg, fn);
        out = true;
#ifdef LA_EPI_TRACE  // debug builds: when the last fold completed
        if (dynamic && tr && lane == 0) tr[TR_WAIT1] = globaltimer();
#endif
      }
      if (!dynamic && fstg && tr && lane == 0) tr[TR_PUBLISH] = globaltimer();  // host: fold done
      if (out) write_out(u.q_row, si.unit);
      if (keep_fb) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&fold_empty[b]);  // staging done: consumers may refill it
      }
    }
    if (lane == 0) {
      if (tr) tr[TR_END] = globaltimer();
      if (dynamic) {  // the last CTA out resets the claim counter for the next launch
        __threadfence();
        if (atomicAdd(&a.counters[CTR_DONE], 1) == int(gridDim.x) - 1) {
          a.counters[CTR_CLAIM] = 0;
          a.counters[CTR_DONE] = 0;
        }
      }
      __threadfence();  // every flag wait of this CTA is over: the last one out advances the epoch
      if (atomicAdd(&a.counters[CTR_EXITED], 1) == int(gridDim.x) - 1) {
        a.counters[CTR_EXITED] = 0;
        *reinterpret_cast<volatile uint32_t*>(&a.counters[CTR_EPOCH]) = epoch;
        if (a.xw > 1) *reinterpret_cast<volatile uint32_t*>(&a.counters[CTR_XEPOCH]) = xepoch;
        __threadfence();
      }
    }
    return;
  }

  // ================================= consumers ==========================================
  const int my_wg = warp / WPS, sub = warp % WPS;  // warp set (= ring slot when NWG == NST)
  int j = 0, k = 0, seg = 0;
#ifdef LA_PROF  // trace fields reused: (publish, wait0, wait1) = consumer warp 0's cycles waiting
  long long prof_wait = 0, prof_work = 0, prof_n = 0;  // for data, in stage(), stages
#endif
  // Give this warp's segment partial to the epilogue warp (double-buffered): wait for a free
  // fold buffer, E::seg_end writes it (called in the loop body, so the State never has its
  // address taken and stays in registers), then signal.
  auto hand_off_wait = [&]() {
    const int b = seg % kFB;
    if (seg >= kFB) mbar_wait(&fold_empty[b], ((seg / kFB) - 1) & 1);
    return b;
  };
  auto hand_off = [&](int b, int v, int unit, int host, int finishing, int s0) {
    if (warp == 0 && lane == 0) seginfo[b] = SegInfo{v, unit, host, finishing, s0, j};
    __syncwarp();
    if (lane == 0) mbar_arrive(&fold_full[b]);
    ++seg;
  };
  for (;;) {
    const int qi = k % kQD;
    mbar_wait(&sq_full[qi], (k / kQD) & 1);
    const SegQ e = squeue[qi];
    const DevUnit u = e.u;
    const int v = e.v;
    if (v < 0) break;
    int it = e.it;
    const int seg_end = e.it_end;
#ifndef LA_EPI_TRACE
    if (dynamic && tr && threadIdx.x == 0) tr[TR_WAIT1] += seg_end - it;  // dynamic: LeanTiles per CTA
#endif
    typename E::State st;
    E::seg_begin(st, a, u, lane, Smem<E>::QB ? static_cast<const void*>(qbuf + qi * Smem<E>::QB)
                                            : static_cast<const void*>(static_cast<const unsigned char*>(a.q) +
                                                                       size_t(u.q_row) * D * sizeof(typename E::QElem)));
    __syncwarp();
    if (lane == 0) mbar_arrive(&sq_empty[qi]);  // entry and Q rows read
    ++k;
    const int seg_s0 = j % NWG;
    for (; it < seg_end; ++it) {
      const int t0 = (it - u.iter_begin) * a.tile_n;
      const int t1 = min(t0 + a.tile_n, u.len);
      for (int s0 = t0; s0 < t1; s0 += a.stage_tokens) {
        if (j % NWG == my_wg) {
          const int rs = j % NST;  // ring slot of stage j
#ifdef LA_PROF
          const long long c0 = clock64();
#endif
          // NWG < NST: slot rs last held stage j - NST of ANOTHER warp set; wait for its
          // release first, so the full-barrier parity below cannot alias that older phase
          if (NWG < NST && j >= NST) mbar_wait(&empty[rs], uint32_t((j / NST) - 1) & 1u);
          mbar_wait(&full[rs], (j / NST) & 1);
#ifdef LA_PROF
          const long long c1 = clock64();
          prof_wait += c1 - c0;
          ++prof_n;
#endif
          if constexpr (EngX<E>::TMEM > 0) {  // the engine releases the slot itself
            E::stage(st, ring + rs * E::STAGE_BYTES, sub, min(a.stage_tokens, t1 - s0), s0, a.scale_log2,
                     lane, a.box_shift, (uint32_t(j / NST) & 1u) | ((uint32_t(j / NWG) & 1u) << 1), &empty[rs]);
          } else {
            E::stage(st, ring + rs * E::STAGE_BYTES, sub, min(a.stage_tokens, t1 - s0), s0, a.scale_log2,
                     lane, a.box_shift);
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[rs]);
          }
#ifdef LA_PROF
          prof_work += clock64() - c1;
#endif
        }
        ++j;
      }
    }
    const int fbuf = hand_off_wait();
    E::seg_end(st, fold + fbuf * FOLD_FLOATS, warp, lane);
    hand_off(fbuf, v, e.unit, e.host, e.finishing, seg_s0);
  }
  hand_off(hand_off_wait(), -1, -1, 0, 0, 0);  // terminator for the epilogue
#ifdef LA_PROF
  if (tr && threadIdx.x == 0) {
    tr[TR_PUBLISH] = prof_wait;
    tr[TR_WAIT0] = prof_work;
    tr[TR_WAIT1] = prof_n;
  }
#endif
  if constexpr (EngX<E>::TMEM > 0) {  // every consumer's tcgen05 work is done: free TMEM
    tc5::fence_before();
    asm volatile("bar.sync 1, %0;" ::"r"(NCW * 32) : "memory");
    if (warp == 0) {
      tc5::fence_after();
      tc5::tmem_dealloc(*E::tmem_base_ptr(), EngX<E>::TMEM);
    }
  }
}

template <class E>
KernelInfo info_of(bool tma) {
  KernelInfo k;
  k.supported = true;
  k.threads = (E::NCW + 1 + EngX<E>::NEP) * 32;  // consumers, producer, epilogue warp(s)
  static_assert(Smem<E>::BYTES <= 232448, "dynamic shared memory exceeds 227 KiB per block");
  k.smem_bytes = Smem<E>::BYTES;
  k.stage_tokens_max = E::STAGE_TOK;
  k.uses_tma_tensor = tma;
  k.fn = reinterpret_cast<const void*>(&la_decode<E>);
  if constexpr (EngX<E>::TMEM > 0) k.box_halves = E::BOX_HALVES;
  if constexpr (EngX<E>::GF) k.global_fold_floats = E::FOLD_BUFS * E::FOLD_FLOATS;
  return k;
}

}  // namespace

// One function per engine family (each defined in its own translation unit).
KernelInfo info_mha(int dtype, int head_dim);
KernelInfo info_gqa(int dtype, int head_dim);
KernelInfo info_fp8(int head_dim, int group);
KernelInfo info_tc5_bf16(int group);
KernelInfo info_tc5_fp16(int group);

}  // namespace la
