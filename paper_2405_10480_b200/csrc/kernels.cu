// sm_100a kernels of libleanattn.so.
//
//  la_decode_mha<T, D, NST, WPS>  -- LeanAttention decode, one persistent launch:
//      stream-K segment walk (Alg2§10-18, §41) + LeanTile online softmax (Alg. 1) +
//      in-kernel fixup through global partials and epoch flags (Alg2§19-36) + finalize
//      (Alg2§38-39).  MHA (T_m = group = 1), CUDA-core fp32 arithmetic.
//  la_combine_kernel<D>           -- sequence-shard combine of (O_r, L_r) (§4.1 operator).
//
// Design:
//  * the last warp (one elected lane) is the producer: it walks the CTA's iteration range and
//    streams each stage (<= 64 tokens of K and V, contiguous in both layouts) HBM -> SMEM
//    with two 1-D TMA bulk copies (cp.async.bulk, SASS UBLKCP) into an NST-deep ring
//    guarded by full/empty mbarriers; L2 evict-first (KV is read exactly once).
//  * NCW = NST * WPS consumer warps: WPS warps own each ring slot and split its 32-key
//    rounds; each warp keeps its own (m, l, O) state (§4.1 partial) and the warps are
//    folded with the re-scaling operator once per segment, so there is no CTA-wide barrier
//    per tile.
//  * QK^T: a key is split over LPK = row_bytes/16 lanes (16 B = one LDS.128 each); every lane
//    accumulates LPK keys' partial dot products with FHFMA (bf16/fp16 x bf16/fp16 + fp32,
//    exact products, fp32 accumulate) and an XOR transpose-butterfly (LPK-1 shuffles, no
//    selects) leaves the full score of key li in lane li.
//  * online softmax in the exp2 domain (scale*log2e folded into one multiply per key);
//    PV with FFMA2 (packed fp32x2) on bf16 -> fp32 widened V.
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <atomic>
#include <cstdint>
#include <string>

#include "la_internal.h"
#include "ptx.cuh"

namespace la {

static std::atomic<int64_t> g_launches{0};
int64_t launch_count() { return g_launches.load(); }
void note_launch() { g_launches.fetch_add(1); }

namespace {

using namespace dev;

// ---------------------------------------------------------------------------------------
// Per-dtype 16-byte chunk arithmetic.
//   dot : acc + sum_e q[e] * k[e] over the chunk's EPL elements (fp32 result)
//   axpy: o[e] += p * v[e]                                         (fp32 accumulators)
// ---------------------------------------------------------------------------------------
template <typename T>
struct Chunk;

template <>
struct Chunk<__nv_bfloat16> {
  static constexpr int EPL = 8;
  struct Q {
    unsigned short h[8];  // one bf16 per entry (exact input values)
  };
  __device__ __forceinline__ static Q load_q(const void* p) {
    const uint4 w = *reinterpret_cast<const uint4*>(p);
    Q q;
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      q.h[2 * i] = static_cast<unsigned short>(ws[i] & 0xffffu);
      q.h[2 * i + 1] = static_cast<unsigned short>(ws[i] >> 16);
    }
    return q;
  }
  // FHFMA.BF16: bf16 x bf16 product is exact in fp32, one rounding on the add.
  __device__ __forceinline__ static float dot(const uint4 k, const Q& q, float acc) {
    asm("{\n\t.reg .b16 l0, h0, l1, h1, l2, h2, l3, h3;\n\t"
        "mov.b32 {l0, h0}, %1;\n\tmov.b32 {l1, h1}, %2;\n\t"
        "mov.b32 {l2, h2}, %3;\n\tmov.b32 {l3, h3}, %4;\n\t"
        "fma.rn.f32.bf16 %0, l0, %5, %0;\n\t"
        "fma.rn.f32.bf16 %0, h0, %6, %0;\n\t"
        "fma.rn.f32.bf16 %0, l1, %7, %0;\n\t"
        "fma.rn.f32.bf16 %0, h1, %8, %0;\n\t"
        "fma.rn.f32.bf16 %0, l2, %9, %0;\n\t"
        "fma.rn.f32.bf16 %0, h2, %10, %0;\n\t"
        "fma.rn.f32.bf16 %0, l3, %11, %0;\n\t"
        "fma.rn.f32.bf16 %0, h3, %12, %0;\n\t}"
        : "+f"(acc)
        : "r"(k.x), "r"(k.y), "r"(k.z), "r"(k.w), "h"(q.h[0]), "h"(q.h[1]), "h"(q.h[2]), "h"(q.h[3]),
          "h"(q.h[4]), "h"(q.h[5]), "h"(q.h[6]), "h"(q.h[7]));
    return acc;
  }
  __device__ __forceinline__ static void axpy(float p, const uint4 v, float2 (&o)[4]) {
    const float2 pp = make_float2(p, p);
    const uint32_t ws[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 vv = make_float2(__uint_as_float(ws[i] << 16), __uint_as_float(ws[i] & 0xffff0000u));
      o[i] = __ffma2_rn(pp, vv, o[i]);
    }
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
    Q q;
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
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
        "fma.rn.f32.f16 %0, l0, %5, %0;\n\t"
        "fma.rn.f32.f16 %0, h0, %6, %0;\n\t"
        "fma.rn.f32.f16 %0, l1, %7, %0;\n\t"
        "fma.rn.f32.f16 %0, h1, %8, %0;\n\t"
        "fma.rn.f32.f16 %0, l2, %9, %0;\n\t"
        "fma.rn.f32.f16 %0, h2, %10, %0;\n\t"
        "fma.rn.f32.f16 %0, l3, %11, %0;\n\t"
        "fma.rn.f32.f16 %0, h3, %12, %0;\n\t}"
        : "+f"(acc)
        : "r"(k.x), "r"(k.y), "r"(k.z), "r"(k.w), "h"(q.h[0]), "h"(q.h[1]), "h"(q.h[2]), "h"(q.h[3]),
          "h"(q.h[4]), "h"(q.h[5]), "h"(q.h[6]), "h"(q.h[7]));
    return acc;
  }
  __device__ __forceinline__ static void axpy(float p, const uint4 v, float2 (&o)[4]) {
    const float2 pp = make_float2(p, p);
    const uint32_t ws[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __half2 h2 = *reinterpret_cast<const __half2*>(&ws[i]);
      o[i] = __ffma2_rn(pp, __half22float2(h2), o[i]);
    }
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
    acc = fmaf(__uint_as_float(k.w), q.f[3], acc);
    return acc;
  }
  __device__ __forceinline__ static void axpy(float p, const uint4 v, float2 (&o)[2]) {
    const float2 pp = make_float2(p, p);
    o[0] = __ffma2_rn(pp, make_float2(__uint_as_float(v.x), __uint_as_float(v.y)), o[0]);
    o[1] = __ffma2_rn(pp, make_float2(__uint_as_float(v.z), __uint_as_float(v.w)), o[1]);
  }
};

// ---------------------------------------------------------------------------------------
// Compile-time configuration of the MHA kernel.
// ---------------------------------------------------------------------------------------
template <typename T, int D, int NST, int WPS>
struct MhaCfg {
  static constexpr int NCW = NST * WPS;                     // consumer warps (WPS per slot)
  static constexpr int ROWB = D * int(sizeof(T));          // bytes of one K (or V) row
  static constexpr int LPK = ROWB / 16;                     // lanes per key
  static constexpr int EPL = 16 / int(sizeof(T));           // elements per lane chunk
  static constexpr int STAGE_TOK = 32768 / (2 * ROWB);      // tokens per ring stage (32 KiB K+V)
  static constexpr int STAGE_BYTES = 2 * STAGE_TOK * ROWB;
  static constexpr int FOLD_FLOATS = NCW * (D + 2);         // per-warp (O[D], m, l)
  static constexpr int THREADS = (NCW + 1) * 32;
  static constexpr int SMEM = NST * STAGE_BYTES + 2 * FOLD_FLOATS * 4 + 2 * NST * 8;
  static_assert(LPK >= 2 && LPK <= 32 && (LPK & (LPK - 1)) == 0, "lanes per key");
  static_assert(STAGE_TOK % 32 == 0, "stage must hold whole 32-key rounds");
  static_assert(D <= NCW * 32, "one consumer thread per output dim in the fold");
};

// One ring stage: ntok (<= STAGE_TOK) keys of one unit.  Updates this warp's (m, l, o).
template <typename T, int D, int NST, int WPS>
__device__ __forceinline__ void process_stage(const unsigned char* __restrict__ st, int r0, int ntok,
                                              const typename Chunk<T>::Q& qf, float scale_log2, int kg,
                                              int li, float& m, float& l,
                                              float2 (&o)[Chunk<T>::EPL / 2]) {
  using C = MhaCfg<T, D, NST, WPS>;
  constexpr int LPK = C::LPK;
  const unsigned char* ks = st;
  const unsigned char* vs = st + C::STAGE_TOK * C::ROWB;
  for (int r = r0; r < ntok; r += 32 * WPS) {  // this warp's 32-key rounds of the stage
    const int kb = r + kg * LPK;  // first key of this lane group in the round
    // ---- S_f = Q_f K_f^T (Alg1§20): lane li accumulates key (jj ^ li), chunk li ----------
    float acc[LPK];
#pragma unroll
    for (int jj = 0; jj < LPK; ++jj) {
      const uint4 w = *reinterpret_cast<const uint4*>(ks + (kb + (jj ^ li)) * C::ROWB + li * 16);
      acc[jj] = Chunk<T>::dot(w, qf, 0.f);
    }
    // XOR transpose-butterfly: afterwards acc[0] of lane li is the full dot of key kb + li
#pragma unroll
    for (int off = LPK / 2; off >= 1; off >>= 1) {
#pragma unroll
      for (int jj = 0; jj < off; ++jj) acc[jj] += __shfl_xor_sync(0xffffffffu, acc[jj + off], off);
    }
    const float s = (kb + li < ntok) ? acc[0] * scale_log2 : -INFINITY;  // reading C5 (mask tail)
    // ---- m_new = max(m, rowmax S_f) (Alg1§21) -------------------------------------------
    float mr = s;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) mr = fmaxf(mr, __shfl_xor_sync(0xffffffffu, mr, off));
    if (mr > m) {  // warp-uniform; e^{m - m_new} rescale of l and O_acc (Alg1§23-24)
      const float alpha = ex2(m - mr);
      l *= alpha;
      const float2 aa = make_float2(alpha, alpha);
#pragma unroll
      for (int e = 0; e < Chunk<T>::EPL / 2; ++e) o[e] = __fmul2_rn(aa, o[e]);
      m = mr;
    }
    // ---- P_f = exp(S_f - m_new); l += rowsum(P_f) (Alg1§22-23) ----------------------------
    const float p = ex2(s - m);
    l += p;
    // ---- O_acc += P_f V_f (Alg1§24): lane li owns dims [li*EPL, li*EPL+EPL) --------------
#pragma unroll
    for (int jj = 0; jj < LPK; ++jj) {
      const float pj = __shfl_sync(0xffffffffu, p, jj, LPK);
      const uint4 w = *reinterpret_cast<const uint4*>(vs + (kb + jj) * C::ROWB + li * 16);
      Chunk<T>::axpy(pj, w, o);
    }
  }
}

template <typename T, int D, int NST, int WPS>
__global__ void __launch_bounds__(MhaCfg<T, D, NST, WPS>::THREADS, 1)
    la_decode_mha(const DecodeArgs a) {
  using C = MhaCfg<T, D, NST, WPS>;
  constexpr int NCW = C::NCW;
  using E = Chunk<T>;
  constexpr int EPL = C::EPL;
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char* ring = smem;
  float* fold = reinterpret_cast<float*>(smem + NST * C::STAGE_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(fold + 2 * C::FOLD_FLOATS);
  uint64_t* empty = full + NST;

  // warp index broadcast from lane 0 so the compiler knows it is warp-uniform
  const int warp = __shfl_sync(0xffffffffu, int(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int g = blockIdx.x;
  const int it0 = a.cta_begin[g], it1 = a.cta_begin[g + 1];
  if (it0 >= it1) return;  // idle CTA (G > I); no barrier below involves it
  unsigned long long* tr = a.trace ? a.trace + size_t(g) * TR_FIELDS : nullptr;
  if (tr && threadIdx.x == 0) {
    tr[TR_SMID] = smid();
    tr[TR_START] = globaltimer();
    tr[TR_PUBLISH] = tr[TR_WAIT0] = tr[TR_WAIT1] = 0;
  }

  // Zero the ring once so rows past the end of a short stage are finite on first use
  // (their scores are masked to -inf, p = 0, and 0 * finite = 0).
  for (int i = threadIdx.x; i < NST * C::STAGE_BYTES / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(ring)[i] = make_uint4(0u, 0u, 0u, 0u);
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], WPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // zero-fill before TMA writes
  __syncthreads();

  if (warp == NCW) {
    // =============================== producer ===========================================
    if (lane == 0) {
      const uint64_t pol = l2_evict_first_policy();
      const unsigned char* gk = static_cast<const unsigned char*>(a.k);
      const unsigned char* gv = static_cast<const unsigned char*>(a.v);
      int j = 0;
      int unit = a.cta_first_unit[g];
      for (int it = it0; it < it1;) {
        const DevUnit u = a.units[unit];
        if (u.iter_end <= it) {
          ++unit;
          continue;
        }
        const int seg_end = min(u.iter_end, it1);
        for (; it < seg_end; ++it) {  // LeanTile iterations of this segment (Alg1§13)
          const int t0 = (it - u.iter_begin) * a.tile_n;  // kk = iter * T_n  (Alg1§14)
          const int t1 = min(t0 + a.tile_n, u.len);
          for (int s0 = t0; s0 < t1; s0 += a.stage_tokens) {  // LoadFragment K, V (Alg1§17-18)
            const int ntok = min(a.stage_tokens, t1 - s0);
            const int slot = j % NST;
            if (j >= NST) mbar_wait(&empty[slot], ((j / NST) - 1) & 1);
            const uint32_t bytes = uint32_t(ntok) * C::ROWB;
            mbar_arrive_expect_tx(&full[slot], 2 * bytes);
            const size_t goff = size_t(u.row0 + s0) * C::ROWB;
            unsigned char* dst = ring + slot * C::STAGE_BYTES;
            bulk_g2s(dst, gk + goff, bytes, &full[slot], pol);
            bulk_g2s(dst + C::STAGE_TOK * C::ROWB, gv + goff, bytes, &full[slot], pol);
            ++j;
          }
        }
        ++unit;
      }
    }
    return;
  }

  // ================================= consumers ==========================================
  // Consumer warp w owns ring slot w / WPS and takes rounds (w % WPS), (w % WPS) + WPS, ...
  // of every stage landing in that slot.  Fixed slot ownership keeps each slot's consumers
  // in stage order, so a wait on the slot's next phase can never alias the previous one.
  const int NCT = NCW * 32;
  const int my_slot = warp / WPS, sub = warp % WPS;
  const int kg = lane / C::LPK, li = lane % C::LPK;
  const int t = threadIdx.x;  // 0 .. NCT-1
  int j = 0, seg = 0;
  int unit = a.cta_first_unit[g];
  for (int it = it0; it < it1;) {
    const DevUnit u = a.units[unit];
    if (u.iter_end <= it) {
      ++unit;
      continue;
    }
    const int seg_end = min(u.iter_end, it1);
    const bool host = (it == u.iter_begin);      // host-block (Alg2§17)
    const bool finishing = (it1 >= u.iter_end);  // finishing-block (Alg2§18)
    const typename E::Q qf = E::load_q(static_cast<const T*>(a.q) + size_t(u.q_row) * D + li * EPL);
    float m = -INFINITY, l = 0.f;                // Alg1§8-9 (per warp)
    float2 o[EPL / 2];
#pragma unroll
    for (int e = 0; e < EPL / 2; ++e) o[e] = make_float2(0.f, 0.f);

    for (; it < seg_end; ++it) {
      const int t0 = (it - u.iter_begin) * a.tile_n;
      const int t1 = min(t0 + a.tile_n, u.len);
      for (int s0 = t0; s0 < t1; s0 += a.stage_tokens) {
        if (j % NST == my_slot) {
          const int ntok = min(a.stage_tokens, t1 - s0);
          mbar_wait(&full[my_slot], (j / NST) & 1);
          process_stage<T, D, NST, WPS>(ring + my_slot * C::STAGE_BYTES, sub * 32, ntok, qf, a.scale_log2,
                                        kg, li, m, l, o);
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[my_slot]);
        }
        ++j;
      }
    }

    // ---- segment end: fold lane groups, then warps, with the re-scaling operator --------
#pragma unroll
    for (int off = C::LPK; off < 32; off <<= 1) {
#pragma unroll
      for (int e = 0; e < EPL / 2; ++e) {
        o[e].x += __shfl_xor_sync(0xffffffffu, o[e].x, off);
        o[e].y += __shfl_xor_sync(0xffffffffu, o[e].y, off);
      }
    }
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) l += __shfl_xor_sync(0xffffffffu, l, off);
    float* fb = fold + (seg & 1) * C::FOLD_FLOATS;
    if (kg == 0) {
#pragma unroll
      for (int e = 0; e < EPL / 2; ++e) {
        fb[warp * (D + 2) + li * EPL + 2 * e] = o[e].x;
        fb[warp * (D + 2) + li * EPL + 2 * e + 1] = o[e].y;
      }
    }
    if (lane == 0) {
      fb[warp * (D + 2) + D] = m;
      fb[warp * (D + 2) + D + 1] = l;
    }
    consumer_bar(NCT);
    float mstar = -INFINITY;
#pragma unroll
    for (int w = 0; w < NCW; ++w) mstar = fmaxf(mstar, fb[w * (D + 2) + D]);
    float lsum = 0.f, oc = 0.f;
#pragma unroll
    for (int w = 0; w < NCW; ++w) {
      const float wt = ex2(fb[w * (D + 2) + D] - mstar);  // idle warp: m = -inf -> 0
      lsum = fmaf(wt, fb[w * (D + 2) + D + 1], lsum);
      if (t < D) oc = fmaf(wt, fb[w * (D + 2) + t], oc);
    }

    if (!host) {
      // ---- non-host: StorePartials(Op[g], mp[g], lp[g]); Signal(flags[g]) (Alg2§19-23) --
      if (t < D) a.part_o[size_t(g) * D + t] = oc;
      if (t == 0) {
        a.part_ml[2 * g] = mstar;
        a.part_ml[2 * g + 1] = lsum;
      }
      consumer_bar(NCT);
      if (t == 0) {
        __threadfence();
        st_release_gpu(&a.flags[g], a.epoch);
        if (tr) tr[TR_PUBLISH] = globaltimer();
      }
    } else {
      if (!finishing) {
        // ---- host, not finishing: Wait(flags[cta]) for cta = g+1 .. last_cta (Alg2§26-28,
        //      reading C9), polled in parallel, then fold in ascending order (§29-35) -----
        if (tr && t == 0) tr[TR_WAIT0] = globaltimer();
        for (int p = g + 1 + t; p <= u.last_cta; p += NCT) {
          while (ld_acquire_gpu(&a.flags[p]) != a.epoch) __nanosleep(20);
        }
        consumer_bar(NCT);
        if (tr && t == 0) tr[TR_WAIT1] = globaltimer();
        for (int p = g + 1; p <= u.last_cta; ++p) {
          const float mp = ld_cg(&a.part_ml[2 * p]);
          const float lp = ld_cg(&a.part_ml[2 * p + 1]);
          const float op = (t < D) ? ld_cg(&a.part_o[size_t(p) * D + t]) : 0.f;
          const float mn = fmaxf(mstar, mp);
          const float wa = ex2(mstar - mn), wb = ex2(mp - mn);
          oc = wa * oc + wb * op;
          lsum = wa * lsum + wb * lp;
          mstar = mn;
        }
      }
      // ---- Write O = diag(l)^-1 O; L = m + log(l) (Alg2§38-39), natural log (C2) -------
      if (t < D) a.out[size_t(u.q_row) * D + t] = oc / lsum;
      if (t == 0 && a.lse) a.lse[u.q_row] = (mstar + log2f(lsum)) * kLn2;
    }
    ++seg;
    ++unit;
  }
  if (tr && t == 0) tr[TR_END] = globaltimer();
}

// ---------------------------------------------------------------------------------------
// Sequence-shard combine: L = ln sum_r e^{L_r}, O = sum_r e^{L_r - L} O_r  (ascending r)
// ---------------------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(D) la_combine_kernel(const float* __restrict__ o_parts,
                                                       const float* __restrict__ lse_parts, int parts,
                                                       int rows, float* __restrict__ out,
                                                       float* __restrict__ lse) {
  const int r = blockIdx.x, c = threadIdx.x;
  float mx = -INFINITY;
  for (int p = 0; p < parts; ++p) mx = fmaxf(mx, lse_parts[size_t(p) * rows + r]);
  float s = 0.f, acc = 0.f;
  for (int p = 0; p < parts; ++p) {
    const float w = expf(lse_parts[size_t(p) * rows + r] - mx);
    s += w;
    acc = fmaf(w, o_parts[(size_t(p) * rows + r) * D + c], acc);
  }
  out[size_t(r) * D + c] = acc / s;
  if (c == 0 && lse) lse[r] = mx + logf(s);
}

template <typename T, int D>
KernelInfo mha_info() {
  constexpr int NST = 6, WPS = 2;
  using C = MhaCfg<T, D, NST, WPS>;
  KernelInfo k;
  k.supported = true;
  k.threads = C::THREADS;
  k.smem_bytes = C::SMEM;
  k.stage_tokens_max = C::STAGE_TOK;
  k.fn = reinterpret_cast<const void*>(&la_decode_mha<T, D, NST, WPS>);
  return k;
}

}  // namespace

KernelInfo decode_kernel_info(int dtype, int head_dim, int group) {
  if (group != 1) return gqa_kernel_info(dtype, head_dim, group);
  if (dtype == LA_BF16 && head_dim == 128) return mha_info<__nv_bfloat16, 128>();
  if (dtype == LA_BF16 && head_dim == 64) return mha_info<__nv_bfloat16, 64>();
  if (dtype == LA_FP16 && head_dim == 128) return mha_info<__half, 128>();
  if (dtype == LA_FP16 && head_dim == 64) return mha_info<__half, 64>();
  if (dtype == LA_FP32 && head_dim == 128) return mha_info<float, 128>();
  if (dtype == LA_FP32 && head_dim == 64) return mha_info<float, 64>();
  return KernelInfo{};
}

int launch_decode(const KernelInfo& ki, const DecodeArgs& a, bool cooperative, void* stream,
                  std::string& err) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(a.grid);
  cfg.blockDim = dim3(ki.threads);
  cfg.dynamicSmemBytes = ki.smem_bytes;
  cfg.stream = static_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // hosts spin on peers: all CTAs co-resident
  attr[0].val.cooperative = cooperative ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  void* args[] = {const_cast<DecodeArgs*>(&a)};
  cudaError_t e = cudaLaunchKernelExC(&cfg, ki.fn, args);
  if (e != cudaSuccess) {
    err = std::string("decode launch: ") + cudaGetErrorString(e);
    cudaGetLastError();
    return 1;
  }
  g_launches.fetch_add(1);
  return 0;
}

int launch_combine(const float* o_parts, const float* lse_parts, int parts, int rows, int head_dim,
                   float* out, float* lse, void* stream, std::string& err) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (head_dim == 128)
    la_combine_kernel<128><<<rows, 128, 0, st>>>(o_parts, lse_parts, parts, rows, out, lse);
  else
    la_combine_kernel<64><<<rows, 64, 0, st>>>(o_parts, lse_parts, parts, rows, out, lse);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    err = std::string("combine launch: ") + cudaGetErrorString(e);
    return 1;
  }
  g_launches.fetch_add(1);
  return 0;
}

}  // namespace la
