// GQA decode kernel: LeanAttention (Alg. 1 + Alg. 2) where an output tile is the T_m = g
// query heads sharing one KV head (reading C3) -- a small dense contraction, so QK^T and PV
// run on the tensor cores.
//
//  * Swap-AB: S^T (16 tokens x 8 heads) = K_f (16 x d) . Q_f^T (d x 8) with mma.sync
//    m16n8k16 (bf16/fp16 in, fp32 accumulate): N = 8 is the GQA group itself, so no MMA
//    row is padding at g = 8 (g = 2, 4 pad N).  PV: O^T (d x 8) += V_f^T (d x 16) . P^T
//    (16 x 8); movmatrix.trans turns the S^T accumulator fragment straight into the P^T
//    B-operand (no shared-memory round trip).
//  * K/V stages arrive by TMA tensor loads (cp.async.bulk.tensor.2d, SASS UTMALDG) in the
//    128-byte swizzled layout, so ldmatrix (K) and ldmatrix.trans (V) are conflict-free.
//  * Producer / ring / slot ownership / segment walk / in-kernel fixup exactly as the MHA
//    kernel (kernels.cu); online softmax per head in the exp2 domain.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <mutex>
#include <string>

#include "la_internal.h"
#include "ptx.cuh"

namespace la {

struct alignas(64) TmapPair {
  CUtensorMap k;
  CUtensorMap v;
};

namespace {

using namespace dev;

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
};

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tm, int c0, int c1, uint64_t* bar,
                                            uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

template <int D, int NST, int WPS>
struct GqaCfg {
  static constexpr int NCW = NST * WPS;
  static constexpr int ST = 64;                   // stage tokens = TMA box rows
  static constexpr int NBOX = D / 64;             // 64-element (128 B) boxes per row
  static constexpr int BOX_BYTES = ST * 128;
  static constexpr int KV_BYTES = NBOX * BOX_BYTES;
  static constexpr int STAGE_BYTES = 2 * KV_BYTES;
  static constexpr int GN = 8;                    // heads per MMA N
  static constexpr int KSTEPS = D / 16;
  static constexpr int FOLD_O = NCW * GN * D;     // per-warp O^T[h][c]
  static constexpr int FOLD_ML = NCW * GN * 2;    // per-warp (m, l) per head
  static constexpr int THREADS = (NCW + 1) * 32;
  static constexpr int SMEM = 1024 + NST * STAGE_BYTES + (FOLD_O + FOLD_ML) * 4 + 2 * NST * 8;
  static_assert(ST == 32 * WPS, "one 32-token round per consumer warp per stage");
};

template <typename T, int D, int NST, int WPS>
__global__ void __launch_bounds__(GqaCfg<D, NST, WPS>::THREADS, 1)
    la_decode_gqa(const DecodeArgs a, const __grid_constant__ TmapPair tm) {
  using C = GqaCfg<D, NST, WPS>;
  constexpr int NCW = C::NCW, GN = C::GN, KS = C::KSTEPS;
  extern __shared__ unsigned char smem_raw[];
  // SWIZZLE_128B destinations need 1024-byte alignment
  unsigned char* ring =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* fold_o = reinterpret_cast<float*>(ring + NST * C::STAGE_BYTES);
  float* fold_ml = fold_o + C::FOLD_O;
  uint64_t* full = reinterpret_cast<uint64_t*>(fold_ml + C::FOLD_ML);
  uint64_t* empty = full + NST;

  const int warp = __shfl_sync(0xffffffffu, int(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int g = blockIdx.x;
  const int it0 = a.cta_begin[g], it1 = a.cta_begin[g + 1];
  if (it0 >= it1) return;
  unsigned long long* tr = a.trace ? a.trace + size_t(g) * TR_FIELDS : nullptr;
  if (tr && threadIdx.x == 0) {
    tr[TR_SMID] = smid();
    tr[TR_START] = globaltimer();
    tr[TR_PUBLISH] = tr[TR_WAIT0] = tr[TR_WAIT1] = 0;
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], WPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm.k)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm.v)) : "memory");
  }
  __syncthreads();

  if (warp == NCW) {
    // =============================== producer ===========================================
    if (lane == 0) {
      const uint64_t pol = l2_evict_first_policy();
      int j = 0;
      int unit = a.cta_first_unit[g];
      for (int it = it0; it < it1;) {
        const DevUnit u = a.units[unit];
        if (u.iter_end <= it) {
          ++unit;
          continue;
        }
        const int seg_end = min(u.iter_end, it1);
        for (; it < seg_end; ++it) {
          const int t0 = (it - u.iter_begin) * a.tile_n;
          const int t1 = min(t0 + a.tile_n, u.len);
          for (int s0 = t0; s0 < t1; s0 += a.stage_tokens) {
            const int slot = j % NST;
            if (j >= NST) mbar_wait(&empty[slot], ((j / NST) - 1) & 1);
            mbar_arrive_expect_tx(&full[slot], C::STAGE_BYTES);  // full boxes (OOB rows zero-filled)
            unsigned char* dst = ring + slot * C::STAGE_BYTES;
            const int row = int(u.row0 + s0);
#pragma unroll
            for (int b = 0; b < C::NBOX; ++b) {
              tma_load_2d(dst + b * C::BOX_BYTES, &tm.k, b * 64, row, &full[slot], pol);
              tma_load_2d(dst + C::KV_BYTES + b * C::BOX_BYTES, &tm.v, b * 64, row, &full[slot], pol);
            }
            ++j;
          }
        }
        ++unit;
      }
    }
    return;
  }

  // ================================= consumers ==========================================
  const int NCT = NCW * 32;
  const int my_slot = warp / WPS, sub = warp % WPS;
  const int gq = lane >> 2, tq = lane & 3;   // mma fragment row group / thread-in-group
  const int t = threadIdx.x;
  const int mi = lane >> 3, ri = lane & 7;   // ldmatrix: matrix index / row within matrix
  int j = 0;
  int unit = a.cta_first_unit[g];
  for (int it = it0; it < it1;) {
    const DevUnit u = a.units[unit];
    if (u.iter_end <= it) {
      ++unit;
      continue;
    }
    const int seg_end = min(u.iter_end, it1);
    const bool host = (it == u.iter_begin);
    const bool finishing = (it1 >= u.iter_end);
    // Q^T B-fragments (exact inputs): b0 = Q[h=gq][16kk + 2tq, +1], b1 = Q[gq][16kk + 8 + 2tq, +1]
    uint32_t qb[KS][2];
    {
      const uint32_t* qrow = reinterpret_cast<const uint32_t*>(static_cast<const T*>(a.q) +
                                                                size_t(u.q_row + gq) * D);
#pragma unroll
      for (int kk = 0; kk < KS; ++kk) {
        qb[kk][0] = gq < a.group ? qrow[8 * kk + tq] : 0u;
        qb[kk][1] = gq < a.group ? qrow[8 * kk + 4 + tq] : 0u;
      }
    }
    // per-warp state: heads hA = 2tq, hB = 2tq + 1
    float m[2] = {-INFINITY, -INFINITY}, l[2] = {0.f, 0.f};
    float o[KS][4];
#pragma unroll
    for (int mm = 0; mm < KS; ++mm) o[mm][0] = o[mm][1] = o[mm][2] = o[mm][3] = 0.f;

    for (; it < seg_end; ++it) {
      const int t0 = (it - u.iter_begin) * a.tile_n;
      const int t1 = min(t0 + a.tile_n, u.len);
      for (int s0 = t0; s0 < t1; s0 += a.stage_tokens) {
        if (j % NST == my_slot) {
          const int ntok = min(a.stage_tokens, t1 - s0);
          mbar_wait(&full[my_slot], (j / NST) & 1);
          unsigned char* st = ring + my_slot * C::STAGE_BYTES;
          const int rb = sub * 32;
          if (rb < ntok) {
            if (rb + 32 > ntok) {
              // rows >= ntok of this round hold the next unit's rows or cache padding: zero
              // this warp's V rows so 0 * (non-finite) cannot reach the accumulator.
              for (int r = rb + (lane >> 3); r < rb + 32; r += 4)
                if (r >= ntok)
#pragma unroll
                  for (int b = 0; b < C::NBOX; ++b)
                    *reinterpret_cast<uint4*>(st + C::KV_BYTES + b * C::BOX_BYTES + r * 128 + (ri << 4)) =
                        make_uint4(0u, 0u, 0u, 0u);
              __syncwarp();
            }
            const uint32_t kbase = smem_u32(st), vbase = smem_u32(st + C::KV_BYTES);
            // ---- S^T = K_f Q_f^T for two 16-token blocks (Alg1§20) ------------------------
            float s[2][4];
#pragma unroll
            for (int blk = 0; blk < 2; ++blk) {
              s[blk][0] = s[blk][1] = s[blk][2] = s[blk][3] = 0.f;
              const int tok = rb + blk * 16 + ri + ((mi & 1) << 3);
#pragma unroll
              for (int kk = 0; kk < KS; ++kk) {
                const int chunk = 2 * kk + (mi >> 1);
                const uint32_t addr = kbase + (chunk >> 3) * C::BOX_BYTES + tok * 128 + (((chunk & 7) ^ (tok & 7)) << 4);
                uint32_t af[4];
                ldsm_x4(addr, af);
                Mma<T>::run(s[blk], af, qb[kk][0], qb[kk][1]);
              }
            }
            // ---- scale, mask the tail (reading C5), running max per head (Alg1§21) -------
            float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
            for (int blk = 0; blk < 2; ++blk) {
              const int r0 = rb + blk * 16 + gq;
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const int tok = r0 + ((e >> 1) << 3);
                s[blk][e] = tok < ntok ? s[blk][e] * a.scale_log2 : -INFINITY;
                mx[e & 1] = fmaxf(mx[e & 1], s[blk][e]);
              }
            }
#pragma unroll
            for (int off = 4; off <= 16; off <<= 1) {
              mx[0] = fmaxf(mx[0], __shfl_xor_sync(0xffffffffu, mx[0], off));
              mx[1] = fmaxf(mx[1], __shfl_xor_sync(0xffffffffu, mx[1], off));
            }
            const bool grow = (mx[0] > m[0]) || (mx[1] > m[1]);
            if (__any_sync(0xffffffffu, grow)) {   // rescale l, O_acc (Alg1§23-24)
              const float mn0 = fmaxf(m[0], mx[0]), mn1 = fmaxf(m[1], mx[1]);
              const float al0 = ex2(m[0] - mn0), al1 = ex2(m[1] - mn1);
              l[0] *= al0;
              l[1] *= al1;
#pragma unroll
              for (int mm = 0; mm < KS; ++mm) {
                o[mm][0] *= al0;
                o[mm][2] *= al0;
                o[mm][1] *= al1;
                o[mm][3] *= al1;
              }
              m[0] = mn0;
              m[1] = mn1;
            }
            // ---- P_f = exp(S_f - m) (Alg1§22); PV (Alg1§24) -----------------------------
#pragma unroll
            for (int blk = 0; blk < 2; ++blk) {
              const float p0 = ex2(s[blk][0] - m[0]), p1 = ex2(s[blk][1] - m[1]);
              const float p2 = ex2(s[blk][2] - m[0]), p3 = ex2(s[blk][3] - m[1]);
              l[0] += p0 + p2;
              l[1] += p1 + p3;
              const uint32_t b0 = movmatrix_t(Mma<T>::pack(p0, p1));
              const uint32_t b1 = movmatrix_t(Mma<T>::pack(p2, p3));
              const int tok = rb + blk * 16 + ri + ((mi >> 1) << 3);
#pragma unroll
              for (int mm = 0; mm < KS; ++mm) {
                const int chunk = 2 * mm + (mi & 1);
                const uint32_t addr = vbase + (chunk >> 3) * C::BOX_BYTES + tok * 128 + (((chunk & 7) ^ (tok & 7)) << 4);
                uint32_t af[4];
                ldsm_x4_t(addr, af);
                Mma<T>::run(o[mm], af, b0, b1);
              }
            }
            if (rb + 32 > ntok) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[my_slot]);
        }
        ++j;
      }
    }

    // ---- segment end: per-head l over the 8 row groups, then fold warps ------------------
#pragma unroll
    for (int off = 4; off <= 16; off <<= 1) {
      l[0] += __shfl_xor_sync(0xffffffffu, l[0], off);
      l[1] += __shfl_xor_sync(0xffffffffu, l[1], off);
    }
    float* fo = fold_o + warp * GN * D;
#pragma unroll
    for (int mm = 0; mm < KS; ++mm) {
      const int c = 16 * mm + gq;
      fo[(2 * tq) * D + c] = o[mm][0];
      fo[(2 * tq + 1) * D + c] = o[mm][1];
      fo[(2 * tq) * D + c + 8] = o[mm][2];
      fo[(2 * tq + 1) * D + c + 8] = o[mm][3];
    }
    if (gq == 0) {
      fold_ml[(warp * GN + 2 * tq) * 2] = m[0];
      fold_ml[(warp * GN + 2 * tq) * 2 + 1] = l[0];
      fold_ml[(warp * GN + 2 * tq + 1) * 2] = m[1];
      fold_ml[(warp * GN + 2 * tq + 1) * 2 + 1] = l[1];
    }
    consumer_bar(NCT);
    constexpr int EPT = (GN * D + (NCW * 32) - 1) / (NCW * 32);   // (head, dim) elements per thread
    float oc[EPT], ms[EPT], ls[EPT];
#pragma unroll
    for (int q = 0; q < EPT; ++q) {
      const int e = t + q * NCT;
      oc[q] = 0.f;
      ms[q] = -INFINITY;
      ls[q] = 0.f;
      if (e < GN * D) {
        const int h = e / D, c = e % D;
#pragma unroll
        for (int w = 0; w < NCW; ++w) ms[q] = fmaxf(ms[q], fold_ml[(w * GN + h) * 2]);
#pragma unroll
        for (int w = 0; w < NCW; ++w) {
          const float wt = ex2(fold_ml[(w * GN + h) * 2] - ms[q]);
          ls[q] = fmaf(wt, fold_ml[(w * GN + h) * 2 + 1], ls[q]);
          oc[q] = fmaf(wt, fold_o[(w * GN + h) * D + c], oc[q]);
        }
      }
    }
    consumer_bar(NCT);   // fold buffer is reused by the next segment

    if (!host) {
      // ---- non-host: StorePartials + Signal (Alg2§19-23) ---------------------------------
#pragma unroll
      for (int q = 0; q < EPT; ++q) {
        const int e = t + q * NCT;
        if (e < GN * D) {
          const int h = e / D, c = e % D;
          if (h < a.group) {
            a.part_o[(size_t(g) * a.group + h) * D + c] = oc[q];
            if (c == 0) {
              a.part_ml[(size_t(g) * a.group + h) * 2] = ms[q];
              a.part_ml[(size_t(g) * a.group + h) * 2 + 1] = ls[q];
            }
          }
        }
      }
      consumer_bar(NCT);
      if (t == 0) {
        __threadfence();
        st_release_gpu(&a.flags[g], a.epoch);
        if (tr) tr[TR_PUBLISH] = globaltimer();
      }
    } else {
      if (!finishing) {
        // ---- host, not finishing: wait for peers g+1 .. last_cta, fold ascending ---------
        if (tr && t == 0) tr[TR_WAIT0] = globaltimer();
        for (int p = g + 1 + t; p <= u.last_cta; p += NCT) {
          while (ld_acquire_gpu(&a.flags[p]) != a.epoch) __nanosleep(20);
        }
        consumer_bar(NCT);
        if (tr && t == 0) tr[TR_WAIT1] = globaltimer();
#pragma unroll
        for (int q = 0; q < EPT; ++q) {
          const int e = t + q * NCT;
          if (e < GN * D) {
            const int h = e / D, c = e % D;
            if (h < a.group) {
              for (int p = g + 1; p <= u.last_cta; ++p) {
                const float mp = ld_cg(&a.part_ml[(size_t(p) * a.group + h) * 2]);
                const float lp = ld_cg(&a.part_ml[(size_t(p) * a.group + h) * 2 + 1]);
                const float op = ld_cg(&a.part_o[(size_t(p) * a.group + h) * D + c]);
                const float mn = fmaxf(ms[q], mp);
                const float wa = ex2(ms[q] - mn), wb = ex2(mp - mn);
                oc[q] = wa * oc[q] + wb * op;
                ls[q] = wa * ls[q] + wb * lp;
                ms[q] = mn;
              }
            }
          }
        }
      }
      // ---- finalize (Alg2§38-39) ----------------------------------------------------------
#pragma unroll
      for (int q = 0; q < EPT; ++q) {
        const int e = t + q * NCT;
        if (e < GN * D) {
          const int h = e / D, c = e % D;
          if (h < a.group) {
            a.out[size_t(u.q_row + h) * D + c] = oc[q] / ls[q];
            if (c == 0 && a.lse) a.lse[u.q_row + h] = (ms[q] + log2f(ls[q])) * kLn2;
          }
        }
      }
    }
    ++unit;
  }
  if (tr && t == 0) tr[TR_END] = globaltimer();
}

template <typename T, int D>
KernelInfo gqa_info() {
  constexpr int NST = 5, WPS = 2;
  using C = GqaCfg<D, NST, WPS>;
  KernelInfo k;
  k.supported = true;
  k.threads = C::THREADS;
  k.smem_bytes = C::SMEM;
  k.stage_tokens_max = C::ST;
  k.uses_tma_tensor = true;
  k.fn = reinterpret_cast<const void*>(&la_decode_gqa<T, D, NST, WPS>);
  return k;
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn(std::string& err) {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  if (!fn) err = "cuTensorMapEncodeTiled unavailable";
  return fn;
}

bool make_tmap(CUtensorMap* tm, const void* base, int64_t rows, int d, int dtype, std::string& err) {
  auto enc = encode_fn(err);
  if (!enc) return false;
  cuuint64_t gdim[2] = {cuuint64_t(d), cuuint64_t(rows)};
  cuuint64_t gstride[1] = {cuuint64_t(d) * 2};
  cuuint32_t box[2] = {64, 64};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(tm, dtype == LA_FP16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                   const_cast<void*>(base), gdim, gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    err = "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")";
    return false;
  }
  return true;
}

}  // namespace

KernelInfo gqa_kernel_info(int dtype, int head_dim, int group) {
  if (group < 2 || group > 8) return KernelInfo{};
  if (dtype == LA_BF16 && head_dim == 128) return gqa_info<__nv_bfloat16, 128>();
  if (dtype == LA_BF16 && head_dim == 64) return gqa_info<__nv_bfloat16, 64>();
  if (dtype == LA_FP16 && head_dim == 128) return gqa_info<__half, 128>();
  if (dtype == LA_FP16 && head_dim == 64) return gqa_info<__half, 64>();
  return KernelInfo{};
}

int launch_decode_tma(const KernelInfo& ki, const DecodeArgs& a, int64_t kv_rows, int head_dim, int dtype,
                      bool cooperative, void* stream, std::string& err) {
  TmapPair tm;
  if (!make_tmap(&tm.k, a.k, kv_rows, head_dim, dtype, err)) return 1;
  if (!make_tmap(&tm.v, a.v, kv_rows, head_dim, dtype, err)) return 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(a.grid);
  cfg.blockDim = dim3(ki.threads);
  cfg.dynamicSmemBytes = ki.smem_bytes;
  cfg.stream = static_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = cooperative ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  void* args[] = {const_cast<DecodeArgs*>(&a), &tm};
  cudaError_t e = cudaLaunchKernelExC(&cfg, ki.fn, args);
  if (e != cudaSuccess) {
    err = std::string("gqa decode launch: ") + cudaGetErrorString(e);
    cudaGetLastError();
    return 1;
  }
  note_launch();
  return 0;
}

}  // namespace la
