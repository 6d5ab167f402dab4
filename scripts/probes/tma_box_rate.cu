// Build: nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/p scripts/probes/<this file>.cu  (run from the repo root)
// Probe: HBM->smem rate of 3-D tensor boxes {64 el, 16 rows, 2 halves} = 4 KiB (the paged page-16
// box) vs issuing warps per CTA, sequential or scattered boxes.  Plus 64-row boxes (16 KiB).
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../../paper_2405_10480_b200/csrc/ptx.cuh"
using namespace la::dev;
constexpr int STAGE = 65536, NS = 3;

__device__ __forceinline__ void tma3(void* dst, const CUtensorMap* tm, int c1, uint64_t* bar) {
  asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
               ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(tm)), "r"(0), "r"(c1), "r"(0), "r"(smem_u32(bar)) : "memory");
}

__global__ void __launch_bounds__(160, 1) probe(const __grid_constant__ CUtensorMap tm, size_t bytes_per_cta, int BR, int W,
                                                int scatter, long long nboxes_total, unsigned long long* sink) {
  extern __shared__ unsigned char smraw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + NS * STAGE);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp >= W) return;
  const int S = BR * 256, per_stage = STAGE / S;
  const size_t nst = bytes_per_cta / STAGE;
  const long long box0 = (long long)blockIdx.x * (long long)(bytes_per_cta / S);
  for (size_t j = 0; j < nst; ++j) {
    const int s = int(j % NS);
    if (j >= NS) mbar_wait(&full[s], uint32_t(((j / NS) - 1) & 1));
    __syncwarp();
    if (warp == 0 && lane == 0) mbar_arrive_expect_tx(&full[s], STAGE);
    if (lane == 0)
      for (int c = warp; c < per_stage; c += W) {
        long long bx = box0 + (long long)j * per_stage + c;
        if (scatter) bx = (bx * 40503ll) % nboxes_total;
        tma3(sm + s * STAGE + c * S, &tm, int(bx * BR), &full[s]);
      }
  }
  for (size_t j = nst > NS ? nst - NS : 0; j < nst; ++j) mbar_wait(&full[j % NS], uint32_t((j / NS) & 1));
  if (threadIdx.x == 0) atomicAdd(sink, (unsigned long long)sm[5]);
}

int main() {
  const size_t total = size_t(4) << 30;
  char* src; cudaMalloc(&src, total); cudaMemset(src, 1, total);
  unsigned long long* sink; cudaMalloc(&sink, 8);
  void* p = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                           const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                           CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill)>(p);
  const int G = 148;
  const size_t per = (total / G) / STAGE * STAGE;
  const int smem = NS * STAGE + 2048;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  struct C { int BR, W, scatter; } cs[] = {{64, 1, 0}, {16, 1, 0}, {16, 2, 0}, {16, 4, 0}, {16, 1, 1}, {16, 2, 1}, {16, 4, 1}, {64, 1, 1}, {8, 1, 1}, {8, 2, 1}, {8, 4, 1}};
  for (auto c : cs) {
    CUtensorMap tm;
    cuuint64_t gdim[3] = {64, cuuint64_t(total / 256), 2};
    cuuint64_t gstr[2] = {256, 128};
    cuuint32_t box[3] = {64, cuuint32_t(c.BR), 2}, es[3] = {1, 1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, src, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) { printf("encode failed %d\n", int(r)); return 1; }
    float best = 1e9;
    for (int it = 0; it < 6; ++it) {
      cudaEventRecord(a);
      probe<<<G, 160, smem>>>(tm, per, c.BR, c.W, c.scatter, (long long)(total / (c.BR * 256)), sink);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (it) best = ms < best ? ms : best;
    }
    cudaError_t e = cudaGetLastError();
    printf("tensor box %2d rows (%5d B)  warps %d  scatter %d : %7.1f us  %7.1f GB/s  (%.1f GB/s per SM) %s\n", c.BR, c.BR * 256,
           c.W, c.scatter, best * 1e3, per * G / (best * 1e-3) / 1e9, per * G / (best * 1e-3) / 1e9 / G, e ? cudaGetErrorString(e) : "");
  }
  return 0;
}
