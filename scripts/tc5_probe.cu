// Checks the tcgen05 descriptor conventions of csrc/tc5.cuh on the GPU before they are used
// in the decode kernel: S^T = K Q^T (A K-major SW128, B K-major SW128, M=128, N=16) and
// O^T = V^T P^T (A = V read MN-major SW128, B = P K-major SW128), against a CPU product.
// Build: nvcc -std=c++17 -O2 -gencode arch=compute_100a,code=sm_100a -I paper_2405_10480_b200/csrc
//        scripts/tc5_probe.cu -o /tmp/tc5_probe
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tc5.cuh"

using namespace la;
__device__ __forceinline__ uint32_t smem32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ uint32_t sw(int row, int byte_in_row) {  // 128-B swizzle in a 1024-B atom
  return uint32_t(row) * 128 + ((((byte_in_row >> 4) ^ (row & 7)) << 4) | (byte_in_row & 15));
}

__global__ void probe(const __nv_bfloat16* K, const __nv_bfloat16* V, const __nv_bfloat16* Q,
                      const __nv_bfloat16* P, float* S, float* O, int mn_swap, const __nv_bfloat16* P2, float* O2) {
  extern __shared__ unsigned char raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  unsigned char *sK = sm, *sV = sm + 32768, *sQ = sm + 65536, *sP = sm + 69632;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 73728);
  uint32_t* taddr_s = reinterpret_cast<uint32_t*>(sm + 73744);
  unsigned char* sP2 = sm + 74752;  // [128 tokens][64 cols] bf16: MN-major B (N contiguous), 128-B swizzle
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  for (int i = t; i < 128 * 128; i += blockDim.x) {
    const int tok = i / 128, d = i % 128;
    const uint32_t o = (d / 64) * 16384 + sw(tok, (d % 64) * 2);
    *reinterpret_cast<__nv_bfloat16*>(sK + o) = K[i];
    *reinterpret_cast<__nv_bfloat16*>(sV + o) = V[i];
  }
  for (int i = t; i < 16 * 128; i += blockDim.x) {
    const int r = i / 128, c = i % 128;  // Q[r][dim c], P[r][token c]
    const uint32_t o = (c / 64) * 2048 + sw(r, (c % 64) * 2);
    *reinterpret_cast<__nv_bfloat16*>(sQ + o) = Q[i];
    *reinterpret_cast<__nv_bfloat16*>(sP + o) = P[i];
  }
  for (int i = t; i < 128 * 64; i += blockDim.x) {
    const int tok = i / 64, n = i % 64;
    *reinterpret_cast<__nv_bfloat16*>(sP2 + sw(tok, n * 2)) = P2[i];
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (warp == 0) tc5::tmem_alloc(taddr_s, 128);
  tc5::fence_before();
  __syncthreads();
  tc5::fence_after();
  const uint32_t tm = *taddr_s;
  if (t == 0) {
    constexpr uint32_t i1 = tc5::idesc_f16(true, 128, 16, false, false);
    constexpr uint32_t i2 = tc5::idesc_f16(true, 128, 16, true, false);
    for (int kk = 0; kk < 8; ++kk) {
      const uint32_t off = (kk / 4) * 0 + (kk % 4) * 32;
      tc5::mma_f16(tm, tc5::sdesc(smem32(sK) + (kk / 4) * 16384 + off, 16, 1024),
                   tc5::sdesc(smem32(sQ) + (kk / 4) * 2048 + off, 16, 1024), i1, kk > 0);
    }
    const uint32_t lbo = mn_swap ? 1024 : 16384, sbo = mn_swap ? 16384 : 1024;
    for (int kk = 0; kk < 8; ++kk) {
      tc5::mma_f16(tm + 32, tc5::sdesc(smem32(sV) + kk * 2048, lbo, sbo),
                   tc5::sdesc(smem32(sP) + (kk / 4) * 2048 + (kk % 4) * 32, 16, 1024), i2, kk > 0);
    }
    constexpr uint32_t i3 = tc5::idesc_f16(true, 128, 64, true, true);
    for (int kk = 0; kk < 8; ++kk)
      tc5::mma_f16(tm + 64, tc5::sdesc(smem32(sV) + kk * 2048, lbo, sbo), tc5::sdesc(smem32(sP2) + kk * 2048, 8192, 1024),
                   i3, kk > 0);
    tc5::commit(bar);
  }
  {
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(smem32(bar)) : "memory");
  }
  tc5::fence_after();
  float v[16];
  tc5::ld16(tm + (uint32_t(32 * warp) << 16), v);
  for (int c = 0; c < 16; ++c) S[(32 * warp + lane) * 16 + c] = v[c];
  tc5::ld16(tm + (uint32_t(32 * warp) << 16) + 32, v);
  for (int c = 0; c < 16; ++c) O[(32 * warp + lane) * 16 + c] = v[c];
  for (int c0 = 0; c0 < 64; c0 += 16) {
    tc5::ld16(tm + (uint32_t(32 * warp) << 16) + 64 + c0, v);
    for (int c = 0; c < 16; ++c) O2[(32 * warp + lane) * 64 + c0 + c] = v[c];
  }
  tc5::fence_before();
  __syncthreads();
  if (warp == 0) tc5::tmem_dealloc(tm, 128);
}

int main() {
  std::vector<__nv_bfloat16> K(128 * 128), V(128 * 128), Q(16 * 128), P(16 * 128), P2(128 * 64);
  std::vector<float> fK(K.size()), fV(V.size()), fQ(Q.size()), fP(P.size()), fP2(P2.size());
  srand(1);
  auto rnd = [] { return float(rand() % 17 - 8) / 8.f; };  // exact in bf16, exact products/sums
  for (size_t i = 0; i < K.size(); ++i) { K[i] = __float2bfloat16(rnd()); fK[i] = __bfloat162float(K[i]); }
  for (size_t i = 0; i < V.size(); ++i) { V[i] = __float2bfloat16(rnd()); fV[i] = __bfloat162float(V[i]); }
  for (size_t i = 0; i < Q.size(); ++i) { Q[i] = __float2bfloat16(rnd()); fQ[i] = __bfloat162float(Q[i]); }
  for (size_t i = 0; i < P.size(); ++i) { P[i] = __float2bfloat16(rnd()); fP[i] = __bfloat162float(P[i]); }
  for (size_t i = 0; i < P2.size(); ++i) { P2[i] = __float2bfloat16(rnd()); fP2[i] = __bfloat162float(P2[i]); }
  __nv_bfloat16 *dK, *dV, *dQ, *dP, *dP2;
  float *dS, *dO, *dO2;
  cudaMalloc(&dP2, P2.size() * 2); cudaMalloc(&dO2, 128 * 64 * 4);
  cudaMemcpy(dP2, P2.data(), P2.size() * 2, cudaMemcpyHostToDevice);
  cudaMalloc(&dK, K.size() * 2); cudaMalloc(&dV, V.size() * 2); cudaMalloc(&dQ, Q.size() * 2); cudaMalloc(&dP, P.size() * 2);
  cudaMalloc(&dS, 128 * 16 * 4); cudaMalloc(&dO, 128 * 16 * 4);
  cudaMemcpy(dK, K.data(), K.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dV, V.data(), V.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dQ, Q.data(), Q.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dP, P.data(), P.size() * 2, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  int rc = 0;
  for (int mn_swap = 0; mn_swap < 2; ++mn_swap) {
    cudaMemset(dS, 0, 128 * 16 * 4); cudaMemset(dO, 0, 128 * 16 * 4);
    probe<<<1, 128, 96 * 1024>>>(dK, dV, dQ, dP, dS, dO, mn_swap, dP2, dO2);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("mn_swap=%d: CUDA error %s\n", mn_swap, cudaGetErrorString(e)); return 2; }
    std::vector<float> S(128 * 16), O(128 * 16);
    cudaMemcpy(S.data(), dS, S.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
    double es = 0, eo = 0;
    for (int tok = 0; tok < 128; ++tok)
      for (int n = 0; n < 16; ++n) {
        double s = 0;
        for (int d = 0; d < 128; ++d) s += double(fK[tok * 128 + d]) * fQ[n * 128 + d];
        es = fmax(es, fabs(s - S[tok * 16 + n]));
      }
    for (int d = 0; d < 128; ++d)
      for (int n = 0; n < 16; ++n) {
        double o = 0;
        for (int tok = 0; tok < 128; ++tok) o += double(fV[tok * 128 + d]) * fP[n * 128 + tok];
        eo = fmax(eo, fabs(o - O[d * 16 + n]));
      }
    std::vector<float> O2(128 * 64);
    cudaMemcpy(O2.data(), dO2, O2.size() * 4, cudaMemcpyDeviceToHost);
    double eo2 = 0;
    for (int d = 0; d < 128; ++d)
      for (int n = 0; n < 64; ++n) {
        double o = 0;
        for (int tok = 0; tok < 128; ++tok) o += double(fV[tok * 128 + d]) * fP2[tok * 64 + n];
        eo2 = fmax(eo2, fabs(o - O2[d * 64 + n]));
      }
    printf("mn_swap=%d  max|S err|=%g  max|O err|=%g  max|O2 (B MN-major, N=64) err|=%g\n", mn_swap, es, eo, eo2);
    if (mn_swap == 0 && (es > 0 || eo > 0 || eo2 > 0)) rc = 1;
  }
  printf(rc ? "PROBE FAIL\n" : "PROBE OK (conventions of tc5.cuh hold)\n");
  return rc;
}
