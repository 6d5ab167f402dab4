// Build: nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/p scripts/probes/<this file>.cu  (run from the repo root)
// Probe: aggregate HBM->smem rate of 1-D bulk copies of S bytes as a function of the number of
// issuing warps per CTA and lanes per warp (is the ~110-cycle per-op cost per warp or per SM?).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2405_10480_b200/csrc/ptx.cuh"
using namespace la::dev;
constexpr int STAGE = 65536, NS = 3;

__global__ void __launch_bounds__(160, 1) probe(const char* src, size_t bytes_per_cta, int S, int W, int lanes, int scatter,
                                                size_t npages_total, unsigned long long* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + NS * STAGE);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp >= W) return;
  const int per_stage = STAGE / S;              // copies per stage
  const size_t nst = bytes_per_cta / STAGE;
  const size_t page0 = size_t(blockIdx.x) * (bytes_per_cta / S);
  for (size_t j = 0; j < nst; ++j) {
    const int s = int(j % NS);
    if (j >= NS) mbar_wait(&full[s], uint32_t(((j / NS) - 1) & 1));
    __syncwarp();
    if (warp == 0 && lane == 0) mbar_arrive_expect_tx(&full[s], STAGE);
    // copies c = warp, warp + W, ... of this stage; within a warp, lanes [0, lanes) round-robin
    int k = 0;
    for (int c = warp; c < per_stage; c += W, ++k) {
      if (k % lanes != lane) continue;
      size_t pg = page0 + j * per_stage + c;
      if (scatter) pg = (pg * 40503ull) % npages_total;
      bulk_g2s_plain(sm + s * STAGE + c * S, src + pg * S, uint32_t(S), &full[s]);
    }
  }
  // drain
  for (size_t j = nst > NS ? nst - NS : 0; j < nst; ++j) mbar_wait(&full[j % NS], uint32_t((j / NS) & 1));
  if (threadIdx.x == 0) atomicAdd(sink, (unsigned long long)sm[5]);
}

int main() {
  const size_t total = size_t(4) << 30;
  char* src; cudaMalloc(&src, total); cudaMemset(src, 1, total);
  unsigned long long* sink; cudaMalloc(&sink, 8);
  const int G = 148;
  const size_t per = (total / G) / STAGE * STAGE;
  const int smem = NS * STAGE + 1024 + 64;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  struct C { int S, W, lanes, scatter; } cs[] = {
    {65536, 1, 1, 0}, {16384, 1, 1, 0}, {4096, 1, 1, 0}, {4096, 1, 16, 0}, {4096, 2, 1, 0}, {4096, 2, 8, 0},
    {4096, 4, 1, 0}, {4096, 4, 4, 0}, {4096, 1, 16, 1}, {4096, 2, 8, 1}, {4096, 4, 4, 1}, {2048, 1, 32, 1}, {2048, 2, 16, 1}, {2048, 4, 8, 1}};
  for (auto c : cs) {
    float best = 1e9;
    for (int it = 0; it < 6; ++it) {
      cudaEventRecord(a);
      probe<<<G, 160, smem>>>(src, per, c.S, c.W, c.lanes, c.scatter, total / c.S, sink);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (it) best = ms < best ? ms : best;
    }
    cudaError_t e = cudaGetLastError();
    printf("S %6d  warps %d  lanes/warp %2d  scatter %d : %7.1f us  %7.1f GB/s  (%.1f GB/s per SM) %s\n", c.S, c.W, c.lanes, c.scatter,
           best * 1e3, per * G / (best * 1e-3) / 1e9, per * G / (best * 1e-3) / 1e9 / G, e ? cudaGetErrorString(e) : "");
  }
  return 0;
}
