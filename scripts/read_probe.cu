// Read-bandwidth probe for B200 (roofline context for the decode kernel).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o read_probe scripts/read_probe.cu
//   ./read_probe [GiB=4] [reps=20]
// (1) bulk:  one CTA per SM, one elected thread streams its contiguous 1/148 of the buffer
//            through a 6 x 32 KiB cp.async.bulk + mbarrier ring, consumers only release
//            slots (no math) -- the decode kernel's data path with the compute removed.
// (2) ldg:   grid-stride 16-byte loads (ld.global.nc.L1::no_allocate), 8 in flight per
//            thread, xor-reduced so nothing is dead code.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

constexpr int NST = 6, STAGE = 32768, NCW = 6;

__global__ void __launch_bounds__((NCW + 1) * 32, 1) bulk_read(const unsigned char* buf, size_t per_cta, unsigned* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + NST * STAGE);
  uint64_t* empty = full + NST;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s32(&full[s])), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s32(&empty[s])), "r"(1));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const unsigned char* base = buf + blockIdx.x * per_cta;
  const int nst = int(per_cta / STAGE);
  if (warp == NCW) {
    if (lane == 0) {
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      for (int j = 0; j < nst; ++j) {
        const int s = j % NST;
        if (j >= NST) {
          uint32_t ok = 0;
          while (!ok)
            asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                         : "=r"(ok) : "r"(s32(&empty[s])), "r"(((j / NST) - 1) & 1) : "memory");
        }
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&full[s])), "r"(STAGE) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                     ::"r"(s32(sm + s * STAGE)), "l"(base + size_t(j) * STAGE), "r"(STAGE), "r"(s32(&full[s])), "l"(pol) : "memory");
      }
    }
    return;
  }
  unsigned acc = 0;
  for (int j = warp; j < nst; j += NCW) {  // warp w owns slot w (NST == NCW)
    const int s = j % NST;
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                   : "=r"(ok) : "r"(s32(&full[s])), "r"((j / NST) & 1) : "memory");
    acc ^= reinterpret_cast<const unsigned*>(sm + s * STAGE)[lane];
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(&empty[s])) : "memory");
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

__global__ void ldg_read(const uint4* buf, size_t n16, unsigned* sink) {
  unsigned acc = 0;
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n16; i += 8 * stride) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const size_t k = i + u * stride;
      if (k < n16)
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(buf + k));
      else
        v[u] = make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

int main(int argc, char** argv) {
  const double gib = argc > 1 ? atof(argv[1]) : 4.0;
  const int reps = argc > 2 ? atoi(argv[2]) : 20;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  size_t per_cta = size_t(gib * (1ull << 30) / sms) / STAGE * STAGE;
  size_t bytes = per_cta * sms;
  unsigned char* buf;
  unsigned* sink;
  CK(cudaMalloc(&buf, bytes));
  CK(cudaMalloc(&sink, 4));
  CK(cudaMemset(buf, 1, bytes));
  const int smem = NST * STAGE + 2 * NST * 8;
  CK(cudaFuncSetAttribute(bulk_read, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int mode = 0; mode < 2; ++mode) {
    for (int w = 0; w < 3; ++w) {
      if (mode == 0) bulk_read<<<sms, (NCW + 1) * 32, smem>>>(buf, per_cta, sink);
      else ldg_read<<<sms * 4, 512>>>(reinterpret_cast<const uint4*>(buf), bytes / 16, sink);
    }
    CK(cudaDeviceSynchronize());
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) {
      if (mode == 0) bulk_read<<<sms, (NCW + 1) * 32, smem>>>(buf, per_cta, sink);
      else ldg_read<<<sms * 4, 512>>>(reinterpret_cast<const uint4*>(buf), bytes / 16, sink);
    }
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double us = ms * 1e3 / reps;
    printf("{\"probe\": \"%s\", \"bytes\": %zu, \"us\": %.1f, \"GBps\": %.1f}\n", mode == 0 ? "tma_bulk_ring" : "ldg128_gridstride",
           bytes, us, bytes / (us * 1e-6) / 1e9);
  }
  return 0;
}
