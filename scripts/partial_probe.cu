// Micro-probe: how fast can one SM read small partials that other SMs have just written and
// released (the static host's fixup read pattern)?  CTAs 1..P write a 512 B partial each,
// __threadfence, release a flag; CTA 0 acquires all flags, then reads every partial with
// 16-byte cp.async (all in flight) -- timed -- and reads them again (timed).  Also times the
// same read pattern on a cold, never-written buffer and on a buffer written by the host
// itself long before.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a scripts/partial_probe.cu -o /tmp/pp && /tmp/pp
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void cp16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cpwait() { asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory"); }

__device__ void read_all(const float* base, int P, int stride_floats, float* sm) {
  const int lane = threadIdx.x & 31;
  for (int x = lane; x < P * 32; x += 32) {
    const int i = x / 32, q = x % 32;
    cp16(sm + 4 * x, base + size_t(1 + i) * stride_floats + 4 * q);
  }
  cpwait();
  __syncwarp();
}

__global__ void probe(float* part, float* cold, unsigned* flags, unsigned epoch, int P, int stride_floats,
                      unsigned long long* out) {
  extern __shared__ float sm[];
  const int g = blockIdx.x;
  if (g > 0) {
    if (threadIdx.x < 32) {
      for (int j = threadIdx.x; j < 128; j += 32) part[size_t(g) * stride_floats + j] = float(g + j);
      __threadfence();
      __syncwarp();
      if (threadIdx.x == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flags + g), "r"(epoch) : "memory");
    }
    return;
  }
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  unsigned long long t0 = gt();
  for (int p = 1 + lane; p <= P; p += 32) {
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + p) : "memory");
    } while (v != epoch);
  }
  __syncwarp();
  unsigned long long t1 = gt();
  read_all(part, P, stride_floats, sm);
  unsigned long long t2 = gt();
  read_all(part, P, stride_floats, sm);
  unsigned long long t3 = gt();
  read_all(cold, P, stride_floats, sm);
  unsigned long long t4 = gt();
  float s = 0.f;
  for (int i = 0; i < P * 128; i += 32) s += sm[i + lane];
  if (lane == 0) {
    out[0] = t1 - t0;
    out[1] = t2 - t1;
    out[2] = t3 - t2;
    out[3] = t4 - t3;
    out[4] = (unsigned long long)(s != 12345.f);
  }
}

int main() {
  const int P = 127;
  for (int stride : {128, 256, 1024}) {
    float *part, *cold;
    unsigned* flags;
    unsigned long long* out;
    cudaMalloc(&part, size_t(P + 1) * stride * 4 * 64);
    cudaMalloc(&cold, size_t(P + 1) * stride * 4 * 64);
    cudaMalloc(&flags, (P + 1) * 4);
    cudaMemset(flags, 0, (P + 1) * 4);
    cudaMallocManaged(&out, 8 * sizeof(unsigned long long));
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    void* flush;
    cudaMalloc(&flush, 512 << 20);
    for (int rep = 0; rep < 6; ++rep) {
      cudaMemset(flush, rep, 512 << 20);
      cudaMemset(cold, 0, size_t(P + 1) * stride * 4);  // in L2, written long before
      probe<<<P + 1, 64, P * 512 + 1024>>>(part, cold, flags, rep + 1, P, stride, out);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(e));
        return 1;
      }
      printf("stride %4d B  wait %6.2f us  read-fresh %6.2f us  reread %6.2f us  read-old %6.2f us\n", stride * 4,
             out[0] / 1e3, out[1] / 1e3, out[2] / 1e3, out[3] / 1e3);
    }
    cudaFree(part);
    cudaFree(cold);
    cudaFree(flags);
    cudaFree(flush);
  }
  return 0;
}
