// Microbenchmark 3: tcgen05.mma (kind::f16, M = 128, K = 16, cta_group::1) issue rate with
// both operands in shared memory, by operand layout: 128-byte swizzled K-major (the body
// convs) vs no-swizzle K-major core matrices (the mode-8 stem: 8-channel planes, LBO = the
// plane distance, SBO = 128 B).  Reports cycles per MMA instruction (N = 128: 64 at peak).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_sw128(uint32_t addr) {
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__device__ __forceinline__ uint64_t desc_none(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

// LA / LB: 0 = SW128, 1 = no swizzle (stem geometry), LA 2 = no swizzle starting one row in
template <int N, int LA, int LB>
__global__ void __launch_bounds__(128, 1) mma_lay(int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* base = (uint8_t*)(((uintptr_t)smem + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) ((uint32_t*)base)[i] = 0;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  const uint32_t sa = smem_u32(base), sb = smem_u32(base + 49152);
  long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0) {
    // stem geometry: A planes 16 KB apart (LBO), rows 16 B apart; B LBO 2048, SBO 128
    // LA = 2: the stem's row-shifted view, start 16 B (one 8-channel row) past a 128 B boundary
    const uint64_t ad = LA == 2 ? desc_none(sa + 16, 16384, 128) : LA ? desc_none(sa, 16384, 128) : desc_sw128(sa);
    const uint64_t bd = LB ? desc_none(sb, 2048, 128) : desc_sw128(sb);
    t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        // SW128: advance 32 B along K inside the atom; no swizzle: shift the start by k rows
        const uint64_t a = LA ? ad + 8 * (k & 3) : ad + 2 * (k & 3);
        const uint64_t b = LB ? bd + 256 * (k & 3) : bd + 2 * (k & 3);
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
            "l"(a), "l"(b), "r"(idesc), "r"((it | k) != 0 ? 1 : 0));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(done) : "r"(smem_u32(&bar)));
    t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

template <typename K>
void report(const char* what, K kern, int sms, int n) {
  const int iters = 2000;
  long long* d;
  cudaMalloc(&d, 256 * sizeof(long long));
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int rep = 0; rep < 2; ++rep) kern<<<sms, 128, 100 * 1024>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[256];
  cudaMemcpy(h, d, sms * sizeof(long long), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < sms; ++i) avg += h[i];
  avg /= sms;
  const double cyc = avg / (iters * 16.0);
  printf("%-40s N=%3d: %s %.1f cyc/MMA, %.0f flop/clk/SM\n", what, n, cudaGetErrorString(e), cyc, 2.0 * 128 * n * 16 / cyc);
  cudaFree(d);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  report("A SW128,   B SW128", mma_lay<128, 0, 0>, sms, 128);
  report("A noswz,   B noswz (mode-8 stem)", mma_lay<128, 1, 1>, sms, 128);
  report("A noswz,   B SW128", mma_lay<128, 1, 0>, sms, 128);
  report("A SW128,   B noswz", mma_lay<128, 0, 1>, sms, 128);
  report("A noswz +16 B (row-shifted), B noswz", mma_lay<128, 2, 1>, sms, 128);
  report("A SW128,   B SW128", mma_lay<64, 0, 0>, sms, 64);
  report("A noswz,   B noswz", mma_lay<64, 1, 1>, sms, 64);
  return 0;
}
