// Microbenchmark: back-to-back tcgen05.mma kind::f16 (M=128, K=16) issue rate per SM for
// several N and smem layouts (SW128 K-major vs no-swizzle K-major).  One CTA per SM, one
// elected thread issues `iters` x 16 MMAs into one TMEM accumulator, commit + wait; the
// kernel reports cycles per MMA.  Operands are zero-filled smem (values irrelevant).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int N, int SWZ>
__global__ void __launch_bounds__(128, 1) mma_rate(int iters, long long* out, int shift) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* base = (uint8_t*)(((uintptr_t)smem + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) ((uint32_t*)base)[i] = 0;
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
  const uint32_t sa = smem_u32(base), sb = smem_u32(base + 32768);
  auto desc = [&](uint32_t addr) -> uint64_t {
    uint64_t d = (uint64_t)((addr >> 4) & 0x3FFF);
    if (SWZ == 128) {
      d |= (uint64_t)(1024 >> 4) << 32;
      d |= (uint64_t)2 << 61;
    } else if (SWZ == 32) {
      d |= (uint64_t)1 << 16;
      d |= (uint64_t)(256 >> 4) << 32;
      d |= (uint64_t)6 << 61;
    } else {
      d |= (uint64_t)(2048 >> 4) << 16;  // LBO: K-adjacent core matrices
      d |= (uint64_t)(128 >> 4) << 32;   // SBO: 8-row groups
    }
    d |= (uint64_t)1 << 46;
    return d;
  };
  long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0) {
    const uint64_t ad = desc(sa), bd = desc(sb);
    t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        // shift: k-th MMA's A start moves by k*shift bytes (row-shifted taps)
        const uint64_t adk = ad + (SWZ == 128 ? 2 * (k & 3) : 0) + ((k * shift) >> 4), bdk = bd + (SWZ == 128 ? 2 * (k & 3) : 0);
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
            "l"(adk), "l"(bdk), "r"(idesc), "r"((it | k) != 0 ? 1 : 0));
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

template <int N, int SWZ>
void run(int sms, int shift = 0) {
  const int iters = 2000;
  long long* d;
  cudaMalloc(&d, sms * sizeof(long long));
  cudaFuncSetAttribute(mma_rate<N, SWZ>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70 * 1024);
  for (int rep = 0; rep < 2; ++rep) mma_rate<N, SWZ><<<sms, 128, 70 * 1024>>>(iters, d, shift);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[256];
  cudaMemcpy(h, d, sms * sizeof(long long), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < sms; ++i) avg += h[i];
  avg /= sms;
  const double cyc = avg / (iters * 16.0);
  printf("shift=%4d N=%3d swz=%3d: %s %.1f cyc/MMA (floor %d), %.0f flop/clk/SM\n", shift, N, SWZ,
         cudaGetErrorString(e), cyc, 128 * N / 256, 2.0 * 128 * N * 16 / cyc);
  cudaFree(d);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<64, 128>(sms);
  run<64, 0>(sms);
  run<128, 128>(sms);
  run<128, 0>(sms);
  run<256, 128>(sms);
  run<256, 0>(sms);
  run<32, 128>(sms);
  for (int sh : {16, 32, 48, 128, 256, 928, 960}) run<64, 0>(sms, sh);
  for (int sh : {32, 64, 256, 1920}) run<64, 32>(sms, sh);
  for (int sh : {128, 256, 1024, 7424}) run<64, 128>(sms, sh);
  for (int sh : {128, 7424}) run<128, 128>(sms, sh);
  return 0;
}
