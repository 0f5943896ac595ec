// Microbenchmark 2: tcgen05.mma issue rate (kind::f16, K=16) per SM for
//   (a) cta_group::2: a CTA pair (cluster of 2), M = 256 (128 rows per SM), the leader issues,
//       each SM holds its A rows and half of B's N rows at the same smem offsets;
//   (b) cta_group::1 with A read from TMEM instead of smem (M = 128).
// Operands are zero-filled (values irrelevant).  Reports cycles per MMA instruction and the
// FLOP/clk per SM it implies (peak 8192).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr) {
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;  // SW128 K-major
  return d;
}

template <int N>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) mma2(int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* base = (uint8_t*)(((uintptr_t)smem + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) ((uint32_t*)base)[i] = 0;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
  const uint32_t sa = smem_u32(base), sb = smem_u32(base + 32768);
  long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0 && rank == 0) {
    const uint64_t ad = sdesc(sa), bd = sdesc(sb);
    t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
            "l"(ad + 2 * (k & 3)), "l"(bd + 2 * (k & 3)), "r"(idesc), "r"((it | k) != 0 ? 1 : 0));
      }
    }
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                     smem_u32(&bar)), "h"((uint16_t)3));
  }
  if (threadIdx.x == 0) {
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(done) : "r"(smem_u32(&bar)));
    t1 = clock64();
    if (rank == 0) out[blockIdx.x / 2] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

// A from TMEM (cta_group::1, M = 128): [d], [a_tmem], b_desc
template <int N>
__global__ void __launch_bounds__(128, 1) mma_ta(int iters, long long* out) {
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
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  const uint32_t sb = smem_u32(base + 32768);
  long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0) {
    const uint64_t bd = sdesc(sb);
    const uint32_t ta = tmem + 256;  // A: 128 lanes x (K/2) columns
    t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
            "r"(ta + 8 * (k & 7)), "l"(bd + 2 * (k & 3)), "r"(idesc), "r"((it | k) != 0 ? 1 : 0));
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
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <typename K>
void report(const char* what, K kern, int grid, int nout, int n, int mrows) {
  const int iters = 2000;
  long long* d;
  cudaMalloc(&d, 256 * sizeof(long long));
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 70 * 1024);
  for (int rep = 0; rep < 2; ++rep) kern<<<grid, 128, 70 * 1024>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[256];
  cudaMemcpy(h, d, nout * sizeof(long long), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < nout; ++i) avg += h[i];
  avg /= nout;
  const double cyc = avg / (iters * 16.0);
  // per SM: mrows rows of the MMA are this SM's
  printf("%-34s N=%3d: %s %.1f cyc/MMA, %.0f flop/clk/SM\n", what, n, cudaGetErrorString(e), cyc,
         2.0 * mrows * n * 16 / cyc);
  cudaFree(d);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int pairs = sms / 2;
  report("cta_group::2 M=256 (per SM 128 rows)", mma2<64>, 2 * pairs, pairs, 64, 128);
  report("cta_group::2 M=256 (per SM 128 rows)", mma2<128>, 2 * pairs, pairs, 128, 128);
  report("cta_group::2 M=256 (per SM 128 rows)", mma2<256>, 2 * pairs, pairs, 256, 128);
  report("cta_group::1 A from TMEM, M=128", mma_ta<64>, sms, sms, 64, 128);
  report("cta_group::1 A from TMEM, M=128", mma_ta<128>, sms, sms, 128, 128);
  report("cta_group::1 A from TMEM, M=128", mma_ta<256>, sms, sms, 256, 128);
  return 0;
}
