// Implicit-GEMM convolution on Blackwell 5th-gen tensor cores (sm_100a).
//
// Row a3 of the hot path: every Conv2d / Linear of the frozen prefix,
// with eval-mode BN folded into the weights and bias, and ReLU, residual add, the
// DenseNet concat (channel-offset store), the bn-relu prologue and the cast fused.
// The storage side "executes the feature extraction part up to the split index"
// (PAPER.md:732); the paper ran it as cuDNN calls on T4 -- this is a B200-first design.
//
//   GEMM view: D[M=N*OH*OW][Cout] = A[M][K] * B[Cout][K]^T, K = KH*KW*C ordered (r, s, c).
//   A = activations gathered from NHWC (implicit im2col), B = packed bf16 weights.
//
// Persistent, warp-specialized CTA (one per SM, 288 threads):
//   warps 0-3  epilogue: TMEM -> registers (tcgen05.ld) -> bias/residual/ReLU -> bf16 store
//   warps 4-7  producer: A tile gather into 128B-swizzled smem (cp.async or a register
//              path for the bn-relu prologue); thread 0 also issues the B tile TMA
//   warp 8     TMEM allocator + single-thread tcgen05.mma issuer (M=128, N=BN, K=16)
// Pipelines: smem ring of STAGES (full/empty mbarriers), two TMEM accumulators
// (tfull/tempty) so the epilogue of tile i overlaps the MMAs of tile i+1.
#include <cuda_bf16.h>

#include "kernels.h"

namespace hapi {
namespace {

constexpr int BM = 128;
constexpr int BK = 64;                 // 64 bf16 = one 128-byte swizzle atom row
constexpr int NUM_EPI_WARPS = 4;
constexpr int PROD_WARP0 = 4;
constexpr int NUM_PROD_THREADS = 128;
constexpr int MMA_WARP = 8;
constexpr int NUM_THREADS = 9 * 32;
constexpr int A_STAGE_BYTES = BM * BK * 2;

template <int BN>
struct Cfg {
  static constexpr int B_STAGE_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_STAGE_BYTES + B_STAGE_BYTES;
  static constexpr int STAGES_RAW = (200 * 1024) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
  static constexpr int TMEM_COLS = (2 * BN <= 32) ? 32 : (2 * BN <= 64) ? 64 : (2 * BN <= 128) ? 128
                                   : (2 * BN <= 256) ? 256 : 512;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256;
};

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  uint32_t done = 0;
  uint32_t spins = 0;
  while (!done) {
    // watchdog: a lost arrival must fail loudly instead of hanging the GPU
    if (++spins == (1u << 30)) __trap();
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint32_t src_size) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_size) : "memory");
}
__device__ __forceinline__ void cp_async8(uint32_t dst, const void* src, uint32_t src_size) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst), "l"(src), "r"(src_size) : "memory");
}
// Arrive on `bar` once all prior cp.async of this thread have landed (pending count is
// incremented first, so this does not consume one of the barrier's expected arrivals).
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// SMEM matrix descriptor: K-major operand, 128-byte swizzle, 8-row atoms 1024 B apart.
__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);        // start address
  d |= (uint64_t)(0) << 16;                      // leading byte offset (unused, swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;              // stride byte offset between 8-row groups
  d |= (uint64_t)1 << 46;                        // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;                        // SWIZZLE_128B
  return d;
}
__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ float2 unpack_bf16x2(uint32_t u) {
  __nv_bfloat162 h = *reinterpret_cast<__nv_bfloat162*>(&u);
  return __bfloat1622float2(h);
}

// ------------------------------------------------------------------ the kernel
template <int BN, int MODE>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    conv_tc_kernel(const ConvArgs a, const __grid_constant__ CUtensorMap tmap_b, int m_tiles, int n_tiles,
                   int k_chunks) {
  using C = Cfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * A_STAGE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + C::STAGES * C::B_STAGE_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], NUM_PROD_THREADS + 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], NUM_EPI_WARPS * 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == PROD_WARP0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_b)) : "memory");
  }
  if (warp == MMA_WARP) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(C::TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int num_tiles = m_tiles * n_tiles;
  const int OHW = a.OH * a.OW;

  if (warp >= PROD_WARP0 && warp < PROD_WARP0 + 4) {
    // ================================================================ producer
    const int pt = threadIdx.x - PROD_WARP0 * 32;
    const char* xb = static_cast<const char*>(a.x);
    const int taps = a.KH * a.KW;
    uint32_t stage = 0, phase = 0;
    constexpr int ROWS = (MODE == 1) ? 16 : 8;       // rows handled per thread
    constexpr int RSTEP = (MODE == 1) ? 8 : 16;      // row stride between them
    const int q = (MODE == 1) ? (pt & 15) : (pt & 7);  // piece index within a 128 B row
    const int rsub = (MODE == 1) ? (pt >> 4) : (pt >> 3);
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      const int tm = tile / n_tiles, tn = tile - (tile / n_tiles) * n_tiles;
      int ih0[ROWS], iw0[ROWS];
      long long ioff[ROWS];
#pragma unroll
      for (int i = 0; i < ROWS; ++i) {
        const long long m = (long long)tm * BM + rsub + RSTEP * i;
        if (m < a.M) {
          const int n = (int)(m / OHW);
          const int rem = (int)(m - (long long)n * OHW);
          const int oh = rem / a.OW, ow = rem - (rem / a.OW) * a.OW;
          ih0[i] = oh * a.stride - a.pad;
          iw0[i] = ow * a.stride - a.pad;
          ioff[i] = (long long)n * a.H * a.W;
        } else {
          ih0[i] = -(1 << 28);
          iw0[i] = 0;
          ioff[i] = 0;
        }
      }
      for (int kc = 0; kc < k_chunks; ++kc) {
        mbar_wait(&empty[stage], phase ^ 1);
        if (pt == 0) {
          mbar_arrive_expect_tx(&full[stage], C::B_STAGE_BYTES);
          tma_load_2d(smem_u32(sB + stage * C::B_STAGE_BYTES), &tmap_b, kc * BK, tn * BN, &full[stage]);
        }
        const uint32_t a_stage = smem_u32(sA + stage * A_STAGE_BYTES);
        if (MODE == 1) {
          // stem: C == 4, one 8-byte piece = one filter tap
          const int tap = kc * 16 + q;
          const int r = tap / a.KW, s = tap - (tap / a.KW) * a.KW;
          const bool tap_ok = tap < taps;
          const uint32_t dst0 = a_stage + rsub * 128 + ((((q >> 1) ^ (rsub & 7))) << 4) + (q & 1) * 8;
#pragma unroll
          for (int i = 0; i < ROWS; ++i) {
            const int ih = ih0[i] + r, iw = iw0[i] + s;
            const bool ok = tap_ok && (unsigned)ih < (unsigned)a.H && (unsigned)iw < (unsigned)a.W;
            const char* src = ok ? xb + ((ioff[i] + (long long)ih * a.W + iw) * a.x_ld) * 2 : xb;
            cp_async8(dst0 + i * 1024, src, ok ? 8u : 0u);
          }
          cp_async_mbar_arrive(&full[stage]);
        } else {
          const int k0 = kc * BK + q * 8;
          const int tap = k0 / a.C;
          const int c = k0 - tap * a.C;
          const int r = tap / a.KW, s = tap - (tap / a.KW) * a.KW;
          const bool tap_ok = tap < taps;
          const uint32_t dst0 = a_stage + rsub * 128 + ((q ^ (rsub & 7)) << 4);
          if (MODE == 0) {
#pragma unroll
            for (int i = 0; i < ROWS; ++i) {
              const int ih = ih0[i] + r, iw = iw0[i] + s;
              const bool ok = tap_ok && (unsigned)ih < (unsigned)a.H && (unsigned)iw < (unsigned)a.W;
              const char* src = ok ? xb + ((ioff[i] + (long long)ih * a.W + iw) * a.x_ld + c) * 2 : xb;
              cp_async16(dst0 + i * 2048, src, ok ? 16u : 0u);
            }
            cp_async_mbar_arrive(&full[stage]);
          } else {
            // bn-relu prologue: A := relu(x * scale[c] + shift[c]); padding stays zero
            uint4 raw[ROWS];
            bool okv[ROWS];
#pragma unroll
            for (int i = 0; i < ROWS; ++i) {
              const int ih = ih0[i] + r, iw = iw0[i] + s;
              okv[i] = tap_ok && (unsigned)ih < (unsigned)a.H && (unsigned)iw < (unsigned)a.W;
              raw[i] = make_uint4(0, 0, 0, 0);
              if (okv[i]) {
                const uint4* src = reinterpret_cast<const uint4*>(xb + ((ioff[i] + (long long)ih * a.W + iw) * a.x_ld + c) * 2);
                raw[i] = __ldg(src);
              }
            }
            float sc[8], sh[8];
            if (tap_ok) {
              const float4 s0 = __ldg(reinterpret_cast<const float4*>(a.pro_scale + c));
              const float4 s1 = __ldg(reinterpret_cast<const float4*>(a.pro_scale + c + 4));
              const float4 h0 = __ldg(reinterpret_cast<const float4*>(a.pro_shift + c));
              const float4 h1 = __ldg(reinterpret_cast<const float4*>(a.pro_shift + c + 4));
              sc[0] = s0.x; sc[1] = s0.y; sc[2] = s0.z; sc[3] = s0.w; sc[4] = s1.x; sc[5] = s1.y; sc[6] = s1.z; sc[7] = s1.w;
              sh[0] = h0.x; sh[1] = h0.y; sh[2] = h0.z; sh[3] = h0.w; sh[4] = h1.x; sh[5] = h1.y; sh[6] = h1.z; sh[7] = h1.w;
            } else {
#pragma unroll
              for (int j = 0; j < 8; ++j) { sc[j] = 0.f; sh[j] = 0.f; }
            }
#pragma unroll
            for (int i = 0; i < ROWS; ++i) {
              uint32_t w4[4] = {raw[i].x, raw[i].y, raw[i].z, raw[i].w};
              uint4 o = make_uint4(0, 0, 0, 0);
              if (okv[i]) {
                uint32_t ov[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  const float2 f = unpack_bf16x2(w4[j]);
                  ov[j] = pack_bf16x2(fmaxf(fmaf(f.x, sc[2 * j], sh[2 * j]), 0.f),
                                      fmaxf(fmaf(f.y, sc[2 * j + 1], sh[2 * j + 1]), 0.f));
                }
                o = make_uint4(ov[0], ov[1], ov[2], ov[3]);
              }
              asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(dst0 + i * 2048), "r"(o.x), "r"(o.y),
                           "r"(o.z), "r"(o.w)
                           : "memory");
            }
            fence_proxy_async_smem();
          }
        }
        mbar_arrive(&full[stage]);
        if (++stage == (uint32_t)C::STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == MMA_WARP) {
    // ================================================================ MMA issuer
    if (lane == 0) {
      // kind::f16 instruction descriptor: D fp32, A/B bf16, both K-major, M=128, N=BN
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                             ((uint32_t)(BM >> 4) << 24);
      uint32_t stage = 0, phase = 0;
      int iter = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++iter) {
        const int acc = iter & 1;
        const uint32_t acc_phase = (iter >> 1) & 1;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kc = 0; kc < k_chunks; ++kc) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t adesc = make_sdesc(smem_u32(sA + stage * A_STAGE_BYTES));
          const uint64_t bdesc = make_sdesc(smem_u32(sB + stage * C::B_STAGE_BYTES));
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            // advance 16 bf16 = 32 bytes along K inside the swizzle atom
            mma_bf16(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, (kc | k) != 0);
          }
          mma_commit(&empty[stage]);
          if (kc == k_chunks - 1) mma_commit(&tfull[acc]);
          if (++stage == (uint32_t)C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else {
    // ================================================================ epilogue
    const int row = warp * 32 + lane;
    __nv_bfloat16* yb = static_cast<__nv_bfloat16*>(a.y);
    const __nv_bfloat16* rb = static_cast<const __nv_bfloat16*>(a.res);
    const bool vec_y = !a.nchw && ((reinterpret_cast<uintptr_t>(a.y) & 15) == 0) && (a.y_ld % 8 == 0);
    const bool vec_r = rb && ((reinterpret_cast<uintptr_t>(a.res) & 15) == 0) && (a.res_ld % 8 == 0);
    int iter = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++iter) {
      const int tm = tile / n_tiles, tn = tile - (tile / n_tiles) * n_tiles;
      const int acc = iter & 1;
      const uint32_t acc_phase = (iter >> 1) & 1;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const long long m = (long long)tm * BM + row;
      const bool mok = m < a.M;
      int img = 0, pix = 0;
      if (a.nchw && mok) {
        img = (int)(m / OHW);
        pix = (int)(m - (long long)img * OHW);
      }
#pragma unroll 1
      for (int j0 = 0; j0 < BN; j0 += 32) {
        uint32_t v[32];
        tmem_ld32(tmem_base + ((uint32_t)(warp * 32) << 16) + acc * BN + j0, v);
        tmem_wait_ld();
        const int n0 = tn * BN + j0;
        if (!mok || n0 >= a.Cout) continue;
        const int nv = min(32, a.Cout - n0);
        float f[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) f[j] = __uint_as_float(v[j]);
        if (a.bias) {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (j < nv) f[j] += __ldg(a.bias + n0 + j);
        }
        if (rb) {
          const __nv_bfloat16* rp = rb + m * a.res_ld + n0;
          if (vec_r && nv == 32) {
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4) {
              const uint4 u = __ldg(reinterpret_cast<const uint4*>(rp) + q4);
              const uint32_t uu[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const float2 g = unpack_bf16x2(uu[j]);
                f[q4 * 8 + 2 * j] += g.x;
                f[q4 * 8 + 2 * j + 1] += g.y;
              }
            }
          } else {
            for (int j = 0; j < nv; ++j) f[j] += __bfloat162float(rp[j]);
          }
        }
        if (a.relu) {
#pragma unroll
          for (int j = 0; j < 32; ++j) f[j] = fmaxf(f[j], 0.f);
        }
        if (a.nchw) {
          __nv_bfloat16* yp = yb + ((long long)img * a.Cout + n0) * OHW + pix;
          for (int j = 0; j < nv; ++j) yp[(long long)j * OHW] = __float2bfloat16_rn(f[j]);
        } else {
          __nv_bfloat16* yp = yb + m * a.y_ld + n0;
          if (vec_y && nv == 32) {
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4) {
              uint4 o;
              o.x = pack_bf16x2(f[q4 * 8 + 0], f[q4 * 8 + 1]);
              o.y = pack_bf16x2(f[q4 * 8 + 2], f[q4 * 8 + 3]);
              o.z = pack_bf16x2(f[q4 * 8 + 4], f[q4 * 8 + 5]);
              o.w = pack_bf16x2(f[q4 * 8 + 6], f[q4 * 8 + 7]);
              reinterpret_cast<uint4*>(yp)[q4] = o;
            }
          } else {
            for (int j = 0; j < nv; ++j) yp[j] = __float2bfloat16_rn(f[j]);
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == MMA_WARP) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(C::TMEM_COLS)
                 : "memory");
  }
}

template <int BN, int MODE>
cudaError_t launch_t(const ConvArgs& a, const CUtensorMap* tmap, int num_sms, cudaStream_t st) {
  using C = Cfg<BN>;
  static bool attr_set = false;  // per-instantiation; benign race (idempotent)
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(conv_tc_kernel<BN, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         C::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const int m_tiles = (int)((a.M + BM - 1) / BM);
  const int n_tiles = (a.Cout + BN - 1) / BN;
  const int k_chunks = (a.K + BK - 1) / BK;
  const int tiles = m_tiles * n_tiles;
  const int grid = tiles < num_sms ? tiles : num_sms;
  if (grid <= 0) return cudaSuccess;
  conv_tc_kernel<BN, MODE><<<grid, NUM_THREADS, C::SMEM_BYTES, st>>>(a, *tmap, m_tiles, n_tiles, k_chunks);
  return cudaGetLastError();
}

template <int BN>
cudaError_t launch_mode(const ConvArgs& a, const CUtensorMap* tmap, int mode, int num_sms, cudaStream_t st) {
  switch (mode) {
    case 0: return launch_t<BN, 0>(a, tmap, num_sms, st);
    case 1: return launch_t<BN, 1>(a, tmap, num_sms, st);
    case 2: return launch_t<BN, 2>(a, tmap, num_sms, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

int conv_tc_pick_bn(int cout) {
  if (cout <= 32) return 32;
  if (cout <= 64) return 64;
  if (cout <= 128) return 128;
  if (cout == 192) return 192;
  return cout % 256 == 0 ? 256 : 128;
}

cudaError_t conv_tc_launch(const ConvArgs& a, const CUtensorMap* tmap_b, int bn, int mode, int num_sms,
                           cudaStream_t st) {
  switch (bn) {
    case 32: return launch_mode<32>(a, tmap_b, mode, num_sms, st);
    case 64: return launch_mode<64>(a, tmap_b, mode, num_sms, st);
    case 128: return launch_mode<128>(a, tmap_b, mode, num_sms, st);
    case 192: return launch_mode<192>(a, tmap_b, mode, num_sms, st);
    case 256: return launch_mode<256>(a, tmap_b, mode, num_sms, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace hapi
