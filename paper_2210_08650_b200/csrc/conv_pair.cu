// Chained 1x1 pair on Blackwell tensor cores (sm_100a): a ResNet bottleneck's last conv and
// the NEXT block's first conv in one persistent kernel.
//
// Rows a3/a5 of the hot path: per 128-pixel tile
//   GEMM1  out = relu(t2 * W3 + bias3 + [x * I | ds(x)])   (conv3 + folded BN + residual,
//          the residual as a second K-concatenated A source against the identity / the
//          fused 1x1 downsample weights -- exactly the single-conv path of conv_tc.cu)
//   GEMM2  t1' = relu(out * W1' + bias1')                  (next block's conv1 + folded BN)
// The block output tile is written to HBM once (it is the next block's residual) and kept
// in shared memory as GEMM2's A operand, so conv1' never re-reads it from HBM: that saves
// the largest activation read of every bottleneck transition (PAPER.md:732 prefix forward;
// layer-at-a-time it is ~0.9 ms of the ResNet-50 b512 step at HBM peak).
//
// Warp roles (11 warps): 0-7 epilogue (thread = TMEM lane; warps w, w+4 split the columns),
// 8 TMA producer of GEMM1 (A + W3 chunks), 9 TMEM allocator + MMA issuer, 10 TMA producer of
// GEMM2's weight chunks (own ring: GEMM2 stages wait on the epilogue, and must not block
// the next tile's GEMM1 prefetch).  (Keeping t2 and the identity block resident in smem
// instead was measured slower: it leaves fewer bytes in flight for the HBM streams.)  TMEM (512 columns): two GEMM1
// accumulators of BN1 = 128 columns (so the epilogue of N tile j overlaps the MMAs of j+1)
// and one GEMM2 accumulator of N2 <= 256 columns.  The GEMM1 epilogue writes each 128-column
// N tile as two 128B-swizzled [128 x 64] bf16 blocks -- the TMA-store staging of `out` and,
// unchanged, K chunks of GEMM2's A operand (2 N tiles in flight = 4 blocks).
//
// Per M tile the MMA order is  G1(0) G1(1) G2(0) G1(2) G2(1) ... G2(last); each producer
// streams its ring in that order.
#include "kernels.h"
#include "tc_ptx.cuh"

namespace hapi {
namespace {
using namespace tcx;

constexpr int PM = 128;                  // rows per tile (MMA M)
constexpr int PK = 64;                   // K chunk (one 128-byte swizzle atom row)
constexpr int BN1 = 128;                 // GEMM1 N tile
constexpr int P_EPI_THREADS = 256;
constexpr int P_PROD_WARP = 8;
constexpr int P_MMA_WARP = 9;
constexpr int P_PROD2_WARP = 10;
constexpr int P_THREADS = 11 * 32;
constexpr int P_S2 = 2;                  // GEMM2 weight ring depth
constexpr int P_SMEM_LIMIT = 232448;
constexpr int P_MAX_STAGES = 8;
constexpr int P_A_BYTES = PM * PK * 2;   // 16 KB
constexpr int P_STG_BYTES = PM * 64 * 2; // one [128 x 64] bf16 block, 16 KB
constexpr int P_MAX_BIAS1 = 512;
constexpr int P_TMEM_ACC2 = 2 * BN1;     // GEMM2 accumulator column base

// named barrier of the two epilogue warps (q, q + 4) that share TMEM lane quarter q
__device__ __forceinline__ void quarter_bar(int q) { asm volatile("bar.sync %0, 64;" ::"r"(2 + q) : "memory"); }

template <int N2>
struct PairCfg {
  static constexpr int STAGE = P_A_BYTES + BN1 * PK * 2;  // GEMM1 ring: A chunk + W3 chunk
  static constexpr int B2_BYTES = N2 * PK * 2;            // GEMM2 ring: one W1' chunk
  static constexpr int FIXED = 4 * P_STG_BYTES + P_S2 * B2_BYTES + (P_MAX_BIAS1 + 256) * 4 + 1024 /*barriers*/ +
                               1024 /*align*/;
};

__device__ __forceinline__ uint32_t idesc_bf16(int n) {
  // kind::f16: D fp32, A/B bf16, both K-major, M = 128, N = n
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(PM >> 4) << 24);
}

template <int N2>
__global__ void __launch_bounds__(P_THREADS, 1)
    conv_pair_kernel(const PairArgs a, const int stages, const __grid_constant__ CUtensorMap tm_a1,
                     const __grid_constant__ CUtensorMap tm_a2, const __grid_constant__ CUtensorMap tm_b1,
                     const __grid_constant__ CUtensorMap tm_id, const __grid_constant__ CUtensorMap tm_b2,
                     const __grid_constant__ CUtensorMap tm_y1, const __grid_constant__ CUtensorMap tm_y2) {
  using C = PairCfg<N2>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* ring = smem;                                  // stages x (A slot | B slot)
  uint8_t* stg = ring + stages * C::STAGE;               // 4 staging / GEMM2-A blocks
  uint8_t* ring2 = stg + 4 * P_STG_BYTES;                // GEMM2 weight chunks
  float* sBias1 = reinterpret_cast<float*>(ring2 + P_S2 * C::B2_BYTES);
  float* sBias2 = sBias1 + P_MAX_BIAS1;
  uint64_t* full = reinterpret_cast<uint64_t*>(sBias2 + 256);
  uint64_t* empty = full + P_MAX_STAGES;
  uint64_t* tfull1 = empty + P_MAX_STAGES;   // GEMM1 accumulator j&1 ready
  uint64_t* tempty1 = tfull1 + 2;            // ... drained
  uint64_t* a2full = tempty1 + 2;            // staging pair j&1 written (GEMM2 may read)
  uint64_t* a2empty = a2full + 2;            // GEMM2 done reading staging pair j&1
  uint64_t* tfull2 = a2empty + 2;
  uint64_t* tempty2 = tfull2 + 1;
  uint64_t* full2 = tempty2 + 1;
  uint64_t* empty2 = full2 + P_S2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(empty2 + P_S2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m_tiles = (int)((a.M + PM - 1) / PM);
  const int nt1 = a.cout1 / BN1;
  const int k12 = a.k1_chunks + a.k2_chunks;
  griddep_launch_dependents();

  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull1[i], 1);
      mbar_init(&tempty1[i], P_EPI_THREADS);
      mbar_init(&a2full[i], P_EPI_THREADS);
      mbar_init(&a2empty[i], 1);
    }
    mbar_init(tfull2, 1);
    mbar_init(tempty2, P_EPI_THREADS);
    for (int i = 0; i < P_S2; ++i) {
      mbar_init(&full2[i], 1);
      mbar_init(&empty2[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == P_PROD_WARP && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_a1)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_b1)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_b2)) : "memory");
  }
  if (warp == P_MMA_WARP) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  griddep_wait();

  if (warp == P_PROD_WARP) {
    // ================================================================ TMA producer
    uint32_t stage = 0, phase = 0;
    auto next = [&]() {
      if (++stage == (uint32_t)stages) { stage = 0; phase ^= 1; }
    };
    auto load_g1 = [&](int j, int kc, int row0) {
      mbar_wait(&empty[stage], phase ^ 1);
      if (elect_one()) {
        uint64_t* bar = &full[stage];
        const uint32_t dA = smem_u32(ring + stage * C::STAGE), dB = dA + P_A_BYTES;
        mbar_arrive_expect_tx(bar, P_A_BYTES + BN1 * PK * 2);
        if (kc < a.k1_chunks) {
          tma_load_2d(dA, &tm_a1, kc * PK, row0, bar);
          tma_load_2d(dB, &tm_b1, kc * PK, j * BN1, bar);
        } else if (a.k2_diag) {
          const int c = kc - a.k1_chunks;  // residual channels j*128 + 64c against identity chunk c
          tma_load_2d(dA, &tm_a2, j * BN1 + c * PK, row0, bar);
          tma_load_2d(dB, &tm_id, 0, -c * PK, bar);
        } else {
          const int c = kc - a.k1_chunks;  // fused 1x1 downsample: its weights follow W3's K columns
          tma_load_2d(dA, &tm_a2, c * PK, row0, bar);
          tma_load_2d(dB, &tm_b1, kc * PK, j * BN1, bar);
        }
      }
      __syncwarp();
      next();
    };
    for (int tile = blockIdx.x; tile < m_tiles; tile += gridDim.x) {
      const int row0 = tile * PM;
      for (int j = 0; j < nt1; ++j)
        for (int kc = 0; kc < k12; ++kc) load_g1(j, kc, row0);
    }
  } else if (warp == P_PROD2_WARP) {
    // ================================================================ GEMM2 weight producer
    uint32_t stage = 0, phase = 0;
    for (int tile = blockIdx.x; tile < m_tiles; tile += gridDim.x) {
      for (int jj = 0; jj < nt1; ++jj) {
        for (int c = 0; c < BN1 / PK; ++c) {
          mbar_wait(&empty2[stage], phase ^ 1);
          if (elect_one()) {
            mbar_arrive_expect_tx(&full2[stage], C::B2_BYTES);
            tma_load_2d(smem_u32(ring2 + stage * C::B2_BYTES), &tm_b2, jj * BN1 + c * PK, 0, &full2[stage]);
          }
          __syncwarp();
          if (++stage == (uint32_t)P_S2) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == P_MMA_WARP) {
    // ================================================================ MMA issuer
    const uint32_t id1 = idesc_bf16(BN1), id2 = idesc_bf16(N2);
    const uint32_t ring0 = smem_u32(ring), stg0 = smem_u32(stg), ring20 = smem_u32(ring2);
    uint32_t stage = 0, phase = 0, stage2 = 0, phase2 = 0;
    int n = 0, it = 0;
    auto next = [&]() {
      if (++stage == (uint32_t)stages) { stage = 0; phase ^= 1; }
    };
    auto gemm2 = [&](int nn, bool first_of_tile) {
      if (first_of_tile) {
        mbar_wait(tempty2, (it & 1) ^ 1);
        tc_fence_after();
      }
      const int bb = nn & 1;
      mbar_wait(&a2full[bb], (nn >> 1) & 1);
      tc_fence_after();
      for (int c = 0; c < BN1 / PK; ++c) {
        mbar_wait(&full2[stage2], phase2);
        tc_fence_after();
        if (elect_one()) {
          const uint64_t ad = make_sdesc(stg0 + (bb * 2 + c) * P_STG_BYTES);
          const uint64_t bd = make_sdesc(ring20 + stage2 * C::B2_BYTES);
#pragma unroll
          for (int k = 0; k < PK / 16; ++k)
            mma_bf16(tmem + P_TMEM_ACC2, ad + 2 * k, bd + 2 * k, id2, (first_of_tile && c == 0 && k == 0) ? 0u : 1u);
          mma_commit(&empty2[stage2]);
        }
        __syncwarp();
        if (++stage2 == (uint32_t)P_S2) { stage2 = 0; phase2 ^= 1; }
      }
      if (elect_one()) mma_commit(&a2empty[bb]);
      __syncwarp();
    };
    for (int tile = blockIdx.x; tile < m_tiles; tile += gridDim.x, ++it) {
      for (int j = 0; j < nt1; ++j, ++n) {
        const int buf = n & 1;
        mbar_wait(&tempty1[buf], ((n >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + buf * BN1;
        for (int kc = 0; kc < k12; ++kc) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (elect_one()) {
            const uint64_t ad = make_sdesc(ring0 + stage * C::STAGE);
            const uint64_t bd = make_sdesc(ring0 + stage * C::STAGE + P_A_BYTES);
#pragma unroll
            for (int k = 0; k < PK / 16; ++k) mma_bf16(d, ad + 2 * k, bd + 2 * k, id1, (kc | k) != 0);
            mma_commit(&empty[stage]);
          }
          __syncwarp();
          next();
        }
        if (elect_one()) mma_commit(&tfull1[buf]);
        __syncwarp();
        if (j >= 1) gemm2(n - 1, j - 1 == 0);
      }
      gemm2(n - 1, nt1 == 1);
      if (elect_one()) mma_commit(tfull2);
      __syncwarp();
    }
  } else if (warp < 8) {
    // ================================================================ epilogues
    const int quarter = warp & 3, gsel = warp >> 2;
    const int row = quarter * 32 + lane;
    const int et = threadIdx.x;
    const bool lead = gsel == 0 && lane == 0;  // issues (and waits for) its row quarter's stores
    for (int i = et; i < a.cout1; i += P_EPI_THREADS) sBias1[i] = a.bias1 ? __ldg(a.bias1 + i) : 0.f;
    for (int i = et; i < N2; i += P_EPI_THREADS) sBias2[i] = a.bias2 ? __ldg(a.bias2 + i) : 0.f;
    epi_bar();
    const uint32_t stg0 = smem_u32(stg);
    const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
    int n = 0, it = 0;
    const int sub_w = (a.W + 1) >> 1, sub_h = (a.H + 1) >> 1;
    for (int tile = blockIdx.x; tile < m_tiles; tile += gridDim.x, ++it) {
      const int row0 = tile * PM;
      // y1_sub: this thread's pixel, if it is an even (row, col) one, goes to the compact map
      uint8_t* dsub = nullptr;
      if (a.y1_sub) {
        const long long m = (long long)row0 + row;
        if (m < a.M) {
          const long long hw = (long long)a.H * a.W;
          const long long nimg = m / hw;
          const int rem = (int)(m - nimg * hw), oh = rem / a.W, ow = rem - (rem / a.W) * a.W;
          if (!((oh | ow) & 1))
            dsub = static_cast<uint8_t*>(a.y1_sub) +
                   (((nimg * sub_h + (oh >> 1)) * sub_w + (ow >> 1)) * a.cout1 + gsel * 32) * 2;
        }
      }
      for (int j = 0; j < nt1; ++j, ++n) {
        const int buf = n & 1;
        mbar_wait(&tfull1[buf], (n >> 1) & 1);
        tc_fence_after();
        // staging pair `buf` was last read by GEMM2(n-2) and by the TMA stores of n-2 (and,
        // for the first N tile of a row tile, by the previous tile's GEMM2-output stores)
        mbar_wait(&a2empty[buf], ((n >> 1) & 1) ^ 1);
        // warps q and q+4 own rows 32q..32q+31 of every staging block (and store exactly those
        // rows), so a 64-thread barrier per row quarter replaces the CTA-wide one
        if (lead) {
          if (j == 0) bulk_wait_read0(); else bulk_wait_read1();
        }
        quarter_bar(quarter);
#pragma unroll
        for (int b = 0; b < 2; ++b) {
          uint32_t v[32];
          tmem_ld32(lane_base + buf * BN1 + b * 64 + gsel * 32, v);
          tmem_wait_ld();
          const uint32_t blk = stg0 + (buf * 2 + b) * P_STG_BYTES;
          const uint32_t bias = smem_u32(sBias1 + j * BN1 + b * 64 + gsel * 32);
#pragma unroll
          for (int c4 = 0; c4 < 4; ++c4) {
            const float4 b0 = lds_f4(bias + c4 * 32), b1 = lds_f4(bias + c4 * 32 + 16);
            const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
            uint32_t o[4];
#pragma unroll
            for (int q = 0; q < 4; ++q)
              o[q] = cvt_relu_bf16x2(__uint_as_float(v[c4 * 8 + 2 * q]) + bb[2 * q],
                                     __uint_as_float(v[c4 * 8 + 2 * q + 1]) + bb[2 * q + 1]);
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(blk + swz_off<128>(row, gsel * 4 + c4)),
                         "r"(o[0]), "r"(o[1]), "r"(o[2]), "r"(o[3])
                         : "memory");
            if (dsub)
              *reinterpret_cast<uint4*>(dsub + (j * BN1 + b * 64 + c4 * 8) * 2) = make_uint4(o[0], o[1], o[2], o[3]);
          }
        }
        tc_fence_before();
        mbar_arrive(&tempty1[buf]);
        fence_proxy_async_smem();
        mbar_arrive(&a2full[buf]);
        quarter_bar(quarter);
        if (lead) {
          if (!a.y1_sub)
            for (int b = 0; b < 2; ++b)
              tma_store_2d(&tm_y1, stg0 + (buf * 2 + b) * P_STG_BYTES + quarter * 32 * 128, j * BN1 + b * 64,
                           row0 + quarter * 32);
          bulk_commit();
        }
      }
      // GEMM2 epilogue: t1' = relu(acc2 + bias2) through staging blocks 0..N2/64-1 (every
      // GEMM2 of this tile has completed -- tfull2 -- so only the store reads are pending)
      mbar_wait(tfull2, it & 1);
      tc_fence_after();
      if (lead) bulk_wait_read0();
      quarter_bar(quarter);
#pragma unroll
      for (int b = 0; b < N2 / 64; ++b) {
        uint32_t v[32];
        tmem_ld32(lane_base + P_TMEM_ACC2 + b * 64 + gsel * 32, v);
        tmem_wait_ld();
        const uint32_t blk = stg0 + b * P_STG_BYTES;
        const uint32_t bias = smem_u32(sBias2 + b * 64 + gsel * 32);
#pragma unroll
        for (int c4 = 0; c4 < 4; ++c4) {
          const float4 b0 = lds_f4(bias + c4 * 32), b1 = lds_f4(bias + c4 * 32 + 16);
          const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
          uint32_t o[4];
#pragma unroll
          for (int q = 0; q < 4; ++q)
            o[q] = cvt_relu_bf16x2(__uint_as_float(v[c4 * 8 + 2 * q]) + bb[2 * q],
                                   __uint_as_float(v[c4 * 8 + 2 * q + 1]) + bb[2 * q + 1]);
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(blk + swz_off<128>(row, gsel * 4 + c4)),
                       "r"(o[0]), "r"(o[1]), "r"(o[2]), "r"(o[3])
                       : "memory");
        }
      }
      tc_fence_before();
      mbar_arrive(tempty2);
      fence_proxy_async_smem();
      quarter_bar(quarter);
      if (lead) {
        for (int b = 0; b < N2 / 64; ++b)
          tma_store_2d(&tm_y2, stg0 + b * P_STG_BYTES + quarter * 32 * 128, b * 64, row0 + quarter * 32);
        bulk_commit();
      }
    }
    if (lead) bulk_wait_all();
  }

  tc_fence_before();
  __syncthreads();
  if (warp == P_MMA_WARP) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

template <int N2>
cudaError_t launch_pair(const PairArgs& a, const PairMaps& mp, int num_sms, cudaStream_t st) {
  using C = PairCfg<N2>;
  static std::atomic<uint64_t> attr_mask{0};
  {
    cudaError_t e = ensure_smem_attr(attr_mask, conv_pair_kernel<N2>, P_SMEM_LIMIT);
    if (e != cudaSuccess) return e;
  }
  int stages = (P_SMEM_LIMIT - C::FIXED) / C::STAGE;
  if (stages > P_MAX_STAGES) stages = P_MAX_STAGES;
  if (stages < 2) return cudaErrorInvalidValue;
  const size_t smem = (size_t)stages * C::STAGE + C::FIXED;
  const long long m_tiles = (a.M + PM - 1) / PM;
  const int grid = (int)(m_tiles < num_sms ? m_tiles : num_sms);
  if (grid <= 0) return cudaSuccess;
  return launch_pdl(conv_pair_kernel<N2>, dim3(grid), dim3(P_THREADS), smem, st, a, stages, *mp.a1, *mp.a2, *mp.b1,
                    *mp.id, *mp.b2, *mp.y1, *mp.y2);
}

}  // namespace

cudaError_t conv_pair_launch(const PairArgs& a, const PairMaps& mp, int n2, int num_sms, cudaStream_t st) {
  if (a.cout1 % BN1 != 0 || a.cout1 > P_MAX_BIAS1 || a.k1_chunks < 1 || a.k2_chunks < 0 ||
      (a.k2_diag && a.k2_chunks != BN1 / PK) || !mp.a1 || !mp.b1 || !mp.b2 || !mp.y1 || !mp.y2 ||
      (a.k2_chunks > 0 && !mp.a2) || (a.k2_diag && !mp.id))
    return cudaErrorInvalidValue;
  switch (n2) {
    case 64: return launch_pair<64>(a, mp, num_sms, st);
    case 128: return launch_pair<128>(a, mp, num_sms, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace hapi
