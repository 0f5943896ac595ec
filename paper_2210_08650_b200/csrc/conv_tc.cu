// Implicit-GEMM convolution on Blackwell 5th-gen tensor cores (sm_100a).
//
// Row a3 of the hot path: every Conv2d / Linear of the frozen prefix,
// with eval-mode BN folded into the weights and bias, and ReLU, residual add, the
// DenseNet concat (channel-offset store), the bn-relu prologue and the cast fused.
// The storage side "executes the feature extraction part up to the split index"
// (PAPER.md:732); the paper ran it as cuDNN calls on T4 -- this is a B200-first design.
//
//   GEMM view: D[M=N*OH*OW][Cout] = A[M][K] * B[Cout][K]^T, K = KH*KW*C ordered (r, s, c).
//   A = activations (implicit im2col of NHWC), B = packed bf16 weights [Cout][Kp].
//
// Persistent, warp-specialized CTA (one per SM, 448 threads):
//   warps 0-7  epilogue: thread = tile row (its TMEM lane; two warps per lane quarter split
//              the columns).  Per 64-column block:
//              tcgen05.ld -> + bias (smem) + residual (swizzled smem block) -> ReLU ->
//              bf16 into a 128B-swizzled staging block (conflict-free) -> one TMA store
//              (2D [M][C] box, or the 4D spatial box of mode 4); NCHW send-buffer writes
//              of the split layer go straight from registers (coalesced per channel)
//   warps 8-11 producer.  A operand per K chunk (one filter tap x 64 channels):
//                mode 3  TMA 2D box {64 ch, 128 rows} of the [M][C] matrix (1x1, stride 1)
//                mode 4  TMA 4D box {64 ch, wb, hb, nb} of the NHWC tensor shifted by the tap
//                        (traversal stride = conv stride; OOB zero fill = conv padding)
//                mode 0  cp.async 16-byte gather (C % 8 == 0: stems)
//                mode 2  register gather with the DenseNet bn-relu prologue
//              B operand: TMA 2D box {64, BN} of the weights.  Both 128-byte swizzled.
//   warp 12    TMEM allocator + tcgen05.mma issuer (one elected lane; M=128, N=BN, K=16)
//   warp 13    residual loader: TMA of the residual blocks into a 2-deep smem ring
// Pipelines: smem ring of STAGES (full/empty mbarriers, depth chosen per launch from the
// smem left after the epilogue buffers), two TMEM accumulators (tfull/tempty) so the
// epilogue of tile i overlaps the MMAs of tile i+1, residual ring (rfull/rempty), and
// double-buffered TMA-store staging (bulk async-groups).
#include <cuda_bf16.h>

#include <cstdlib>
#include <type_traits>

#include "kernels.h"
#include "tc_ptx.cuh"

namespace hapi {
namespace {
using namespace tcx;

constexpr int BM = 128;
constexpr int BK = 64;                 // 64 bf16 = one 128-byte swizzle atom row
constexpr int NUM_EPI_WARPS = 8;     // two per TMEM lane quarter, splitting the columns
constexpr int NUM_EPI_THREADS = NUM_EPI_WARPS * 32;
constexpr int PROD_WARP0 = 8;
constexpr int NUM_PROD_THREADS = 128;
constexpr int MMA_WARP = 12;
constexpr int RES_WARP = 13;
constexpr int XFORM_TMA_WARP = 14;   // mode 7: TMA issuer while warps 8-11 transform
constexpr int NUM_THREADS = 15 * 32;
constexpr int M8_POOL_WARP0 = 9;      // mode 8: warps 9-11, 13, 14 pool while 0-7 drain TMEM
constexpr int M8_POOL_THREADS = 160;
constexpr int M8_ROWS = 5;            // mode 8: padded s2d rows per tile (2 stem rows + 3 taps)
constexpr int M8_CHUNKS = M8_ROWS * 4; // mode 8: K chunks (s2d row x tap column), K = 16 each
constexpr int A_STAGE_BYTES = BM * BK * 2;
constexpr int SMEM_LIMIT = 232448;                           // 227 KB opt-in per CTA
constexpr int MAX_STAGES = 8;
constexpr int MAX_B_STAGES = 16;  // mode 6 weight ring
constexpr int MAX_A_STAGES = 8;   // mode 6 / mode 8 halo rings
constexpr int MAX_RES = 8;        // residual ring depth

// Static part of the shared-memory carve-up; the pipeline depth is chosen per launch.
template <int BN>
struct Cfg {
  static constexpr int SB = BN < 64 ? BN : 64;               // epilogue block width (columns)
  static constexpr int SB_BYTES = SB * 2 * BM;               // one [128 x SB] bf16 block (swizzled)
  static constexpr int SWZ = SB * 2;                         // 64- or 128-byte swizzle of that block
  static constexpr int B_STAGE_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_STAGE_BYTES + B_STAGE_BYTES;
  static constexpr int TMEM_COLS = (2 * BN <= 32) ? 32 : (2 * BN <= 64) ? 64 : (2 * BN <= 128) ? 128
                                   : (2 * BN <= 256) ? 256 : 512;
  static constexpr int FIXED = 2 * SB_BYTES /*out staging*/ + BN * 4 /*bias*/ + 1024 /*align*/ + 1024 /*barriers*/;
  static_assert((3 * MAX_B_STAGES + 2 * MAX_A_STAGES + 2 * MAX_RES + 17) * 8 + 4 <= 1024, "barrier area");
  static int stages(bool res) {
    int s = (SMEM_LIMIT - FIXED - (res ? 2 * SB_BYTES : 0)) / STAGE_BYTES;
    return s > MAX_STAGES ? MAX_STAGES : s;
  }
  static int smem_bytes(int stages, bool res) { return stages * STAGE_BYTES + FIXED + (res ? 2 * SB_BYTES : 0); }
};

// Tile geometry shared by producer, epilogue and loaders.
struct Geo {
  int mode;
  int wb, hb, nb;              // mode 4 spatial tile
  int tiles_w, tiles_h;        // mode 4
  int m_tiles, n_tiles, k_chunks, cblocks;
  int k1_chunks;               // chunks of the first A source (the rest come from tmap_a2)
  int a_bytes;                 // TMA modes: bytes of one A box
  int stages;                  // smem pipeline depth (A and B rings; mode 6: B ring)
  int a_stages, a_stage_bytes; // mode 6: halo ring depth and slot size
  int we;                      // mode 6: extended tile width (OW + KW - 1)
  int has_res;                 // residual tiles streamed by the loader warp
  int tma_out;                 // 1: epilogue writes via TMA store (NHWC views); 0: NCHW direct
  int res_box_bytes;           // bytes of one residual box
  int b_res;                   // 1: all weight chunks resident in smem (one N tile), loaded once
  int cps;                     // K chunks per pipeline stage (modes 3/4: 2 when BN <= 128)
  int pro_c;                   // mode 7: channels of the smem scale/shift tables (C rounded to 64)
  int ph, pw, pq, strips, n_tasks;  // mode 8: pooled map, pool columns per strip, strips/image, tasks
  int nseg, seg_rows, tlen;         // mode 8: pooled-row segments per (image, strip pair), rows per
                                    // segment, tiles per task (= seg_rows + 1: a warm-up tile first)
  int ring_bytes;                   // mode 8: two [2 we x 128 B] buffers of vertically pooled rows
  int res_depth;                    // residual ring depth (blocks of [128 x SB] in flight)
  int mt;                           // M sub-tiles per tile sharing each B stage (mode 6: 1 or 2)
  int mc;                           // 1: 2-CTA cluster, each weight chunk multicast to both CTAs
  int n_pairs;                      // mc: (M-tile pair, N tile) work items
  int pool2;                        // mode 4, hb = 2 tiles: 2x2/s2 maxpool fused into the epilogue
                                    // (y is the pooled map; only pooled pixels reach HBM)
};

// Row i (0..127) of m-tile tm -> output pixel index m, or -1 when the row is padding.
__device__ __forceinline__ long long row_to_m(const ConvArgs& a, const Geo& g, int tm, int i) {
  if (g.mode == 6) {
    const int h = i / g.we, w = i - (i / g.we) * g.we;
    const int th = tm % g.tiles_h, n = tm / g.tiles_h;
    const int oh = th * g.hb + h;
    if (w >= a.OW || h >= g.hb || oh >= a.OH) return -1;
    return ((long long)n * a.OH + oh) * a.OW + w;
  }
  if (g.mode != 4) {
    const long long m = (long long)tm * BM + i;
    return m < a.M ? m : -1;
  }
  const int per_img = g.hb * g.wb;
  if (i >= g.nb * per_img) return -1;
  const int tw = tm % g.tiles_w;
  const int th = (tm / g.tiles_w) % g.tiles_h;
  const int tb = tm / (g.tiles_w * g.tiles_h);
  const int ni = i / per_img, rem = i - ni * per_img;
  const int hi = rem / g.wb, wi = rem - hi * g.wb;
  const int n = tb * g.nb + ni, oh = th * g.hb + hi, ow = tw * g.wb + wi;
  if (n >= a.N || oh >= a.OH || ow >= a.OW) return -1;
  return ((long long)n * a.OH + oh) * a.OW + ow;
}

// k-th tile of this CTA (-1 when done).  Mode 8 hands out whole (image, strip pair) tasks so a
// CTA walks one task's pooled rows in order (the previous stem row stays in registers).
__device__ __forceinline__ int tile_at(const Geo& g, int k, int num_tiles) {
  if (g.mode == 8) {
    const int task = blockIdx.x + (k / g.tlen) * gridDim.x;
    return task < g.n_tasks ? task * g.tlen + (k - (k / g.tlen) * g.tlen) : -1;
  }
  if (g.mc) {
    // the two CTAs of a cluster walk the same (M-tile pair, N tile) items in lockstep, rank r
    // taking M tile 2p + r (beyond the last tile: OOB loads read zeros, stores are clipped)
    const int q = (int)(blockIdx.x >> 1) + k * (int)(gridDim.x >> 1);
    if (q >= g.n_pairs) return -1;
    const int tp = q / g.n_tiles, tn = q - tp * g.n_tiles;
    return (2 * tp + (int)(blockIdx.x & 1)) * g.n_tiles + tn;
  }
  const int t = blockIdx.x + k * gridDim.x;
  return t < num_tiles ? t : -1;
}

// Spatial origin of m-tile tm in mode 4 (output coordinates).
__device__ __forceinline__ void tile_origin(const Geo& g, int tm, int* w0, int* h0, int* b0) {
  if (g.mode == 8) {  // (image, strip pair, segment, tile): strip coordinate 2p, s2d rows from 2po
    const int t = tm % g.tlen, task = tm / g.tlen;
    const int seg = task % g.nseg, pt = task / g.nseg;
    const int po = seg * g.seg_rows - 1 + t;  // t = 0: the warm-up tile (pooled row before the segment)
    *b0 = pt / g.strips;              // g.strips = strip pairs per image in mode 8
    *w0 = 2 * (pt % g.strips);
    *h0 = 2 * po;                     // -2 for the first segment: TMA zero fill
    return;
  }
  const int tw = tm % g.tiles_w, th = (tm / g.tiles_w) % g.tiles_h, tb = tm / (g.tiles_w * g.tiles_h);
  *w0 = tw * g.wb;
  *h0 = th * g.hb;
  *b0 = tb * g.nb;
}

// Row of the output box (staging / residual block) that tile row i lands in, or -1.
__device__ __forceinline__ int staging_row(const Geo& g, int i, int OW) {
  if (g.mode != 6) return i;
  const int h = i / g.we, w = i - (i / g.we) * g.we;
  return (w < OW && h < g.hb) ? h * OW + w : -1;
}

// ------------------------------------------------------------------ the kernel
template <int BN, int MODE>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    conv_tc_kernel(const ConvArgs a, const Geo g, const __grid_constant__ CUtensorMap tmap_a,
                   const __grid_constant__ CUtensorMap tmap_b, const __grid_constant__ CUtensorMap tmap_y,
                   const __grid_constant__ CUtensorMap tmap_r, const __grid_constant__ CUtensorMap tmap_a2,
                   const __grid_constant__ CUtensorMap tmap_b2, const __grid_constant__ CUtensorMap tmap_bh) {
  using C = Cfg<BN>;
  constexpr int SB = C::SB;
  // MODE 9 = halo mode 6 with two M sub-tiles per B stage (g.mode stays 6 for the geometry)
  // MODE 10 = im2col mode 5 with two M sub-tiles per weight stage
  constexpr bool HALO = (MODE == 6 || MODE == 9);
  constexpr bool IM2COL = (MODE == 5 || MODE == 10);
  // MODE 11 = 1x1 mode 3 with two M sub-tiles per weight chunk (g.mode stays 3)
  constexpr int MT = (MODE == 9 || MODE == 10 || MODE == 11 || MODE == 12) ? 2 : 1;
  constexpr bool PRO = (MODE == 7 || MODE == 12);  // TMA A with the bn-relu prologue in smem (12: two M sub-tiles)
  constexpr bool FLAT = (MODE == 3 || MODE == 11);  // 2D [M][C] TMA tiles
  // TMEM accumulator buffers: two (the epilogue of tile i overlaps the MMAs of tile i+1) unless
  // MT x BN x 2 exceeds the 512 columns -- MODE 10 at BN = 256 keeps one buffer of 2 x 256 columns
  // (the weight stream halves; the MMAs wait for each tile pair's drain)
  // MODE 8 (the stem, N = 128): four buffers, so the MMAs run up to three pooled rows ahead of the
  // epilogue / pooling chain (each pooled row costs that chain more than its 20 MMAs)
  constexpr int NACC = MODE == 8 ? 4 : (MT * BN * 2 <= 512) ? 2 : 1;
  constexpr int TMEM_ALLOC = MODE == 8 ? 512 : NACC == 2 ? C::TMEM_COLS * MT : BN * MT;
  constexpr bool TMA_A = (FLAT || MODE == 4 || IM2COL || HALO || PRO || MODE == 8);
  constexpr bool SPATIAL = (MODE == 4 || HALO || MODE == 8);
  // 1x1 TMA tiles (mode 3): the epilogue stores per-warp [32 x 32] boxes through the 7th map
  // (tmap_bh, free in mode 3: no multicast there); the CTA-wide staging path is compiled only
  // into the other modes.  (Measured: -3..-5% on the epilogue-bound 1x1 convs.  Tried on the
  // im2col modes too: +7..9% on the MMA-bound 3x3 convs, so they keep the staging block.)
  constexpr bool WARP_STORE = FLAT;
  const int S = g.stages;
  const int AS = (HALO || MODE == 8) ? g.a_stages : S;
  constexpr int CPS = (MODE == 3 && BN <= 128) ? 2 : 1;  // == g.cps (host); mode 4 measured better at 1
  const int ASZ = HALO ? MT * g.a_stage_bytes : MODE == 8 ? g.a_stage_bytes : MT * CPS * A_STAGE_BYTES;  // A slot
  const int BSZ = CPS * C::B_STAGE_BYTES;                               // B ring slot
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = sA + AS * ASZ;
  uint8_t* sY = sB + (g.b_res ? g.k_chunks * C::B_STAGE_BYTES : S * BSZ);  // 2 output staging blocks
  uint8_t* sR = sY + (MODE == 8 ? g.ring_bytes : 2 * C::SB_BYTES);  // residual ring (if has_res)
  float* sBias = reinterpret_cast<float*>(sR + (g.has_res ? g.res_depth * C::SB_BYTES : 0));
  float* sScale = sBias + BN;                                   // mode 7 prologue tables
  float* sShift = sScale + (PRO ? g.pro_c : 0);
  uint64_t* full = reinterpret_cast<uint64_t*>(sShift + (PRO ? g.pro_c : 0));
  uint64_t* empty = full + MAX_B_STAGES;
  uint64_t* afull = empty + MAX_B_STAGES;    // mode 6 halo ring
  uint64_t* aempty = afull + MAX_A_STAGES;
  uint64_t* tfull = aempty + MAX_A_STAGES;
  uint64_t* tempty = tfull + 4;
  uint64_t* rfull = tempty + 4;
  uint64_t* rempty = rfull + MAX_RES;
  uint64_t* bres = rempty + MAX_RES;         // resident weights landed
  uint64_t* lfull = bres + 1;                // mode 7: raw A tile landed (before the transform)
  uint64_t* pready = lfull + MAX_B_STAGES;   // mode 8: stem rows of a tile in the ring
  uint64_t* pfree = pready + 4;              // mode 8: pooling of a tile done (its ring rows free)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pfree + 4);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  griddep_launch_dependents();

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], PRO ? NUM_PROD_THREADS : (TMA_A ? 1 : NUM_PROD_THREADS + 1));
      mbar_init(&empty[s], g.mc ? 2 : 1);  // mc: both CTAs' MMAs release the multicast stage
      mbar_init(&lfull[s], 1);
    }
    for (int i = 0; i < MAX_A_STAGES; ++i) {
      mbar_init(&afull[i], 1);
      mbar_init(&aempty[i], 1);
    }
    for (int i = 0; i < 4; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], (MODE == 4 && g.pool2) ? NUM_EPI_THREADS / 2 : NUM_EPI_THREADS);
    }
    for (int i = 0; i < MAX_RES; ++i) {
      mbar_init(&rfull[i], 1);
      mbar_init(&rempty[i], NUM_EPI_THREADS);
    }
    mbar_init(bres, 1);
    for (int i = 0; i < 4; ++i) {
      mbar_init(&pready[i], NUM_EPI_THREADS);
      mbar_init(&pfree[i], M8_POOL_THREADS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == PROD_WARP0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_b)) : "memory");
    if (TMA_A) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_a)) : "memory");
  }
  if (warp == MMA_WARP) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_ALLOC)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  if (g.mc) cluster_sync_all();  // peers' barriers initialised before any multicast lands
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  griddep_wait();  // the previous kernel's outputs are visible from here on

  const int num_tiles = (g.m_tiles + MT - 1) / MT * g.n_tiles;
  const int OHW = a.OH * a.OW;

  if (PRO && warp == XFORM_TMA_WARP) {
    // ================================================================ mode 7 / 12 loader
    uint32_t stage = 0, phase = 0;
    for (int k_ = 0, tile = tile_at(g, 0, num_tiles); tile >= 0; tile = tile_at(g, ++k_, num_tiles)) {
      const int tm = (tile / g.n_tiles) * MT, tn = tile - (tile / g.n_tiles) * g.n_tiles;
      for (int kc = 0; kc < g.k_chunks; ++kc) {
        mbar_wait(&empty[stage], phase ^ 1);
        if (elect_one()) {
          mbar_arrive_expect_tx(&lfull[stage], MT * g.a_bytes + C::B_STAGE_BYTES);
          tma_load_2d(smem_u32(sA + stage * ASZ), &tmap_a, kc * BK, tm * BM, &lfull[stage]);
          if (MT > 1)  // MODE 12: the second M sub-tile (rows past M read as zeros)
            tma_load_2d(smem_u32(sA + stage * ASZ + A_STAGE_BYTES), &tmap_a, kc * BK, (tm + 1) * BM, &lfull[stage]);
          tma_load_2d(smem_u32(sB + stage * BSZ), &tmap_b, kc * BK, tn * BN, &lfull[stage]);
        }
        __syncwarp();
        if (++stage == (uint32_t)S) { stage = 0; phase ^= 1; }
      }
    }
  } else if (PRO && warp >= PROD_WARP0 && warp < PROD_WARP0 + 4) {
    // ================================================================ mode 7 transform
    // bn-relu prologue applied in shared memory: thread = tile row, its 8 swizzled 16-byte
    // chunks (conflict-free), channel = chunk ^ (row & 7) inside the 64-channel block
    const int pt = threadIdx.x - PROD_WARP0 * 32;
    for (int i = pt; i < g.pro_c; i += NUM_PROD_THREADS) {
      sScale[i] = i < a.C ? __ldg(a.pro_scale + i) : 0.f;
      sShift[i] = i < a.C ? __ldg(a.pro_shift + i) : 0.f;
    }
    asm volatile("bar.sync 2, 128;" ::: "memory");
    // thread -> logical 8-channel group j = pt % 8 of rows pt/8 + 16 i: the group's scale and
    // shift live in registers for the whole stage; 8 consecutive threads cover one 128-byte
    // row (conflict-free), physical chunk = j ^ (row & 7)
    const int j = pt & 7, r0 = pt >> 3;
    uint32_t stage = 0, phase = 0;
    for (int k_ = 0, tile = tile_at(g, 0, num_tiles); tile >= 0; tile = tile_at(g, ++k_, num_tiles)) {
      for (int kc = 0; kc < g.k_chunks; ++kc) {
        const int c0 = kc * BK + j * 8;
        const float4 s0 = lds_f4(smem_u32(sScale + c0));
        const float4 s1 = lds_f4(smem_u32(sScale + c0 + 4));
        const float4 h0 = lds_f4(smem_u32(sShift + c0));
        const float4 h1 = lds_f4(smem_u32(sShift + c0 + 4));
        const float sc[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
        const float sh[8] = {h0.x, h0.y, h0.z, h0.w, h1.x, h1.y, h1.z, h1.w};
        mbar_wait(&lfull[stage], phase);
#pragma unroll 1
        for (int sub = 0; sub < MT; ++sub) {  // MODE 12: both M sub-tiles of the stage
        const uint32_t base = smem_u32(sA + stage * ASZ) + sub * A_STAGE_BYTES;
        uint32_t w[8][4];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int r = r0 + 16 * i;
          asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(w[i][0]), "=r"(w[i][1]), "=r"(w[i][2]), "=r"(w[i][3])
                       : "r"(base + r * 128 + ((j ^ (r & 7)) << 4)));
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int r = r0 + 16 * i;
          uint32_t o[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float2 f = unpack_bf16x2(w[i][q]);
            o[q] = pack_bf16x2(fmaxf(fmaf(f.x, sc[2 * q], sh[2 * q]), 0.f), fmaxf(fmaf(f.y, sc[2 * q + 1], sh[2 * q + 1]), 0.f));
          }
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(base + r * 128 + ((j ^ (r & 7)) << 4)),
                       "r"(o[0]), "r"(o[1]), "r"(o[2]), "r"(o[3])
                       : "memory");
        }
        }
        fence_proxy_async_smem();
        mbar_arrive(&full[stage]);
        if (++stage == (uint32_t)S) { stage = 0; phase ^= 1; }
      }
    }
  } else if (MODE == 8 && ((warp >= M8_POOL_WARP0 && warp < PROD_WARP0 + 4) || warp == RES_WARP ||
                            warp == XFORM_TMA_WARP)) {
    // ================================================================ mode 8 pooling
    // Horizontal half of the 3x3/s2/p1 max: the epilogue already took the vertical max over
    // stem rows 2po-1..2po+1 into V (one row per strip column); pooled column q of strip k =
    // max(V[2qo], V[2qo+1], V[2qo+2]).  Item = (strip, pooled column, 8-channel group): three
    // swizzled 16-byte smem reads, one 16-byte global store.
    const int pt = (warp < PROD_WARP0 + 4 ? warp - M8_POOL_WARP0 : warp - RES_WARP + 3) * 32 + lane;
    __nv_bfloat16* yb = static_cast<__nv_bfloat16*>(a.y);
    // this thread's items (strip k, pooled column qo, channel group cg) are the same in every
    // tile: their smem offsets and pooled-column offsets are computed once
    constexpr int M8_MAX_ITEMS = 3;            // ceil(2 x 30 x 8 / 160)
    uint32_t off[M8_MAX_ITEMS][3];
    int qcol[M8_MAX_ITEMS], cgo[M8_MAX_ITEMS];
    int n_items = 0;
    for (int item = pt; item < 2 * g.pq * 8 && n_items < M8_MAX_ITEMS; item += M8_POOL_THREADS, ++n_items) {
      const int k = item / (g.pq * 8), rem = item - k * (g.pq * 8);
      const int qo = rem >> 3, cg = rem & 7;
#pragma unroll
      for (int dc = 0; dc < 3; ++dc) {
        const int x = 2 * qo + dc;
        off[n_items][dc] = (uint32_t)((k * g.we + x) * 128 + ((cg ^ (x & 7)) << 4));
      }
      qcol[n_items] = k * g.pq + qo;
      cgo[n_items] = cg * 8;
    }
    int t = 0, task = blockIdx.x;
    for (int it = 0; task < g.n_tasks; ++it) {
      const int pt = task / g.nseg, seg = task - pt * g.nseg;
      const int img = pt / g.strips, pair = pt - img * g.strips;
      const int po = seg * g.seg_rows - 1 + t;
      mbar_wait(&pready[it & 3], (it >> 2) & 1);
      if (t > 0 && po < g.ph) {  // the warm-up tile only seeds the vertical pool; rows past ph are dead
        const uint32_t vbuf = smem_u32(sY) + (uint32_t)((it & 3) * (g.ring_bytes / 4));
        __nv_bfloat16* yrow = yb + (((long long)img * g.ph + po) * g.pw + 2 * pair * g.pq) * a.y_ld;
        const int qlim = g.pw - 2 * pair * g.pq;
#pragma unroll
        for (int i = 0; i < M8_MAX_ITEMS; ++i) {
          if (i >= n_items || qcol[i] >= qlim) continue;
          uint32_t mx[4] = {0u, 0u, 0u, 0u};
#pragma unroll
          for (int dc = 0; dc < 3; ++dc) {
            uint32_t u[4];
            asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3])
                         : "r"(vbuf + off[i][dc]));
#pragma unroll
            for (int j = 0; j < 4; ++j) mx[j] = bf16x2_max(mx[j], u[j]);
          }
          *reinterpret_cast<uint4*>(yrow + (long long)qcol[i] * a.y_ld + cgo[i]) = make_uint4(mx[0], mx[1], mx[2], mx[3]);
        }
      }
      mbar_arrive(&pfree[it & 3]);
      if (++t == g.tlen) {
        t = 0;
        task += gridDim.x;
      }
    }
  } else if (MODE == 8 && warp < NUM_EPI_WARPS) {
    // ================================================================ mode 8 epilogue
    // TMEM lane = strip column (strip k = row / we, column x = row % we); accumulator columns
    // 0-63 = stem row 2po, 64-127 = stem row 2po+1 (the MMA's N covers both rows).  Each thread
    // holds 32 channels of both rows, relu(+bias) in fp32, and keeps row 2po+1 in registers for
    // the next pooled row: V = max(row 2po-1, row 2po, row 2po+1) is the vertical pool, written
    // once to smem for the pooling warps (ReLU >= 0, so padding is 0; max commutes with the
    // bf16 rounding, so V equals pooling the rounded stem map).
    const int quarter = warp & 3;
    const int gsel = warp >> 2;
    const int row = quarter * 32 + lane;
    const int k = row / g.we, x = row - (row / g.we) * g.we;
    const bool live = k < 2 && x < 2 * g.pq + 1;
    float prev[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) prev[j] = 0.f;
    // a task = (image, strip pair, segment of seg_rows pooled rows); its first tile is the
    // pooled row before the segment (stem rows -2, -1 -- all padding -- for the first segment),
    // whose only use is to leave relu(stem row 2 h0 - 1) in prev for the segment's first row
    int t = 0, task = blockIdx.x;
    for (int it = 0; task < g.n_tasks; ++it) {
      const int acc = it & 3;
      const int pt = task / g.nseg;
      const int pair = pt % g.strips;
      const int po = (task - pt * g.nseg) * g.seg_rows - 1 + t;
      const int stem_col = 2 * (2 * pair + k) * g.pq - 1 + x;
      const bool valid = live && stem_col >= 0 && stem_col < a.OW;
      const bool valid0 = valid && 2 * po >= 0 && 2 * po < a.OH;  // padding positions are -inf
      const bool valid1 = valid && 2 * po + 1 >= 0 && 2 * po + 1 < a.OH;
      mbar_wait(&tfull[acc], (it >> 2) & 1);
      tc_fence_after();
      uint32_t v0[32], v1[32];
      const uint32_t tb = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * BN + gsel * 32;
      tmem_ld32(tb, v0);
      tmem_ld32(tb + 64, v1);
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      mbar_wait(&pfree[it & 3], ((it >> 2) & 1) ^ 1);
      if (live) {
        const uint32_t dst = smem_u32(sY) + (uint32_t)((it & 3) * (g.ring_bytes / 4) + row * 128);
        // the channel half is a compile-time constant inside, so the bias parameter reads are
        // immediate constant-bank operands of the adds
        auto vpool = [&](auto G) {
          constexpr int GS = decltype(G)::value;
#pragma unroll
          for (int c4 = 0; c4 < 4; ++c4) {
            uint32_t o[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              float f[2];
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                // prev >= 0, so max(prev, a, b) = max(prev, relu(a), relu(b)); padding is -inf
                const int c = c4 * 8 + 2 * j + h;
                const float bc = a.bias_u[GS * 32 + c];
                const float a0 = valid0 ? __uint_as_float(v0[c]) + bc : -INFINITY;
                const float a1 = valid1 ? __uint_as_float(v1[c]) + bc : -INFINITY;
                f[h] = fmaxf(fmaxf(prev[c], a0), a1);
                prev[c] = fmaxf(a1, 0.f);
              }
              o[j] = pack_bf16x2(f[0], f[1]);
            }
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(dst + (((GS * 4 + c4) ^ (x & 7)) << 4)),
                         "r"(o[0]), "r"(o[1]), "r"(o[2]), "r"(o[3])
                         : "memory");
          }
        };
        if (gsel == 0) vpool(std::integral_constant<int, 0>{});
        else vpool(std::integral_constant<int, 1>{});
      }
      fence_proxy_async_smem();
      mbar_arrive(&pready[it & 3]);
      if (++t == g.tlen) {
        t = 0;
        task += gridDim.x;
      }
    }
  } else if (warp >= PROD_WARP0 && warp < PROD_WARP0 + 4) {
    // ================================================================ producer
    const int pt = threadIdx.x - PROD_WARP0 * 32;
    if (TMA_A && MODE != 8 && g.b_res && warp == PROD_WARP0) {
      // all weight chunks of the single N tile, once per CTA
      if (elect_one()) {
        mbar_arrive_expect_tx(bres, (uint32_t)g.k_chunks * C::B_STAGE_BYTES);
        for (int c = 0; c < g.k_chunks; ++c) {
          if (a.k2_diag && c >= g.k1_chunks)
            tma_load_2d(smem_u32(sB + c * C::B_STAGE_BYTES), &tmap_b2, 0, -(c - g.k1_chunks) * BK, bres);
          else
            tma_load_2d(smem_u32(sB + c * C::B_STAGE_BYTES), &tmap_b, c * BK, 0, bres);
        }
      }
      __syncwarp();
    }
    if (MODE == 8) {
      // stem: resident weights (20 K chunks x [2 k-halves][128 n][8], 80 KB) once, then per
      // tile one 5D box {8 ch, we cols, 2 strips, 5 s2d rows, 1} per 8-channel plane: smem
      // [row][strip][col] x 16 B, so each (row, tap column) K chunk is a row-shifted view
      if (warp == PROD_WARP0) {
        if (elect_one()) {
          mbar_arrive_expect_tx(bres, M8_CHUNKS * 4096);
          bulk_load_1d(smem_u32(sB), a.w, M8_CHUNKS * 4096, bres);
        }
        __syncwarp();
        uint32_t ast = 0, aph = 0;
        const uint32_t plane_stride = (uint32_t)g.a_stage_bytes / 2;
        for (int k_ = 0, tile = tile_at(g, 0, num_tiles); tile >= 0; tile = tile_at(g, ++k_, num_tiles)) {
          int w0, h0, b0;
          tile_origin(g, tile, &w0, &h0, &b0);
          mbar_wait(&aempty[ast], aph ^ 1);
          if (elect_one()) {
            mbar_arrive_expect_tx(&afull[ast], g.a_bytes);
            const uint32_t dst = smem_u32(sA + ast * ASZ);
            tma_load_5d(dst, &tmap_a, 0, 0, w0, h0, b0, &afull[ast]);
            tma_load_5d(dst + plane_stride, &tmap_a, 8, 0, w0, h0, b0, &afull[ast]);
          }
          __syncwarp();
          if (++ast == (uint32_t)AS) { ast = 0; aph ^= 1; }
        }
      }
    } else if (HALO) {
      // halo mode: one [(hb+KH-1) x we] pixel box per 64-channel block, then the taps' weights
      if (warp == PROD_WARP0) {
        uint32_t stage = 0, phase = 0, ast = 0, aph = 0;
        const int taps = a.KH * a.KW;
        for (int k_ = 0, tile = tile_at(g, 0, num_tiles); tile >= 0; tile = tile_at(g, ++k_, num_tiles)) {
          const int tm0 = (tile / g.n_tiles) * MT, tn = tile - (tile / g.n_tiles) * g.n_tiles;
          const int nsub = g.m_tiles - tm0 < MT ? g.m_tiles - tm0 : MT;
          for (int cb = 0; cb < g.cblocks; ++cb) {
            mbar_wait(&aempty[ast], aph ^ 1);
            if (elect_one()) {
              // one halo box per M sub-tile (they share every B stage below)
              mbar_arrive_expect_tx(&afull[ast], g.a_bytes * nsub);
              for (int sub = 0; sub < nsub; ++sub) {
                int ow0, oh0, b0;
                tile_origin(g, tm0 + sub, &ow0, &oh0, &b0);
                tma_load_4d(smem_u32(sA + ast * ASZ + sub * g.a_stage_bytes), &tmap_a, cb * BK, ow0 - a.pad,
                            oh0 - a.pad, b0, &afull[ast]);
              }
            }
            __syncwarp();
            if (++ast == (uint32_t)AS) { ast = 0; aph ^= 1; }
            if (g.b_res) continue;
            for (int t = 0; t < taps; ++t) {
              mbar_wait(&empty[stage], phase ^ 1);
              if (elect_one()) {
                mbar_arrive_expect_tx(&full[stage], C::B_STAGE_BYTES);
                tma_load_2d(smem_u32(sB + stage * C::B_STAGE_BYTES), &tmap_b, t * a.C + cb * BK, tn * BN, &full[stage]);
              }
              __syncwarp();
              if (++stage == (uint32_t)S) { stage = 0; phase ^= 1; }
            }
          }
        }
      }
    } else if (TMA_A) {
      // mode 4 with one K chunk per tile (the VGG stem): the producer's per-tile work (tile
      // coordinates: a chain of integer divisions) is longer than the tile's 4 MMAs, so warps
      // 8-11 each take every 4th tile (tile k_ uses stage k_ mod S, as with one producer)
      const int np = (MODE == 4 && g.k_chunks == 1 && !g.mc && S > 4) ? 4 : 1;
      const int pw = warp - PROD_WARP0;
      if (pw < np) {
        uint32_t stage = (uint32_t)pw, phase = 0;
        for (int k_ = pw, tile = tile_at(g, pw, num_tiles); tile >= 0; tile = tile_at(g, k_ += np, num_tiles)) {
          const int tm = (tile / g.n_tiles) * MT, tn = tile - (tile / g.n_tiles) * g.n_tiles;
          // (MT == 1: always one, even for the out-of-range partner tile of an odd multicast pair)
          const int nsub = MT == 1 ? 1 : (g.m_tiles - tm < MT ? g.m_tiles - tm : MT);
          int ow0 = 0, oh0 = 0, b0 = 0, w0 = 0, h0 = 0;
          int w1 = 0, h1 = 0, b1 = 0;  // MODE 10: origin of the second M sub-tile
          int ow1o = 0, oh1o = 0;      // ... in output coordinates (fused-downsample source)
          if (SPATIAL) {
            tile_origin(g, tm, &ow0, &oh0, &b0);
            w0 = ow0 * a.stride - a.pad;
            h0 = oh0 * a.stride - a.pad;
          } else if (IM2COL) {
            // flat tile: its first output pixel (n, oh, ow) -> im2col start position
            const long long m0 = (long long)tm * BM;
            b0 = (int)(m0 / OHW);
            const int rem = (int)(m0 - (long long)b0 * OHW);
            oh0 = rem / a.OW;
            ow0 = rem - oh0 * a.OW;
            w0 = ow0 * a.stride - a.pad;
            h0 = oh0 * a.stride - a.pad;
            if (MT > 1) {
              const long long m1 = m0 + BM;
              b1 = (int)(m1 / OHW);
              const int rem1 = (int)(m1 - (long long)b1 * OHW);
              const int oh1 = rem1 / a.OW, ow1 = rem1 - (rem1 / a.OW) * a.OW;
              w1 = ow1 * a.stride - a.pad;
              h1 = oh1 * a.stride - a.pad;
              ow1o = ow1;
              oh1o = oh1;
            }
          }
          int cb = 0, r = 0, sft = 0;  // (tap, channel block) of chunk kc, tracked incrementally
#pragma unroll 1
          for (int kc = 0; kc < g.k_chunks; kc += CPS) {
            const int nch = g.k_chunks - kc < CPS ? g.k_chunks - kc : CPS;
            mbar_wait(&empty[stage], phase ^ 1);
            if (elect_one()) {
              mbar_arrive_expect_tx(&full[stage], nch * (nsub * g.a_bytes + (g.b_res ? 0 : C::B_STAGE_BYTES)));
              int cb_j = cb, r_j = r, s_j = sft;
#pragma unroll 1
              for (int j = 0; j < nch; ++j) {
                const int ck = kc + j;
                const uint32_t dA = smem_u32(sA + stage * ASZ + j * A_STAGE_BYTES);
                if (ck >= g.k1_chunks) {
                  // second A source: the fused downsample (1x1/stride2 over the block input), or
                  // the identity residual (k2_diag) -- channel block tn*BN + 64 j of the residual
                  // against chunk j of the shared identity (tmap_b2)
                  const int c2 = ck - g.k1_chunks + (a.k2_diag ? tn * (BN / BK) : 0);
                  if (FLAT)
                    tma_load_2d(dA, &tmap_a2, c2 * BK, tm * BM, &full[stage]);
                  else if (IM2COL) {
                    tma_load_im2col_4d(dA, &tmap_a2, c2 * BK, ow0 * a.stride2, oh0 * a.stride2, b0, 0, 0, &full[stage]);
                    if (MT > 1 && nsub > 1)  // MODE 10: the second M sub-tile's downsample rows
                      tma_load_im2col_4d(dA + A_STAGE_BYTES, &tmap_a2, c2 * BK, ow1o * a.stride2, oh1o * a.stride2, b1,
                                         0, 0, &full[stage]);
                  }
                  else
                    tma_load_4d(dA, &tmap_a2, c2 * BK, ow0 * a.stride2, oh0 * a.stride2, b0, &full[stage]);
                } else if (FLAT) {
                  tma_load_2d(dA, &tmap_a, ck * BK, tm * BM, &full[stage]);
                  if (MT > 1 && nsub > 1)  // MODE 11: the second M sub-tile of the weight chunk
                    tma_load_2d(dA + A_STAGE_BYTES, &tmap_a, ck * BK, (tm + 1) * BM, &full[stage]);
                } else if (IM2COL) {
                  tma_load_im2col_4d(dA, &tmap_a, cb_j * BK, w0, h0, b0, (uint16_t)s_j, (uint16_t)r_j, &full[stage]);
                  if (MT > 1 && nsub > 1)
                    tma_load_im2col_4d(dA + A_STAGE_BYTES, &tmap_a, cb_j * BK, w1, h1, b1, (uint16_t)s_j, (uint16_t)r_j,
                                       &full[stage]);
                } else {
                  tma_load_4d(dA, &tmap_a, cb_j * BK, w0 + s_j, h0 + r_j, b0, &full[stage]);
                }
                if (!g.b_res) {
                  const uint32_t dB = smem_u32(sB + stage * BSZ + j * C::B_STAGE_BYTES);
                  if (a.k2_diag && ck >= g.k1_chunks)
                    tma_load_2d(dB, &tmap_b2, 0, -(ck - g.k1_chunks) * BK, &full[stage]);
                  else if (g.mc)  // my half of the weight chunk, multicast into both CTAs
                    tma_load_2d_mc(dB + (blockIdx.x & 1) * (BN / 2) * 128, &tmap_bh, ck * BK,
                                   tn * BN + (int)(blockIdx.x & 1) * (BN / 2), &full[stage], 3);
                  else
                    tma_load_2d(dB, &tmap_b, ck * BK, tn * BN, &full[stage]);
                }
                if (++cb_j == g.cblocks) {
                  cb_j = 0;
                  if (++s_j == a.KW) { s_j = 0; ++r_j; }
                }
              }
            }
            __syncwarp();
            if (++stage == (uint32_t)S) { stage = 0; phase ^= 1; }
#pragma unroll 1
            for (int j = 0; j < nch; ++j) {
              if (++cb == g.cblocks) {
                cb = 0;
                if (++sft == a.KW) { sft = 0; ++r; }
              }
            }
          }
          if (np > 1) {  // skip the other producers' stages (np < S: at most one wrap)
            stage += (uint32_t)(np - 1);
            if (stage >= (uint32_t)S) { stage -= (uint32_t)S; phase ^= 1; }
          }
        }
      }
    } else {
      const char* xb = static_cast<const char*>(a.x);
      const int taps = a.KH * a.KW;
      uint32_t stage = 0, phase = 0;
      const int q = pt & 7;          // 16-byte piece index within a 128-byte row
      const int rsub = pt >> 3;      // rows rsub + 16 i
      for (int k_ = 0, tile = tile_at(g, 0, num_tiles); tile >= 0; tile = tile_at(g, ++k_, num_tiles)) {
        const int tm = tile / g.n_tiles, tn = tile - (tile / g.n_tiles) * g.n_tiles;
        int ih0[8], iw0[8];
        long long ioff[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const long long m = (long long)tm * BM + rsub + 16 * i;
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
        for (int kc = 0; kc < g.k_chunks; ++kc) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (pt == 0) {
            mbar_arrive_expect_tx(&full[stage], C::B_STAGE_BYTES);
            tma_load_2d(smem_u32(sB + stage * C::B_STAGE_BYTES), &tmap_b, kc * BK, tn * BN, &full[stage]);
          }
          const uint32_t a_stage = smem_u32(sA + stage * A_STAGE_BYTES);
          const int k0 = kc * BK + q * 8;
          const int tap = k0 / a.C;
          const int c = k0 - tap * a.C;
          const int r = tap / a.KW, s = tap - (tap / a.KW) * a.KW;
          const bool tap_ok = tap < taps;
          const uint32_t dst0 = a_stage + rsub * 128 + ((q ^ (rsub & 7)) << 4);
          if (MODE == 0) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int ih = ih0[i] + r, iw = iw0[i] + s;
              const bool ok = tap_ok && (unsigned)ih < (unsigned)a.H && (unsigned)iw < (unsigned)a.W;
              const char* src = ok ? xb + ((ioff[i] + (long long)ih * a.W + iw) * a.x_ld + c) * 2 : xb;
              cp_async16(dst0 + i * 2048, src, ok ? 16u : 0u);
            }
            cp_async_mbar_arrive(&full[stage]);
          } else {
            // bn-relu prologue: A := relu(x * scale[c] + shift[c]); padding stays zero
            uint4 raw[8];
            bool okv[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
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
            for (int i = 0; i < 8; ++i) {
              const uint32_t w4[4] = {raw[i].x, raw[i].y, raw[i].z, raw[i].w};
              uint32_t ov[4] = {0u, 0u, 0u, 0u};
              if (okv[i]) {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  const float2 f = unpack_bf16x2(w4[j]);
                  ov[j] = pack_bf16x2(fmaxf(fmaf(f.x, sc[2 * j], sh[2 * j]), 0.f),
                                      fmaxf(fmaf(f.y, sc[2 * j + 1], sh[2 * j + 1]), 0.f));
                }
              }
              asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(dst0 + i * 2048), "r"(ov[0]), "r"(ov[1]),
                           "r"(ov[2]), "r"(ov[3])
                           : "memory");
            }
            fence_proxy_async_smem();
          }
          mbar_arrive(&full[stage]);
          if (++stage == (uint32_t)S) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == MMA_WARP) {
    // ================================================================ MMA issuer
    // The whole warp runs the loop (waits, descriptor math in uniform registers); one
    // elected lane issues the MMAs and their commits.
    {
      // kind::f16 instruction descriptor: D fp32, A/B bf16, both K-major, M=128, N=BN
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                             ((uint32_t)(BM >> 4) << 24);
      const uint32_t sA0 = smem_u32(sA), sB0 = smem_u32(sB);
      uint32_t stage = 0, phase = 0, ast = 0, aph = 0;
      if (TMA_A && g.b_res) mbar_wait(bres, 0);
      int iter = 0;
      for (int k_ = 0, tile = tile_at(g, 0, num_tiles); tile >= 0; tile = tile_at(g, ++k_, num_tiles), ++iter) {
        const int acc = iter % NACC;
        const uint32_t acc_phase = (iter / NACC) & 1;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * MT * BN;
        const int nsub_mma = MT > 1 ? (g.m_tiles - (tile / g.n_tiles) * MT < MT ? g.m_tiles - (tile / g.n_tiles) * MT : MT) : 1;
        if (MODE == 8) {
          // 20 K chunks (s2d row rho, tap column s), K = 16 each, N = 128 = both stem rows of
          // the tile (row 2po uses tap row rho, row 2po+1 tap row rho-1; the weight block holds
          // zeros where a tap does not apply).  A = the box planes of row rho shifted by s
          // columns; M rows = [strip 0 columns | strip 1 columns].  N = 128 runs the tensor
          // core at full rate where two N = 64 tiles were smem-bound (tools/micro/mma_rate.cu).
          const uint32_t plane_stride = (uint32_t)g.a_stage_bytes / 2;
          const uint32_t row_stride = (uint32_t)(2 * g.we * 16);
          mbar_wait(&afull[ast], aph);
          tc_fence_after();
          if (elect_one()) {
            // descriptors built once and advanced by adds (start-address field, 16-byte units):
            // a single lane issues the 20 MMAs back to back
            const uint64_t a0 = make_sdesc_none(sA0 + ast * ASZ, plane_stride, 128);
            const uint64_t b0 = make_sdesc_none(sB0, 2048, 128);
            const uint32_t rs16 = row_stride >> 4;
#pragma unroll
            for (int rho = 0; rho < M8_ROWS; ++rho) {
#pragma unroll
              for (int sft = 0; sft < 4; ++sft)
                mma_bf16(d_tmem, a0 + rho * rs16 + sft, b0 + (rho * 4 + sft) * 256, idesc, (rho | sft) != 0);
            }
            mma_commit(&aempty[ast]);
            mma_commit(&tfull[acc]);
          }
          __syncwarp();
          if (++ast == (uint32_t)AS) { ast = 0; aph ^= 1; }
          continue;
        }
        if (HALO) {
          // tap (r, s) reads the halo shifted by r*we + s rows (the extra we - OW columns per
          // row are garbage rows of the tile, discarded by the epilogue).  With mt = 2 every B
          // stage feeds the MMAs of two M sub-tiles (halves the weight traffic from L2).
          const int tm0 = (tile / g.n_tiles) * MT;
          const int nsub = g.m_tiles - tm0 < MT ? g.m_tiles - tm0 : MT;
          const uint32_t d_base = tmem_base + acc * MT * BN;
          uint32_t accum = 0;
          for (int cb = 0; cb < g.cblocks; ++cb) {
            mbar_wait(&afull[ast], aph);
            tc_fence_after();
            const uint32_t a_base = sA0 + ast * ASZ;
            // descriptors built once per channel block and advanced by adds (start-address
            // field in 16-byte units): tap (r, s) = + (r*we + s) * 8, next K16 step = + 2
            const uint64_t a0 = make_sdesc(a_base);
            const uint64_t a1 = make_sdesc(a_base + (MT > 1 ? g.a_stage_bytes : 0));
            const uint32_t rstep = (uint32_t)g.we * 8u;
            if (g.b_res) {
              // weights resident: all taps of this channel block in one burst
              if (elect_one()) {
                uint64_t bd = make_sdesc(sB0 + cb * C::B_STAGE_BYTES);
                const uint32_t bstep = (uint32_t)(g.cblocks * C::B_STAGE_BYTES) >> 4;
                const int taps = a.KH * a.KW, kw = a.KW;
                const uint32_t wrap = rstep - (uint32_t)(kw - 1) * 8u;
                uint32_t off = 0;
                int sft = 0;
                // one flat tap loop (unrolled by the compiler) keeps the MMAs back to back
#pragma unroll 4
                for (int t = 0; t < taps; ++t) {
                  const uint32_t first = (cb | t) != 0;
#pragma unroll
                  for (int k = 0; k < BK / 16; ++k)
                    mma_bf16(d_base, a0 + off + 2 * k, bd + 2 * k, idesc, k ? 1u : first);
                  if (MT > 1 && nsub > 1) {
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k)
                      mma_bf16(d_base + BN, a1 + off + 2 * k, bd + 2 * k, idesc, k ? 1u : first);
                  }
                  bd += bstep;
                  if (++sft == kw) { sft = 0; off += wrap; } else { off += 8u; }
                }
                mma_commit(&aempty[ast]);
              }
              __syncwarp();
              if (++ast == (uint32_t)AS) { ast = 0; aph ^= 1; }
              continue;
            }
            {
              const int taps = a.KH * a.KW, kw = a.KW;
              const uint32_t wrap = rstep - (uint32_t)(kw - 1) * 8u;
              uint32_t off = 0;
              int sft = 0;
              for (int t = 0; t < taps; ++t) {
                mbar_wait(&full[stage], phase);
                tc_fence_after();
                if (elect_one()) {
                  const uint64_t bd = make_sdesc(sB0 + (int)stage * C::B_STAGE_BYTES);
#pragma unroll
                  for (int k = 0; k < BK / 16; ++k) mma_bf16(d_base, a0 + off + 2 * k, bd + 2 * k, idesc, accum | k);
                  if (MT > 1 && nsub > 1) {
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k)
                      mma_bf16(d_base + BN, a1 + off + 2 * k, bd + 2 * k, idesc, accum | k);
                  }
                  mma_commit(&empty[stage]);
                }
                __syncwarp();
                accum = 1;
                if (++stage == (uint32_t)S) { stage = 0; phase ^= 1; }
                if (++sft == kw) { sft = 0; off += wrap; } else { off += 8u; }
              }
            }
            if (elect_one()) mma_commit(&aempty[ast]);
            __syncwarp();
            if (++ast == (uint32_t)AS) { ast = 0; aph ^= 1; }
          }
          if (elect_one()) mma_commit(&tfull[acc]);
          __syncwarp();
          continue;
        }
#pragma unroll 1
        for (int kc = 0; kc < g.k_chunks; kc += CPS) {
          const int nch = g.k_chunks - kc < CPS ? g.k_chunks - kc : CPS;
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (elect_one()) {
#pragma unroll 1
            for (int j = 0; j < nch; ++j) {
              const uint64_t adesc = make_sdesc(sA0 + stage * ASZ + j * A_STAGE_BYTES);
              const uint64_t bdesc =
                  make_sdesc(g.b_res ? sB0 + (kc + j) * C::B_STAGE_BYTES : sB0 + stage * BSZ + j * C::B_STAGE_BYTES);
#pragma unroll
              for (int k = 0; k < BK / 16; ++k) {
                // advance 16 bf16 = 32 bytes along K inside the 128-byte swizzle atom
                mma_bf16(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, ((kc + j) | k) != 0);
              }
              if (MT > 1 && nsub_mma > 1) {  // MODE 10: the second M sub-tile shares the weight chunk
                const uint64_t adesc1 = adesc + (A_STAGE_BYTES >> 4);
#pragma unroll
                for (int k = 0; k < BK / 16; ++k)
                  mma_bf16(d_tmem + BN, adesc1 + 2 * k, bdesc + 2 * k, idesc, ((kc + j) | k) != 0);
              }
            }
            if (g.mc)
              mma_commit_mc(&empty[stage], 3);  // both CTAs' producers refill this multicast stage
            else
              mma_commit(&empty[stage]);
            if (kc + nch >= g.k_chunks) mma_commit(&tfull[acc]);
          }
          __syncwarp();
          if (++stage == (uint32_t)S) { stage = 0; phase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == RES_WARP) {
    // ================================================================ residual loader
    // Streams the [128 x SB] residual blocks of every output tile, in the order the
    // epilogue consumes them, into a 2-deep smem ring (TMA, same swizzle as the staging).
    if (g.has_res && lane == 0) {
      uint32_t rs = 0, rph = 0;
      for (int k_ = 0, tile = tile_at(g, 0, num_tiles); tile >= 0; tile = tile_at(g, ++k_, num_tiles)) {
        const int tm = tile / g.n_tiles, tn = tile - (tile / g.n_tiles) * g.n_tiles;
        int w0 = 0, h0 = 0, b0 = 0;
        if (SPATIAL) tile_origin(g, tm, &w0, &h0, &b0);
        for (int jb = 0; jb < BN; jb += SB) {
          const int n0 = tn * BN + jb;
          if (n0 >= a.Cout) break;
          mbar_wait(&rempty[rs], rph ^ 1);
          mbar_arrive_expect_tx(&rfull[rs], g.res_box_bytes);
          const uint32_t dst = smem_u32(sR + rs * C::SB_BYTES);
          if (SPATIAL)
            tma_load_4d(dst, &tmap_r, n0, w0, h0, b0, &rfull[rs]);
          else
            tma_load_2d(dst, &tmap_r, n0, tm * BM, &rfull[rs]);
          if (++rs == (uint32_t)g.res_depth) { rs = 0; rph ^= 1; }
        }
      }
    }
  } else if (warp < NUM_EPI_WARPS) {
    // ================================================================ epilogue
    // Thread = tile row (its TMEM lane); warps w and w+4 share lane quarter w%4 and take
    // alternate 32-column sub-chunks.  Per SB-column block: TMEM -> registers, + bias
    // (smem) + residual (TMA-prefetched swizzled smem block), ReLU, bf16 -> swizzled
    // staging block (conflict-free 16-byte stores) -> one TMA store per block.
    const int quarter = warp & 3, gsel = warp >> 2;
    const int row = quarter * 32 + lane;
    const int srow = staging_row(g, row, a.OW);  // row of the TMA box this thread fills (-1: none)
    const int et = threadIdx.x;  // 0..255
    __nv_bfloat16* yb = static_cast<__nv_bfloat16*>(a.y);
    const __nv_bfloat16* rb = static_cast<const __nv_bfloat16*>(a.res);
    uint32_t rs = 0, rph = 0;
    int blk = 0;
    int iter = 0, bias_tn = -1;
    if (MODE == 4 && g.pool2) {
      // conv + 2x2/s2 maxpool, [2 x wb] tiles, one N tile (host-checked): the per-tile epilogue is
      // a latency chain (TMEM drain -> staging -> pooled stores) far longer than the tile's
      // K = 192 MMAs, so two groups of 4 warps (each covering all four TMEM lane quarters and
      // all BN columns) take alternate tiles = alternate accumulator buffers, with their own
      // staging block and named barrier, and the two chains overlap.
      for (int j = et; j < BN; j += NUM_EPI_THREADS) sBias[j] = (a.bias && j < a.Cout) ? __ldg(a.bias + j) : 0.f;
      epi_bar();
      const int grp = gsel, eg = et & 127;
      const uint32_t stg = smem_u32(sY + grp * C::SB_BYTES);
      const int pq = g.wb >> 1, nchunk = BN / 8, PW = a.OW >> 1;
      __nv_bfloat16* yp = static_cast<__nv_bfloat16*>(a.y);
      // the group's tiles are k_ = grp, grp + 2, ...: without multicast (one N tile) the tile index
      // advances by 2 x gridDim.x, so its coordinates are carried forward instead of re-divided
      const bool inc = !g.mc && g.n_tiles == 1;
      const int TW = g.tiles_w, TH = g.tiles_h, D = 2 * (int)gridDim.x;
      const int dw = D % TW, dh = (D / TW) % TH, db = D / (TW * TH);
      int tw = 0, th = 0, tb = 0;
      for (int k_ = grp, tile = tile_at(g, grp, num_tiles); tile >= 0; tile = tile_at(g, k_ += 2, num_tiles)) {
        const int acc = grp;  // == k_ & 1
        mbar_wait(&tfull[acc], (k_ >> 1) & 1);
        tc_fence_after();
        int w0 = 0, h0 = 0, b0 = 0;
        if (!inc) {
          tile_origin(g, tile / g.n_tiles, &w0, &h0, &b0);
        } else {
          if (k_ == grp) {
            tw = tile % TW; th = (tile / TW) % TH; tb = tile / (TW * TH);
          } else {
            tw += dw;
            int c = tw >= TW ? 1 : 0;
            tw -= c * TW;
            th += dh + c;
            c = th >= TH ? 1 : 0;
            th -= c * TH;
            tb += db + c;
          }
          w0 = tw * g.wb; h0 = th * g.hb; b0 = tb * g.nb;
        }
        const uint32_t t_row = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * BN;
#pragma unroll
        for (int sub = 0; sub < BN / 32; ++sub) {
          uint32_t v[32];
          tmem_ld32(t_row + sub * 32, v);
          tmem_wait_ld();
#pragma unroll
          for (int c4 = 0; c4 < 4; ++c4) {
            const int chunk = sub * 4 + c4;
            const uint32_t ba = smem_u32(sBias + chunk * 8);
            const float4 b0v = lds_f4(ba), b1v = lds_f4(ba + 16);
            const float bb[8] = {b0v.x, b0v.y, b0v.z, b0v.w, b1v.x, b1v.y, b1v.z, b1v.w};
            float f[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              f[j] = __uint_as_float(v[c4 * 8 + j]) + bb[j];
              if (a.relu) f[j] = fmaxf(f[j], 0.f);
            }
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(stg + swz_off<C::SWZ>(row, chunk)),
                         "r"(pack_bf16x2(f[0], f[1])), "r"(pack_bf16x2(f[2], f[3])), "r"(pack_bf16x2(f[4], f[5])),
                         "r"(pack_bf16x2(f[6], f[7]))
                         : "memory");
          }
        }
        tc_fence_before();
        mbar_arrive(&tempty[acc]);
        asm volatile("bar.sync %0, 128;" ::"r"(3 + grp) : "memory");  // the group's staging is complete
        for (int it = eg; it < pq * nchunk; it += NUM_EPI_THREADS / 2) {
          const int q = it / nchunk, c = it - q * nchunk;
          uint32_t r[4][4];
#pragma unroll
          for (int d = 0; d < 4; ++d) {
            const int srow_d = (d >> 1) * g.wb + 2 * q + (d & 1);
            asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(r[d][0]), "=r"(r[d][1]), "=r"(r[d][2]), "=r"(r[d][3])
                         : "r"(stg + swz_off<C::SWZ>(srow_d, c)));
          }
          uint4 o;
          o.x = bf16x2_max(bf16x2_max(r[0][0], r[1][0]), bf16x2_max(r[2][0], r[3][0]));
          o.y = bf16x2_max(bf16x2_max(r[0][1], r[1][1]), bf16x2_max(r[2][1], r[3][1]));
          o.z = bf16x2_max(bf16x2_max(r[0][2], r[1][2]), bf16x2_max(r[2][2], r[3][2]));
          o.w = bf16x2_max(bf16x2_max(r[0][3], r[1][3]), bf16x2_max(r[2][3], r[3][3]));
          const long long pix = ((long long)b0 * (a.OH >> 1) + (h0 >> 1)) * PW + (w0 >> 1) + q;
          *reinterpret_cast<uint4*>(yp + pix * a.y_ld + c * 8) = o;
        }
        asm volatile("bar.sync %0, 128;" ::"r"(3 + grp) : "memory");  // staging reads done
      }
      iter = -1;  // (the generic loop below is skipped)
    }
    for (int k_ = 0, tile = (iter < 0 ? -1 : tile_at(g, 0, num_tiles)); tile >= 0;
         tile = tile_at(g, ++k_, num_tiles), ++iter) {
      const int tn = tile - (tile / g.n_tiles) * g.n_tiles;
      const int acc = NACC == 2 ? (iter & 1) : 0;
      const uint32_t acc_phase = NACC == 2 ? ((iter >> 1) & 1) : (iter & 1);
      // bias of this tile's columns -> smem, only when the N tile changes (a global load per
      // tile would put an L2 round trip on every tile of the epilogue-bound small-K convs;
      // the previous tile's readers are past the last epi_bar of that tile)
      if (tn != bias_tn) {
        // (the per-warp store path has no CTA-wide barrier of its own: fence the table here)
        if constexpr (WARP_STORE) epi_bar();
        for (int j = et; j < BN; j += NUM_EPI_THREADS) {
          const int n = tn * BN + j;
          sBias[j] = (a.bias && n < a.Cout) ? __ldg(a.bias + n) : 0.f;
        }
        if constexpr (WARP_STORE) epi_bar();
        bias_tn = tn;
      }
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      // one M tile's epilogue (twice per tile in MODE 9)
      auto epilogue_tile = [&](const int tm, const uint32_t t_row) {
      if (!g.tma_out) {
        // final layer straight into the NCHW send buffer (consecutive rows = consecutive
        // pixels, so thread-per-row stores are coalesced per channel)
        epi_bar();
        const long long m = row_to_m(a, g, tm, row);
        int img = 0, pix = 0;
        if (m >= 0) {
          img = (int)(m / OHW);
          pix = (int)(m - (long long)img * OHW);
        }
#pragma unroll 1
        for (int j0 = gsel * 32; j0 < BN; j0 += 64) {
          uint32_t v[32];
          tmem_ld32(t_row + j0, v);
          tmem_wait_ld();
          const int n0 = tn * BN + j0;
          if (m < 0 || n0 >= a.Cout) continue;
          __nv_bfloat16* yp = yb + ((long long)img * a.Cout + n0) * OHW + pix;
          const __nv_bfloat16* rp = rb ? rb + m * a.res_ld + n0 : nullptr;
          // residual: the thread's 32 channels as four 16-byte loads (not 32 scalar loads)
          float res[32];
          const bool full32 = n0 + 32 <= a.Cout;
          if (rp && full32 && (a.res_ld % 8) == 0) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const uint4 u = __ldg(reinterpret_cast<const uint4*>(rp) + q);
              const uint32_t uu[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
              for (int h = 0; h < 4; ++h) {
                const float2 f2 = unpack_bf16x2(uu[h]);
                res[q * 8 + 2 * h] = f2.x;
                res[q * 8 + 2 * h + 1] = f2.y;
              }
            }
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) res[j] = (rp && n0 + j < a.Cout) ? __bfloat162float(rp[j]) : 0.f;
          }
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            if (n0 + j < a.Cout) {
              float f = __uint_as_float(v[j]) + sBias[j0 + j] + res[j];
              if (a.relu) f = fmaxf(f, 0.f);
              yp[(long long)j * OHW] = __float2bfloat16_rn(f);
            }
          }
        }
        epi_bar();
      } else if constexpr (WARP_STORE) {
        // flat tiles: every warp stages and stores its own [32 rows x 32 cols] boxes (its TMEM
        // lane quarter x its column half of each SB block), so no CTA-wide barrier sits between
        // the TMEM drain and the stores; per-warp double buffer of 2 KB (64-byte swizzle)
        for (int jb = 0; jb < BN; jb += SB) {
          const int n0 = tn * BN + jb;
          if (n0 >= a.Cout) break;  // uniform
          if (g.has_res) mbar_wait(&rfull[rs], rph);
          const uint32_t rsm = smem_u32(sR + rs * C::SB_BYTES);
#pragma unroll
          for (int sub = gsel; sub < SB / 32; sub += 2) {
            const uint32_t stg = smem_u32(sY) + (uint32_t)(warp * 2 + (blk & 1)) * 2048u;
            if (lane == 0) bulk_wait_read1();  // this buffer's store (two boxes ago) has read it
            __syncwarp();
            uint32_t v[32];
            tmem_ld32(t_row + jb + sub * 32, v);
            tmem_wait_ld();
#pragma unroll
            for (int c4 = 0; c4 < 4; ++c4) {
              const int chunk = sub * 4 + c4;
              float f[8];
              {
                const uint32_t ba = smem_u32(sBias + jb + chunk * 8);
                const float4 b0 = lds_f4(ba), b1 = lds_f4(ba + 16);
                const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
                for (int j = 0; j < 8; ++j) f[j] = __uint_as_float(v[c4 * 8 + j]) + bb[j];
              }
              if (g.has_res) {
                uint32_t r0, r1, r2, r3;
                asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                             : "r"(rsm + swz_off<C::SWZ>(row, chunk)));
                const uint32_t rr[4] = {r0, r1, r2, r3};
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  const float2 r2f = unpack_bf16x2(rr[j]);
                  f[2 * j] += r2f.x;
                  f[2 * j + 1] += r2f.y;
                }
              }
              if (a.relu) {
#pragma unroll
                for (int j = 0; j < 8; ++j) f[j] = fmaxf(f[j], 0.f);
              }
              asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(stg + swz_off<64>(lane, c4)),
                           "r"(pack_bf16x2(f[0], f[1])), "r"(pack_bf16x2(f[2], f[3])), "r"(pack_bf16x2(f[4], f[5])),
                           "r"(pack_bf16x2(f[6], f[7]))
                           : "memory");
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_2d(&tmap_bh, stg, n0 + sub * 32, tm * BM + quarter * 32);
              bulk_commit();
            }
            ++blk;
          }
          if (g.has_res) {
            mbar_arrive(&rempty[rs]);
            if (++rs == (uint32_t)g.res_depth) { rs = 0; rph ^= 1; }
          }
        }
      } else {
        int w0 = 0, h0 = 0, b0 = 0;
        if (SPATIAL) tile_origin(g, tm, &w0, &h0, &b0);
        for (int jb = 0; jb < BN; jb += SB) {
          const int n0 = tn * BN + jb;
          if (n0 >= a.Cout) break;  // uniform
          const int buf = blk & 1;
          const uint32_t stg = smem_u32(sY + buf * C::SB_BYTES);
          // staging block `buf` was last stored two blocks ago: wait until TMA read it
          if (et == 0) bulk_wait_read1();
          epi_bar();
          if (g.has_res) mbar_wait(&rfull[rs], rph);
          const uint32_t rsm = smem_u32(sR + rs * C::SB_BYTES);
#pragma unroll
          for (int sub = gsel; sub < SB / 32; sub += 2) {
            uint32_t v[32];
            tmem_ld32(t_row + jb + sub * 32, v);
            tmem_wait_ld();
#pragma unroll
            for (int c4 = 0; c4 < 4; ++c4) {  // 8 columns = one 16-byte chunk
              const int chunk = sub * 4 + c4;
              float f[8];
              {
                const uint32_t ba = smem_u32(sBias + jb + chunk * 8);
                const float4 b0 = lds_f4(ba), b1 = lds_f4(ba + 16);
                const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
                for (int j = 0; j < 8; ++j) f[j] = __uint_as_float(v[c4 * 8 + j]) + bb[j];
              }
              if (srow < 0) continue;
              if (g.has_res) {
                uint32_t r0, r1, r2, r3;
                asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                             : "r"(rsm + swz_off<C::SWZ>(srow, chunk)));
                const uint32_t rr[4] = {r0, r1, r2, r3};
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  const float2 r2f = unpack_bf16x2(rr[j]);
                  f[2 * j] += r2f.x;
                  f[2 * j + 1] += r2f.y;
                }
              }
              if (a.relu) {
#pragma unroll
                for (int j = 0; j < 8; ++j) f[j] = fmaxf(f[j], 0.f);
              }
              asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(stg + swz_off<C::SWZ>(srow, chunk)),
                           "r"(pack_bf16x2(f[0], f[1])), "r"(pack_bf16x2(f[2], f[3])), "r"(pack_bf16x2(f[4], f[5])),
                           "r"(pack_bf16x2(f[6], f[7]))
                           : "memory");
            }
          }
          if (g.has_res) {
            mbar_arrive(&rempty[rs]);
            if (++rs == (uint32_t)g.res_depth) { rs = 0; rph ^= 1; }
          }
          fence_proxy_async_smem();
          epi_bar();
          if (et == 0) {
            if (SPATIAL)
              tma_store_4d(&tmap_y, stg, n0, w0, h0, b0);
            else
              tma_store_2d(&tmap_y, stg, n0, tm * BM);
            bulk_commit();
          }
          ++blk;
        }
      }
      };
      const int tm0 = (tile / g.n_tiles) * MT;
      const uint32_t t_row0 = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * MT * BN;
      epilogue_tile(tm0, t_row0);
      if (MT > 1 && tm0 + 1 < g.m_tiles) epilogue_tile(tm0 + 1, t_row0 + BN);
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
    }
    if (WARP_STORE ? lane == 0 : et == 0) bulk_wait_all();  // (per-warp stores: each warp's lane 0 owns groups)
  }

  tc_fence_before();
  __syncthreads();
  if (g.mc) cluster_sync_all();  // no CTA leaves while its peer may still signal it
  if (warp == MMA_WARP) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_ALLOC)
                 : "memory");
  }
}

bool bres_enabled() {  // HAPI_BRES=1: also keep weights resident in modes 3/4 (experiment)
  static const bool on = [] {
    const char* e = std::getenv("HAPI_BRES");
    return e && e[0] == '1';
  }();
  return on;
}

// 2-CTA weight multicast is correct (parity-tested) but measured neutral-to-slower on
// ResNet-50 b512 (+1.5%: the weight stream is not the limiter), so it is opt-in: HAPI_CLUSTER=1.
bool cluster_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("HAPI_CLUSTER");
    return e && e[0] == '1';
  }();
  return on;
}

// Residual ring depth: the deepest ring that costs no pipeline stage (measured on ResNet-50
// b512: depth 3 beats 2 by 8% on the +res convs; depth 4/6 lose a BN=256 stage and are slower).
// HAPI_RES_DEPTH overrides.
int res_depth_pick(int stage_bytes, int fixed, int sb_bytes) {
  static const int forced = [] {
    const char* e = std::getenv("HAPI_RES_DEPTH");
    return e ? std::atoi(e) : 0;
  }();
  if (forced) return forced < 2 ? 2 : (forced > MAX_RES ? MAX_RES : forced);
  auto stages = [&](int d) { return (SMEM_LIMIT - fixed - d * sb_bytes) / stage_bytes; };
  const int s2 = stages(2) > MAX_STAGES ? MAX_STAGES : stages(2);
  int d = 2;
  while (d < MAX_RES && stages(d + 1) >= s2) ++d;
  return d;
}

template <int BN, int MODE>
cudaError_t launch_t(const ConvArgs& a, Geo g, const ConvMaps& mp, int num_sms, cudaStream_t st) {
  using C = Cfg<BN>;
  static std::atomic<uint64_t> attr_mask{0};  // per instantiation, one bit per device
  {
    cudaError_t e = ensure_smem_attr(attr_mask, conv_tc_kernel<BN, MODE>, SMEM_LIMIT);
    if (e != cudaSuccess) return e;
  }
  g.res_box_bytes = (g.mode == 4 || g.mode == 6) ? C::SB * 2 * g.wb * g.hb * g.nb : C::SB_BYTES;
  int smem;
  g.cps = (g.mode == 3 && BN <= 128 && g.mt == 1) ? 2 : 1;
  g.res_depth = res_depth_pick(g.cps * C::STAGE_BYTES, C::FIXED, C::SB_BYTES);
  const int res_bytes = g.has_res ? g.res_depth * C::SB_BYTES : 0;
  const int bres_bytes = g.k_chunks * C::B_STAGE_BYTES;
  const bool tma_a = g.mode == 3 || g.mode == 4 || g.mode == 5 || g.mode == 6 || g.mode == 8;
  const int a_ring = g.a_stages * g.mt * g.a_stage_bytes;  // mode 6 halo ring
  const int a_min = g.mode == 6 ? a_ring : 4 * A_STAGE_BYTES;
  // resident weights: measured win in halo mode; in modes 3/4 (e.g. the stem) it was slower
  g.b_res = tma_a && g.n_tiles == 1 && (g.mode == 6 || bres_enabled()) &&
            C::FIXED + res_bytes + a_min + bres_bytes <= SMEM_LIMIT;
  const int pro_bytes = g.mode == 7 ? 8 * g.pro_c : 0;
  if (g.mode == 8) {
    g.b_res = 1;
    g.stages = 2;  // B ring unused (placeholder for the barrier init loop)
    if (2 * g.we > BM) return cudaErrorInvalidValue;
    const int ring_extra = g.ring_bytes > 2 * C::SB_BYTES ? g.ring_bytes - 2 * C::SB_BYTES : 0;
    smem = g.a_stages * g.a_stage_bytes + bres_bytes + C::FIXED + ring_extra;
    if (smem > SMEM_LIMIT) return cudaErrorInvalidValue;
  } else if (g.mode == 6) {
    if (g.b_res) {
      g.stages = 1;  // B ring unused
      smem = a_ring + bres_bytes + C::FIXED + res_bytes;
    } else {
      const int rest = SMEM_LIMIT - C::FIXED - res_bytes - a_ring;
      g.stages = rest / C::B_STAGE_BYTES;
      if (g.stages > MAX_B_STAGES) g.stages = MAX_B_STAGES;
      if (g.stages < 2) return cudaErrorInvalidValue;
      smem = a_ring + g.stages * C::B_STAGE_BYTES + C::FIXED + res_bytes;
    }
  } else if (g.b_res) {
    g.stages = (SMEM_LIMIT - C::FIXED - res_bytes - bres_bytes) / (g.cps * g.mt * A_STAGE_BYTES);
    if (g.stages > MAX_STAGES) g.stages = MAX_STAGES;
    smem = g.stages * g.cps * g.mt * A_STAGE_BYTES + bres_bytes + C::FIXED + res_bytes;
  } else {
    const int stage_bytes = g.cps * (g.mt * A_STAGE_BYTES + C::B_STAGE_BYTES);
    g.stages = (SMEM_LIMIT - C::FIXED - res_bytes - pro_bytes) / stage_bytes;
    if (g.stages > MAX_STAGES) g.stages = MAX_STAGES;
    smem = g.stages * stage_bytes + C::FIXED + res_bytes + pro_bytes;
  }
  if (g.stages < 2 && !(g.mode == 6 && g.b_res)) return cudaErrorInvalidValue;
  // 2-CTA clusters with multicast weights: the generic TMA path, weights streamed (not
  // resident), no identity block, at least two M tiles; every weight chunk then crosses L2
  // once per CTA pair instead of once per CTA
  g.mc = 0;
  if ((g.mode == 4 || g.mode == 5) && g.mt == 1 && !g.b_res && !a.k2_diag && BN >= 128 && mp.bh &&
      g.m_tiles >= 2 && cluster_enabled()) {
    g.mc = 1;
    g.n_pairs = (g.m_tiles + 1) / 2 * g.n_tiles;
  }
  const int tiles = g.mode == 8 ? g.n_tasks : g.mc ? 2 * g.n_pairs : (g.m_tiles + g.mt - 1) / g.mt * g.n_tiles;
  int grid = tiles < num_sms ? tiles : num_sms;
  if (g.mc) grid &= ~1;
  if (grid <= 0) return cudaSuccess;
  const CUtensorMap* b = mp.b;
  if (!g.mc)
    return launch_pdl(conv_tc_kernel<BN, MODE>, dim3(grid), dim3(NUM_THREADS), (size_t)smem, st, a, g,
                      mp.a ? *mp.a : *b, *b, mp.y ? *mp.y : *b, mp.r ? *mp.r : *b, mp.a2 ? *mp.a2 : *b,
                      mp.b2 ? *mp.b2 : *b, ((MODE == 3 || MODE == 11) && mp.yw) ? *mp.yw : *b);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(NUM_THREADS);
  cfg.dynamicSmemBytes = (size_t)smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, conv_tc_kernel<BN, MODE>, a, g, mp.a ? *mp.a : *b, *b, mp.y ? *mp.y : *b,
                            mp.r ? *mp.r : *b, mp.a2 ? *mp.a2 : *b, mp.b2 ? *mp.b2 : *b, *mp.bh);
}

template <int BN>
cudaError_t launch_mode(const ConvArgs& a, const Geo& g, const ConvMaps& mp, int num_sms, cudaStream_t st) {
  switch (g.mode) {
    case 0: return launch_t<BN, 0>(a, g, mp, num_sms, st);
    case 2: return launch_t<BN, 2>(a, g, mp, num_sms, st);
    case 3:
      if (g.mt == 2) {
        if constexpr (BN == 128 || BN == 256) return launch_t<BN, 11>(a, g, mp, num_sms, st);
        return cudaErrorInvalidValue;
      }
      return launch_t<BN, 3>(a, g, mp, num_sms, st);
    case 4: return launch_t<BN, 4>(a, g, mp, num_sms, st);
    case 5:
      if (g.mt == 2) {
        if constexpr (BN <= 128 || BN == 256) return launch_t<BN, 10>(a, g, mp, num_sms, st);
        return cudaErrorInvalidValue;
      }
      return launch_t<BN, 5>(a, g, mp, num_sms, st);
    case 6:
      if (g.mt == 2) {
        if constexpr (BN <= 128) return launch_t<BN, 9>(a, g, mp, num_sms, st);
        return cudaErrorInvalidValue;
      }
      return launch_t<BN, 6>(a, g, mp, num_sms, st);
    case 7:
      if (g.mt == 2) {
        if constexpr (BN == 128) return launch_t<BN, 12>(a, g, mp, num_sms, st);
        return cudaErrorInvalidValue;
      }
      return launch_t<BN, 7>(a, g, mp, num_sms, st);
    case 8:
      if constexpr (BN == 128) return launch_t<BN, 8>(a, g, mp, num_sms, st);
      return cudaErrorInvalidValue;
  }
  return cudaErrorInvalidValue;
}

}  // namespace

bool dual_m_ntiles_enabled() {  // HAPI_DUAL_M_NT=1: MODE 10 at BN = 256 also when Cout > 256 (experiment)
  static const bool on = [] {
    const char* e = std::getenv("HAPI_DUAL_M_NT");
    return e && e[0] == '1';
  }();
  return on;
}

bool dual_m_ds_enabled() {  // HAPI_DUAL_M_DS=1: ... also with the fused 1x1/s2 downsample source (experiment)
  static const bool on = [] {
    const char* e = std::getenv("HAPI_DUAL_M_DS");
    return e && e[0] == '1';
  }();
  return on;
}

bool dual_m1x1_enabled() {  // HAPI_DUAL_M1X1=1: 1x1 convs with two M sub-tiles per weight chunk (MODE 11)
  static const bool on = [] {
    const char* e = std::getenv("HAPI_DUAL_M1X1");
    return e && e[0] == '1';
  }();
  return on;
}

bool dual_m256_enabled() {  // HAPI_DUAL_M256=0: im2col convs at BN = 256 with one M tile per weight chunk
  static const bool on = [] {
    const char* e = std::getenv("HAPI_DUAL_M256");
    return !(e && e[0] == '0');
  }();
  return on;
}

bool dual_m_pro_enabled() {  // MODE 12 (mode 7 with two M sub-tiles); HAPI_DUAL_M_PRO=0: off
  static const bool on = [] {
    const char* e = std::getenv("HAPI_DUAL_M_PRO");
    return !(e && e[0] == '0');
  }();
  return on;
}

bool dual_m32_enabled() {  // the halo mode's two M sub-tiles also at BN = 32 (DenseNet 3x3); HAPI_DUAL_M32=0: off
  static const bool on = [] {
    const char* e = std::getenv("HAPI_DUAL_M32");
    return !(e && e[0] == '0');
  }();
  return on;
}

bool dual_m_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("HAPI_DUAL_M");
    return !(e && e[0] == '0');
  }();
  return on;
}

int conv_tc_pick_bn(int cout) {
  if (cout <= 32) return 32;
  if (cout <= 64) return 64;
  if (cout <= 128) return 128;
  if (cout == 192) return 192;
  return cout % 256 == 0 ? 256 : 128;
}

int conv_tc_store_cols(int bn) { return bn < 64 ? bn : 64; }

void conv_tc_spatial_tile(int OH, int OW, int N, int* wb, int* hb, int* nb) {
  const int tiles_w = (OW + BM - 1) / BM;
  *wb = (OW + tiles_w - 1) / tiles_w;
  const int hmax = BM / *wb;
  const int tiles_h = (OH + hmax - 1) / hmax;
  *hb = (OH + tiles_h - 1) / tiles_h;
  *nb = 1;
  if (*hb == OH && tiles_w == 1) {
    *nb = BM / (*wb * *hb);
    if (*nb > N) *nb = N;
    if (*nb < 1) *nb = 1;
  }
}

cudaError_t conv_tc_launch(const ConvArgs& a, const ConvMaps& mp, int bn, int mode, int wb, int hb, int nb, int num_sms,
                           cudaStream_t st) {
  Geo g{};
  g.mode = mode;
  g.mt = 1;
  g.n_tiles = (a.Cout + bn - 1) / bn;
  g.has_res = a.res != nullptr;
  g.tma_out = !a.nchw;
  if (mode == 8) {
    // stem conv fused with the 3x3/s2/p1 maxpool: a tile is one pooled row of a pair of
    // strips of pq pooled columns (2 pq + 1 stem columns + 3 tap columns = we box columns per
    // strip); tasks = images x strip pairs, each walked row by row by one CTA
    if (a.Cout > 64 || a.C != BK || a.stride != 1 || bn != 128) return cudaErrorInvalidValue;
    g.pw = (a.OW - 1) / 2 + 1;
    g.ph = (a.OH - 1) / 2 + 1;
    const int S = (g.pw + 29) / 30;
    g.pq = (g.pw + S - 1) / S;
    g.strips = (S + 1) / 2;                    // strip pairs
    // pooled rows split into nseg segments per (image, strip pair) so the task count fills the
    // last wave (b512 at 224: 512 tasks = 3.46 waves -> 1024 = 6.92); each segment pays one
    // warm-up tile.  Pick the split with the shortest makespan, waves x (seg_rows + 1)
    {
      const int pairs = a.N * g.strips;
      long long best = -1;
      static const int max_seg = [] {  // HAPI_STEM_SEG=0: one task per (image, strip pair)
        const char* e = std::getenv("HAPI_STEM_SEG");
        return (e && e[0] == '0') ? 1 : 8;
      }();
      for (int ns = 1; ns <= max_seg && ns <= g.ph; ++ns) {
        const int rows = (g.ph + ns - 1) / ns;
        const long long waves = ((long long)pairs * ns + num_sms - 1) / num_sms;
        const long long span = waves * (rows + 1);
        if (best < 0 || span < best) { best = span; g.nseg = ns; g.seg_rows = rows; }
      }
      g.tlen = g.seg_rows + 1;
      g.n_tasks = pairs * g.nseg;
    }
    g.we = 2 * g.pq + 4;
    g.wb = 2 * g.pq + 1; g.hb = 2; g.nb = 1;
    g.tiles_w = 1; g.tiles_h = 1;
    g.m_tiles = g.n_tasks * g.tlen;
    g.cblocks = 1;
    g.k_chunks = 5;                            // resident weights: 5 x 16 KB = 20 chunks x 4 KB
    g.a_bytes = 2 * (16 * g.we * 2 * M8_ROWS); // two planes of [5 rows][2 strips][we] x 16 B
    {
      // the MMA of the last row reads 128 rows + 3 shifted columns past that row's start
      const int plane = ((M8_ROWS - 1) * 2 * g.we + 128 + 3) * 16;
      const int pstride = (plane + 127) / 128 * 128;
      g.a_stage_bytes = 2 * pstride;
    }
    g.a_stages = 4;
    g.ring_bytes = 4 * 2 * g.we * 128;         // four buffers of vertically pooled rows
    g.tma_out = 0;
  } else if (mode == 6) {
    // halo tile: full output rows (wb = OW), hb rows, one image; extended width we = OW + KW - 1
    if (a.stride != 1 || a.C % BK != 0) return cudaErrorInvalidValue;
    g.we = a.OW + a.KW - 1;
    g.wb = a.OW; g.hb = hb; g.nb = 1;
    g.tiles_w = 1;
    g.tiles_h = (a.OH + hb - 1) / hb;
    g.m_tiles = g.tiles_h * a.N;
    g.cblocks = a.C / BK;
    g.k_chunks = a.KH * a.KW * g.cblocks;
    g.a_bytes = BK * 2 * g.we * (hb + a.KH - 1);
    const int rows_read = (a.KH - 1) * g.we + (a.KW - 1) + BM;   // by the last tap's MMA
    const int rows = rows_read > g.a_bytes / 128 ? rows_read : g.a_bytes / 128;
    g.a_stage_bytes = (rows * 128 + 1023) / 1024 * 1024;
    g.a_stages = 2;
    // two M sub-tiles per B stage (TMEM: 2 buffers x 2 sub-tiles x BN <= 512 columns): halves
    // the weight stream from L2 -- measured -25% on ResNet-50 stage-2 3x3 (BN=128); at BN=64
    // the MMA is smem-bound and it lost 9%, so BN=128 -- and BN=32 (DenseNet's 3x3 128->32: the
    // 4-row halo box halves the input re-read of the 2-row one, -12%) -- if >= 4 B stages still fit
    {
      const int sb = bn < 64 ? bn : 64;
      const int fixed = 2 * sb * 2 * BM + bn * 4 + 2048;
      const int need = 2 * g.a_stages * g.a_stage_bytes + fixed + 4 * bn * BK * 2;
      if ((bn == 128 || (bn == 32 && dual_m32_enabled())) && g.n_tiles == 1 && !a.res && need <= SMEM_LIMIT && dual_m_enabled()) g.mt = 2;
    }
  } else if (mode == 4) {
    if (a.pool2) {
      if (hb != 2 || nb != 1 || (wb & 1) || a.OW % wb != 0 || (a.OH & 1) || a.res || a.nchw || a.y_ld % 8 != 0 ||
          a.k2_chunks > 0 || bn > 64 || a.Cout != bn)
        return cudaErrorInvalidValue;
      g.pool2 = 1;
    }
    g.wb = wb; g.hb = hb; g.nb = nb;
    g.tiles_w = (a.OW + wb - 1) / wb;
    g.tiles_h = (a.OH + hb - 1) / hb;
    g.m_tiles = g.tiles_w * g.tiles_h * ((a.N + nb - 1) / nb);
    g.cblocks = a.C / BK;
    g.k_chunks = a.KH * a.KW * g.cblocks;
    g.a_bytes = BK * 2 * wb * hb * nb;
  } else {
    g.m_tiles = (int)((a.M + BM - 1) / BM);
    g.k_chunks = (a.K + BK - 1) / BK;
    g.cblocks = a.C / BK;
    g.a_bytes = A_STAGE_BYTES;
    if (mode == 7) {
      // TMA-loaded 1x1 A with the bn-relu prologue applied in smem (C % 8 == 0)
      if (a.KH != 1 || a.KW != 1 || a.stride != 1 || a.pad != 0 || a.C % 8 != 0 || !a.pro_scale || !mp.a)
        return cudaErrorInvalidValue;
      g.pro_c = (a.C + BK - 1) / BK * BK;
    }
  }
  // im2col convs at BN = 128: two M sub-tiles share every weight chunk (halves the L2 weight
  // stream; TMEM 2 x 2 x 128 columns)
  if (mode == 5 && bn == 128 && g.n_tiles == 1 && !a.res && a.k2_chunks == 0 && dual_m_enabled()) g.mt = 2;
  // ... and at BN = 256 (one accumulator buffer of 2 x 256 columns): the 3x3 convs of ResNet-50
  // stage 3 move 1.38 GB through L2 per launch at BN = 256 x 1 M tile (the weights re-read per
  // 128-pixel tile are two thirds of it); two M tiles per weight chunk cut that to ~0.9 GB
  if (mode == 5 && bn == 256 && !a.res && !a.k2_diag && dual_m_enabled() && dual_m256_enabled() &&
      (g.n_tiles == 1 || dual_m_ntiles_enabled()) && (a.k2_chunks == 0 || dual_m_ds_enabled()))
    g.mt = 2;
  // 1x1 convs without a residual (every bottleneck's conv1) likewise: the K = 512..2048 weight
  // chunks are re-read per 128-row tile otherwise (ResNet-50 stage 3 conv1: 411 of 616 MB through
  // L2 per launch).  Measured a loss (stage-3 conv1 +8%, layer3.0.conv1 +16%: with one TMEM
  // buffer the short-K tiles wait for every drain), so opt-in: HAPI_DUAL_M1X1=1 (MODE 11)
  if (mode == 3 && (bn == 256 || bn == 128) && !a.res && a.k2_chunks == 0 && a.nchw == 0 && dual_m_enabled() &&
      dual_m1x1_enabled() && (long long)((g.m_tiles + 1) / 2) * g.n_tiles >= 2LL * num_sms)
    g.mt = 2;
  // the DenseNet bottleneck 1x1 convs (bn-relu prologue, long K = 64..1000): two M sub-tiles per
  // weight chunk halve the weight stream from L2 (MODE 12)
  if (mode == 7 && bn == 128 && g.n_tiles == 1 && !a.res && a.nchw == 0 && dual_m_enabled() && dual_m_pro_enabled())
    g.mt = 2;
  g.k1_chunks = g.k_chunks;
  if (a.k2_chunks > 0) {
    if ((mode != 3 && mode != 4 && mode != 5) || !mp.a2 || (a.k2_diag && (!mp.b2 || bn > 256))) return cudaErrorInvalidValue;
    g.k_chunks += a.k2_chunks;
  }
  if ((mode == 3 || mode == 4 || mode == 5 || mode == 6 || mode == 8) && (!mp.a || a.C % BK != 0)) return cudaErrorInvalidValue;
  if (g.tma_out && !mp.y) return cudaErrorInvalidValue;
  if (g.tma_out && mode == 3 && !mp.yw) return cudaErrorInvalidValue;  // per-warp store map
  if (g.has_res && g.tma_out && !mp.r) return cudaErrorInvalidValue;
  if (g.has_res && !g.tma_out) g.has_res = 0;  // NCHW path reads the residual directly
  switch (bn) {
    case 32: return launch_mode<32>(a, g, mp, num_sms, st);
    case 64: return launch_mode<64>(a, g, mp, num_sms, st);
    case 128: return launch_mode<128>(a, g, mp, num_sms, st);
    case 192: return launch_mode<192>(a, g, mp, num_sms, st);
    case 256: return launch_mode<256>(a, g, mp, num_sms, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace hapi
