// A whole ResNet bottleneck in one kernel on a CTA pair (sm_100a, tcgen05.mma.cta_group::2):
//   t1  = relu(x  * W1 + b1)            1x1, C -> 64      (BN1 folded)
//   t2  = relu(t1 (*) W2 + b2)          3x3/s1/p1, 64 -> 64
//   out = relu(t2 * W3 + b3 + x)        1x1, 64 -> C, identity residual
// Rows a3/a5 of the hot path; the prefix forward "executes the feature extraction
// part up to the split index" -- this is the block-level fusion SURVEY 7.2 H1
// plans for the HBM-bound stage-1 blocks: x is read from HBM once (the residual comes back
// from L2), t1 and t2 never leave the SMs.
//
// Why a CTA pair: the three weight tensors (136 KB bf16 at C = 256) plus the x ring, the t1
// row ring and t2 do not fit one SM's 227 KB.  With cta_group::2 every MMA is M = 256 (128
// rows from each CTA) and each CTA holds only its half of B's N rows: 68 KB of resident
// weights per CTA.  The two CTAs walk the same (image pair, row pair) tiles in lockstep, CTA r
// on image 2i + r; the leader (rank 0) issues every MMA.
//
// Tiles: one tile = two image rows x 64 positions (position p = column p - 1; 0 and >= W+1
// are zero padding), M = 128 per CTA.  Rolling rows: a segment of row pairs [pa, pb] of one
// image pair is computed as   step k:  C2(pa + k - 3)   C1(pa - 1 + k)   C3(pa + k - 4)
// (the C1 tiles -1 and PR produce the zero rows above and below the image).  t1 lives in a
// ring of six 8 KB row slots (row r -> slot (r + 1) mod 6) plus shadow copies of slots 0, 1,
// so the four rows 2p-1 .. 2p+2 conv2 reads are always one contiguous window; each 3x3 tap is
// the window shifted by (dr * 64 + dc - 1) positions (row-shifted SW128 descriptors).
// Every TMEM lane is one tile position in all three GEMMs, so an epilogue thread handles the
// same position through E1 (t1 row slot), E2 (t2) and E3 (+ residual, global store).
//
// Warps (448 threads per CTA): 0-7 E3 (lane quarter w & 3, column half w >> 2 of the C output
// columns), 8-11 E1 and E2 (lane quarter w & 3, all 64 columns) -- separate warps so the
// residual-and-store epilogue of tile p overlaps the t1/t2 epilogues of tiles p+1, p+2 --,
// 12 TMA producer (weights once, then the x chunks), 13 TMEM allocator + (leader) MMA issuer.
//
// Memory path (DESIGN.md section 10 has the measurements): x is TMA-read with an L2 evict_last
// policy and re-read as the residual by E3 with evict_first (its last use), so the residual
// comes from L2; the output streams out with evict_first.  E3 owns one position per lane and
// moves it with 256-bit loads / stores; the biases are kernel parameters (uniform operands).
// E3's global accesses are the kernel's limiter (the MMA issuer waits on D3 draining).
#include <cstdio>
#include <cuda_bf16.h>

#include "kernels.h"
#include "tc_ptx.cuh"

namespace hapi {
namespace {
using namespace tcx;

#ifndef BLK_UWARP
#define BLK_UWARP 1  // warp index through shfl: uniform registers, no S2R rematerialization in loops
#endif
#ifndef BLK_HINT
#define BLK_HINT 1  // L2 eviction hints: x evict_last until its residual read, out evict_first
#endif
#ifndef BLK_EXP
#define BLK_EXP 0  // experiment switches for A/B builds only (1 no residual, 2 no store, 4 no x TMA,
                   // 8 E1 ignores C2DONE, 16 C2 one tap row, 32 print wait cycles,
                   // 64 L2 prefetch of x two tiles ahead (measured: extra DRAM reads), 128 x TMA evict_normal, 256 out evict_normal)
#endif
#if BLK_EXP & 32
#define PW(i, stmt) do { const long long t_ = clock64(); stmt; pw[i] += clock64() - t_; } while (0)
#else
#define PW(i, stmt) stmt
#endif
constexpr int B_THREADS = 480;
constexpr int B_E12_WARP0 = 8;          // warps 8-11: E1 and E2 (one per TMEM lane quarter)
constexpr int B_PROD_WARP = 12;
constexpr int B_MMA_WARP = 13;
constexpr int B_XDS_WARP = 14;          // ds blocks: TMA producer of the x tile's second copy (downsample A)
constexpr int B_XS = 4;                 // x ring stages (one 64-channel chunk of a tile each; ds blocks: 3)
constexpr int B_SLOTS = 6;              // t1 row slots (+2 shadows)
constexpr int B_ROW = 64 * 128;         // one t1 row slot: 64 positions x 64 ch bf16
constexpr int B_CHUNK = 128 * 128;      // one [128 x 64] bf16 operand block (16 KB)
constexpr int B_SMEM = 232448;

struct BlkLayout {
  // byte offsets from the 1024-aligned base (identical in both CTAs of the pair)
  int w1, w2, w3, wds, x, xds, t1, t2, bars, total, xs;
  __host__ __device__ static BlkLayout make(int C, int Cout, int ds) {
    BlkLayout L{};
    int o = 0;
    L.w1 = o; o += (C / 64) * (32 * 128);          // W1 half: C/64 chunks of [32 n x 64 k]
    L.w2 = o; o += 9 * (32 * 128);                 // W2 half: 9 taps x [32 x 64]
    L.w3 = o; o += (Cout / 2) * 128;               // W3 half: [Cout/2 n x 64 k]
    L.wds = o; o += ds ? (C / 64) * (Cout / 2) * 128 : 0;  // Wds half: C/64 chunks of [Cout/2 x 64]
    L.xs = ds ? 3 : B_XS;
    L.x = o; o += L.xs * B_CHUNK;
    L.xds = o; o += ds ? B_CHUNK : 0;              // the x tile again, for the downsample MMA
    o += 1024;                                     // guard before the t1 ring (position -1)
    L.t1 = o; o += (B_SLOTS + 2) * B_ROW + 1024;   // ring + 2 shadows + guard after
    L.t2 = o; o += B_CHUNK;
    L.bars = o; o += 512;
    L.total = o + 1024;                            // + alignment slack
    return L;
  }
};

// mbarrier indices (uint64 each) inside the bars area
enum {
  XFULL = 0,            // [B_XS]  leader: both CTAs' x chunk landed (tx bytes of both)
  XEMPTY = 4,           // [B_XS]  each: C1 consumed the stage (leader's commit, multicast)
  WFULL = 8,            // leader: both CTAs' weight halves landed
  D1FULL = 9,           // [2] each: C1 accumulator ready (commit multicast)
  D1EMPTY = 11,         // [2] leader: both epilogues drained D1 (16 warp arrivals)
  D2FULL = 13,          // [2]
  D2EMPTY = 15,         // [2]
  D3FULL = 17,          // each
  D3EMPTY = 18,         // leader
  T1READY = 19,         // [4] leader: E1 of a C1 tile written in both CTAs (16 warp arrivals)
  C2DONE = 23,          // [2] each: C2 finished reading the t1 window (commit multicast)
  T2READY = 25,         // leader: E2 written in both CTAs
  C3DONE = 26,          // each: C3 finished reading t2
  XDSFULL = 27,         // ds: leader: both CTAs' second x tile landed
  XDSEMPTY = 28,        // ds: each: the downsample MMA read it (commit multicast)
  NBARS = 29
};

// wait on a barrier that collects arrivals from the peer CTA.  CTA-scope acquire: the waiter is
// the MMA warp, whose reads of the peer's shared memory happen in the async proxy (a
// cluster-scope acquire compiles to CCTL.IVALL + MEMBAR per poll: measured to stall the
// whole kernel)
__device__ __forceinline__ void mbar_wait_cl(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  uint32_t done = 0, spins = 0;
  uint64_t t0 = 0;
  while (!done) {
    if ((++spins & 1023u) == 0) {
      uint64_t now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (t0 == 0) t0 = now;
      else if (now - t0 > HAPI_WATCHDOG_NS) __trap();
    }
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
  }
}

__device__ __forceinline__ uint32_t mapa_leader(uint32_t local) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(local));
  return r;
}
__device__ __forceinline__ void arrive_remote(uint32_t cluster_addr) {
  // (default .release.cta semantics: a cluster-scope release would put a MEMBAR on every arrival;
  // the data behind these arrivals is consumed by the MMA's async proxy, ordered by the
  // writers' fence.proxy.async)
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// TMA into this CTA's smem, completing on the LEADER's mbarrier (CTA-pair form)
__device__ __forceinline__ void tma2_load_2d(uint32_t dst, const CUtensorMap* map, int x, int y, uint32_t bar_leader) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar_leader)
      : "memory");
}
__device__ __forceinline__ void tma2_load_4d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                             uint32_t bar_leader, uint64_t policy) {
#if BLK_HINT
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, %4, %5}], [%6], %7;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar_leader), "l"(policy)
      : "memory");
#else
  (void)policy;
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar_leader)
      : "memory");
#endif
}
// L2 eviction policies: x stays in L2 between its TMA read (C1) and its residual read (E3),
// which is its last use; the output streams through
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void mma2(uint32_t d, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(ad), "l"(bd), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void commit2(uint64_t* bar) {  // arrive on `bar` in both CTAs
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                   smem_u32(bar)),
               "h"((uint16_t)3)
               : "memory");
}
__device__ __forceinline__ uint32_t idesc2(int n) {  // kind::f16, fp32 D, bf16 A/B K-major, M = 256
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
}

// 256-bit global accesses (one full 32 B sector per lane)
__device__ __forceinline__ void ldg256(const void* p, uint4& a, uint4& b, uint64_t policy) {
#if BLK_HINT
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8], %9;"
      : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
      : "l"(p), "l"(policy));
#else
  (void)policy;
  asm("ld.global.nc.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
      : "l"(p));
#endif
}
__device__ __forceinline__ void stg256(void* p, const uint4& a, const uint4& b, uint64_t policy) {
#if BLK_HINT
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8}, %9;" ::"l"(p),
               "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w), "l"(policy)
               : "memory");
#else
  (void)policy;
  asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(a.x), "r"(a.y), "r"(a.z),
               "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w)
               : "memory");
#endif
}
// packed fp32x2 add (FADD2), round-to-nearest like two scalar adds
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
  float2 r;
  asm("{\n\t.reg .b64 ra, rb, rc;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "add.rn.f32x2 rc, ra, rb;\n\tmov.b64 {%0, %1}, rc;\n\t}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}


// Segment schedule: the pair's tile range [t0, t1) over (image pair, row pair) tiles, split at
// image-pair boundaries.  next_segment() yields (image pair, pa, pb).
struct Seg {
  int ip, pa, pb;
};
__device__ __forceinline__ bool seg_at(int t, int t1, int PR, Seg* s) {
  if (t >= t1) return false;
  s->ip = t / PR;
  s->pa = t - s->ip * PR;
  const int end = (s->ip + 1) * PR < t1 ? (s->ip + 1) * PR : t1;
  s->pb = s->pa + (end - t) - 1;
  return true;
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(B_THREADS, 1)
    conv_block_kernel(const __grid_constant__ BlockArgs a, const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_w1,
                      const __grid_constant__ CUtensorMap tm_w2, const __grid_constant__ CUtensorMap tm_w3,
                      const __grid_constant__ CUtensorMap tm_wds) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const BlkLayout L = BlkLayout::make(a.C, a.Cout, a.ds);
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + L.bars);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + NBARS);
  const uint32_t rank = cluster_ctarank();
#if BLK_UWARP
  const int warp = __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0);  // warp-uniform: kept in uniform registers
#else
  const int warp = threadIdx.x >> 5;
#endif
  const int lane = threadIdx.x & 31;
  const int PR = (a.H + 1) / 2;                 // row pairs per image
  const int npairs = (a.N + 1) / 2;             // image pairs
  const int T = npairs * PR;
  const int cl = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int t0 = (int)((long long)T * cl / ncl), t1 = (int)((long long)T * (cl + 1) / ncl);
  const int kc1 = a.C / 64;                     // K chunks of C1
  griddep_launch_dependents();
#if BLK_EXP & 32
  unsigned long long pw[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const long long t_start = clock64();
#endif

  if (threadIdx.x == 0) {
    for (int i = 0; i < L.xs; ++i) {
      mbar_init(&bars[XFULL + i], 1);
      mbar_init(&bars[XEMPTY + i], 1);
    }
    mbar_init(&bars[WFULL], 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bars[D1FULL + i], 1);
      mbar_init(&bars[D1EMPTY + i], 8);
      mbar_init(&bars[D2FULL + i], 1);
      mbar_init(&bars[D2EMPTY + i], 8);
      mbar_init(&bars[C2DONE + i], 1);
    }
    mbar_init(&bars[D3FULL], 1);
    mbar_init(&bars[D3EMPTY], 16);
    for (int i = 0; i < 4; ++i) mbar_init(&bars[T1READY + i], 8);
    mbar_init(&bars[T2READY], 8);
    mbar_init(&bars[C3DONE], 1);
    mbar_init(&bars[XDSFULL], 1);
    mbar_init(&bars[XDSEMPTY], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // zero the t1 guards and shadows once (the ring slots are always written before read)
  for (int i = threadIdx.x; i < 1024 / 16; i += B_THREADS) {
    *reinterpret_cast<uint4*>(base + L.t1 - 1024 + i * 16) = make_uint4(0, 0, 0, 0);
    *reinterpret_cast<uint4*>(base + L.t1 + (B_SLOTS + 2) * B_ROW + i * 16) = make_uint4(0, 0, 0, 0);
  }
  if (warp == B_MMA_WARP) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // both CTAs' barriers initialised before any cross-CTA signal
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  griddep_wait();

  const uint32_t sbase = smem_u32(base);
  const uint32_t bar0 = smem_u32(bars);
  auto lbar = [&](int i) { return bar0 + 8u * (uint32_t)i; };  // local shared address of barrier i

  if (warp == B_PROD_WARP) {
    // ================================================================ producer
    if (elect_one()) {
      const uint32_t wbar = mapa_leader(lbar(WFULL));
      if (rank == 0) mbar_arrive_expect_tx(&bars[WFULL], 2u * (uint32_t)(L.x - L.w1));
      for (int c = 0; c < kc1; ++c) tma2_load_2d(sbase + L.w1 + c * 4096, &tm_w1, c * 64, (int)rank * 32, wbar);
      for (int t = 0; t < 9; ++t) tma2_load_2d(sbase + L.w2 + t * 4096, &tm_w2, t * 64, (int)rank * 32, wbar);
      tma2_load_2d(sbase + L.w3, &tm_w3, 0, (int)rank * (a.Cout / 2), wbar);
      if (a.ds)
        for (int c = 0; c < kc1; ++c)
          tma2_load_2d(sbase + L.wds + c * (a.Cout / 2) * 128, &tm_wds, c * 64, (int)rank * (a.Cout / 2), wbar);
    }
    __syncwarp();
    const uint64_t pol_last = (BLK_EXP & 128) ? policy_evict_normal() : policy_evict_last();
    uint32_t st = 0, ph = 0;
    Seg s;
    for (int t = t0; seg_at(t, t1, PR, &s); t += s.pb - s.pa + 1) {
      const int img = 2 * s.ip + (int)rank;  // beyond N: TMA zero fill, stores skipped
      for (int q = s.pa - 1; q <= s.pb + 1; ++q) {
        // warm L2 with the rows two tiles ahead: the 4-stage ring holds one tile, so the
        // loads of the next tile have only about one step to arrive
        if ((BLK_EXP & 64) && q + 2 <= s.pb + 1 && elect_one())
          for (int c = 0; c < kc1; ++c)
#if BLK_HINT
            asm volatile("cp.async.bulk.prefetch.tensor.4d.L2.global.L2::cache_hint [%0, {%1, %2, %3, %4}], %5;" ::"l"(
                             reinterpret_cast<uint64_t>(&tm_x)), "r"(c * 64), "r"(-1), "r"(2 * (q + 2)), "r"(img), "l"(pol_last)
                         : "memory");
#else
            asm volatile("cp.async.bulk.prefetch.tensor.4d.L2.global [%0, {%1, %2, %3, %4}];" ::"l"(
                             reinterpret_cast<uint64_t>(&tm_x)), "r"(c * 64), "r"(-1), "r"(2 * (q + 2)), "r"(img)
                         : "memory");
#endif
        __syncwarp();
        for (int c = 0; c < kc1; ++c) {
          PW(0, mbar_wait(&bars[XEMPTY + st], ph ^ 1));
          if (BLK_EXP & 4) {
            if (rank == 0 && elect_one()) mbar_arrive(&bars[XFULL + st]);
          } else if (elect_one()) {
            if (rank == 0) mbar_arrive_expect_tx(&bars[XFULL + st], 2u * B_CHUNK);
            tma2_load_4d(sbase + L.x + st * B_CHUNK, &tm_x, c * 64, -1, 2 * q, img, mapa_leader(lbar(XFULL + st)), pol_last);
          }
          __syncwarp();
          if (++st == (uint32_t)L.xs) { st = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == B_XDS_WARP) {
    // ================================================================ ds: second x copy
    // The downsample MMA of tile p runs with C3(p), three steps after C1(p) consumed x(p) from
    // the ring, so x(p) is read again (from L2: the ring's TMA loads mark it evict_last) into
    // one slot, as soon as the previous tile's downsample MMA released it.
    if (a.ds) {
      const uint64_t pol_last = policy_evict_last();
      int n = 0;
      Seg s;
      for (int t = t0; seg_at(t, t1, PR, &s); t += s.pb - s.pa + 1) {
        const int img = 2 * s.ip + (int)rank;
        for (int p = s.pa; p <= s.pb; ++p, ++n) {
          mbar_wait(&bars[XDSEMPTY], (n & 1) ^ 1);
          if (elect_one()) {
            if (rank == 0) mbar_arrive_expect_tx(&bars[XDSFULL], 2u * (uint32_t)(kc1 * B_CHUNK));
            for (int c = 0; c < kc1; ++c)
              tma2_load_4d(sbase + L.xds + c * B_CHUNK, &tm_x, c * 64, -1, 2 * p, img, mapa_leader(lbar(XDSFULL)),
                           pol_last);
          }
          __syncwarp();
        }
      }
    }
  } else if (warp == B_MMA_WARP) {
    // ================================================================ MMA issuer (leader)
    if (rank == 0) {
      const uint32_t id64 = idesc2(64), id256 = idesc2(a.Cout);
      mbar_wait_cl(&bars[WFULL], 0);
      tc_fence_after();
      uint32_t st = 0, ph = 0;
      int n1 = 0, n2 = 0, n3 = 0;  // C1 / C2 / C3 tiles issued so far (buffer + phase counters)
      Seg s;
      for (int t = t0; seg_at(t, t1, PR, &s); t += s.pb - s.pa + 1) {
        const int n = s.pb - s.pa + 1;
        const int c1b = n1;  // C1 sequence number of this segment's first tile (row pair pa - 1)
        for (int k = 0; k <= n + 3; ++k) {
          if (k <= n + 1) {
            // C1(q = pa - 1 + k): x chunks x W1 half -> D1[n1 & 1]
            const int b = n1 & 1;
            PW(0, mbar_wait_cl(&bars[D1EMPTY + b], ((n1 >> 1) & 1) ^ 1));
            tc_fence_after();
            for (int c = 0; c < kc1; ++c) {
              PW(1, mbar_wait_cl(&bars[XFULL + st], ph));
              tc_fence_after();
              if (elect_one()) {
                const uint64_t ad = make_sdesc(sbase + L.x + st * B_CHUNK);
                const uint64_t bd = make_sdesc(sbase + L.w1 + c * 4096);
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) mma2(tmem + b * 64, ad + 2 * kk, bd + 2 * kk, id64, (c | kk) != 0);
                commit2(&bars[XEMPTY + st]);
                if (c == kc1 - 1) commit2(&bars[D1FULL + b]);
              }
              __syncwarp();
              if (++st == (uint32_t)L.xs) { st = 0; ph ^= 1; }
            }
            ++n1;
          }
          if (k >= 3 && k <= n + 2) {
            // C2(p = pa + k - 3): t1 window rows 2p-1 .. 2p+2, written by the E1s of C1 tiles
            // p - 1 .. p + 1 (in order, so waiting for the last suffices)
            const int p = s.pa + k - 3;
            const int need = c1b + (p + 1) - (s.pa - 1);  // sequence number of C1(p + 1), issued last step
            PW(2, mbar_wait_cl(&bars[T1READY + (need & 3)], (need >> 2) & 1));
            const int b = n2 & 1;
            PW(3, mbar_wait_cl(&bars[D2EMPTY + b], ((n2 >> 1) & 1) ^ 1));
            tc_fence_after();
            if (elect_one()) {
              const int slot = ((2 * p) % B_SLOTS + B_SLOTS) % B_SLOTS;  // slot of row 2p-1
              const uint32_t win = sbase + L.t1 + slot * B_ROW;
              const uint64_t a0 = make_sdesc(win);
              const uint64_t b0 = make_sdesc(sbase + L.w2);
              uint32_t first = 0;
#pragma unroll 1
              for (int dr = 0; dr < ((BLK_EXP & 16) ? 1 : 3); ++dr) {
#pragma unroll
                for (int dc = 0; dc < 3; ++dc) {
                  // shift (dr * 64 + dc - 1) positions of 128 B = 8 descriptor units each
                  const int64_t sh = (int64_t)(dr * 64 + dc - 1) * 8;
                  const uint64_t ad = a0 + (uint64_t)sh;
                  const uint64_t bd = b0 + (uint64_t)((dr * 3 + dc) * 4096 >> 4);
#pragma unroll
                  for (int kk = 0; kk < 4; ++kk) {
                    mma2(tmem + 128 + b * 64, ad + 2 * kk, bd + 2 * kk, id64, first | kk);
                  }
                  first = 1;
                }
              }
              commit2(&bars[C2DONE + (n2 & 1)]);
              commit2(&bars[D2FULL + b]);
            }
            __syncwarp();
            ++n2;
          }
          if (k >= 4) {
            // C3(p = pa + k - 4): t2 x W3 half -> D3
            PW(4, mbar_wait_cl(&bars[T2READY], n3 & 1));
            PW(5, mbar_wait_cl(&bars[D3EMPTY], (n3 & 1) ^ 1));
            if (a.ds) mbar_wait_cl(&bars[XDSFULL], n3 & 1);
            tc_fence_after();
            if (elect_one()) {
              const uint64_t ad = make_sdesc(sbase + L.t2);
              const uint64_t bd = make_sdesc(sbase + L.w3);
#pragma unroll
              for (int kk = 0; kk < 4; ++kk) mma2(tmem + 256, ad + 2 * kk, bd + 2 * kk, id256, kk != 0);
              commit2(&bars[C3DONE]);
              if (a.ds) {
                // the residual is the downsample: D3 += x(p) * Wds over the C input channels,
                // from the second copy of the x tile
                for (int c = 0; c < kc1; ++c) {
                  const uint64_t xd = make_sdesc(sbase + L.xds + c * B_CHUNK);
                  const uint64_t wd = make_sdesc(sbase + L.wds + c * (a.Cout / 2) * 128);
#pragma unroll
                  for (int kk = 0; kk < 4; ++kk) mma2(tmem + 256, xd + 2 * kk, wd + 2 * kk, id256, 1u);
                }
                commit2(&bars[XDSEMPTY]);
              }
              commit2(&bars[D3FULL]);
            }
            __syncwarp();
            ++n3;
          }
        }
      }
    }
  } else if (warp >= B_E12_WARP0 && warp < B_E12_WARP0 + 4) {
    // ================================================================ E1 / E2 warps
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;        // TMEM lane = tile position
    const int ri = row >> 6, pos = row & 63;    // row in tile, padded position
    const int col = pos - 1;
    const bool col_ok = col >= 0 && col < a.W;
    const uint32_t lanebase = tmem + ((uint32_t)(quarter * 32) << 16);
    const uint32_t t1ready_l = mapa_leader(lbar(T1READY));
    const uint32_t t2ready_l = mapa_leader(lbar(T2READY));
    const uint32_t d1empty_l = mapa_leader(lbar(D1EMPTY));
    const uint32_t d2empty_l = mapa_leader(lbar(D2EMPTY));
    auto warp_arrive = [&](uint32_t cluster_bar) {
      __syncwarp();
      if (elect_one()) arrive_remote(cluster_bar);
    };
    // relu(v + bias) of 32 accumulator columns (bias: kernel parameter, uniform) -> 16 bf16x2
    auto act32 = [&](const uint32_t (&v)[32], const float* bias, bool ok, uint32_t (&o)[16]) {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const float2 z = add2(make_float2(__uint_as_float(v[2 * j]), __uint_as_float(v[2 * j + 1])),
                              make_float2(bias[2 * j], bias[2 * j + 1]));
        o[j] = ok ? cvt_relu_bf16x2(z.x, z.y) : 0u;
      }
    };
    int n1 = 0, n2 = 0;
    Seg s;
    for (int t = t0; seg_at(t, t1, PR, &s); t += s.pb - s.pa + 1) {
      const int n = s.pb - s.pa + 1;
      const int c2b = n2;  // C2s issued before this segment
      for (int k = 0; k <= n + 2; ++k) {
        if (k <= n + 1) {
          // ---- E1(q): relu(D1 + b1) -> t1 row slot of row 2q + ri (zero outside the image)
          const int q = s.pa - 1 + k;
          const int r = 2 * q + ri;
          const bool ok = col_ok && r >= 0 && r < a.H;
          const int b = n1 & 1;
          PW(0, mbar_wait(&bars[D1FULL + b], (n1 >> 1) & 1));
          tc_fence_after();
          uint32_t v0[32], v1[32];
          tmem_ld32(lanebase + b * 64, v0);
          tmem_ld32(lanebase + b * 64 + 32, v1);
          tmem_wait_ld();
          tc_fence_before();
          warp_arrive(d1empty_l + 8u * b);
          // the slots of rows 2q, 2q+1 held rows 2q-6, 2q-5, last read by C2(q - 2) -- the C2
          // the MMA warp issues right after C1(q); at a segment start, by the previous
          // segment's last C2.  Wait for the latest C2 issued up to this step.
          {
            const int issued = c2b + (k >= 3 ? ((k < n + 2 ? k : n + 2) - 2) : 0);
            if (!(BLK_EXP & 8) && issued > 0) PW(1, mbar_wait(&bars[C2DONE + ((issued - 1) & 1)], ((issued - 1) >> 1) & 1));
          }
          const int slot = ((r + 1) % B_SLOTS + B_SLOTS) % B_SLOTS;
          const uint32_t rowaddr = sbase + L.t1 + slot * B_ROW + pos * 128;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            uint32_t o[16];
            act32(h ? v1 : v0, a.b1 + h * 32, ok, o);
#pragma unroll
            for (int c4 = 0; c4 < 4; ++c4) {
              const uint32_t off = (((h * 4 + c4) ^ (pos & 7)) << 4);
              asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(rowaddr + off), "r"(o[4 * c4]),
                           "r"(o[4 * c4 + 1]), "r"(o[4 * c4 + 2]), "r"(o[4 * c4 + 3])
                           : "memory");
              if (slot < 2)  // shadow copy after the ring (keeps every 4-row window contiguous)
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(rowaddr + B_SLOTS * B_ROW + off),
                             "r"(o[4 * c4]), "r"(o[4 * c4 + 1]), "r"(o[4 * c4 + 2]), "r"(o[4 * c4 + 3])
                             : "memory");
            }
          }
          fence_proxy_async_smem();
          warp_arrive(t1ready_l + 8u * (n1 & 3));
          ++n1;
        }
        if (k >= 3 && k <= n + 2) {
          // ---- E2(p): relu(D2 + b2) -> t2
          const int b = n2 & 1;
          PW(2, mbar_wait(&bars[D2FULL + b], (n2 >> 1) & 1));
          tc_fence_after();
          uint32_t v0[32], v1[32];
          tmem_ld32(lanebase + 128 + b * 64, v0);
          tmem_ld32(lanebase + 128 + b * 64 + 32, v1);
          tmem_wait_ld();
          tc_fence_before();
          warp_arrive(d2empty_l + 8u * b);
          if (n2 >= 1) PW(3, mbar_wait(&bars[C3DONE], (n2 - 1) & 1));  // C3 of the previous tile read t2
          const uint32_t rowaddr = sbase + L.t2 + row * 128;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            uint32_t o[16];
            act32(h ? v1 : v0, a.b2 + h * 32, true, o);
#pragma unroll
            for (int c4 = 0; c4 < 4; ++c4)
              asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(rowaddr + (((h * 4 + c4) ^ (row & 7)) << 4)),
                           "r"(o[4 * c4]), "r"(o[4 * c4 + 1]), "r"(o[4 * c4 + 2]), "r"(o[4 * c4 + 3])
                           : "memory");
          }
          fence_proxy_async_smem();
          warp_arrive(t2ready_l);
          ++n2;
        }
      }
    }
  } else if (warp < 8) {
    // ================================================================ E3 warps
    // Each lane owns one tile position (its TMEM lane) and moves that position's C/2-channel
    // half row with 256-bit loads / stores: every access writes or reads a full 32 B sector,
    // with no data exchange between lanes.
    const int quarter = warp & 3;
#if BLK_UWARP
    const int gsel = warp >> 2;
#else
    const int gsel = __shfl_sync(0xffffffffu, warp >> 2, 0);  // warp-uniform (bias reads use uniform registers)
#endif
    const int row = quarter * 32 + lane;
    const int ri = row >> 6, pos = row & 63;
    const int col = pos - 1;
    const bool col_ok = col >= 0 && col < a.W;
    const uint32_t lanebase = tmem + ((uint32_t)(quarter * 32) << 16);
    const uint32_t d3empty_l = mapa_leader(lbar(D3EMPTY));
    const __nv_bfloat16* xg = static_cast<const __nv_bfloat16*>(a.x);
    __nv_bfloat16* yg = static_cast<__nv_bfloat16*>(a.y);
    const int nsub = a.Cout / 64;               // 32-column blocks of this warp's half (<= 4)
    // the residual of a tile (this thread's C/2 channels, <= 8 x 32 B) is loaded one tile
    // ahead, 32 B at a time: right after step hs of tile p consumed its residual registers,
    // they are reloaded with tile p+1's, so each L2 round trip overlaps a whole tile
    uint4 res[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) res[j] = make_uint4(0, 0, 0, 0);
    const uint64_t pol_first = policy_evict_first();
    const uint64_t pol_out = (BLK_EXP & 256) ? policy_evict_normal() : pol_first;
    auto tile_addr = [&](int img, int p, bool& okk, const __nv_bfloat16*& xr, __nv_bfloat16*& yrr) {
      const int r = 2 * p + ri;
      okk = img < a.N && col_ok && r < a.H;
      const long long pix = ((long long)img * a.H + (okk ? r : 0)) * a.W + (okk ? col : 0);
      xr = xg + pix * a.x_ld + gsel * (a.Cout / 2);
      yrr = yg + pix * a.y_ld + gsel * (a.Cout / 2);
    };
    int n3 = 0;
    Seg s;
    bool have = seg_at(t0, t1, PR, &s);
    int p = have ? s.pa : 0;
    int t = t0;
    bool ok = false;
    const __nv_bfloat16* xr = xg;
    __nv_bfloat16* yr = yg;
    if (have) {
      tile_addr(2 * s.ip + (int)rank, p, ok, xr, yr);
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (!(BLK_EXP & 1) && !a.ds && ok && j < nsub * 2) ldg256(xr + j * 16, res[2 * j], res[2 * j + 1], pol_first);
    }
    while (have) {
      // the next tile in C3 order
      Seg sn = s;
      int pn = p + 1, tn = t;
      bool have_n = true;
      if (pn > s.pb) {
        tn = t + s.pb - s.pa + 1;
        have_n = seg_at(tn, t1, PR, &sn);
        pn = have_n ? sn.pa : 0;
      }
      bool ok_n = false;
      const __nv_bfloat16* xr_n = xg;
      __nv_bfloat16* yr_n = yg;
      if (have_n) tile_addr(2 * sn.ip + (int)rank, pn, ok_n, xr_n, yr_n);
      // ---- E3(p): relu(D3 + b3 + x) -> out (global, valid positions only)
      PW(0, mbar_wait(&bars[D3FULL], n3 & 1));
      tc_fence_after();
      // 16 accumulator columns per step; the TMEM load of step hs + 1 is in flight while
      // step hs computes and stores
      const uint32_t d3 = lanebase + 256 + gsel * (a.Cout / 2);
      uint32_t va[16], vb[16];
      tmem_ld16(d3, va);
      tmem_wait_ld();
#pragma unroll
      for (int hs = 0; hs < 8; ++hs) {
        if (hs >= 2 * nsub) break;
        uint32_t (&v)[16] = (hs & 1) ? vb : va;
        uint32_t (&vn)[16] = (hs & 1) ? va : vb;
        const bool last = hs == 2 * nsub - 1;
        if (!last) tmem_ld16(d3 + (hs + 1) * 16, vn);
        uint4 oq[2];
#pragma unroll
        for (int qq = 0; qq < 2; ++qq) {
          const int q = hs * 2 + qq;            // 8-channel group within the half row
          const uint4 rr = res[q];
          const uint32_t uu[4] = {rr.x, rr.y, rr.z, rr.w};
          const float* bb = a.b3 + gsel * (a.Cout / 2) + q * 8;  // uniform constant-bank operands
          uint32_t o[4];
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const float2 f = unpack_bf16x2(uu[h]);
            const int c = qq * 8 + 2 * h;
            const float2 z = add2(add2(make_float2(__uint_as_float(v[c]), __uint_as_float(v[c + 1])),
                                       make_float2(bb[2 * h], bb[2 * h + 1])), f);
            o[h] = cvt_relu_bf16x2(z.x, z.y);
          }
          oq[qq] = make_uint4(o[0], o[1], o[2], o[3]);
        }
        if (!(BLK_EXP & 1) && !a.ds && ok_n) ldg256(xr_n + hs * 16, res[2 * hs], res[2 * hs + 1], pol_first);
        if (ok && !(BLK_EXP & 2)) stg256(yr + hs * 16, oq[0], oq[1], pol_out);
        tmem_wait_ld();
        if (hs == 2 * nsub - 2) {               // D3 fully loaded (the last step's load landed)
          tc_fence_before();
          __syncwarp();
          if (elect_one()) arrive_remote(d3empty_l);
        }
      }
      ++n3;
      s = sn;
      p = pn;
      t = tn;
      have = have_n;
      ok = ok_n;
      yr = yr_n;
    }
  }

#if BLK_EXP & 32
  if (blockIdx.x < 2 && lane == 0 && (warp == 0 || warp == 4 || warp == 8 || warp == B_PROD_WARP || warp == B_MMA_WARP))
    printf("blkprof cta %d warp %2d total %lld w0 %llu w1 %llu w2 %llu w3 %llu w4 %llu w5 %llu\n", blockIdx.x, warp,
           clock64() - t_start, pw[0], pw[1], pw[2], pw[3], pw[4], pw[5]);
#endif
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // no CTA frees TMEM or exits while its peer may still signal it
  if (warp == B_MMA_WARP) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

}  // namespace

int conv_block_smem_bytes(int C, int Cout, int ds) { return BlkLayout::make(C, Cout, ds).total; }

cudaError_t conv_block_launch(const BlockArgs& a, const BlockMaps& mp, int num_sms, cudaStream_t st) {
  if (a.C % 64 != 0 || a.C > 256 || a.Cout % 64 != 0 || a.Cout > 256 || a.W > 62 || a.W < 1 || a.H < 1 || a.N < 1 ||
      !mp.x || !mp.w1 || !mp.w2 || !mp.w3 || (a.ds ? !mp.wds : a.Cout != a.C))
    return cudaErrorInvalidValue;
  const int smem = BlkLayout::make(a.C, a.Cout, a.ds).total;
  if (smem > B_SMEM) return cudaErrorInvalidValue;
  static std::atomic<uint64_t> attr_mask{0};
  {
    // one attribute for every variant: the identity and downsample layouts differ in size, and a
    // smaller first launch must not leave the attribute too low for a later, larger one
    cudaError_t e = ensure_smem_attr(attr_mask, conv_block_kernel, B_SMEM);
    if (e != cudaSuccess) return e;
  }
  const long long tiles = (long long)((a.N + 1) / 2) * ((a.H + 1) / 2);
  int clusters = num_sms / 2;
  if (tiles < clusters) clusters = (int)tiles;
  if (clusters < 1) return cudaSuccess;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * clusters);
  cfg.blockDim = dim3(B_THREADS);
  cfg.dynamicSmemBytes = (size_t)smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, conv_block_kernel, a, *mp.x, *mp.w1, *mp.w2, *mp.w3, a.ds ? *mp.wds : *mp.w3);
}

}  // namespace hapi
