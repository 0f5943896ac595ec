// Kernel argument structs and launchers (host-callable).  Activations are NHWC
// (channels-last) with an explicit pixel stride `ld` (elements between consecutive
// pixels) so that DenseNet's concatenated block buffers can be read and written
// in place by channel offset.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <utility>

namespace hapi {

// Programmatic dependent launch: every kernel of the plan is launched with the PDL
// attribute, calls griddep_launch_dependents() early and griddep_wait() before its first
// global-memory access, so its prologue (barrier init, TMEM alloc, descriptor prefetch)
// overlaps the previous kernel's tail.  HAPI_PDL=0 disables it.
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("HAPI_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is per device: `mask` (one static per
// kernel instantiation) remembers the device ordinals (< 64) it was applied on.
template <typename K>
cudaError_t ensure_smem_attr(std::atomic<uint64_t>& mask, K kern, int bytes) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = dev < 64 ? (1ull << dev) : 0;
  if (bit && (mask.load(std::memory_order_acquire) & bit)) return cudaSuccess;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess && bit) mask.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}

#ifdef __CUDACC__
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
#endif

// Implicit-GEMM convolution: M = N*OH*OW output pixels, N = Cout, K = KH*KW*C.
struct ConvArgs {
  const void* x;        // input NHWC, pointer already offset to the first consumed channel
  int N, H, W, C;       // C = channels consumed per pixel
  int x_ld;             // elements between pixels of x
  int KH, KW, stride, pad;
  int OH, OW;
  int Cout;
  int K;                // KH*KW*C
  const void* w;        // packed weights (see pack_* in model.cu)
  const float* bias;    // [Cout] fp32 or nullptr
  const float* pro_scale;  // [C] fp32 or nullptr: A := relu(A*scale + shift) (DenseNet bn-relu)
  const float* pro_shift;
  const void* res;      // residual NHWC (same dtype as y) or nullptr
  int res_ld;
  void* y;              // output: NHWC (pointer offset to channel offset) or NCHW base
  int y_ld;
  int relu;             // apply ReLU after bias/residual
  int nchw;             // 1: y is contiguous NCHW [N][Cout][OH][OW]
  long long M;
  // optional second A source, K-concatenated after the first (a ResNet downsample 1x1 conv
  // fused into the block's last conv): k2_chunks 64-channel chunks of a 1x1 conv with
  // stride `stride2` over its own input (TMA modes only)
  int k2_chunks;
  int stride2;
  // k2_diag = 1: the second source is the identity residual (same rows and channels as the
  // output) against an identity weight block; each N tile multiplies only its diagonal
  // BN-channel block (k2_chunks = BN / 64 chunks per tile)
  int k2_diag;
  // fp32 SIMT path: split-K over `ksplit` slices (small grids); raw partial sums go to
  // ws [ksplit][M][Cout] fp32 and a second kernel adds them in slice order (deterministic)
  // with the bias / residual / ReLU epilogue
  int ksplit;
  float* ws;
  // mode 4 with [2 x wb] tiles (wb even, OW % wb == 0, OH even): a 2x2/s2 maxpool follows the
  // conv and is fused into the epilogue; y / y_ld describe the pooled [N][OH/2][OW/2] map
  int pool2;
  // mode 8 (stem + maxpool, Cout <= 64): the bias BY VALUE, read as uniform constant-bank
  // operands by the epilogue (a register copy per thread spilled next to its accumulators)
  float bias_u[64];
};

// tcgen05 / TMEM / TMA path (bf16 activations, fp32 accumulation).  A-operand modes:
//   0  cp.async 16-byte gather (C % 8 == 0): stems (space-to-depth / padded input)
//   2  register gather with the bn-relu prologue (C % 8 == 0): DenseNet
//   3  TMA 2D {64, 128} over the [M][C] matrix (1x1 stride-1 convs, linear layers)
//   4  TMA 4D {64, wb*s, hb*s, nb} per filter tap over NHWC, traversal stride s
// tmap_a: A tensor map (modes 3/4, else nullptr); tmap_b: 2D map over the packed
// [Cout][Kp] bf16 weights with box {64, bn}.
struct ConvMaps {
  const CUtensorMap* a;  // A operand (modes 3/4) or nullptr
  const CUtensorMap* a2; // second A source (k2_chunks > 0) or nullptr
  const CUtensorMap* b2; // k2_diag: the shared 64x64 bf16 identity block, box {64, BN}, loaded at row -64c
  const CUtensorMap* b;  // weights
  const CUtensorMap* bh; // weights with a {64, bn/2} box (2-CTA multicast halves) or nullptr
  const CUtensorMap* y;  // output view (NHWC epilogue via TMA store) or nullptr for NCHW
  const CUtensorMap* r;  // residual view or nullptr
  const CUtensorMap* yw; // output view with a {32, 32} box, 64B swizzle (per-warp epilogue stores) or nullptr
};
// Chained 1x1 pair (conv_pair.cu): a bottleneck's conv3 (+ residual as second A source) and
// the next block's conv1 per 128-row tile; the block output tile stays in smem as conv1's A.
struct PairArgs {
  long long M;          // rows (pixels) of both GEMMs
  int k1_chunks;        // conv3 K / 64 (A from a1, B from b1 columns)
  int k2_chunks;        // second A source chunks per 128-wide N tile: diag = 2, fused ds = its K / 64
  int k2_diag;          // 1: identity residual (a2 channel block of the N tile x identity b2-id)
  int cout1;            // conv3 output channels (multiple of 128, <= 2048)
  const float* bias1;   // [cout1] conv3 bias (+ ds bias)
  const float* bias2;   // [n2] next conv1 bias
  void* y1_sub;         // non-null: store the block output only at even (row, col) pixels, as a
                        // compact [N][(H+1)/2][(W+1)/2][cout1] bf16 tensor (y1 map unused)
  int H, W;             // pixel grid of the M rows (for y1_sub)
};
struct PairMaps {
  const CUtensorMap* a1;  // t2 [M][K1], box {64, 128}
  const CUtensorMap* a2;  // residual / ds input [M][C2], box {64, 128}
  const CUtensorMap* b1;  // conv3 weights [cout1][Kp], box {64, 128}
  const CUtensorMap* id;  // 64x64 identity block, box {64, 128}, loaded at row -64c
  const CUtensorMap* b2;  // next conv1 weights [n2][cout1], box {64, n2}
  const CUtensorMap* y1;  // block output view [M][cout1], box {64, 32} (one row quarter), 128B swizzle
  const CUtensorMap* y2;  // next conv1 output view [M][n2], box {64, 32}, 128B swizzle
};
cudaError_t conv_pair_launch(const PairArgs& a, const PairMaps& mp, int n2, int num_sms, cudaStream_t st);

// A whole identity bottleneck (1x1 C->64, 3x3 64->64, 1x1 64->C + x, each + folded BN + ReLU) on
// a CTA pair (conv_block.cu): x is read once, t1/t2 stay on chip.  C <= 256, W <= 62.
struct BlockArgs {
  int N, H, W, C;        // x: NHWC [N][H][W][C] bf16 (C = block input channels)
  int Cout;              // y: NHWC [N][H][W][Cout]; identity blocks: Cout == C
  int ds;                // 1: the residual is the block's 1x1/s1 downsample of x (+BN), an MMA
                         // over a second copy of the x tile (ResNet layer1.0); 0: identity
  const void* x; int x_ld;
  void* y; int y_ld;     // must not alias x
  // folded BN biases BY VALUE (kernel parameter space): every epilogue lane adds the same
  // bias, which the FADD2s then read as uniform constant-bank operands (no shared loads)
  float b1[64];
  float b2[64];
  float b3[256];         // [Cout], Cout <= 256 (ds: conv3's and the downsample's biases summed)
};
struct BlockMaps {
  const CUtensorMap* x;   // 4D {C, W, H, N} over x, box {64, 64, 2, 1}, SW128
  const CUtensorMap* w1;  // 2D over W1 [64][C], box {64, 32}, SW128
  const CUtensorMap* w2;  // 2D over W2 [64][576] (taps (r, s) x 64 channels), box {64, 32}, SW128
  const CUtensorMap* w3;  // 2D over W3 [Cout][64], box {64, Cout/2}, SW128
  const CUtensorMap* wds; // ds: 2D over Wds [Cout][C], box {64, Cout/2}, SW128 (else nullptr)
};
cudaError_t conv_block_launch(const BlockArgs& a, const BlockMaps& mp, int num_sms, cudaStream_t st);
int conv_block_smem_bytes(int C, int Cout, int ds);

int conv_tc_pick_bn(int cout);
int conv_tc_store_cols(int bn);  // columns per epilogue TMA box (64, or bn if smaller)
void conv_tc_spatial_tile(int OH, int OW, int N, int* wb, int* hb, int* nb);
cudaError_t conv_tc_launch(const ConvArgs& a, const ConvMaps& maps, int bn, int mode, int wb, int hb, int nb,
                           int num_sms, cudaStream_t st);

// SIMT fp32 path (weights packed [K][Cout] fp32).
cudaError_t conv_simt_launch(const ConvArgs& a, cudaStream_t st);
// split-K factor for a small SIMT conv grid (1 = no split)
int conv_simt_ksplit(long long M, int Cout, int K, int num_sms);

// NCHW fp32 images -> NHWC activations.  layout 0: fp32, C=3.  layout 1: bf16, C=8
// (channels 3..7 zero).  layout 2: bf16 space-to-depth 2x2 with a zero border ->
// [N][H/2+3][wp][16] (wp >= W/2+4); padded pixel (i+2, j+3) channel (a*2+b)*3+c holds image pixel
// (2i+a, 2j+b) channel c; channels 12..15 and the border are zero.
// u8 ingest: the images arrive as uint8 NCHW and each value becomes
// scale[c] * u + shift[c] in fp32 before the same packing (fp32 images: nrm == nullptr).
struct InNorm {
  float scale[3], shift[3];
};
cudaError_t pack_input_launch(const void* img, const InNorm* nrm, void* y, int N, int H, int W, int layout, int wp,
                              cudaStream_t st);
// Contiguous NCHW [N][C][HW] (act dtype, es = 2 or 4 bytes) -> NHWC with pixel stride y_ld.
cudaError_t unpack_nchw_launch(const void* x, int N, int C, int HW, void* y, int y_ld, int es, cudaStream_t st);

// Window pooling, NHWC -> NHWC.  mode 0 = max (-inf padding), 1 = avg (count k*k).
struct PoolArgs {
  const void* x; int N, H, W, C, x_ld;
  void* y; int OH, OW, y_ld;
  int k, stride, pad, mode;
  // optional bn-relu prologue: x := relu(x * pro_scale[c] + pro_shift[c]) before pooling (the
  // DenseNet transition commuted to bn-relu -> avgpool -> 1x1 conv, model.cu)
  const float* pro_scale = nullptr;
  const float* pro_shift = nullptr;
};
cudaError_t pool_launch(const PoolArgs& a, int is_bf16, cudaStream_t st);

// Adaptive average pooling (PyTorch bins), optional ReLU on the input first.
struct AdaptiveArgs {
  const void* x; int N, H, W, C, x_ld;
  void* y; int OH, OW, y_ld;
  int relu_in;
};
cudaError_t adaptive_avgpool_launch(const AdaptiveArgs& a, int is_bf16, cudaStream_t st);

// y = x*scale[c] + shift[c] (optionally ReLU); scale == nullptr means identity affine.
struct EltArgs {
  const void* x; int N, HW, C, x_ld;
  void* y; int y_ld;
  const float* scale; const float* shift; int relu;
};
cudaError_t bn_act_launch(const EltArgs& a, int is_bf16, cudaStream_t st);

// NHWC view (ld, already channel-offset) -> contiguous NCHW [N][C][HW] (the send buffer).
cudaError_t pack_output_launch(const void* x, int N, int HW, int C, int x_ld, void* y,
                               int is_bf16, cudaStream_t st);

}  // namespace hapi
