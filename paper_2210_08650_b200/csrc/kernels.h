// Kernel argument structs and launchers (host-callable).  Activations are NHWC
// (channels-last) with an explicit pixel stride `ld` (elements between consecutive
// pixels) so that DenseNet's concatenated block buffers can be read and written
// in place by channel offset.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>

namespace hapi {

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
};

// tcgen05 / TMEM / TMA path (bf16 activations, fp32 accumulation).
//   mode 0: A gathered with 16-byte cp.async (C % 8 == 0)
//   mode 1: A gathered with 8-byte cp.async (C == 4; the packed stem input)
//   mode 2: A via registers with the bn-relu prologue (C % 8 == 0)
// tmap_b: 2D tensor map over the packed [Cout][Kp] bf16 weights, box {64, bn}.
int conv_tc_pick_bn(int cout);
cudaError_t conv_tc_launch(const ConvArgs& a, const CUtensorMap* tmap_b, int bn, int mode,
                           int num_sms, cudaStream_t st);

// SIMT fp32 path (weights packed [K][Cout] fp32).
cudaError_t conv_simt_launch(const ConvArgs& a, cudaStream_t st);

// NCHW fp32 images -> NHWC activations: fp32 with C=3 (is_bf16=0) or bf16 padded to C=4.
cudaError_t pack_input_launch(const float* img, void* y, int N, int H, int W, int is_bf16,
                              cudaStream_t st);

// Window pooling, NHWC -> NHWC.  mode 0 = max (-inf padding), 1 = avg (count k*k).
struct PoolArgs {
  const void* x; int N, H, W, C, x_ld;
  void* y; int OH, OW, y_ld;
  int k, stride, pad, mode;
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
