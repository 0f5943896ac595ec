// fp32 implicit-GEMM convolution on CUDA cores (FFMA, fp32 accumulate).
//
// The fp32 activation path of the hot path (HAPI_F32): B200 tensor cores have no fp32
// mode and TF32 misses the 1e-5 tolerance, so the paper's fp32
// precision (reading R7) is served by SIMT FFMA.  Same fusion surface as the tcgen05
// kernel: folded-BN bias, bn-relu prologue, residual, ReLU, channel-offset / NCHW store.
//
// Tile 64 (pixels) x 64 (out channels) x 16 (K), 256 threads, 4x4 outputs per thread,
// register-prefetched double buffering through shared memory.
#include "kernels.h"

namespace hapi {
namespace {

constexpr int TM = 64, TN = 64, TK = 16;

__global__ void __launch_bounds__(256)
    conv_simt_kernel(const ConvArgs a) {
  __shared__ float As[2][TK][TM + 4];
  __shared__ float Bs[2][TK][TN];

  griddep_launch_dependents();
  griddep_wait();
  const int tid = threadIdx.x;
  const long long m_base = (long long)blockIdx.x * TM;
  const int n_base = blockIdx.y * TN;
  const float* x = static_cast<const float*>(a.x);
  const float* w = static_cast<const float*>(a.w);
  const int OHW = a.OH * a.OW;

  // A loader: row = tid / 4 (64 rows), k = (tid % 4) * 4 + j (16 k)
  const int a_row = tid >> 2;
  const int a_k = (tid & 3) * 4;
  const long long am = m_base + a_row;
  int ih0 = -(1 << 28), iw0 = 0;
  long long ioff = 0;
  if (am < a.M) {
    const int n = (int)(am / OHW);
    const int rem = (int)(am - (long long)n * OHW);
    const int oh = rem / a.OW, ow = rem % a.OW;
    ih0 = oh * a.stride - a.pad;
    iw0 = ow * a.stride - a.pad;
    ioff = (long long)n * a.H * a.W;
  }
  // B loader: k = tid / 16, n = (tid % 16) * 4 + j
  const int b_k = tid >> 4;
  const int b_n = (tid & 15) * 4;

  float ra[4], rb[4];
  auto load_tile = [&](int k0) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int k = k0 + a_k + j;
      float v = 0.f;
      if (k < a.K) {
        const int tap = k / a.C;
        const int c = k - tap * a.C;
        const int r = tap / a.KW, s = tap % a.KW;
        const int ih = ih0 + r, iw = iw0 + s;
        if ((unsigned)ih < (unsigned)a.H && (unsigned)iw < (unsigned)a.W) {
          v = __ldg(x + (ioff + (long long)ih * a.W + iw) * a.x_ld + c);
          if (a.pro_scale) v = fmaxf(fmaf(v, __ldg(a.pro_scale + c), __ldg(a.pro_shift + c)), 0.f);
        }
      }
      ra[j] = v;
    }
    const int kb = k0 + b_k;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n_base + b_n + j;
      rb[j] = (kb < a.K && n < a.Cout) ? __ldg(w + (long long)kb * a.Cout + n) : 0.f;
    }
  };
  auto store_tile = [&](int buf) {
#pragma unroll
    for (int j = 0; j < 4; ++j) As[buf][a_k + j][a_row] = ra[j];
#pragma unroll
    for (int j = 0; j < 4; ++j) Bs[buf][b_k][b_n + j] = rb[j];
  };

  const int ty = tid >> 4, tx = tid & 15;
  float acc[4][4] = {};
  const int nk = (a.K + TK - 1) / TK;
  load_tile(0);
  store_tile(0);
  __syncthreads();
  for (int kt = 0; kt < nk; ++kt) {
    const int cur = kt & 1;
    if (kt + 1 < nk) load_tile((kt + 1) * TK);
#pragma unroll
    for (int kk = 0; kk < TK; ++kk) {
      float av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = As[cur][kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = Bs[cur][kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    if (kt + 1 < nk) store_tile(cur ^ 1);
    __syncthreads();
  }

  float* y = static_cast<float*>(a.y);
  const float* res = static_cast<const float*>(a.res);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const long long m = m_base + ty * 4 + i;
    if (m >= a.M) continue;
    int img = 0, pix = 0;
    if (a.nchw) {
      img = (int)(m / OHW);
      pix = (int)(m - (long long)img * OHW);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n_base + tx * 4 + j;
      if (n >= a.Cout) continue;
      float v = acc[i][j];
      if (a.bias) v += __ldg(a.bias + n);
      if (res) v += __ldg(res + m * a.res_ld + n);
      if (a.relu) v = fmaxf(v, 0.f);
      if (a.nchw)
        y[((long long)img * a.Cout + n) * OHW + pix] = v;
      else
        y[m * a.y_ld + n] = v;
    }
  }
}

}  // namespace

cudaError_t conv_simt_launch(const ConvArgs& a, cudaStream_t st) {
  const long long mt = (a.M + TM - 1) / TM;
  const int nt = (a.Cout + TN - 1) / TN;
  if (mt <= 0 || nt <= 0) return cudaSuccess;
  dim3 grid((unsigned)mt, (unsigned)nt);
  return launch_pdl(conv_simt_kernel, grid, dim3(256), 0, st, a);
}

}  // namespace hapi
