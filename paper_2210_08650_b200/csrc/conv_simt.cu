// fp32 implicit-GEMM convolution on CUDA cores (FFMA, fp32 accumulate).
//
// The fp32 activation path of the hot path (HAPI_F32): B200 tensor cores have no fp32
// mode and TF32 misses the 1e-5 tolerance, so the paper's fp32
// precision (reading R7) is served by SIMT FFMA.  Same fusion surface as the tcgen05
// kernel: folded-BN bias, bn-relu prologue, residual, ReLU, channel-offset / NCHW store.
//
// Tile 128 (pixels) x 64 (out channels) x 16 (K), 256 threads, 8x4 outputs per thread
// (float4 shared loads), register-prefetched double buffering through shared memory; small
// grids split K (see conv_simt_launch).
#include "kernels.h"

namespace hapi {
namespace {

constexpr int TM = 128, TN = 64, TK = 16;
constexpr int RM = 8, RN = 4;                 // outputs per thread (rows x cols)
constexpr int KTAB = 1024;                    // (r, s, c) table for the generic gather

__global__ void __launch_bounds__(256)
    conv_simt_kernel(const ConvArgs a) {
  __shared__ __align__(16) float As[2][TK][TM + 4];
  __shared__ __align__(16) float Bs[2][TK][TN];
  __shared__ int ktab[KTAB];                  // generic gather: k -> (r << 20) | (s << 10) | c

  griddep_launch_dependents();
  const int tid = threadIdx.x;
  // fast path (C % 16 == 0, 16-byte aligned rows): a 16-wide K tile lies inside one filter tap,
  // so each thread's 8 consecutive channels are one bounds check and two float4 loads
  const bool fast = (a.C % TK == 0) && (a.x_ld % 4 == 0) && (a.Cout % 4 == 0) && !a.pro_scale;
  const bool table = !fast && a.K <= KTAB && a.C < 1024 && a.KW < 1024;
  if (table) {
    for (int k = tid; k < a.K; k += 256) {
      const int tap = k / a.C, c = k - (k / a.C) * a.C;
      ktab[k] = ((tap / a.KW) << 20) | ((tap % a.KW) << 10) | c;
    }
  }
  griddep_wait();
  const long long m_base = (long long)blockIdx.x * TM;
  const int n_base = blockIdx.y * TN;
  const float* x = static_cast<const float*>(a.x);
  const float* w = static_cast<const float*>(a.w);
  const int OHW = a.OH * a.OW;

  // A loader: row = tid / 2 (128 rows), k = (tid % 2) * 8 + j (16 k)
  const int a_row = tid >> 1;
  const int a_k = (tid & 1) * 8;
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
  if (table) __syncthreads();

  float ra[8], rb[4];
  auto load_tile = [&](int k0) {
    if (fast) {
      const int tap = k0 / a.C;
      const int c = k0 - tap * a.C + a_k;
      const int r = tap / a.KW, s = tap - (tap / a.KW) * a.KW;
      const int ih = ih0 + r, iw = iw0 + s;
      float4 v0 = make_float4(0.f, 0.f, 0.f, 0.f), v1 = v0;
      if (k0 < a.K && (unsigned)ih < (unsigned)a.H && (unsigned)iw < (unsigned)a.W) {
        const float4* src = reinterpret_cast<const float4*>(x + (ioff + (long long)ih * a.W + iw) * a.x_ld + c);
        v0 = __ldg(src);
        v1 = __ldg(src + 1);
      }
      ra[0] = v0.x; ra[1] = v0.y; ra[2] = v0.z; ra[3] = v0.w;
      ra[4] = v1.x; ra[5] = v1.y; ra[6] = v1.z; ra[7] = v1.w;
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int k = k0 + a_k + j;
        float v = 0.f;
        if (k < a.K) {
          int r, s, c;
          if (table) {
            const int e = ktab[k];
            r = e >> 20; s = (e >> 10) & 1023; c = e & 1023;
          } else {
            const int tap = k / a.C;
            c = k - tap * a.C;
            r = tap / a.KW; s = tap % a.KW;
          }
          const int ih = ih0 + r, iw = iw0 + s;
          if ((unsigned)ih < (unsigned)a.H && (unsigned)iw < (unsigned)a.W) {
            v = __ldg(x + (ioff + (long long)ih * a.W + iw) * a.x_ld + c);
            if (a.pro_scale) v = fmaxf(fmaf(v, __ldg(a.pro_scale + c), __ldg(a.pro_shift + c)), 0.f);
          }
        }
        ra[j] = v;
      }
    }
    const int kb = k0 + b_k;
    if (a.Cout % 4 == 0) {
      float4 u = make_float4(0.f, 0.f, 0.f, 0.f);
      if (kb < a.K && n_base + b_n < a.Cout) u = __ldg(reinterpret_cast<const float4*>(w + (long long)kb * a.Cout + n_base + b_n));
      rb[0] = u.x; rb[1] = u.y; rb[2] = u.z; rb[3] = u.w;
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int n = n_base + b_n + j;
        rb[j] = (kb < a.K && n < a.Cout) ? __ldg(w + (long long)kb * a.Cout + n) : 0.f;
      }
    }
  };
  auto store_tile = [&](int buf) {
#pragma unroll
    for (int j = 0; j < 8; ++j) As[buf][a_k + j][a_row] = ra[j];
    *reinterpret_cast<float4*>(&Bs[buf][b_k][b_n]) = make_float4(rb[0], rb[1], rb[2], rb[3]);
  };

  // thread (ty, tx): rows ty*8 .. +8, columns tx*4 .. +4
  const int ty = tid >> 4, tx = tid & 15;
  float acc[RM][RN] = {};
  // K slice of this CTA (split-K: blockIdx.z of ksplit; slices are whole TK tiles)
  const int nk_all = (a.K + TK - 1) / TK;
  const int ks = a.ksplit > 1 ? a.ksplit : 1;
  const int per = (nk_all + ks - 1) / ks;
  const int kt0 = blockIdx.z * per;
  const int nk = (kt0 + per < nk_all ? kt0 + per : nk_all) - kt0;
  if (nk > 0) {
    load_tile(kt0 * TK);
    store_tile(0);
    __syncthreads();
    for (int kt = 0; kt < nk; ++kt) {
      const int cur = kt & 1;
      if (kt + 1 < nk) load_tile((kt0 + kt + 1) * TK);
#pragma unroll
      for (int kk = 0; kk < TK; ++kk) {
        const float4 a0 = *reinterpret_cast<const float4*>(&As[cur][kk][ty * RM]);
        const float4 a1 = *reinterpret_cast<const float4*>(&As[cur][kk][ty * RM + 4]);
        const float4 b0 = *reinterpret_cast<const float4*>(&Bs[cur][kk][tx * RN]);
        const float av[RM] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
        const float bv[RN] = {b0.x, b0.y, b0.z, b0.w};
#pragma unroll
        for (int i = 0; i < RM; ++i)
#pragma unroll
          for (int j = 0; j < RN; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
      }
      if (kt + 1 < nk) store_tile(cur ^ 1);
      __syncthreads();
    }
  }
  if (ks > 1) {
    // raw partial sums; the reduce kernel applies the epilogue
    float* wz = a.ws + (long long)blockIdx.z * a.M * a.Cout;
#pragma unroll
    for (int i = 0; i < RM; ++i) {
      const long long m = m_base + ty * RM + i;
      if (m >= a.M) continue;
#pragma unroll
      for (int j = 0; j < RN; ++j) {
        const int n = n_base + tx * RN + j;
        if (n < a.Cout) wz[m * a.Cout + n] = acc[i][j];
      }
    }
    return;
  }

  float* y = static_cast<float*>(a.y);
  const float* res = static_cast<const float*>(a.res);
#pragma unroll
  for (int i = 0; i < RM; ++i) {
    const long long m = m_base + ty * RM + i;
    if (m >= a.M) continue;
    int img = 0, pix = 0;
    if (a.nchw) {
      img = (int)(m / OHW);
      pix = (int)(m - (long long)img * OHW);
    }
#pragma unroll
    for (int j = 0; j < RN; ++j) {
      const int n = n_base + tx * RN + j;
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

// out = epilogue(sum over slices, in slice order) -- one thread per output element
__global__ void __launch_bounds__(256) splitk_reduce_kernel(const ConvArgs a) {
  griddep_launch_dependents();
  griddep_wait();
  const long long total = a.M * a.Cout;
  const long long stride = (long long)gridDim.x * blockDim.x;
  float* y = static_cast<float*>(a.y);
  const float* res = static_cast<const float*>(a.res);
  const int OHW = a.OH * a.OW;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
    const long long m = e / a.Cout;
    const int n = (int)(e - m * a.Cout);
    float v = 0.f;
    for (int z = 0; z < a.ksplit; ++z) v += a.ws[(long long)z * total + e];
    if (a.bias) v += __ldg(a.bias + n);
    if (res) v += __ldg(res + m * a.res_ld + n);
    if (a.relu) v = fmaxf(v, 0.f);
    if (a.nchw) {
      const int img = (int)(m / OHW), pix = (int)(m - (long long)img * OHW);
      y[((long long)img * a.Cout + n) * OHW + pix] = v;
    } else {
      y[m * a.y_ld + n] = v;
    }
  }
}

}  // namespace

cudaError_t conv_simt_launch(const ConvArgs& a, cudaStream_t st) {
  const long long mt = (a.M + TM - 1) / TM;
  const int nt = (a.Cout + TN - 1) / TN;
  if (mt <= 0 || nt <= 0) return cudaSuccess;
  const int ks = a.ksplit > 1 && a.ws ? a.ksplit : 1;
  dim3 grid((unsigned)mt, (unsigned)nt, (unsigned)ks);
  ConvArgs b = a;
  b.ksplit = ks;
  cudaError_t e = launch_pdl(conv_simt_kernel, grid, dim3(256), 0, st, b);
  if (e != cudaSuccess || ks == 1) return e;
  const long long total = a.M * a.Cout;
  long long blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  return launch_pdl(splitk_reduce_kernel, dim3((unsigned)blocks), dim3(256), 0, st, b);
}

int conv_simt_ksplit(long long M, int Cout, int K, int num_sms) {
  // split K when the output grid leaves most of the GPU idle (small batches: config 1)
  const long long tiles = ((M + TM - 1) / TM) * ((Cout + TN - 1) / TN);
  const int nk = (K + TK - 1) / TK;
  int ks = 1;
  while (ks < 8 && tiles * ks < 2LL * num_sms && nk / (ks * 2) >= 16) ks *= 2;
  return ks;
}

}  // namespace hapi
