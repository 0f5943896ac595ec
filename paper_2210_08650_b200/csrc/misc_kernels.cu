// Memory-bound kernels of the hot path:
//   pack_input   a1: caller NCHW fp32 (or u8, normalised on the fly) images -> NHWC activations (bf16 padded to C=4)
//   pool         a4: max 3x3/s2 (-inf padding), max 2x2/s2, avg 2x2/s2 (DenseNet transitions)
//   adaptive     a4: adaptive / global average pool (ResNet avgpool, DenseNet classifier)
//   bn_act       a5: unfused eval BN (+ReLU) at split points inside a DenseNet transition,
//                    norm5, and strided channel copies into a DenseNet block buffer
//   pack_output  a7: NHWC activation -> the contiguous NCHW send buffer
// All are coalesced along channels with 16-byte vector accesses where alignment allows.
#include <cuda_bf16.h>

#include "kernels.h"

namespace hapi {
namespace {

template <typename T>
__device__ __forceinline__ float to_f(T v);
template <>
__device__ __forceinline__ float to_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }
template <typename T>
__device__ __forceinline__ T from_f(float v);
template <>
__device__ __forceinline__ float from_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

// V consecutive elements of T (16 bytes when V*sizeof(T) == 16).
template <typename T, int V>
struct Vec {
  T v[V];
};
template <typename T, int V>
__device__ __forceinline__ void load_vec(const T* p, float (&f)[V]) {
  if constexpr (V * sizeof(T) == 16) {
    const uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
    const Vec<T, V> t = *reinterpret_cast<const Vec<T, V>*>(&u);
#pragma unroll
    for (int i = 0; i < V; ++i) f[i] = to_f<T>(t.v[i]);
  } else {
#pragma unroll
    for (int i = 0; i < V; ++i) f[i] = to_f<T>(p[i]);
  }
}
template <typename T, int V>
__device__ __forceinline__ void store_vec(T* p, const float (&f)[V]) {
  if constexpr (V * sizeof(T) == 16) {
    Vec<T, V> t;
#pragma unroll
    for (int i = 0; i < V; ++i) t.v[i] = from_f<T>(f[i]);
    *reinterpret_cast<uint4*>(p) = *reinterpret_cast<const uint4*>(&t);
  } else {
#pragma unroll
    for (int i = 0; i < V; ++i) p[i] = from_f<T>(f[i]);
  }
}

__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

// ---------------------------------------------------------------- pack_input
// one input value: fp32 as is, u8 through the per-channel affine (one FFMA)
__device__ __forceinline__ float in_val(const float* p, const InNorm&, int) { return __ldg(p); }
__device__ __forceinline__ float in_val(const uint8_t* p, const InNorm& nrm, int c) {
  return fmaf((float)__ldg(p), nrm.scale[c], nrm.shift[c]);
}

template <typename T>
__global__ void pack_input_kernel(const T* __restrict__ img, void* __restrict__ y, int N, int H, int W, int layout,
                                  int wp, const InNorm nrm) {
  griddep_launch_dependents();
  griddep_wait();
  const int HW = H * W;
  if (layout == 2) {
    // space-to-depth 2x2 with a zero border (rows: 2 before, 1 after; columns: 3 before, 1
    // after) so the stem's 4x4 windows -- and the stem+pool kernel's boxes, which start one
    // column left of the stem's first column -- never leave the buffer: one thread per padded
    // pixel of the (H/2+3) x (W/2+4) grid
    const int H2 = H / 2, W2 = W / 2, HP = H2 + 3, WP = wp;
    const long long total = (long long)N * HP * WP;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
      const long long n = t / (HP * WP);
      const int rem = (int)(t - n * HP * WP);
      const int i = rem / WP - 2, j = rem - (rem / WP) * WP - 3;
      float v[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) v[c] = 0.f;
      if (i >= 0 && i < H2 && j >= 0 && j < W2) {
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int b = 0; b < 2; ++b) {
            const T* src = img + n * 3 * HW + (long long)(2 * i + a) * W + (2 * j + b);
#pragma unroll
            for (int c = 0; c < 3; ++c) v[(a * 2 + b) * 3 + c] = in_val(src + c * HW, nrm, c);
          }
      }
      uint4 o0, o1;
      o0.x = pack2(v[0], v[1]); o0.y = pack2(v[2], v[3]); o0.z = pack2(v[4], v[5]); o0.w = pack2(v[6], v[7]);
      o1.x = pack2(v[8], v[9]); o1.y = pack2(v[10], v[11]); o1.z = pack2(v[12], v[13]); o1.w = pack2(v[14], v[15]);
      uint4* yo = reinterpret_cast<uint4*>(y) + t * 2;
      yo[0] = o0;
      yo[1] = o1;
    }
    return;
  }
  if (layout == 4) {
    // 3x3/s1/p1 stem on a 3-channel image (VGG), im2col in the pack: pixel (y, x) holds the
    // 27 taps (r, s, c) of its 3x3 window (zeros outside the image) padded to 64 channels, so
    // the stem is a 1x1 conv over plain NHWC rows.  One thread per pixel gathers its 27 taps
    // (loads coalesced across the block's consecutive pixels) into shared memory; the block
    // then writes its 256 x 128 B output span with consecutive 16-byte stores.
    __shared__ uint4 tap_s[256][4];
    const long long total = (long long)N * HW;
    for (long long base = (long long)blockIdx.x * blockDim.x; base < total; base += (long long)gridDim.x * blockDim.x) {
      const long long pix = base + threadIdx.x;
      if (pix < total) {
        const long long n = pix / HW;
        const int rem = (int)(pix - n * HW), yy = rem / W, xx = rem - (rem / W) * W;
        float v[28];
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          const int iy = yy + r - 1;
#pragma unroll
          for (int s_ = 0; s_ < 3; ++s_) {
            const int ix = xx + s_ - 1;
            const bool in = iy >= 0 && iy < H && ix >= 0 && ix < W;
            const T* src = img + n * 3 * HW + (long long)iy * W + ix;
#pragma unroll
            for (int c = 0; c < 3; ++c) v[(r * 3 + s_) * 3 + c] = in ? in_val(src + c * HW, nrm, c) : 0.f;
          }
        }
        v[27] = 0.f;
#pragma unroll
        for (int q = 0; q < 3; ++q)
          tap_s[threadIdx.x][q] = make_uint4(pack2(v[q * 8 + 0], v[q * 8 + 1]), pack2(v[q * 8 + 2], v[q * 8 + 3]),
                                             pack2(v[q * 8 + 4], v[q * 8 + 5]), pack2(v[q * 8 + 6], v[q * 8 + 7]));
        tap_s[threadIdx.x][3] = make_uint4(pack2(v[24], v[25]), pack2(v[26], v[27]), 0u, 0u);
      }
      __syncthreads();
      const long long npix = total - base < (long long)blockDim.x ? total - base : (long long)blockDim.x;
      uint4* yo = reinterpret_cast<uint4*>(y) + base * 8;
      for (int t = threadIdx.x; t < npix * 8; t += blockDim.x) {
        const int p = t >> 3, part = t & 7;
        yo[t] = part < 4 ? tap_s[p][part] : make_uint4(0u, 0u, 0u, 0u);
      }
      __syncthreads();
    }
    return;
  }
  if (layout == 3) {
    // 3x3/s1/p1 stem on a 3-channel image (VGG): NHWC padded to 8 channels with a zero border
    // (one row above and below, one column left, wp - W - 1 right), so the stem reads each
    // filter row as one 8-pixel x 8-channel window (64 contiguous bf16) starting at padded
    // column ow: one thread per padded pixel of the (H+2) x wp grid
    const int HP = H + 2, WP = wp;
    const long long total = (long long)N * HP * WP;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
      const long long n = t / (HP * WP);
      const int rem = (int)(t - n * HP * WP);
      const int i = rem / WP - 1, j = rem - (rem / WP) * WP - 1;
      float v[3] = {0.f, 0.f, 0.f};
      if (i >= 0 && i < H && j >= 0 && j < W) {
        const T* src = img + n * 3 * HW + (long long)i * W + j;
#pragma unroll
        for (int c = 0; c < 3; ++c) v[c] = in_val(src + c * HW, nrm, c);
      }
      uint4 o;
      o.x = pack2(v[0], v[1]); o.y = pack2(v[2], 0.f); o.z = 0u; o.w = 0u;
      reinterpret_cast<uint4*>(y)[t] = o;
    }
    return;
  }
  const long long total = (long long)N * HW;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long n = i / HW;
    const long long p = i - n * HW;
    const T* src = img + n * 3 * HW + p;
    const float r = in_val(src, nrm, 0), g = in_val(src + HW, nrm, 1), b = in_val(src + 2 * HW, nrm, 2);
    if (layout == 1) {
      uint4 o;
      o.x = pack2(r, g);
      o.y = pack2(b, 0.f);
      o.z = 0u;
      o.w = 0u;
      reinterpret_cast<uint4*>(y)[i] = o;
    } else {
      float* yo = static_cast<float*>(y) + i * 3;
      yo[0] = r; yo[1] = g; yo[2] = b;
    }
  }
}

// ---------------------------------------------------------------- pooling
template <typename T, int V>
__global__ void pool_kernel(const PoolArgs a) {
  griddep_launch_dependents();
  griddep_wait();
  const int cg = a.C / V;
  const long long total = (long long)a.N * a.OH * a.OW * cg;
  const T* x = static_cast<const T*>(a.x);
  T* y = static_cast<T*>(a.y);
  const float inv = 1.f / (float)(a.k * a.k);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(i % cg) * V;
    const long long pix = i / cg;
    const int ow = (int)(pix % a.OW);
    const int oh = (int)((pix / a.OW) % a.OH);
    const long long n = pix / ((long long)a.OW * a.OH);
    float acc[V];
#pragma unroll
    for (int j = 0; j < V; ++j) acc[j] = a.mode == 0 ? -INFINITY : 0.f;
    for (int r = 0; r < a.k; ++r) {
      const int ih = oh * a.stride - a.pad + r;
      if ((unsigned)ih >= (unsigned)a.H) continue;
      for (int s = 0; s < a.k; ++s) {
        const int iw = ow * a.stride - a.pad + s;
        if ((unsigned)iw >= (unsigned)a.W) continue;
        float f[V];
        load_vec<T, V>(x + ((n * a.H + ih) * a.W + iw) * a.x_ld + c, f);
        if (a.pro_scale) {
#pragma unroll
          for (int j = 0; j < V; ++j) f[j] = fmaxf(fmaf(f[j], __ldg(a.pro_scale + c + j), __ldg(a.pro_shift + c + j)), 0.f);
        }
#pragma unroll
        for (int j = 0; j < V; ++j) acc[j] = a.mode == 0 ? fmaxf(acc[j], f[j]) : acc[j] + f[j];
      }
    }
    if (a.mode == 1) {
#pragma unroll
      for (int j = 0; j < V; ++j) acc[j] *= inv;
    }
    store_vec<T, V>(y + pix * a.y_ld + c, acc);
  }
}

// 2x2/s2/p0 pooling on bf16 NHWC (VGG maxpools, DenseNet transition avgpools): every window is
// in bounds, so one thread reads its four 16-byte channel vectors with no bounds tests and 32-bit
// index arithmetic.  Same operations in the same order as pool_kernel (bitwise identical).
template <int MODE>
__global__ void __launch_bounds__(256) pool2x2_bf16_kernel(const PoolArgs a) {
  griddep_launch_dependents();
  griddep_wait();
  const unsigned cg = (unsigned)a.C / 8u;
  const unsigned total = (unsigned)a.N * a.OH * a.OW * cg;
  const __nv_bfloat16* x = static_cast<const __nv_bfloat16*>(a.x);
  __nv_bfloat16* y = static_cast<__nv_bfloat16*>(a.y);
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const unsigned pix = i / cg;
    const unsigned c = (i - pix * cg) * 8u;
    const unsigned row = pix / (unsigned)a.OW;  // n * OH + oh
    const unsigned ow = pix - row * (unsigned)a.OW;
    const unsigned n = row / (unsigned)a.OH;
    const unsigned oh = row - n * (unsigned)a.OH;
    const __nv_bfloat16* p0 = x + ((size_t)(n * a.H + 2u * oh) * a.W + 2u * ow) * a.x_ld + c;
    const __nv_bfloat16* p1 = p0 + (size_t)a.W * a.x_ld;
    float f[4][8];
    load_vec<__nv_bfloat16, 8>(p0, f[0]);
    load_vec<__nv_bfloat16, 8>(p0 + a.x_ld, f[1]);
    load_vec<__nv_bfloat16, 8>(p1, f[2]);
    load_vec<__nv_bfloat16, 8>(p1 + a.x_ld, f[3]);
    if (a.pro_scale) {  // bn-relu prologue (commuted DenseNet transition)
      float sc[8], sh[8];
      load_vec<float, 4>(a.pro_scale + c, *reinterpret_cast<float(*)[4]>(sc));
      load_vec<float, 4>(a.pro_scale + c + 4, *reinterpret_cast<float(*)[4]>(sc + 4));
      load_vec<float, 4>(a.pro_shift + c, *reinterpret_cast<float(*)[4]>(sh));
      load_vec<float, 4>(a.pro_shift + c + 4, *reinterpret_cast<float(*)[4]>(sh + 4));
#pragma unroll
      for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int j = 0; j < 8; ++j) f[t][j] = fmaxf(fmaf(f[t][j], sc[j], sh[j]), 0.f);
    }
    float acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float v = MODE == 0 ? -INFINITY : 0.f;
#pragma unroll
      for (int t = 0; t < 4; ++t) v = MODE == 0 ? fmaxf(v, f[t][j]) : v + f[t][j];
      acc[j] = MODE == 0 ? v : v * 0.25f;
    }
    store_vec<__nv_bfloat16, 8>(y + (size_t)pix * a.y_ld + c, acc);
  }
}

template <typename T, int V>
__global__ void adaptive_kernel(const AdaptiveArgs a) {
  griddep_launch_dependents();
  griddep_wait();
  const int cg = a.C / V;
  const long long total = (long long)a.N * a.OH * a.OW * cg;
  const T* x = static_cast<const T*>(a.x);
  T* y = static_cast<T*>(a.y);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(i % cg) * V;
    const long long pix = i / cg;
    const int ow = (int)(pix % a.OW);
    const int oh = (int)((pix / a.OW) % a.OH);
    const long long n = pix / ((long long)a.OW * a.OH);
    // PyTorch bins: [floor(i*H/o), ceil((i+1)*H/o))
    const int h0 = (oh * a.H) / a.OH, h1 = ((oh + 1) * a.H + a.OH - 1) / a.OH;
    const int w0 = (ow * a.W) / a.OW, w1 = ((ow + 1) * a.W + a.OW - 1) / a.OW;
    float acc[V];
#pragma unroll
    for (int j = 0; j < V; ++j) acc[j] = 0.f;
    for (int ih = h0; ih < h1; ++ih)
      for (int iw = w0; iw < w1; ++iw) {
        float f[V];
        load_vec<T, V>(x + ((n * a.H + ih) * a.W + iw) * a.x_ld + c, f);
#pragma unroll
        for (int j = 0; j < V; ++j) acc[j] += a.relu_in ? fmaxf(f[j], 0.f) : f[j];
      }
    const float inv = 1.f / (float)((h1 - h0) * (w1 - w0));
#pragma unroll
    for (int j = 0; j < V; ++j) acc[j] *= inv;
    store_vec<T, V>(y + pix * a.y_ld + c, acc);
  }
}

template <typename T, int V>
__global__ void bn_act_kernel(const EltArgs a) {
  griddep_launch_dependents();
  griddep_wait();
  const int cg = a.C / V;
  const long long total = (long long)a.N * a.HW * cg;
  const T* x = static_cast<const T*>(a.x);
  T* y = static_cast<T*>(a.y);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(i % cg) * V;
    const long long pix = i / cg;
    float f[V];
    load_vec<T, V>(x + pix * a.x_ld + c, f);
#pragma unroll
    for (int j = 0; j < V; ++j) {
      float v = f[j];
      if (a.scale) v = fmaf(v, __ldg(a.scale + c + j), __ldg(a.shift + c + j));
      if (a.relu) v = fmaxf(v, 0.f);
      f[j] = v;
    }
    store_vec<T, V>(y + pix * a.y_ld + c, f);
  }
}

// NHWC (ld) -> NCHW through a 32x32 shared-memory tile: coalesced on both sides.
template <typename T>
__global__ void pack_output_kernel(const T* __restrict__ x, int HW, int C, int x_ld, T* __restrict__ y) {
  griddep_launch_dependents();
  griddep_wait();
  __shared__ T tile[32][33];
  const int p0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
  const long long n = blockIdx.z;
  const int tx = threadIdx.x, ty = threadIdx.y;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int p = p0 + ty + 8 * i, c = c0 + tx;
    if (p < HW && c < C) tile[ty + 8 * i][tx] = x[(n * HW + p) * x_ld + c];
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int c = c0 + ty + 8 * i, p = p0 + tx;
    if (p < HW && c < C) y[(n * C + c) * HW + p] = tile[tx][ty + 8 * i];
  }
}

// NCHW [N][C][HW] -> NHWC [N*HW][y_ld] (the suffix path's input: the split-layer send
// buffer of the storage side becomes the client's first activation)
template <typename T>
__global__ void unpack_nchw_kernel(const T* __restrict__ x, int HW, int C, T* __restrict__ y, int y_ld) {
  griddep_launch_dependents();
  griddep_wait();
  __shared__ T tile[32][33];
  const int c0 = blockIdx.x * 32, p0 = blockIdx.y * 32;
  const long long n = blockIdx.z;
  const int tx = threadIdx.x, ty = threadIdx.y;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int c = c0 + ty + 8 * i, p = p0 + tx;
    if (p < HW && c < C) tile[ty + 8 * i][tx] = x[(n * C + c) * HW + p];
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int p = p0 + ty + 8 * i, c = c0 + tx;
    if (p < HW && c < C) y[(n * HW + p) * y_ld + c] = tile[tx][ty + 8 * i];
  }
}

// bf16 NHWC -> NCHW with 16-byte accesses on both sides: a 64-pixel x 64-channel tile is read
// as 8-channel vectors along C and written as 8-pixel vectors along HW (HW % 8 == 0, C % 8 == 0)
__global__ void __launch_bounds__(256) pack_output_v8_kernel(const __nv_bfloat16* __restrict__ x, int HW, int C,
                                                             int x_ld, __nv_bfloat16* __restrict__ y) {
  griddep_launch_dependents();
  griddep_wait();
  // [channel][pixel]; the 16-byte pixel chunk of row r is stored at chunk ^ (r >> 3) so the
  // transposing scalar stores of a warp (8 channel rows 8 apart) hit 8 different bank groups
  // (a padded 72-element row maps rows 8 apart to the same bank: 8-way conflicts, 3.2 TB/s).
  __shared__ __align__(16) __nv_bfloat16 tile[64][64];
  const int p0 = blockIdx.x * 64, c0 = blockIdx.y * 64;
  const long long n = blockIdx.z;
  const int t = threadIdx.x;
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int idx = t + k * 256;              // 64 pixels x 8 channel-chunks
    const int pp = idx >> 3, cc = (idx & 7) * 8;
    const int p = p0 + pp, c = c0 + cc;
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (p < HW && c < C) v = __ldg(reinterpret_cast<const uint4*>(x + (n * HW + p) * x_ld + c));
    const __nv_bfloat16* e = reinterpret_cast<const __nv_bfloat16*>(&v);
#pragma unroll
    for (int j = 0; j < 8; ++j) tile[cc + j][(((pp >> 3) ^ ((cc + j) >> 3)) << 3) | (pp & 7)] = e[j];
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int idx = t + k * 256;              // 64 channels x 8 pixel-chunks
    const int cc = idx >> 3, pp = (idx & 7) * 8;
    const int c = c0 + cc, p = p0 + pp;
    if (c < C && p < HW)
      *reinterpret_cast<uint4*>(y + (n * C + c) * HW + p) =
          *reinterpret_cast<const uint4*>(&tile[cc][((pp >> 3) ^ (cc >> 3)) << 3]);
  }
}

inline int grid_for(long long total, int block) {
  long long g = (total + block - 1) / block;
  if (g > 148 * 32) g = 148 * 32;
  return (int)(g > 0 ? g : 1);
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace

cudaError_t unpack_nchw_launch(const void* x, int N, int C, int HW, void* y, int y_ld, int es, cudaStream_t st) {
  if (N <= 0 || C <= 0 || HW <= 0) return cudaSuccess;
  dim3 grid((C + 31) / 32, (HW + 31) / 32, N), block(32, 8);
  if (es == 2)
    launch_pdl(unpack_nchw_kernel<__nv_bfloat16>, grid, block, 0, st, static_cast<const __nv_bfloat16*>(x), HW, C,
               static_cast<__nv_bfloat16*>(y), y_ld);
  else
    launch_pdl(unpack_nchw_kernel<float>, grid, block, 0, st, static_cast<const float*>(x), HW, C,
               static_cast<float*>(y), y_ld);
  return cudaGetLastError();
}

cudaError_t pack_input_launch(const void* img, const InNorm* nrm, void* y, int N, int H, int W, int layout, int wp,
                              cudaStream_t st) {
  const long long total = layout == 2 ? (long long)N * (H / 2 + 3) * wp
                          : layout == 3 ? (long long)N * (H + 2) * wp
                          : (long long)N * H * W;
  const dim3 grid(grid_for(total, 256)), block(256);
  if (nrm)
    launch_pdl(pack_input_kernel<uint8_t>, grid, block, 0, st, static_cast<const uint8_t*>(img), y, N, H, W, layout, wp,
               *nrm);
  else
    launch_pdl(pack_input_kernel<float>, grid, block, 0, st, static_cast<const float*>(img), y, N, H, W, layout, wp,
               InNorm{});
  return cudaGetLastError();
}

// HAPI_POOL_GENERIC=1: every pool through pool_kernel (A/B of the 2x2 specialisation).
static bool pool_generic() {
  static const bool on = [] {
    const char* e = std::getenv("HAPI_POOL_GENERIC");
    return e && e[0] == '1';
  }();
  return on;
}

cudaError_t pool_launch(const PoolArgs& a, int is_bf16, cudaStream_t st) {
  const long long pix = (long long)a.N * a.OH * a.OW;
  if (is_bf16) {
    const bool vec8 = a.C % 8 == 0 && a.x_ld % 8 == 0 && a.y_ld % 8 == 0 && aligned16(a.x) && aligned16(a.y);
    if (vec8 && a.k == 2 && a.stride == 2 && a.pad == 0 && a.OH * 2 <= a.H && a.OW * 2 <= a.W &&
        pix * (a.C / 8) < (1ll << 31) && !pool_generic()) {
      if (a.mode == 0)
        launch_pdl(pool2x2_bf16_kernel<0>, dim3(grid_for(pix * (a.C / 8), 256)), dim3(256), 0, st, a);
      else
        launch_pdl(pool2x2_bf16_kernel<1>, dim3(grid_for(pix * (a.C / 8), 256)), dim3(256), 0, st, a);
    } else if (vec8)
      launch_pdl(pool_kernel<__nv_bfloat16, 8>, dim3(grid_for(pix * (a.C / 8), 256)), dim3(256), 0, st, a);
    else
      launch_pdl(pool_kernel<__nv_bfloat16, 1>, dim3(grid_for(pix * a.C, 256)), dim3(256), 0, st, a);
  } else {
    if (a.C % 4 == 0 && a.x_ld % 4 == 0 && a.y_ld % 4 == 0 && aligned16(a.x) && aligned16(a.y))
      launch_pdl(pool_kernel<float, 4>, dim3(grid_for(pix * (a.C / 4), 256)), dim3(256), 0, st, a);
    else
      launch_pdl(pool_kernel<float, 1>, dim3(grid_for(pix * a.C, 256)), dim3(256), 0, st, a);
  }
  return cudaGetLastError();
}

cudaError_t adaptive_avgpool_launch(const AdaptiveArgs& a, int is_bf16, cudaStream_t st) {
  const long long pix = (long long)a.N * a.OH * a.OW;
  if (is_bf16) {
    if (a.C % 8 == 0 && a.x_ld % 8 == 0 && a.y_ld % 8 == 0 && aligned16(a.x) && aligned16(a.y))
      launch_pdl(adaptive_kernel<__nv_bfloat16, 8>, dim3(grid_for(pix * (a.C / 8), 256)), dim3(256), 0, st, a);
    else
      launch_pdl(adaptive_kernel<__nv_bfloat16, 1>, dim3(grid_for(pix * a.C, 256)), dim3(256), 0, st, a);
  } else {
    if (a.C % 4 == 0 && a.x_ld % 4 == 0 && a.y_ld % 4 == 0 && aligned16(a.x) && aligned16(a.y))
      launch_pdl(adaptive_kernel<float, 4>, dim3(grid_for(pix * (a.C / 4), 256)), dim3(256), 0, st, a);
    else
      launch_pdl(adaptive_kernel<float, 1>, dim3(grid_for(pix * a.C, 256)), dim3(256), 0, st, a);
  }
  return cudaGetLastError();
}

cudaError_t bn_act_launch(const EltArgs& a, int is_bf16, cudaStream_t st) {
  const long long pix = (long long)a.N * a.HW;
  if (is_bf16) {
    if (a.C % 8 == 0 && a.x_ld % 8 == 0 && a.y_ld % 8 == 0 && aligned16(a.x) && aligned16(a.y))
      launch_pdl(bn_act_kernel<__nv_bfloat16, 8>, dim3(grid_for(pix * (a.C / 8), 256)), dim3(256), 0, st, a);
    else
      launch_pdl(bn_act_kernel<__nv_bfloat16, 1>, dim3(grid_for(pix * a.C, 256)), dim3(256), 0, st, a);
  } else {
    if (a.C % 4 == 0 && a.x_ld % 4 == 0 && a.y_ld % 4 == 0 && aligned16(a.x) && aligned16(a.y))
      launch_pdl(bn_act_kernel<float, 4>, dim3(grid_for(pix * (a.C / 4), 256)), dim3(256), 0, st, a);
    else
      launch_pdl(bn_act_kernel<float, 1>, dim3(grid_for(pix * a.C, 256)), dim3(256), 0, st, a);
  }
  return cudaGetLastError();
}

// Small maps whose HW is not a multiple of 8 (7x7 splits: VGG s=21, ResNet s=20): one block per
// (image, 64-channel group).  The group's output is one contiguous span of 64 * HW elements, so
// the block gathers its HW x 64 input with 16-byte loads, transposes into a shared copy of that
// span, and writes it back with 16-byte stores.
__global__ void __launch_bounds__(256) pack_output_span_kernel(const __nv_bfloat16* __restrict__ x, int HW, int C,
                                                               int x_ld, __nv_bfloat16* __restrict__ y) {
  griddep_launch_dependents();
  griddep_wait();
  extern __shared__ __align__(16) unsigned char span_raw[];
  __nv_bfloat16* span = reinterpret_cast<__nv_bfloat16*>(span_raw);  // [64][HW]
  const int c0 = blockIdx.x * 64;
  const long long n = blockIdx.y;
  for (int idx = threadIdx.x; idx < HW * 8; idx += blockDim.x) {
    const int p = idx >> 3, cc = (idx & 7) * 8;
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(x + (n * HW + p) * x_ld + c0 + cc));
    const __nv_bfloat16* e = reinterpret_cast<const __nv_bfloat16*>(&v);
#pragma unroll
    for (int j = 0; j < 8; ++j) span[(cc + j) * HW + p] = e[j];
  }
  __syncthreads();
  uint4* dst = reinterpret_cast<uint4*>(y + (n * C + c0) * HW);
  const uint4* src = reinterpret_cast<const uint4*>(span);
  for (int i = threadIdx.x; i < HW * 8; i += blockDim.x) dst[i] = src[i];  // 64 * HW / 8 vectors
}

cudaError_t pack_output_launch(const void* x, int N, int HW, int C, int x_ld, void* y, int is_bf16, cudaStream_t st) {
  const size_t es = is_bf16 ? 2 : 4;
  if (HW == 1) {  // NHWC == NCHW: a strided row copy
    return cudaMemcpy2DAsync(y, C * es, x, (size_t)x_ld * es, C * es, N, cudaMemcpyDeviceToDevice, st);
  }
  if (is_bf16 && HW % 8 == 0 && C % 8 == 0 && x_ld % 8 == 0 && aligned16(x) && aligned16(y)) {
    launch_pdl(pack_output_v8_kernel, dim3((HW + 63) / 64, (C + 63) / 64, N), dim3(256), 0, st,
               static_cast<const __nv_bfloat16*>(x), HW, C, x_ld, static_cast<__nv_bfloat16*>(y));
    return cudaGetLastError();
  }
  if (is_bf16 && C % 64 == 0 && HW <= 256 && x_ld % 8 == 0 && aligned16(x) && aligned16(y) && N <= 65535) {
    launch_pdl(pack_output_span_kernel, dim3(C / 64, N), dim3(256), (size_t)64 * HW * 2, st,
               static_cast<const __nv_bfloat16*>(x), HW, C, x_ld, static_cast<__nv_bfloat16*>(y));
    return cudaGetLastError();
  }
  dim3 grid((HW + 31) / 32, (C + 31) / 32, N), block(32, 8);
  if (is_bf16)
    launch_pdl(pack_output_kernel<__nv_bfloat16>, dim3(grid), dim3(block), 0, st, static_cast<const __nv_bfloat16*>(x), HW, C, x_ld,
                                                             static_cast<__nv_bfloat16*>(y));
  else
    launch_pdl(pack_output_kernel<float>, dim3(grid), dim3(block), 0, st, static_cast<const float*>(x), HW, C, x_ld, static_cast<float*>(y));
  return cudaGetLastError();
}

}  // namespace hapi
