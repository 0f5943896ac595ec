// Executor half of the C ABI: model creation (BN folding, weight packing, TMA
// descriptors), split-aware launch plans (fusion never crosses the split boundary,
// SURVEY.md 7.2 H3), the liveness-planned activation arena, and the launch loop of
// hapi_prefix_forward ("executes the feature extraction part up to the split index",
// PAPER.md:732; COS batch decoupled from the request, PAPER.md:732/740/750 -> chunking).
#include <cuda.h>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "arch.h"
#include "common.h"
#include "kernels.h"

using namespace hapi;

namespace hapi {

namespace {
thread_local std::string g_err;
}

hapi_status set_error(hapi_status st, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}
void clear_error() { g_err.clear(); }
const char* last_error_cstr() { return g_err.c_str(); }

}  // namespace hapi

namespace {

constexpr double BN_EPS = 1e-5;

// ---------------------------------------------------------------- TMA encode (driver entry point)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

typedef CUresult (*EncodeIm2colFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t, const cuuint32_t*,
                                   CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                   CUtensorMapFloatOOBfill);

EncodeIm2colFn get_im2col_fn() {
  static EncodeIm2colFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeIm2colFn>(p);
  }
  return fn;
}

bool im2col_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("HAPI_IM2COL");
    return !(e && e[0] == '0');
  }();
  return on;
}

EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

bool prologue_tma_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("HAPI_PRO_TMA");
    return !(e && e[0] == '0');
  }();
  return on;
}

bool stem_pool_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("HAPI_STEM_POOL");
    return !(e && e[0] == '0');
  }();
  return on;
}

bool block_enabled() {  // whole identity bottlenecks on a CTA pair (conv_block.cu); HAPI_BLOCK=0: off
  static const bool on = [] {
    const char* e = std::getenv("HAPI_BLOCK");
    return !(e && e[0] == '0');
  }();
  return on;
}

bool block_ds_enabled() {  // HAPI_BLOCK_DS=0: the downsample block (ResNet layer1.0) stays unfused
  static const bool on = [] {
    const char* e = std::getenv("HAPI_BLOCK_DS");
    return !(e && e[0] == '0');
  }();
  return on;
}

bool pair_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("HAPI_PAIR");
    return !(e && e[0] == '0');
  }();
  return on;
}

bool stem_col_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("HAPI_STEM_COL");
    return !(e && e[0] == '0');
  }();
  return on;
}

bool win3_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("HAPI_WIN3");
    return !(e && e[0] == '0');
  }();
  return on;
}

bool sub_store_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("HAPI_SUB_STORE");
    return !(e && e[0] == '0');
  }();
  return on;
}

bool res_identity_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("HAPI_RES_GEMM");
    return !(e && e[0] == '0');
  }();
  return on;
}

bool halo_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("HAPI_HALO");
    return !(e && e[0] == '0');
  }();
  return on;
}

bool commute_enabled() {  // HAPI_COMMUTE=0: DenseNet transitions as bn-relu-conv, then avgpool
  static const bool on = [] {
    const char* e = std::getenv("HAPI_COMMUTE");
    return !(e && e[0] == '0');
  }();
  return on;
}

bool fused_ds_disabled() {
  static const bool off = [] {
    const char* e = std::getenv("HAPI_FUSE_DS");
    return e && e[0] == '0';
  }();
  return off;
}

// ---------------------------------------------------------------- model structures
struct ConvW {
  int cs = 0;        // channels per pixel consumed (stored)
  int cout = 0, kh = 1, kw = 1, stride = 1, pad = 0;
  int K = 0, Kp = 0;
  void* w = nullptr;           // bf16 [Cout][Kp] (tc) or fp32 [K][Cout] (simt)
  void* w8 = nullptr;          // s2d stem, mode 8: bf16 [chunk 20][k half 2][n 128][8] (no-swizzle K-major)
  float* bias = nullptr;       // [Cout]
  std::vector<float> hbias;    // host copy of bias (the block kernel takes it by value)
  float* pro_scale = nullptr;  // [cs]
  float* pro_shift = nullptr;
  CUtensorMap tmap;
  CUtensorMap tmap_half;         // {64, bn/2} box: each CTA of a 2-CTA cluster loads one half
  bool has_half = false;
  int bn = 0, mode = 0;
  double real_flops_per_px = 0;  // 2 * K_real * Cout
  int K2 = 0, cs2 = 0, stride2 = 1;  // fused downsample source (bf16): 1x1/stride2 over cs2 channels
  bool res_identity = false;         // K2 columns are an identity block: + residual inside the GEMM
};

enum OpType { OP_PACK_IN, OP_CONV, OP_POOL, OP_ADAPTIVE, OP_BNACT, OP_PACK_OUT, OP_PAIR, OP_UNPACK, OP_BLOCK };

struct View {
  int buf = -1;       // -1: external (caller out, or caller images for PACK_IN input)
  int C = 0, H = 0, W = 0, ld = 0, coff = 0;
};

struct Op {
  OpType t;
  View in, out, res;
  bool has_res = false, relu = false, nchw_out = false, relu_in = false;
  int conv = -1;
  int pk = 0, ps = 0, pp = 0, pmode = 0;
  const float* scale = nullptr;  // bn_act (device)
  const float* shift = nullptr;
  uint32_t kind = 0;             // plan_info kernel class
  double flops = 0, bytes = 0;   // per image
  std::string desc;              // human-readable (hapi_plan_describe)
  int tc_mode = 0;               // conv_tc A-operand mode
  int wb = 0, hb = 0, nb = 0;    // mode 4 spatial tile
  int layout = 0;                // pack_in layout
  bool s2d_view = false;         // stem over the padded space-to-depth window view
  int conv_oh = 0, conv_ow = 0;  // mode 8: stem map size (out is the pooled map)
  CUtensorMap tmap_a;            // modes 3/4 (built after the arena is placed)
  CUtensorMap tmap_y;            // NHWC output view (TMA-store epilogue)
  CUtensorMap tmap_r;            // residual view
  CUtensorMap tmap_yw;           // NHWC output view with a {32, 32} box (per-warp epilogue stores)
  bool has_yw = false;
  bool dual = false;             // second A source (fused downsample) = in2
  View in2;
  CUtensorMap tmap_a2;
  // OP_PAIR (conv_pair.cu): conv = the bottleneck's conv3, conv2 = the next block's conv1,
  // out = block output, out2 = next conv1 output
  int conv2 = -1;
  View out2;
  CUtensorMap tmap_b1;           // conv3 weights with a {64, 128} box
  CUtensorMap tmap_y2;
  int ksplit = 1;                // fp32 SIMT split-K slices (partial sums in `ws`)
  View ws;
  // OP_PAIR whose block output is read only by a later 1x1/stride-2 downsample: `out` holds
  // just the even (row, col) pixels of the full_h x full_w map, the consumer reads it with
  // in2_stride = 1
  bool sub_out = false;
  int full_h = 0, full_w = 0;
  bool pool2 = false;            // mode-4 conv with the following 2x2/s2 maxpool in its epilogue (out = pooled)
  // OP_BLOCK (conv_block.cu): conv = conv1, conv2 = conv2, conv3 = conv3 of an identity
  // bottleneck; in = x, out = block output; maps over x and the three weight tensors
  int conv3 = -1;
  int conv4 = -1;                // OP_BLOCK with a downsample: its 1x1 conv (else -1)
  CUtensorMap bmap_x, bmap_w1, bmap_w2, bmap_w3, bmap_wds;
  int in2_stride = 0;            // 0: the conv's own stride2
};

struct Buf {
  int64_t per_img = 0;  // bytes per image
  int first = -1, last = -1;
  int64_t offset = 0;   // per-image-scaled offset is not used; absolute offset for max_batch
};

struct Plan {
  int split = 0;
  std::vector<Op> ops;
  std::vector<Buf> bufs;
  int64_t arena_bytes = 0;
  int64_t out_bytes_per_img = 0;
};

}  // namespace

// Device weights (packed convs, bias/BN vectors, the identity block) of a model, shared by
// the models made from it with hapi_model_create_shared; freed with the last of them.
struct WeightStore {
  int device = 0;
  std::vector<void*> ptrs;
  ~WeightStore() {
    int prev = -1;
    cudaGetDevice(&prev);
    if (prev != device) cudaSetDevice(device);
    for (void* p : ptrs) cudaFree(p);
    if (prev >= 0 && prev != device) cudaSetDevice(prev);
  }
};

struct hapi_model {
  hapi_model_desc d;
  std::shared_ptr<WeightStore> wstore;  // owned (or shared) weight allocations
  const ArchDesc* arch = nullptr;
  bool bf16 = true;
  int es = 2;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  std::vector<ConvW> convs;
  std::map<std::string, int> conv_index;
  std::map<std::string, std::pair<float*, float*>> bn_cache;  // unfused BN: device scale/shift
  std::vector<const float*> host_params;  // valid during create only
  std::vector<void*> allocs;
  int64_t weight_bytes = 0;
  uint32_t start = 0;                          // suffix models: input = layer `start` output
  int64_t in_bytes_per_img = 0;                // suffix models: bytes of one input activation
  void* ident = nullptr;                       // shared 64x64 bf16 identity block (residual in GEMM)
  CUtensorMap ident_map128, ident_map256;      // box {64, 128} / {64, 256}
  std::vector<Plan> plans;  // index split - min_split
  void* arena = nullptr;
  int64_t arena_bytes = 0;
  // host pipeline (desc.host_chunk > 0): streams, events and staging made at create time
  int64_t stage_bytes = 0;              // device bytes of the four staging buffers
  uint32_t host_chunk = 0;              // images per staging slot
  cudaStream_t copy_stream = nullptr;   // host path: H2D copies
  cudaStream_t out_stream = nullptr;    // host path: D2H copies (separate, so the next H2D never
                                        // queues behind a D2H that waits for compute)
  void* stage_in[2] = {nullptr, nullptr};
  void* stage_out[2] = {nullptr, nullptr};
  int64_t stage_out_bytes = 0;
  cudaEvent_t ev[8] = {};
  bool host_ready = false;
  uint64_t host_seq = 0;                // host-path chunks enqueued so far (slot parity, reuse waits)
  // CUDA graphs of one chunk's launch sequence, keyed by (split, batch, images, out)
  struct GraphEntry {
    uint32_t split;
    int nb;
    bool u8;
    const void* images;
    void* out;
    cudaGraphExec_t exec;
  };
  std::vector<GraphEntry> graphs;
  cudaStream_t cap_stream = nullptr;
  // u8 ingest (hapi_prefix_forward_u8 & co.): x = scale[c] * u + shift[c]
  InNorm u8norm = {{1.f / 255.f, 1.f / 255.f, 1.f / 255.f}, {0.f, 0.f, 0.f}};
};

namespace {

// ---------------------------------------------------------------- helpers
// Every entry point runs on the model's device and leaves the caller's current device as
// it found it (a process may hold models on several GPUs).
struct DeviceGuard {
  int prev = -1;
  bool switched = false;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) == cudaSuccess && prev != dev) switched = cudaSetDevice(dev) == cudaSuccess;
  }
  ~DeviceGuard() {
    if (switched) cudaSetDevice(prev);
  }
};

hapi_status dev_alloc(hapi_model* m, size_t bytes, void** p, bool weights) {
  if (bytes == 0) bytes = 16;
  cudaError_t e = cudaMalloc(p, bytes);
  if (e != cudaSuccess)
    return set_error(e == cudaErrorMemoryAllocation ? HAPI_ERR_OUT_OF_MEMORY : HAPI_ERR_CUDA, "cudaMalloc(%zu): %s", bytes,
                     cudaGetErrorString(e));
  if (weights) {
    m->wstore->ptrs.push_back(*p);
    m->weight_bytes += (int64_t)bytes;
  } else {
    m->allocs.push_back(*p);
  }
  return HAPI_OK;
}

template <typename T>
hapi_status upload(hapi_model* m, const std::vector<T>& h, T** dptr) {
  void* p;
  hapi_status st = dev_alloc(m, h.size() * sizeof(T), &p, true);
  if (st != HAPI_OK) return st;
  cudaError_t e = cudaMemcpy(p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return set_error(HAPI_ERR_CUDA, "cudaMemcpy: %s", cudaGetErrorString(e));
  *dptr = static_cast<T*>(p);
  return HAPI_OK;
}

uint16_t f2bf(float f) {  // round-to-nearest-even
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7f800000u) == 0x7f800000u) return (uint16_t)(u >> 16) | ((u & 0xffff) ? 0x40 : 0);
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

const float* P(hapi_model* m, const std::string& name, int64_t expect_numel) {
  if (m->host_params.empty()) return nullptr;  // a shared-weight model finds every conv in the cache
  int i = m->arch->find_param(name);
  if (i < 0) return nullptr;
  if (m->arch->params[i].numel() != expect_numel) return nullptr;
  return m->host_params[i];
}

// BN eval as y = x*scale + shift (fp64)
bool bn_affine(hapi_model* m, const std::string& bn, int c, std::vector<double>& scale, std::vector<double>& shift) {
  const float* g = P(m, bn + ".weight", c);
  const float* b = P(m, bn + ".bias", c);
  const float* mu = P(m, bn + ".running_mean", c);
  const float* var = P(m, bn + ".running_var", c);
  if (!g || !b || !mu || !var) return false;
  scale.resize(c);
  shift.resize(c);
  for (int i = 0; i < c; ++i) {
    scale[i] = (double)g[i] / std::sqrt((double)var[i] + BN_EPS);
    shift[i] = (double)b[i] - (double)mu[i] * scale[i];
  }
  return true;
}

struct ConvSpec {
  std::string wname, bname, fold_bn, pro_bn;
  int cin = 0, cout = 0, k = 1, stride = 1, pad = 0;
  int cs = 0;            // stored channels per pixel of the input view (4 for the bf16 stem)
  int fh = 0, fw = 0;    // linear on a flattened (cin/(fh*fw), fh, fw) map: permute columns
  bool linear = false;
  bool s2d = false;      // 7x7/s2/p3 stem re-expressed as 4x4/s1/p2 on a 2x2 space-to-depth input
  bool col3 = false;     // 3x3/s1/p1 stem on 3 channels (VGG) over the im2col-packed input: a 1x1
                         // conv over 64 channels (k = (r*3+s)*3+c < 27)
  bool win3 = false;     // 3x3/s1/p1 stem on 3 channels (VGG) over the zero-bordered 8-channel input,
                         // each filter row one 8-pixel x 8-channel window: stored as KH=3, KW=8, C=8
  // fused downsample (bf16): out = conv(x1) + ds(x2) with ds a 1x1/stride2 conv + folded BN,
  // packed as extra K columns after the first conv's
  std::string w2name, fold2;
  int cin2 = 0, stride2 = 1;
  // identity residual as the second A source (bf16 1x1): K2 = cout identity columns, so
  // out = relu(conv(x) + bias + res) comes out of the accumulator (no epilogue residual read)
  bool res_identity = false;
};

hapi_status make_conv(hapi_model* m, const ConvSpec& s, int* out_idx) {
  std::string key = s.wname + "|" + s.bname + "|" + s.fold_bn + "|" + s.pro_bn + "|" + std::to_string(s.cs) + "|" +
                    std::to_string(s.fh) + "x" + std::to_string(s.fw) + (s.s2d ? "|s2d" : "") + (s.win3 ? "|win3" : "") + (s.col3 ? "|col3" : "") + "|" +
                    s.w2name + "|" +
                    s.fold2 + (s.res_identity ? "|resid" : "");
  auto it = m->conv_index.find(key);
  if (it != m->conv_index.end()) {
    *out_idx = it->second;
    return HAPI_OK;
  }
  const int kk = s.linear ? 1 : s.k;
  const int64_t wn = (int64_t)s.cout * s.cin * kk * kk;
  const float* w = P(m, s.wname, wn);
  if (!w) return set_error(HAPI_ERR_INVALID_MODEL, "param %s missing or wrong shape", s.wname.c_str());
  const float* b0 = nullptr;
  if (!s.bname.empty() && !(b0 = P(m, s.bname, s.cout)))
    return set_error(HAPI_ERR_INVALID_MODEL, "param %s missing", s.bname.c_str());
  std::vector<double> fs, fb;
  if (!s.fold_bn.empty() && !bn_affine(m, s.fold_bn, s.cout, fs, fb))
    return set_error(HAPI_ERR_INVALID_MODEL, "bn %s missing", s.fold_bn.c_str());
  const float* w2 = nullptr;
  std::vector<double> fs2, fb2;
  if (!s.w2name.empty()) {
    if (!m->bf16) return set_error(HAPI_ERR_UNSUPPORTED, "fused downsample is a bf16-path feature");
    if (!(w2 = P(m, s.w2name, (int64_t)s.cout * s.cin2)))
      return set_error(HAPI_ERR_INVALID_MODEL, "param %s missing or wrong shape", s.w2name.c_str());
    if (!bn_affine(m, s.fold2, s.cout, fs2, fb2)) return set_error(HAPI_ERR_INVALID_MODEL, "bn %s missing", s.fold2.c_str());
  }

  ConvW cw;
  cw.cs = s.cs;
  cw.cout = s.cout;
  cw.kh = cw.kw = s.s2d ? 4 : kk;
  if (s.win3) cw.kw = 8;
  if (s.col3) cw.kh = cw.kw = 1;
  cw.stride = s.s2d ? 1 : s.stride;
  cw.pad = s.s2d ? 2 : ((s.win3 || s.col3) ? 0 : s.pad);
  cw.K = cw.kh * cw.kw * s.cs;
  cw.real_flops_per_px = 2.0 * ((double)kk * kk * s.cin + s.cin2) * s.cout;
  cw.K2 = w2 ? s.cin2 : 0;
  cw.cs2 = s.cin2;
  cw.stride2 = s.stride2;
  if (s.res_identity) {
    // the residual joins as a second A source against the model's shared identity block (no
    // extra weight columns stored)
    if (!m->bf16 || w2) return set_error(HAPI_ERR_UNSUPPORTED, "identity residual source is a bf16, no-downsample feature");
    cw.cs2 = s.cout;
    cw.stride2 = 1;
    cw.res_identity = true;
  }
  // element (o, k) of the GEMM B operand, k ordered (r, s, c) over the stored input channels
  auto wval = [&](int o, int r, int t, int c) -> double {
    if (s.s2d) {
      // stored tap (r, t) of the 4x4 kernel, channel c = (a*2+b)*3 + ch of the 2x2 block:
      // original tap (2r+a-1, 2t+b-1) of the 7x7 kernel (zero outside it)
      if (c >= 12) return 0.0;
      const int blk = c / 3, ch = c % 3, aa = blk / 2, bb = blk % 2;
      const int orr = 2 * r + aa - 1, ott = 2 * t + bb - 1;
      if (orr < 0 || orr >= kk || ott < 0 || ott >= kk) return 0.0;
      double v = w[(((int64_t)o * s.cin + ch) * kk + orr) * kk + ott];
      if (!fs.empty()) v *= fs[o];
      return v;
    }
    if (s.col3) {
      // packed channel c = (r * 3 + t) * 3 + ch of the 1x1 conv
      if (c >= 27) return 0.0;
      const int rr = c / 9, tt = (c % 9) / 3, ch = c % 3;
      double v = w[(((int64_t)o * s.cin + ch) * kk + rr) * kk + tt];
      if (!fs.empty()) v *= fs[o];
      return v;
    }
    if (s.win3) {
      // window pixel t of filter row r: original tap (r, t) for t < 3, channel c < 3
      if (t >= kk || c >= s.cin) return 0.0;
      double v = w[(((int64_t)o * s.cin + c) * kk + r) * kk + t];
      if (!fs.empty()) v *= fs[o];
      return v;
    }
    if (c >= s.cin) return 0.0;  // padded stored channel
    double v;
    if (s.linear) {
      // torchvision flattens NCHW: column c*fh*fw + h*fw + w; our input is NHWC-flattened
      const int hw = s.fh * s.fw;
      const int cf = s.cin / hw;
      const int pix = c / cf, ch = c % cf;
      v = w[(int64_t)o * s.cin + (int64_t)ch * hw + pix];
    } else {
      v = w[(((int64_t)o * s.cin + c) * kk + r) * kk + t];
    }
    if (!fs.empty()) v *= fs[o];
    return v;
  };
  std::vector<float> bias(s.cout, 0.f);
  bool has_bias = b0 || !fs.empty();
  for (int o = 0; o < s.cout; ++o) {
    double bv = b0 ? (double)b0[o] : 0.0;
    if (!fs.empty()) bv = bv * fs[o] + fb[o];
    if (w2) bv += fb2[o];
    bias[o] = (float)bv;
  }
  const int taps = cw.kh * cw.kw;
  const int gk = cw.kw;
  if (m->bf16) {
    if (w2 && cw.K % 64 != 0) return set_error(HAPI_ERR_UNSUPPORTED, "fused downsample needs K1 %% 64 == 0");
    cw.Kp = (cw.K + cw.K2 + 7) / 8 * 8;
    std::vector<uint16_t> hw((size_t)s.cout * cw.Kp, 0);
    for (int o = 0; o < s.cout; ++o) {
      for (int tap = 0; tap < taps; ++tap)
        for (int c = 0; c < s.cs; ++c)
          hw[(size_t)o * cw.Kp + tap * s.cs + c] = f2bf((float)wval(o, tap / gk, tap % gk, c));
      for (int c = 0; c < cw.K2; ++c)
        hw[(size_t)o * cw.Kp + cw.K + c] = f2bf((float)((double)w2[(int64_t)o * s.cin2 + c] * fs2[o]));
    }
    uint16_t* dw;
    hapi_status st = upload(m, hw, &dw);
    if (st != HAPI_OK) return st;
    cw.w = dw;
    if (s.s2d && s.cout <= 64) {
      // stem+pool kernel (mode 8): 20 K chunks (padded s2d row rho 0..4, tap column s 0..3) of
      // [k half 2][n 128][8] (no-swizzle core matrices): n < 64 computes stem row 2po with tap
      // row rho, n >= 64 stem row 2po+1 with tap row rho-1; zero where the tap row is outside 0..3
      std::vector<uint16_t> h8((size_t)20 * 2 * 128 * 8, 0);
      for (int rho = 0; rho < 5; ++rho)
        for (int sc = 0; sc < 4; ++sc)
          for (int kh = 0; kh < 2; ++kh)
            for (int n = 0; n < 128; ++n) {
              const int o = n & 63, r = n < 64 ? rho : rho - 1;
              if (o >= s.cout || r < 0 || r > 3) continue;
              for (int j = 0; j < 8; ++j)
                h8[((((size_t)(rho * 4 + sc)) * 2 + kh) * 128 + n) * 8 + j] =
                    hw[(size_t)o * cw.Kp + (r * 4 + sc) * 16 + kh * 8 + j];
            }
      uint16_t* d8;
      if ((st = upload(m, h8, &d8)) != HAPI_OK) return st;
      cw.w8 = d8;
    }
    cw.bn = conv_tc_pick_bn(s.cout);
    if (s.res_identity) {
      if (cw.bn != 128 && cw.bn != 256) return set_error(HAPI_ERR_UNSUPPORTED, "identity residual needs BN 128/256");
      if (!m->ident) {
        // one 64x64 block: K chunk c of the N-row identity is this block at row offset c*64,
        // loaded at row coordinate -c*64 (the rows outside it are TMA out-of-bounds zeros)
        std::vector<uint16_t> id(64 * 64, 0);
        for (int i = 0; i < 64; ++i) id[(size_t)i * 64 + i] = 0x3F80;  // bf16 1.0
        uint16_t* did;
        if ((st = upload(m, id, &did)) != HAPI_OK) return st;
        m->ident = did;
        EncodeTiledFn enc0 = get_encode_fn();
        if (!enc0) return set_error(HAPI_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
        cuuint64_t dims[2] = {64, 64};
        cuuint64_t strides[1] = {128};
        cuuint32_t estr[2] = {1, 1};
        for (int bn2 : {128, 256}) {
          cuuint32_t box[2] = {64, (cuuint32_t)bn2};
          CUresult r = enc0(bn2 == 128 ? &m->ident_map128 : &m->ident_map256, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                            m->ident, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
          if (r != CUDA_SUCCESS) return set_error(HAPI_ERR_CUDA, "identity tensor map failed (%d)", (int)r);
        }
      }
    }
    EncodeTiledFn enc = get_encode_fn();
    if (!enc) return set_error(HAPI_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {(cuuint64_t)cw.Kp, (cuuint64_t)s.cout};
    cuuint64_t strides[1] = {(cuuint64_t)cw.Kp * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)cw.bn};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(&cw.tmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, cw.w, dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_error(HAPI_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d) for %s", (int)r, s.wname.c_str());
    if (cw.bn >= 128) {
      cuuint32_t boxh[2] = {64, (cuuint32_t)(cw.bn / 2)};
      r = enc(&cw.tmap_half, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, cw.w, dims, strides, boxh, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) return set_error(HAPI_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d) for %s", (int)r, s.wname.c_str());
      cw.has_half = true;
    }
  } else {
    cw.Kp = cw.K;
    std::vector<float> hw((size_t)cw.K * s.cout, 0.f);
    for (int o = 0; o < s.cout; ++o)
      for (int tap = 0; tap < taps; ++tap)
        for (int c = 0; c < s.cs; ++c)
          hw[(size_t)(tap * s.cs + c) * s.cout + o] = (float)wval(o, tap / gk, tap % gk, c);
    float* dw;
    hapi_status st = upload(m, hw, &dw);
    if (st != HAPI_OK) return st;
    cw.w = dw;
  }
  if (has_bias) {
    cw.hbias = bias;
    hapi_status st = upload(m, bias, &cw.bias);
    if (st != HAPI_OK) return st;
  }
  if (!s.pro_bn.empty()) {
    std::vector<double> ps, ph;
    if (!bn_affine(m, s.pro_bn, s.cin, ps, ph)) return set_error(HAPI_ERR_INVALID_MODEL, "bn %s missing", s.pro_bn.c_str());
    std::vector<float> fps(ps.begin(), ps.end()), fph(ph.begin(), ph.end());
    hapi_status st = upload(m, fps, &cw.pro_scale);
    if (st == HAPI_OK) st = upload(m, fph, &cw.pro_shift);
    if (st != HAPI_OK) return st;
    cw.mode = 2;
  } else {
    cw.mode = 0;
  }
  if (m->bf16 && s.cs % 8 != 0)
    return set_error(HAPI_ERR_UNSUPPORTED, "tensor-core conv needs C %% 8 == 0 (%s, C=%d)", s.wname.c_str(), s.cs);
  m->convs.push_back(cw);
  *out_idx = (int)m->convs.size() - 1;
  m->conv_index[key] = *out_idx;
  return HAPI_OK;
}

// ---------------------------------------------------------------- plan builder
struct Builder {
  hapi_model* m;
  Plan p;
  int new_buf(int64_t per_img_bytes) {
    Buf b;
    b.per_img = per_img_bytes;
    p.bufs.push_back(b);
    return (int)p.bufs.size() - 1;
  }
  View compact(int C, int H, int W) {
    View v;
    v.buf = new_buf((int64_t)C * H * W * m->es);
    v.C = C; v.H = H; v.W = W; v.ld = C; v.coff = 0;
    return v;
  }
  Op& emit(Op o) {
    p.ops.push_back(o);
    return p.ops.back();
  }
  hapi_status conv(const ConvSpec& cs, const View& in, const View& out, bool relu, const View* res, Op** op_out = nullptr,
                   const View* in2 = nullptr) {
    int ci;
    hapi_status st = make_conv(m, cs, &ci);
    if (st != HAPI_OK) return st;
    Op o;
    o.t = OP_CONV;
    o.in = in; o.out = out; o.conv = ci; o.relu = relu;
    if (res) { o.res = *res; o.has_res = true; }
    if (in2) { o.in2 = *in2; o.dual = true; }
    o.kind = m->bf16 ? 0 : 1;
    const ConvW& w = m->convs[ci];
    if (m->bf16) {
      o.tc_mode = w.mode;
      if (w.mode == 2 && w.kh == 1 && w.kw == 1 && w.stride == 1 && w.pad == 0 && prologue_tma_enabled()) {
        o.tc_mode = 7;  // TMA-loaded A, bn-relu applied in shared memory
      } else if (in2) {
        // fused downsample: both A sources must produce rows in the same order
        if (w.kh == 1 && w.kw == 1 && w.stride == 1 && w.pad == 0 && cs.stride2 == 1) {
          o.tc_mode = 3;
        } else if (im2col_enabled()) {
          o.tc_mode = 5;  // flat 128-row tiles, both sources through im2col TMA
        } else {
          conv_tc_spatial_tile(out.H, out.W, (int)m->d.max_batch, &o.wb, &o.hb, &o.nb);
          o.tc_mode = 4;
        }
      } else if (cs.s2d || cs.win3) {
        // space-to-depth stem (4x4/s1 over 16-channel pixels): read as a window view whose
        // rows are 4 adjacent padded pixels (128 B), W stride 32 B -> KH=4, KW=1, C=64 mode 4;
        // the VGG 3x3 stem likewise: rows of 8 padded 8-channel pixels, W stride 16 B, KH=3
        conv_tc_spatial_tile(out.H, out.W, (int)m->d.max_batch, &o.wb, &o.hb, &o.nb);
        o.tc_mode = 4;
        o.s2d_view = true;
      } else if (w.mode == 0 && w.cs % 64 == 0) {
        const int we = out.W + w.kw - 1;
        if (w.kh == 1 && w.kw == 1 && w.stride == 1 && w.pad == 0) {
          o.tc_mode = 3;
        } else if (w.stride == 1 && w.kh > 1 && we <= 128 && halo_enabled() &&
                   out.W * ((out.H + ((out.H + 128 / we - 1) / (128 / we)) - 1) / ((out.H + 128 / we - 1) / (128 / we))) >=
                       (w.bn <= 64 ? 64 : 96)) {
          // halo mode: one input box per 64-channel block, taps from row-shifted descriptors.
          // Only when a tile keeps enough of its 128 rows valid: halo beats im2col at 116 and 112
          // valid rows (ResNet-50 stage 1 -47%, stage 2 -18%); at 98 (14x14 maps) it was +10% in
          // round 1 and is now equal on ResNet-50 stage 3 and -2% on the ResNet-18 b200 step, so
          // the threshold is 96 (it was 108 for wide non-residual convs).  Narrow-N convs (their
          // MMA is smem-bound, and im2col writes 9x the A bytes into smem) take halo tiles from 64
          // valid rows: one 80-column row per tile at 320 px, DenseNet121 s=9 +25%, ResNet-50 +6%
          const int hmax = 128 / we;
          const int tiles_h = (out.H + hmax - 1) / hmax;
          o.hb = (out.H + tiles_h - 1) / tiles_h;
          o.wb = out.W;
          o.nb = 1;
          o.tc_mode = 6;
        } else if (im2col_enabled()) {
          o.tc_mode = 5;  // strided / small maps: im2col TMA per tap, full 128-row tiles
        } else if (w.stride <= 2) {
          conv_tc_spatial_tile(out.H, out.W, (int)m->d.max_batch, &o.wb, &o.hb, &o.nb);
          if (o.wb * w.stride <= 256 && o.hb * w.stride <= 256) o.tc_mode = 4;
        }
      }
    }
    const double px = (double)out.H * out.W;
    o.flops = w.real_flops_per_px * px;
    o.bytes = ((double)in.H * in.W * (cs.linear ? in.C : cs.cin) + px * w.cout * (res ? 2 : 1) +
               (in2 ? (double)in2->H * in2->W * in2->C : 0.0)) * m->es;
    char d[256];
    std::snprintf(d, sizeof(d), "%s %dx%d/s%d C%d->%d %dx%d->%dx%d bn%d mode%d%s%s%s%s%s", cs.wname.c_str(), w.kh,
                  w.kw, w.stride, w.cs, w.cout, in.H, in.W, out.H, out.W, w.bn, o.tc_mode, relu ? " relu" : "",
                  res ? " +res" : "", cs.pro_bn.empty() ? "" : " prologue", cs.s2d ? " s2d" : "",
                  in2 ? (cs.res_identity ? " +res(in GEMM)" : " +fused-downsample") : "");
    o.desc = d;
    emit(o);
    if (op_out) *op_out = &p.ops.back();
    return HAPI_OK;
  }
  void pool(const View& in, const View& out, int k, int s, int pad, int mode) {
    Op o;
    o.t = OP_POOL;
    o.in = in; o.out = out; o.pk = k; o.ps = s; o.pp = pad; o.pmode = mode;
    o.kind = 2;
    o.bytes = ((double)in.H * in.W * in.C + (double)out.H * out.W * out.C) * m->es;
    char d[128];
    std::snprintf(d, sizeof(d), "%s %dx%d/s%d p%d C%d %dx%d->%dx%d", mode ? "avgpool" : "maxpool", k, k, s, pad, in.C,
                  in.H, in.W, out.H, out.W);
    o.desc = d;
    emit(o);
  }
};

bool is_fresh_output(const Plan& p, int buf) {
  // buf written by the last op only and read by nobody
  int refs = 0;
  for (const Op& o : p.ops) {
    if (o.in.buf == buf && o.t != OP_PACK_IN) ++refs;
    if (o.has_res && o.res.buf == buf) ++refs;
    if (o.dual && o.in2.buf == buf) ++refs;
    if (o.out.buf == buf) ++refs;
  }
  return refs == 1 && !p.ops.empty() && p.ops.back().out.buf == buf;
}

hapi_status build_plan(hapi_model* m, int split, Plan* out, bool retarget) {
  Builder b{m};
  b.p.split = split;
  const ArchDesc& A = *m->arch;
  const int H0 = (int)m->d.in_h, W0 = (int)m->d.in_w;
  // a1: pack the caller's NCHW fp32 images.  bf16: ResNet/DenseNet stems (7x7/s2/p3) read a
  // 2x2 space-to-depth layout (16 channels at H/2 x W/2) so the stem gathers 16-byte pieces;
  // other stems read the image padded to 8 channels.
  const ModDesc& m0 = A.mods[0];
  const int start = (int)m->start;
  const bool s2d = start == 0 && m->bf16 && m0.kind == MK_CONV && m0.k == 7 && m0.stride == 2 && m0.pad == 3 &&
                   m0.cin == 3 && H0 % 2 == 0 && W0 % 2 == 0;
  const bool win3 = start == 0 && m->bf16 && m0.kind == MK_CONV && m0.k == 3 && m0.stride == 1 && m0.pad == 1 &&
                    m0.cin == 3 && win3_enabled();
  const bool col3 = win3 && stem_col_enabled();
  const int layout = !m->bf16 ? 0 : (s2d ? 2 : (col3 ? 4 : (win3 ? 3 : 1)));
  View cur;
  if (start == 0) {
    // s2d padded width: 3 zero columns on the left, >= 1 on the right, and room for the
    // stem+pool kernel's last strip box (S strips of 2 pq stem columns, box width 2 pq + 4)
    const int sw = W0 / 2, spw = (sw - 1) / 2 + 1, sS = (spw + 29) / 30, spq = (spw + sS - 1) / sS;
    const int WP = std::max(sw, 2 * sS * spq) + 4;
    cur = layout == 2   ? b.compact(16, H0 / 2 + 3, WP)
          : layout == 3 ? b.compact(8, H0 + 2, W0 + 8)
          : layout == 4 ? b.compact(64, H0, W0)
                        : b.compact(layout == 1 ? 8 : 3, H0, W0);
    Op o;
    o.t = OP_PACK_IN;
    o.out = cur;
    o.kind = 3;
    o.layout = layout;
    o.bytes = (double)H0 * W0 * 3 * 4 + (double)cur.C * cur.H * cur.W * m->es;
    b.emit(o);
  } else {
    // suffix plan: the input is layer `start`'s output in the send-buffer
    // layout (contiguous NCHW, act dtype) -- unpacked to NHWC, then layers start+1..split
    Shape sh{3, H0, W0, false};
    for (int k = 0; k < start; ++k) {
      bool ok;
      sh = infer(A.mods[k], sh, &ok);
      if (!ok) return set_error(HAPI_ERR_INVALID_MODEL, "layer %s empty", A.mods[k].name.c_str());
    }
    cur = sh.flat ? b.compact(sh.c, 1, 1) : b.compact(sh.c, sh.h, sh.w);
    Op o;
    o.t = OP_UNPACK;
    o.out = cur;
    o.kind = 3;
    o.bytes = 2.0 * (double)cur.C * cur.H * cur.W * m->es;
    o.desc = "unpack layer " + std::to_string(start) + " (NCHW -> NHWC)";
    b.emit(o);
  }
  const auto& mods = A.mods;
  int i = start;
  hapi_status st;
  while (i < split) {
    const ModDesc& md = mods[i];
    switch (md.kind) {
      case MK_CONV: {
        const bool fold = i + 1 < split && mods[i + 1].kind == MK_BN;
        const int j = i + 1 + (fold ? 1 : 0);
        const bool relu = j < split && mods[j].kind == MK_RELU;
        ConvSpec cs;
        cs.wname = md.name + ".weight";
        cs.bname = md.bias ? md.name + ".bias" : "";
        cs.fold_bn = fold ? mods[i + 1].name : "";
        cs.cin = md.cin; cs.cout = md.cout; cs.k = md.k; cs.stride = md.stride; cs.pad = md.pad;
        cs.cs = cur.C;
        cs.s2d = (i == 0 && s2d);
        cs.col3 = (i == 0 && col3);
        cs.win3 = (i == 0 && win3 && !col3);
        const int ih = (cs.s2d || cs.win3) ? H0 : cur.H, iw = (cs.s2d || cs.win3) ? W0 : cur.W;
        const int oh = out_dim(ih, md.k, md.stride, md.pad), ow = out_dim(iw, md.k, md.stride, md.pad);
        const int jp = j + (relu ? 1 : 0);
        if (cs.s2d && relu && md.cout <= 64 && jp < split && mods[jp].kind == MK_MAXPOOL && mods[jp].k == 3 &&
            mods[jp].stride == 2 && mods[jp].pad == 1 && stem_pool_enabled()) {
          // stem conv + bn + relu + 3x3/s2/p1 maxpool in one kernel (tcgen05 mode 8): the stem
          // map never reaches HBM
          View o = b.compact(md.cout, out_dim(oh, 3, 2, 1), out_dim(ow, 3, 2, 1));
          Op* op = nullptr;
          if ((st = b.conv(cs, cur, o, relu, nullptr, &op)) != HAPI_OK) return st;
          if (!m->convs[op->conv].w8) return set_error(HAPI_ERR_UNSUPPORTED, "stem weights for mode 8 missing");
          op->tc_mode = 8;
          op->conv_oh = oh; op->conv_ow = ow;
          const int pw = o.W, strips = (pw + 29) / 30, pq = (pw + strips - 1) / strips;
          op->wb = 2 * pq + 1; op->hb = 2; op->nb = 1;
          const ConvW& w = m->convs[op->conv];
          op->flops = w.real_flops_per_px * (double)oh * ow;
          op->bytes = ((double)cur.H * cur.W * cur.C + (double)o.H * o.W * o.C) * m->es;
          op->desc += " +maxpool3/s2 mode8";
          cur = o;
          i = jp + 1;
          break;
        }
        if ((cs.win3 || cs.col3) && relu && jp < split && mods[jp].kind == MK_MAXPOOL && mods[jp].k == 2 && mods[jp].stride == 2 &&
            mods[jp].pad == 0 && oh % 2 == 0 && ow % 2 == 0 && stem_pool_enabled()) {
          // VGG stem + relu + 2x2/s2 maxpool: [2 x wb] tiles, the epilogue writes only the pooled
          // row (the 224x224x64 stem map never reaches HBM)
          int wbp = 0;
          for (int d = 64; d >= 2; d -= 2)
            if (ow % d == 0) { wbp = d; break; }
          if (wbp > 0) {
            View o = b.compact(md.cout, oh / 2, ow / 2);
            Op* op = nullptr;
            if ((st = b.conv(cs, cur, o, relu, nullptr, &op)) != HAPI_OK) return st;
            if (cs.col3 && op->tc_mode == 3) {
              // the im2col-packed stem is a 1x1 conv: read it with mode-4 spatial boxes instead
              // of flat 2D tiles so the epilogue sees [2 x wb] pixel blocks to pool
              op->tc_mode = 4;
              const size_t mp_ = op->desc.find("mode3");
              if (mp_ != std::string::npos) op->desc.replace(mp_, 5, "mode4");
            }
            if (op->tc_mode == 4) {
              op->pool2 = true;
              op->conv_oh = oh; op->conv_ow = ow;
              op->wb = wbp; op->hb = 2; op->nb = 1;
              const ConvW& w = m->convs[op->conv];
              op->flops = w.real_flops_per_px * (double)oh * ow;
              op->bytes = ((double)cur.H * cur.W * cur.C + (double)o.H * o.W * o.C) * m->es;
              op->desc += " +maxpool2/s2";
              cur = o;
              i = jp + 1;
              break;
            }
            return set_error(HAPI_ERR_UNSUPPORTED, "VGG stem+pool: unexpected conv mode");
          }
        }
        View o = b.compact(md.cout, oh, ow);
        if ((st = b.conv(cs, cur, o, relu, nullptr)) != HAPI_OK) return st;
        cur = o;
        i = j + (relu ? 1 : 0);
        break;
      }
      case MK_BN: {
        if (i + 3 < split && mods[i + 1].kind == MK_RELU && mods[i + 2].kind == MK_CONV && mods[i + 2].k == 1 &&
            mods[i + 2].stride == 1 && mods[i + 2].pad == 0 && !mods[i + 2].bias && mods[i + 3].kind == MK_AVGPOOL &&
            mods[i + 3].k == 2 && mods[i + 3].stride == 2 && mods[i + 3].pad == 0 && cur.H % 2 == 0 &&
            cur.W % 2 == 0 && commute_enabled()) {
          // DenseNet transition with its pool inside the prefix: avgpool2x2(conv1x1(relu(bn x)))
          // = conv1x1(avgpool2x2(relu(bn x))) (a bias-free 1x1 conv and a 2x2 mean are both
          // linear and act on different axes), so pool first -- the conv then runs on a quarter
          // of the pixels and the C/2-channel full-size map never reaches HBM
          const ModDesc& cv = mods[i + 2];
          float *dsc, *dsh;
          auto it = m->bn_cache.find(md.name);
          if (it != m->bn_cache.end()) {
            dsc = it->second.first;
            dsh = it->second.second;
          } else {
            std::vector<double> sc, sh;
            if (!bn_affine(m, md.name, md.cin, sc, sh)) return set_error(HAPI_ERR_INVALID_MODEL, "bn %s", md.name.c_str());
            std::vector<float> fsc(sc.begin(), sc.end()), fsh(sh.begin(), sh.end());
            if ((st = upload(m, fsc, &dsc)) != HAPI_OK || (st = upload(m, fsh, &dsh)) != HAPI_OK) return st;
            m->bn_cache[md.name] = {dsc, dsh};
          }
          View pooled = b.compact(cur.C, cur.H / 2, cur.W / 2);
          b.pool(cur, pooled, 2, 2, 0, 1);
          b.p.ops.back().scale = dsc;
          b.p.ops.back().shift = dsh;
          b.p.ops.back().desc = "bn-relu + avgpool 2x2/s2 (transition commuted) C" + std::to_string(cur.C);
          ConvSpec cs;
          cs.wname = cv.name + ".weight";
          cs.cin = cv.cin; cs.cout = cv.cout; cs.k = 1; cs.stride = 1; cs.pad = 0;
          cs.cs = pooled.C;
          View o = b.compact(cv.cout, pooled.H, pooled.W);
          if ((st = b.conv(cs, pooled, o, false, nullptr)) != HAPI_OK) return st;
          cur = o;
          i += 4;
        } else if (i + 2 < split && mods[i + 1].kind == MK_RELU && mods[i + 2].kind == MK_CONV) {
          // DenseNet transition norm -> relu -> conv: bn-relu prologue on the conv's A operand
          const ModDesc& cv = mods[i + 2];
          ConvSpec cs;
          cs.wname = cv.name + ".weight";
          cs.pro_bn = md.name;
          cs.cin = cv.cin; cs.cout = cv.cout; cs.k = cv.k; cs.stride = cv.stride; cs.pad = cv.pad;
          cs.cs = cur.C;
          View o = b.compact(cv.cout, out_dim(cur.H, cv.k, cv.stride, cv.pad), out_dim(cur.W, cv.k, cv.stride, cv.pad));
          if ((st = b.conv(cs, cur, o, false, nullptr)) != HAPI_OK) return st;
          cur = o;
          i += 3;
        } else {
          const bool relu = i + 1 < split && mods[i + 1].kind == MK_RELU;
          float *dsc, *dsh;
          auto it = m->bn_cache.find(md.name);
          if (it != m->bn_cache.end()) {
            dsc = it->second.first;
            dsh = it->second.second;
          } else {
            std::vector<double> sc, sh;
            if (!bn_affine(m, md.name, md.cin, sc, sh)) return set_error(HAPI_ERR_INVALID_MODEL, "bn %s", md.name.c_str());
            std::vector<float> fsc(sc.begin(), sc.end()), fsh(sh.begin(), sh.end());
            if ((st = upload(m, fsc, &dsc)) != HAPI_OK || (st = upload(m, fsh, &dsh)) != HAPI_OK) return st;
            m->bn_cache[md.name] = {dsc, dsh};
          }
          View o = b.compact(cur.C, cur.H, cur.W);
          Op op;
          op.t = OP_BNACT;
          op.in = cur; op.out = o; op.scale = dsc; op.shift = dsh; op.relu = relu;
          op.kind = 4;
          op.bytes = 2.0 * cur.C * cur.H * cur.W * m->es;
          b.emit(op);
          cur = o;
          i += 1 + (relu ? 1 : 0);
        }
        break;
      }
      case MK_RELU: {
        View o = b.compact(cur.C, cur.H, cur.W);
        Op op;
        op.t = OP_BNACT;
        op.in = cur; op.out = o; op.relu = true;
        op.kind = 4;
        op.bytes = 2.0 * cur.C * cur.H * cur.W * m->es;
        b.emit(op);
        cur = o;
        i += 1;
        break;
      }
      case MK_MAXPOOL:
      case MK_AVGPOOL: {
        View o = b.compact(cur.C, out_dim(cur.H, md.k, md.stride, md.pad), out_dim(cur.W, md.k, md.stride, md.pad));
        b.pool(cur, o, md.k, md.stride, md.pad, md.kind == MK_MAXPOOL ? 0 : 1);
        cur = o;
        i += 1;
        break;
      }
      case MK_ADAPTIVE: {
        if (!(cur.H == md.oh && cur.W == md.ow)) {
          View o = b.compact(cur.C, md.oh, md.ow);
          Op op;
          op.t = OP_ADAPTIVE;
          op.in = cur; op.out = o;
          op.kind = 2;
          op.bytes = ((double)cur.C * cur.H * cur.W + (double)cur.C * md.oh * md.ow) * m->es;
          b.emit(op);
          cur = o;
        }
        i += 1;
        break;
      }
      case MK_DROPOUT:
        i += 1;  // identity; flatten is a view
        break;
      case MK_LINEAR:
      case MK_DENSE_CLS: {
        if (md.kind == MK_DENSE_CLS) {
          View o = b.compact(cur.C, 1, 1);
          Op op;
          op.t = OP_ADAPTIVE;
          op.in = cur; op.out = o; op.relu_in = true;
          op.kind = 2;
          op.bytes = ((double)cur.C * cur.H * cur.W + cur.C) * m->es;
          b.emit(op);
          cur = o;
        }
        if (cur.ld != cur.C || cur.coff != 0) return set_error(HAPI_ERR_UNSUPPORTED, "linear on a strided view");
        const bool relu = md.kind == MK_LINEAR && i + 1 < split && mods[i + 1].kind == MK_RELU;
        ConvSpec cs;
        cs.wname = md.name + ".weight";
        cs.bname = md.name + ".bias";
        cs.cin = md.cin; cs.cout = md.cout; cs.k = 1;
        cs.linear = true;
        cs.fh = cur.H; cs.fw = cur.W;
        cs.cs = cur.C * cur.H * cur.W;
        if (cs.cs != md.cin) return set_error(HAPI_ERR_INVALID_MODEL, "linear %s input %d != %d", md.name.c_str(), cs.cs, md.cin);
        View in = cur;
        in.C = cs.cs; in.H = 1; in.W = 1; in.ld = cs.cs;
        View o = b.compact(md.cout, 1, 1);
        if ((st = b.conv(cs, in, o, relu, nullptr)) != HAPI_OK) return st;
        cur = o;
        i += 1 + (relu ? 1 : 0);
        break;
      }
      case MK_BASIC:
      case MK_BOTTLENECK: {
        const std::string& p = md.name;
        const int OH = out_dim(cur.H, 3, md.stride, 1), OW = out_dim(cur.W, 3, md.stride, 1);
        View x = cur;
        if (md.kind == MK_BOTTLENECK && m->bf16 && md.stride == 1 && md.planes == 64 && md.cout % 64 == 0 &&
            md.cout <= 256 && (md.ds ? block_ds_enabled() : md.cout == cur.C) && cur.C % 64 == 0 && cur.C <= 256 &&
            cur.W <= 62 && cur.ld == cur.C && cur.coff == 0 && block_enabled()) {
          // the whole block on a CTA pair: x read once (the residual from L2), t1/t2 on chip
          ConvSpec c1, c2, c3;
          c1.wname = p + ".conv1.weight"; c1.fold_bn = p + ".bn1";
          c1.cin = md.cin; c1.cout = 64; c1.k = 1; c1.cs = x.C;
          c2.wname = p + ".conv2.weight"; c2.fold_bn = p + ".bn2";
          c2.cin = 64; c2.cout = 64; c2.k = 3; c2.pad = 1; c2.cs = 64;
          c3.wname = p + ".conv3.weight"; c3.fold_bn = p + ".bn3";
          c3.cin = 64; c3.cout = md.cout; c3.k = 1; c3.cs = 64;
          int i1, i2, i3, i4 = -1;
          if ((st = make_conv(m, c1, &i1)) != HAPI_OK || (st = make_conv(m, c2, &i2)) != HAPI_OK ||
              (st = make_conv(m, c3, &i3)) != HAPI_OK)
            return st;
          if (md.ds) {
            // ResNet layer1.0: the residual is the 1x1/s1 downsample of x (+BN), an MMA over a
            // second copy of the x tile inside the same kernel
            ConvSpec cd;
            cd.wname = p + ".downsample.0.weight"; cd.fold_bn = p + ".downsample.1";
            cd.cin = md.cin; cd.cout = md.cout; cd.k = 1; cd.cs = x.C;
            if ((st = make_conv(m, cd, &i4)) != HAPI_OK) return st;
          }
          Op o;
          o.t = OP_BLOCK;
          o.in = x;
          o.out = b.compact(md.cout, cur.H, cur.W);
          o.conv = i1; o.conv2 = i2; o.conv3 = i3; o.conv4 = i4;
          o.kind = 0;
          const double px = (double)cur.H * cur.W;
          o.flops = (m->convs[i1].real_flops_per_px + m->convs[i2].real_flops_per_px + m->convs[i3].real_flops_per_px +
                     (i4 >= 0 ? m->convs[i4].real_flops_per_px : 0.0)) * px;
          o.bytes = px * (x.C + md.cout) * m->es;   // x once (the residual re-read comes from L2) + out
          char d[160];
          std::snprintf(d, sizeof(d), "block[%s 1x1 C%d->64, 3x3 64->64, 1x1 64->%d %s] %dx%d (CTA pair)", p.c_str(),
                        x.C, md.cout, md.ds ? "+ds 1x1" : "+res", cur.H, cur.W);
          o.desc = d;
          b.emit(o);
          cur = o.out;
          i += 1;
          break;
        }
        View t;
        if (md.kind == MK_BOTTLENECK) {
          View t1 = b.compact(md.planes, cur.H, cur.W);
          ConvSpec c1;
          c1.wname = p + ".conv1.weight"; c1.fold_bn = p + ".bn1";
          c1.cin = md.cin; c1.cout = md.planes; c1.k = 1; c1.cs = x.C;
          if ((st = b.conv(c1, x, t1, true, nullptr)) != HAPI_OK) return st;
          t = b.compact(md.planes, OH, OW);
          ConvSpec c2;
          c2.wname = p + ".conv2.weight"; c2.fold_bn = p + ".bn2";
          c2.cin = md.planes; c2.cout = md.planes; c2.k = 3; c2.stride = md.stride; c2.pad = 1; c2.cs = md.planes;
          if ((st = b.conv(c2, t1, t, true, nullptr)) != HAPI_OK) return st;
        } else {
          t = b.compact(md.planes, OH, OW);
          ConvSpec c1;
          c1.wname = p + ".conv1.weight"; c1.fold_bn = p + ".bn1";
          c1.cin = md.cin; c1.cout = md.planes; c1.k = 3; c1.stride = md.stride; c1.pad = 1; c1.cs = x.C;
          if ((st = b.conv(c1, x, t, true, nullptr)) != HAPI_OK) return st;
        }
        // bf16: the downsample 1x1 joins the last conv as a second K-concatenated A source
        const bool fuse_ds = md.ds && m->bf16 && x.C % 64 == 0 && md.planes % 64 == 0 && !fused_ds_disabled();
        View idn = x;
        if (md.ds && !fuse_ds) {
          idn = b.compact(md.cout, OH, OW);
          ConvSpec cd;
          cd.wname = p + ".downsample.0.weight"; cd.fold_bn = p + ".downsample.1";
          cd.cin = md.cin; cd.cout = md.cout; cd.k = 1; cd.stride = md.stride; cd.cs = x.C;
          if ((st = b.conv(cd, x, idn, false, nullptr)) != HAPI_OK) return st;
        }
        ConvSpec cl;
        if (md.kind == MK_BOTTLENECK) {
          cl.wname = p + ".conv3.weight"; cl.fold_bn = p + ".bn3";
          cl.cin = md.planes; cl.cout = md.cout; cl.k = 1; cl.cs = md.planes;
        } else {
          cl.wname = p + ".conv2.weight"; cl.fold_bn = p + ".bn2";
          cl.cin = md.planes; cl.cout = md.cout; cl.k = 3; cl.pad = 1; cl.cs = md.planes;
        }
        if (fuse_ds) {
          // out = relu(bn(conv(t)) + bn_ds(conv1x1_s(x))) in one GEMM, into a fresh buffer
          cl.w2name = p + ".downsample.0.weight";
          cl.fold2 = p + ".downsample.1";
          cl.cin2 = md.cin;
          cl.stride2 = md.stride;
          View o = b.compact(md.cout, OH, OW);
          if ((st = b.conv(cl, t, o, true, nullptr, nullptr, &x)) != HAPI_OK) return st;
          cur = o;
        } else if (md.kind == MK_BOTTLENECK && m->bf16 && md.cout % 64 == 0 && md.planes % 64 == 0 &&
                   md.planes <= 128 && res_identity_enabled()) {
          // out = relu(bn(conv(t)) + idn): idn is a second K-concatenated A source against an
          // identity weight block (diagonal block per N tile), written in place over idn.  The
          // epilogue-bound small-K convs gain (stage 1: -16%, stage 2: -11%, measured); from
          // K = 256 the extra BN-deep MMA work cancels the gain (stage 3 equal, stage 4 +21%)
          cl.res_identity = true;
          if ((st = b.conv(cl, t, idn, true, nullptr, nullptr, &idn)) != HAPI_OK) return st;
          cur = idn;
        } else {
          // out = relu(bn(conv(t)) + idn), written in place over idn
          if ((st = b.conv(cl, t, idn, true, &idn)) != HAPI_OK) return st;
          cur = idn;
        }
        i += 1;
        break;
      }
      case MK_DENSEBLOCK: {
        const int C0 = md.cin, Ct = md.cout;
        View blk = b.compact(Ct, cur.H, cur.W);
        View head = blk;
        head.C = C0;
        if (retarget && cur.buf >= 0 && is_fresh_output(b.p, cur.buf) && cur.ld == cur.C && cur.coff == 0) {
          // retarget the producing op (pool0 / transition pool) into the block buffer
          b.p.ops.back().out = head;
          b.p.bufs[cur.buf].per_img = 0;
        } else {
          Op op;
          op.t = OP_BNACT;
          op.in = cur; op.out = head;
          op.kind = 4;
          op.bytes = 2.0 * C0 * cur.H * cur.W * m->es;
          b.emit(op);
        }
        View tmid = b.compact(md.bn_size * md.growth, cur.H, cur.W);
        for (int j = 0; j < md.nlayers; ++j) {
          const std::string q = md.name + ".denselayer" + std::to_string(j + 1);
          const int cj = C0 + md.growth * j;
          View in = blk;
          in.C = cj;
          ConvSpec c1;
          c1.wname = q + ".conv1.weight"; c1.pro_bn = q + ".norm1"; c1.fold_bn = q + ".norm2";
          c1.cin = cj; c1.cout = md.bn_size * md.growth; c1.k = 1; c1.cs = cj;
          if ((st = b.conv(c1, in, tmid, true, nullptr)) != HAPI_OK) return st;
          View o = blk;
          o.C = md.growth;
          o.coff = cj;
          ConvSpec c2;
          c2.wname = q + ".conv2.weight";
          c2.cin = md.bn_size * md.growth; c2.cout = md.growth; c2.k = 3; c2.pad = 1; c2.cs = md.bn_size * md.growth;
          if ((st = b.conv(c2, tmid, o, false, nullptr)) != HAPI_OK) return st;
        }
        cur = blk;
        i += 1;
        break;
      }
    }
  }

  // fp32 path: split K of convs whose output grid would leave most SMs idle (small batches,
  // config 1).  The [ksplit][M][Cout] workspace is an arena buffer live only during the conv,
  // capped so that in + out + workspace stays within the plan's largest in + out (the
  // per-image peak the planner's P(s) already covers, section 4.3).
  if (!m->bf16) {
    std::vector<Op>& ops = b.p.ops;
    double peak = 0;
    for (const Op& o : ops)
      if (o.t == OP_CONV)
        peak = std::max(peak, ((double)o.in.H * o.in.W * o.in.ld + (double)o.out.H * o.out.W * o.out.ld) * m->es);
    for (size_t k = 0; k < ops.size(); ++k) {
      if (ops[k].t != OP_CONV) continue;
      const ConvW& w = m->convs[ops[k].conv];
      const View in = ops[k].in, out = ops[k].out;
      int ks = conv_simt_ksplit((long long)m->d.max_batch * out.H * out.W, w.cout, w.K, m->num_sms);
      const double io = ((double)in.H * in.W * in.ld + (double)out.H * out.W * out.ld) * m->es;
      const double wsb = (double)out.H * out.W * w.cout * m->es;
      while (ks > 1 && io + ks * wsb > peak) ks /= 2;
      if (ks > 1) {
        View ws = b.compact(w.cout * ks, out.H, out.W);
        ops[k].ksplit = ks;
        ops[k].ws = ws;
      }
    }
  }

  // Peephole: a bottleneck's last conv (1x1, residual or stride-1 downsample as second A
  // source) directly followed by the next block's 1x1 conv1 reading its output becomes one
  // OP_PAIR launch -- the block output tile stays in smem as conv1's A operand.
  if (m->bf16 && pair_enabled()) {
    std::vector<Op>& ops = b.p.ops;
    for (size_t k = 0; k + 1 < ops.size(); ++k) {
      Op& A = ops[k];
      const Op& B = ops[k + 1];
      if (A.t != OP_CONV || B.t != OP_CONV || A.tc_mode != 3 || !A.dual || A.has_res || !A.relu || A.nchw_out) continue;
      if (B.tc_mode != 3 || B.dual || B.has_res || !B.relu || B.nchw_out) continue;
      const ConvW& wa = m->convs[A.conv];
      const ConvW& wb = m->convs[B.conv];
      const bool ds1 = !wa.res_identity && wa.stride2 == 1 && wa.K2 % 64 == 0 && wa.K2 > 0;
      if (!(wa.res_identity || ds1) || wa.kh != 1 || wa.K % 64 != 0 || wa.cout % 128 != 0 || wa.cout > 2048) continue;
      if (wb.kh != 1 || wb.stride != 1 || wb.pro_scale || wb.cs != wa.cout || wb.bn != wb.cout ||
          (wb.cout != 64 && wb.cout != 128) || wa.K > 128 || wa.cout > 512)
        continue;
      if (B.in.buf != A.out.buf || B.in.coff != A.out.coff || B.in.ld != A.out.ld || A.out.buf < 0 || B.out.buf < 0 ||
          A.out.ld != A.out.C || B.out.ld != B.out.C)
        continue;
      Op P = A;
      P.t = OP_PAIR;
      P.conv2 = B.conv;
      P.out2 = B.out;
      P.flops = A.flops + B.flops;
      P.bytes = A.bytes + (double)B.out.H * B.out.W * B.out.C * m->es;
      P.desc = "pair[" + A.desc + " => " + B.desc + "]";
      ops[k] = P;
      ops.erase(ops.begin() + (long)k + 1);
    }
  }

  // a7: deliver layer `split` into the caller's buffer as contiguous NCHW.
  Plan& p = b.p;
  b.p.out_bytes_per_img = (int64_t)cur.C * cur.H * cur.W * m->es;
  Op& last = p.ops.back();
  const bool compact = cur.ld == cur.C && cur.coff == 0;
  const bool same_view = cur.buf >= 0 && last.out.buf == cur.buf && last.out.C == cur.C && last.out.ld == cur.ld &&
                         last.out.coff == cur.coff;
  const bool can_direct = same_view && compact && last.t != OP_PACK_IN &&
                          !(last.t == OP_CONV && (last.tc_mode == 8 || last.pool2));
  static const bool nchw_epi = [] {  // HAPI_NCHW_EPI=0: last conv stores NHWC, then the split pack
    const char* e = std::getenv("HAPI_NCHW_EPI");
    return !(e && e[0] == '0');
  }();
  if (can_direct && last.t == OP_CONV && nchw_epi) {
    last.out.buf = -1;
    last.nchw_out = true;
  } else if (can_direct && cur.H == 1 && cur.W == 1 && (last.t == OP_POOL || last.t == OP_ADAPTIVE || last.t == OP_BNACT)) {
    last.out.buf = -1;
  } else {
    Op op;
    op.t = OP_PACK_OUT;
    op.in = cur;
    op.out.buf = -1;
    op.kind = 3;
    op.bytes = 2.0 * cur.C * cur.H * cur.W * m->es;
    b.emit(op);
  }
  // A pair's block output whose only other reader is the next stage's fused 1x1/stride-2
  // downsample is stored at stride 2 (a quarter of the bytes; the pair's GEMM2 takes the full
  // tile from shared memory either way).
  if (m->bf16 && sub_store_enabled()) {
    for (size_t k = 0; k < p.ops.size(); ++k) {
      Op& P = p.ops[k];
      if (P.t != OP_PAIR || P.out.buf < 0 || P.out.ld != P.out.C || P.out.coff != 0) continue;
      const int buf = P.out.buf;
      int uses = 0;
      Op* ds = nullptr;
      for (size_t q = k + 1; q < p.ops.size(); ++q) {  // (earlier ops may share the buffer: in-place residuals)
        Op& o = p.ops[q];
        if (o.t != OP_PACK_IN && o.in.buf == buf) ++uses;
        if (o.has_res && o.res.buf == buf) ++uses;
        if (o.dual && o.in2.buf == buf) { ++uses; ds = &o; }
        if (o.out.buf == buf || (o.t == OP_PAIR && o.out2.buf == buf) || (o.ksplit > 1 && o.ws.buf == buf)) uses += 2;
      }
      if (uses != 1 || !ds || ds->t != OP_CONV || (ds->tc_mode != 4 && ds->tc_mode != 5)) continue;
      const ConvW& wd = m->convs[ds->conv];
      const int sh = (P.out.H + 1) / 2, sw = (P.out.W + 1) / 2;
      if (wd.res_identity || wd.stride2 != 2 || ds->in2.coff != 0 || ds->in2.ld != P.out.ld || ds->out.H != sh ||
          ds->out.W != sw)
        continue;
      const View sub = b.compact(P.out.C, sh, sw);
      P.sub_out = true;
      P.full_h = P.out.H;
      P.full_w = P.out.W;
      P.out = sub;
      P.bytes -= 0.75 * (double)P.full_h * P.full_w * P.out.C * m->es;
      P.desc += " (block output stored at stride 2)";
      ds->in2 = sub;
      ds->in2_stride = 1;
    }
  }
  // liveness + first-fit arena placement (sizes at max_batch)
  for (size_t k = 0; k < p.ops.size(); ++k) {
    const Op& o = p.ops[k];
    auto touch = [&](int buf) {
      if (buf < 0) return;
      Buf& bb = p.bufs[buf];
      if (bb.first < 0) bb.first = (int)k;
      bb.last = (int)k;
    };
    if (o.t != OP_PACK_IN) touch(o.in.buf);
    if (o.has_res) touch(o.res.buf);
    if (o.dual) touch(o.in2.buf);
    touch(o.out.buf);
    if (o.t == OP_PAIR) touch(o.out2.buf);
    if (o.ksplit > 1) touch(o.ws.buf);
  }
  const int64_t B = m->d.max_batch;
  std::vector<int> order;
  for (size_t k = 0; k < p.bufs.size(); ++k)
    if (p.bufs[k].first >= 0 && p.bufs[k].per_img > 0) order.push_back((int)k);
  std::sort(order.begin(), order.end(), [&](int a, int c) { return p.bufs[a].per_img * B > p.bufs[c].per_img * B; });
  std::vector<int> placed;
  int64_t top = 0;
  for (int id : order) {
    Buf& bb = p.bufs[id];
    const int64_t sz = (bb.per_img * B + 255) / 256 * 256;
    // candidate offsets: 0 and the end of every overlapping placed buffer
    std::vector<int64_t> cands{0};
    for (int q : placed) {
      const Buf& o = p.bufs[q];
      if (o.last < bb.first || o.first > bb.last) continue;
      cands.push_back(o.offset + (o.per_img * B + 255) / 256 * 256);
    }
    std::sort(cands.begin(), cands.end());
    for (int64_t off : cands) {
      bool ok = true;
      for (int q : placed) {
        const Buf& o = p.bufs[q];
        if (o.last < bb.first || o.first > bb.last) continue;
        const int64_t oe = o.offset + (o.per_img * B + 255) / 256 * 256;
        if (off < oe && o.offset < off + sz) { ok = false; break; }
      }
      if (ok) { bb.offset = off; break; }
    }
    placed.push_back(id);
    top = std::max(top, bb.offset + sz);
  }
  p.arena_bytes = top;
  *out = std::move(b.p);
  return HAPI_OK;
}

// ---------------------------------------------------------------- launching
inline char* vptr(hapi_model* m, const Plan& p, const View& v, void* ext) {
  char* base = v.buf < 0 ? static_cast<char*>(ext) : static_cast<char*>(m->arena) + p.bufs[v.buf].offset;
  return base + (int64_t)v.coff * m->es;
}

hapi_status launch_op(hapi_model* m, const Plan& p, const Op& o, int nb, const void* images, bool in_u8, void* out,
                      cudaStream_t st) {
  cudaError_t e = cudaSuccess;
  const int isb = m->bf16 ? 1 : 0;
  switch (o.t) {
    case OP_PACK_IN:
      e = pack_input_launch(images, in_u8 ? &m->u8norm : nullptr, vptr(m, p, o.out, out), nb, (int)m->d.in_h,
                            (int)m->d.in_w, o.layout, o.out.W, st);
      break;
    case OP_UNPACK:
      e = unpack_nchw_launch(images, nb, o.out.C, o.out.H * o.out.W, vptr(m, p, o.out, out), o.out.ld, m->es, st);
      break;
    case OP_PAIR: {
      const ConvW& wa = m->convs[o.conv];
      const ConvW& wb = m->convs[o.conv2];
      PairArgs a;
      a.M = o.sub_out ? (long long)nb * o.full_h * o.full_w : (long long)nb * o.out.H * o.out.W;
      a.y1_sub = o.sub_out ? vptr(m, p, o.out, out) : nullptr;
      a.H = o.sub_out ? o.full_h : o.out.H;
      a.W = o.sub_out ? o.full_w : o.out.W;
      a.k1_chunks = wa.K / 64;
      a.k2_diag = wa.res_identity ? 1 : 0;
      a.k2_chunks = wa.res_identity ? 2 : wa.K2 / 64;
      a.cout1 = wa.cout;
      a.bias1 = wa.bias;
      a.bias2 = wb.bias;
      PairMaps mp;
      mp.a1 = &o.tmap_a;
      mp.a2 = &o.tmap_a2;
      mp.b1 = &o.tmap_b1;
      mp.id = &m->ident_map128;
      mp.b2 = &wb.tmap;
      mp.y1 = &o.tmap_y;
      mp.y2 = &o.tmap_y2;
      e = conv_pair_launch(a, mp, wb.cout, m->num_sms, st);
      break;
    }
    case OP_CONV: {
      const ConvW& w = m->convs[o.conv];
      ConvArgs a;
      a.pool2 = o.pool2 ? 1 : 0;
      a.ksplit = 1;
      a.ws = nullptr;
      a.x = vptr(m, p, o.in, out);
      a.N = nb; a.H = o.in.H; a.W = o.in.W; a.C = w.cs; a.x_ld = o.in.ld;
      a.KH = w.kh; a.KW = w.kw; a.stride = w.stride; a.pad = w.pad;
      a.OH = o.out.H; a.OW = o.out.W;
      a.Cout = w.cout;
      a.K = w.K;
      a.w = w.w;
      a.bias = w.bias;
      for (int i = 0; i < 64; ++i) a.bias_u[i] = i < (int)w.hbias.size() ? w.hbias[i] : 0.f;
      a.pro_scale = w.pro_scale;
      a.pro_shift = w.pro_shift;
      a.res = o.has_res ? vptr(m, p, o.res, out) : nullptr;
      a.res_ld = o.has_res ? o.res.ld : 0;
      a.y = vptr(m, p, o.out, out);
      a.y_ld = o.out.ld;
      a.relu = o.relu;
      a.nchw = o.nchw_out;
      a.M = (long long)nb * a.OH * a.OW;
      a.k2_chunks = o.dual ? (w.res_identity ? w.bn / 64 : w.K2 / 64) : 0;
      a.stride2 = o.in2_stride ? o.in2_stride : w.stride2;
      a.k2_diag = w.res_identity ? 1 : 0;
      if (o.s2d_view) {  // window view geometry (see finalize_tmaps)
        a.C = 64; a.KH = w.kh; a.KW = 1; a.stride = 1; a.pad = 0;
      }
      if (o.pool2) {  // the kernel iterates the conv map; y is the 2x2-pooled map
        a.OH = o.conv_oh; a.OW = o.conv_ow;
        a.M = (long long)nb * a.OH * a.OW;
      }
      if (o.tc_mode == 8) {  // the kernel iterates the stem map; y is the pooled map
        a.OH = o.conv_oh; a.OW = o.conv_ow;
        a.w = w.w8;
        a.M = (long long)nb * a.OH * a.OW;
      }
      if (m->bf16) {
        ConvMaps mp;
        mp.a = (o.tc_mode >= 3) ? &o.tmap_a : nullptr;
        mp.a2 = o.dual ? &o.tmap_a2 : nullptr;
        mp.b2 = w.res_identity ? (w.bn == 256 ? &m->ident_map256 : &m->ident_map128) : nullptr;
        mp.b = &w.tmap;
        mp.bh = w.has_half ? &w.tmap_half : nullptr;
        mp.y = o.nchw_out ? nullptr : &o.tmap_y;
        mp.r = (o.has_res && !o.nchw_out) ? &o.tmap_r : nullptr;
        mp.yw = o.has_yw ? &o.tmap_yw : nullptr;
        e = conv_tc_launch(a, mp, o.tc_mode == 8 ? 128 : w.bn, o.tc_mode, o.wb, o.hb, o.nb, m->num_sms, st);
      } else {
        a.ksplit = o.ksplit;
        a.ws = o.ksplit > 1 ? reinterpret_cast<float*>(vptr(m, p, o.ws, out)) : nullptr;
        e = conv_simt_launch(a, st);
      }
      break;
    }
    case OP_POOL: {
      PoolArgs a;
      a.x = vptr(m, p, o.in, out);
      a.N = nb; a.H = o.in.H; a.W = o.in.W; a.C = o.in.C; a.x_ld = o.in.ld;
      a.y = vptr(m, p, o.out, out);
      a.OH = o.out.H; a.OW = o.out.W; a.y_ld = o.out.buf < 0 ? o.out.C : o.out.ld;
      a.k = o.pk; a.stride = o.ps; a.pad = o.pp; a.mode = o.pmode;
      a.pro_scale = o.scale;
      a.pro_shift = o.shift;
      e = pool_launch(a, isb, st);
      break;
    }
    case OP_ADAPTIVE: {
      AdaptiveArgs a;
      a.x = vptr(m, p, o.in, out);
      a.N = nb; a.H = o.in.H; a.W = o.in.W; a.C = o.in.C; a.x_ld = o.in.ld;
      a.y = vptr(m, p, o.out, out);
      a.OH = o.out.H; a.OW = o.out.W; a.y_ld = o.out.buf < 0 ? o.out.C : o.out.ld;
      a.relu_in = o.relu_in;
      e = adaptive_avgpool_launch(a, isb, st);
      break;
    }
    case OP_BNACT: {
      EltArgs a;
      a.x = vptr(m, p, o.in, out);
      a.N = nb; a.HW = o.in.H * o.in.W; a.C = o.in.C; a.x_ld = o.in.ld;
      a.y = vptr(m, p, o.out, out);
      a.y_ld = o.out.buf < 0 ? o.out.C : o.out.ld;
      a.scale = o.scale; a.shift = o.shift; a.relu = o.relu;
      e = bn_act_launch(a, isb, st);
      break;
    }
    case OP_PACK_OUT:
      e = pack_output_launch(vptr(m, p, o.in, out), nb, o.in.H * o.in.W, o.in.C, o.in.ld, out, isb, st);
      break;
    case OP_BLOCK: {
      BlockArgs a;
      a.N = nb; a.H = o.in.H; a.W = o.in.W; a.C = o.in.C;
      a.Cout = o.out.C;
      a.ds = o.conv4 >= 0 ? 1 : 0;
      a.x = vptr(m, p, o.in, out); a.x_ld = o.in.ld;
      a.y = vptr(m, p, o.out, out); a.y_ld = o.out.ld;
      auto fill = [&](float* dst, int n, const ConvW& cw) {
        for (int i = 0; i < n; ++i) dst[i] = (int)cw.hbias.size() == n ? cw.hbias[i] : 0.f;
      };
      std::memset(a.b3, 0, sizeof(a.b3));
      fill(a.b1, 64, m->convs[o.conv]);
      fill(a.b2, 64, m->convs[o.conv2]);
      fill(a.b3, a.Cout, m->convs[o.conv3]);
      if (a.ds) {  // conv3's and the downsample's folded biases land in the same accumulator
        const ConvW& wd = m->convs[o.conv4];
        for (int i = 0; i < a.Cout; ++i) a.b3[i] += (int)wd.hbias.size() == a.Cout ? wd.hbias[i] : 0.f;
      }
      BlockMaps mp;
      mp.x = &o.bmap_x; mp.w1 = &o.bmap_w1; mp.w2 = &o.bmap_w2; mp.w3 = &o.bmap_w3;
      mp.wds = o.conv4 >= 0 ? &o.bmap_wds : nullptr;
      e = conv_block_launch(a, mp, m->num_sms, st);
      break;
    }
  }
  if (e != cudaSuccess)
    return set_error(HAPI_ERR_CUDA, "launch of %s failed: %s", o.desc.empty() ? "op" : o.desc.c_str(), cudaGetErrorString(e));
  return HAPI_OK;
}

// HAPI_NVTX=1: one NVTX range per launch (fused group), named by its plan description -- the
// per-layer timeline the paper plots in Nsight; with HAPI_GRAPH=0, since a
// replayed CUDA graph emits no host-side ranges
bool nvtx_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("HAPI_NVTX");
    return e && e[0] == '1';
  }();
  return on;
}

hapi_status run_chunk(hapi_model* m, const Plan& p, int nb, const void* images, bool in_u8, void* out, cudaStream_t st,
                      cudaEvent_t* evs = nullptr) {
  const bool nvtx = nvtx_enabled();
  for (size_t k = 0; k < p.ops.size(); ++k) {
    if (evs) cudaEventRecord(evs[k], st);
    if (nvtx) nvtxRangePushA(p.ops[k].desc.empty() ? "op" : p.ops[k].desc.c_str());
    hapi_status s = launch_op(m, p, p.ops[k], nb, images, in_u8, out, st);
    if (nvtx) nvtxRangePop();
    if (s != HAPI_OK) return s;
  }
  if (evs) cudaEventRecord(evs[p.ops.size()], st);
  return HAPI_OK;
}

// TMA descriptors of the A operand (modes 3/4) need the placed arena, so they are
// encoded once after allocation.  The batch dimension spans max_batch images; smaller
// calls read (and then discard) rows past the batch inside the same buffer.
hapi_status encode_bf16(CUtensorMap* map, int rank, void* base, const cuuint64_t* dims, const cuuint64_t* strides,
                        const cuuint32_t* box, const cuuint32_t* estr, CUtensorMapSwizzle swz, const std::string& what) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return set_error(HAPI_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, base, dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(HAPI_ERR_CUDA, "tensor map encode failed (%d): %s", (int)r, what.c_str());
  return HAPI_OK;
}

// im2col map for mode 5: {C, W, H, N} NHWC view; the bounding box of traversal positions is
// [-pad, dim - 1 + pad - (k - 1)] per spatial dim, walked with the conv stride, so a load at
// (ow*s - pad, oh*s - pad, n) with tap offsets (s, r) yields the A tile of 128 consecutive
// output pixels for that tap (padding = OOB zero fill); box = 64 channels x 128 pixels.
hapi_status encode_im2col(hapi_model* m, void* base, const View& v, int C, int kh, int kw, int stride, int pad,
                          CUtensorMap* map, const std::string& what) {
  EncodeIm2colFn enc = get_im2col_fn();
  if (!enc) return set_error(HAPI_ERR_CUDA, "cuTensorMapEncodeIm2col unavailable");
  const cuuint64_t ld = (cuuint64_t)v.ld * 2;
  cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)v.W, (cuuint64_t)v.H, (cuuint64_t)m->d.max_batch};
  cuuint64_t strides[3] = {ld, ld * v.W, ld * v.W * v.H};
  int lower[2] = {-pad, -pad};
  int upper[2] = {pad - (kw - 1), pad - (kh - 1)};
  cuuint32_t estr[4] = {1, (cuuint32_t)stride, (cuuint32_t)stride, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, base, dims, strides, lower, upper, 64, 128, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(HAPI_ERR_CUDA, "im2col tensor map encode failed (%d): %s", (int)r, what.c_str());
  return HAPI_OK;
}

// Map over an NHWC activation view with the conv's tile geometry: 2D [M][C] with a
// {cols, 128} box for linear tiles, 4D {C, W, H, N} with a {cols, wb, hb, nb} box for
// mode-4 spatial tiles.  The batch extent is max_batch.
hapi_status encode_view(hapi_model* m, const Plan& p, const Op& o, const View& v, int cols, CUtensorMap* map,
                        const char* what, int rows = 128) {
  const cuuint64_t es = 2, ld = (cuuint64_t)v.ld;
  const CUtensorMapSwizzle swz = cols * 2 == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
  void* base = vptr(m, p, v, nullptr);
  if (o.tc_mode == 4 || o.tc_mode == 6) {
    cuuint64_t dims[4] = {(cuuint64_t)v.C, (cuuint64_t)v.W, (cuuint64_t)v.H, (cuuint64_t)m->d.max_batch};
    cuuint64_t strides[3] = {ld * es, ld * es * v.W, ld * es * v.W * v.H};
    cuuint32_t box[4] = {(cuuint32_t)cols, (cuuint32_t)o.wb, (cuuint32_t)o.hb, (cuuint32_t)o.nb};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    return encode_bf16(map, 4, base, dims, strides, box, estr, swz, o.desc + " " + what);
  }
  cuuint64_t dims[2] = {(cuuint64_t)v.C, (cuuint64_t)m->d.max_batch * v.H * v.W};
  cuuint64_t strides[1] = {ld * es};
  cuuint32_t box[2] = {(cuuint32_t)cols, (cuuint32_t)rows};
  cuuint32_t estr[2] = {1, 1};
  return encode_bf16(map, 2, base, dims, strides, box, estr, swz, o.desc + " " + what);
}

// TMA descriptors over arena views need the placed arena, so they are encoded once after
// allocation.  The batch extent is max_batch; smaller calls touch rows past the batch
// inside the same arena buffers only (never the caller's output, which is written by the
// NCHW path).
hapi_status finalize_tmaps(hapi_model* m) {
  if (!m->bf16) return HAPI_OK;
  for (Plan& p : m->plans) {
    for (Op& o : p.ops) {
      if (o.t == OP_BLOCK) {
        const ConvW &w1 = m->convs[o.conv], &w2 = m->convs[o.conv2], &w3 = m->convs[o.conv3];
        const cuuint64_t ld = (cuuint64_t)o.in.ld * 2;
        cuuint64_t xd[4] = {(cuuint64_t)o.in.C, (cuuint64_t)o.in.W, (cuuint64_t)o.in.H, (cuuint64_t)m->d.max_batch};
        cuuint64_t xs[3] = {ld, ld * o.in.W, ld * o.in.W * o.in.H};
        cuuint32_t xb[4] = {64, 64, 2, 1};
        cuuint32_t e4[4] = {1, 1, 1, 1};
        hapi_status st = encode_bf16(&o.bmap_x, 4, vptr(m, p, o.in, nullptr), xd, xs, xb, e4, CU_TENSOR_MAP_SWIZZLE_128B,
                                     o.desc + " x");
        auto wmap = [&](CUtensorMap* mp, const ConvW& w, int rows) {
          cuuint64_t dd[2] = {(cuuint64_t)w.Kp, (cuuint64_t)w.cout};
          cuuint64_t ss[1] = {(cuuint64_t)w.Kp * 2};
          cuuint32_t bb[2] = {64, (cuuint32_t)rows};
          return encode_bf16(mp, 2, w.w, dd, ss, bb, e4, CU_TENSOR_MAP_SWIZZLE_128B, o.desc + " w");
        };
        if (st == HAPI_OK) st = wmap(&o.bmap_w1, w1, 32);
        if (st == HAPI_OK) st = wmap(&o.bmap_w2, w2, 32);
        if (st == HAPI_OK) st = wmap(&o.bmap_w3, w3, w3.cout / 2);
        if (st == HAPI_OK && o.conv4 >= 0) st = wmap(&o.bmap_wds, m->convs[o.conv4], m->convs[o.conv4].cout / 2);
        if (st != HAPI_OK) return st;
        continue;
      }
      if (o.t != OP_CONV && o.t != OP_PAIR) continue;
      const ConvW& w = m->convs[o.conv];
      hapi_status st = HAPI_OK;
      if (o.t == OP_PAIR) {
        // conv3 weights with the pair kernel's 128-row N tile, and the next conv1's output view
        EncodeTiledFn enc = get_encode_fn();
        if (!enc) return set_error(HAPI_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
        cuuint64_t dims[2] = {(cuuint64_t)w.Kp, (cuuint64_t)w.cout};
        cuuint64_t strides[1] = {(cuuint64_t)w.Kp * 2};
        cuuint32_t box[2] = {64, 128};
        cuuint32_t estr[2] = {1, 1};
        CUresult r = enc(&o.tmap_b1, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w.w, dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return set_error(HAPI_ERR_CUDA, "pair weight tensor map failed (%d)", (int)r);
        // the pair kernel stores one 32-row quarter of a [128 x 64] staging block per box
        if ((st = encode_view(m, p, o, o.out2, 64, &o.tmap_y2, "Y2", 32)) != HAPI_OK) return st;
      }
      if (o.tc_mode == 8) {
        // stem+pool boxes over the padded s2d input [N][HP][WP][16] as a 5D view
        // {16 ch, we cols, S strips (stride 2 pq cols), HP rows, N}: one box {8, we, 2, 5, 1}
        // per 8-channel plane lands as [row][strip][col] x 16 B.  Column x of strip k is
        // padded column 2 k pq + x = stem column 2 k pq - 1 + x (3 zero columns on the left).
        const int pw = o.out.W, S = (pw + 29) / 30, pq = (pw + S - 1) / S, we = 2 * pq + 4;
        void* base = vptr(m, p, o.in, nullptr);
        const cuuint64_t px = (cuuint64_t)o.in.ld * 2;
        cuuint64_t dims[5] = {16, (cuuint64_t)we, (cuuint64_t)S, (cuuint64_t)o.in.H, (cuuint64_t)m->d.max_batch};
        cuuint64_t strides[4] = {px, px * 2 * pq, px * o.in.W, px * o.in.W * o.in.H};
        cuuint32_t box[5] = {8, (cuuint32_t)we, 2, 5, 1};
        cuuint32_t estr[5] = {1, 1, 1, 1, 1};
        st = encode_bf16(&o.tmap_a, 5, base, dims, strides, box, estr, CU_TENSOR_MAP_SWIZZLE_NONE, o.desc + " stem 5D");
        if (st != HAPI_OK) return st;
      } else if (o.s2d_view) {
        // overlapping window view of the padded s2d input: element (e, w, h, n) at
        // base + n*HP*WP*32 + h*WP*32 + (w+1)*32 + 2e, e < 64 spans 4 adjacent pixels (stem
        // column w starts at padded column w+1: the buffer has 3 zero columns on the left)
        // (the VGG 3x3 window view, KW = 8: 8-channel pixels, 16 B, and output column w starts
        // at padded column w -- one zero column on the left)
        const bool win3 = w.kw == 8;
        void* base = static_cast<char*>(vptr(m, p, o.in, nullptr)) + (win3 ? 0 : o.in.ld * 2);
        const cuuint64_t px = (cuuint64_t)o.in.ld * 2;  // 32 B (s2d) / 16 B (win3)
        const int stem_w = (o.tc_mode == 8 || o.pool2) ? o.conv_ow : o.out.W;
        cuuint64_t dims[4] = {64, (cuuint64_t)stem_w, (cuuint64_t)o.in.H, (cuuint64_t)m->d.max_batch};
        cuuint64_t strides[3] = {px, px * o.in.W, px * o.in.W * o.in.H};
        cuuint32_t box[4] = {64, (cuuint32_t)o.wb, (cuuint32_t)o.hb, (cuuint32_t)o.nb};
        cuuint32_t estr[4] = {1, 1, 1, 1};
        st = encode_bf16(&o.tmap_a, 4, base, dims, strides, box, estr, CU_TENSOR_MAP_SWIZZLE_128B, o.desc + " A");
        if (st != HAPI_OK) return st;
      } else if (o.tc_mode == 6) {
        void* base = vptr(m, p, o.in, nullptr);
        const cuuint64_t ld = (cuuint64_t)o.in.ld * 2;
        const int we = o.out.W + w.kw - 1;
        cuuint64_t dims[4] = {(cuuint64_t)w.cs, (cuuint64_t)o.in.W, (cuuint64_t)o.in.H, (cuuint64_t)m->d.max_batch};
        cuuint64_t strides[3] = {ld, ld * o.in.W, ld * o.in.W * o.in.H};
        cuuint32_t box[4] = {64, (cuuint32_t)we, (cuuint32_t)(o.hb + w.kh - 1), 1};
        cuuint32_t estr[4] = {1, 1, 1, 1};
        st = encode_bf16(&o.tmap_a, 4, base, dims, strides, box, estr, CU_TENSOR_MAP_SWIZZLE_128B, o.desc + " halo");
        if (st != HAPI_OK) return st;
      } else if (o.tc_mode == 5) {
        if ((st = encode_im2col(m, vptr(m, p, o.in, nullptr), o.in, w.cs, w.kh, w.kw, w.stride, w.pad, &o.tmap_a,
                                o.desc + " A im2col")) != HAPI_OK)
          return st;
      } else if (o.tc_mode == 3 || o.tc_mode == 4 || o.tc_mode == 7) {
        void* base = vptr(m, p, o.in, nullptr);
        const cuuint64_t es = 2, ld = (cuuint64_t)o.in.ld;
        if (o.tc_mode == 3 || o.tc_mode == 7) {
          cuuint64_t dims[2] = {(cuuint64_t)w.cs, (cuuint64_t)m->d.max_batch * o.in.H * o.in.W};
          cuuint64_t strides[1] = {ld * es};
          cuuint32_t box[2] = {64, 128};
          cuuint32_t estr[2] = {1, 1};
          st = encode_bf16(&o.tmap_a, 2, base, dims, strides, box, estr, CU_TENSOR_MAP_SWIZZLE_128B, o.desc + " A");
        } else {
          const cuuint32_t sd = (cuuint32_t)w.stride;
          cuuint64_t dims[4] = {(cuuint64_t)w.cs, (cuuint64_t)o.in.W, (cuuint64_t)o.in.H, (cuuint64_t)m->d.max_batch};
          cuuint64_t strides[3] = {ld * es, ld * es * o.in.W, ld * es * o.in.W * o.in.H};
          cuuint32_t box[4] = {64, (cuuint32_t)o.wb * sd, (cuuint32_t)o.hb * sd, (cuuint32_t)o.nb};
          cuuint32_t estr[4] = {1, sd, sd, 1};
          st = encode_bf16(&o.tmap_a, 4, base, dims, strides, box, estr, CU_TENSOR_MAP_SWIZZLE_128B, o.desc + " A");
        }
        if (st != HAPI_OK) return st;
      }
      if (o.dual && o.tc_mode == 5) {
        if ((st = encode_im2col(m, vptr(m, p, o.in2, nullptr), o.in2, w.cs2, 1, 1, o.in2_stride ? o.in2_stride : w.stride2, 0, &o.tmap_a2,
                                o.desc + " A2 im2col")) != HAPI_OK)
          return st;
      } else if (o.dual) {
        void* base2 = vptr(m, p, o.in2, nullptr);
        const cuuint64_t ld2 = (cuuint64_t)o.in2.ld * 2;
        if (o.tc_mode == 3) {
          cuuint64_t dims[2] = {(cuuint64_t)w.cs2, (cuuint64_t)m->d.max_batch * o.in2.H * o.in2.W};
          cuuint64_t strides[1] = {ld2};
          cuuint32_t box[2] = {64, 128};
          cuuint32_t estr[2] = {1, 1};
          st = encode_bf16(&o.tmap_a2, 2, base2, dims, strides, box, estr, CU_TENSOR_MAP_SWIZZLE_128B, o.desc + " A2");
        } else {
          const cuuint32_t sd = (cuuint32_t)(o.in2_stride ? o.in2_stride : w.stride2);
          cuuint64_t dims[4] = {(cuuint64_t)w.cs2, (cuuint64_t)o.in2.W, (cuuint64_t)o.in2.H, (cuuint64_t)m->d.max_batch};
          cuuint64_t strides[3] = {ld2, ld2 * o.in2.W, ld2 * o.in2.W * o.in2.H};
          cuuint32_t box[4] = {64, (cuuint32_t)o.wb * sd, (cuuint32_t)o.hb * sd, (cuuint32_t)o.nb};
          cuuint32_t estr[4] = {1, sd, sd, 1};
          st = encode_bf16(&o.tmap_a2, 4, base2, dims, strides, box, estr, CU_TENSOR_MAP_SWIZZLE_128B, o.desc + " A2");
        }
        if (st != HAPI_OK) return st;
      }
      if (!o.nchw_out && o.tc_mode != 8) {
        const int cols = conv_tc_store_cols(w.bn);
        if ((st = encode_view(m, p, o, o.out, cols, &o.tmap_y, "Y", o.t == OP_PAIR ? 32 : 128)) != HAPI_OK) return st;
        if (o.t == OP_CONV && o.tc_mode == 3) {
          // 1x1 tiles: per-warp [32 rows x 32 channels] store boxes
          void* base = vptr(m, p, o.out, nullptr);
          cuuint64_t dims[2] = {(cuuint64_t)o.out.C, (cuuint64_t)m->d.max_batch * o.out.H * o.out.W};
          cuuint64_t strides[1] = {(cuuint64_t)o.out.ld * 2};
          cuuint32_t box[2] = {32, 32};
          cuuint32_t estr[2] = {1, 1};
          if ((st = encode_bf16(&o.tmap_yw, 2, base, dims, strides, box, estr, CU_TENSOR_MAP_SWIZZLE_64B,
                                o.desc + " Yw")) != HAPI_OK)
            return st;
          o.has_yw = true;
        }
        if (o.has_res && (st = encode_view(m, p, o, o.res, cols, &o.tmap_r, "R")) != HAPI_OK) return st;
      }
    }
  }
  return HAPI_OK;
}

bool graphs_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("HAPI_GRAPH");
    return !(e && e[0] == '0');
  }();
  return on;
}

// One chunk through the plan, replayed from a cached CUDA graph (captured on first use;
// PDL attributes become programmatic edges).  Falls back to direct launches if capture fails.
hapi_status run_chunk_graph(hapi_model* m, const Plan& p, int nb, const void* images, bool in_u8, void* out) {
  if (!graphs_enabled()) return run_chunk(m, p, nb, images, in_u8, out, m->stream);
  for (auto& g : m->graphs)
    if (g.split == (uint32_t)p.split && g.nb == nb && g.u8 == in_u8 && g.images == images && g.out == out) {
      HAPI_CUDA_TRY(cudaGraphLaunch(g.exec, m->stream));
      return HAPI_OK;
    }
  if (!m->cap_stream) HAPI_CUDA_TRY(cudaStreamCreateWithFlags(&m->cap_stream, cudaStreamNonBlocking));
  HAPI_CUDA_TRY(cudaStreamBeginCapture(m->cap_stream, cudaStreamCaptureModeThreadLocal));
  hapi_status st = run_chunk(m, p, nb, images, in_u8, out, m->cap_stream);
  cudaGraph_t graph = nullptr;
  cudaError_t e = cudaStreamEndCapture(m->cap_stream, &graph);
  if (st != HAPI_OK) {
    if (graph) cudaGraphDestroy(graph);
    return st;
  }
  if (e != cudaSuccess) return set_error(HAPI_ERR_CUDA, "graph capture: %s", cudaGetErrorString(e));
  // Same (split, chunk size) with other buffers (the serving case: a caching allocator hands
  // out new pointers): the topology is identical, so update that executable graph's kernel
  // parameters in place instead of instantiating another one.
  for (auto& g : m->graphs) {
    if (g.split != (uint32_t)p.split || g.nb != nb || g.u8 != in_u8) continue;
    cudaGraphExecUpdateResultInfo info;
    if (cudaGraphExecUpdate(g.exec, graph, &info) == cudaSuccess) {
      cudaGraphDestroy(graph);
      g.images = images;
      g.out = out;
      HAPI_CUDA_TRY(cudaGraphLaunch(g.exec, m->stream));
      return HAPI_OK;
    }
    cudaGetLastError();  // a refused update is not an error: instantiate below
    break;
  }
  cudaGraphExec_t exec = nullptr;
  e = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) return set_error(HAPI_ERR_CUDA, "graph instantiate: %s", cudaGetErrorString(e));
  if (m->graphs.size() >= 16) {
    cudaGraphExecDestroy(m->graphs.front().exec);
    m->graphs.erase(m->graphs.begin());
  }
  m->graphs.push_back({(uint32_t)p.split, nb, in_u8, images, out, exec});
  HAPI_CUDA_TRY(cudaGraphLaunch(exec, m->stream));
  return HAPI_OK;
}

const Plan* get_plan(hapi_model* m, uint32_t split) {
  if (split < m->d.min_split || split > m->d.max_split) return nullptr;
  return &m->plans[split - m->d.min_split];
}

// Host path (f2): two staging slots of host_chunk images in and split outputs out, plus the
// copy streams and events, all made at create time so hapi_prefix_forward_host never
// allocates and hapi_model_device_bytes reports them.
hapi_status host_setup(hapi_model* m) {
  const uint32_t c = std::min<uint32_t>(m->d.host_chunk, m->d.max_batch);
  const int64_t img_bytes = 12ll * m->d.in_h * m->d.in_w;
  int64_t max_out = 0;
  for (const Plan& q : m->plans) max_out = std::max(max_out, q.out_bytes_per_img);
  HAPI_CUDA_TRY(cudaStreamCreateWithFlags(&m->copy_stream, cudaStreamNonBlocking));
  HAPI_CUDA_TRY(cudaStreamCreateWithFlags(&m->out_stream, cudaStreamNonBlocking));
  for (auto& e : m->ev) HAPI_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  m->host_ready = true;  // streams/events exist: destroy releases them
  for (int k = 0; k < 2; ++k) {
    hapi_status st = dev_alloc(m, (size_t)img_bytes * c, &m->stage_in[k], false);
    if (st == HAPI_OK) st = dev_alloc(m, (size_t)max_out * c, &m->stage_out[k], false);
    if (st != HAPI_OK) return st;
  }
  m->host_chunk = c;
  m->stage_bytes = 2 * ((int64_t)img_bytes * c + max_out * c);
  return HAPI_OK;
}

// One launch plan per split in [min_split, max_split] (two candidates each: pool written
// straight into the DenseNet block buffer, or through a compact buffer + copy; the smaller
// arena is kept), then the arena, the TMA descriptors over it and the host-path staging.
hapi_status plans_and_arena(hapi_model* m) {
  for (uint32_t s = m->d.min_split; s <= m->d.max_split; ++s) {
    Plan p, p2;
    hapi_status st = build_plan(m, (int)s, &p, true);
    if (st == HAPI_OK) st = build_plan(m, (int)s, &p2, false);
    if (st != HAPI_OK) return st;
    if (p2.arena_bytes < p.arena_bytes) p = std::move(p2);
    m->arena_bytes = std::max(m->arena_bytes, p.arena_bytes);
    m->plans.push_back(std::move(p));
  }
  hapi_status st = dev_alloc(m, (size_t)m->arena_bytes, &m->arena, false);
  if (st == HAPI_OK) st = finalize_tmaps(m);
  if (st == HAPI_OK && m->start == 0 && m->d.host_chunk > 0) st = host_setup(m);
  return st;
}

}  // namespace

extern "C" {

static hapi_status create_impl(const hapi_model_desc* desc, uint32_t start, const float* const* params,
                               uint32_t n_params, hapi_model** out);

hapi_status hapi_model_create(const hapi_model_desc* desc, const float* const* params, uint32_t n_params, hapi_model** out) {
  return create_impl(desc, 0, params, n_params, out);
}

hapi_status hapi_model_create_suffix(const hapi_model_desc* desc, uint32_t start_idx, const float* const* params,
                                     uint32_t n_params, hapi_model** out) {
  clear_error();
  if (!desc) return set_error(HAPI_ERR_INVALID_ARGUMENT, "null desc");
  if (start_idx < 1 || start_idx >= desc->min_split)
    return set_error(HAPI_ERR_INVALID_ARGUMENT, "start_idx %u must be in [1, min_split)", start_idx);
  return create_impl(desc, start_idx, params, n_params, out);
}

static hapi_status create_impl(const hapi_model_desc* desc, uint32_t start, const float* const* params,
                               uint32_t n_params, hapi_model** out) {
  clear_error();
  if (!desc || !out || (!params && n_params)) return set_error(HAPI_ERR_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  const ArchDesc* A = get_arch(desc->arch);
  if (!A) return set_error(HAPI_ERR_INVALID_MODEL, "unknown arch %d", (int)desc->arch);
  if (desc->act != HAPI_F32 && desc->act != HAPI_BF16) return set_error(HAPI_ERR_INVALID_ARGUMENT, "dtype");
  const uint32_t L = (uint32_t)A->mods.size();
  if (desc->min_split < 1 || desc->min_split > desc->max_split || desc->max_split > L)
    return set_error(HAPI_ERR_INVALID_ARGUMENT, "split range [%u,%u] not within [1,%u]", desc->min_split, desc->max_split, L);
  if (desc->max_batch < 1) return set_error(HAPI_ERR_INVALID_ARGUMENT, "max_batch = 0");
  if (n_params != A->params.size())
    return set_error(HAPI_ERR_INVALID_MODEL, "n_params %u != %zu", n_params, A->params.size());
  for (uint32_t k = 0; k < n_params; ++k)
    if (!params[k]) return set_error(HAPI_ERR_INVALID_ARGUMENT, "params[%u] is null", k);
  // shape validity at this image size
  int64_t in_numel = 3ll * desc->in_h * desc->in_w;
  {
    Shape s{3, (int)desc->in_h, (int)desc->in_w, false};
    for (uint32_t k = 0; k < desc->max_split; ++k) {
      bool ok;
      s = infer(A->mods[k], s, &ok);
      if (!ok) return set_error(HAPI_ERR_INVALID_MODEL, "layer %s empty at %ux%u", A->mods[k].name.c_str(), desc->in_h, desc->in_w);
      if (k + 1 == start) in_numel = s.numel();
    }
  }
  int ndev = 0;
  HAPI_CUDA_TRY(cudaGetDeviceCount(&ndev));
  if (desc->device < 0 || desc->device >= ndev) return set_error(HAPI_ERR_INVALID_ARGUMENT, "device %d", desc->device);
  DeviceGuard dg(desc->device);
  std::unique_ptr<hapi_model> m(new hapi_model());
  m->wstore = std::make_shared<WeightStore>();
  m->wstore->device = desc->device;
  m->d = *desc;
  m->arch = A;
  m->bf16 = desc->act == HAPI_BF16;
  m->es = m->bf16 ? 2 : 4;
  m->start = start;
  m->in_bytes_per_img = start ? in_numel * m->es : in_numel * 4;
  HAPI_CUDA_TRY(cudaDeviceGetAttribute(&m->num_sms, cudaDevAttrMultiProcessorCount, desc->device));
  if (m->bf16) {
    int major = 0, minor = 0;
    HAPI_CUDA_TRY(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, desc->device));
    HAPI_CUDA_TRY(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, desc->device));
    if (major != 10 || minor != 0)
      return set_error(HAPI_ERR_UNSUPPORTED, "bf16 tcgen05 path is built for sm_100a; device is sm_%d%d", major, minor);
  }
  m->host_params.assign(params, params + n_params);
  hapi_status st = plans_and_arena(m.get());
  m->host_params.clear();
  if (st != HAPI_OK) {
    hapi_model_destroy(m.release());
    return st;
  }
  *out = m.release();
  return HAPI_OK;
}

hapi_status hapi_model_create_shared(const hapi_model* base, uint32_t max_batch, uint32_t host_chunk, hapi_model** out) {
  clear_error();
  if (!base || !out) return set_error(HAPI_ERR_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  if (max_batch < 1) return set_error(HAPI_ERR_INVALID_ARGUMENT, "max_batch = 0");
  DeviceGuard dg(base->d.device);
  std::unique_ptr<hapi_model> m(new hapi_model());
  m->wstore = base->wstore;  // weights shared, freed with the last model holding them
  m->d = base->d;
  m->d.max_batch = max_batch;
  m->d.host_chunk = host_chunk;
  m->arch = base->arch;
  m->bf16 = base->bf16;
  m->es = base->es;
  m->num_sms = base->num_sms;
  m->start = base->start;
  m->in_bytes_per_img = base->in_bytes_per_img;
  m->convs = base->convs;            // device pointers into the shared store
  m->conv_index = base->conv_index;  // every conv of the plans is found here (no host params)
  m->bn_cache = base->bn_cache;
  m->ident = base->ident;
  m->ident_map128 = base->ident_map128;
  m->ident_map256 = base->ident_map256;
  hapi_status st = plans_and_arena(m.get());
  if (st != HAPI_OK) {
    hapi_model_destroy(m.release());
    return st;
  }
  *out = m.release();
  return HAPI_OK;
}

hapi_status hapi_model_set_stream(hapi_model* m, void* s) {
  clear_error();
  if (!m) return set_error(HAPI_ERR_INVALID_ARGUMENT, "null model");
  m->stream = static_cast<cudaStream_t>(s);
  return HAPI_OK;
}

hapi_status hapi_suffix_forward(hapi_model* m, uint32_t end_idx, const void* acts, uint64_t batch, void* out) {
  clear_error();
  if (!m || !acts || !out) return set_error(HAPI_ERR_INVALID_ARGUMENT, "null argument");
  if (m->start == 0) return set_error(HAPI_ERR_INVALID_ARGUMENT, "not a suffix model (use hapi_prefix_forward)");
  if (batch == 0) return set_error(HAPI_ERR_INVALID_ARGUMENT, "batch = 0");
  DeviceGuard dg(m->d.device);
  const Plan* p = get_plan(m, end_idx);
  if (!p) return set_error(HAPI_ERR_INVALID_ARGUMENT, "end_idx %u outside [%u,%u]", end_idx, m->d.min_split, m->d.max_split);
  HAPI_CUDA_TRY(cudaGetLastError());
  const bool use_graph = (batch + m->d.max_batch - 1) / m->d.max_batch <= 4;
  for (uint64_t c0 = 0; c0 < batch; c0 += m->d.max_batch) {
    const int nb = (int)std::min<uint64_t>(m->d.max_batch, batch - c0);
    const float* ci = reinterpret_cast<const float*>(static_cast<const char*>(acts) + c0 * m->in_bytes_per_img);
    void* co = static_cast<char*>(out) + c0 * p->out_bytes_per_img;
    hapi_status st = use_graph ? run_chunk_graph(m, *p, nb, ci, false, co) : run_chunk(m, *p, nb, ci, false, co, m->stream);
    if (st != HAPI_OK) return st;
  }
  return HAPI_OK;
}

static hapi_status prefix_forward_impl(hapi_model* m, uint32_t split_idx, const void* images, bool in_u8, uint64_t batch,
                                       void* out) {
  clear_error();
  if (!m || !images || !out) return set_error(HAPI_ERR_INVALID_ARGUMENT, "null argument");
  if (m->start != 0) return set_error(HAPI_ERR_INVALID_ARGUMENT, "suffix model: use hapi_suffix_forward");
  if (batch == 0) return set_error(HAPI_ERR_INVALID_ARGUMENT, "batch = 0");
  DeviceGuard dg(m->d.device);
  const Plan* p = get_plan(m, split_idx);
  if (!p) return set_error(HAPI_ERR_INVALID_ARGUMENT, "split_idx %u outside [%u,%u]", split_idx, m->d.min_split, m->d.max_split);
  HAPI_CUDA_TRY(cudaGetLastError());
  const int64_t img_bytes = 3ll * m->d.in_h * m->d.in_w * (in_u8 ? 1 : 4);
  // graphs are keyed by the chunk's pointers: replay them for calls of up to a few chunks,
  // launch directly when a large call would only thrash the cache
  const bool use_graph = (batch + m->d.max_batch - 1) / m->d.max_batch <= 4;
  for (uint64_t c0 = 0; c0 < batch; c0 += m->d.max_batch) {
    const int nb = (int)std::min<uint64_t>(m->d.max_batch, batch - c0);
    const void* ci = static_cast<const char*>(images) + c0 * img_bytes;
    void* co = static_cast<char*>(out) + c0 * p->out_bytes_per_img;
    hapi_status st = use_graph ? run_chunk_graph(m, *p, nb, ci, in_u8, co) : run_chunk(m, *p, nb, ci, in_u8, co, m->stream);
    if (st != HAPI_OK) return st;
  }
  return HAPI_OK;
}

hapi_status hapi_prefix_forward(hapi_model* m, uint32_t split_idx, const float* images, uint64_t batch, void* out) {
  return prefix_forward_impl(m, split_idx, images, false, batch, out);
}

hapi_status hapi_prefix_forward_u8(hapi_model* m, uint32_t split_idx, const uint8_t* images, uint64_t batch, void* out) {
  return prefix_forward_impl(m, split_idx, images, true, batch, out);
}

hapi_status hapi_model_set_u8_norm(hapi_model* m, const float* scale, const float* shift) {
  clear_error();
  if (!m || !scale || !shift) return set_error(HAPI_ERR_INVALID_ARGUMENT, "null argument");
  for (int c = 0; c < 3; ++c)
    if (!std::isfinite(scale[c]) || !std::isfinite(shift[c]))
      return set_error(HAPI_ERR_INVALID_ARGUMENT, "non-finite scale/shift");
  DeviceGuard dg(m->d.device);
  // captured graphs hold the old values as kernel parameters: no call may still be replaying them
  HAPI_CUDA_TRY(cudaStreamSynchronize(m->stream));
  for (int c = 0; c < 3; ++c) {
    m->u8norm.scale[c] = scale[c];
    m->u8norm.shift[c] = shift[c];
  }
  for (auto& g : m->graphs)
    if (g.u8) cudaGraphExecDestroy(g.exec);
  m->graphs.erase(std::remove_if(m->graphs.begin(), m->graphs.end(), [](const hapi_model::GraphEntry& g) { return g.u8; }),
                  m->graphs.end());
  return HAPI_OK;
}

hapi_status hapi_prefix_forward_timed(hapi_model* m, uint32_t split_idx, const float* images, uint64_t batch, void* out,
                                      float* ms, uint32_t cap) {
  clear_error();
  if (!m || !images || !out) return set_error(HAPI_ERR_INVALID_ARGUMENT, "null argument");
  if (m->start != 0) return set_error(HAPI_ERR_INVALID_ARGUMENT, "suffix model: use hapi_suffix_forward");
  if (batch == 0 || batch > m->d.max_batch) return set_error(HAPI_ERR_INVALID_ARGUMENT, "batch must be in [1, max_batch]");
  DeviceGuard dg(m->d.device);
  const Plan* p = get_plan(m, split_idx);
  if (!p) return set_error(HAPI_ERR_INVALID_ARGUMENT, "split_idx %u outside [%u,%u]", split_idx, m->d.min_split, m->d.max_split);
  std::vector<cudaEvent_t> evs(p->ops.size() + 1);
  for (auto& e : evs) HAPI_CUDA_TRY(cudaEventCreate(&e));
  hapi_status st = run_chunk(m, *p, (int)batch, images, false, out, m->stream, evs.data());
  if (st == HAPI_OK) {
    cudaError_t e = cudaEventSynchronize(evs.back());
    if (e != cudaSuccess) st = set_error(HAPI_ERR_CUDA, "sync: %s", cudaGetErrorString(e));
  }
  if (st == HAPI_OK && ms)
    for (size_t k = 0; k < p->ops.size() && k < cap; ++k) cudaEventElapsedTime(&ms[k], evs[k], evs[k + 1]);
  for (auto& e : evs) cudaEventDestroy(e);
  return st;
}

static hapi_status forward_host_enqueue(hapi_model* m, uint32_t split_idx, const void* images, bool in_u8,
                                        uint64_t batch, void* out, bool ramp_fill);

hapi_status hapi_prefix_forward_host(hapi_model* m, uint32_t split_idx, const float* images, uint64_t batch, void* out) {
  hapi_status st = forward_host_enqueue(m, split_idx, images, false, batch, out, true);
  if (st != HAPI_OK) return st;
  return hapi_host_sync(m);
}

hapi_status hapi_prefix_forward_host_async(hapi_model* m, uint32_t split_idx, const float* images, uint64_t batch,
                                           void* out) {
  // (no half-size first chunk: in a stream of calls the H2D of this call's first chunk overlaps
  // the previous call's compute, so the fill the ramp shortens is not exposed)
  return forward_host_enqueue(m, split_idx, images, false, batch, out, false);
}

hapi_status hapi_prefix_forward_host_u8(hapi_model* m, uint32_t split_idx, const uint8_t* images, uint64_t batch,
                                        void* out) {
  hapi_status st = forward_host_enqueue(m, split_idx, images, true, batch, out, true);
  if (st != HAPI_OK) return st;
  return hapi_host_sync(m);
}

hapi_status hapi_prefix_forward_host_async_u8(hapi_model* m, uint32_t split_idx, const uint8_t* images, uint64_t batch,
                                              void* out) {
  return forward_host_enqueue(m, split_idx, images, true, batch, out, false);
}

hapi_status hapi_host_sync(hapi_model* m) {
  clear_error();
  if (!m) return set_error(HAPI_ERR_INVALID_ARGUMENT, "null model");
  if (!m->host_ready) return HAPI_OK;
  DeviceGuard dg(m->d.device);
  HAPI_CUDA_TRY(cudaStreamSynchronize(m->copy_stream));
  HAPI_CUDA_TRY(cudaStreamSynchronize(m->out_stream));
  HAPI_CUDA_TRY(cudaStreamSynchronize(m->stream));
  return HAPI_OK;
}

static hapi_status forward_host_enqueue(hapi_model* m, uint32_t split_idx, const void* images, bool in_u8,
                                        uint64_t batch, void* out, bool ramp_fill) {
  clear_error();
  if (!m || !images || !out) return set_error(HAPI_ERR_INVALID_ARGUMENT, "null argument");
  if (m->start != 0) return set_error(HAPI_ERR_INVALID_ARGUMENT, "suffix model: use hapi_suffix_forward");
  if (batch == 0) return set_error(HAPI_ERR_INVALID_ARGUMENT, "batch = 0");
  const Plan* p = get_plan(m, split_idx);
  if (!p) return set_error(HAPI_ERR_INVALID_ARGUMENT, "split_idx %u outside [%u,%u]", split_idx, m->d.min_split, m->d.max_split);
  if (m->host_chunk == 0)
    return set_error(HAPI_ERR_INVALID_ARGUMENT, "model created with host_chunk = 0 (no host-path staging)");
  DeviceGuard dg(m->d.device);
  const int64_t img_bytes = 3ll * m->d.in_h * m->d.in_w * (in_u8 ? 1 : 4);  // (staging slots are fp32-sized)
  // ev[0..1] h2d done, ev[2..3] compute done, ev[4..5] d2h done (slot reuse)
  cudaStream_t cs = m->stream, xs = m->copy_stream, ys = m->out_stream;
  // sub-chunks so the H2D copy of chunk i+1 and the D2H of chunk i-1 overlap compute of chunk i
  // (H2D and D2H on their own streams: PCIe is full duplex).  Chunk = the staging slot
  // (create time; ~3/16 of a 512 batch measured best on ResNet-50)
  uint64_t B = m->host_chunk;
  if (const char* e = std::getenv("HAPI_HOST_CHUNK")) B = std::min<uint64_t>(B, std::max(1, std::atoi(e)));
  // chunk schedule: a half-size first chunk (its H2D copy is the pipeline fill nothing overlaps),
  // then full chunks, the remainder last (HAPI_HOST_RAMP=0: equal chunks)
  std::vector<uint64_t> sizes;
  {
    static const bool ramp = [] {
      const char* e = std::getenv("HAPI_HOST_RAMP");
      return !(e && e[0] == '0');
    }();
    uint64_t left = batch;
    if (ramp_fill && ramp && B >= 32 && batch >= 2 * B) {
      sizes.push_back(B / 2);
      left -= B / 2;
    }
    while (left > 0) {
      sizes.push_back(std::min<uint64_t>(B, left));
      left -= sizes.back();
    }
  }
  const uint64_t nchunks = sizes.size();
  uint64_t c0 = 0;
  // chunk numbering continues across calls (host_seq), so consecutive asynchronous calls keep
  // alternating the two staging slots and wait on the chunk that last used a slot -- the H2D of
  // the next call's first chunk overlaps the compute of this call's last one
  for (uint64_t c = 0; c < nchunks; c0 += sizes[c], ++c) {
    const uint64_t gc = m->host_seq++;
    const int k = (int)(gc & 1);
    const int nb = (int)sizes[c];
    if (gc >= 2) HAPI_CUDA_TRY(cudaStreamWaitEvent(xs, m->ev[2 + k], 0));  // stage_in[k] free once chunk gc-2 computed
    HAPI_CUDA_TRY(cudaMemcpyAsync(m->stage_in[k], reinterpret_cast<const char*>(images) + c0 * img_bytes,
                                  (size_t)nb * img_bytes, cudaMemcpyHostToDevice, xs));
    HAPI_CUDA_TRY(cudaEventRecord(m->ev[k], xs));
    HAPI_CUDA_TRY(cudaStreamWaitEvent(cs, m->ev[k], 0));
    if (gc >= 2) HAPI_CUDA_TRY(cudaStreamWaitEvent(cs, m->ev[4 + k], 0));  // stage_out[k] drained
    hapi_status st = run_chunk_graph(m, *p, nb, m->stage_in[k], in_u8, m->stage_out[k]);
    if (st != HAPI_OK) return st;
    HAPI_CUDA_TRY(cudaEventRecord(m->ev[2 + k], cs));
    HAPI_CUDA_TRY(cudaStreamWaitEvent(ys, m->ev[2 + k], 0));
    HAPI_CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(out) + c0 * p->out_bytes_per_img, m->stage_out[k],
                                  (size_t)nb * p->out_bytes_per_img, cudaMemcpyDeviceToHost, ys));
    HAPI_CUDA_TRY(cudaEventRecord(m->ev[4 + k], ys));
  }
  return HAPI_OK;
}

hapi_status hapi_model_device_bytes(const hapi_model* m, uint64_t* wb, uint64_t* ab) {
  clear_error();
  if (!m) return set_error(HAPI_ERR_INVALID_ARGUMENT, "null model");
  if (wb) *wb = (uint64_t)m->weight_bytes;
  if (ab) *ab = (uint64_t)(m->arena_bytes + m->stage_bytes);
  return HAPI_OK;
}

hapi_status hapi_plan_describe(const hapi_model* m, uint32_t split_idx, uint32_t op, char* buf, uint32_t cap) {
  clear_error();
  if (!m || !buf || cap == 0) return set_error(HAPI_ERR_INVALID_ARGUMENT, "null argument");
  if (split_idx < m->d.min_split || split_idx > m->d.max_split) return set_error(HAPI_ERR_INVALID_ARGUMENT, "split_idx");
  const Plan& p = m->plans[split_idx - m->d.min_split];
  if (op >= p.ops.size()) return set_error(HAPI_ERR_INVALID_ARGUMENT, "op index");
  static const char* names[] = {"pack_in", "conv", "pool", "adaptive_avgpool", "bn_act", "pack_out", "pair", "unpack", "block"};
  const Op& o = p.ops[op];
  std::snprintf(buf, cap, "%s%s%s", o.desc.empty() ? names[o.t] : o.desc.c_str(), o.out.buf < 0 ? " ->out" : "",
                o.nchw_out ? "(nchw)" : "");
  return HAPI_OK;
}

hapi_status hapi_plan_info(const hapi_model* m, uint32_t split_idx, uint32_t* n, uint32_t* kind, double* flops,
                           double* bytes, uint32_t cap) {
  clear_error();
  if (!m || !n) return set_error(HAPI_ERR_INVALID_ARGUMENT, "null argument");
  if (split_idx < m->d.min_split || split_idx > m->d.max_split) return set_error(HAPI_ERR_INVALID_ARGUMENT, "split_idx");
  const Plan& p = m->plans[split_idx - m->d.min_split];
  *n = (uint32_t)p.ops.size();
  for (size_t k = 0; k < p.ops.size() && k < cap; ++k) {
    if (kind) kind[k] = p.ops[k].kind;
    if (flops) flops[k] = p.ops[k].flops;
    if (bytes) bytes[k] = p.ops[k].bytes;
  }
  return HAPI_OK;
}

void hapi_model_destroy(hapi_model* m) {
  if (!m) return;
  DeviceGuard dg(m->d.device);
  for (auto& g : m->graphs) cudaGraphExecDestroy(g.exec);
  if (m->cap_stream) cudaStreamDestroy(m->cap_stream);
  if (m->host_ready) {
    cudaStreamSynchronize(m->copy_stream);
    cudaStreamSynchronize(m->out_stream);
    for (auto& e : m->ev) cudaEventDestroy(e);
    cudaStreamDestroy(m->copy_stream);
    cudaStreamDestroy(m->out_stream);
  }
  for (void* p : m->allocs) cudaFree(p);
  delete m;
}

const char* hapi_last_error(void) { return last_error_cstr(); }

const char* hapi_build_info(void) {
  return "hapi-b200 (sm_100a tcgen05/TMEM/TMA implicit-GEMM conv; fp32 SIMT path); built " __DATE__ " " __TIME__;
}

}  // extern "C"
