// Arch descriptors: canonical layer lists (reading R2), parameter specs in
// torchvision state_dict order, and closed-form shape inference.  Host-only.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "hapi.h"

namespace hapi {

enum ModKind {
  MK_CONV,        // Conv2d (+bias)
  MK_BN,          // BatchNorm2d (eval)
  MK_RELU,
  MK_MAXPOOL,
  MK_AVGPOOL,     // DenseNet transition pool (2x2/s2)
  MK_ADAPTIVE,    // AdaptiveAvgPool2d(oh, ow)
  MK_DROPOUT,     // identity; flattens (first classifier module)
  MK_LINEAR,
  MK_BASIC,       // ResNet BasicBlock (atomic)
  MK_BOTTLENECK,  // ResNet Bottleneck (atomic)
  MK_DENSEBLOCK,  // DenseNet _DenseBlock (atomic)
  MK_DENSE_CLS    // relu -> adaptive_avg_pool(1) -> flatten -> linear
};

struct Shape {
  int c = 0, h = 0, w = 0;
  bool flat = false;  // [F] with F = c (h = w = 1)
  int64_t numel() const { return flat ? (int64_t)c : (int64_t)c * h * w; }
};

struct ModDesc {
  ModKind kind;
  std::string name;
  int cin = 0, cout = 0, k = 0, stride = 1, pad = 0;
  bool bias = false;
  int planes = 0;       // ResNet blocks
  bool ds = false;      // ResNet downsample branch
  int nlayers = 0;      // dense block
  int growth = 32, bn_size = 4;
  int oh = 0, ow = 0;   // adaptive pool
  int first_param = 0;  // index of the module's first param in the arch param list
  int64_t weight_elems = 0, vec_elems = 0;  // for W(s)
};

struct ParamSpec {
  std::string name;
  int ndim;
  int64_t dims[4];
  int64_t numel() const {
    int64_t n = 1;
    for (int i = 0; i < ndim; ++i) n *= dims[i];
    return n;
  }
};

struct ArchDesc {
  hapi_arch arch;
  int freeze;
  std::vector<ModDesc> mods;
  std::vector<ParamSpec> params;
  int find_param(const std::string& name) const;
};

// Returns nullptr for an unknown arch.  Descriptors are built once and cached.
const ArchDesc* get_arch(hapi_arch arch);

// Output shape of module m given its input shape; ok=false if an output dim <= 0
// or the input does not match.
Shape infer(const ModDesc& m, const Shape& in, bool* ok);

int out_dim(int in, int k, int stride, int pad);

}  // namespace hapi
