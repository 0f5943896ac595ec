// Canonical layer lists of AlexNet, ResNet18/50, VGG11 and DenseNet121 (torchvision
// definitions; block-atomic "split at block boundary", Table 2 PAPER.md:939;
// DESIGN.md reading R2), with parameters registered in torchvision state_dict order.
#include "arch.h"

#include <mutex>

namespace hapi {

int out_dim(int in, int k, int stride, int pad) {
  int num = in + 2 * pad - k;
  if (num < 0) return 0;
  return num / stride + 1;
}

int ArchDesc::find_param(const std::string& name) const {
  for (size_t i = 0; i < params.size(); ++i)
    if (params[i].name == name) return (int)i;
  return -1;
}

namespace {

struct Builder {
  ArchDesc a;
  void p1(const std::string& n, int64_t d0) { a.params.push_back({n, 1, {d0, 0, 0, 0}}); }
  void p2(const std::string& n, int64_t d0, int64_t d1) { a.params.push_back({n, 2, {d0, d1, 0, 0}}); }
  void p4(const std::string& n, int64_t o, int64_t i, int64_t k) { a.params.push_back({n, 4, {o, i, k, k}}); }
  void bn_params(const std::string& n, int c) {
    p1(n + ".weight", c); p1(n + ".bias", c); p1(n + ".running_mean", c); p1(n + ".running_var", c);
  }
  void conv_params(const std::string& n, int cin, int cout, int k, bool bias) {
    p4(n + ".weight", cout, cin, k);
    if (bias) p1(n + ".bias", cout);
  }
  ModDesc& push(ModDesc m) {
    a.mods.push_back(m);
    return a.mods.back();
  }
  void conv(const std::string& n, int cin, int cout, int k, int s, int p, bool bias) {
    ModDesc m{MK_CONV, n};
    m.cin = cin; m.cout = cout; m.k = k; m.stride = s; m.pad = p; m.bias = bias;
    m.first_param = (int)a.params.size();
    m.weight_elems = (int64_t)cout * cin * k * k;
    m.vec_elems = bias ? cout : 0;
    conv_params(n, cin, cout, k, bias);
    push(m);
  }
  void bn(const std::string& n, int c) {
    ModDesc m{MK_BN, n};
    m.cin = m.cout = c;
    m.first_param = (int)a.params.size();
    m.vec_elems = 2 * c;
    bn_params(n, c);
    push(m);
  }
  void simple(ModKind k, const std::string& n) { push(ModDesc{k, n}); }
  void pool(ModKind kind, const std::string& n, int k, int s, int p) {
    ModDesc m{kind, n};
    m.k = k; m.stride = s; m.pad = p;
    push(m);
  }
  void adaptive(const std::string& n, int oh, int ow) {
    ModDesc m{MK_ADAPTIVE, n};
    m.oh = oh; m.ow = ow;
    push(m);
  }
  void linear(const std::string& n, int fin, int fout) {
    ModDesc m{MK_LINEAR, n};
    m.cin = fin; m.cout = fout; m.bias = true;
    m.first_param = (int)a.params.size();
    m.weight_elems = (int64_t)fin * fout;
    m.vec_elems = fout;
    p2(n + ".weight", fout, fin); p1(n + ".bias", fout);
    push(m);
  }
};

ArchDesc build_alexnet() {
  Builder b;
  b.a.arch = HAPI_ALEXNET; b.a.freeze = 17;
  b.conv("features.0", 3, 64, 11, 4, 2, true); b.simple(MK_RELU, "features.1");
  b.pool(MK_MAXPOOL, "features.2", 3, 2, 0);
  b.conv("features.3", 64, 192, 5, 1, 2, true); b.simple(MK_RELU, "features.4");
  b.pool(MK_MAXPOOL, "features.5", 3, 2, 0);
  b.conv("features.6", 192, 384, 3, 1, 1, true); b.simple(MK_RELU, "features.7");
  b.conv("features.8", 384, 256, 3, 1, 1, true); b.simple(MK_RELU, "features.9");
  b.conv("features.10", 256, 256, 3, 1, 1, true); b.simple(MK_RELU, "features.11");
  b.pool(MK_MAXPOOL, "features.12", 3, 2, 0);
  b.adaptive("avgpool", 6, 6);
  b.simple(MK_DROPOUT, "classifier.0"); b.linear("classifier.1", 256 * 36, 4096);
  b.simple(MK_RELU, "classifier.2"); b.simple(MK_DROPOUT, "classifier.3");
  b.linear("classifier.4", 4096, 4096); b.simple(MK_RELU, "classifier.5");
  b.linear("classifier.6", 4096, 1000);
  return b.a;
}

ArchDesc build_resnet(bool bottleneck, const int* layers, hapi_arch id) {
  Builder b;
  b.a.arch = id; b.a.freeze = bottleneck ? 21 : 11;
  b.conv("conv1", 3, 64, 7, 2, 3, false);
  b.bn("bn1", 64);
  b.simple(MK_RELU, "relu");
  b.pool(MK_MAXPOOL, "maxpool", 3, 2, 1);
  int cin = 64, exp = bottleneck ? 4 : 1;
  const int widths[4] = {64, 128, 256, 512};
  for (int li = 0; li < 4; ++li) {
    for (int bi = 0; bi < layers[li]; ++bi) {
      int planes = widths[li], stride = (li > 0 && bi == 0) ? 2 : 1;
      std::string p = "layer" + std::to_string(li + 1) + "." + std::to_string(bi);
      ModDesc m{bottleneck ? MK_BOTTLENECK : MK_BASIC, p};
      m.cin = cin; m.planes = planes; m.cout = planes * exp; m.stride = stride;
      m.ds = stride != 1 || cin != planes * exp;
      m.first_param = (int)b.a.params.size();
      if (!bottleneck) {
        b.conv_params(p + ".conv1", cin, planes, 3, false); b.bn_params(p + ".bn1", planes);
        b.conv_params(p + ".conv2", planes, planes, 3, false); b.bn_params(p + ".bn2", planes);
        m.weight_elems = (int64_t)planes * cin * 9 + (int64_t)planes * planes * 9;
        m.vec_elems = 4 * planes;
      } else {
        b.conv_params(p + ".conv1", cin, planes, 1, false); b.bn_params(p + ".bn1", planes);
        b.conv_params(p + ".conv2", planes, planes, 3, false); b.bn_params(p + ".bn2", planes);
        b.conv_params(p + ".conv3", planes, planes * 4, 1, false); b.bn_params(p + ".bn3", planes * 4);
        m.weight_elems = (int64_t)planes * cin + (int64_t)planes * planes * 9 + (int64_t)planes * 4 * planes;
        m.vec_elems = 2 * (planes + planes + 4 * planes);
      }
      if (m.ds) {
        b.conv_params(p + ".downsample.0", cin, planes * exp, 1, false);
        b.bn_params(p + ".downsample.1", planes * exp);
        m.weight_elems += (int64_t)planes * exp * cin;
        m.vec_elems += 2 * planes * exp;
      }
      b.push(m);
      cin = planes * exp;
    }
  }
  b.adaptive("avgpool", 1, 1);
  b.linear("fc", cin, 1000);
  return b.a;
}

ArchDesc build_vgg11() {
  Builder b;
  b.a.arch = HAPI_VGG11; b.a.freeze = 25;
  const int cfg[] = {64, -1, 128, -1, 256, 256, -1, 512, 512, -1, 512, 512, -1};
  int idx = 0, cin = 3;
  for (int v : cfg) {
    if (v < 0) {
      b.pool(MK_MAXPOOL, "features." + std::to_string(idx), 2, 2, 0);
      idx += 1;
    } else {
      b.conv("features." + std::to_string(idx), cin, v, 3, 1, 1, true);
      b.simple(MK_RELU, "features." + std::to_string(idx + 1));
      cin = v;
      idx += 2;
    }
  }
  b.adaptive("avgpool", 7, 7);
  b.linear("classifier.0", 512 * 49, 4096); b.simple(MK_RELU, "classifier.1");
  b.simple(MK_DROPOUT, "classifier.2");
  b.linear("classifier.3", 4096, 4096); b.simple(MK_RELU, "classifier.4");
  b.simple(MK_DROPOUT, "classifier.5");
  b.linear("classifier.6", 4096, 1000);
  return b.a;
}

ArchDesc build_densenet121() {
  Builder b;
  b.a.arch = HAPI_DENSENET121; b.a.freeze = 20;
  b.conv("features.conv0", 3, 64, 7, 2, 3, false);
  b.bn("features.norm0", 64);
  b.simple(MK_RELU, "features.relu0");
  b.pool(MK_MAXPOOL, "features.pool0", 3, 2, 1);
  const int blocks[4] = {6, 12, 24, 16};
  int c = 64;
  for (int bi = 0; bi < 4; ++bi) {
    std::string p = "features.denseblock" + std::to_string(bi + 1);
    ModDesc m{MK_DENSEBLOCK, p};
    m.cin = c; m.nlayers = blocks[bi]; m.cout = c + 32 * blocks[bi];
    m.first_param = (int)b.a.params.size();
    for (int j = 0; j < blocks[bi]; ++j) {
      std::string q = p + ".denselayer" + std::to_string(j + 1);
      int cj = c + 32 * j;
      b.bn_params(q + ".norm1", cj); b.conv_params(q + ".conv1", cj, 128, 1, false);
      b.bn_params(q + ".norm2", 128); b.conv_params(q + ".conv2", 128, 32, 3, false);
      m.weight_elems += (int64_t)128 * cj + 32 * 128 * 9;
      m.vec_elems += 2 * cj + 2 * 128;
    }
    b.push(m);
    c += 32 * blocks[bi];
    if (bi != 3) {
      std::string t = "features.transition" + std::to_string(bi + 1);
      b.bn(t + ".norm", c);
      b.simple(MK_RELU, t + ".relu");
      b.conv(t + ".conv", c, c / 2, 1, 1, 0, false);
      b.pool(MK_AVGPOOL, t + ".pool", 2, 2, 0);
      c /= 2;
    }
  }
  b.bn("features.norm5", c);
  ModDesc m{MK_DENSE_CLS, "classifier"};
  m.cin = c; m.cout = 1000; m.bias = true;
  m.first_param = (int)b.a.params.size();
  m.weight_elems = (int64_t)c * 1000; m.vec_elems = 1000;
  b.p2("classifier.weight", 1000, c); b.p1("classifier.bias", 1000);
  b.push(m);
  return b.a;
}

}  // namespace

const ArchDesc* get_arch(hapi_arch arch) {
  static std::once_flag once;
  static ArchDesc descs[5];
  std::call_once(once, [] {
    const int r18[4] = {2, 2, 2, 2}, r50[4] = {3, 4, 6, 3};
    descs[0] = build_alexnet();
    descs[1] = build_resnet(false, r18, HAPI_RESNET18);
    descs[2] = build_resnet(true, r50, HAPI_RESNET50);
    descs[3] = build_vgg11();
    descs[4] = build_densenet121();
  });
  if ((int)arch < 0 || (int)arch > 4) return nullptr;
  return &descs[(int)arch];
}

Shape infer(const ModDesc& m, const Shape& in, bool* ok) {
  Shape o = in;
  *ok = true;
  auto spatial = [&](int k, int s, int p) {
    o.h = out_dim(in.h, k, s, p);
    o.w = out_dim(in.w, k, s, p);
  };
  switch (m.kind) {
    case MK_CONV:
      if (in.flat || in.c != m.cin) *ok = false;
      o.c = m.cout; spatial(m.k, m.stride, m.pad);
      break;
    case MK_BN: case MK_RELU:
      break;
    case MK_MAXPOOL: case MK_AVGPOOL:
      spatial(m.k, m.stride, m.pad);
      break;
    case MK_ADAPTIVE:
      o.h = m.oh; o.w = m.ow;
      break;
    case MK_DROPOUT:
      if (!in.flat) { o.c = (int)in.numel(); o.h = o.w = 1; o.flat = true; }
      break;
    case MK_LINEAR:
      if (in.numel() != m.cin) *ok = false;
      o.c = m.cout; o.h = o.w = 1; o.flat = true;
      break;
    case MK_BASIC: case MK_BOTTLENECK:
      if (in.flat || in.c != m.cin) *ok = false;
      o.c = m.cout; spatial(3, m.stride, 1);
      break;
    case MK_DENSEBLOCK:
      if (in.flat || in.c != m.cin) *ok = false;
      o.c = m.cout;
      break;
    case MK_DENSE_CLS:
      if (in.flat || in.c != m.cin) *ok = false;
      o.c = m.cout; o.h = o.w = 1; o.flat = true;
      break;
  }
  if (o.c <= 0 || o.h <= 0 || o.w <= 0) *ok = false;
  return o;
}

}  // namespace hapi
