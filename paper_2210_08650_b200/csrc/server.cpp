// The HAPI server loop of one GPU (section 4.5) on top of
// the scheduler (scheduler.cpp) and the executor (model.cu), through the public C ABI only:
// registered frozen models hold the device weights once; every admitted request runs on its
// own stream with a model sharing those weights and an arena for its COS batch.
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "common.h"
#include "hapi.h"

using hapi::clear_error;
using hapi::set_error;

namespace {
struct DevGuard {
  int prev = -1;
  bool sw = false;
  explicit DevGuard(int d) {
    if (cudaGetDevice(&prev) == cudaSuccess && prev != d) sw = cudaSetDevice(d) == cudaSuccess;
  }
  ~DevGuard() {
    if (sw) cudaSetDevice(prev);
  }
};
}  // namespace

struct hapi_server {
  hapi_server_config cfg;
  hapi_scheduler* sched = nullptr;
  struct Entry {
    hapi_model* base;
    hapi_model_desc desc;
    std::vector<uint64_t> w, p;  // W(s), P(s) for s = 1..L
  };
  std::vector<Entry> models;
  struct Req {
    uint32_t model, split;
    const float* images;
    uint64_t n;
    void* out;
    hapi_model* inst = nullptr;
    cudaStream_t stream = nullptr;
    cudaEvent_t done = nullptr;
    bool launched = false, retired = false;
  };
  std::vector<Req> reqs;  // index = scheduler id (both dense, in submission order)

  void release(Req& r) {
    if (r.done) cudaEventDestroy(r.done);
    if (r.stream) cudaStreamDestroy(r.stream);
    if (r.inst) hapi_model_destroy(r.inst);
    r.done = nullptr;
    r.stream = nullptr;
    r.inst = nullptr;
  }
};

extern "C" {

hapi_status hapi_server_create(const hapi_server_config* cfg, hapi_server** out) {
  clear_error();
  if (!cfg || !out) return set_error(HAPI_ERR_INVALID_ARGUMENT, "null argument");
  if (cfg->b_min < 1) return set_error(HAPI_ERR_INVALID_ARGUMENT, "b_min = 0");
  hapi_server* s = new hapi_server();
  s->cfg = *cfg;
  hapi_status st = hapi_scheduler_create(&cfg->sched, &s->sched);
  if (st != HAPI_OK) {
    delete s;
    return st;
  }
  *out = s;
  return HAPI_OK;
}

hapi_status hapi_server_add_model(hapi_server* s, const hapi_model_desc* desc, const float* const* params,
                                  uint32_t n_params, uint32_t* model_id) {
  clear_error();
  if (!s || !desc || !model_id) return set_error(HAPI_ERR_INVALID_ARGUMENT, "null argument");
  hapi_model_desc d = *desc;
  d.device = s->cfg.device;
  d.max_batch = 1;  // the registered model only holds the weights; requests get their own arenas
  d.host_chunk = 0;
  const int32_t L = hapi_num_layers(d.arch);
  if (L < 0) return set_error(HAPI_ERR_INVALID_MODEL, "unknown arch");
  hapi_server::Entry e;
  e.desc = d;
  e.w.resize(L);
  e.p.resize(L);
  std::vector<uint64_t> o(L);
  uint64_t l0;
  hapi_status st = hapi_layer_sizes(d.arch, d.in_h, d.in_w, d.act, &l0, o.data(), e.p.data(), e.w.data(), (uint32_t)L);
  if (st != HAPI_OK) return st;
  if ((st = hapi_model_create(&d, params, n_params, &e.base)) != HAPI_OK) return st;
  s->models.push_back(e);
  *model_id = (uint32_t)s->models.size() - 1;
  return HAPI_OK;
}

hapi_status hapi_server_submit(hapi_server* s, uint64_t now_us, uint32_t model_id, uint32_t split_idx, uint32_t b_max,
                               const float* images, uint64_t n, void* out, uint64_t* req_id) {
  clear_error();
  if (!s || !images || !out || !req_id) return set_error(HAPI_ERR_INVALID_ARGUMENT, "null argument");
  if (model_id >= s->models.size()) return set_error(HAPI_ERR_INVALID_ARGUMENT, "unknown model %u", model_id);
  const auto& e = s->models[model_id];
  if (split_idx < e.desc.min_split || split_idx > e.desc.max_split)
    return set_error(HAPI_ERR_INVALID_ARGUMENT, "split %u outside [%u,%u]", split_idx, e.desc.min_split, e.desc.max_split);
  if (n == 0 || b_max == 0) return set_error(HAPI_ERR_INVALID_ARGUMENT, "n = 0 or b_max = 0");
  hapi_adapt_request r;
  r.arrival_seq = 0;
  r.model_bytes = e.w[split_idx - 1];  // M_r(model) = W(s)
  r.data_bytes = e.p[split_idx - 1];   // M_r(data) = P(s)
  r.b_max = b_max;
  r.b_min = s->cfg.b_min < b_max ? s->cfg.b_min : b_max;
  uint64_t id;
  hapi_status st = hapi_scheduler_submit(s->sched, now_us, &r, &id);
  if (st != HAPI_OK) return st;
  hapi_server::Req q;
  q.model = model_id;
  q.split = split_idx;
  q.images = images;
  q.n = n;
  q.out = out;
  s->reqs.push_back(q);
  *req_id = id;
  return HAPI_OK;
}

hapi_status hapi_server_step(hapi_server* s, uint64_t now_us, uint32_t* n_active) {
  clear_error();
  if (!s) return set_error(HAPI_ERR_INVALID_ARGUMENT, "null server");
  DevGuard dg(s->cfg.device);
  // (1) retire completed requests: their memory returns to the scheduler
  for (uint64_t i = 0; i < s->reqs.size(); ++i) {
    auto& r = s->reqs[i];
    if (!r.launched || r.retired) continue;
    const cudaError_t q = cudaEventQuery(r.done);
    if (q == cudaErrorNotReady) continue;
    if (q != cudaSuccess) return set_error(HAPI_ERR_CUDA, "request %llu: %s", (unsigned long long)i, cudaGetErrorString(q));
    s->release(r);
    r.retired = true;
    hapi_status st = hapi_scheduler_finish(s->sched, i);
    if (st != HAPI_OK) return st;
  }
  // (2) a scheduling round if the trigger holds, (3) launch what it admitted
  std::vector<uint64_t> ids(s->reqs.size() + 1);
  std::vector<uint32_t> bs(s->reqs.size() + 1);
  uint32_t n = 0;
  hapi_status st = hapi_scheduler_poll(s->sched, now_us, ids.data(), bs.data(), (uint32_t)ids.size(), &n);
  if (st != HAPI_OK) return st;
  for (uint32_t k = 0; k < n; ++k) {
    auto& r = s->reqs[ids[k]];
    if ((st = hapi_model_create_shared(s->models[r.model].base, bs[k], 0, &r.inst)) != HAPI_OK) return st;
    HAPI_CUDA_TRY(cudaStreamCreateWithFlags(&r.stream, cudaStreamNonBlocking));
    HAPI_CUDA_TRY(cudaEventCreateWithFlags(&r.done, cudaEventDisableTiming));
    if ((st = hapi_model_set_stream(r.inst, r.stream)) != HAPI_OK) return st;
    if ((st = hapi_prefix_forward(r.inst, r.split, r.images, r.n, r.out)) != HAPI_OK) return st;
    HAPI_CUDA_TRY(cudaEventRecord(r.done, r.stream));
    r.launched = true;
  }
  if (n_active) {
    uint32_t a = 0;
    for (const auto& r : s->reqs) a += !r.retired;
    *n_active = a;
  }
  return HAPI_OK;
}

hapi_status hapi_server_query(const hapi_server* s, uint64_t req_id, uint32_t* state, uint32_t* batch,
                              uint64_t* device_bytes) {
  clear_error();
  if (!s) return set_error(HAPI_ERR_INVALID_ARGUMENT, "null server");
  if (state || batch) {
    hapi_status st = hapi_scheduler_query(s->sched, req_id, state, batch, nullptr);
    if (st != HAPI_OK) return st;
    // the scheduler marks a request RUNNING when admitted; DONE only once its forward completed
  }
  if (device_bytes) {
    uint64_t t = 0, w, a;
    for (const auto& e : s->models)
      if (hapi_model_device_bytes(e.base, &w, &a) == HAPI_OK) t += w + a;
    for (const auto& r : s->reqs)
      if (r.inst && hapi_model_device_bytes(r.inst, &w, &a) == HAPI_OK) t += w + a;
    *device_bytes = t;
  }
  return HAPI_OK;
}

void hapi_server_destroy(hapi_server* s) {
  if (!s) return;
  DevGuard dg(s->cfg.device);
  for (auto& r : s->reqs) {
    if (r.stream) cudaStreamSynchronize(r.stream);
    s->release(r);
  }
  for (auto& e : s->models) hapi_model_destroy(e.base);
  hapi_scheduler_destroy(s->sched);
  delete s;
}

}  // extern "C"
