// Planner half of the C ABI: per-layer sizes (Alg. 1 profile_model, PAPER.md:795-800,
// done analytically), the memory profile of section 4.3, Alg. 1's split
// choice and Eq. 4's single-request COS batch.
// Pure integer host code; u64 with overflow checks.
#include <cstdio>
#include <algorithm>
#include <cstring>
#include <vector>
#include <string>

#include "arch.h"
#include "common.h"

using namespace hapi;

namespace {

constexpr uint64_t U64MAX = ~0ull;

bool mul_ok(uint64_t a, uint64_t b, uint64_t* r) {
  if (a != 0 && b > U64MAX / a) return false;
  *r = a * b;
  return true;
}
bool add_ok(uint64_t a, uint64_t b, uint64_t* r) {
  if (b > U64MAX - a) return false;
  *r = a + b;
  return true;
}

struct Sizes {
  uint64_t l0;
  std::vector<uint64_t> out, peak, w;
};

hapi_status compute_sizes(hapi_arch arch, uint32_t in_h, uint32_t in_w, hapi_dtype act, Sizes* sz) {
  const ArchDesc* a = get_arch(arch);
  if (!a) return set_error(HAPI_ERR_INVALID_MODEL, "unknown arch %d", (int)arch);
  if (act != HAPI_F32 && act != HAPI_BF16) return set_error(HAPI_ERR_INVALID_ARGUMENT, "unknown dtype");
  if (in_h == 0 || in_w == 0 || in_h > 65536 || in_w > 65536)
    return set_error(HAPI_ERR_INVALID_MODEL, "image size %ux%u", in_h, in_w);
  const uint64_t ab = act == HAPI_F32 ? 4 : 2;
  sz->l0 = 3ull * in_h * in_w * 4ull;
  Shape s{3, (int)in_h, (int)in_w, false};
  uint64_t prev = sz->l0, peak = 0, w = 0;
  for (const ModDesc& m : a->mods) {
    bool ok;
    s = infer(m, s, &ok);
    if (!ok) return set_error(HAPI_ERR_INVALID_MODEL, "layer %s has an empty output at %ux%u", m.name.c_str(), in_h, in_w);
    uint64_t ls, pk, wt, vt;
    if (!mul_ok((uint64_t)s.numel(), ab, &ls) || !add_ok(prev, ls, &pk) ||
        !mul_ok((uint64_t)m.weight_elems, ab, &wt) || !mul_ok((uint64_t)m.vec_elems, 4, &vt) ||
        !add_ok(w, wt, &w) || !add_ok(w, vt, &w))
      return set_error(HAPI_ERR_INVALID_ARGUMENT, "u64 overflow in layer sizes");
    if (pk > peak) peak = pk;
    sz->out.push_back(ls);
    sz->peak.push_back(peak);
    sz->w.push_back(w);
    prev = ls;
  }
  return HAPI_OK;
}

}  // namespace

extern "C" {

int32_t hapi_num_layers(hapi_arch arch) {
  const ArchDesc* a = get_arch(arch);
  return a ? (int32_t)a->mods.size() : -(int32_t)HAPI_ERR_INVALID_MODEL;
}

int32_t hapi_freeze_index(hapi_arch arch) {
  const ArchDesc* a = get_arch(arch);
  return a ? a->freeze : -(int32_t)HAPI_ERR_INVALID_MODEL;
}

hapi_status hapi_layer_sizes(hapi_arch arch, uint32_t in_h, uint32_t in_w, hapi_dtype act,
                             uint64_t* input_bytes, uint64_t* out_bytes, uint64_t* peak_bytes,
                             uint64_t* weight_bytes, uint32_t capacity) {
  clear_error();
  const ArchDesc* a = get_arch(arch);
  if (!a) return set_error(HAPI_ERR_INVALID_MODEL, "unknown arch %d", (int)arch);
  const uint32_t L = (uint32_t)a->mods.size();
  if ((out_bytes || peak_bytes || weight_bytes) && capacity < L)
    return set_error(HAPI_ERR_INVALID_ARGUMENT, "capacity %u < L = %u", capacity, L);
  Sizes sz;
  hapi_status st = compute_sizes(arch, in_h, in_w, act, &sz);
  if (st != HAPI_OK) return st;
  if (input_bytes) *input_bytes = sz.l0;
  for (uint32_t i = 0; i < L; ++i) {
    if (out_bytes) out_bytes[i] = sz.out[i];
    if (peak_bytes) peak_bytes[i] = sz.peak[i];
    if (weight_bytes) weight_bytes[i] = sz.w[i];
  }
  return HAPI_OK;
}

hapi_status hapi_choose_split(const hapi_split_query* q, hapi_split_result* r, uint32_t* candidates) {
  clear_error();
  if (!q || !r) return set_error(HAPI_ERR_INVALID_ARGUMENT, "null query/result");
  std::memset(r, 0, sizeof(*r));
  const ArchDesc* a = get_arch(q->arch);
  if (!a) return set_error(HAPI_ERR_INVALID_MODEL, "unknown arch %d", (int)q->arch);
  const uint32_t L = (uint32_t)a->mods.size();
  if (q->freeze_idx < 1 || q->freeze_idx > L) return set_error(HAPI_ERR_INVALID_ARGUMENT, "freeze_idx %u not in [1,%u]", q->freeze_idx, L);
  if (q->training_batch < 1) return set_error(HAPI_ERR_INVALID_ARGUMENT, "training_batch = 0");
  if (q->link_bytes_per_s < 1) return set_error(HAPI_ERR_INVALID_ARGUMENT, "link_bytes_per_s = 0");
  if (q->threshold_ms < 1) return set_error(HAPI_ERR_INVALID_ARGUMENT, "threshold_ms = 0");
  if (q->b_min < 1 || q->b_min > q->b_max) return set_error(HAPI_ERR_INVALID_ARGUMENT, "b_min/b_max");
  Sizes sz;
  hapi_status st = compute_sizes(q->arch, q->in_h, q->in_w, q->act, &sz);
  if (st != HAPI_OK) return st;

  // C = network bandwidth x 1 s (threshold_ms / 1000), integer division.
  uint64_t Cms;
  if (!mul_ok(q->link_bytes_per_s, q->threshold_ms, &Cms)) return set_error(HAPI_ERR_INVALID_ARGUMENT, "overflow in C");
  const uint64_t C = Cms / 1000;

  // Candidate selection: l_s < l0 and s <= freeze, ascending; winner: first with
  // l_s * training_batch < C, default freeze.
  uint32_t winner = q->freeze_idx, ncand = 0;
  bool found = false;
  for (uint32_t s = 1; s <= q->freeze_idx; ++s) {
    if (!(sz.out[s - 1] < sz.l0)) continue;
    if (candidates) candidates[ncand] = s;
    ++ncand;
    if (!found) {
      uint64_t bytes;
      if (!mul_ok(sz.out[s - 1], q->training_batch, &bytes)) return set_error(HAPI_ERR_INVALID_ARGUMENT, "overflow l_s*batch");
      if (bytes < C) { winner = s; found = true; }
    }
  }
  r->split_idx = winner;
  r->n_candidates = ncand;
  if (!mul_ok(sz.out[winner - 1], q->training_batch, &r->bytes_per_iteration))
    return set_error(HAPI_ERR_INVALID_ARGUMENT, "overflow bytes_per_iteration");

  // Eq. 4, one request: largest b in [b_min, b_max] with W + b*P <= budget.
  const uint64_t W = sz.w[winner - 1], P = sz.peak[winner - 1];
  uint64_t minneed;
  if (!mul_ok(q->b_min, P, &minneed)) minneed = U64MAX;
  if (q->hbm_budget_bytes < W || q->hbm_budget_bytes - W < minneed) {
    r->cos_batch = 0;
    r->est_bytes = W;
    return set_error(HAPI_ERR_INFEASIBLE, "budget %llu < W(s) + b_min*P(s)", (unsigned long long)q->hbm_budget_bytes);
  }
  uint64_t b = (q->hbm_budget_bytes - W) / P;
  if (b > q->b_max) b = q->b_max;
  r->cos_batch = (uint32_t)b;
  r->est_bytes = W + b * P;  // <= budget, no overflow
  return HAPI_OK;
}

int32_t hapi_num_params(hapi_arch arch) {
  const ArchDesc* a = get_arch(arch);
  return a ? (int32_t)a->params.size() : -(int32_t)HAPI_ERR_INVALID_MODEL;
}

hapi_status hapi_param_info(hapi_arch arch, uint32_t idx, char* name_buf, uint32_t name_cap,
                            int64_t dims[4], uint32_t* ndim) {
  clear_error();
  const ArchDesc* a = get_arch(arch);
  if (!a) return set_error(HAPI_ERR_INVALID_MODEL, "unknown arch %d", (int)arch);
  if (idx >= a->params.size()) return set_error(HAPI_ERR_INVALID_ARGUMENT, "param index %u", idx);
  const ParamSpec& p = a->params[idx];
  if (name_buf && name_cap > 0) {
    std::snprintf(name_buf, name_cap, "%s", p.name.c_str());
  }
  if (dims) for (int i = 0; i < 4; ++i) dims[i] = i < p.ndim ? p.dims[i] : 0;
  if (ndim) *ndim = (uint32_t)p.ndim;
  return HAPI_OK;
}

// Section 4.5 batch adaptation: Eq. 4 over the queued requests of one GPU,
// readings F1-F4 in include/hapi.h.  Host-only, pure.
hapi_status hapi_adapt_batches(const hapi_adapt_request* reqs, uint32_t n, uint64_t available_bytes,
                               uint32_t max_concurrency, uint32_t* batch, uint64_t* used_bytes) {
  clear_error();
  if (n > 0 && (!reqs || !batch)) return set_error(HAPI_ERR_INVALID_ARGUMENT, "null requests/batch");
  for (uint32_t i = 0; i < n; ++i)
    if (reqs[i].b_min < 1 || reqs[i].b_min > reqs[i].b_max)
      return set_error(HAPI_ERR_INVALID_ARGUMENT, "request %u: b_min/b_max", i);
  std::vector<uint32_t> order(n);
  for (uint32_t i = 0; i < n; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(),
                   [&](uint32_t x, uint32_t y) { return reqs[x].arrival_seq < reqs[y].arrival_seq; });
  if (max_concurrency > 0 && order.size() > max_concurrency) order.resize(max_concurrency);  // F3
  // floor footprint sum_r (b_min * data + model); u64 with overflow treated as "does not fit"
  auto floor_need = [&](const std::vector<uint32_t>& ids, uint64_t* out) {
    uint64_t t = 0;
    for (uint32_t i : ids) {
      uint64_t x;
      if (!mul_ok(reqs[i].b_min, reqs[i].data_bytes, &x) || !add_ok(x, reqs[i].model_bytes, &x) || !add_ok(t, x, &t))
        return false;
    }
    *out = t;
    return true;
  };
  uint64_t need = 0;
  while (!order.empty() && (!floor_need(order, &need) || need > available_bytes)) order.pop_back();  // F1
  for (uint32_t i = 0; i < n; ++i) batch[i] = 0;
  uint64_t rem = available_bytes;
  if (!order.empty()) {
    rem -= need;
    for (uint32_t i : order) batch[i] = reqs[i].b_min;
    // F2 unit water-filling: one more sample to the smallest b (earliest arrival on ties) that
    // is below its b_max and whose M(data) still fits.  Computed a level at a time: the unit
    // process raises every eligible request at the minimum level m once, in arrival order,
    // before any goes to m + 2, so while the group's summed M(data) fits, whole levels are
    // granted at once (up to the next occupied level or the group's smallest b_max); a level
    // that does not fit completely is finished one unit step at a time.  Cost O(n^2) levels
    // instead of O(n * b_max) unit steps.
    auto eligible = [&](uint32_t i) { return batch[i] < reqs[i].b_max && reqs[i].data_bytes <= rem; };
    for (;;) {
      uint32_t m = UINT32_MAX;
      for (uint32_t i : order)
        if (eligible(i)) m = std::min(m, batch[i]);
      if (m == UINT32_MAX) break;
      uint64_t S = 0, levels = UINT64_MAX;
      bool ovf = false;
      for (uint32_t i : order) {
        if (!eligible(i)) continue;
        if (batch[i] == m) {
          if (!add_ok(S, reqs[i].data_bytes, &S)) ovf = true;
          levels = std::min<uint64_t>(levels, (uint64_t)reqs[i].b_max - m);
        } else {
          levels = std::min<uint64_t>(levels, (uint64_t)batch[i] - m);  // next occupied level
        }
      }
      if (!ovf && S > 0) levels = std::min<uint64_t>(levels, rem / S);
      if (!ovf && levels >= 1) {
        for (uint32_t i : order)
          if (eligible(i) && batch[i] == m) batch[i] += (uint32_t)levels;
        rem -= levels * S;  // <= rem (levels <= rem / S)
        continue;
      }
      for (uint32_t i : order)  // partial level: one unit step, first minimum by arrival
        if (eligible(i) && batch[i] == m) {
          batch[i] += 1;
          rem -= reqs[i].data_bytes;
          break;
        }
    }
  }
  if (used_bytes) *used_bytes = available_bytes - rem;
  return HAPI_OK;
}

hapi_status hapi_partition_requests(uint32_t n, uint32_t n_gpus, uint32_t* gpu_of) {
  clear_error();
  if (n_gpus < 1) return set_error(HAPI_ERR_INVALID_ARGUMENT, "n_gpus = 0");
  if (n > 0 && !gpu_of) return set_error(HAPI_ERR_INVALID_ARGUMENT, "null gpu_of");
  for (uint32_t i = 0; i < n; ++i) gpu_of[i] = i % n_gpus;  // F4 round-robin by arrival
  return HAPI_OK;
}

}  // extern "C"
