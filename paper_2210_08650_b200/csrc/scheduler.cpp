// The HAPI server's batch-adaptation loop for one GPU (section 4.5,
// PAPER.md:841-866): queue, trigger (available memory + an unaccounted request), wait
// window, one Eq. 4 round per trigger through hapi_adapt_batches, deferred requests carried
// into the next round after a request finishes.  Readings F5-F8 in include/hapi.h.
// Host-only; the caller supplies the clock, so the loop is deterministic and testable.
#include <algorithm>
#include <cstdint>
#include <vector>

#include "common.h"
#include "hapi.h"

using hapi::clear_error;
using hapi::set_error;

struct hapi_scheduler {
  hapi_scheduler_config cfg;
  struct Req {
    uint64_t arrival, model_bytes, data_bytes;
    uint32_t b_min, b_max;
    uint32_t state, batch;
  };
  std::vector<Req> reqs;  // index = id (ids are dense, in submission order)
  uint64_t last_now = 0;

  uint64_t available() const {
    // F6: M_total - M(occupied) - sum over running requests of (W_r + b_r P_r), floored at 0
    uint64_t used = cfg.occupied_bytes;
    for (const Req& r : reqs)
      if (r.state == HAPI_REQ_RUNNING) {
        const unsigned __int128 u = (unsigned __int128)used + r.model_bytes + (unsigned __int128)r.batch * r.data_bytes;
        used = u > UINT64_MAX ? UINT64_MAX : (uint64_t)u;
      }
    return cfg.total_bytes > used ? cfg.total_bytes - used : 0;
  }
  uint32_t running() const {
    uint32_t n = 0;
    for (const Req& r : reqs) n += r.state == HAPI_REQ_RUNNING;
    return n;
  }
};

extern "C" {

hapi_status hapi_scheduler_create(const hapi_scheduler_config* cfg, hapi_scheduler** out) {
  clear_error();
  if (!cfg || !out) return set_error(HAPI_ERR_INVALID_ARGUMENT, "null argument");
  if (cfg->occupied_bytes > cfg->total_bytes) return set_error(HAPI_ERR_INVALID_ARGUMENT, "occupied > total");
  hapi_scheduler* s = new hapi_scheduler();
  s->cfg = *cfg;
  *out = s;
  return HAPI_OK;
}

hapi_status hapi_scheduler_submit(hapi_scheduler* s, uint64_t now_us, const hapi_adapt_request* r, uint64_t* id) {
  clear_error();
  if (!s || !r || !id) return set_error(HAPI_ERR_INVALID_ARGUMENT, "null argument");
  if (r->b_min < 1 || r->b_min > r->b_max) return set_error(HAPI_ERR_INVALID_ARGUMENT, "b_min/b_max");
  if (now_us < s->last_now) return set_error(HAPI_ERR_INVALID_ARGUMENT, "clock went backwards");
  s->last_now = now_us;
  s->reqs.push_back({now_us, r->model_bytes, r->data_bytes, r->b_min, r->b_max, HAPI_REQ_QUEUED, 0});
  *id = s->reqs.size() - 1;
  return HAPI_OK;
}

hapi_status hapi_scheduler_poll(hapi_scheduler* s, uint64_t now_us, uint64_t* ids, uint32_t* batches, uint32_t cap,
                                uint32_t* n_admitted) {
  clear_error();
  if (!s || !n_admitted || (cap > 0 && (!ids || !batches))) return set_error(HAPI_ERR_INVALID_ARGUMENT, "null argument");
  if (now_us < s->last_now) return set_error(HAPI_ERR_INVALID_ARGUMENT, "clock went backwards");
  s->last_now = now_us;
  *n_admitted = 0;
  // condition (2): an unaccounted request; F5: its wait window has passed
  uint64_t t_first = UINT64_MAX;
  for (const auto& r : s->reqs)
    if (r.state == HAPI_REQ_QUEUED) t_first = std::min(t_first, r.arrival);
  if (t_first == UINT64_MAX) return HAPI_OK;
  const uint32_t n_run = s->running();
  const uint64_t avail = s->available();
  if (avail == 0 || (s->cfg.max_concurrency > 0 && n_run >= s->cfg.max_concurrency)) return HAPI_OK;  // (1), F6
  if (now_us - t_first < s->cfg.wait_us) return HAPI_OK;
  // F7: unaccounted + deferred requests in arrival order (ties: submission order = id)
  std::vector<uint32_t> pool;
  for (uint32_t i = 0; i < s->reqs.size(); ++i)
    if (s->reqs[i].state == HAPI_REQ_QUEUED || s->reqs[i].state == HAPI_REQ_DEFERRED) pool.push_back(i);
  std::stable_sort(pool.begin(), pool.end(), [&](uint32_t a, uint32_t b) { return s->reqs[a].arrival < s->reqs[b].arrival; });
  std::vector<hapi_adapt_request> ar(pool.size());
  for (size_t k = 0; k < pool.size(); ++k) {
    const auto& r = s->reqs[pool[k]];
    ar[k] = {(uint64_t)k, r.model_bytes, r.data_bytes, r.b_min, r.b_max};
  }
  std::vector<uint32_t> b(pool.size(), 0);
  const uint32_t cap_left = s->cfg.max_concurrency > 0 ? s->cfg.max_concurrency - n_run : 0;
  hapi_status st = hapi_adapt_batches(ar.data(), (uint32_t)ar.size(), avail, cap_left, b.data(), nullptr);
  if (st != HAPI_OK) return st;
  uint32_t n = 0;
  for (uint32_t x : b) n += x > 0;
  if (n > cap) return set_error(HAPI_ERR_INVALID_ARGUMENT, "round admits %u requests, output capacity %u", n, cap);
  n = 0;
  for (size_t k = 0; k < pool.size(); ++k) {
    auto& r = s->reqs[pool[k]];
    if (b[k] > 0) {
      r.state = HAPI_REQ_RUNNING;
      r.batch = b[k];
      ids[n] = pool[k];
      batches[n] = b[k];
      ++n;
    } else {
      r.state = HAPI_REQ_DEFERRED;
    }
  }
  *n_admitted = n;
  return HAPI_OK;
}

hapi_status hapi_scheduler_finish(hapi_scheduler* s, uint64_t id) {
  clear_error();
  if (!s || id >= s->reqs.size()) return set_error(HAPI_ERR_INVALID_ARGUMENT, "unknown request");
  auto& r = s->reqs[id];
  if (r.state != HAPI_REQ_RUNNING) return set_error(HAPI_ERR_INVALID_ARGUMENT, "request %llu is not running", (unsigned long long)id);
  r.state = HAPI_REQ_DONE;
  r.batch = 0;
  for (auto& q : s->reqs)  // F8
    if (q.state == HAPI_REQ_DEFERRED) q.state = HAPI_REQ_QUEUED;
  return HAPI_OK;
}

hapi_status hapi_scheduler_query(const hapi_scheduler* s, uint64_t id, uint32_t* state, uint32_t* batch,
                                 uint64_t* available) {
  clear_error();
  if (!s) return set_error(HAPI_ERR_INVALID_ARGUMENT, "null scheduler");
  if (available) *available = s->available();
  if (state || batch) {
    if (id >= s->reqs.size()) return set_error(HAPI_ERR_INVALID_ARGUMENT, "unknown request");
    if (state) *state = s->reqs[id].state;
    if (batch) *batch = s->reqs[id].batch;
  }
  return HAPI_OK;
}

void hapi_scheduler_destroy(hapi_scheduler* s) { delete s; }

}  // extern "C"
