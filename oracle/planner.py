"""Oracle planner: per-layer sizes, memory estimate, Alg. 1 split choice, Eq. 4 batch.

TEST INFRASTRUCTURE ONLY (see oracle/ops.py header).

Exact integer arithmetic (Python ints, checked against the u64 range) following
SURVEY.md section 8(b):

* ``l_s`` = numel(output of layer s) x bytes(act); ``l_0`` = 3*H*W*4, the fp32 input
  tensor per sample (Alg. 1 line 9 ``size(iteration_input)/len(iteration_input)``,
  PAPER.md:805; reading A3).
* ``P(s)`` = max_{1<=i<=s} (l_{i-1} + l_i): "the memory used by the most expensive
  layer (i.e. maximum input plus output size across all layers)" (section 4.3,
  PAPER.md:767), over the storage-side partition (reading A13).
* ``W(s)`` = sum_{i<=s} [weight elems x bytes(act) + (bias + BN gamma/beta elems) x 4]
  (the "model size" of the partition; BN running buffers not counted).
* est(b, s) = W(s) + b * P(s) (correction term 0; reading A14).
* Alg. 1: candidates = {l <= freeze : l_l < l_0} ascending;
  C = link bytes/s x threshold (1 s: "network bandwidth times 1s");
  winner = first candidate with l_l x training_batch < C, else freeze.  Line 16's
  ``winner = intermediate_sizes[l]`` is read as ``winner = l`` (reading A6).
* Eq. 4 for a single request: the largest integer b in
  [b_min, b_max] with W + b*P <= budget; infeasible when b_min does not fit
  ("removes one request at a time and retries"; reading A15).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List

from . import archs

U64_MAX = (1 << 64) - 1
ACT_BYTES = {"f32": 4, "bf16": 2}


def _u64(v: int) -> int:
    if v < 0 or v > U64_MAX:
        raise OverflowError(v)
    return v


def _numel(shape):
    n = 1
    for d in shape:
        n *= d
    return n


@dataclass
class LayerSizes:
    input_bytes: int
    out_bytes: List[int]
    peak_bytes: List[int]
    weight_bytes: List[int]


def layer_sizes(arch: str, in_h: int = 224, in_w: int = 224, act: str = "f32") -> LayerSizes:
    """profile_model (Alg. 1 lines 1-5) done analytically: shapes are static."""
    if in_h <= 0 or in_w <= 0:
        raise ValueError("image size")
    ab = ACT_BYTES[act]
    l0 = _u64(3 * in_h * in_w * 4)
    shp = (3, in_h, in_w)
    outs, peaks, wts = [], [], []
    prev, peak, w = l0, 0, 0
    for m in archs.layers(arch):
        shp = m.shape_fn(shp)
        if min(shp) <= 0:
            raise ValueError(f"layer {m.name} has empty output {shp} at {in_h}x{in_w}")
        ls = _u64(_numel(shp) * ab)
        peak = max(peak, _u64(prev + ls))
        w = _u64(w + m.weight_elems * ab + m.vec_elems * 4)
        outs.append(ls)
        peaks.append(peak)
        wts.append(w)
        prev = ls
    return LayerSizes(l0, outs, peaks, wts)


def choose_split_idx(intermediate_sizes: List[int], input_size: int, freeze_idx: int,
                     training_batch: int, C: int):
    """Alg. 1 choose_split_idx lines 11-19, indices 1-based.  Returns (winner, candidates)."""
    # candidate selection phase (line 12)
    potential_layers = [l for l in range(1, len(intermediate_sizes) + 1)
                        if intermediate_sizes[l - 1] < input_size and l <= freeze_idx]
    # winner selection phase (lines 14-19)
    winner = freeze_idx
    for l in potential_layers:
        if _u64(intermediate_sizes[l - 1] * training_batch) < C:
            winner = l
            break
    return winner, potential_layers


@dataclass
class SplitQuery:
    arch: str
    freeze_idx: int
    training_batch: int
    link_bytes_per_s: int
    hbm_budget_bytes: int
    b_min: int = 25
    b_max: int = 2000
    threshold_ms: int = 1000
    act: str = "f32"
    in_h: int = 224
    in_w: int = 224


@dataclass
class SplitResult:
    status: str                 # "ok" | "infeasible"
    split_idx: int
    cos_batch: int
    bytes_per_iteration: int
    est_bytes: int
    candidates: List[int] = field(default_factory=list)


def choose_split(q: SplitQuery) -> SplitResult:
    sz = layer_sizes(q.arch, q.in_h, q.in_w, q.act)
    L = len(sz.out_bytes)
    if not (1 <= q.freeze_idx <= L) or q.training_batch < 1 or q.link_bytes_per_s < 1 \
            or q.threshold_ms < 1 or q.b_min < 1 or q.b_min > q.b_max:
        raise ValueError("invalid argument")
    C = _u64(q.link_bytes_per_s * q.threshold_ms) // 1000
    s, cands = choose_split_idx(sz.out_bytes, sz.input_bytes, q.freeze_idx, q.training_batch, C)
    bpi = _u64(sz.out_bytes[s - 1] * q.training_batch)
    W, P = sz.weight_bytes[s - 1], sz.peak_bytes[s - 1]
    if q.hbm_budget_bytes < W or q.hbm_budget_bytes - W < _u64(q.b_min * P):
        return SplitResult("infeasible", s, 0, bpi, W, cands)
    b = min(q.b_max, (q.hbm_budget_bytes - W) // P)
    return SplitResult("ok", s, b, bpi, _u64(W + b * P), cands)


def estimate(arch: str, split_idx: int, batch: int, act: str = "f32", in_h: int = 224, in_w: int = 224) -> int:
    """est(b, s) = W(s) + b * P(s)."""
    sz = layer_sizes(arch, in_h, in_w, act)
    return _u64(sz.weight_bytes[split_idx - 1] + batch * sz.peak_bytes[split_idx - 1])


# ---------------------------------------------------------------- section 4.5
# Multi-request batch adaptation, Eq. 4 over all queued requests of one
# GPU:  maximise sum_r b_r * M_r(data) + M_r(model)  s.t.  b_min,r <= b_r <= b_max,r  and
# sum_r (b_r * M_r(data) + M_r(model)) <= M_total - M_occupied.  The paper gives the problem,
# not a solver; readings (F1-F4):
#   F1 infeasible -> "removes one request at a time and retries": the most
#      recently arrived request is deferred first (deferred ids are a suffix of arrival order);
#   F2 solver: unit water-filling -- start every request at b_min, then repeatedly give one
#      more sample to the request with the smallest current b (ties: earliest arrival) that is
#      below its b_max and whose M_r(data) still fits; stop when none does.  The objective is
#      then within max_r M_r(data) of the optimum (every request is at b_max or cannot grow);
#   F3 the static concurrency cap ("capped statically") defers the requests
#      beyond the first `max_concurrency` by arrival before the memory check;
#   F4 requests are spread over GPUs round-robin by arrival ("distributes requests evenly",
#      PAPER.md:862), and the adaptation runs per GPU.

@dataclass
class AdaptRequest:
    arrival_seq: int
    model_bytes: int         # M_r(model) = W(s)
    data_bytes: int          # M_r(data) per sample = P(s)
    b_min: int
    b_max: int


def adapt_batches(reqs: List[AdaptRequest], available: int, max_concurrency: int = 0):
    """-> (batch per request in input order, 0 = deferred; memory used)."""
    for r in reqs:
        if not (1 <= r.b_min <= r.b_max):
            raise ValueError("b_min/b_max")
    order = sorted(range(len(reqs)), key=lambda i: (reqs[i].arrival_seq, i))
    active = order[:max_concurrency] if max_concurrency > 0 else list(order)

    def floor_need(ids):
        return sum(reqs[i].b_min * reqs[i].data_bytes + reqs[i].model_bytes for i in ids)

    while active and floor_need(active) > available:
        active.pop()                                  # most recent arrival first (F1)
    b = [0] * len(reqs)
    for i in active:
        b[i] = reqs[i].b_min
    rem = available - floor_need(active) if active else available
    while True:
        best = None
        for i in active:                              # arrival order: first minimum wins ties
            r = reqs[i]
            if b[i] < r.b_max and r.data_bytes <= rem and (best is None or b[i] < b[best]):
                best = i
        if best is None:
            break
        b[best] += 1
        rem -= reqs[best].data_bytes
    used = sum(b[i] * reqs[i].data_bytes + reqs[i].model_bytes for i in active)
    return b, used


def partition_requests(n: int, n_gpus: int) -> List[int]:
    """GPU of each request (requests given in arrival order): round-robin (F4)."""
    if n_gpus < 1:
        raise ValueError("n_gpus")
    return [i % n_gpus for i in range(n)]
