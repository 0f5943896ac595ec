"""Section 4.5 batch adaptation: the oracle pinned to hand-computed
examples, brute force and invariants, then the C ABI checked against the oracle.

Pins (independent of the oracle's code):
* worked examples computed by hand from Eq. 4: an unconstrained request
  reaches b_max; a capacity-bound one saturates memory exactly; two identical requests share
  the slack evenly; infeasible floors defer the latest arrival;
* brute force over every (b_1..b_k) tuple on small instances: the water-filling objective is
  within max_r M_r(data) of the true optimum of Eq. 4;
* invariants on random instances: feasibility, bounds, maximality at slack, determinism,
  deferred set = suffix of arrival order, the static cap.
"""
import itertools
import random

import pytest

from oracle.planner import AdaptRequest as R
from oracle.planner import adapt_batches, partition_requests


def _objective(reqs, b):
    return sum(bi * r.data_bytes + r.model_bytes for r, bi in zip(reqs, b) if bi > 0)


# ------------------------------------------------------------------ hand-computed examples
def test_unconstrained_request_reaches_b_max():
    # 1000*10 + 1000 = 11,000 <= 20,000
    assert adapt_batches([R(0, 1000, 10, 25, 1000)], 20000) == ([1000], 11000)


def test_capacity_bound_request_saturates_memory():
    # 1000 + b*10 <= 5000  ->  b = 400, exactly 5000 bytes
    assert adapt_batches([R(0, 1000, 10, 25, 1000)], 5000) == ([400], 5000)


def test_identical_requests_share_the_slack():
    # floors 25+25 = 50 of 120 bytes; the remaining 70 split evenly -> 60 + 60 = 120
    assert adapt_batches([R(0, 0, 1, 25, 100), R(1, 0, 1, 25, 100)], 120) == ([60, 60], 120)


def test_infeasible_floor_defers_latest_arrival():
    # floors 3*25 = 75 > 60: the latest (arrival 2) is deferred, the other two share 60
    reqs = [R(0, 0, 1, 25, 100), R(2, 0, 1, 25, 100), R(1, 0, 1, 25, 100)]
    b, used = adapt_batches(reqs, 60)
    assert b == [30, 0, 30] and used == 60


def test_nothing_fits_and_empty_queue():
    assert adapt_batches([R(0, 100, 10, 25, 50)], 349) == ([0], 0)   # 100 + 250 = 350 > 349
    assert adapt_batches([], 10**9) == ([], 0)


def test_static_cap_defers_beyond_first_by_arrival():
    reqs = [R(5, 0, 1, 1, 10), R(1, 0, 1, 1, 10), R(3, 0, 1, 1, 10)]
    b, _ = adapt_batches(reqs, 1000, max_concurrency=2)
    assert b == [0, 10, 10]


def test_bad_bounds_rejected():
    with pytest.raises(ValueError):
        adapt_batches([R(0, 0, 1, 0, 10)], 100)
    with pytest.raises(ValueError):
        adapt_batches([R(0, 0, 1, 11, 10)], 100)


def test_partition_round_robin():
    assert partition_requests(5, 2) == [0, 1, 0, 1, 0]
    assert partition_requests(0, 3) == []
    assert partition_requests(6, 3) == [0, 1, 2, 0, 1, 2]
    with pytest.raises(ValueError):
        partition_requests(3, 0)


# ------------------------------------------------------------------ brute force
def _random_instance(rng, k, bmax_cap):
    reqs = []
    for i in range(k):
        bmin = rng.randint(1, 4)
        reqs.append(R(rng.randint(0, 9), rng.randint(0, 40), rng.randint(0, 9), bmin, rng.randint(bmin, bmax_cap)))
    return reqs


def test_near_optimal_against_brute_force():
    rng = random.Random(2210)
    for _ in range(300):
        k = rng.randint(1, 3)
        reqs = _random_instance(rng, k, 9)
        avail = rng.randint(0, 250)
        b, used = adapt_batches(reqs, avail)
        kept = [i for i in range(k) if b[i] > 0]
        # exhaustive optimum over the same kept set (the removal rule decides the set)
        best = 0
        for tup in itertools.product(*[range(reqs[i].b_min, reqs[i].b_max + 1) for i in kept]):
            mem = sum(t * reqs[i].data_bytes + reqs[i].model_bytes for t, i in zip(tup, kept))
            if mem <= avail:
                best = max(best, mem)
        assert used == _objective(reqs, b) <= avail
        gap = max([reqs[i].data_bytes for i in kept], default=0)
        assert best - used <= gap, (reqs, avail, b, best)


def test_invariants_random():
    rng = random.Random(7)
    for _ in range(2000):
        k = rng.randint(0, 6)
        reqs = _random_instance(rng, k, 60)
        avail = rng.randint(0, 2000)
        cap = rng.choice([0, 0, 2, 4])
        b, used = adapt_batches(reqs, avail, cap)
        assert (b, used) == adapt_batches(reqs, avail, cap)                     # determinism
        assert used <= avail and used == _objective(reqs, b)                     # feasibility
        order = sorted(range(k), key=lambda i: (reqs[i].arrival_seq, i))
        kept = [b[i] > 0 for i in order]
        assert kept == sorted(kept, reverse=True)                                # deferred = suffix
        if cap:
            assert sum(kept) <= cap
        for i in range(k):
            if b[i]:
                assert reqs[i].b_min <= b[i] <= reqs[i].b_max                    # bounds
                # maximality: nobody who could still grow fits one more sample
                assert b[i] == reqs[i].b_max or reqs[i].data_bytes > avail - used


# ------------------------------------------------------------------ C ABI == oracle
def test_abi_matches_oracle():
    import paper_2210_08650_b200 as H
    rng = random.Random(11)
    for _ in range(3000):
        k = rng.randint(0, 8)
        reqs = _random_instance(rng, k, rng.choice([9, 60, 3000]))
        for r in reqs:
            r.data_bytes *= rng.choice([1, 1000, 150_000])
            r.model_bytes *= rng.choice([1, 10**6])
        avail = rng.randint(0, 4 * 10**8)
        cap = rng.choice([0, 3])
        want = adapt_batches(reqs, avail, cap)
        got = H.hapi_adapt_batches([(r.arrival_seq, r.model_bytes, r.data_bytes, r.b_min, r.b_max) for r in reqs],
                                   avail, cap)
        assert got == want, (reqs, avail, cap)
    assert H.hapi_partition_requests(7, 3) == partition_requests(7, 3)
    with pytest.raises(H.HapiError):
        H.hapi_adapt_batches([(0, 0, 1, 5, 4)], 100)
    with pytest.raises(H.HapiError):
        H.hapi_partition_requests(3, 0)


def test_abi_with_planner_sizes():
    """End to end with the paper's own quantities: M(model) = W(s), M(data) = P(s) of
    ResNet50 s=21 and DenseNet121 s=9 requests sharing one 80 GB budget."""
    import paper_2210_08650_b200 as H
    from oracle import planner
    reqs = []
    for seq, (arch, s) in enumerate([("resnet50", 21), ("densenet121", 9), ("resnet50", 21)]):
        sz = planner.layer_sizes(arch, act="bf16")
        reqs.append(R(seq, sz.weight_bytes[s - 1], sz.peak_bytes[s - 1], 25, 2000))
    want = adapt_batches(reqs, 80 * 10**9)
    got = H.hapi_adapt_batches([(r.arrival_seq, r.model_bytes, r.data_bytes, r.b_min, r.b_max) for r in reqs],
                               80 * 10**9)
    assert got == want and all(b == 2000 for b in got[0])
    tight = sum(r.model_bytes + 25 * r.data_bytes for r in reqs) + 10**8
    b, used = H.hapi_adapt_batches([(r.arrival_seq, r.model_bytes, r.data_bytes, r.b_min, r.b_max) for r in reqs],
                                   tight)
    assert all(25 <= x <= 2000 for x in b) and used <= tight


def test_abi_large_b_max_is_fast_and_exact():
    """The C solver grants whole levels to the group at the minimum level (the
    unit loop cost O(n * b_max)); the result still equals the oracle's unit process, and u32
    b_max no longer means minutes of host time."""
    import time

    import paper_2210_08650_b200 as H
    reqs = [(0, 10, 3, 1, 10 ** 7), (1, 20, 3, 1, 10 ** 7), (2, 0, 5, 2, 4_000_000_000)]
    t0 = time.perf_counter()
    got, used = H.hapi_adapt_batches(reqs, 10 ** 10)
    assert time.perf_counter() - t0 < 0.5
    assert got[:2] == [10 ** 7, 10 ** 7] and used <= 10 ** 10
    small = [R(i, m, d, lo, hi) for i, (_, m, d, lo, hi) in enumerate(reqs[:2])]
    want, wused = adapt_batches([R(r.arrival_seq, r.model_bytes, r.data_bytes, r.b_min, 300) for r in small], 1000)
    got2, gused = H.hapi_adapt_batches([(r.arrival_seq, r.model_bytes, r.data_bytes, r.b_min, 300) for r in small], 1000)
    assert (got2, gused) == (want, wused)
