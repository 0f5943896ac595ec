"""Section 4.5's server loop: the oracle (oracle/scheduler.py) is pinned by
hand-worked traces of the paper's rules -- trigger conditions, the wait window, deferral and
carry-over into the next round after a request finishes, the static concurrency cap -- and
the C ABI (hapi_scheduler_*) must reproduce the oracle exactly on random event traces."""
import random

import pytest

from oracle.scheduler import DEFERRED, DONE, QUEUED, RUNNING, Scheduler

MB = 1 << 20


def test_wait_window_collects_requests_in_quick_succession():
    s = Scheduler(total_bytes=1000 * MB, occupied_bytes=100 * MB, wait_us=500)
    a = s.submit(0, 50 * MB, 1 * MB, 25, 100)
    assert s.poll(100) == []                       # still inside the window
    b = s.submit(300, 50 * MB, 1 * MB, 25, 100)
    got = s.poll(500)                              # window of the first arrival passed
    assert [r for r, _ in got] == [a, b]
    # 800 MB free for 100 MB of models: both reach b_max = 100 (2 x 100 MB of data)
    assert [b_ for _, b_ in got] == [100, 100]
    assert s.available() == 1000 * MB - 100 * MB - 2 * (50 * MB + 100 * MB)


def test_no_round_without_unaccounted_request_or_memory():
    s = Scheduler(total_bytes=300 * MB, occupied_bytes=0)
    assert s.poll(0) == []                         # condition (2): nothing queued
    a = s.submit(0, 100 * MB, 1 * MB, 25, 200)
    assert s.poll(0) == [(a, 200)]                 # 100 + 200 = 300 MB: memory now exhausted
    b = s.submit(1, 10 * MB, 1 * MB, 25, 50)
    assert s.poll(2) == []                         # condition (1): no available memory
    assert s.state(b) == (QUEUED, 0)
    s.finish(a)
    assert s.poll(3) == [(b, 50)]


def test_infeasible_round_defers_latest_then_carries_over_after_finish():
    s = Scheduler(total_bytes=200 * MB, occupied_bytes=0)
    a = s.submit(0, 60 * MB, 1 * MB, 25, 30)
    b = s.submit(0, 60 * MB, 1 * MB, 25, 30)
    c = s.submit(0, 60 * MB, 1 * MB, 25, 30)
    got = s.poll(0)                                # floors 3 x 85 MB > 200 MB: drop c (latest)
    assert [r for r, _ in got] == [a, b]
    assert s.state(c) == (DEFERRED, 0)
    assert s.poll(10) == []                        # c is accounted; no new request -> no round
    s.finish(a)
    assert s.state(c)[0] == QUEUED                 # "part of the next batch assignment round"
    assert s.poll(11) == [(c, 30)]
    assert s.state(a) == (DONE, 0) and s.state(b)[0] == RUNNING


def test_static_concurrency_cap():
    s = Scheduler(total_bytes=10_000 * MB, occupied_bytes=0, max_concurrency=2)
    ids = [s.submit(0, 10 * MB, 1 * MB, 25, 50) for _ in range(3)]
    assert [r for r, _ in s.poll(0)] == ids[:2]
    assert s.state(ids[2]) == (DEFERRED, 0)
    d = s.submit(5, 10 * MB, 1 * MB, 25, 50)
    assert s.poll(6) == []                         # cap reached: condition (1) fails
    s.finish(ids[0])
    assert [r for r, _ in s.poll(7)] == [ids[2]]   # earliest arrival first; d waits
    assert s.state(d) == (DEFERRED, 0)


def test_errors():
    s = Scheduler(100, 0)
    with pytest.raises(ValueError):
        s.submit(0, 1, 1, 5, 4)
    a = s.submit(0, 1, 1, 1, 1)
    with pytest.raises(ValueError):
        s.finish(a)                                # queued, not running
    with pytest.raises(KeyError):
        s.finish(99)


def _trace(rng, sched_o, sched_c, steps=120):
    now, ids = 0, []
    for _ in range(steps):
        now += rng.choice([0, 0, 1, 5, 50, 400])
        op = rng.random()
        if op < 0.45:
            m, d = rng.choice([0, 10, 47]) * MB, rng.choice([1, 3, 7]) * MB // rng.choice([1, 4])
            lo = rng.randint(1, 30)
            hi = lo + rng.randint(0, 200)
            a = sched_o.submit(now, m, d, lo, hi)
            b = sched_c.submit(now, m, d, lo, hi)
            assert a == b
            ids.append(a)
        elif op < 0.8:
            assert sched_o.poll(now) == sched_c.poll(now)
        else:
            run = [i for i in ids if sched_o.state(i)[0] == RUNNING]
            if run:
                i = rng.choice(run)
                sched_o.finish(i)
                sched_c.finish(i)
        for i in ids:
            assert sched_o.state(i) == sched_c.state(i)
        assert sched_o.available() == sched_c.available()


def test_abi_matches_oracle_on_random_traces():
    import paper_2210_08650_b200 as H
    rng = random.Random(5)
    for _ in range(200):
        total = rng.choice([200, 1000, 5000]) * MB
        occ = rng.choice([0, 50]) * MB
        cap = rng.choice([0, 0, 2, 3])
        wait = rng.choice([0, 10, 300])
        o = Scheduler(total, occ, cap, wait)
        c = H.Scheduler(total, occ, cap, wait)
        _trace(rng, o, c)
        c.close()


def test_abi_errors():
    import paper_2210_08650_b200 as H
    with pytest.raises(H.HapiError):
        H.Scheduler(10, 20)
    s = H.Scheduler(100, 0)
    with pytest.raises(H.HapiError):
        s.submit(0, 1, 1, 5, 4)
    s.submit(10, 1, 1, 1, 1)
    with pytest.raises(H.HapiError):
        s.submit(5, 1, 1, 1, 1)                    # clock went backwards
    with pytest.raises(H.HapiError):
        s.finish(0)                                # not running
    with pytest.raises(H.HapiError):
        s.finish(7)                                # unknown
