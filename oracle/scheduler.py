"""Oracle of the HAPI server's batch-adaptation loop (section 4.5).

TEST INFRASTRUCTURE ONLY (see oracle/ops.py header).

PAPER.md:841: "This algorithm runs repeatedly at the HAPI server.  A new run of the
algorithm is triggered when two conditions hold: (1) there is available GPU memory for new
requests, and (2) there exists at least one queued request that has not yet been accounted
for in the previous runs of the algorithm. ... the HAPI server waits for new requests for a
small amount of time."  The algorithm "takes into account the already-running requests ...
but not the future requests".  PAPER.md:864: "if the server cannot solve the problem it
removes one request at a time and retries until a solution is found.  The removed requests
become part of the next batch assignment round, typically after some existing requests
finish."  PAPER.md:866: "the concurrency level is capped statically".

Readings (F5-F8; F1-F4 are planner.adapt_batches'):
  F5 wait window: a round runs at the first poll with now >= t_first + wait, t_first the
     earliest arrival among the unaccounted requests (a bounded delay that collects the
     requests that arrive "in quick succession");
  F6 available memory = M_total - M_occupied - sum over running requests of
     (W_r + b_r * P_r); condition (1) is available > 0 and, with a static cap, fewer running
     requests than the cap;
  F7 a round's request set = the unaccounted requests plus the deferred ones (they "become
     part of the next batch assignment round"); the cap passed to adapt_batches is the
     static cap minus the running count; admitted requests run, the rest are deferred
     (accounted);
  F8 a request finishing returns its memory and makes the deferred requests unaccounted
     again (with their original arrival times), so the next poll may run a round for them
     ("typically after some existing requests finish").
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, List, Tuple

from .planner import AdaptRequest, adapt_batches

QUEUED, DEFERRED, RUNNING, DONE = 0, 1, 2, 3


@dataclass
class _Req:
    rid: int
    arrival: int
    model_bytes: int
    data_bytes: int
    b_min: int
    b_max: int
    state: int = QUEUED
    batch: int = 0


class Scheduler:
    def __init__(self, total_bytes: int, occupied_bytes: int, max_concurrency: int = 0, wait_us: int = 0):
        self.total, self.occupied = total_bytes, occupied_bytes
        self.cap, self.wait = max_concurrency, wait_us
        self.reqs: Dict[int, _Req] = {}
        self.next_id = 0

    def submit(self, now: int, model_bytes: int, data_bytes: int, b_min: int, b_max: int) -> int:
        if not 1 <= b_min <= b_max:
            raise ValueError("b_min/b_max")
        rid = self.next_id
        self.next_id += 1
        self.reqs[rid] = _Req(rid, now, model_bytes, data_bytes, b_min, b_max)
        return rid

    def _running(self) -> List[_Req]:
        return [r for r in self.reqs.values() if r.state == RUNNING]

    def available(self) -> int:
        used = self.occupied + sum(r.model_bytes + r.batch * r.data_bytes for r in self._running())
        return self.total - used if self.total > used else 0

    def poll(self, now: int) -> List[Tuple[int, int]]:
        """-> [(request id, COS batch)] admitted by this poll's round (empty: no round)."""
        queued = [r for r in self.reqs.values() if r.state == QUEUED]
        if not queued:
            return []                                             # condition (2)
        n_run = len(self._running())
        avail = self.available()
        if avail == 0 or (self.cap > 0 and n_run >= self.cap):
            return []                                             # condition (1), F6
        if now < min(r.arrival for r in queued) + self.wait:
            return []                                             # wait window, F5
        pool = sorted([r for r in self.reqs.values() if r.state in (QUEUED, DEFERRED)],
                      key=lambda r: (r.arrival, r.rid))          # F7
        cap = self.cap - n_run if self.cap > 0 else 0
        b, _ = adapt_batches([AdaptRequest(k, r.model_bytes, r.data_bytes, r.b_min, r.b_max)
                              for k, r in enumerate(pool)], avail, cap)
        out = []
        for r, bb in zip(pool, b):
            if bb > 0:
                r.state, r.batch = RUNNING, bb
                out.append((r.rid, bb))
            else:
                r.state = DEFERRED
        return out

    def finish(self, rid: int) -> None:
        r = self.reqs[rid]
        if r.state != RUNNING:
            raise ValueError("not running")
        r.state, r.batch = DONE, 0
        for q in self.reqs.values():                              # F8
            if q.state == DEFERRED:
                q.state = QUEUED

    def state(self, rid: int) -> Tuple[int, int]:
        r = self.reqs[rid]
        return r.state, r.batch
