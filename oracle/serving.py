"""Pure-Python restatement of the reference serving loop — TEST INFRASTRUCTURE ONLY.

Follows fragserve/simulator.py for a fixed deployment:
  event heap keyed (t, rank, seq)               simulator.py:39, 244-246
  _gen_request / _next_gen / _arrive             simulator.py:353-385
  _enqueue / _service / _stage_done              simulator.py:387-426
  run loop (REPLAN pushes consume seqs)          simulator.py:430-463
Pinned bit-for-bit against the golden logs of the unmodified reference (tests/golden/serving,
scripts/make_golden.py).  Used by tests and as the CPU event-loop baseline in bench.py.
"""
from __future__ import annotations

import bisect
import heapq
from collections import deque

import numpy as np

R_REPLAN, R_GEN, R_ARRIVE, R_TIMEOUT, R_DONE = range(5)
EPS = 1e-9


class _Req:
    __slots__ = ("seq", "cid", "gen", "slo", "deadline", "worst", "stages", "idx", "enq", "status", "done")


class _Stage:
    __slots__ = ("batch", "free", "budget", "lat", "queue", "armed")


def simulate_fixed(dep, clients, horizon_s, epoch_s, latency, poisson=False, seed=0, on_batch=None):
    """Returns (records [(client, gen, done, deadline, status)], dispatch [(t, stage, k, seqs)]).

    `on_batch(stage_index, k, t)` may return a service time to use instead of the table (the CPU
    execution baseline plugs real measured execution in here)."""
    horizon = horizon_s * 1000.0
    epoch_ms = epoch_s * 1000.0
    stages = []
    for s in dep.stages:
        st = _Stage()
        st.batch, st.free, st.budget = s.batch, s.instances, s.budget_ms
        st.lat = {}
        st.queue = deque()
        st.armed = None
        stages.append((s, st))
    by_id = {c.client_id: c for c in clients}
    ids = sorted(by_id)
    rngs = {cid: np.random.default_rng((seed, i)) for i, cid in enumerate(ids)} if poisson else {}
    events = []
    counter = [0]
    records = []
    dispatch = []

    def push(t, rank, payload):
        counter[0] += 1
        heapq.heappush(events, (t, rank, counter[0], payload))

    def next_gen(cid, now):
        c = by_id[cid]
        if poisson:
            return now + float(rngs[cid].exponential(1000.0 / c.rate_rps))
        return now + 1000.0 / c.rate_rps

    def lat_for(i, k):
        spec, st = stages[i]
        v = st.lat.get(k)
        if v is None:
            v = latency(spec, k)
            st.lat[k] = v
        return v

    def service(i, now):
        spec, st = stages[i]
        q = st.queue
        while st.free > 0 and q:
            if len(q) >= st.batch:
                k = st.batch
            elif now - q[0].enq >= st.budget - EPS:
                k = len(q)
            else:
                break
            batch = [q.popleft() for _ in range(k)]
            st.free -= 1
            dispatch.append((now, i, k, tuple(r.seq for r in batch)))
            lat = on_batch(i, k, now) if on_batch is not None else lat_for(i, k)
            push(now + lat, R_DONE, (i, batch))
        if q:
            head = q[0]
            tfire = head.enq + st.budget
            if tfire > now + EPS and st.armed != head.seq:
                st.armed = head.seq
                push(tfire, R_TIMEOUT, (i, head.seq))

    def enqueue(i, req, now):
        req.enq = now
        stages[i][1].queue.append(req)
        service(i, now)

    def complete(req, now):
        req.status = "completed"
        req.done = now

    def gen_request(cid, now):
        c = by_id[cid]
        r = _Req()
        r.seq, r.cid, r.gen, r.slo = counter[0], cid, now, c.slo_ms
        r.deadline = now + c.slo_ms
        r.worst, r.stages, r.idx, r.enq, r.status, r.done = 0.0, (), 0, 0.0, "inflight", None
        records.append(r)
        route = dep.routes.get(cid)
        if route is None:
            r.status = "dropped"
            return
        mobile = c.mobile_ms[route.point]
        j = bisect.bisect_right(c.trace_t_s, now / 1000.0) - 1
        bw = c.trace_mbps[j] if j >= 0 else c.trace_mbps[0]
        arrive = now + mobile + c.payload_bytes[route.point] * 8.0 / (bw * 1e6) * 1000.0
        r.stages = route.stages
        r.worst = route.worst_rem_ms
        push(arrive, R_ARRIVE, r)

    def arrive(r, now):
        if now - r.gen + r.worst > r.slo + EPS:
            r.status = "dropped"
            return
        if not r.stages:
            complete(r, now)
            return
        enqueue(r.stages[0], r, now)

    def stage_done(i, batch, now):
        stages[i][1].free += 1
        for r in batch:
            r.idx += 1
            if r.idx < len(r.stages):
                enqueue(r.stages[r.idx], r, now)
            else:
                complete(r, now)
        service(i, now)

    if epoch_ms > 0:
        k = 1
        while k * epoch_ms < horizon:
            push(k * epoch_ms, R_REPLAN, k)
            k += 1
    for cid in ids:
        first = next_gen(cid, 0.0) if poisson else 0.0
        if first < horizon:
            push(first, R_GEN, cid)
    while events and events[0][0] <= horizon + EPS:
        now, rank, _, payload = heapq.heappop(events)
        if rank == R_REPLAN:
            continue
        if rank == R_GEN:
            gen_request(payload, now)
            nxt = next_gen(payload, now)
            if nxt < horizon:
                push(nxt, R_GEN, payload)
        elif rank == R_ARRIVE:
            arrive(payload, now)
        elif rank == R_TIMEOUT:
            i, seq = payload
            if stages[i][1].armed == seq:
                stages[i][1].armed = None
                service(i, now)
        else:
            i, batch = payload
            stage_done(i, batch, now)
    return [(r.cid, r.gen, r.done, r.deadline, r.status) for r in records], dispatch
