"""Serving: a deployed plan driven by the native event loop (libgx gx_serve_*).

`serve()` is the executor-side counterpart of fragserve's `simulate(..., fixed_plan=plan)`
(simulator.py:536-538): same clients, same arrival process, same batching/admission semantics,
same report schema (SimReport, simulator.py:121-183).  Two clocks:

  * virtual — batch service time comes from a latency table (a CostModel's latency(model, start,
    end, k, share), exactly what _StageRT.latency_for asks, simulator.py:95-100).  Dispatch order,
    batch composition and every request record are bit-identical to the reference; this is the
    parity mode.
  * wall    — every dispatched batch really executes on the B200 (gather -> span kernels ->
    scatter on a free instance's stream, SM-bounded by the stage's share) and completes when its
    CUDA event fires.  This is the measurement mode for SLO-met requests/sec.
  * replay  — the virtual clock's dispatch decisions (bit-identical to the reference) with every
    batch also executed on the B200 and the real activations flowing align -> shared; per-request
    outputs come back for numerics parity against the fp32 oracle.
"""
from __future__ import annotations

import ctypes as C
import json
import math
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .errors import ValidationError
from .plan import Deployment

_EPS = 1e-9
STATUS = {0: "completed", 1: "dropped", 2: "inflight"}


@dataclass(frozen=True)
class ClientView:
    """The parts of a fragserve ClientSpec (workload.py:98-117) the serving loop needs."""

    client_id: str
    rate_rps: float
    slo_ms: float
    trace_t_s: tuple[float, ...]
    trace_mbps: tuple[float, ...]
    mobile_ms: tuple[float, ...]  # cumulative device latency per boundary (profiles.py:109-131)
    payload_bytes: tuple[int, ...]  # ModelSpec.payload_bytes(p) for p = 0..N

    @classmethod
    def from_reference(cls, client) -> "ClientView":
        model = client.model
        n = model.layer_count
        return cls(client.client_id, float(client.rate_rps), float(client.slo_ms),
                   tuple(float(t) for t in client.trace.times_s), tuple(float(v) for v in client.trace.mbps),
                   tuple(client.device.mobile_ms(model.model_id, p) for p in range(n + 1)),
                   tuple(int(model.payload_bytes(p)) for p in range(n + 1)))

    def to_doc(self) -> dict:
        return {"client_id": self.client_id, "rate_rps": self.rate_rps, "slo_ms": self.slo_ms,
                "trace_t_s": list(self.trace_t_s), "trace_mbps": list(self.trace_mbps),
                "mobile_ms": list(self.mobile_ms), "payload_bytes": list(self.payload_bytes)}

    @classmethod
    def from_doc(cls, d: dict) -> "ClientView":
        return cls(d["client_id"], float(d["rate_rps"]), float(d["slo_ms"]), tuple(d["trace_t_s"]),
                   tuple(d["trace_mbps"]), tuple(d["mobile_ms"]), tuple(int(x) for x in d["payload_bytes"]))


@dataclass
class ServeReport:
    """Same fields and serialisation as the reference SimReport (simulator.py:121-183)."""

    planner: str
    horizon_s: float
    generated: int
    completed: int
    dropped: int
    in_flight: int
    latency_p50_ms: float | None
    latency_p95_ms: float | None
    latency_p99_ms: float | None
    max_latency_ms: float | None
    slo_violation_rate: float | None
    drop_rate: float
    requests: list[tuple]
    config: dict = field(default_factory=dict)
    dispatch: list[tuple] | None = None  # (t_ms, stage index, k, (request seqs...))
    placement: list[tuple] | None = None  # per dispatched batch: (instance index, GPU)
    outputs: np.ndarray | None = None  # replay / wall with return_outputs: [request, out elems]
    sampled: tuple | None = None  # sample_outputs: (request indices, [n, out elems] fp32)
    wall_ms: float = 0.0
    batches: int = 0
    kernels: int = 0

    @property
    def slo_met(self) -> int:
        """#{completed and done <= deadline} (the metric's numerator)."""
        return sum(1 for _c, _g, d, dl, s in self.requests if s == "completed" and d <= dl + _EPS)

    def to_json_dict(self) -> dict:
        return {
            "format_version": 1, "planner": self.planner, "horizon_s": self.horizon_s,
            "generated": self.generated, "completed": self.completed, "dropped": self.dropped,
            "in_flight": self.in_flight,
            "latency_ms": {"p50": self.latency_p50_ms, "p95": self.latency_p95_ms, "p99": self.latency_p99_ms,
                           "max": self.max_latency_ms},
            "slo_violation_rate": self.slo_violation_rate, "drop_rate": self.drop_rate, "config": self.config,
        }

    def to_json(self) -> str:
        return json.dumps(self.to_json_dict(), sort_keys=True, indent=2) + "\n"

    def requests_csv(self) -> str:
        lines = ["client,gen_ms,done_ms,latency_ms,deadline_ms,status"]
        for client_id, gen, done, deadline, status in self.requests:
            if done is None:
                done_s = lat_s = ""
            else:
                done_s = f"{done:.6f}"
                lat_s = f"{done - gen:.6f}"
            lines.append(f"{client_id},{gen:.6f},{done_s},{lat_s},{deadline:.6f},{status}")
        return "\n".join(lines) + "\n"


def _report(planner, horizon_s, client_ids, cl, gen, done, dl, status, config) -> ServeReport:
    """_Sim._report (simulator.py:465-498) over the native records."""
    n = len(gen)
    completed = status == 0
    dropped = int((status == 1).sum())
    ncomp = int(completed.sum())
    lats = (done - gen)[completed]
    if ncomp:
        p50, p95, p99 = (float(x) for x in np.percentile(lats, [50, 95, 99]))
        mx = float(lats.max())
        viol = int((done[completed] > dl[completed] + _EPS).sum())
        viol_rate = viol / ncomp
    else:
        p50 = p95 = p99 = mx = None
        viol_rate = None
    reqs = [(client_ids[cl[i]], float(gen[i]), None if status[i] != 0 else float(done[i]), float(dl[i]),
             STATUS[int(status[i])]) for i in range(n)]
    return ServeReport(planner, horizon_s, n, ncomp, dropped, n - ncomp - dropped, p50, p95, p99, mx, viol_rate,
                       dropped / n if n else 0.0, reqs, config)


class _Keep:
    """Keeps ctypes buffers alive for the duration of a native call."""

    def __init__(self):
        self.items = []

    def __call__(self, x):
        self.items.append(x)
        return x


def serve(deployment: Deployment, clients: list[ClientView], horizon_s: float, *, epoch_s: float = 0.0,
          latency=None, instances=None, ctx=None, poisson: bool = False, seed: int = 0,
          record_dispatch: bool = False, ingress=None, ingress_from_host: bool = False,
          egress_to_host: bool = False, slot_bytes: int = 0, max_inflight: int = 4096,
          planner: str | None = None, plan_latency=None, return_outputs: bool = False,
          epochs: list | None = None, result_rows: int = 0, sample_outputs: int = 0,
          drain_s: float = 0.0, top1: int = 0, lane_policy: int = 0) -> ServeReport:
    """Run one plan for one horizon.

    latency: callable (StageSpec, k) -> ms for the virtual clock (None -> wall clock).
    instances: per stage index, a list of `StageInstance` (wall clock; with `latency` too: replay).
    ingress: (client id, route point), client id, or route point (first match wins) ->
    (pointer, bytes, channels) of the client's fp32 entry activation (device memory, or pinned host
    memory with `ingress_from_host`).
    slot_bytes: per-request device slot size; 0 lets the library size it from the routes (the
    largest DMA-copied ingress / intermediate boundary); a smaller value than a route needs raises.
    max_inflight: device slots (requests in flight with a slot); result_rows: final outputs kept
    (a ring; 0 = max_inflight) — return_outputs needs result_rows >= completed requests.
    drain_s: wall clock only — after the horizon, keep serving already-generated requests for up
    to this long (no new arrivals), so requests generated near the horizon complete and count.
    sample_outputs: keep the logits of up to this many completed requests still held in the ring
    (the most recent completions, distinct clients first) as report.sampled = (request indices,
    [n, elems] fp32) — output spot-checks of long serving runs.
    top1: GX_TOP1_* (0 none, 1 logits + top-1, 2 top-1 only): the final stage's scatter also writes
    each request's argmax (K9, classifier chains); report.top1 = int32 per request (-1: none).
    lane_policy: GX_LANE_* (graft_exec.h): 0 one lane per hardware queue with 4 queues reserved for
    short stages (default), 1 least-loaded of 64 lanes, 2 the same with stream priorities by expected
    batch time, 3 one lane per hardware queue, earliest expected free lane.
    plan_latency: optional (StageSpec, k) -> ms the plan assumed; on the wall clock it is only
    compared with the observed batch times in the GX_SERVE_DEBUG summary.
    epochs: plan transitions under churn, one entry per epoch (Deployment / None = keep /
    "infeasible"); `deployment` is then ignored and stage indices (latency, instances, the
    dispatch log) run over the concatenated stages of the deployments in epoch order.
    """
    keep = _Keep()
    wall = latency is None
    replay = latency is not None and instances is not None
    gpu = wall or replay
    ids = sorted(c.client_id for c in clients)
    by_id = {c.client_id: c for c in clients}
    # plan transitions (simulator.py:297-349): epochs[e] is the Deployment put in place at epoch
    # e's REPLAN, None keeps the previous one, "infeasible" clears the routes (simulator.py:320-324).
    # Stages of every deployment stay alive (in-flight requests drain on the stages they were
    # routed to); they are numbered in deployment order, as the reference creates _StageRT objects.
    if epochs is None:
        epochs = [deployment]
    deps, eff, cur = [], [], -1
    for e, d in enumerate(epochs):
        if d is None:
            if e == 0:
                raise ValidationError("epoch 0 needs a deployment")
        elif isinstance(d, str):
            if d != "infeasible":
                raise ValidationError(f"bad epoch entry {d!r}")
            cur = -1
        else:
            deps.append(d)
            cur = len(deps) - 1
        eff.append(cur)
    stages, offset = [], []
    for d in deps:
        offset.append(len(stages))
        stages.extend(d.stages)
    st_arr = (N.GxServeStage * max(1, len(stages)))()
    for i, s in enumerate(stages):
        st_arr[i].batch, st_arr[i].instances, st_arr[i].budget_ms = s.batch, s.instances, s.budget_ms
        st_arr[i].out_final = 0
        lat_fn = plan_latency if wall else latency
        if lat_fn is not None:
            lat = (C.c_double * (s.batch + 1))(0.0, *[float(lat_fn(s, k)) for k in range(1, s.batch + 1)])
            st_arr[i].lat_ms = keep(lat)
        if s.gpus is not None:  # placement (placement.py:24-70): GPU of each instance
            if len(s.gpus) != s.instances:
                raise ValidationError(f"stage {s.stage_id}: placement lists {len(s.gpus)} GPUs for {s.instances} "
                                      f"instances")
            st_arr[i].inst_gpu = keep((C.c_int32 * s.instances)(*s.gpus))
        if gpu:
            insts = instances[i]
            if len(insts) != s.instances:
                raise ValidationError(f"stage {s.stage_id}: {len(insts)} executor instances for {s.instances}")
            arr = (C.c_void_p * len(insts))(*[x.handle.value for x in insts])
            st_arr[i].inst = keep(arr)
            st_arr[i].out_final = 1 if insts[0].final else 0
    # one native route per (deployment, client): the reference keeps one _Route per client per plan
    route_docs = []
    route_of = {}
    for di, d in enumerate(deps):
        for cid in ids:
            c = by_id[cid]
            r = d.routes.get(cid)
            if r is None:
                continue
            rt = N.GxServeRoute()
            rt.n_stages = len(r.stages)
            for j, si in enumerate(r.stages):
                rt.stage[j] = offset[di] + si
            rt.worst_rem_ms = r.worst_rem_ms
            rt.mobile_ms = c.mobile_ms[r.point]
            rt.payload_bytes = c.payload_bytes[r.point]
            rt.ingress_dtype = N.GX_F32  # the client wire format (fp32), token ids at a BERT boundary 0
            if gpu and r.stages:
                ch = instances[offset[di] + r.stages[0]][0].model.chain
                if ch.boundary_shape(r.point)[3] == N.GX_I32:
                    rt.ingress_dtype = N.GX_I32
            if ingress is not None:
                key = (cid, r.point) if (cid, r.point) in ingress else cid if cid in ingress else r.point
                ptr, nbytes, channels = ingress[key]
                rt.ingress, rt.ingress_bytes, rt.ingress_channels = ptr, nbytes, channels
            route_docs.append(rt)
            route_of[(di, cid)] = len(route_docs) - 1
    cl_arr = (N.GxServeClient * max(1, len(ids)))()
    for ci, cid in enumerate(ids):
        c = by_id[cid]
        per_epoch = [route_of.get((d, cid), -1) if d >= 0 else -1 for d in eff]
        cl_arr[ci].rate_rps, cl_arr[ci].slo_ms, cl_arr[ci].route = c.rate_rps, c.slo_ms, per_epoch[0]
        if len(per_epoch) > 1:
            er = keep((C.c_int32 * len(per_epoch))(*per_epoch))
            cl_arr[ci].epoch_route, cl_arr[ci].n_epoch_route = er, len(per_epoch)
        if poisson:
            # the reference draws gaps lazily from default_rng((seed, i)) in client-id order
            # (simulator.py:240-242, 382-384); draw enough of the same stream up front
            rng = np.random.default_rng((seed, ci))
            n = int(horizon_s * c.rate_rps * 3 + 64)
            gaps = rng.exponential(1000.0 / c.rate_rps, size=n)
            g = keep((C.c_double * n)(*gaps))
            cl_arr[ci].gen_gaps_ms, cl_arr[ci].n_gaps = g, n
        tt = keep((C.c_double * len(c.trace_t_s))(*c.trace_t_s))
        tm = keep((C.c_double * len(c.trace_mbps))(*c.trace_mbps))
        cl_arr[ci].trace_t_s, cl_arr[ci].trace_mbps, cl_arr[ci].n_trace = tt, tm, len(c.trace_t_s)
    rt_arr = (N.GxServeRoute * max(1, len(route_docs)))(*route_docs)
    cfg = N.GxServeCfg()
    cfg.horizon_ms = horizon_s * 1000.0
    cfg.epoch_ms = epoch_s * 1000.0
    cfg.clock = N.GX_CLOCK_WALL if wall else N.GX_CLOCK_REPLAY if replay else N.GX_CLOCK_VIRTUAL
    cfg.record_dispatch = 1 if record_dispatch else 0
    # True / "zero_copy": the gather reads pinned host memory over PCIe; "dma": copy at arrival
    cfg.ingress_from_host = {False: 0, True: 1, "zero_copy": 1, "dma": 2}[ingress_from_host]
    cfg.egress_to_host = 1 if egress_to_host else 0
    cfg.slot_bytes = slot_bytes
    cfg.max_inflight = max_inflight
    cfg.result_rows = result_rows
    cfg.drain_ms = drain_s * 1000.0 if wall else 0.0
    cfg.top1 = int(top1)
    cfg.lane_policy = int(lane_policy)
    L = N.lib()
    h = C.c_void_p()
    ctx_handle = ctx.handle if ctx is not None else C.c_void_p(0)
    if gpu and ctx is None:
        raise ValidationError("executing batches needs an executor context")
    if not gpu and ctx is None:
        ctx_handle = C.c_void_p(1)  # virtual clock never touches the device; any non-null handle
    N.check(L.gx_serve_create(ctx_handle, len(stages), st_arr, len(route_docs), rt_arr, len(ids), cl_arr,
                              C.byref(cfg), C.byref(h)), "gx_serve_create")
    try:
        N.check(L.gx_serve_run(h), "gx_serve_run")
        n = C.c_int64()
        N.check(L.gx_serve_count_requests(h, C.byref(n)))
        n = n.value
        cl = np.zeros(n, np.int32)
        gen = np.zeros(n)
        done = np.zeros(n)
        dl = np.zeros(n)
        status = np.zeros(n, np.int32)
        P = lambda a, t: a.ctypes.data_as(C.POINTER(t))  # noqa: E731
        N.check(L.gx_serve_requests(h, P(cl, C.c_int32), P(gen, C.c_double), P(done, C.c_double), P(dl, C.c_double),
                                    P(status, C.c_int32)))
        wall_ms = C.c_double()
        nb = C.c_int64()
        nk = C.c_int64()
        N.check(L.gx_serve_stats(h, C.byref(wall_ms), C.byref(nb), C.byref(nk)))
        top1_out = None
        if top1 and gpu:
            top1_out = np.full(n, -1, np.int32)
            held = C.c_int64()
            allreq = np.arange(n, dtype=np.int64)
            N.check(L.gx_serve_top1_for(h, n, allreq.ctypes.data_as(C.POINTER(C.c_int64)), P(top1_out, C.c_int32),
                                        C.byref(held)), "gx_serve_top1_for")
        outputs = None
        if return_outputs and gpu and top1 != N.GX_TOP1_ONLY:
            final = [x for x in (instances or []) if x and x[0].final]
            elems = final[0][0].out_elems if final else 0
            outputs = np.zeros((max(1, n), max(1, elems)), np.float32)
            if elems:
                N.check(L.gx_serve_outputs(h, outputs.ctypes.data_as(C.POINTER(C.c_float)), outputs.shape[0], elems),
                        "gx_serve_outputs")
        sampled = None
        if sample_outputs and gpu and top1 != N.GX_TOP1_ONLY:
            final = [x for x in (instances or []) if x and x[0].final]
            elems = final[0][0].out_elems if final else 0
            comp = np.nonzero(status == 0)[0]
            if elems and comp.size:
                order = np.ascontiguousarray(comp[np.argsort(done[comp], kind="stable")][::-1][:4 * sample_outputs],
                                             dtype=np.int64)
                arr = np.empty((order.size, elems), np.float32)
                held = C.c_int64()
                N.check(L.gx_serve_outputs_for(h, order.size, order.ctypes.data_as(C.POINTER(C.c_int64)),
                                               arr.ctypes.data_as(C.POINTER(C.c_float)), elems, C.byref(held)),
                        "gx_serve_outputs_for")
                good = [j for j in range(order.size) if not np.isnan(arr[j]).any()]
                seen, pick = set(), []
                for j in good:  # distinct clients first, then repeats
                    if cl[order[j]] not in seen:
                        seen.add(cl[order[j]])
                        pick.append(j)
                pick += [j for j in good if j not in set(pick)][:max(0, sample_outputs - len(pick))]
                pick = sorted(pick[:sample_outputs])
                sampled = (order[pick], arr[pick])
        dispatch = placement = None
        if record_dispatch:
            nbat = C.c_int64()
            nit = C.c_int64()
            N.check(L.gx_serve_count_dispatch(h, C.byref(nbat), C.byref(nit)))
            t = np.zeros(nbat.value)
            si = np.zeros(nbat.value, np.int32)
            kk = np.zeros(nbat.value, np.int32)
            sq = np.zeros(nit.value, np.int64)
            N.check(L.gx_serve_dispatch(h, P(t, C.c_double), P(si, C.c_int32), P(kk, C.c_int32), P(sq, C.c_int64)))
            dispatch = []
            off = 0
            for i in range(nbat.value):
                dispatch.append((float(t[i]), int(si[i]), int(kk[i]), tuple(int(x) for x in sq[off:off + kk[i]])))
                off += kk[i]
            pi = np.zeros(nbat.value, np.int32)
            pg = np.zeros(nbat.value, np.int32)
            N.check(L.gx_serve_dispatch_placement(h, P(pi, C.c_int32), P(pg, C.c_int32)))
            placement = [(int(a), int(b)) for a, b in zip(pi, pg)]
    finally:
        L.gx_serve_destroy(h)
    rep = _report(planner or deps[0].planner, horizon_s, ids, cl, gen, done, dl, status,
                  {"clock": "wall" if wall else "replay" if replay else "virtual", "horizon_s": horizon_s,
                   "poisson": poisson, "seed": seed, "clients": len(ids)})
    rep.dispatch = dispatch
    rep.placement = placement
    rep.outputs = outputs
    rep.sampled = sampled
    rep.top1 = top1_out
    rep.wall_ms, rep.batches, rep.kernels = float(wall_ms.value), int(nb.value), int(nk.value)
    return rep


def slo_met_rps(rep: ServeReport) -> float:
    """SLO-met requests/sec over the horizon."""
    return rep.slo_met / rep.horizon_s if rep.horizon_s > 0 else math.nan
