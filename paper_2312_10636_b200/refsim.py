"""Seam 2 in code: the reference's own simulator driving the B200 executor.

fragserve's `_Sim` (simulator.py:227-498) prices every dispatched batch with a cost-model lookup:
`_service` pops k requests FIFO and schedules `_R_DONE` at now + `_StageRT.latency_for(k)`
(simulator.py:396-416, 95-100).  `b200_sim_class(fragserve.simulator)` returns a `_Sim` subclass
whose batches really execute: the hook is `_push`, where every `_R_DONE` event carries exactly the
batch `_service` just popped (stage, [requests]).  The batch is gathered from each request's
current activation (its client's entry activation, or the output the request's alignment stage
left), run on a `StageInstance` of the stage's span, and each request's output is kept for the
next stage or as its result.  Everything else — arrivals, admission, batching, timers, hand-off,
the report — is the reference's code, unmodified.

Two clocks:
  * measured=False (replay): completion times stay the reference's virtual ones, so records and
    dispatch are bit-identical to `simulate(...)`, and every output is real (numerics parity);
  * measured=True: a batch completes at dispatch time + its measured GPU time (CUDA events around
    the synchronous run), i.e. the reference's event loop with the cost table replaced by the
    B200 — `_StageRT.latency_for` answered by execution.

The reference's `_deploy` cannot resolve merged fragment ids; pass the merged
fragments the planner used as `merged_fragments` and they are used for routing instead.
"""
from __future__ import annotations

from typing import Callable

import torch


class StagePool:
    """Executor instances per planned span (model, start, end, batch, share) on one GPU."""

    def __init__(self, models: dict, ctx, device: int = 0):
        from .engine import StageInstance

        self._make = StageInstance
        self.models = models  # model_id -> DeviceModel
        self.ctx = ctx
        self.device = device
        self.pool = {}

    def instance(self, stage):
        key = (stage.model_id, stage.start, stage.end, stage.batch, stage.share)
        inst = self.pool.get(key)
        if inst is None:
            dm = self.models[stage.model_id]
            inst = self._make(dm, stage.start, stage.end, stage.batch, self.ctx.sm_budget(stage.share))
            self.pool[key] = inst
        return inst


def b200_sim_class(S):
    """A `_Sim` subclass of the given fragserve.simulator module that executes every batch."""

    class B200Sim(S._Sim):
        def __init__(self, scenario, cost, planner, cfg, fixed_plan=None, *, pool: StagePool,
                     ingress: Callable, measured: bool = False, merged_fragments=None):
            super().__init__(scenario, cost, planner, cfg, fixed_plan=fixed_plan)
            self.pool = pool
            self.ingress = ingress  # (client_id, point) -> entry activation (device tensor, fp32)
            self.measured = measured
            self.merged = merged_fragments
            self.current = {}  # request seq -> its activation at its next stage
            self.outputs = {}  # request seq -> final output (host tensor)
            self.batches = []  # (stage span, k, request seqs, GPU ms) per executed batch
            self._ev = None

        def _deploy(self, plan, fragments):
            return super()._deploy(plan, self.merged if self.merged is not None else fragments)

        def _execute(self, stage, batch) -> float:
            inst = self.pool.instance(stage)
            chain = inst.model.chain
            xs = []
            for req in batch:
                x = self.current.pop(req.seq, None)
                if x is None:  # first stage of the route: the client's own entry activation
                    x = self.ingress(req.client_id, stage.start)
                xs.append(x)
            if self._ev is None:
                self._ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            e0, e1 = self._ev
            e0.record(torch.cuda.current_stream())
            outs = inst.run(xs, src_channels=chain.ingress_channels(stage.start))
            e1.record(torch.cuda.current_stream())
            e1.synchronize()
            ms = e0.elapsed_time(e1)
            for req, y in zip(batch, outs):
                if inst.final:
                    self.outputs[req.seq] = y.float().cpu()
                else:
                    self.current[req.seq] = y
            self.batches.append(((stage.start, stage.end), len(batch), tuple(r.seq for r in batch), ms))
            return ms

        def _push(self, t, rank, payload):
            if rank == S._R_DONE:
                stage, batch = payload
                ms = self._execute(stage, batch)
                if self.measured:  # now + measured GPU time instead of now + latency_for(k)
                    t = t - stage.latency_for(len(batch), self.cost) + ms
            super()._push(t, rank, payload)

    return B200Sim

