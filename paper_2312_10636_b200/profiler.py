"""B200 profile sweep -> the reference's profile CSV (profiles.py:24, 405-454).

Each row is the measured latency of one span [a, b) at batch k on an SM budget equal to the GPU
share, including the ragged gather and the output scatter (the reference budgets inter-stage
transfer as 0 ms; measuring it keeps the planner's budgets honest).  Rows are made
monotone (non-decreasing in batch, non-increasing in share) before writing, because
TableCostModel rejects non-monotone tables (profiles.py:347-371) and measurement noise is not
a property of the span.
"""
from __future__ import annotations

import math
from pathlib import Path

import numpy as np

from .device import context
from .engine import DeviceModel, StageInstance

PROFILE_HEADER = "model,start_layer,end_layer,batch,gpu_share,latency_ms"


class Background:
    """Keeps the SMs outside the measured instance busy with a full-model batch-16 instance on its
    own stream, so profiled latencies include HBM/L2 contention from co-located stages (the
    serving condition: the placement packs a GPU to 99%, placement.py:24)."""

    def __init__(self, dmodel: DeviceModel):
        import threading

        import torch

        self.dm = dmodel
        self.torch = torch
        self.threading = threading
        self.inst = {}
        chain = dmodel.chain
        self.src = torch.randn(chain.boundary_elems(0), device=f"cuda:{dmodel.device}")
        self.dst = torch.empty(16 * chain.boundary_elems(chain.n_units), device=f"cuda:{dmodel.device}")
        self.thread = None

    def start(self, sm_budget: int):
        from . import _native as N

        if sm_budget < 1:
            return
        inst = self.inst.get(sm_budget)
        if inst is None:
            inst = StageInstance(self.dm, 0, self.dm.n_units, 16, sm_budget)
            self.inst[sm_budget] = inst
        chain = self.dm.chain
        out = chain.boundary_elems(chain.n_units)
        srcs = [self.src.data_ptr()] * 16
        dsts = [self.dst.data_ptr() + i * out * 4 for i in range(16)]
        self.stop_flag = False

        def loop():
            while not self.stop_flag:
                for _ in range(3):
                    inst.run_ptrs(16, srcs, [N.GX_F32] * 16, dsts, N.GX_F32, chain.input_channels)
                inst.stream.synchronize()

        self.thread = self.threading.Thread(target=loop, daemon=True)
        self.thread.start()

    def stop(self):
        if self.thread is not None:
            self.stop_flag = True
            self.thread.join()
            self.thread = None


def sweep(dmodel: DeviceModel, spans, batches, shares, iters: int = 10, log=None, contended: bool = False,
          capacity: int = 99) -> list[tuple]:
    ctx = context(dmodel.device)
    bg = Background(dmodel) if contended else None
    rows = []
    for a, b in spans:
        grid = np.full((len(batches), len(shares)), np.nan)
        for j, share in enumerate(shares):
            budget = ctx.sm_budget(share)
            st = StageInstance(dmodel, a, b, max(batches), budget)
            for k in batches:
                st.kernel_count(k)  # capture before the background starts
            if bg is not None:
                bg.start(ctx.sm_count * capacity // 100 - budget)
            try:
                for i, k in enumerate(batches):
                    grid[i, j] = st.profile(k, iters)
            finally:
                if bg is not None:
                    bg.stop()
            del st
        # monotone upper envelope: non-decreasing in batch, non-increasing in share
        grid = np.maximum.accumulate(grid, axis=0)
        order = np.argsort(shares)
        g2 = grid[:, order]
        g2 = np.maximum.accumulate(g2[:, ::-1], axis=1)[:, ::-1]
        grid[:, order] = g2
        for i, k in enumerate(batches):
            for j, share in enumerate(shares):
                rows.append((dmodel.chain.model_id, a, b, k, share, float(grid[i, j])))
        if log:
            log(f"span [{a},{b}) k=1..{max(batches)} share 100: "
                + " ".join(f"{grid[i, shares.index(100)] if 100 in shares else grid[i, -1]:.3f}"
                           for i in range(len(batches))))
    return rows


def write_csv(rows, path, echo: dict | None = None):
    lines = []
    for k, v in (echo or {}).items():
        lines.append(f"# {k}={v}")
    lines.append(PROFILE_HEADER)
    for m, a, b, k, s, lat in rows:
        lines.append(f"{m},{a},{b},{k},{s},{lat:.6f}")
    Path(path).write_text("\n".join(lines) + "\n")


def read_csv(path) -> dict:
    """(model, a, b, k, share) -> ms (the rows a TableCostModel would ingest)."""
    out = {}
    for ln in Path(path).read_text().splitlines():
        if not ln or ln.startswith("#") or ln.startswith("model,"):
            continue
        m, a, b, k, s, lat = ln.split(",")
        out[(m, int(a), int(b), int(k), int(s))] = float(lat)
    return out


class TableLatency:
    """Conservative lookup with the TableCostModel rule (round batch up, share down;
    profiles.py:373-385), for the executor's own virtual-clock runs."""

    def __init__(self, table: dict):
        self.cells = {}
        for (m, a, b, k, s), v in table.items():
            self.cells.setdefault((m, a, b), {})[(k, s)] = v

    def __call__(self, model_id, start, end, batch, share) -> float:
        if start == end:
            return 0.0
        cells = self.cells.get((model_id, start, end))
        if not cells:
            return math.inf
        best = math.inf
        for (k, s), v in cells.items():
            if k >= batch and s <= share:
                best = min(best, v)
        return best
