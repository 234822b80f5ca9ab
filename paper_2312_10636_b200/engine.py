"""Executor objects over libgx: a unit chain resident on one GPU and its stage instances.

`DeviceModel` is a ModelSpec (profiles.py:31-87) made executable; `StageInstance` is one
instance of a planned stage (StagePlan, realign.py:50-67; _StageRT, simulator.py:76-100): span
[start, end), max batch b, SM budget from the plan's share.  `StageInstance.run` is the real
execution behind _StageRT.latency_for(k).
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _native as N
from .device import context
from .errors import ValidationError
from .models import UnitChain


class DeviceModel:
    def __init__(self, chain: UnitChain, device: int = 0):
        self.chain = chain
        self.device = device
        self.ctx = context(device)
        descs = (N.GxTensor * len(chain.tensors))()
        for i, (H, W, Cc, dt) in enumerate(chain.tensors):
            descs[i].H, descs[i].W, descs[i].C, descs[i].dtype = H, W, Cc, dt
            descs[i].s2d = chain.tensor_s2d.get(i, 0)
        ops = (N.GxOp * len(chain.ops))(*chain.ops)
        blob = chain.blob.bytes()
        self.handle = C.c_void_p()
        with torch.cuda.device(device):
            N.check(N.lib().gx_model_create(
                self.ctx.handle, chain.model_id.encode(), len(chain.tensors), descs, len(chain.ops), ops,
                chain.n_units, N.i32_array(chain.unit_first_op), N.i32_array(chain.boundary),
                blob.ctypes.data_as(C.c_void_p), blob.nbytes, C.byref(self.handle)), "gx_model_create")
        self.weight_bytes = blob.nbytes
        dt = C.c_int32()
        N.check(N.lib().gx_model_dtype(self.handle, C.byref(dt)))
        self.dtype = dt.value  # GX_BF16 or GX_F32 (fp32 execution mode)

    @property
    def n_units(self) -> int:
        return self.chain.n_units

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                N.lib().gx_model_destroy(h)
            except Exception:  # noqa: BLE001 - interpreter teardown
                pass
            self.handle = None


def _gx_dtype(t: torch.Tensor) -> int:
    """Element type of a request's entry tensor: fp32 client ingress, bf16 from an alignment
    stage, int32 token ids (BERT boundary 0)."""
    return {torch.float32: N.GX_F32, torch.bfloat16: N.GX_BF16, torch.int32: N.GX_I32}[t.dtype]


def placed_instances(dep, models: dict, work_conserving: bool = True, capacity: int = 99) -> list:
    """Executor instances of a deployment placed across the GPUs of one box: instance i of stage s
    runs on GPU s.gpus[i] (the plan's placement, placement.py:24-70; None = GPU 0).  `models` maps
    a plan GPU index to the DeviceModel resident on it.  SM budgets are assigned per GPU from the
    shares of the instances placed on that GPU (Context.sm_budgets; `capacity` > 100 oversubscribes,
    DESIGN.md §6.1)."""
    per_gpu = {}
    for si, s in enumerate(dep.stages):
        for i, g in enumerate(s.gpus if s.gpus is not None else (0,) * s.instances):
            per_gpu.setdefault(g, []).append((si, i, s.share))
    budget = {}
    for g, lst in per_gpu.items():
        if g not in models:
            raise ValidationError(f"plan places instances on GPU {g} but no model is resident there")
        bs = models[g].ctx.sm_budgets([(share, 1) for _si, _i, share in lst], capacity=capacity,
                                      work_conserving=work_conserving)
        for (si, i, _share), b in zip(lst, bs):
            budget[(si, i)] = (g, b)
    out = []
    for si, s in enumerate(dep.stages):
        row = []
        for i in range(s.instances):
            g, b = budget[(si, i)]
            row.append(StageInstance(models[g], s.start, s.end, s.batch, b))
        out.append(row)
    return out


class StageInstance:
    """One executor instance of span [start, end) bounded to `sm_budget` SMs."""

    def __init__(self, model: DeviceModel, start: int, end: int, max_batch: int, sm_budget: int,
                 stream: torch.cuda.Stream | None = None, exec_mode: int = N.GX_EXEC_GRAPH):
        if not 0 <= start < end <= model.n_units:
            raise ValidationError(f"bad span [{start}, {end}) for model {model.chain.model_id!r}")
        self.model = model
        self.start, self.end, self.max_batch, self.sm_budget = start, end, max_batch, sm_budget
        self.handle = C.c_void_p()
        # the stream is torch-owned so tensors freed on it are tracked by torch's allocator
        self.stream = stream or torch.cuda.Stream(device=model.device)
        with torch.cuda.device(model.device):
            N.check(N.lib().gx_stage_create(model.handle, start, end, max_batch, sm_budget, model.dtype,
                                            C.c_void_p(self.stream.cuda_stream), C.byref(self.handle)),
                    "gx_stage_create")
            if exec_mode != N.GX_EXEC_GRAPH:
                N.check(N.lib().gx_stage_set_exec(self.handle, exec_mode), "gx_stage_set_exec")
        chain = model.chain
        self.in_channels = chain.boundary_shape(start)[2]
        self.out_elems = chain.boundary_elems(end)
        self.final = end == chain.n_units
        self.dtype = model.dtype
        # element type of the stage output: fp32 logits, else the chain's compute type
        self.out_dtype = N.GX_F32 if self.final else model.dtype
        self.out_elem_bytes = 4 if self.out_dtype == N.GX_F32 else 2

    def run_ptrs(self, k: int, src, src_dtypes, dst, dst_dtype: int, src_channels: int = 0):
        N.check(N.lib().gx_stage_run(self.handle, k, N.ptr_array(src), N.i32_array(src_dtypes), src_channels,
                                     N.ptr_array(dst), dst_dtype), "gx_stage_run")

    def run(self, inputs: list[torch.Tensor], out_dtype: torch.dtype | None = None,
            src_channels: int = 0) -> list[torch.Tensor]:
        """Execute one batch: inputs are per-request entry activations (NHWC, fp32 or bf16)."""
        k = len(inputs)
        if not 1 <= k <= self.max_batch:
            raise ValidationError(f"batch {k} outside 1..{self.max_batch}")
        out_dtype = out_dtype or (torch.float32 if self.out_dtype == N.GX_F32 else torch.bfloat16)
        dev = torch.device("cuda", self.model.device)
        outs = [torch.empty(self.out_elems, dtype=out_dtype, device=dev) for _ in range(k)]
        cur = torch.cuda.current_stream(dev)
        self.stream.wait_stream(cur)
        self.run_ptrs(k, [t.data_ptr() for t in inputs], [_gx_dtype(t) for t in inputs],
                      [o.data_ptr() for o in outs], N.GX_F32 if out_dtype == torch.float32 else N.GX_BF16,
                      src_channels)
        cur.wait_stream(self.stream)
        return outs

    def run_top1(self, inputs: list[torch.Tensor], logits: bool = True, src_channels: int = 0):
        """Execute one batch of a classifier's final stage with the top-1 (K9) fused into the
        scatter: returns (per-request fp32 logits or None, int32 [k] argmax on the device)."""
        k = len(inputs)
        if not self.final:
            raise ValidationError("top-1 is computed by the stage that ends at the chain output")
        if not 1 <= k <= self.max_batch:
            raise ValidationError(f"batch {k} outside 1..{self.max_batch}")
        dev = torch.device("cuda", self.model.device)
        outs = [torch.empty(self.out_elems, dtype=torch.float32, device=dev) for _ in range(k)] if logits else None
        top1 = torch.full((k,), -1, dtype=torch.int32, device=dev)
        cur = torch.cuda.current_stream(dev)
        self.stream.wait_stream(cur)
        N.check(N.lib().gx_stage_run_top1(self.handle, None, k, N.ptr_array([t.data_ptr() for t in inputs]),
                                          N.i32_array([_gx_dtype(t) for t in inputs]), src_channels,
                                          N.ptr_array([o.data_ptr() for o in outs]) if logits else None,
                                          N.ptr_array([top1.data_ptr() + 4 * i for i in range(k)]), None),
                "gx_stage_run_top1")
        cur.wait_stream(self.stream)
        return outs, top1

    def profile(self, k: int, iters: int = 20) -> float:
        ms = C.c_float()
        N.check(N.lib().gx_stage_profile(self.handle, k, iters, C.byref(ms)), "gx_stage_profile")
        return float(ms.value)

    def profile_ops(self, k: int, iters: int = 20) -> list[dict]:
        """Each op of the span alone at batch k: median ms and algorithmic FLOPs / bytes."""
        L = N.lib()
        n = C.c_int()
        N.check(L.gx_stage_op_count(self.handle, C.byref(n)))
        n = n.value
        ms, fl, by, kd = (C.c_float * n)(), (C.c_double * n)(), (C.c_double * n)(), (C.c_int32 * n)()
        N.check(L.gx_stage_profile_ops(self.handle, k, iters, n, ms, fl, by, kd), "gx_stage_profile_ops")
        # logical FLOPs of convs with zero-padded channels (UnitChain.op_flops_scale)
        chain = self.model.chain
        first = chain.unit_first_op[self.start]
        scale = [getattr(chain, "op_flops_scale", {}).get(first + i, 1.0) for i in range(n)]
        return [{"op": i, "kind": int(kd[i]), "ms": float(ms[i]), "flops": float(fl[i]) * scale[i],
                 "bytes": float(by[i])} for i in range(n)]

    def kernel_count(self, k: int) -> int:
        n = C.c_int()
        N.check(N.lib().gx_stage_kernel_count(self.handle, k, C.byref(n)))
        return n.value

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                N.lib().gx_stage_destroy(h)
            except Exception:  # noqa: BLE001
                pass
            self.handle = None
