"""Per-GPU executor context and single-op launch helpers over torch device tensors.

torch is the plumbing here (device memory, streams); every kernel that runs is libgx's.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _native as N
from .errors import InfeasibleError

_CTXS: dict[int, "Context"] = {}


class Context:
    """One libgx context per CUDA device (gx_init)."""

    def __init__(self, device: int = 0):
        if not torch.cuda.is_available():
            raise InfeasibleError("no CUDA device: the B200 executor has no CPU path")
        self.device = device
        self.handle = C.c_void_p()
        with torch.cuda.device(device):
            N.check(N.lib().gx_init(device, C.byref(self.handle)), "gx_init")
        n = C.c_int()
        N.check(N.lib().gx_sm_count(self.handle, C.byref(n)))
        self.sm_count = n.value

    def sm_budget(self, share: int) -> int:
        """MPS-style percentage share -> SM count for bounded persistent grids."""
        if not 1 <= share <= 100:
            raise ValueError(f"gpu share must be an integer in 1..100, got {share}")
        return max(1, -(-share * self.sm_count // 100))

    def sm_budgets(self, shares_instances, capacity: int = 99, work_conserving: bool = True) -> list[int]:
        """SM budget per instance for a whole deployment on this GPU.

        The plan's share is a floor (what the planner was promised).  With
        `work_conserving`, SMs the plan leaves idle are handed out in proportion to the planned
        shares, so a plan using 32% of the GPU does not leave 68% of the SMs dark; the total never
        exceeds `capacity`% of the SMs (placement capacity, placement.py:24)."""
        total = sum(s * n for s, n in shares_instances)
        if total <= 0:
            return []
        scale = max(1.0, capacity / total) if work_conserving else 1.0
        cap = self.sm_count * capacity // 100
        out, floor = [], []
        for s, n in shares_instances:
            f = min(self.sm_budget(s), self.sm_count)  # the profiled budget: never handed out less
            b = max(f, min(int(s * scale * self.sm_count / 100), self.sm_count))
            out.extend([b] * n)
            floor.extend([f] * n)
        # rounding can overshoot the capacity: trim only SMs handed out above the floors
        while sum(out) > cap:
            i = max(range(len(out)), key=lambda j: out[j] - floor[j])
            if out[i] <= floor[i]:
                break
            out[i] -= 1
        return out


def context(device: int = 0) -> Context:
    ctx = _CTXS.get(device)
    if ctx is None:
        ctx = Context(device)
        _CTXS[device] = ctx
    return ctx


def gx_dtype(t: torch.dtype) -> int:
    if t == torch.bfloat16:
        return N.GX_BF16
    if t == torch.float32:
        return N.GX_F32
    raise TypeError(f"unsupported dtype {t}")


def tensor_desc(H, W, Cc, dtype=N.GX_BF16) -> N.GxTensor:
    t = N.GxTensor()
    t.H, t.W, t.C, t.dtype = H, W, Cc, dtype
    return t


def run_op(op: N.GxOp, tensors: list[torch.Tensor], descs: list[N.GxTensor], weights: torch.Tensor,
           k: int, sm_budget: int = 0, stream: torch.cuda.Stream | None = None):
    """Run one op on caller tensors (batch-major, per-sample layout given by `descs`)."""
    ctx = context(tensors[0].device.index or 0)
    stream = stream or torch.cuda.current_stream()
    tarr = (N.GxTensor * len(descs))(*descs)
    parr = N.ptr_array([t.data_ptr() for t in tensors])
    N.check(N.lib().gx_run_op(ctx.handle, C.byref(op), tarr, parr, C.c_void_p(weights.data_ptr()), k,
                              sm_budget, C.c_void_p(stream.cuda_stream)), "gx_run_op")


class WeightBlob:
    """Host-side packing of one model's weights into the layout libgx expects (graft_exec.h)."""

    ALIGN = 1024

    def __init__(self):
        self.parts: list[np.ndarray] = []
        self.size = 0

    def _add(self, arr: np.ndarray) -> int:
        raw = np.ascontiguousarray(arr).view(np.uint8).reshape(-1)
        off = self.size
        pad = (-raw.size) % self.ALIGN
        self.parts.append(raw)
        if pad:
            self.parts.append(np.zeros(pad, np.uint8))
        self.size += raw.size + pad
        return off

    def add_bf16(self, t: torch.Tensor) -> int:
        return self._add(t.detach().to(torch.bfloat16).contiguous().view(torch.int16).cpu().numpy())

    def add_f32(self, t: torch.Tensor) -> int:
        return self._add(t.detach().to(torch.float32).contiguous().cpu().numpy())

    def bytes(self) -> np.ndarray:
        if not self.parts:
            return np.zeros(self.ALIGN, np.uint8)
        return np.concatenate(self.parts)


def pack_conv_weight(w: torch.Tensor, cin_pad: int | None = None) -> torch.Tensor:
    """[Cout, Cin, R, S] fp32 -> [Cout, Kpad] with K ordered (r, s, cin), zero padded."""
    cout, cin, r, s = w.shape
    cin_pad = cin_pad or cin
    wt = w.permute(0, 2, 3, 1)  # Cout, R, S, Cin
    if cin_pad != cin:
        wt = torch.nn.functional.pad(wt, (0, cin_pad - cin))
    wt = wt.reshape(cout, r * s * cin_pad)
    kpad = -(-wt.shape[1] // 64) * 64
    if kpad != wt.shape[1]:
        wt = torch.nn.functional.pad(wt, (0, kpad - wt.shape[1]))
    return wt.contiguous()
