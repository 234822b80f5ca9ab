"""ctypes binding of libgx (include/graft_exec.h).

There is no CPU fallback: importing the executor without the built library, or creating a
context without a B200, raises.  Errors from the C ABI are mapped onto the reference's
exception hierarchy (fragserve/errors.py:4-17) via `errors.raise_for_status`.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

from .errors import raise_for_status

LIB_PATH = Path(__file__).resolve().parent / "_gx.so"
ABI_VERSION = 3

GX_BF16, GX_F32, GX_I32 = 0, 1, 2
(GX_OP_CONV, GX_OP_MAXPOOL, GX_OP_AVGPOOL, GX_OP_GAP, GX_OP_FC, GX_OP_LINEAR, GX_OP_LAYERNORM,
 GX_OP_ATTENTION, GX_OP_EMBED, GX_OP_COPY, GX_OP_FLATTEN_NCHW) = range(1, 12)
GX_ACT_NONE, GX_ACT_RELU, GX_ACT_GELU = 0, 1, 2
GX_OPF_COUNT_INCLUDE_PAD, GX_OPF_NO_HALO, GX_OPF_FC_SIMT, GX_OPF_DS = 1, 2, 4, 8
GX_CLOCK_VIRTUAL, GX_CLOCK_WALL, GX_CLOCK_REPLAY = 0, 1, 2
GX_EXEC_GRAPH, GX_EXEC_SPAN = 0, 1
GX_TOP1_NONE, GX_TOP1_WITH_LOGITS, GX_TOP1_ONLY = 0, 1, 2
GX_LANE_SPLIT, GX_LANE_LEAST_LOADED, GX_LANE_PRIO_BY_TIME, GX_LANE_EARLIEST, GX_LANE_EDF = 0, 1, 2, 3, 4


class GxTensor(C.Structure):
    _fields_ = [("H", C.c_int32), ("W", C.c_int32), ("C", C.c_int32), ("dtype", C.c_int32), ("s2d", C.c_int32)]


class GxOp(C.Structure):
    _fields_ = [
        ("kind", C.c_int32), ("in_", C.c_int32), ("in2", C.c_int32), ("out", C.c_int32),
        ("out_coff", C.c_int32), ("act", C.c_int32),
        ("R", C.c_int32), ("S", C.c_int32), ("sh", C.c_int32), ("sw", C.c_int32),
        ("ph", C.c_int32), ("pw", C.c_int32), ("Cin", C.c_int32), ("Cout", C.c_int32),
        ("heads", C.c_int32), ("flags", C.c_int32),
        ("w_off", C.c_int64), ("b_off", C.c_int64), ("w2_off", C.c_int64), ("w3_off", C.c_int64),
        ("eps", C.c_float), ("ph_hi", C.c_int32), ("pw_hi", C.c_int32), ("reserved", C.c_int32),
    ]


def make_op(kind, in_, out, in2=-1, out_coff=0, act=GX_ACT_NONE, R=1, S=1, sh=1, sw=1, ph=0, pw=0,
            Cin=0, Cout=0, heads=0, flags=0, w_off=-1, b_off=-1, w2_off=-1, w3_off=-1, eps=0.0, ph_hi=-1,
            pw_hi=-1, reserved=0):
    op = GxOp()
    op.kind, op.in_, op.in2, op.out, op.out_coff, op.act = kind, in_, in2, out, out_coff, act
    op.R, op.S, op.sh, op.sw, op.ph, op.pw = R, S, sh, sw, ph, pw
    op.Cin, op.Cout, op.heads, op.flags = Cin, Cout, heads, flags
    op.w_off, op.b_off, op.w2_off, op.w3_off, op.eps = w_off, b_off, w2_off, w3_off, eps
    op.ph_hi, op.pw_hi, op.reserved = ph_hi, pw_hi, reserved
    return op


class GxServeStage(C.Structure):
    _fields_ = [("batch", C.c_int32), ("instances", C.c_int32), ("budget_ms", C.c_double),
                ("lat_ms", C.POINTER(C.c_double)), ("inst", C.POINTER(C.c_void_p)),
                ("in_boundary_elems_is_input", C.c_int32), ("out_final", C.c_int32),
                ("inst_gpu", C.POINTER(C.c_int32))]


class GxServeRoute(C.Structure):
    _fields_ = [("n_stages", C.c_int32), ("stage", C.c_int32 * 2), ("worst_rem_ms", C.c_double),
                ("mobile_ms", C.c_double), ("payload_bytes", C.c_int64), ("ingress", C.c_void_p),
                ("ingress_bytes", C.c_int64), ("ingress_dtype", C.c_int32), ("ingress_channels", C.c_int32)]


class GxServeClient(C.Structure):
    _fields_ = [("rate_rps", C.c_double), ("slo_ms", C.c_double), ("route", C.c_int32),
                ("gen_gaps_ms", C.POINTER(C.c_double)), ("n_gaps", C.c_int64),
                ("trace_t_s", C.POINTER(C.c_double)), ("trace_mbps", C.POINTER(C.c_double)),
                ("n_trace", C.c_int64), ("epoch_route", C.POINTER(C.c_int32)), ("n_epoch_route", C.c_int64)]


class GxServeCfg(C.Structure):
    _fields_ = [("horizon_ms", C.c_double), ("epoch_ms", C.c_double), ("clock", C.c_int32),
                ("record_dispatch", C.c_int32), ("ingress_from_host", C.c_int32),
                ("egress_to_host", C.c_int32), ("slot_bytes", C.c_int64),
                ("max_inflight", C.c_int32), ("warmup_requests_skip", C.c_int32), ("result_rows", C.c_int64),
                ("drain_ms", C.c_double), ("top1", C.c_int32), ("lane_policy", C.c_int32)]


_lib = None


def lib():
    """Load libgx once.  Raises if the library was not built (no silent fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(
            f"libgx not built: {LIB_PATH} is missing; run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(str(LIB_PATH))
    vp, i32, i64, dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    P = C.POINTER
    sig = {
        "gx_abi_version": (i32, []),
        "gx_last_error": (i32, [C.c_char_p, C.c_size_t]),
        "gx_init": (i32, [C.c_int, P(vp)]),
        "gx_destroy": (i32, [vp]),
        "gx_sm_count": (i32, [vp, P(C.c_int)]),
        "gx_model_create": (i32, [vp, C.c_char_p, C.c_int, P(GxTensor), C.c_int, P(GxOp), C.c_int,
                                  P(i32), P(i32), vp, C.c_size_t, P(vp)]),
        "gx_model_destroy": (i32, [vp]),
        "gx_model_tensor_elems": (i32, [vp, C.c_int, P(i64)]),
        "gx_model_dtype": (i32, [vp, P(i32)]),
        "gx_stage_create": (i32, [vp, C.c_int, C.c_int, C.c_int, C.c_int, i32, vp, P(vp)]),
        "gx_stage_run_async": (i32, [vp, vp, C.c_int, P(vp), P(i32), i32, P(vp), i32, vp]),
        "gx_stage_run_top1": (i32, [vp, vp, C.c_int, P(vp), P(i32), i32, P(vp), P(vp), vp]),
        "gx_stage_set_exec": (i32, [vp, i32]),
        "gx_stage_destroy": (i32, [vp]),
        "gx_stage_stream": (i32, [vp, P(vp)]),
        "gx_stage_run": (i32, [vp, C.c_int, P(vp), P(i32), i32, P(vp), i32]),
        "gx_stage_profile": (i32, [vp, C.c_int, C.c_int, P(C.c_float)]),
        "gx_stage_kernel_count": (i32, [vp, C.c_int, P(C.c_int)]),
        "gx_stage_op_count": (i32, [vp, P(C.c_int)]),
        "gx_debug_trace": (i32, [P(i64), i64]),
        "gx_stage_profile_ops": (i32, [vp, C.c_int, C.c_int, C.c_int, P(C.c_float), P(dbl), P(dbl), P(i32)]),
        "gx_run_op": (i32, [vp, P(GxOp), P(GxTensor), P(vp), vp, C.c_int, C.c_int, vp]),
        "gx_gather": (i32, [vp, C.c_int, P(vp), P(i32), i64, i32, i32, vp, C.c_int, vp]),
        "gx_scatter": (i32, [vp, C.c_int, vp, i32, i64, P(vp), i32, C.c_int, vp]),
        "gx_gather_ex": (i32, [vp, C.c_int, P(vp), P(i32), i32, i32, i32, i32, i32, vp, i32, C.c_int, vp]),
        "gx_serve_create": (i32, [vp, C.c_int, P(GxServeStage), C.c_int, P(GxServeRoute), C.c_int,
                                  P(GxServeClient), P(GxServeCfg), P(vp)]),
        "gx_serve_run": (i32, [vp]),
        "gx_serve_count_requests": (i32, [vp, P(i64)]),
        "gx_serve_requests": (i32, [vp, P(i32), P(dbl), P(dbl), P(dbl), P(i32)]),
        "gx_serve_count_dispatch": (i32, [vp, P(i64), P(i64)]),
        "gx_serve_dispatch": (i32, [vp, P(dbl), P(i32), P(i32), P(i64)]),
        "gx_serve_stats": (i32, [vp, P(dbl), P(i64), P(i64)]),
        "gx_serve_dispatch_placement": (i32, [vp, P(i32), P(i32)]),
        "gx_serve_destroy": (i32, [vp]),
        "gx_serve_outputs": (i32, [vp, P(C.c_float), i64, i64]),
        "gx_serve_outputs_for": (i32, [vp, i64, P(i64), P(C.c_float), i64, P(i64)]),
        "gx_serve_top1_for": (i32, [vp, i64, P(i64), P(i32), P(i64)]),
    }
    for name, (res, args) in sig.items():
        if not hasattr(L, name):
            continue
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    if L.gx_abi_version() != ABI_VERSION:
        raise ImportError(f"libgx ABI version {L.gx_abi_version()} != {ABI_VERSION} (rebuild the library)")
    _lib = L
    return L


def last_error() -> str:
    buf = C.create_string_buffer(2048)
    lib().gx_last_error(buf, len(buf))
    return buf.value.decode(errors="replace")


def check(rc: int, what: str = "libgx"):
    if rc != 0:
        raise_for_status(rc, f"{what}: {last_error()}")


def ptr_array(ptrs):
    arr = (C.c_void_p * len(ptrs))()
    for i, p in enumerate(ptrs):
        arr[i] = C.c_void_p(int(p))
    return arr


def i32_array(vals):
    arr = (C.c_int32 * len(vals))()
    for i, v in enumerate(vals):
        arr[i] = int(v)
    return arr
