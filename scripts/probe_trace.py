"""Print the on-device timeline of one persistent span launch (development aid)."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

from paper_2312_10636_b200 import _native as N  # noqa: E402
from paper_2312_10636_b200.engine import DeviceModel, StageInstance  # noqa: E402
from paper_2312_10636_b200.models import build_chain  # noqa: E402

NAMES = {1: "conv", 2: "maxpool", 3: "avgpool", 4: "gap", 5: "fc", 6: "linear", 10: "copy"}
budget = int(sys.argv[1]) if len(sys.argv) > 1 else 4
k = int(sys.argv[2]) if len(sys.argv) > 2 else 1
a, b = (int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "0,18").split(","))
chain = build_chain("resnet50")
dm = DeviceModel(chain)
st = StageInstance(dm, a, b, 16, budget)
L = N.lib()
L.gx_stage_span_trace.restype = C.c_int32
L.gx_stage_span_trace.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_int64), C.c_int64, C.POINTER(C.c_int)]
cap = budget * 200 * 4
buf = (C.c_int64 * cap)()
nops = C.c_int()
for _ in range(3):
    N.check(L.gx_stage_span_trace(st.handle, k, buf, cap, C.byref(nops)))
n = nops.value
t = np.array(buf[: budget * n * 4], dtype=np.int64).reshape(budget, n, 4).astype(np.float64)
t0 = t[t > 0].min()
t = np.where(t > 0, (t - t0) / 1000.0, np.nan)
ops = [chain.ops[i] for i in range(chain.unit_first_op[a], chain.unit_first_op[b])]
print(f"span [{a},{b}) budget={budget} k={k}: total {np.nanmax(t):.1f} us over {n} ops")
prev_end = 0.0
for j in range(n):
    op = ops[j]
    start = np.nanmin(t[:, j, 2])
    end = np.nanmax(t[:, j, 3])
    pa0 = np.nanmin(t[:, j, 0])
    pa1 = np.nanmax(t[:, j, 1])
    desc = NAMES.get(op.kind, str(op.kind))
    if op.kind == 1:
        desc += f" {op.R}x{op.S}/{op.sh} {op.Cin}->{op.Cout}" + (" +res" if op.in2 >= 0 else "")
    print(f"{j:3d} {desc:28s} start {start:8.1f} end {end:8.1f} dur {end - prev_end:7.1f} us  "
          f"prodA [{pa0:8.1f}, {pa1:8.1f}]")
    prev_end = end
