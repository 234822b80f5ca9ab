"""Per-tile epilogue / MMA timeline of one conv launch (CTA 0) from the GX_CONV_DBG&16 trace."""
import ctypes as C
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2312_10636_b200 import _native as N  # noqa: E402
from scripts.bench_conv import SHAPES, run  # noqa: E402

name = sys.argv[1]
budget = int(sys.argv[2]) if len(sys.argv) > 2 else 3
run(name, *SHAPES[name], budget=budget, iters=1)
n = 8 * 8192 + 4096
buf = (C.c_int64 * n)()
N.check(N.lib().gx_debug_trace(buf, n))
a = np.frombuffer(buf, dtype=np.int64)
kb = a[:4 * 8192].reshape(-1, 4)
ep = a[4 * 8192:8 * 8192].reshape(-1, 4)
mm = a[8 * 8192:8 * 8192 + 4096]
nt = int((ep[:, 0] > 0).sum())
t0 = kb[0, 0]
print(f"{name}: tiles(CTA0)={nt}")
print(f"  epilogue: tfull->emit done median {np.median(ep[:nt,1]-ep[:nt,0]):.0f} clk; emit done->store issued {np.median(ep[:nt,2]-ep[:nt,1]):.0f}")
print(f"  tile interval (tfull exits) median {np.median(np.diff(ep[:nt,0])):.0f} clk; MMA tempty-exit interval {np.median(np.diff(mm[:nt])):.0f}")
for t in range(min(nt, 8)):
    print(f"  t{t}: mma_tempty {mm[t]-t0:7d} epi_tfull {ep[t,0]-t0:7d} emit_done {ep[t,1]-t0:7d} store {ep[t,2]-t0:7d}")
