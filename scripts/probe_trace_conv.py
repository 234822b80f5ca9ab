"""Per-iteration producer / MMA timeline of one conv launch (CTA 0) from the GX_CONV_DBG&16 trace."""
import ctypes as C
import os
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2312_10636_b200 import _native as N  # noqa: E402
from scripts.bench_conv import SHAPES, run  # noqa: E402

name = sys.argv[1]
budget = int(sys.argv[2]) if len(sys.argv) > 2 else 3
run(name, *SHAPES[name], budget=budget, iters=1)
buf = (C.c_int64 * (8192 * 4))()
N.check(N.lib().gx_debug_trace(buf, 8192 * 4))
N.check(N.lib().gx_debug_trace(buf, 8192 * 4)) if False else None
a = np.frombuffer(buf, dtype=np.int64).reshape(-1, 4)
n = int((a[:, 1] > 0).sum())
a = a[:n]
t0 = a[0, 0]
print(f"{name} dbg={os.environ.get('GX_CONV_DBG')} iterations={n}")
d_full = np.diff(a[:, 1])
d_prod = np.diff(a[:, 0])
print(f"  MMA thread: full-wait exit interval median {np.median(d_full):.0f} clk, mean {d_full.mean():.0f}")
print(f"  producer:   empty-wait exit interval median {np.median(d_prod):.0f} clk, mean {d_prod.mean():.0f}")
print(f"  MMA issue span (full->commit) median {np.median(a[:, 2] - a[:, 1]):.0f} clk")
print(f"  producer lead (MMA full exit - producer empty exit) median {np.median(a[:, 1] - a[:, 0]):.0f} clk")
for i in range(0, min(n, 24)):
    print(f"  it {i:3d}: prod {a[i,0]-t0:8d}  mma_full {a[i,1]-t0:8d}  mma_commit {a[i,2]-t0:8d}")
