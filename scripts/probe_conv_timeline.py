"""Tile-level timeline of one conv launch on CTA 0 (development build, GX_CONV_DBG=16): per k-block
the producer's empty-wait exit and the MMA thread's full-wait exit / commit; per tile the MMA
thread's accumulator-free exit and the epilogue's accumulator-full exit / drain end / store issue.

  GX_BUILD_DEV=1 python -c "import __graft_entry__ as g; g.build()"
  GX_CONV_DBG=16 python scripts/probe_conv_timeline.py l1_1x1_256_64 2
"""
import ctypes as C
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2312_10636_b200 import _native as N  # noqa: E402
from scripts.bench_conv import SHAPES, run  # noqa: E402

name = sys.argv[1]
budget = int(sys.argv[2]) if len(sys.argv) > 2 else 2
run(name, *SHAPES[name], budget=budget, iters=1)
n_all = 8 * 8192 + 4096
buf = (C.c_int64 * n_all)()
N.check(N.lib().gx_debug_trace(buf, n_all))
a = np.frombuffer(buf, dtype=np.int64)
kb = a[:4 * 8192].reshape(-1, 4)
epi = a[4 * 8192:8 * 8192].reshape(-1, 4)
mt = a[8 * 8192:8 * 8192 + 4096]
nk = int((kb[:, 1] > 0).sum())
nt = int((epi[:, 0] > 0).sum())
t0 = min(x for x in (kb[0, 0], kb[0, 1], mt[0]) if x > 0)
print(f"{name} budget={budget}: {nk} k-block iterations, {nt} tiles on CTA 0, span {(epi[nt-1,1]-t0)} clk")
print(f"  k-block: MMA full-exit interval median {np.median(np.diff(kb[:nk,1])):.0f} clk; "
      f"producer empty-exit interval median {np.median(np.diff(kb[:nk,0])):.0f}")
print(f"  tile: MMA acc-free interval median {np.median(np.diff(mt[:nt])):.0f} clk; epilogue start interval "
      f"median {np.median(np.diff(epi[:nt,0])):.0f}; epilogue drain (start->end) median "
      f"{np.median(epi[:nt,1]-epi[:nt,0]):.0f}")
print(f"  epilogue start - MMA acc-free (same tile) median {np.median(epi[:nt,0]-mt[:nt]):.0f} clk")
for i in range(min(nk, 12)):
    print(f"  kb {i:3d}: prod_empty_exit {kb[i,0]-t0:8d}  mma_full_exit {kb[i,1]-t0:8d}  mma_commit {kb[i,2]-t0:8d}")
for t in range(min(nt, 12)):
    print(f"  tile {t:3d}: mma_acc_free {mt[t]-t0:8d}  epi_start {epi[t,0]-t0:8d}  epi_end {epi[t,1]-t0:8d}"
          f"  store {epi[t,2]-t0 if epi[t,2] else -1:8d}")
