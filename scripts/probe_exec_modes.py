"""Graph (per-op kernels, PDL) vs span (one persistent kernel, grid barriers) execution of one
stage batch: median span latency per (span, k, budget)."""
import sys

sys.path.insert(0, ".")
from paper_2312_10636_b200 import _native as N  # noqa: E402
from paper_2312_10636_b200.engine import DeviceModel, StageInstance  # noqa: E402
from paper_2312_10636_b200.models import build_chain  # noqa: E402

chain = build_chain("resnet50")
dm = DeviceModel(chain)
for pt in (sys.argv[1] if len(sys.argv) > 1 else "17:18:1:2,15:18:1:2,14:18:2:2,9:18:4:2,2:18:16:2").split(","):
    a, b, k, bud = (int(x) for x in pt.split(":"))
    st = StageInstance(dm, a, b, k, bud)
    g = st.profile(k, 20)
    try:
        N.check(N.lib().gx_stage_set_exec(st.handle, N.GX_EXEC_SPAN))
        sp = st.profile(k, 20)
    except Exception as e:  # noqa: BLE001
        sp = f"n/a ({e})"
    print(f"[{a},{b}) k={k} budget={bud}: graph {g * 1000:.1f} us  span {sp if isinstance(sp, str) else f'{sp * 1000:.1f} us'}",
          flush=True)
