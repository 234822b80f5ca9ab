"""Host-side cost of one gx_stage_run dispatch (development aid)."""
import ctypes as C
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2312_10636_b200 import _native as N  # noqa: E402
from paper_2312_10636_b200.engine import DeviceModel, StageInstance  # noqa: E402
from paper_2312_10636_b200.models import build_chain  # noqa: E402

chain = build_chain("resnet50")
dm = DeviceModel(chain)
L = N.lib()
for (a, b) in ((0, 18), (9, 18), (15, 18), (17, 18)):
    st = StageInstance(dm, a, b, 16, 2)
    x = torch.randn(chain.ingress_elems(a), device="cuda")
    out = torch.empty(chain.boundary_elems(b), device="cuda")
    src = N.ptr_array([x.data_ptr()])
    dt = N.i32_array([N.GX_F32])
    dst = N.ptr_array([out.data_ptr()])
    ch = chain.ingress_channels(a)
    for _ in range(3):
        L.gx_stage_run(st.handle, 1, src, dt, ch, dst, N.GX_F32 if b == 18 else N.GX_BF16)
    torch.cuda.synchronize()
    n = 200
    t0 = time.perf_counter()
    for _ in range(n):
        L.gx_stage_run(st.handle, 1, src, dt, ch, dst, N.GX_F32 if b == 18 else N.GX_BF16)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"span [{a},{b}) kernels={st.kernel_count(1)} host {1e6 * (t1 - t0) / n:.1f} us/dispatch, "
          f"device {1e6 * (t2 - t0) / n:.1f} us/dispatch (2 SMs)", flush=True)
