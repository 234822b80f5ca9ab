"""Run one dispatched batch of a stage (gather -> span graph -> scatter) for an ncu capture.

  ncu --set full -k regex:conv_tc -c 60 -o gpurun_out/stage python scripts/ncu_stage.py resnet50 0 18 8 3
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2312_10636_b200.engine import DeviceModel, StageInstance  # noqa: E402
from paper_2312_10636_b200.models import build_chain  # noqa: E402

name, a, b, k, budget = sys.argv[1], *(int(x) for x in sys.argv[2:6])
chain = build_chain(name)
dm = DeviceModel(chain)
st = StageInstance(dm, a, b, k, budget)
H, W, C, _ = chain.boundary_shape(a)
xs = [torch.rand(chain.ingress_elems(a), device="cuda") for _ in range(k)]
out = st.run(xs, src_channels=chain.ingress_channels(a))
torch.cuda.synchronize()
print(f"ran span [{a},{b}) k={k} budget={budget}: {st.kernel_count(k)} kernels")
