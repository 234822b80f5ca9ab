"""One conv op as a one-unit chain: span kernel vs per-op path (development aid)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
import torch.nn as nn  # noqa: E402

from paper_2312_10636_b200.engine import DeviceModel, StageInstance  # noqa: E402
from paper_2312_10636_b200.models import ChainBuilder  # noqa: E402

CASES = {"l1_3x3": (56, 64, 64, 3, 1, 1), "l3_3x3": (14, 256, 256, 3, 1, 1), "l4_3x3": (7, 512, 512, 3, 1, 1),
         "l3_1x1": (14, 1024, 256, 1, 1, 0)}
budget = int(sys.argv[1]) if len(sys.argv) > 1 else 4
for name, (hw, cin, cout, r, s, p) in CASES.items():
    b = ChainBuilder("single")
    x = b.tensor(hw, hw, cin)
    b.begin_unit(x)
    conv = nn.Conv2d(cin, cout, r, s, p, bias=False)
    y = b.conv(x, conv, None, relu=True)
    chain = b.finish(y)
    chain.input_channels = cin
    dm = DeviceModel(chain)
    st = StageInstance(dm, 0, 1, 16, budget)
    res = []
    for k in (1, 4, 16):
        res.append(f"k={k} {st.profile(k, 30) * 1000:8.1f} us")
    print(f"{os.environ.get('GX_EXEC', 'span'):5s} {name:8s} budget={budget} " + "  ".join(res), flush=True)
