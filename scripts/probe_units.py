"""Per-unit error of libgx vs the fp32 oracle (development aid)."""
import sys
import torch
sys.path.insert(0, ".")
from oracle.units import nchw_to_nhwc, run_span, units_for
from paper_2312_10636_b200.engine import DeviceModel, StageInstance
from paper_2312_10636_b200.models import build_chain, torch_model

name = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
res = 299 if name == "inception_v3" else 224
m = torch_model(name)
chain = build_chain(name, module=m)
dm = DeviceModel(chain)
units = units_for(name, m)
x = torch.randn(2, 3, res, res, generator=torch.Generator().manual_seed(1))
acts = [x]
for u in range(chain.n_units):
    acts.append(run_span(units, u, u + 1, acts[-1]))
for u in range(chain.n_units):
    st = StageInstance(dm, u, u + 1, max_batch=2, sm_budget=148)
    inp = [nchw_to_nhwc(acts[u][i:i+1])[0].contiguous().cuda() for i in range(2)]
    got = torch.stack(st.run(inp, out_dtype=torch.float32, src_channels=3 if u == 0 else 0)).cpu()
    ref = nchw_to_nhwc(acts[u + 1]).reshape(2, -1)
    got = got.view(2, -1)
    rel = ((got - ref).norm() / ref.norm()).item()
    print(f"unit {u:2d} rel={rel:.4e} ref_norm={ref.norm():.3e} out_shape={chain.boundary_shape(u+1)}")
