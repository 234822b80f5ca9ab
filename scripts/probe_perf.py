"""Quick span-latency probe on the GPU (development aid)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2312_10636_b200.engine import DeviceModel, StageInstance
from paper_2312_10636_b200.models import build_chain

name = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
chain = build_chain(name)
dm = DeviceModel(chain)
N = chain.n_units
budgets = [int(a) for a in sys.argv[2].split(",")] if len(sys.argv) > 2 else (148, 74, 30)
ks = [int(a) for a in sys.argv[3].split(",")] if len(sys.argv) > 3 else (1, 4, 8, 16, 32)
for budget in budgets:
    st = StageInstance(dm, 0, N, max_batch=32, sm_budget=budget)
    for k in ks:
        ms = st.profile(k, 20)
        gflop = sum(chain.unit_flops) * k / 1e9
        print(f"{name} sms={budget:3d} k={k:2d} {ms*1000:8.1f} us  {k/ms*1000:9.0f} img/s  {gflop/ms:7.1f} TFLOP/s"
              f"  kernels={st.kernel_count(k)}", flush=True)
