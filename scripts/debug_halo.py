"""Halo conv debug: per-tap error vs torch (development aid)."""
import os
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402
import torch.nn.functional as F  # noqa: E402

from paper_2312_10636_b200 import _native as N  # noqa: E402
from paper_2312_10636_b200.device import WeightBlob, pack_conv_weight, run_op, tensor_desc  # noqa: E402

k, H, W, C, Co = 1, 56, 56, 64, 64
g = torch.Generator().manual_seed(0)
x = torch.randn(k, H, W, C, generator=g).to(torch.bfloat16)
for dbg in ("0", "32"):
    os.environ["GX_CONV_DBG"] = dbg
    for tap in (0, 1, 3, 4, 8):
        w = torch.zeros(Co, C, 3, 3)
        w[:, :, tap // 3, tap % 3] = torch.randn(Co, C, generator=g) / 8
        b = torch.zeros(Co)
        ref = F.conv2d(x.float().permute(0, 3, 1, 2), w.to(torch.bfloat16).float(), b, padding=1).permute(0, 2, 3, 1)
        blob = WeightBlob()
        w_off = blob.add_bf16(pack_conv_weight(w))
        b_off = blob.add_f32(b)
        wdev = torch.from_numpy(blob.bytes()).cuda()
        y = torch.full((k, H, W, Co), float("nan"), dtype=torch.bfloat16, device="cuda")
        op = N.make_op(N.GX_OP_CONV, 0, 1, R=3, S=3, sh=1, sw=1, ph=1, pw=1, Cin=C, Cout=Co, w_off=w_off, b_off=b_off)
        run_op(op, [x.cuda(), y], [tensor_desc(H, W, C), tensor_desc(H, W, Co)], wdev, k, 3)
        torch.cuda.synchronize()
        got = y.float().cpu()
        rel = ((got - ref).norm() / ref.norm()).item()
        # is got a shifted version of ref?
        best = None
        for dy in (-2, -1, 0, 1, 2):
            for dx in (-2, -1, 0, 1, 2):
                sh = torch.roll(ref, shifts=(dy, dx), dims=(1, 2))
                r2 = ((got[:, 3:-3, 3:-3] - sh[:, 3:-3, 3:-3]).norm() / sh[:, 3:-3, 3:-3].norm()).item()
                if best is None or r2 < best[0]:
                    best = (round(r2, 4), dy, dx)
        print(f"dbg={dbg} tap={tap} rel={rel:.4f} best_shift={best}", flush=True)
