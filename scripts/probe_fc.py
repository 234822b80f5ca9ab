"""FC (ResNet head 2048 -> 1000, fp32 logits) at small batch on a few SMs, CUDA-graph timed."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2312_10636_b200 import _native as N  # noqa: E402
from paper_2312_10636_b200.device import WeightBlob, run_op, tensor_desc  # noqa: E402

K, O = 2048, 1000
blob = WeightBlob()
w_off = blob.add_bf16(torch.randn(O, K) * 0.02)
b_off = blob.add_f32(torch.zeros(O))
wdev = torch.from_numpy(blob.bytes()).cuda()
for k, bud in [(1, 2), (1, 6), (4, 6), (16, 6)]:
    x = torch.randn(k, K, device="cuda").to(torch.bfloat16)
    y = torch.empty(k, O, device="cuda")
    op = N.make_op(N.GX_OP_FC, 0, 1, Cin=K, Cout=O, w_off=w_off, b_off=b_off)
    descs = [tensor_desc(1, 1, K), tensor_desc(1, 1, O, N.GX_F32)]
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        run_op(op, [x, y], descs, wdev, k, bud, stream=s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(20):
            run_op(op, [x, y], descs, wdev, k, bud, stream=s)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"fc 2048->1000 k={k} budget={bud}: {e0.elapsed_time(e1) * 1000 / 20:.1f} us", flush=True)
