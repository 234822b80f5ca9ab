"""Conv kernel microbenchmark (development aid): back-to-back launches timed with CUDA events."""
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2312_10636_b200 import _native as N
from paper_2312_10636_b200.device import WeightBlob, pack_conv_weight, run_op, tensor_desc

SHAPES = {  # name: (k, H, W, Cin, Cout, R, S, stride, pad)
    "l1_1x1_256_64": (16, 56, 56, 256, 64, 1, 1, 1, 0),
    "l1_3x3_64": (16, 56, 56, 64, 64, 3, 3, 1, 1),
    "l3_1x1_1024_256": (16, 14, 14, 1024, 256, 1, 1, 1, 0),
    "l3_3x3_256": (16, 14, 14, 256, 256, 3, 3, 1, 1),
    "l4_3x3_512": (16, 7, 7, 512, 512, 3, 3, 1, 1),
    "big_gemm": (64, 32, 32, 1024, 256, 1, 1, 1, 0),
    "stem": (16, 224, 224, 8, 64, 7, 7, 2, 3),
}


def run(name, k, H, W, Cin, Cout, R, S, stride, pad, budget=0, iters=50):
    dev = "cuda"
    res = name.endswith("_res")
    Ho = (H + 2 * pad - R) // stride + 1
    Wo = (W + 2 * pad - S) // stride + 1
    blob = WeightBlob()
    w_off = blob.add_bf16(pack_conv_weight(torch.randn(Cout, Cin, R, S) * 0.05))
    b_off = blob.add_f32(torch.zeros(Cout))
    wdev = torch.from_numpy(blob.bytes()).to(dev)
    x = torch.randn(k, H, W, Cin, device=dev).to(torch.bfloat16)
    y = torch.empty(k, Ho, Wo, Cout, device=dev, dtype=torch.bfloat16)
    op = N.make_op(N.GX_OP_CONV, 0, 1, in2=2 if res else -1, act=N.GX_ACT_RELU, R=R, S=S, sh=stride, sw=stride,
                   ph=pad, pw=pad, Cin=Cin, Cout=Cout, w_off=w_off, b_off=b_off)
    descs = [tensor_desc(H, W, Cin), tensor_desc(Ho, Wo, Cout), tensor_desc(Ho, Wo, Cout)]
    tens = [x, y, torch.randn(k, Ho, Wo, Cout, device=dev).to(torch.bfloat16)]
    for _ in range(3):
        run_op(op, tens, descs, wdev, k, budget)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(iters):
        run_op(op, tens, descs, wdev, k, budget)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1000 / iters
    flops = 2.0 * k * Ho * Wo * Cout * Cin * R * S
    hbm = (x.numel() + y.numel()) * 2 + Cout * Cin * R * S * 2
    print(f"{name:18s} BN={os.environ.get('GX_BN', 'auto'):4s} st={os.environ.get('GX_STAGES', 'auto'):4s} "
          f"{us:8.2f} us  {flops / us / 1e6:7.1f} TFLOP/s  {hbm / us / 1e3:7.1f} GB/s(min HBM)", flush=True)




def run_graph(name, k, H, W, Cin, Cout, R, S, stride, pad, budget=0, iters=50):
    """Same, but the launches are replayed from a CUDA graph (no host overhead per launch)."""
    dev = "cuda"
    Ho = (H + 2 * pad - R) // stride + 1
    Wo = (W + 2 * pad - S) // stride + 1
    blob = WeightBlob()
    w_off = blob.add_bf16(pack_conv_weight(torch.randn(Cout, Cin, R, S) * 0.05))
    b_off = blob.add_f32(torch.zeros(Cout))
    wdev = torch.from_numpy(blob.bytes()).to(dev)
    x = torch.randn(k, H, W, Cin, device=dev).to(torch.bfloat16)
    y = torch.empty(k, Ho, Wo, Cout, device=dev, dtype=torch.bfloat16)
    op = N.make_op(N.GX_OP_CONV, 0, 1, act=N.GX_ACT_RELU, R=R, S=S, sh=stride, sw=stride, ph=pad, pw=pad, Cin=Cin,
                   Cout=Cout, w_off=w_off, b_off=b_off)
    descs = [tensor_desc(H, W, Cin), tensor_desc(Ho, Wo, Cout)]
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        run_op(op, [x, y], descs, wdev, k, budget)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(iters):
            run_op(op, [x, y], descs, wdev, k, budget)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1000 / iters
    flops = 2.0 * k * Ho * Wo * Cout * Cin * R * S
    print(f"{name:18s} GRAPH {us:8.2f} us  {flops / us / 1e6:7.1f} TFLOP/s", flush=True)


SHAPES["tiny"] = (1, 8, 8, 64, 64, 1, 1, 1, 0)
SHAPES["l3_1x1_256_1024_k16_res"] = (16, 14, 14, 256, 1024, 1, 1, 1, 0)
SHAPES["l3_1x1_256_1024_k16"] = (16, 14, 14, 256, 1024, 1, 1, 1, 0)
SHAPES["l2_1x1_128_512_k16_res"] = (16, 28, 28, 128, 512, 1, 1, 1, 0)
SHAPES["l1_1x1_64_256_k8"] = (8, 56, 56, 64, 256, 1, 1, 1, 0)
SHAPES["l1_3x3_64_k8"] = (8, 56, 56, 64, 64, 3, 3, 1, 1)
SHAPES["l3_3x3_256_k8"] = (8, 14, 14, 256, 256, 3, 3, 1, 1)
SHAPES["l3_1x1_1024_256_k8"] = (8, 14, 14, 1024, 256, 1, 1, 1, 0)
SHAPES["l4_3x3_512_k8"] = (8, 7, 7, 512, 512, 3, 3, 1, 1)

SHAPES["l1_3x3_k1"] = (1, 56, 56, 64, 64, 3, 3, 1, 1)
SHAPES["l1_1x1_64_256_k16_res"] = (16, 56, 56, 64, 256, 1, 1, 1, 0)
SHAPES["l1_1x1_64_256_k16"] = (16, 56, 56, 64, 256, 1, 1, 1, 0)
SHAPES["l1_1x1_256_64_k16"] = (16, 56, 56, 256, 64, 1, 1, 1, 0)
SHAPES["l1_1x1_64_64_k16"] = (16, 56, 56, 64, 64, 1, 1, 1, 0)
SHAPES["l1_3x3_64_k16"] = (16, 56, 56, 64, 64, 3, 3, 1, 1)
SHAPES["l2_3x3_128_k16"] = (16, 28, 28, 128, 128, 3, 3, 1, 1)
SHAPES["l3_3x3_k1"] = (1, 14, 14, 256, 256, 3, 3, 1, 1)
SHAPES["l1_1x1_576_k1"] = (1, 56, 56, 576, 64, 1, 1, 1, 0)
# the layer4 tail at batch 1 (stages [15,18) / [17,18) of the serving plans)
SHAPES["l4_1x1_2048_512_k1"] = (1, 7, 7, 2048, 512, 1, 1, 1, 0)
SHAPES["l4_3x3_512_k1"] = (1, 7, 7, 512, 512, 3, 3, 1, 1)
SHAPES["l4_1x1_512_2048_k1_res"] = (1, 7, 7, 512, 2048, 1, 1, 1, 0)
SHAPES["l4_1x1_512_2048_k4_res"] = (4, 7, 7, 512, 2048, 1, 1, 1, 0)


if __name__ == "__main__":
    names = sys.argv[1].split(",") if len(sys.argv) > 1 else list(SHAPES)
    budget = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    graph = os.environ.get("GRAPH", "0") == "1"
    for n in names:
        (run_graph if graph else run)(n, *SHAPES[n], budget=budget)
