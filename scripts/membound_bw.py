"""Achieved HBM bandwidth of the bandwidth-bound kernels (pool, GAP, gather, scatter, LayerNorm,
channel copy, FC weight streaming) launched alone on the whole GPU with inputs far larger than L2,
timed with CUDA events on the launching stream (north star (2): "BN/pool/activation kernels are
bandwidth-bound ... evidenced by achieved HBM GB/s against the peak").  Algorithmic bytes = every
logical input and output byte once (gx_api.cu op_work).  Run under
`ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --iters 1` for the
DRAM-side counts.

  python scripts/membound_bw.py --out profiles/r01_membound_bw.csv
"""
from __future__ import annotations

import argparse
import csv
import ctypes as C
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--out", default=None)
    ap.add_argument("--no-torch", action="store_true", help="skip the PyTorch reference rows")
    args = ap.parse_args()

    import torch

    from paper_2312_10636_b200 import _native as N
    from paper_2312_10636_b200.device import WeightBlob, context, run_op, tensor_desc

    ctx = context(0)
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] if (ROOT / "MEASURED_PEAKS.json").exists() \
        else 6650.0
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    rows = []

    def timed(name, shape, nbytes, fn, reps=10):
        for _ in range(3):
            fn()
        ts = []
        for _ in range(args.iters):
            # the GPU sleeps while the host enqueues `reps` launches behind the start event, so the
            # event interval is device time only (a ctypes launch costs ~20-40 us of host time,
            # comparable to these kernels)
            torch.cuda._sleep(int(2e6))
            e0.record(s)
            for _ in range(reps):
                fn()
            e1.record(s)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) / reps)
        ms = sorted(ts)[len(ts) // 2]
        gbs = nbytes / (ms * 1e-3) / 1e9
        rows.append({"kernel": name, "shape": shape, "mbytes": round(nbytes / 1e6, 1), "us": round(ms * 1e3, 1),
                     "gbs": round(gbs, 1), "peak_gbs": peak, "frac": round(gbs / peak, 3)})
        print(f"{name:14s} {shape:34s} {nbytes / 1e6:8.1f} MB {ms * 1e3:8.1f} us {gbs:7.1f} GB/s  {gbs / peak:.3f}",
              flush=True)

    bf = torch.bfloat16
    wz = torch.zeros(1 << 20, dtype=torch.uint8, device="cuda")
    # ResNet stem max pool 3x3/2 (112x112x64 -> 56x56), k = 128
    k = 128
    x = torch.randn(k, 112, 112, 64, device="cuda").to(bf)
    y = torch.empty(k, 56, 56, 64, dtype=bf, device="cuda")
    op = N.make_op(N.GX_OP_MAXPOOL, 0, 1, R=3, S=3, sh=2, sw=2, ph=1, pw=1, flags=1)
    timed("maxpool", "3x3/2 112x112x64 k=128", x.numel() * 2 + y.numel() * 2,
          lambda: run_op(op, [x, y], [tensor_desc(112, 112, 64), tensor_desc(56, 56, 64)], wz, k))
    # Inception avg pool 3x3/1 p1 (35x35x288), k = 256
    k = 256
    x = torch.randn(k, 35, 35, 288, device="cuda").to(bf)
    y = torch.empty(k, 35, 35, 288, dtype=bf, device="cuda")
    op = N.make_op(N.GX_OP_AVGPOOL, 0, 1, R=3, S=3, sh=1, sw=1, ph=1, pw=1, flags=1)
    timed("avgpool", "3x3/1 35x35x288 k=256", x.numel() * 4,
          lambda: run_op(op, [x, y], [tensor_desc(35, 35, 288), tensor_desc(35, 35, 288)], wz, k))
    # GAP 7x7x2048, k = 1024
    k = 1024
    x = torch.randn(k, 7, 7, 2048, device="cuda").to(bf)
    y = torch.empty(k, 2048, dtype=bf, device="cuda")
    op = N.make_op(N.GX_OP_GAP, 0, 1)
    timed("gap", "7x7x2048 k=1024", x.numel() * 2 + y.numel() * 2,
          lambda: run_op(op, [x, y], [tensor_desc(7, 7, 2048), tensor_desc(1, 1, 2048)], wz, k))
    # LayerNorm over BERT rows (seq 128 x 768), k = 1024
    k = 1024
    x = torch.randn(k, 128, 768, device="cuda").to(bf)
    y = torch.empty_like(x)
    blob = WeightBlob()
    g_off = blob.add_f32(torch.ones(768))
    b_off = blob.add_f32(torch.zeros(768))
    wln = torch.from_numpy(blob.bytes()).cuda()
    op = N.make_op(N.GX_OP_LAYERNORM, 0, 1, Cin=768, Cout=768, w_off=g_off, b_off=b_off, eps=1e-12)
    timed("layernorm", "128x768 k=1024", x.numel() * 4,
          lambda: run_op(op, [x, y], [tensor_desc(128, 1, 768), tensor_desc(128, 1, 768)], wln, k))
    # channel copy into a concat slice (Inception), 35x35x(64 of 288), k = 1024
    k = 1024
    x = torch.randn(k, 35, 35, 64, device="cuda").to(bf)
    y = torch.empty(k, 35, 35, 288, dtype=bf, device="cuda")
    op = N.make_op(N.GX_OP_COPY, 0, 1, Cin=64, out_coff=96)
    timed("copy_channels", "35x35x64 -> slice of 288, k=1024", x.numel() * 4,
          lambda: run_op(op, [x, y], [tensor_desc(35, 35, 64), tensor_desc(35, 35, 288)], wz, k))
    # ragged gather of fp32 client activations (112x112x64) into one bf16 batch, k = 64
    k, pix, cc = 64, 112 * 112, 64
    srcs = [torch.randn(pix * cc, device="cuda") for _ in range(k)]
    dst = torch.empty(k, pix * cc, dtype=bf, device="cuda")
    sp = N.ptr_array([t.data_ptr() for t in srcs])
    dts = (C.c_int32 * k)(*([N.GX_F32] * k))
    timed("gather", "fp32 112x112x64 -> bf16, k=64", k * pix * cc * 6,
          lambda: N.check(N.lib().gx_gather(ctx.handle, k, sp, dts, pix, cc, cc, C.c_void_p(dst.data_ptr()), 0,
                                            C.c_void_p(s.cuda_stream)), "gx_gather"))
    # scatter of a bf16 batch into per-request slots, k = 64
    outs = [torch.empty(pix * cc, dtype=bf, device="cuda") for _ in range(k)]
    op_ = N.ptr_array([t.data_ptr() for t in outs])
    timed("scatter", "bf16 112x112x64 rows -> slots, k=64", k * pix * cc * 4,
          lambda: N.check(N.lib().gx_scatter(ctx.handle, k, C.c_void_p(dst.data_ptr()), N.GX_BF16, pix * cc, op_,
                                             N.GX_BF16, 0, C.c_void_p(s.cuda_stream)), "gx_scatter"))
    # FC weight streaming at batch 1 (VGG-16 fc6: 25088 -> 4096, 205 MB of weights), both paths
    K, O = 25088, 4096
    blob = WeightBlob()
    w_off = blob.add_bf16(torch.randn(O, K) * 0.01)
    b_off = blob.add_f32(torch.zeros(O))
    wfc = torch.from_numpy(blob.bytes()).cuda()
    x = torch.randn(1, 7, 7, 512, device="cuda").to(bf)
    y = torch.empty(1, O, dtype=bf, device="cuda")
    for path, flags in (("tcgen05", 0), ("simt", N.GX_OPF_FC_SIMT)):  # the op flag selects the path
        op = N.make_op(N.GX_OP_FC, 0, 1, Cin=K, Cout=O, w_off=w_off, b_off=b_off, flags=flags)
        timed(f"fc_{path}", "25088->4096 k=1 (VGG fc6)", K * O * 2 + O * 4 + K * 2 + O * 2,
              lambda op=op: run_op(op, [x, y], [tensor_desc(7, 7, 512), tensor_desc(1, 1, O)], wfc, 1))
    # the same traffic through PyTorch's own kernels (library ceilings on this box, not ours): a
    # plain copy, a strided slice copy, a channels-last max pool and a spatial sum
    if not args.no_torch:
        a = torch.randn(1024, 35, 35, 64, device="cuda").to(bf)
        b = torch.empty_like(a)
        timed("torch_copy", "contiguous 1024x35x35x64 bf16", a.numel() * 4, lambda: b.copy_(a))
        y = torch.empty(1024, 35, 35, 288, dtype=bf, device="cuda")
        timed("torch_slice", "35x35x64 -> slice of 288, k=1024", a.numel() * 4, lambda: y[..., 96:160].copy_(a))
        x = torch.randn(128, 64, 112, 112, device="cuda").to(bf).to(memory_format=torch.channels_last)
        timed("torch_maxpool", "3x3/2 112x112x64 k=128 (NHWC)", x.numel() * 2 + x.numel() // 2,
              lambda: torch.nn.functional.max_pool2d(x, 3, 2, 1))
        g = torch.randn(1024, 7, 7, 2048, device="cuda").to(bf)
        timed("torch_gap", "7x7x2048 k=1024 (sum dim 1,2)", g.numel() * 2 + 1024 * 2048 * 2,
              lambda: g.sum(dim=(1, 2)))
    if args.out:
        with open(args.out, "w", newline="") as f:
            w = csv.DictWriter(f, fieldnames=list(rows[0].keys()))
            w.writeheader()
            w.writerows(rows)


if __name__ == "__main__":
    main()
