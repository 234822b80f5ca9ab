"""Per-kernel roofline table: every op of a span launched alone (gx_stage_profile_ops) at batch k on
an SM budget, its algorithmic FLOPs / bytes (FLOPs = 2*M*N*K unpadded; bytes = every
logical input, weight, bias, residual and output byte once) against the measured peaks scaled by
budget/SMs (tensor) and min(HBM, per-SM L2 feed x budget) (memory).  Writes a CSV and prints a summary per operating point.

  python scripts/kernel_roofline.py --model resnet50 --points 0:18:16:148,0:18:8:3,2:18:1:2 \
      --out profiles/r01_kernel_roofline.csv
"""
from __future__ import annotations

import argparse
import csv
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

KIND = {1: "conv", 2: "maxpool", 3: "avgpool", 4: "gap", 5: "fc", 6: "linear", 7: "layernorm", 8: "attention",
        9: "embed", 10: "copy", 11: "flatten"}


# one SM's measured L2->SM feed (bulk copies, 2x64 KB in flight, scripts/native/sm_feed_probe.cu,
# profiles/r01_sm_feed_probe.log): the memory roofline of a kernel confined to a few SMs, whose
# working set (weights, activations) is L2-resident; HBM caps it for large budgets
SM_FEED_GBS = 166.3


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d["bf16_tflops"], d["hbm_gbs"], "measured"
    return 1590.0, 6650.0, "fallback"


def describe(chain, op_index):
    op = chain.ops[op_index]
    ti = chain.tensors[op.in_]
    to = chain.tensors[op.out]
    if op.kind == 1:
        return f"{op.R}x{op.S}/{op.sh} {ti[0]}x{ti[1]}x{op.Cin}->{to[0]}x{to[1]}x{op.Cout}" + \
            (" +res" if op.in2 >= 0 else "")
    if op.kind in (2, 3):
        return f"{op.R}x{op.S}/{op.sh} {ti[0]}x{ti[1]}x{ti[2]}->{to[0]}x{to[1]}"
    if op.kind == 5:
        return f"{op.Cin}->{op.Cout}"
    if op.kind == 6:
        return f"S={ti[0]} {op.Cin}->{op.Cout}"
    return f"{ti[0]}x{ti[1]}x{ti[2]}"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="resnet50")
    ap.add_argument("--points", default="0:18:16:148,0:18:8:3,2:18:1:2",
                    help="start:end:k:sm_budget,...")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()

    from paper_2312_10636_b200.device import context
    from paper_2312_10636_b200.engine import DeviceModel, StageInstance
    from paper_2312_10636_b200.models import build_chain

    tc_peak, hbm_peak, src = peaks()
    chain = build_chain(args.model)
    dm = DeviceModel(chain, 0)
    sms = context(0).sm_count
    rows = []
    for pt in args.points.split(","):
        a, b, k, budget = (int(x) for x in pt.split(":"))
        st = StageInstance(dm, a, b, k, budget)
        whole = st.profile(k, args.iters)
        ops = st.profile_ops(k, args.iters)
        first = chain.unit_first_op[a]
        scale = budget / sms
        tot_ms = sum(o["ms"] for o in ops)
        frac_w = 0.0
        for o in ops:
            t = o["ms"] * 1e-3
            tf = o["flops"] / t / 1e12 if t > 0 else 0.0
            gb = o["bytes"] / t / 1e9 if t > 0 else 0.0
            # persistent tensor-core kernels (conv / linear / FC) run on `budget` CTAs = SMs; attention
            # launches up to 4 CTAs per budget SM and the bandwidth kernels budget x 8 blocks of 256
            # threads, which the block scheduler spreads over up to 4x / 8x as many SMs (a budget is a
            # grid size, not an SM partition)
            spread = budget if o["kind"] in (1, 5, 6) else min(sms, (4 if o["kind"] == 8 else 8) * budget)
            t_tc = o["flops"] / (tc_peak * spread / sms * 1e12)
            mem_peak = min(hbm_peak, SM_FEED_GBS * spread)
            t_hbm = o["bytes"] / (mem_peak * 1e9)
            frac = max(t_tc, t_hbm) / t if t > 0 else 0.0
            frac_w += frac * o["ms"]
            rows.append({"model": args.model, "start": a, "end": b, "k": k, "sm_budget": budget,
                         "op": first + o["op"], "kind": KIND.get(o["kind"], str(o["kind"])),
                         "shape": describe(chain, first + o["op"]), "us": round(o["ms"] * 1000, 2),
                         "gflop": round(o["flops"] / 1e9, 4), "mbytes": round(o["bytes"] / 1e6, 4),
                         "tflops": round(tf, 2), "gbs": round(gb, 1), "bound": "tensor" if t_tc >= t_hbm else "memory",
                         "roofline_us": round(max(t_tc, t_hbm) * 1e6, 2), "frac": round(frac, 3)})
        print(f"# span [{a},{b}) k={k} budget={budget} SMs: graph {whole * 1000:.1f} us, sum of ops "
              f"{tot_ms * 1000:.1f} us over {len(ops)} ops, time-weighted roofline frac "
              f"{frac_w / max(tot_ms, 1e-12):.3f} (peaks {src}: {tc_peak} TF/s x {budget}/{sms}; memory min({hbm_peak}, {SM_FEED_GBS} x SMs touched: budget, or 8 x budget for the bandwidth kernels) GB/s)",
              flush=True)
        by_kind = {}
        for r in rows[-len(ops):]:
            d = by_kind.setdefault(r["kind"], [0.0, 0.0, 0])
            d[0] += r["us"]
            d[1] += r["roofline_us"]
            d[2] += 1
        for kname, (us, roof, n) in sorted(by_kind.items(), key=lambda x: -x[1][0]):
            print(f"#   {kname:9s} n={n:3d} {us:9.1f} us ({100 * us / (tot_ms * 1000):5.1f}%)  roofline {roof:8.1f} us "
                  f"-> frac {roof / us:.3f}", flush=True)
        del st
    if args.out:
        with open(args.out, "w", newline="") as f:
            w = csv.DictWriter(f, fieldnames=list(rows[0].keys()))
            w.writeheader()
            w.writerows(rows)
        print(f"# wrote {len(rows)} rows to {args.out}")


if __name__ == "__main__":
    main()
