"""Benchmark: SLO-met requests/sec for re-aligned ResNet-50 fragment groups on B200.

Workload (BASELINE.json configs[1]): a fleet of ResNet-50 clients at 30 rps cut at 8 partition
points, planned by the unmodified reference planner (merge -> group -> re-align -> placement)
against the measured B200 profile table; tests/golden/workload/resnet50_c<N>.json.  The executor
serves that plan in real time: requests arrive on the wall clock (gen + mobile prefix + link
transfer), are batched per stage exactly as the reference simulator batches them, and every
dispatched batch runs on the GPU (ragged gather -> span kernels -> scatter) on an instance bounded
to the stage's SM share.

A step is one serving window of `--window` seconds of arrivals.  `value` counts requests generated
in the K timed windows that complete within their deadline, divided by the timed window time;
valid only when p99 latency <= SLO.  Entry activations are resident in HBM for `value`; `e2e`
repeats the measurement with each request's activation copied host->device at arrival and its
logits written back to pinned host memory.

Multi-GPU (torchrun): one process per GPU, each serving its own independent fleet of the same
size (groups share no tensors; no collective on the data path): scaling "weak".

--impl reference: the reference's serving path on the host CPU — the oracle restatement of its
event loop (pinned bit-exact to the reference) driven by fp32 CPU execution times of the same
spans measured on this host (bounded sample).
"""
from __future__ import annotations

import argparse
import glob
import json
import math
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "SLO-met requests/sec (p99<=SLO) for re-aligned ResNet-50 groups"
UNIT = "req/s"


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d.get("bf16_tflops_sustained", 1401.0), d.get("bf16_tflops", 1659.7), d.get("hbm_gbs", 6538.6), "measured"
    return 1400.0, 1590.0, 6650.0, "fallback"


def _workloads(name: str, all_plans: bool = False):
    """Planned fleets <name>_c<N>.json in ascending (clients, latency_scale) order; with all_plans
    also the fleets planned against the load-calibrated table (<name>_s<F>_c<N>.json)."""
    pats = [f"{name}_c[0-9]*.json"] + ([f"{name}_s*_c[0-9]*.json"] if all_plans else [])
    files = [f for pat in pats for f in glob.glob(str(ROOT / "tests" / "golden" / "workload" / pat))]
    docs = [json.loads(Path(f).read_text()) for f in files]
    return sorted(docs, key=lambda d: (d["clients_n"], d.get("latency_scale", 1.0), -d.get("merge_threshold", 0.2)))


def _workload(name: str, clients: int | None):
    files = sorted(glob.glob(str(ROOT / "tests" / "golden" / "workload" / f"{name}_c[0-9]*.json")),
                   key=lambda f: int(f.rsplit("_c", 1)[1].split(".")[0]))
    if not files:
        raise SystemExit(f"no workload fixtures for {name}; run scripts/make_workload.py")
    if clients is not None:
        files = [f for f in files if f.endswith(f"_c{clients}.json")]
        if not files:
            raise SystemExit(f"no workload fixture with {clients} clients")
    return json.loads(Path(files[-1]).read_text())


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region (B200_PROFILING.md)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                if out.returncode == 0 and out.stdout.strip():
                    self.samples.append([x.strip() for x in out.stdout.strip().split(",")])
            except Exception:  # noqa: BLE001 - clocks are best-effort telemetry
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = sorted(float(s[1]) for s in self.samples)
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for s in self.samples:
            for n, v in zip(names, s[5:9]):
                if v.strip().lower() in ("active", "1"):
                    reasons.add(n)
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": float(self.samples[0][2]), "reasons": sorted(reasons),
                "samples": len(self.samples)}


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2312_10636_b200 import _native as N
    from paper_2312_10636_b200.device import context
    from paper_2312_10636_b200.engine import DeviceModel, StageInstance
    from paper_2312_10636_b200.models import build_chain
    from paper_2312_10636_b200.plan import deploy
    from paper_2312_10636_b200.serving import ClientView, serve

    world, rank, local = _dist()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = context(local)
    chain = build_chain(args.model)
    dm = DeviceModel(chain, local)

    class Fleet:
        """One planned fleet made executable on this GPU: stage instances + ingress templates."""

        def __init__(self, wl):
            self.wl = wl
            self.dep = deploy(wl["plan"], wl["fragments"])
            self.clients = [ClientView.from_doc(c) for c in wl["clients"]]
            budgets = ctx.sm_budgets([(s.share, s.instances) for s in self.dep.stages],
                                     work_conserving=not args.strict_shares)
            it = iter(budgets)
            self.instances = [[StageInstance(dm, s.start, s.end, s.batch, next(it)) for _ in range(s.instances)]
                              for s in self.dep.stages]
            g = torch.Generator(device="cuda").manual_seed(1234)
            self.dev_in, self.host_in = {}, {}
            slot = 0
            for p in sorted({r.point for r in self.dep.routes.values()}):
                ch = chain.ingress_channels(p)
                x = torch.randn(chain.ingress_elems(p), device="cuda", generator=g)
                if p > 0:
                    x = x.clamp_min(0)  # post-ReLU client activations
                self.dev_in[p] = (x, x.data_ptr(), x.numel() * 4, ch)
                h = x.cpu().pin_memory()
                self.host_in[p] = (h, h.data_ptr(), h.numel() * 4, ch)
                slot = max(slot, x.numel() * 4, chain.boundary_elems(p) * 2)
            for s in self.dep.stages:
                slot = max(slot, chain.boundary_elems(s.end) * 2)
            self.slot_bytes = (slot + 255) // 256 * 256
            for s, insts in zip(self.dep.stages, self.instances):  # capture every (instance, k) graph
                for inst in insts:
                    for k in range(1, s.batch + 1):
                        inst.kernel_count(k)
            torch.cuda.synchronize()

        def serve(self, horizon, host=False):
            ingress = {p: (v[1], v[2], v[3]) for p, v in (self.host_in if host else self.dev_in).items()}
            return serve(self.dep, self.clients, horizon, ctx=ctx, instances=self.instances, ingress=ingress,
                         ingress_from_host=(args.e2e_ingress if host else False), egress_to_host=host,
                         slot_bytes=self.slot_bytes,
                         max_inflight=args.max_inflight)

    def p99_of(rep, t_lo_ms=0.0):
        lats = sorted(d - g for _c, g, d, _dl, s in rep.requests if s == "completed" and g >= t_lo_ms)
        return lats[min(len(lats) - 1, int(math.ceil(0.99 * len(lats))) - 1)] if lats else math.inf

    def all_ok(ok: bool) -> bool:
        if world > 1:
            flag = torch.tensor([1 if ok else 0], device="cuda")
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
            ok = bool(flag.item())
        return ok

    # the achievable-throughput search runs over every planned fleet of the model: plans made
    # against the measured table and against the load-calibrated table (make_workload.py --scale),
    # with the reference's default merge threshold and a lower one (--merge 0.05: fewer, larger
    # merged fragments -> fewer stage instances competing for the 32 hardware queues)
    workloads = _workloads(args.plans or args.model, all_plans=args.plans is None)
    key = lambda w: (w["clients_n"], w.get("latency_scale", 1.0), -w.get("merge_threshold", 0.2))  # noqa: E731
    if args.clients is not None:
        fleet = Fleet(_workload(args.plans or args.model, args.clients))
    else:
        # achievable-throughput search: the largest planned fleet whose served
        # p99 stays within the SLO with < 1% drops, probed for 3 s each (p99 over arrivals after
        # the first second) from the top down; the timed run below re-checks and steps down
        fleet = None
        for wl in reversed(workloads):
            cand = Fleet(wl)
            rep = cand.serve(3.0)
            ok = p99_of(rep, 1000.0) <= wl["slo_ms"] and rep.dropped <= 0.01 * max(1, rep.generated)
            if rank == 0:
                print(f"# probe clients={wl['clients_n']} scale={wl.get('latency_scale', 1.0)} "
                      f"merge={wl.get('merge_threshold', 0.2)}: "
                      f"p99={p99_of(rep, 1000.0):.1f} ms "
                      f"met/s={rep.slo_met / 3.0:.0f} -> {'ok' if ok else 'over'}", file=sys.stderr, flush=True)
            if all_ok(ok):
                fleet = cand
                break
            del cand
        if fleet is None:
            fleet = Fleet(workloads[0])

    window = args.window
    W, K = args.warmup, args.steps
    horizon = (W + K) * window

    def one_run(fleet, host: bool):
        dep = fleet.dep
        ingress = {p: (v[1], v[2], v[3]) for p, v in (fleet.host_in if host else fleet.dev_in).items()}
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        rep = fleet.serve(horizon, host=host)
        e1.record()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t_lo, t_hi = W * window * 1000.0, horizon * 1000.0
        timed = [r for r in rep.requests if t_lo <= r[1] < t_hi]
        met = sum(1 for _c, _g, d, dl, s in timed if s == "completed" and d <= dl + 1e-9)
        lats = sorted(d - gg for _c, gg, d, _dl, s in timed if s == "completed")
        p99 = lats[min(len(lats) - 1, int(math.ceil(0.99 * len(lats))) - 1)] if lats else math.inf
        dropped = sum(1 for r in timed if r[4] == "dropped")
        return {"met": met, "generated": len(timed), "dropped": dropped, "p99": p99, "wall_ms": rep.wall_ms,
                "device_ms": e0.elapsed_time(e1), "kernels": rep.kernels, "batches": rep.batches,
                "h2d": sum(ingress[dep.routes[r[0]].point][1] for r in timed if r[0] in dep.routes) if host else 0,
                "d2h": sum(1 for r in timed if r[4] == "completed") * chain.boundary_elems(chain.n_units) * 4
                if host else 0}

    with ClockSampler(local) as clk:
        res = one_run(fleet, host=False)
        # the timed run is the verdict: if its p99 misses the SLO (or >1% drops), step down to the
        # next smaller planned fleet and measure again
        smaller = [w for w in reversed(workloads) if key(w) < key(fleet.wl)]
        while args.clients is None and smaller and not all_ok(
                res["p99"] <= fleet.wl["slo_ms"] and res["dropped"] <= 0.01 * max(1, res["generated"])):
            if rank == 0:
                print(f"# timed clients={fleet.wl['clients_n']}: p99={res['p99']:.1f} ms -> over, stepping down",
                      file=sys.stderr, flush=True)
            del fleet
            fleet = Fleet(smaller.pop(0))
            res = one_run(fleet, host=False)
    wl, dep, clients, instances = fleet.wl, fleet.dep, fleet.clients, fleet.instances
    slo = wl["slo_ms"]
    # e2e: the same achievable-throughput rule through the host path (each request's ingress
    # DMA-copied from pinned host memory at arrival, or read in place by the gather with
    # --e2e-ingress zero_copy; logits written to mapped host memory), from this fleet down
    e2e_fleet = fleet
    res_e2e = one_run(fleet, host=True)
    if args.clients is None:
        # host ingress makes the tail noisier than the resident run: a near miss (p99 within 2x the
        # SLO) is retried once before stepping down
        retried = False
        # fleets whose host->device demand exceeds ~85% of the measured PCIe Gen5 x16 rate (46 GB/s
        # for 1 MB copies, scripts/probe_h2d_streams.py) queue on the link without bound: skip them
        def h2d_gbs(w):
            by_id = {c["client_id"]: c for c in w["clients"]}
            return sum(by_id[cid]["rate_rps"] * by_id[cid]["payload_bytes"][f["start_layer"]]
                       for f in w["fragments"] for cid in f["clients"]) / 1e9

        cands = [w for w in reversed(workloads) if key(w) < key(wl) and h2d_gbs(w) <= 0.85 * 46.0]
        while True:
            ok = all_ok(res_e2e["p99"] <= slo and res_e2e["dropped"] <= 0.01 * max(1, res_e2e["generated"]))
            if rank == 0:
                print(f"# e2e clients={e2e_fleet.wl['clients_n']} scale={e2e_fleet.wl.get('latency_scale', 1.0)}: "
                      f"p99={res_e2e['p99']:.1f} ms -> "
                      f"{'ok' if ok else 'over'}", file=sys.stderr, flush=True)
            if ok:
                break
            if not retried and res_e2e["p99"] <= 2.0 * slo:
                retried = True
                res_e2e = one_run(e2e_fleet, host=True)
                continue
            if not cands:
                break
            if e2e_fleet is not fleet:
                del e2e_fleet
            e2e_fleet = Fleet(cands.pop(0))
            retried = False
            res_e2e = one_run(e2e_fleet, host=True)

    # roofline of the dominant kernel, the implicit-GEMM conv (conv_tc_kernel, plus conv_halo_kernel
    # for wide 3x3 layers: >=90% of GPU time in every launch list under profiles/): the busiest stage's span, each conv launched alone on the stage's stream
    # and timed with CUDA events (gx_stage_profile_ops), algorithmic FLOPs = 2*M*N*K unpadded per
    # launch, peak = measured burst bf16 x (stage SM budget / SMs) since the kernel is timed alone.
    def stage_flops(i):
        s = dep.stages[i]
        return s.instances * s.batch * sum(chain.unit_flops[s.start:s.end])

    busiest = max(range(len(dep.stages)), key=stage_flops)
    st = dep.stages[busiest]
    inst = instances[busiest][0]
    span_ms = inst.profile(st.batch, 20)
    ops = inst.profile_ops(st.batch, 10)
    convs = [o for o in ops if o["kind"] in (N.GX_OP_CONV, N.GX_OP_LINEAR)]
    conv_ms = sum(o["ms"] for o in convs)
    conv_flops = sum(o["flops"] for o in convs)
    conv_bytes = sum(o["bytes"] for o in convs)
    sustained, burst, hbm, src = _peaks()
    achieved = conv_flops / (conv_ms * 1e-3) / 1e12
    peak_scaled = burst * inst.sm_budget / ctx.sm_count
    span_flops = st.batch * sum(chain.unit_flops[st.start:st.end])
    traffic = None
    ncu_path = ROOT / "profiles" / "ncu_conv_summary.json"
    key = f"{args.model}:{st.start}:{st.end}:{st.batch}:{inst.sm_budget}"
    if ncu_path.exists():
        ent = json.loads(ncu_path.read_text()).get(key)
        if ent:
            traffic = {"dram_bytes_per_launch": ent["dram_bytes_per_launch"],
                       "l2_to_smem_bytes_per_launch": ent.get("tma_bytes_per_launch"),
                       "algorithmic_bytes_per_launch": round(conv_bytes / max(1, len(convs))),
                       "source": f"profiles/ncu_conv_summary.json[{key}] ({ent['launches']} launches, ncu --set full)"}
    stats = torch.tensor([res["met"], res["generated"], res["dropped"], res_e2e["met"], res["kernels"],
                          res["h2d"], res_e2e["h2d"], res_e2e["d2h"]], dtype=torch.float64, device="cuda")
    times = torch.tensor([res["device_ms"], res_e2e["device_ms"], res["p99"], res_e2e["p99"]], dtype=torch.float64,
                         device="cuda")
    if world > 1:
        dist.all_reduce(stats)
        dist.all_reduce(times, op=dist.ReduceOp.MAX)
    timed_s = K * window
    value = stats[0].item() / timed_s
    e2e_value = stats[3].item() / timed_s
    p99, p99_e2e = times[2].item(), times[3].item()
    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline:
            # the CPU path's own achievable rate: the smallest planned fleet (no fleet meets the SLO
            # on the host), plus the same CPU path on this run's plan for reference
            wl0 = _workloads(args.plans or args.model)[0]
            cpu = cpu_baseline(args, wl0, deploy(wl0["plan"], wl0["fragments"]), chain)
            cpu["sample"] += f" ({wl0['clients_n']}-client fleet)"
            cpu["value_on_bench_plan"] = cpu_baseline(args, wl, dep, chain, budget_s=10.0)["value"]
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": round(window * 1000.0, 3), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded random-init weights, random activations)",
            "config": {"workload": f"{args.model} re-aligned fragment groups, {wl['clients_n']} clients x "
                                   f"{wl['rate_rps']:.0f} rps per GPU, 8 cut points, plan from the reference planner "
                                   f"on the measured B200 profile table, SM-share partitioning",
                       "model": args.model, "latency_scale": wl.get("latency_scale", 1.0),
                       "merge_threshold": wl.get("merge_threshold", 0.2),
                       "clients_per_gpu": wl["clients_n"], "offered_rps_per_gpu":
                           wl["clients_n"] * wl["rate_rps"], "slo_ms": round(slo, 3), "window_s": window,
                       "stages": len(dep.stages), "instances": sum(s.instances for s in dep.stages),
                       "plan_resource": wl["plan"]["total_resource"], "parallelism": f"replica-per-gpu x{world}",
                       "l2": "inputs resident; working set per stage < L2, serving windows not flushed"},
            "p99_ms": round(p99, 3), "p99_ok": p99 <= slo, "generated": int(stats[1].item()),
            "dropped": int(stats[2].item()),
            "e2e": {"value": round(e2e_value, 1), "unit": UNIT, "p99_ms": round(p99_e2e, 3),
                    "p99_ok": p99_e2e <= slo, "clients_per_gpu": e2e_fleet.wl["clients_n"],
                    "latency_scale": e2e_fleet.wl.get("latency_scale", 1.0),
                    "merge_threshold": e2e_fleet.wl.get("merge_threshold", 0.2),
                    "path": ("serve() with host ingress: gather kernels read fp32 entry activations from pinned "
                             "host memory over PCIe (zero-copy), logits scattered to mapped host memory")
                    if args.e2e_ingress == "zero_copy" else
                    ("serve() with host ingress: each request's fp32 entry activation DMA-copied from pinned host "
                     "memory into a device slot at arrival (copy engine, per-request event the batch waits on), "
                     "logits scattered to mapped host memory"),
                    "h2d_bytes_per_step": int(stats[6].item() / K), "d2h_bytes_per_step": int(stats[7].item() / K)},
            "gpu_launches": int(stats[4].item()),
            "roofline": {"bound": "tensor",
                         "kernel": f"implicit-GEMM conv (conv_tc_kernel / conv_halo_kernel) x{len(convs)} launches of "
                                   f"span [{st.start},{st.end}) k={st.batch} "
                                   f"on {inst.sm_budget} SMs (busiest stage, planned share {st.share}%)",
                         "achieved": round(achieved, 2), "peak": round(peak_scaled, 2), "unit": "TFLOP/s",
                         "frac": round(achieved / peak_scaled, 4), "traffic": traffic,
                         "avg_launch_us": round(conv_ms * 1000 / max(1, len(convs)), 2),
                         "flops_per_launch": round(conv_flops / max(1, len(convs))),
                         "peak_source": f"{src} bf16_tflops burst ({burst}) x {inst.sm_budget}/{ctx.sm_count} SMs",
                         "span": {"graph_ms": round(span_ms, 4), "kernels": inst.kernel_count(st.batch),
                                  "tflops": round(span_flops / (span_ms * 1e-3) / 1e12, 2),
                                  "frac_of_sustained": round(span_flops / (span_ms * 1e-3) / 1e12 /
                                                             (sustained * inst.sm_budget / ctx.sm_count), 4)}},
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _cpu_stage_latency(chain_name, spans_k, budget_s):
    """fp32 CPU forward time per (span, k) on this host (the reference's compute path restated)."""
    import torch

    from oracle.units import run_span, units_for
    from paper_2312_10636_b200.models import build_chain, torch_model

    torch.set_num_threads(os.cpu_count() or 1)
    m = torch_model(chain_name)
    units = units_for(chain_name, m)
    chain = build_chain(chain_name, module=m)
    out = {}
    t_start = time.time()
    for (a, b), ks in spans_k.items():
        for k in ks:
            if time.time() - t_start > budget_s:
                break
            if a == 0:
                x = torch.randn(k, 3, 224, 224)
            else:
                H, W, Cc, _ = chain.boundary_shape(a)
                x = torch.randn(k, Cc, H, W).clamp_min(0)
            run_span(units, a, b, x)  # warm
            best = math.inf
            for _ in range(2):  # best of two timed passes
                t0 = time.perf_counter()
                run_span(units, a, b, x)
                best = min(best, (time.perf_counter() - t0) * 1000.0)
            out[(a, b, k)] = best
    return out


def cpu_baseline(args, wl, dep, chain, budget_s: float = 20.0):
    """The CPU path on this host: oracle event loop + measured fp32 CPU span latencies."""
    from oracle.serving import simulate_fixed
    from paper_2312_10636_b200.serving import ClientView

    spans_k = {}
    for s in dep.stages:
        spans_k.setdefault((s.start, s.end), set()).update({1, s.batch})
    spans_k = {k: sorted(v) for k, v in spans_k.items()}
    t0 = time.time()
    lat = _cpu_stage_latency(args.model, spans_k, budget_s)

    def latency(spec, k):
        lo = lat.get((spec.start, spec.end, 1))
        hi = lat.get((spec.start, spec.end, spec.batch))
        if lo is None:
            return 1e9
        if hi is None or spec.batch == 1:
            return lo * k
        return lo + (hi - lo) * (k - 1) / (spec.batch - 1)

    clients = [ClientView.from_doc(c) for c in wl["clients"]]
    horizon = args.steps * args.window
    # one host CPU executes every dispatched batch, one after another (all cores per batch)
    busy_until = [0.0]
    by_index = list(dep.stages)

    def on_batch(i, k, now):
        start = max(now, busy_until[0])
        busy_until[0] = start + latency(by_index[i], k)
        return busy_until[0] - now

    recs, _ = simulate_fixed(dep, clients, horizon, 0.0, latency, on_batch=on_batch)
    met = sum(1 for _c, _g, d, dl, s in recs if s == "completed" and d <= dl + 1e-9)
    return {"value": round(met / horizon, 2), "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
            "sample": f"fp32 CPU forward of {len(lat)} (span, k) points of this plan (best of 2 timed passes, "
                      f"{time.time() - t0:.1f}s) driving the oracle event loop over a {horizon:.1f}s horizon"}


def run_reference(args):
    world, rank, _ = _dist()
    if rank != 0:
        return
    from paper_2312_10636_b200.models import build_chain
    from paper_2312_10636_b200.plan import deploy

    # the achievable-throughput rule steps the fleet down until p99 <= SLO; on the host CPU no fleet
    # gets there, so the arm reports the smallest planned fleet (the most favourable to the CPU)
    wl = _workload(args.plans or args.model, args.clients) if args.clients is not None else _workloads(args.plans or args.model)[0]
    dep = deploy(wl["plan"], wl["fragments"])
    chain = build_chain(args.model)
    vals = []
    cpu = None
    for _ in range(max(1, args.steps)):
        cpu = cpu_baseline(args, wl, dep, chain, budget_s=max(5.0, 120.0 / max(1, args.steps)))
        vals.append(cpu["value"])
    value = sum(vals) / len(vals)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": args.window * 1000.0, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{args.model} re-aligned fragment groups, {wl['clients_n']} clients, CPU path",
                       "model": args.model},
            "cpu_baseline": cpu, "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                                         "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--window", type=float, default=1.0, help="seconds of arrivals per step")
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--model", default="resnet50")
    ap.add_argument("--plans", default=None,
                    help="workload fixture tag (default: the model; e.g. resnet50_s1.5 = plans made against the "
                         "profile table scaled by the served/profiled latency ratio)")
    ap.add_argument("--clients", type=int, default=None, help="fleet size per GPU (default: largest feasible plan)")
    ap.add_argument("--max-inflight", type=int, default=8192)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-ingress", choices=("zero_copy", "dma"), default="dma",
                    help="e2e host ingress: a copy-engine DMA of each request into a device slot at arrival "
                         "(default), or the gather reading pinned host memory over PCIe (zero_copy)")
    ap.add_argument("--strict-shares", action="store_true",
                    help="SM budget = planned share exactly (default: work-conserving, share is a floor)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
