"""Benchmark: SLO-met requests/sec for re-aligned ResNet-50 fragment groups on B200.

Workload (BASELINE.json configs[1]): a fleet of ResNet-50 clients at 30 rps cut at 8 partition
points, planned by the unmodified reference planner (merge -> group -> re-align -> placement)
against the measured B200 profile table; tests/golden/workload/resnet50*_c<N>.json.  The executor
serves that plan in real time: requests arrive on the wall clock (gen + mobile prefix + link
transfer), are batched per stage exactly as the reference simulator batches them, and every
dispatched batch runs on the GPU (ragged gather -> span kernels -> scatter) on an instance bounded
to the stage's SM share.  Every client ships its OWN fp32 entry activation (seeded, distinct per
client, resident in HBM for `value`; in pinned host memory, DMA-copied at arrival, for `e2e`).

A step is one serving window of `--window` seconds of arrivals.  `value` counts requests generated
in the K timed windows that complete within their deadline, divided by the timed window time;
valid only when p99 latency <= SLO.  After the last window no new requests are generated and the
ones already generated are served for `--drain` more seconds, so the last window's tail is
measured; requests still unfinished after that count as misses (latency +inf in the p99).

Output parity of the measured run: the last completions of the timed run (logits still held in
the result ring) are spot-checked against the fp32 CPU forward of their client's activation in the
CPU leg (`output_check`).

Multi-GPU (torchrun): one process per GPU, each serving its own independent fleet of the same
size (groups share no tensors; no collective on the data path): scaling "weak".

--impl reference: the reference's CPU path on the host (see run_reference / cpu_paths).
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
# --config: the BASELINE.json configs served on the same path (model, fixture tag, metric, workload)
CONFIGS = {
    "resnet50": ("resnet50", None, METRIC,
                 "resnet50 re-aligned fragment groups, {n} clients x {rps} rps per GPU, 8 cut points, plan from the "
                 "reference planner on the measured B200 profile table, SM-share partitioning"),
    "vgg16_churn": ("vgg16", "vgg16_churn", "SLO-met requests/sec (p99<=SLO) for VGG-16 fragment groups under "
                    "partition-point churn",
                    "vgg16 fragment groups under network-trace-driven partition-point churn: {n} clients x {rps} rps "
                    "per GPU on a fast/slow bandwidth trace (half out of phase), re-partitioned and re-planned by "
                    "the reference every 2-s epoch, plan transitions served on the wall clock"),
    "inception_v3": ("inception_v3", "inception_v3", "SLO-met requests/sec (p99<=SLO) for re-aligned "
                     "Inception-v3 groups",
                     "inception_v3 multi-branch re-aligned fragment groups (ragged gather across concat "
                     "boundaries), {n} clients x {rps} rps per GPU, 8 cut points at the Mixed blocks"),
    "bert_base": ("bert_base", "bert_base", "SLO-met requests/sec (p99<=SLO) for re-aligned BERT-base "
                  "encoder groups, seq 128",
                  "bert_base encoder fragments split at layer boundaries (cuts 0/3/6/9), seq 128, {n} clients x "
                  "{rps} rps per GPU, shared-suffix GEMM batching"),
}
UNIT = "req/s"
PCIE_GBS = 46.0  # measured H2D for 1 MB pinned copies on these hosts (scripts/probe_h2d_streams.py)


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d.get("bf16_tflops_sustained", 1401.0), d.get("bf16_tflops", 1659.7), d.get("hbm_gbs", 6538.6), "measured"
    return 1400.0, 1590.0, 6650.0, "fallback"


def _fkey(w):
    return (w["clients_n"], w.get("latency_scale", 1.0), -w.get("merge_threshold", 0.2))


def _family(w):
    return (w.get("latency_scale", 1.0), w.get("merge_threshold", 0.2))


def _workloads(name: str, all_plans: bool = False):
    """Planned fleets <name>_c<N>.json in ascending (clients, latency_scale) order; with all_plans
    also the fleets planned against the load-calibrated table (<name>_s<F>[_m<T>]_c<N>.json)."""
    pats = [f"{name}_c[0-9]*.json"] + ([f"{name}_s*_c[0-9]*.json"] if all_plans else [])
    files = [f for pat in pats for f in glob.glob(str(ROOT / "tests" / "golden" / "workload" / pat))]
    docs = [json.loads(Path(f).read_text()) for f in files]
    # plans for an N-GPU box (<tag>_g<N>_c*) belong to --placement plan only
    gpus = int(name.rsplit("_g", 1)[1]) if "_g" in name else 1
    return sorted((d for d in docs if d.get("gpus", 1) == gpus), key=_fkey)


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


def _plans(wl) -> list:
    return [e["plan"] for e in wl["epochs"] if e["kind"] == "deploy"] if "epochs" in wl else [wl["plan"]]


def _align_stages(wl) -> int:
    """Alignment stages of the plan (of the largest epoch plan for a churn fleet)."""
    return max(sum(1 for g in pl["groups"] for lv in g["levels"] for a in lv["align"] if a["span"][0] != a["span"][1])
               for pl in _plans(wl))


def _plan_resource(wl) -> int:
    return max(pl["total_resource"] for pl in _plans(wl))


def _h2d_gbs(w) -> float:
    by_id = {c["client_id"]: c for c in w["clients"]}
    frs = [e["fragments"] for e in w["epochs"] if e["kind"] == "deploy"] if "epochs" in w else [w["fragments"]]
    return max(sum(by_id[cid]["rate_rps"] * by_id[cid]["payload_bytes"][f["start_layer"]]
                   for f in fr for cid in f["clients"]) for fr in frs) / 1e9


def _p99(lats):
    lats = sorted(lats)
    return lats[min(len(lats) - 1, int(math.ceil(0.99 * len(lats))) - 1)] if lats else math.inf


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


def _lscpu() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=5).stdout
        kv = dict(line.split(":", 1) for line in out.splitlines() if ":" in line)
        return (f"{kv.get('Model name', '?').strip()}, {kv.get('Socket(s)', '?').strip()} socket(s), "
                f"{kv.get('CPU(s)', '?').strip()} CPUs")
    except Exception:  # noqa: BLE001
        return "lscpu unavailable"


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2312_10636_b200 import _native as N
    from paper_2312_10636_b200.device import context
    from paper_2312_10636_b200.engine import DeviceModel, StageInstance
    from paper_2312_10636_b200.models import build_chain
    from paper_2312_10636_b200.plan import deploy, deploy_epochs
    from paper_2312_10636_b200.serving import ClientView, serve

    world, rank, local = _dist()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = context(local)
    chain = build_chain(args.model)
    dm = DeviceModel(chain, local)

    class Fleet:
        """One planned fleet made executable on this GPU: stage instances plus every client's own
        fp32 entry activation (one seeded tensor per (client, cut point), post-ReLU at inner
        boundaries).  A churn fleet (BASELINE configs[2]) carries one deployment per epoch, put in
        place at that epoch's REPLAN (simulator.py:297-349); stages of every deployment stay alive
        so requests drain on the stages they were routed to."""

        def __init__(self, wl, strict: bool = False):
            self.wl = wl
            if "epochs" in wl:
                self.epochs = deploy_epochs(wl["epochs"])
                self.deps = [d for d in self.epochs if d is not None and not isinstance(d, str)]
            else:
                self.epochs = None
                self.deps = [deploy(wl["plan"], wl["fragments"])]
            self.dep = self.deps[0]
            self.stages = [s for d in self.deps for s in d.stages]
            self.clients = [ClientView.from_doc(c) for c in wl["clients"]]
            self.instances = []
            for d in self.deps:  # each deployment gets its planned shares on the whole GPU
                it = iter(ctx.sm_budgets([(s.share, s.instances) for s in d.stages], work_conserving=not strict,
                                         capacity=int(round(99 * args.sm_oversubscribe))))
                self.instances += [[StageInstance(dm, s.start, s.end, s.batch, next(it)) for _ in range(s.instances)]
                                   for s in d.stages]
            keys = sorted({(cid, r.point) for d in self.deps for cid, r in d.routes.items()})
            sizes = [chain.ingress_elems(p) for _cid, p in keys]
            pads = [-(-n // 16) * 16 for n in sizes]  # every client slice 64-byte aligned (16-byte vectors)
            g = torch.Generator(device="cuda").manual_seed(1234 + rank)
            self.act = torch.randn(sum(pads), device="cuda", generator=g)  # one slab, a slice per client
            self.dev_in, self.slices, off = {}, {}, 0
            for key, n, npad in zip(keys, sizes, pads):
                p = key[1]
                if chain.boundary_shape(p)[3] == N.GX_I32:  # BERT boundary 0: token ids (int32 bits)
                    self.act[off:off + n].view(torch.int32).random_(0, 30522, generator=g)
                elif p > 0 and chain.relu_boundary(p):
                    self.act[off:off + n].clamp_(min=0)
                self.slices[key] = (off, n, p)
                self.dev_in[key] = (self.act.data_ptr() + off * 4, n * 4, chain.ingress_channels(p))
                off += npad
            self.host = None
            self.host_in = None
            for s, insts in zip(self.stages, self.instances):  # capture every (instance, k) graph
                for inst in insts:
                    for k in range(1, s.batch + 1):
                        inst.kernel_count(k)
            torch.cuda.synchronize()

        def point_of(self, cid, gen_ms):
            """The cut point a request generated at gen_ms was routed at (routes are chosen at
            generation, simulator.py:353-366; a REPLAN at the same instant fires first, rank 0 <
            _R_GEN, simulator.py:40), None if it had no route."""
            if self.epochs is None:
                return self.dep.routes[cid].point
            ep = self.wl["epoch_s"] * 1000.0
            e = min(int(gen_ms // ep), len(self.epochs) - 1)
            di = -1
            for j in range(e + 1):
                d = self.epochs[j]
                if isinstance(d, str):
                    di = -1
                elif d is not None:
                    di = sum(1 for x in self.epochs[:j] if x is not None and not isinstance(x, str))
            r = self.deps[di].routes.get(cid) if di >= 0 else None
            return r.point if r is not None else None

        def pin(self):
            if self.host is None:
                self.host = torch.empty(self.act.numel(), dtype=torch.float32, pin_memory=True)
                self.host.copy_(self.act.cpu())
                base = self.host.data_ptr()
                self.host_in = {key: (base + off * 4, n * 4, self.dev_in[key][2])
                                for key, (off, n, _p) in self.slices.items()}
            return self.host_in

        def activation(self, cid, p):
            off, n, _p = self.slices[(cid, p)]
            return self.act[off:off + n].cpu()

        def serve(self, horizon, host=False, drain=0.0, sample=0):
            extra = {} if self.epochs is None else {"epochs": self.epochs, "epoch_s": self.wl["epoch_s"]}
            return serve(self.dep, self.clients, horizon, ctx=ctx, instances=self.instances, **extra,
                         ingress=self.pin() if host else self.dev_in,
                         ingress_from_host=(args.e2e_ingress if host else False), egress_to_host=host,
                         max_inflight=self.max_inflight(), drain_s=drain, sample_outputs=sample,
                         lane_policy={"split": 0, "least": 1, "time": 2, "earliest": 3, "edf": 4}[args.lanes])

        def max_inflight(self):
            """Device slots: at least --max-inflight, and 1.5x the requests an SLO's worth of
            arrivals keeps in flight (a request finding no free slot is an admission drop)."""
            rps = sum(c.rate_rps for c in self.clients)
            return max(args.max_inflight, int(math.ceil(1.5 * rps * self.wl["slo_ms"] / 1000.0)))

    def all_ok(ok: bool) -> bool:
        if world > 1:
            flag = torch.tensor([1 if ok else 0], device="cuda")
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
            ok = bool(flag.item())
        return ok

    def log(msg):
        if rank == 0:
            print(msg, file=sys.stderr, flush=True)

    window = args.window
    W, K = args.warmup, args.steps
    horizon = (W + K) * window

    def one_run(fleet, host: bool, sample: int = 0):
        """The measured serving run: W warm-up windows + K timed windows + the drain."""
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        rep = fleet.serve(horizon, host=host, drain=args.drain, sample=sample)
        e1.record()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t_lo, t_hi = W * window * 1000.0, horizon * 1000.0
        timed = [r for r in rep.requests if t_lo <= r[1] < t_hi]
        met = sum(1 for _c, _g, d, dl, s in timed if s == "completed" and d <= dl + 1e-9)
        # unfinished after the drain = missed: +inf in the p99
        lats = [(d - gg) if s == "completed" else math.inf for _c, gg, d, _dl, s in timed if s != "dropped"]
        dropped = sum(1 for r in timed if r[4] == "dropped")
        ing = fleet.dev_in
        return {"met": met, "generated": len(timed), "dropped": dropped, "p99": _p99(lats),
                "unfinished": sum(1 for r in timed if r[4] == "inflight"), "wall_ms": rep.wall_ms,
                "device_ms": e0.elapsed_time(e1), "kernels": rep.kernels, "batches": rep.batches, "rep": rep,
                "h2d": sum(ing[(c, fleet.point_of(c, g))][1] for c, g, _d, _dl, s in timed
                           if s != "dropped" and (c, fleet.point_of(c, g)) in ing) if host else 0,
                "d2h": sum(1 for r in timed if r[4] == "completed") * chain.boundary_elems(chain.n_units) * 4
                if host else 0}

    def passes(res, wl):
        return res["p99"] <= wl["slo_ms"] and res["dropped"] <= 0.01 * max(1, res["generated"])

    def search(cands, probe_s=3.0, strict=False):
        """Achievable throughput: the largest planned fleet whose served p99 stays
        within the SLO with < 1% drops, probed for `probe_s` seconds from the top down (p99 over
        arrivals after the first second)."""
        for wl in reversed(cands):
            cand = Fleet(wl, strict)
            rep = cand.serve(probe_s)
            lats = [d - g for _c, g, d, _dl, s in rep.requests if s == "completed" and g >= 1000.0]
            ok = _p99(lats) <= wl["slo_ms"] and rep.dropped <= 0.01 * max(1, rep.generated)
            log(f"# probe clients={wl['clients_n']} scale={wl.get('latency_scale', 1.0)} "
                f"merge={wl.get('merge_threshold', 0.2)}{' strict' if strict else ''}: p99={_p99(lats):.1f} ms "
                f"met/s={rep.slo_met / probe_s:.0f} -> {'ok' if ok else 'over'}")
            if all_ok(ok):
                return cand
            del cand
        return Fleet(cands[0], strict)

    def timed_search(fleet, cands, host=False, sample=0, strict=False, retry_near=False):
        """The timed run is the verdict: on a miss, step down to the next smaller fleet."""
        res = one_run(fleet, host, sample)
        first = res
        smaller = [w for w in reversed(cands) if _fkey(w) < _fkey(fleet.wl)]
        retried = False
        while not all_ok(passes(res, fleet.wl)) and smaller:
            log(f"# timed clients={fleet.wl['clients_n']}{' e2e' if host else ''}: p99={res['p99']:.1f} ms -> over")
            if retry_near and not retried and res["p99"] <= 2.0 * fleet.wl["slo_ms"]:
                retried = True  # host ingress makes the tail noisier: one retry of a near miss
                res = one_run(fleet, host, sample)
                continue
            retried = False
            fleet = Fleet(smaller.pop(0), strict)
            res = one_run(fleet, host, sample)
        return fleet, res, first

    all_wl = _workloads(args.plans or args.model, all_plans=args.all_plans)
    sample = 256 if (rank == 0 and not args.no_cpu_baseline) else 0
    with ClockSampler(local) as clk:
        if args.clients is not None:
            fleet = Fleet(_workload(args.plans or args.model, args.clients))
            res = one_run(fleet, False, sample)
        else:
            fleet = search(all_wl)
            fleet, res, _ = timed_search(fleet, all_wl, sample=sample)
    wl, stages, instances = fleet.wl, fleet.stages, fleet.instances
    slo = wl["slo_ms"]
    log(f"# value: clients={wl['clients_n']} met/s={res['met'] / (K * window):.0f} p99={res['p99']:.1f} ms")

    # e2e through the host path, same plan family as `value` (same latency scale and merge
    # threshold): first the value fleet itself, then down the family to the fleets whose PCIe
    # demand fits the link (fleets above ~85% of it queue on the copy engine without bound)
    family = [w for w in all_wl if _family(w) == _family(wl)]
    e2e_cands = [w for w in family if _fkey(w) < _fkey(wl) and _h2d_gbs(w) <= 0.92 * PCIE_GBS]
    if not e2e_cands:  # the value fleet's family has no fleet within the link: the nearest family that does
        fams = sorted({_family(w) for w in all_wl if _h2d_gbs(w) <= 0.92 * PCIE_GBS},
                      key=lambda f: (abs(f[0] - _family(wl)[0]), abs(f[1] - _family(wl)[1])))
        if fams:
            e2e_cands = [w for w in all_wl if _family(w) == fams[0] and _h2d_gbs(w) <= 0.92 * PCIE_GBS]
    res_e2e = one_run(fleet, True)
    e2e_on_value = res_e2e
    e2e_fleet = fleet
    if args.clients is None and not all_ok(passes(res_e2e, wl)) and e2e_cands:
        log(f"# e2e on the value fleet: p99={res_e2e['p99']:.1f} ms (PCIe demand {_h2d_gbs(wl):.1f} GB/s) -> "
            f"down the family")
        e2e_fleet = Fleet(e2e_cands[-1])
        e2e_fleet, res_e2e, _ = timed_search(e2e_fleet, e2e_cands, host=True, retry_near=True)

    # variants beside the tuned line: the same fleet with the planned shares as hard SM budgets,
    # and the best fleet planned against the UNSCALED measured table (latency_scale 1, default merge)
    variants = {}
    if not args.no_variants and args.clients is None:
        fs = Fleet(wl, strict=True)
        rs = one_run(fs, False)
        variants["strict_shares_same_fleet"] = {
            "value": round(rs["met"] / (K * window), 1), "p99_ms": round(rs["p99"], 3), "p99_ok": passes(rs, wl),
            "clients_per_gpu": wl["clients_n"]}
        del fs
        unscaled = [w for w in all_wl if _family(w) == (1.0, 0.2)]
        if unscaled:
            fu = search(unscaled)
            fu, ru, _ = timed_search(fu, unscaled)
            variants["latency_scale_1_default_merge"] = {
                "value": round(ru["met"] / (K * window), 1), "p99_ms": round(ru["p99"], 3),
                "p99_ok": passes(ru, fu.wl), "clients_per_gpu": fu.wl["clients_n"],
                "align_stages": _align_stages(fu.wl)}
            del fu

    # roofline of the dominant kernel, the implicit-GEMM conv (conv_tc_kernel, plus conv_halo_kernel
    # for wide 3x3 layers: >=90% of GPU time in every launch list under profiles/): the busiest
    # stage's span, each conv launched alone on the stage's stream and timed with CUDA events
    # (gx_stage_profile_ops), algorithmic FLOPs = 2*M*N*K unpadded per launch, peak = measured burst
    # bf16 x (stage SM budget / SMs) since the kernel is timed alone.
    def stage_flops(i):
        s = stages[i]
        return s.instances * s.batch * sum(chain.unit_flops[s.start:s.end])

    busiest = max(range(len(stages)), key=stage_flops)
    st = stages[busiest]
    inst = instances[busiest][0]
    span_ms = inst.profile(st.batch, 20)
    ops = inst.profile_ops(st.batch, 10)
    convs = [o for o in ops if o["kind"] in (N.GX_OP_CONV, N.GX_OP_LINEAR, N.GX_OP_FC)]
    conv_ms = sum(o["ms"] for o in convs)
    conv_flops = sum(o["flops"] for o in convs)
    conv_bytes = sum(o["bytes"] for o in convs)
    sustained, burst, hbm, src = _peaks()
    achieved = conv_flops / (conv_ms * 1e-3) / 1e12
    peak_scaled = burst * inst.sm_budget / ctx.sm_count
    # attainable time per conv on its SM budget: the tensor peak or the per-SM L2<->SM data path,
    # whichever binds (profiles/r02_sm_feed_probe.log: bulk reads 86 B/clk, stores 31.5 B/clk, a
    # concurrent read + write stream ~25 B/clk each), reads = inputs + weights + residual, writes =
    # the output; the K=64 1x1 convs of layer1/2 write 2 bytes per 128 FLOP and sit on the write path
    first_op = chain.unit_first_op[st.start]
    clk_hz = 1.965e9
    att_s = 0.0
    for o in convs:
        op = chain.ops[first_op + o["op"]]
        oh, ow, oc, dt = chain.tensors[op.out]  # (not W / H: W is the warm-up window count)
        wbytes = st.batch * oh * ow * (op.Cout or oc) * (4 if dt == N.GX_F32 else 2)
        rbytes = max(0.0, o["bytes"] - wbytes)
        t_tc = o["flops"] / (burst * 1e12 * inst.sm_budget / ctx.sm_count)
        t_mem = max(rbytes / 86.0, wbytes / 31.5, (rbytes + wbytes) / 50.0) / inst.sm_budget / clk_hz
        att_s += max(t_tc, t_mem)
    span_flops = st.batch * sum(chain.unit_flops[st.start:st.end])
    traffic = None
    ncu_path = ROOT / "profiles" / "ncu_conv_summary.json"
    nkey = f"{args.model}:{st.start}:{st.end}:{st.batch}:{inst.sm_budget}"
    if ncu_path.exists():
        ent = json.loads(ncu_path.read_text()).get(nkey)
        if ent:
            traffic = {"dram_bytes_per_launch": ent["dram_bytes_per_launch"],
                       "l2_to_smem_bytes_per_launch": ent.get("tma_bytes_per_launch"),
                       "algorithmic_bytes_per_launch": round(conv_bytes / max(1, len(convs))),
                       "tensor_pipe_pct": ent.get("tensor_pct"),
                       "source": f"profiles/ncu_conv_summary.json[{nkey}] ({ent['launches']} launches, ncu --set full)"}
    stats = torch.tensor([res["met"], res["generated"], res["dropped"], res_e2e["met"], res["kernels"],
                          res["h2d"], res_e2e["h2d"], res_e2e["d2h"], res["unfinished"], e2e_on_value["met"]],
                         dtype=torch.float64, device="cuda")
    times = torch.tensor([res["device_ms"], res_e2e["device_ms"], res["p99"], res_e2e["p99"], e2e_on_value["p99"]],
                         dtype=torch.float64, device="cuda")
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
            cpu = cpu_paths(args, budget_s=args.cpu_budget)
            # output parity of the measured run, on the CPU leg: the sampled completions of the
            # timed run vs the fp32 CPU forward of their clients' activations
            cpu["output_check"] = output_check(args.model, res["rep"], fleet)
        line = {
            "metric": args.metric, "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": K,
            "warmup": W, "ms_per_step": round(window * 1000.0, 3), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded random-init weights, a distinct seeded "
                                                          "fp32 activation per client)",
            "config": {"workload": args.workload.format(n=wl["clients_n"], rps=f"{wl['rate_rps']:.0f}"),
                       "model": args.model, "latency_scale": wl.get("latency_scale", 1.0),
                       "merge_threshold": wl.get("merge_threshold", 0.2), "align_stages": _align_stages(wl),
                       "clients_per_gpu": wl["clients_n"], "offered_rps_per_gpu":
                           wl["clients_n"] * wl["rate_rps"], "slo_ms": round(slo, 3), "window_s": window,
                       "drain_s": args.drain, "stages": len(stages),
                       "instances": sum(s.instances for s in stages),
                       "plan_resource": _plan_resource(wl), "parallelism": f"replica-per-gpu x{world}",
                       "sm_budgets": "work-conserving (planned share is a floor)",
                       "l2": "per-client activations in HBM (2+ GB > L2), weights L2-resident per stage"},
            "p99_ms": round(p99, 3), "p99_ok": p99 <= slo, "generated": int(stats[1].item()),
            "dropped": int(stats[2].item()), "unfinished_after_drain": int(stats[8].item()),
            "e2e": {"value": round(e2e_value, 1), "unit": UNIT, "p99_ms": round(p99_e2e, 3),
                    "p99_ok": p99_e2e <= e2e_fleet.wl["slo_ms"], "clients_per_gpu": e2e_fleet.wl["clients_n"],
                    "latency_scale": e2e_fleet.wl.get("latency_scale", 1.0),
                    "merge_threshold": e2e_fleet.wl.get("merge_threshold", 0.2),
                    "align_stages": _align_stages(e2e_fleet.wl),
                    "pcie_demand_gbs": round(_h2d_gbs(e2e_fleet.wl), 1),
                    "on_value_fleet": {"value": round(stats[9].item() / timed_s, 1),
                                       "p99_ms": round(times[4].item(), 3),
                                       "pcie_demand_gbs": round(_h2d_gbs(wl), 1)},
                    "path": ("serve() with host ingress: gather kernels read fp32 entry activations from pinned "
                             "host memory over PCIe (zero-copy), logits scattered to mapped host memory")
                    if args.e2e_ingress == "zero_copy" else
                    ("serve() with host ingress: each request's fp32 entry activation DMA-copied from pinned host "
                     "memory into a device slot at arrival (copy engine, per-request event the batch waits on), "
                     "logits scattered to mapped host memory"),
                    "h2d_bytes_per_step": int(stats[6].item() / K), "d2h_bytes_per_step": int(stats[7].item() / K)},
            "variants": variants,
            "gpu_launches": int(stats[4].item()),
            "roofline": {"bound": "tensor",
                         "kernel": f"implicit-GEMM conv (conv_tc_kernel / conv_halo_kernel) x{len(convs)} launches of "
                                   f"span [{st.start},{st.end}) k={st.batch} "
                                   f"on {inst.sm_budget} SMs (busiest stage, planned share {st.share}%)",
                         "achieved": round(achieved, 2), "peak": round(peak_scaled, 2), "unit": "TFLOP/s",
                         "frac": round(achieved / peak_scaled, 4), "traffic": traffic,
                         "attainable": {"frac": round(att_s / (conv_ms * 1e-3), 4),
                                        "us": round(att_s * 1e6, 1), "measured_us": round(conv_ms * 1000, 1),
                                        "model": "per conv max(FLOPs / tensor peak x budget/148, per-SM data "
                                                 "path: reads/86, writes/31.5, (reads+writes)/50 B/clk x budget)"},
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


def run_placed(args):
    """--placement plan (N > 1): ONE fleet planned for the whole N-GPU box by the reference planner
    (plan_realigned with gpus=N packs and places every stage instance, placement.py:24-70;
    tests/golden/workload/<model>_s2_m0_g<N>_c*.json), served by one host loop on rank 0 that runs
    instance i of stage s on GPU placement[s][i]; stage FIFOs stay global (simulator.py:91), a batch
    prefers a free instance on the GPU holding its activations, and an alignment output produced on
    another GPU is gathered over NVLink (peer access) — no NCCL on the data path.  Other ranks only
    hold their GPU and wait.  Same metric and JSON line as the replica mode."""
    import datetime

    import torch
    import torch.distributed as dist

    from paper_2312_10636_b200.device import context
    from paper_2312_10636_b200.engine import DeviceModel, placed_instances
    from paper_2312_10636_b200.models import build_chain
    from paper_2312_10636_b200.plan import deploy
    from paper_2312_10636_b200.serving import ClientView, serve

    world, rank, local = _dist()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local), timeout=datetime.timedelta(hours=2))
    if rank == 0:
        chain = build_chain(args.model)
        models = {g: DeviceModel(chain, g) for g in range(world)}
        fleets = _workloads(f"{args.model}_s2_m0_g{world}")
        if not fleets:
            raise SystemExit(f"no {world}-GPU fleets: run scripts/make_workload.py {args.model} ... --gpus {world}")
        W, K, window = args.warmup, args.steps, args.window
        horizon = (W + K) * window

        def build(wl):
            dep = deploy(wl["plan"], wl["fragments"])
            inst = placed_instances(dep, models, capacity=int(round(99 * args.sm_oversubscribe)))
            clients = [ClientView.from_doc(c) for c in wl["clients"]]
            ingress, keep = {}, []
            for cid in sorted(c.client_id for c in clients if c.client_id in dep.routes):
                r = dep.routes[cid]
                home = dep.stages[r.stages[0]].gpus[0] if r.stages and dep.stages[r.stages[0]].gpus else 0
                g = torch.Generator(device=f"cuda:{home}").manual_seed(1234 + len(keep))
                x = torch.randn(chain.ingress_elems(r.point), device=f"cuda:{home}", generator=g)
                if r.point > 0:
                    x.clamp_(min=0)
                keep.append(x)
                ingress[cid] = (x.data_ptr(), x.numel() * 4, chain.ingress_channels(r.point))
            for s, row in zip(dep.stages, inst):
                for i in row:
                    for k in range(1, s.batch + 1):
                        i.kernel_count(k)
            return dep, inst, clients, ingress, keep

        def measure(wl, secs):
            dep, inst, clients, ingress, keep = build(wl)
            for g in range(world):
                torch.cuda.synchronize(g)
            rep = serve(dep, clients, secs, ctx=context(0), instances=inst, ingress=ingress,
                        max_inflight=args.max_inflight, drain_s=args.drain)
            t_lo, t_hi = (W * window * 1000.0, secs * 1000.0) if secs == horizon else (1000.0, secs * 1000.0)
            timed = [r for r in rep.requests if t_lo <= r[1] < t_hi]
            lats = [(d - g) if s == "completed" else math.inf for _c, g, d, _dl, s in timed if s != "dropped"]
            met = sum(1 for _c, _g, d, dl, s in timed if s == "completed" and d <= dl + 1e-9)
            dropped = sum(1 for r in timed if r[4] == "dropped")
            ok = _p99(lats) <= wl["slo_ms"] and dropped <= 0.01 * max(1, len(timed))
            return {"met": met, "p99": _p99(lats), "ok": ok, "kernels": rep.kernels, "generated": len(timed),
                    "dropped": dropped}

        chosen, res = fleets[0], None
        with ClockSampler(0) as clk:
            for wl in reversed(fleets):
                probe = measure(wl, 3.0)
                print(f"# placed probe clients={wl['clients_n']}: p99={probe['p99']:.1f} ms -> "
                      f"{'ok' if probe['ok'] else 'over'}", file=sys.stderr, flush=True)
                if probe["ok"]:
                    chosen = wl
                    break
            res = measure(chosen, horizon)
        n_inst = collections_counter(s for g in chosen["plan"]["groups"] for lv in g["levels"]
                                     for st in [lv["shared"], *lv["align"]] for s in (st["gpu"] or []))
        value = res["met"] / (K * window)
        line = {"metric": args.metric, "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
                "ms_per_step": window * 1000.0, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "bf16", "data": "synthetic (seeded random-init weights, a distinct activation per client)",
                "config": {"workload": f"{args.model} re-aligned fragment groups, ONE {chosen['clients_n']}-client "
                                       f"fleet planned for {world} GPUs and placed by the reference planner",
                           "parallelism": f"placement-faithful x{world} (one host loop, peer-access hand-off)",
                           "instances_per_gpu": dict(n_inst), "slo_ms": chosen["slo_ms"]},
                "p99_ms": round(res["p99"], 3), "p99_ok": res["ok"], "generated": res["generated"],
                "dropped": res["dropped"], "gpu_launches": res["kernels"], "clocks": clk.summary(),
                "e2e": None, "roofline": None, "cpu_baseline": None}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def collections_counter(it):
    import collections

    return collections.Counter(it)


# ------------------------------------------------------------------------------------------------
# CPU legs (the only place bench.py touches oracle/: the checker and the CPU baseline)
# ------------------------------------------------------------------------------------------------

def output_check(model, rep, fleet, tol=2e-2):
    """The sampled completions of the measured run vs the fp32 CPU forward of the same client
    activation: max relative L2 error and top-1 agreement (decisive fp32 top-1 only)."""
    import torch

    from oracle.units import nhwc_to_nchw, run_span, units_for
    from paper_2312_10636_b200.models import build_chain, torch_model

    if rep.sampled is None or len(rep.sampled[0]) == 0:
        return {"checked": 0, "sampled": 0}
    t0 = time.time()
    torch.set_num_threads(os.cpu_count() or 1)
    m = torch_model(model)
    units = units_for(model, m)
    ch = build_chain(model, module=m)
    idx, outs = rep.sampled
    cids = [rep.requests[i][0] for i in idx]
    points = [fleet.point_of(rep.requests[i][0], rep.requests[i][1]) for i in idx]
    by_point = {}
    for j, (cid, p) in enumerate(zip(cids, points)):
        if p is not None:
            by_point.setdefault(p, []).append(j)
    classifier = model != "bert_base"  # BERT's final output is the hidden state: no top-1
    rels, agree, decisive = [], 0, 0
    units_bf16, relaxed, passed = None, [], []
    for p, js in by_point.items():
        for b0 in range(0, len(js), 16):
            part = js[b0:b0 + 16]
            xs = []
            for j in part:
                a = fleet.activation(cids[j], p)
                H, W, Cc, _ = ch.boundary_shape(p)
                if not classifier:
                    xs.append(a.view(torch.int32).view(1, H) if p == 0 else a.view(1, H, Cc))
                elif p == 0:
                    f = ch.tensor_s2d.get(ch.boundary[0], 1)
                    xs.append(a.view(1, H * f, W * f, ch.input_channels))
                else:
                    xs.append(a.view(1, H, W, Cc))
            xin = nhwc_to_nchw(torch.cat(xs))
            ref = run_span(units, p, ch.n_units, xin)
            for jj, (r, j) in enumerate(zip(ref, part)):
                got = torch.from_numpy(outs[j])
                r = r.reshape(-1)
                rel = ((got - r).norm() / r.norm()).item()
                within = rel <= tol
                if model == "inception_v3" and rel > tol:
                    # random-init Inception-v3 amplifies bf16 rounding ~20x (test_models_gpu.py): the
                    # bound is 1.25x the framework's own bf16 error on the same suffix and input
                    if units_bf16 is None:
                        import copy
                        units_bf16 = units_for(model, copy.deepcopy(m).to(torch.bfloat16))
                    fb = run_span(units_bf16, p, ch.n_units, xin[jj:jj + 1].to(torch.bfloat16)).float().reshape(-1)
                    bound = 1.25 * ((fb - r).norm() / r.norm()).item()
                    relaxed.append((rel, bound))
                    within = rel <= bound
                rels.append(rel)
                passed.append(within)
                top2 = r.topk(2).values
                if classifier and (top2[0] - top2[1]) > 0.02 * (r.max() - r.min()):
                    decisive += 1
                    agree += int(int(got.argmax()) == int(r.argmax()))
    if not rels:
        return {"checked": 0, "sampled": len(idx), "unresolved_points": sum(1 for p in points if p is None),
                "examples": [list(rep.requests[i][:2]) for i in idx[:3]]}
    return {"checked": len(rels), "distinct_clients": len(set(cids)), "cut_points": sorted(by_point),
            "max_rel_l2": round(max(rels), 6), "median_rel_l2": round(sorted(rels)[len(rels) // 2], 6),
            "top1_decisive": decisive, "top1_agree": agree, "tolerance": tol,
            "inception_bf16_bound": ({"samples": len(relaxed), "max_rel_l2": round(max(a for a, _ in relaxed), 6),
                                      "max_bound": round(max(b for _, b in relaxed), 6),
                                      "rule": "rel <= max(2e-2, 1.25 x torch-bf16 error of the same suffix on the "
                                              "same input), as tests/test_replay_gpu.py"} if relaxed else None),
            "ok": all(passed) and agree == decisive, "cpu_s": round(time.time() - t0, 1),
            "oracle": "fp32 CPU forward (oracle/units.py, torchvision definitions) of each sampled request's "
                      "client activation; requests are the last completions of the timed run"}


def _ref_import():
    """The unmodified reference installed under baseline/_ref (pip --target), else the source tree."""
    for p in (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")):
        if (p / "fragserve" / "__init__.py").exists():
            sys.path.insert(0, str(p))
            import fragserve  # noqa: F401

            return str(p)
    return None


def reference_cpu_path(wl, repeats=3):
    """The reference's own CPU path on this host: plan_realigned per epoch
    (best of N, as pkg/benchmarks/bench_kernels.py:30-37) on this fleet's fragments, checked equal
    to the committed plan, and simulate(fixed_plan=plan) throughput (simulated requests and heap
    events per wall second; _deploy resolves merged fragments, the SURVEY §0.6 defect)."""
    where = _ref_import()
    if where is None:
        return {"unavailable": "reference not installed (baseline/_ref) and source tree absent"}
    if "epochs" in wl:
        return {"unavailable": "churn fleets are re-planned per epoch by the reference's own loop "
                               "(scripts/make_config_fleets.py); timed on the static fleets only"}
    import logging

    import fragserve
    logging.getLogger("fragserve").setLevel(logging.ERROR)  # per-client "offloading is pointless" notes
    from fragserve import (BandwidthTrace, ClientSpec, DeviceProfile, LayerSpec, ModelSpec, Scenario, SimConfig,
                           load_profiles, plan_to_dict)
    from fragserve import simulator as S
    from fragserve.merging import MergeConfig, merge_fragments
    from fragserve.planners import plan_realigned
    from fragserve.workload import Fragment, transfer_ms

    ms = wl["model_spec"]
    spec = ModelSpec(ms["model_id"], ms["input_bytes"],
                     tuple(LayerSpec(x["compute_weight"], x["output_bytes"]) for x in ms["layers"]))
    cuts = wl["cuts"]
    clients, frags = [], []
    for c in wl["clients"]:
        j = int(c["client_id"][1:])
        p = cuts[j % len(cuts)]
        dev = DeviceProfile(f"dev_{c['client_id']}", {spec.model_id: tuple(c["mobile_ms"])})
        cl = ClientSpec(c["client_id"], dev, spec, c["rate_rps"], c["slo_ms"],
                        BandwidthTrace(tuple(c["trace_t_s"]), tuple(c["trace_mbps"])))
        clients.append(cl)
        t = cl.slo_ms - dev.mobile_ms(spec.model_id, p) - transfer_ms(spec.payload_bytes(p), c["trace_mbps"][0])
        frags.append(Fragment(cl.client_id, spec.model_id, p, t, cl.rate_rps, frozenset({cl.client_id})))
    table = ROOT / wl["profile"]
    scale = wl.get("latency_scale", 1.0)
    if scale != 1.0:
        import tempfile
        out = []
        for ln in table.read_text().splitlines():
            if ln.startswith("#") or ln.startswith("model,"):
                out.append(ln)
                continue
            f = ln.split(",")
            f[-1] = f"{float(f[-1]) * scale:.6f}"
            out.append(",".join(f))
        table = Path(tempfile.mkdtemp()) / "table.csv"
        table.write_text("\n".join(out) + "\n")
    cost = load_profiles(table, batch_max=16)
    mcfg = MergeConfig(threshold=wl.get("merge_threshold", 0.2))
    models = {spec.model_id: spec}
    plan = plan_realigned(frags, models, cost, gpus=1, capacity=99, merge_cfg=mcfg)  # warm (numba JIT)
    best = math.inf
    for _ in range(repeats):
        t0 = time.perf_counter()
        plan = plan_realigned(frags, models, cost, gpus=1, capacity=99, merge_cfg=mcfg)
        best = min(best, time.perf_counter() - t0)
    same_plan = plan_to_dict(plan) == wl["plan"]
    merged = merge_fragments(frags, mcfg, cost, models)

    class Sim(S._Sim):
        n_events = 0

        def _push(self, t, rank, payload):
            Sim.n_events += 1
            super()._push(t, rank, payload)

        def _deploy(self, plan, fragments):
            return super()._deploy(plan, merged)

    horizon = 5.0
    sc = Scenario(tuple(clients), 1, 60.0, models)
    t0 = time.perf_counter()
    srep = Sim(sc, cost, "realign", SimConfig(horizon_s=horizon, merge_cfg=mcfg), fixed_plan=plan).run()
    wall = time.perf_counter() - t0
    return {"source": where, "fragserve": getattr(fragserve, "__version__", "0.1.0"),
            "plan_realigned_ms_per_epoch": round(best * 1000.0, 2), "plan_fragments": len(frags),
            "plan_equals_committed": same_plan,
            "simulate_req_per_s": round(srep.generated / wall, 1), "simulate_events_per_s": round(Sim.n_events / wall, 1),
            "simulate_horizon_s": horizon, "simulate_wall_s": round(wall, 2),
            "note": "the reference executes no DNN: simulate() prices each batch with the cost table"}


def cpu_serving_rate(model, budget_s=40.0, horizon_s=3.0, tag=None):
    """The CPU restatement of the execution step as a steady-state rate: the
    reference's batching (oracle event loop, pinned bit-exact to the reference) with every
    dispatched batch executed for real — fp32 torch forward of the span on all host cores, one
    batch at a time (the host CPU is one executor) — on growing client prefixes of the smallest
    planned fleet (the workload's cut mix, cheapest cuts first).  Returns the largest prefix whose
    p99 meets the SLO with < 1% drops, plus the CPU's execution rate on the dispatched batches."""
    import torch

    from oracle.serving import simulate_fixed
    from oracle.units import run_span, units_for
    from paper_2312_10636_b200.models import build_chain, torch_model
    from paper_2312_10636_b200.plan import deploy
    from paper_2312_10636_b200.serving import ClientView

    torch.set_num_threads(os.cpu_count() or 1)
    m = torch_model(model)
    units = units_for(model, m)
    chain = build_chain(model, module=m)
    wl = (_workloads(tag, all_plans=True) if tag else _workloads(model) or _workloads(model, all_plans=True))[0]
    first = next(e for e in wl["epochs"] if e["kind"] == "deploy") if "epochs" in wl else wl
    dep = deploy(first["plan"], first["fragments"])
    # clients in descending id order: the cut mix cycles from the cheapest suffix (cut 17) down to
    # the full model (cut 0), so every prefix is the most favourable fleet of its size for the CPU
    allc = sorted((ClientView.from_doc(c) for c in wl["clients"]), key=lambda c: c.client_id, reverse=True)
    inputs = {}

    def x_for(a, k):
        if (a, k) not in inputs:
            H, W, Cc, _ = chain.boundary_shape(a)
            if model == "bert_base":
                inputs[(a, k)] = torch.randint(0, 30522, (k, H)) if a == 0 else torch.randn(k, H, Cc)
            elif a == 0:
                f = chain.tensor_s2d.get(chain.boundary[0], 1)
                inputs[(a, k)] = torch.randn(k, chain.input_channels, H * f, W * f)
            else:
                inputs[(a, k)] = torch.randn(k, Cc, H, W).clamp_min(0)
        return inputs[(a, k)]

    t_start = time.time()
    best, tried, exec_imgs, exec_s = None, [], 0, 0.0
    for n in range(1, len(allc) + 1):
        if time.time() - t_start > budget_s:
            break
        busy = [0.0]

        def on_batch(i, k, now):
            nonlocal exec_imgs, exec_s
            s = dep.stages[i]
            t0 = time.perf_counter()
            run_span(units, s.start, s.end, x_for(s.start, k))
            dt = (time.perf_counter() - t0) * 1000.0
            exec_imgs += k
            exec_s += dt / 1000.0
            start = max(now, busy[0])
            busy[0] = start + dt
            return busy[0] - now

        recs, _ = simulate_fixed(dep, allc[:n], horizon_s, 0.0, lambda spec, k: 0.0, on_batch=on_batch)
        t_lo, t_hi = 500.0, horizon_s * 1000.0 - 300.0
        timed = [r for r in recs if t_lo <= r[1] < t_hi]
        lats = [(d - g) if s == "completed" else math.inf for _c, g, d, _dl, s in timed if s != "dropped"]
        met = sum(1 for _c, _g, d, dl, s in timed if s == "completed" and d <= dl + 1e-9)
        dropped = sum(1 for r in timed if r[4] == "dropped")
        p99 = _p99(lats)
        ok = p99 <= wl["slo_ms"] and dropped <= 0.01 * max(1, len(timed))
        tried.append({"clients": n, "p99_ms": round(p99, 1) if p99 < math.inf else None,
                      "met_per_s": round(met / ((t_hi - t_lo) / 1000.0), 1), "ok": ok})
        if not ok:
            break
        best = tried[-1]
    value = best["met_per_s"] if best else 0.0
    return {"value": value, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
            "host": _lscpu(),
            "sample": (f"{best['clients'] if best else 0} clients of the {wl['clients_n']}-client fleet "
                       f"(its cut cycle {wl.get('cuts', 'of epoch 0')} from the cheapest cut down, {wl['rate_rps']:.0f} rps each), {horizon_s:.0f} s of arrivals per size, every "
                       f"dispatched batch run as fp32 torch on {os.cpu_count()} threads (no interpolation)"),
            "search": tried,
            "cpu_exec_img_per_s": round(exec_imgs / exec_s, 2) if exec_s else None,
            "wall_s": round(time.time() - t_start, 1)}


def cpu_paths(args, budget_s=40.0):
    """Both CPU legs: the steady-state CPU serving rate (the baseline value) and the reference's
    own planner / simulator timings on the headline fleet."""
    out = cpu_serving_rate(args.model, budget_s=budget_s, tag=args.plans)
    head = [w for w in _workloads(args.plans or args.model, all_plans=True)]
    try:
        out["reference_path"] = reference_cpu_path(head[-1] if head else _workloads(args.model)[-1])
        out["reference_path"]["fleet_clients"] = (head[-1] if head else {}).get("clients_n")
    except Exception as e:  # noqa: BLE001 - the reference leg is reported, never fatal
        out["reference_path"] = {"error": f"{type(e).__name__}: {e}"}
    return out


def run_reference(args):
    world, rank, _ = _dist()
    if rank != 0:
        return
    vals = []
    cpu = None
    for _ in range(max(1, args.steps)):
        cpu = cpu_serving_rate(args.model, budget_s=max(20.0, 150.0 / max(1, args.steps)), tag=args.plans)
        vals.append(cpu["value"])
    value = sum(vals) / len(vals)
    head = _workloads(args.plans or args.model, all_plans=True)
    try:
        cpu["reference_path"] = reference_cpu_path(head[-1])
    except Exception as e:  # noqa: BLE001
        cpu["reference_path"] = {"error": f"{type(e).__name__}: {e}"}
    line = {"impl": "reference", "metric": args.metric, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": args.window * 1000.0, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{args.model} re-aligned fragment groups (the workload's cut mix), CPU path",
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
    ap.add_argument("--drain", type=float, default=0.5, help="seconds served after the last window (no new arrivals)")
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", choices=tuple(CONFIGS), default="resnet50",
                    help="BASELINE.json config: resnet50 (configs[1], the headline), vgg16_churn (configs[2]), "
                         "inception_v3 (configs[3]), bert_base (configs[4])")
    ap.add_argument("--model", default=None, help="override the config's model")
    ap.add_argument("--plans", default=None,
                    help="workload fixture tag (default: the model; e.g. resnet50_s1.5 = plans made against the "
                         "profile table scaled by the served/profiled latency ratio)")
    ap.add_argument("--clients", type=int, default=None, help="fleet size per GPU (default: largest feasible plan)")
    ap.add_argument("--max-inflight", type=int, default=8192)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-variants", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=40.0, help="seconds for the CPU serving-rate search")
    ap.add_argument("--e2e-ingress", choices=("zero_copy", "dma"), default="dma",
                    help="e2e host ingress: a copy-engine DMA of each request into a device slot at arrival "
                         "(default), or the gather reading pinned host memory over PCIe (zero_copy)")
    ap.add_argument("--sm-oversubscribe", type=float, default=4.0,
                    help="work-conserving SM budgets may sum to this multiple of the GPU's SMs (at most 32 "
                         "batches execute at once, one per hardware queue: budgets summing to 1x leave SMs idle)")
    ap.add_argument("--lanes", choices=("split", "least", "time", "earliest", "edf"), default="split",
                    help="stream-lane policy (graft_exec.h GX_LANE_*): one lane per hardware queue with queues "
                         "reserved for short stages (default), least-loaded of 64 lanes, the same with priorities "
                         "by expected batch time, or one lane per hardware queue, earliest free")
    ap.add_argument("--placement", choices=("replicas", "plan"), default="replicas",
                    help="N > 1: an independent fleet per GPU (default), or one fleet planned and placed across "
                         "the N GPUs (run_placed)")
    args = ap.parse_args()
    model, tag, args.metric, args.workload = CONFIGS[args.config]
    args.model = args.model or model
    args.all_plans = args.plans is None  # the config's plan families (load-calibrated tables, merge thresholds)
    args.plans = args.plans or tag
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    elif args.placement == "plan" and int(os.environ.get("WORLD_SIZE", "1")) > 1:
        run_placed(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
