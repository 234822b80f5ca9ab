"""Generate golden serving fixtures by running the UNMODIFIED reference (fragserve) here.

For each case: the reference planner's plan (plan_to_dict), the fragments it planned, the clients,
the per-stage latency tables `_StageRT.latency_for` would use, and the reference simulator's
output under `simulate(..., fixed_plan=plan)`: every request record and the dispatch log
(time, stage, k, request seqs) captured by a `_Sim._push` hook.  The executor's native serving
loop (virtual clock) and the oracle restatement must reproduce these bit for bit.

Needs /root/reference (this container only).  Usage: python scripts/make_golden.py
"""
from __future__ import annotations

import json
import math
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(ROOT))

import fragserve  # noqa: E402
from fragserve import (AllocConfig, BandwidthTrace, ClientSpec, DeviceProfile, ExecutionPlan, GroupPlan,  # noqa: E402
                       LayerSpec, Level, ModelSpec, Scenario, SimConfig, StagePlan, SyntheticCostModel,
                       load_scenario, plan_to_dict)
from fragserve import simulator as S  # noqa: E402
from fragserve.merging import merge_fragments  # noqa: E402
from fragserve.workload import generate_epoch  # noqa: E402

from paper_2312_10636_b200.serving import ClientView  # noqa: E402

OUT = ROOT / "tests" / "golden" / "serving"


class RecordingSim(S._Sim):
    """_Sim with the dispatch log captured and merged fragments resolvable in _deploy."""

    def __init__(self, *a, merged_fragments=None, **k):
        super().__init__(*a, **k)
        self.dispatch = []
        self.stage_objs = []
        self.epoch_log = []
        self._merged = merged_fragments

    def _push(self, t, rank, payload):
        if rank == S._R_DONE:
            stage, batch = payload
            self.dispatch.append((self._now, self.stage_objs.index(stage), len(batch), [r.seq for r in batch]))
        super()._push(t, rank, payload)

    def _service(self, stage, now):
        self._now = now
        return super()._service(stage, now)

    def _plan_epoch(self, epoch, t_s):
        self._epoch_kind = "keep"
        super()._plan_epoch(epoch, t_s)
        if self._epoch_kind == "keep" and not self.routes:
            self._epoch_kind = "infeasible"
        self.epoch_log.append(self._epoch_deploy if self._epoch_kind == "deploy" else {"kind": self._epoch_kind})

    def _deploy(self, plan, fragments):
        # creation order of _StageRT objects == the executor's deployment stage order
        orig = S._StageRT

        objs = self.stage_objs
        if self._merged is None and getattr(self, "remerge", False):
            # the planner merged fragments (ids 'first+N'): resolve them by re-running the
            # deterministic merge instead of the reference's KeyError
            ids = {f.fragment_id for f in fragments}
            if any(m not in ids for g in plan.groups for lv in g.levels for m in lv.shared.members):
                fragments = merge_fragments(fragments, self.cfg.merge_cfg, self.cost, self.scenario.models,
                                            cap=self.cfg.realign_cfg.instance_cap,
                                            max_share=self.cfg.realign_cfg.max_share)
        self._epoch_kind = "deploy"
        first = len(objs)
        self._epoch_deploy = {"kind": "deploy", "plan": plan_to_dict(plan),
                              "fragments": [frag_doc(f) for f in fragments], "first_stage": first}

        class Tracked(orig):
            def __init__(self, st):
                super().__init__(st)
                objs.append(self)

        S._StageRT = Tracked
        try:
            return super()._deploy(plan, self._merged if self._merged is not None else fragments)
        finally:
            S._StageRT = orig


def latency_tables(plan, cost):
    out = {}
    for gi, g in enumerate(plan.groups):
        for li, lv in enumerate(g.levels):
            for ai, st in enumerate(list(lv.align) + [lv.shared]):
                sid = f"g{gi}.l{li}.align{ai}" if ai < len(lv.align) else f"g{gi}.l{li}.shared"
                if st.is_null:
                    continue
                out[sid] = [0.0] + [cost.latency(st.model_id, st.start, st.end, k, st.alloc.share)
                                    for k in range(1, st.alloc.batch + 1)]
    return out


def frag_doc(f):
    return {"fragment_id": f.fragment_id, "start_layer": f.start_layer, "clients": sorted(f.clients)}


def run_case(name, scenario, cost, planner, cfg, plan=None, fragments=None, merged=None):
    if plan is None:
        wl = generate_epoch(scenario.clients, 0.0, cost)
        fragments = list(wl.fragments)
        plan = S._Sim(scenario, cost, planner, cfg)._run_planner(wl.fragments)
        if merged is not None:
            merged = merge_fragments(wl.fragments, cfg.merge_cfg, cost, scenario.models,
                                     cap=cfg.realign_cfg.instance_cap, max_share=cfg.realign_cfg.max_share)
    sim = RecordingSim(scenario, cost, planner, cfg, fixed_plan=plan, merged_fragments=merged)
    rep = sim.run()
    doc = {
        "name": name,
        "reference": "fragserve " + fragserve.__version__,
        "plan": plan_to_dict(plan),
        "fragments": [frag_doc(f) for f in (merged if merged is not None else fragments)],
        "clients": [ClientView.from_reference(c).to_doc() for c in sorted(scenario.clients, key=lambda c: c.client_id)],
        "latency": latency_tables(plan, cost),
        "horizon_s": cfg.horizon_s, "epoch_s": scenario.epoch_s, "poisson": cfg.poisson, "seed": cfg.seed,
        "expected": {
            "requests": [[c, g, d, dl, s] for c, g, d, dl, s in rep.requests],
            "dispatch": sim.dispatch,
            "summary": {"generated": rep.generated, "completed": rep.completed, "dropped": rep.dropped,
                        "in_flight": rep.in_flight, "p99": rep.latency_p99_ms,
                        "slo_violation_rate": rep.slo_violation_rate},
        },
    }
    OUT.mkdir(parents=True, exist_ok=True)
    (OUT / f"{name}.json").write_text(json.dumps(doc, separators=(",", ":")) + "\n")
    print(f"{name}: generated={rep.generated} completed={rep.completed} dropped={rep.dropped} "
          f"batches={len(sim.dispatch)} stages={len(sim.stage_objs)}")


def closed_form_cases():
    # test_simulator.py:35-56: two-layer model, hand-built fixed plans
    m2 = ModelSpec("m2", 50_000, (LayerSpec(1.0, 2_000), LayerSpec(5.0, 1_000_000)))
    dev = DeviceProfile("dev", {"m2": (0.0, 12.0, 112.0)})
    cost = SyntheticCostModel({"m2": m2}, c0=1.0, c1=0.25, kappa=0.9, batch_max=16)

    def plan(budget, batch, instances=1):
        st = StagePlan("m2", 0, 2, 5.0, budget, AllocConfig(100, batch, instances), ("c0",))
        return ExecutionPlan("fixed", (GroupPlan((Level(0, (), st),)),), 100 * instances)

    for name, rate, budget, batch, inst, hz in (("closed_partial_batch", 5.0, 30.0, 8, 1, 2.0),
                                                  ("closed_full_batch", 50.0, 30.0, 2, 2, 1.0),
                                                  ("closed_inflight_horizon", 5.0, 30.0, 8, 1, 0.035)):
        client = ClientSpec("c0", dev, m2, rate, 100.0, BandwidthTrace((0.0,), (40.0,)))
        sc = Scenario((client,), 1, 10.0, {"m2": m2})
        frags = list(generate_epoch(sc.clients, 0.0, cost).fragments)
        run_case(name, sc, cost, "realign", SimConfig(horizon_s=hz), plan=plan(budget, batch, inst), fragments=frags)


def resnet18_case():
    """BASELINE.json configs[0]: ResNet-18 fragments at 3 partition points, plan from the reference
    CPU planner.  One client per cut p in {2, 4, 6}; each client's device is cheap up to its cut and
    prohibitively slow after it, so the reference's own partition_client (workload.py:145-176) picks
    exactly that cut.  Server latency: the reference's SyntheticCostModel over the unit chain's
    GFLOP weights, with a large per-batch fixed cost (c0) and a small per-request one (c1), at
    300 rps per client: re-alignment pays and plan_realigned (planners.py:81-100) builds ONE level
    at point 6 with alignment stages [2, 6) and [4, 6) feeding a shared [6, 10) suffix, i.e. the
    align -> shared ragged gather the executor must get right.  The golden drives the GPU replay
    test (tests/test_replay_gpu.py)."""
    from fragserve.workload import partition_client

    from paper_2312_10636_b200.models import build_chain

    chain = build_chain("resnet18")
    doc = chain.model_spec_doc()
    spec = ModelSpec(doc["model_id"], doc["input_bytes"],
                     tuple(LayerSpec(l["compute_weight"], l["output_bytes"]) for l in doc["layers"]))
    cost = SyntheticCostModel({spec.model_id: spec}, c0=2.0, c1=0.05, kappa=0.9, batch_max=8)
    n = spec.layer_count
    clients = []
    for j, p in enumerate((2, 4, 6)):
        cum = [0.0]
        for u in range(n):
            cum.append(cum[-1] + (0.2 if u < p else 500.0))
        dev = DeviceProfile(f"dev{j}", {spec.model_id: tuple(cum)})
        c = ClientSpec(f"c{j}", dev, spec, 300.0, 100.0, BandwidthTrace((0.0,), (2000.0 + 100.0 * j,)))
        frag = partition_client(c, 2000.0 + 100.0 * j, cost)
        assert frag is not None and frag.start_layer == p, (j, p, frag)
        clients.append(c)
    sc = Scenario(tuple(clients), 1, 10.0, {spec.model_id: spec})
    run_case("resnet18_3cuts_realign", sc, cost, "realign", SimConfig(horizon_s=0.15))


def realign_model_case(name, model, cuts, horizon_s, seed_rate=300.0, slo=100.0):
    """One client per cut of `cuts` (each client's device cheap up to its cut, prohibitively slow
    after it, so the reference's partition_client picks exactly that cut); the reference's
    SyntheticCostModel over the unit chain's GFLOP weights; the first (c0, c1, kappa) whose
    plan_realigned output re-aligns (>= 1 alignment stage) is recorded.  Covers BASELINE configs
    beyond ResNet: Inception-v3 (concat gather across Mixed blocks) and BERT-base (encoder
    fragments split at layer boundaries)."""
    from fragserve.planners import plan_realigned
    from fragserve.workload import generate_epoch, partition_client

    from paper_2312_10636_b200.models import build_chain

    chain = build_chain(model)
    doc = chain.model_spec_doc()
    spec = ModelSpec(doc["model_id"], doc["input_bytes"],
                     tuple(LayerSpec(l["compute_weight"], l["output_bytes"]) for l in doc["layers"]))
    n = spec.layer_count
    for c0, c1, kappa, rate in ((2.0, 0.05, 0.9, seed_rate), (1.0, 0.05, 0.9, seed_rate), (4.0, 0.05, 0.5, seed_rate),
                                (2.0, 0.2, 0.9, seed_rate), (2.0, 0.05, 0.9, 2 * seed_rate),
                                (1.0, 0.05, 0.5, 2 * seed_rate), (0.5, 0.02, 0.9, seed_rate)):
        cost = SyntheticCostModel({spec.model_id: spec}, c0=c0, c1=c1, kappa=kappa, batch_max=8)
        clients = []
        for j, p in enumerate(cuts):
            cum = [0.0]
            for u in range(n):
                cum.append(cum[-1] + (0.2 if u < p else 500.0))
            dev = DeviceProfile(f"dev{j}", {spec.model_id: tuple(cum)})
            c = ClientSpec(f"c{j}", dev, spec, rate, slo, BandwidthTrace((0.0,), (4000.0 + 100.0 * j,)))
            frag = partition_client(c, 4000.0 + 100.0 * j, cost)
            if frag is None or frag.start_layer != p:
                break
            clients.append(c)
        if len(clients) != len(cuts):
            continue
        try:
            plan = plan_realigned(list(generate_epoch(clients, 0.0, cost).fragments), {spec.model_id: spec}, cost,
                                  gpus=1, capacity=99)
        except fragserve.InfeasibleError:
            continue
        if not any(not a.is_null for g in plan.groups for lv in g.levels for a in lv.align):
            continue
        sc = Scenario(tuple(clients), 1, 10.0, {spec.model_id: spec})
        print(f"{name}: c0={c0} c1={c1} kappa={kappa} rate={rate}")
        run_case(name, sc, cost, "realign", SimConfig(horizon_s=horizon_s))
        return
    raise SystemExit(f"{name}: no parameter set re-aligns")


def vgg16_churn_case():
    """BASELINE.json configs[3rd]: VGG-16 fragment groups under network-trace-driven partition-point
    churn.  Four clients on a steppy bandwidth trace (fast -> slow -> fast, one step per epoch):
    the reference's partition_client moves their cuts each epoch, the simulator re-plans
    (simulator.py:297-349) and deploys a new plan while in-flight requests drain on the old
    stages (drain-old / start-new).  Recorded per epoch: the deployed plan (or keep /
    infeasible), the merged fragments, every stage's latency table in deployment order, and the
    simulator's request records and dispatch log.  Drives test_serving_cpu (virtual clock, bit-
    exact) and tests/test_replay_gpu.py (every batch executed on the B200)."""
    from fragserve.workload import partition_client

    from paper_2312_10636_b200.models import build_chain

    chain = build_chain("vgg16")
    doc = chain.model_spec_doc()
    spec = ModelSpec(doc["model_id"], doc["input_bytes"],
                     tuple(LayerSpec(l["compute_weight"], l["output_bytes"]) for l in doc["layers"]))
    cost = SyntheticCostModel({spec.model_id: spec}, c0=0.5, c1=0.1, kappa=0.9, batch_max=8)
    # handset: the conv blocks run at ~1 ms/GFLOP, the three FC layers (0.4 GB of weights) are
    # memory-bound and slow on the device -> at low bandwidth the argmin cut is after the conv
    # blocks (p = 5, 100 KB payload), at high bandwidth everything is offloaded (p = 0)
    cum = [0.0]
    for u, l in enumerate(spec.layers):
        cum.append(cum[-1] + (1.0 * l.compute_weight if u < 5 else 30.0))
    clients = []
    for j in range(4):
        dev = DeviceProfile(f"phone{j}", {spec.model_id: tuple(cum)})
        hi, lo = 4000.0 + 500.0 * j, 60.0 + 10.0 * j
        trace = BandwidthTrace((0.0, 0.1, 0.2), (hi, lo, hi))
        clients.append(ClientSpec(f"v{j}", dev, spec, 40.0, 110.0, trace))
        p_hi = partition_client(clients[-1], hi, cost).start_layer
        p_lo = partition_client(clients[-1], lo, cost).start_layer
        assert p_hi != p_lo, (j, p_hi, p_lo)
    sc = Scenario(tuple(clients), 1, 0.1, {spec.model_id: spec})
    cfg = SimConfig(horizon_s=0.3)
    sim = RecordingSim(sc, cost, "realign", cfg)
    sim.remerge = True
    rep = sim.run()
    lat = []
    for ep in sim.epoch_log:
        if ep["kind"] != "deploy":
            continue
        for g in ep["plan"]["groups"]:
            for lv in g["levels"]:
                for st in list(lv["align"]) + [lv["shared"]]:
                    if st["instances"]:
                        lat.append([0.0] + [cost.latency(st["model"], st["span"][0], st["span"][1], k, st["share"])
                                            for k in range(1, st["batch"] + 1)])
    assert len(lat) == len(sim.stage_objs), (len(lat), len(sim.stage_objs))
    out = {
        "name": "vgg16_churn_realign", "reference": "fragserve " + fragserve.__version__,
        "epochs": sim.epoch_log,
        "clients": [ClientView.from_reference(c).to_doc() for c in sorted(sc.clients, key=lambda c: c.client_id)],
        "latency_by_stage": lat,
        "horizon_s": cfg.horizon_s, "epoch_s": sc.epoch_s, "poisson": cfg.poisson, "seed": cfg.seed,
        "expected": {
            "requests": [[c, g, d, dl, st] for c, g, d, dl, st in rep.requests],
            "dispatch": sim.dispatch,
            "summary": {"generated": rep.generated, "completed": rep.completed, "dropped": rep.dropped,
                        "in_flight": rep.in_flight, "p99": rep.latency_p99_ms},
        },
    }
    (OUT.parent / "churn").mkdir(parents=True, exist_ok=True)
    (OUT.parent / "churn" / "vgg16_churn_realign.json").write_text(json.dumps(out, separators=(",", ":")) + "\n")
    kinds = [e["kind"] for e in sim.epoch_log]
    print(f"vgg16_churn_realign: epochs={kinds} generated={rep.generated} completed={rep.completed} "
          f"dropped={rep.dropped} batches={len(sim.dispatch)} stages={len(sim.stage_objs)}")


def main():
    realign_model_case("inception_v3_3cuts_realign", "inception_v3", (7, 10, 15), 0.1)
    realign_model_case("bert_base_3cuts_realign", "bert_base", (3, 6, 9), 0.1)
    vgg16_churn_case()
    resnet18_case()
    closed_form_cases()
    scen = REF / "scenarios"
    sc, cost = load_scenario(scen / "slo-guarantee" / "scenario.json")
    run_case("slo_guarantee_realign", sc, cost, "realign", SimConfig(horizon_s=10.0))
    run_case("slo_guarantee_independent_poisson", sc, cost, "independent",
             SimConfig(horizon_s=6.0, seed=3, poisson=True))
    sc, cost = load_scenario(scen / "shared-suffix" / "scenario.json")
    run_case("shared_suffix_realign", sc, cost, "realign", SimConfig(horizon_s=5.0))
    sc, cost = load_scenario(scen / "demo" / "scenario.json")
    run_case("demo_realign", sc, cost, "realign", SimConfig(horizon_s=65.0))
    sc, cost = load_scenario(scen / "merge-fleet" / "scenario.json")
    # merging fires here: the reference's own _deploy raises KeyError; the recording
    # sim deploys the merged fragments instead (the documented fix the executor applies too)
    run_case("merge_fleet_realign_fixed_deploy", sc, cost, "realign", SimConfig(horizon_s=2.0), merged=True)
    run_case("merge_fleet_realign_poisson", sc, cost, "realign", SimConfig(horizon_s=2.0, poisson=True, seed=1),
             merged=True)


if __name__ == "__main__":
    main()
