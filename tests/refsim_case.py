"""The reference-side scenario of the resnet18_3cuts_realign golden, rebuilt with fragserve's own
classes (as scripts/make_golden.py builds it), for the Seam 2 tests (paper_2312_10636_b200/refsim.py).
fragserve comes from baseline/_ref (the pip --target install that travels to the GPU box) or the
reference source tree."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def fragserve_available() -> bool:
    for p in (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")):
        if (p / "fragserve" / "__init__.py").exists():
            if str(p) not in sys.path:
                sys.path.insert(0, str(p))
            return True
    return False


def resnet18_case(chain):
    import fragserve
    from fragserve import (BandwidthTrace, ClientSpec, DeviceProfile, LayerSpec, ModelSpec, Scenario, SimConfig,
                           SyntheticCostModel)
    from fragserve import simulator as S
    from fragserve.workload import generate_epoch

    doc = chain.model_spec_doc()
    spec = ModelSpec(doc["model_id"], doc["input_bytes"],
                     tuple(LayerSpec(x["compute_weight"], x["output_bytes"]) for x in doc["layers"]))
    cost = SyntheticCostModel({spec.model_id: spec}, c0=2.0, c1=0.05, kappa=0.9, batch_max=8)
    n = spec.layer_count
    clients = []
    for j, p in enumerate((2, 4, 6)):
        cum = [0.0]
        for u in range(n):
            cum.append(cum[-1] + (0.2 if u < p else 500.0))
        dev = DeviceProfile(f"dev{j}", {spec.model_id: tuple(cum)})
        clients.append(ClientSpec(f"c{j}", dev, spec, 300.0, 100.0, BandwidthTrace((0.0,), (2000.0 + 100.0 * j,))))
    sc = Scenario(tuple(clients), 1, 10.0, {spec.model_id: spec})
    cfg = SimConfig(horizon_s=0.15)
    wl = generate_epoch(sc.clients, 0.0, cost)
    plan = S._Sim(sc, cost, "realign", cfg)._run_planner(wl.fragments)
    return fragserve, S, sc, cost, cfg, plan
