"""Seam 2 on the B200: the reference's own simulator (fragserve, from baseline/_ref) executing every
dispatched batch on the executor through refsim.B200Sim.

Replay (measured=False): the reference's records stay bit-identical to the golden, and every
completed request's output is the real ResNet-18 forward of its client's input (fp32 oracle,
<= 2e-2, same top-1 where decisive), alignment outputs flowing into the shared stage.
Measured (measured=True): completion times come from CUDA-event timings of the real batches; every
admitted request completes and its latency is the reference's arrival time plus measured GPU time.
"""
import json

import pytest
import torch

from conftest import GOLDEN
from refsim_case import fragserve_available, resnet18_case

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not fragserve_available(), reason="fragserve (baseline/_ref) absent")]


def _run(measured):
    from oracle.units import nchw_to_nhwc, run_span, units_for
    from paper_2312_10636_b200.device import context
    from paper_2312_10636_b200.engine import DeviceModel
    from paper_2312_10636_b200.models import build_chain, torch_model
    from paper_2312_10636_b200.refsim import StagePool, b200_sim_class

    m = torch_model("resnet18")
    chain = build_chain("resnet18", module=m)
    units = units_for("resnet18", m)
    fragserve, S, sc, cost, cfg, plan = resnet18_case(chain)
    pool = StagePool({"resnet18": DeviceModel(chain)}, context(0))
    images, acts, expected = {}, {}, {}
    for j, c in enumerate(sorted(sc.clients, key=lambda c: c.client_id)):
        images[c.client_id] = torch.randn(1, 3, 224, 224, generator=torch.Generator().manual_seed(500 + j))
        expected[c.client_id] = run_span(units, 0, chain.n_units, images[c.client_id])[0]

    def ingress(cid, point):
        key = (cid, point)
        if key not in acts:
            acts[key] = nchw_to_nhwc(run_span(units, 0, point, images[cid]))[0].contiguous().cuda()
        return acts[key]

    sim = b200_sim_class(S)(sc, cost, "realign", cfg, fixed_plan=plan, pool=pool, ingress=ingress, measured=measured)
    rep = sim.run()
    return sim, rep, expected


def test_reference_simulator_replays_on_the_executor():
    sim, rep, expected = _run(measured=False)
    golden = json.loads((GOLDEN / "serving" / "resnet18_3cuts_realign.json").read_text())
    assert [list(r) for r in rep.requests] == golden["expected"]["requests"]
    recs = sim.records
    done = 0
    for r in recs:
        if r.status != "completed":
            continue
        got, ref = sim.outputs[r.seq].reshape(-1), expected[r.client_id]
        assert ((got - ref).norm() / ref.norm()).item() < 2e-2
        top2 = ref.topk(2).values
        if (top2[0] - top2[1]) > 0.02 * (ref.max() - ref.min()):
            assert int(got.argmax()) == int(ref.argmax())
        done += 1
    assert done == golden["expected"]["summary"]["completed"] > 20
    assert {span for span, *_ in sim.batches} >= {(2, 6), (4, 6), (6, 10)}


def test_reference_simulator_priced_by_measured_execution():
    sim, rep, _ = _run(measured=True)
    assert rep.completed > 20 and rep.generated == rep.completed + rep.dropped + rep.in_flight
    # every batch was timed on the device; latencies now reflect B200 execution, not the cost table
    assert all(ms > 0 for *_x, ms in sim.batches)
    assert rep.latency_p99_ms is not None and rep.latency_p99_ms < 100.0
