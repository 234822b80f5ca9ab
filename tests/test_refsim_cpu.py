"""Seam 2 without a GPU: the reference's own _Sim drives the executor hook (refsim.B200Sim).

With the execution stubbed (no device here), the subclass must leave the reference's behaviour
untouched — request records identical to the golden the unmodified simulator produced
(tests/golden/serving/resnet18_3cuts_realign.json) — and hand the executor exactly the batches the
reference dispatched, in order (the dispatch log's k and request seqs)."""
import json

import pytest

from conftest import GOLDEN
from refsim_case import fragserve_available, resnet18_case

pytestmark = pytest.mark.skipif(not fragserve_available(), reason="fragserve (baseline/_ref or /root/reference) absent")


def test_b200sim_hook_sees_the_reference_dispatch():
    from paper_2312_10636_b200.models import build_chain
    from paper_2312_10636_b200.refsim import b200_sim_class

    fragserve, S, sc, cost, cfg, plan = resnet18_case(build_chain("resnet18"))
    golden = json.loads((GOLDEN / "serving" / "resnet18_3cuts_realign.json").read_text())
    assert fragserve.plan_to_dict(plan) == golden["plan"]

    class Stubbed(b200_sim_class(S)):
        def _execute(self, stage, batch):
            self.batches.append(((stage.start, stage.end), len(batch), tuple(r.seq for r in batch), 0.0))
            return 0.0

    sim = Stubbed(sc, cost, "realign", cfg, fixed_plan=plan, pool=None, ingress=None)
    rep = sim.run()
    assert [list(r) for r in rep.requests] == golden["expected"]["requests"]
    assert [(k, seqs) for _span, k, seqs, _ms in sim.batches] == [(k, tuple(q)) for _t, _s, k, q in
                                                                   golden["expected"]["dispatch"]]
    spans = {span for span, *_ in sim.batches}
    assert {(2, 6), (4, 6), (6, 10)} <= spans  # alignment stages and the shared suffix all ran
