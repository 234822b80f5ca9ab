"""Serving parity without a GPU: the executor's native event loop (virtual clock) and the oracle
restatement vs golden logs of the unmodified reference simulator (scripts/make_golden.py).

Bit-exact: every request record (client, gen_ms, done_ms, deadline_ms, status) and every
dispatched batch (time, stage, k, request seqs in FIFO order)."""
import json

import pytest

from conftest import GOLDEN
from paper_2312_10636_b200.plan import deploy
from paper_2312_10636_b200.serving import ClientView, serve

CASES = sorted(p.stem for p in (GOLDEN / "serving").glob("*.json"))


def _load(name):
    doc = json.loads((GOLDEN / "serving" / f"{name}.json").read_text())
    dep = deploy(doc["plan"], doc["fragments"])
    clients = [ClientView.from_doc(c) for c in doc["clients"]]
    lat = doc["latency"]
    return doc, dep, clients, (lambda st, k: lat[st.stage_id][k])


def _expected_dispatch(doc):
    return [(t, s, k, tuple(seqs)) for t, s, k, seqs in doc["expected"]["dispatch"]]


@pytest.mark.parametrize("name", CASES)
def test_native_loop_matches_reference(name):
    doc, dep, clients, latency = _load(name)
    rep = serve(dep, clients, doc["horizon_s"], epoch_s=doc["epoch_s"], latency=latency, poisson=doc["poisson"],
                seed=doc["seed"], record_dispatch=True)
    exp = doc["expected"]
    got = [list(r) for r in rep.requests]
    assert len(got) == len(exp["requests"])
    assert got == exp["requests"]
    assert rep.dispatch == _expected_dispatch(doc)
    s = exp["summary"]
    assert (rep.generated, rep.completed, rep.dropped, rep.in_flight) == (s["generated"], s["completed"],
                                                                          s["dropped"], s["in_flight"])
    assert rep.latency_p99_ms == s["p99"]


@pytest.mark.parametrize("name", CASES)
def test_oracle_restatement_matches_reference(name):
    from oracle.serving import simulate_fixed
    doc, dep, clients, latency = _load(name)
    recs, dispatch = simulate_fixed(dep, clients, doc["horizon_s"], doc["epoch_s"], latency, doc["poisson"],
                                    doc["seed"])
    assert [list(r) for r in recs] == doc["expected"]["requests"]
    assert dispatch == _expected_dispatch(doc)


def test_closed_form_partial_batch_latency():
    # test_simulator.py:155-169: 10 ms uplink + 30 ms batching wait + 6.0 ms service
    doc, dep, clients, latency = _load("closed_partial_batch")
    rep = serve(dep, clients, doc["horizon_s"], epoch_s=doc["epoch_s"], latency=latency)
    assert rep.generated == rep.completed == 10
    for _c, gen, done, _dl, status in rep.requests:
        assert status == "completed"
        assert done - gen == pytest.approx(46.0, abs=1e-9)


def test_closed_form_full_batch_latency():
    doc, dep, clients, latency = _load("closed_full_batch")
    rep = serve(dep, clients, doc["horizon_s"], epoch_s=doc["epoch_s"], latency=latency)
    lat2 = 6.0 * 1.25
    for i, (_c, gen, done, _dl, status) in enumerate(rep.requests):
        assert done - gen == pytest.approx((30.0 if i % 2 == 0 else 10.0) + lat2, abs=1e-9)


def test_inflight_at_horizon_csv_row():
    doc, dep, clients, latency = _load("closed_inflight_horizon")
    rep = serve(dep, clients, doc["horizon_s"], epoch_s=doc["epoch_s"], latency=latency)
    assert rep.in_flight == 1
    row = rep.requests_csv().splitlines()[1]
    assert row.startswith("c0,0.000000,,,") and row.endswith("inflight")


def test_churn_plan_transitions_match_reference():
    """VGG-16 under partition-point churn (BASELINE configs: network-trace-driven churn): three
    epochs, each deploying a new reference plan at its REPLAN (cuts 0 -> 5 -> 0); requests in flight
    drain on the stages they were routed to.  Records and dispatch log bit-exact."""
    from paper_2312_10636_b200.plan import deploy_epochs

    doc = json.loads((GOLDEN / "churn" / "vgg16_churn_realign.json").read_text())
    epochs = deploy_epochs(doc["epochs"])
    assert sum(1 for e in epochs if e is not None and not isinstance(e, str)) == 3
    stages = [s for e in epochs if e is not None and not isinstance(e, str) for s in e.stages]
    table = {id(s): doc["latency_by_stage"][i] for i, s in enumerate(stages)}
    clients = [ClientView.from_doc(c) for c in doc["clients"]]
    rep = serve(None, clients, doc["horizon_s"], epoch_s=doc["epoch_s"], latency=lambda st, k: table[id(st)][k],
                record_dispatch=True, epochs=epochs)
    exp = doc["expected"]
    assert [list(r) for r in rep.requests] == exp["requests"]
    assert rep.dispatch == [(t, s, k, tuple(q)) for t, s, k, q in exp["dispatch"]]
    assert {s for _t, s, _k, _q in rep.dispatch} == {0, 1, 2}  # every epoch's stage served batches


def test_empty_fleet_and_zero_horizon():
    """Edge cases of the event loop: no clients, and a horizon shorter than the first arrival."""
    doc, dep, clients, latency = _load("closed_partial_batch")
    rep = serve(dep, [], 1.0, latency=latency)
    assert (rep.generated, rep.completed, rep.dropped) == (0, 0, 0)
    assert rep.latency_p99_ms is None and rep.requests_csv().count("\n") == 1
    rep = serve(dep, clients, 0.0, latency=latency)
    assert rep.completed == 0
