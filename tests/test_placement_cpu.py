"""Placement-faithful routing without a GPU (placement.py:24-70).

A plan whose stages are placed across two GPUs — an alignment stage [1, 2) on GPU 1 feeding a
shared suffix [2, 18) with one instance on each GPU — served on the virtual clock with the
placement handed to the native loop.  Checked: (1) placement never changes the reference's
timing: the records equal the oracle restatement's (oracle/serving.py); (2) every batch runs on an
instance of its own stage, on the GPU the placement gives that instance; (3) the same-GPU
preference: a batch goes to the GPU holding most of its requests' activations (alignment outputs
on GPU 1, direct arrivals at their first-stage instance-0 GPU 0) unless that GPU's instance is busy.
"""
from oracle.serving import simulate_fixed
from paper_2312_10636_b200.plan import deploy
from paper_2312_10636_b200.serving import ClientView, serve

N_UNITS = 18


def _stage(sid, span, share, batch, instances, members, gpus, budget):
    return {"stage_id": sid, "model": "resnet50", "span": list(span), "demand_rps": 0.0, "budget_ms": budget,
            "share": share, "batch": batch, "instances": instances, "members": members, "gpu": gpus}


def _case():
    plan = {"planner": "realign", "total_resource": 22, "groups": [{"levels": [{
        "point": 2,
        "align": [_stage("g0.l0.align0", (1, 2), 2, 4, 1, ["fa"], [1], 3.0),
                  _stage("g0.l0.align1", (2, 2), 0, 0, 0, ["fd"], None, 0.0)],
        "shared": _stage("g0.l0.shared", (2, N_UNITS), 10, 8, 2, ["fa", "fd"], [0, 1], 6.0)}]}]}
    frags = [{"fragment_id": "fa", "start_layer": 1, "clients": [f"a{i}" for i in range(10)]},
             {"fragment_id": "fd", "start_layer": 2, "clients": [f"d{i}" for i in range(10)]}]
    clients = [ClientView(cid, 40.0 + 3 * i, 200.0, (0.0,), (1000.0,), tuple(0.5 * p for p in range(N_UNITS + 1)),
                          tuple(1000 for _ in range(N_UNITS + 1)))
               for i, cid in enumerate([f"a{i}" for i in range(10)] + [f"d{i}" for i in range(10)])]
    return deploy(plan, frags), clients


def _lat(st, k):
    return (0.4 + 0.05 * k) if st.end == 2 else (2.5 + 0.3 * k)


def test_placed_plan_routes_by_placement_and_prefers_the_activations_gpu():
    dep, clients = _case()
    assert [s.gpus for s in dep.stages] == [(0, 1), (1,)]
    rep = serve(dep, clients, 2.0, latency=_lat, record_dispatch=True)
    recs, _ = simulate_fixed(dep, clients, 2.0, 0.0, _lat)
    assert [tuple(r) for r in rep.requests] == [tuple(r) for r in recs]
    busy = {}  # (stage, instance) -> [(t0, t1)]
    remote = preferred = 0
    shared = dep.stage_index("g0.l0.shared")
    align = dep.stage_index("g0.l0.align0")
    from_align = set()
    for (t, si, k, seqs), (inst, gpu) in zip(rep.dispatch, rep.placement):
        st = dep.stages[si]
        assert 0 <= inst < st.instances and gpu == st.gpus[inst]
        if si == align:
            from_align.update(seqs)
        else:
            on1 = sum(1 for q in seqs if q in from_align)
            major = 1 if on1 * 2 > k else 0 if on1 * 2 < k else None
            if major is not None and gpu != major:
                other = st.gpus.index(major)
                assert any(t0 <= t < t1 - 1e-9 for t0, t1 in busy.get((si, other), [])), (t, seqs)
                remote += 1
            elif major is not None:
                preferred += 1
        busy.setdefault((si, inst), []).append((t, t + _lat(st, k)))
    assert preferred > remote > 0  # both happen at this load; busy-forced remote gathers are the minority
