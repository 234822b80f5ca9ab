"""N>1 path without a GPU: two ranks (gloo, 127.0.0.1) each serve an independent fleet with the
native loop (virtual clock), exactly like bench.py's weak-scaling replicas, and the metric is
aggregated with an all-reduce of counts (sum) and timings (max).  Groups share no tensors, so
there is no data-path collective to test."""
import json
import os
import socket

import pytest
import torch.multiprocessing as mp

from conftest import GOLDEN


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank(rank, world, port, name, out):
    import torch
    import torch.distributed as dist

    from paper_2312_10636_b200.plan import deploy
    from paper_2312_10636_b200.serving import ClientView, serve

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    doc = json.loads((GOLDEN / "serving" / f"{name}.json").read_text())
    dep = deploy(doc["plan"], doc["fragments"])
    clients = [ClientView.from_doc(c) for c in doc["clients"]]
    lat = doc["latency"]
    rep = serve(dep, clients, doc["horizon_s"], epoch_s=doc["epoch_s"], latency=lambda st, k: lat[st.stage_id][k],
                poisson=True, seed=rank)  # a different arrival draw per replica
    counts = torch.tensor([float(rep.slo_met), float(rep.generated)], dtype=torch.float64)
    worst = torch.tensor([rep.latency_p99_ms or 0.0], dtype=torch.float64)
    mine = counts.clone()
    dist.all_reduce(counts)
    dist.all_reduce(worst, op=dist.ReduceOp.MAX)
    out[rank] = (mine.tolist(), counts.tolist(), worst.item(), rep.latency_p99_ms)
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_weak_scaling_aggregation():
    world = 2
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_rank, args=(world, port, "slo_guarantee_realign", out), nprocs=world, join=True)
        res = dict(out)
    per_rank = [res[r][0] for r in range(world)]
    total = res[0][1]
    assert total == res[1][1]  # every rank sees the same aggregate
    assert total[0] == sum(p[0] for p in per_rank) and total[1] == sum(p[1] for p in per_rank)
    assert res[0][2] == max(res[r][3] for r in range(world))
    assert per_rank[0][1] > 0 and per_rank[1][1] > 0
