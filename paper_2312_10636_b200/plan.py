"""Plan ingestion: the reference's plan types / plan JSON -> an executable deployment.

Input is either a fragserve `ExecutionPlan` (realign.py:50-103, duck-typed: no import of the
reference is needed) or the plan JSON document `fragserve plan` writes (plan_to_dict,
simulator.py:186-219, plus the cmd_plan header cli.py:121-123).  Output mirrors
_Sim._deploy (simulator.py:275-295): one runtime stage per align StagePlan and per level's shared
StagePlan, and per client a route (entry point, stage list, worst-case remaining time).

Deviation, documented: the reference's _deploy looks merged fragment ids ('u0n4+1',
merging.py:52) up in a table built from the *unmerged* fragments and raises KeyError whenever
merging fires.  Here the caller passes the fragments the planner actually planned
(the merged ones, whose `clients` sets hold every absorbed client, merging.py:44-56), so every
plan member resolves.
"""
from __future__ import annotations

import json
from dataclasses import dataclass, field
from pathlib import Path

from .errors import ValidationError


@dataclass(frozen=True)
class StageSpec:
    """One planned stage (StagePlan + its placement)."""

    stage_id: str
    model_id: str
    start: int
    end: int
    share: int
    batch: int
    instances: int
    budget_ms: float
    members: tuple[str, ...]
    gpus: tuple[int, ...] | None = None

    @property
    def is_null(self) -> bool:
        return self.start == self.end


@dataclass(frozen=True)
class RouteSpec:
    """_Route (simulator.py:103-107): entry point, stage indices, worst-case remaining ms."""

    point: int
    stages: tuple[int, ...]
    worst_rem_ms: float


@dataclass
class Deployment:
    planner: str
    stages: list[StageSpec] = field(default_factory=list)
    routes: dict[str, RouteSpec] = field(default_factory=dict)
    total_resource: int | None = None

    def stage_index(self, stage_id: str) -> int:
        for i, s in enumerate(self.stages):
            if s.stage_id == stage_id:
                return i
        raise KeyError(stage_id)


def _stage_from_obj(sid: str, st, placement) -> StageSpec:
    gpus = None
    if placement is not None and sid in placement:
        gpus = tuple(int(g) for g in placement[sid])
    return StageSpec(sid, st.model_id, int(st.start), int(st.end), int(st.alloc.share), int(st.alloc.batch),
                     int(st.alloc.instances), float(st.budget_ms), tuple(st.members), gpus)


def _stage_from_doc(d: dict) -> StageSpec:
    gpus = tuple(int(g) for g in d["gpu"]) if d.get("gpu") is not None else None
    return StageSpec(d["stage_id"], d["model"], int(d["span"][0]), int(d["span"][1]), int(d["share"]),
                     int(d["batch"]), int(d["instances"]), float(d["budget_ms"]), tuple(d["members"]), gpus)


def _levels(plan):
    """Yield (group index, level index, point, [align StageSpec], shared StageSpec)."""
    if isinstance(plan, dict):
        for gi, g in enumerate(plan["groups"]):
            for li, lv in enumerate(g["levels"]):
                yield gi, li, int(lv["point"]), [_stage_from_doc(a) for a in lv["align"]], _stage_from_doc(lv["shared"])
        return
    placement = getattr(plan, "placement", None)
    for gi, g in enumerate(plan.groups):
        for li, lv in enumerate(g.levels):
            align = [_stage_from_obj(f"g{gi}.l{li}.align{ai}", st, placement) for ai, st in enumerate(lv.align)]
            yield gi, li, int(lv.point), align, _stage_from_obj(f"g{gi}.l{li}.shared", lv.shared, placement)


def deploy(plan, fragments) -> Deployment:
    """Deploy a plan: mirrors _Sim._deploy (simulator.py:275-295).

    `fragments`: iterable of objects with fragment_id / start_layer / clients (fragserve
    Fragment, workload.py:120-138), or dicts with those keys.  Merged fragments must be included
    (see module docstring).
    """
    table = {}
    for f in fragments:
        if isinstance(f, dict):
            table[f["fragment_id"]] = (int(f["start_layer"]), frozenset(f["clients"]))
        else:
            table[f.fragment_id] = (int(f.start_layer), frozenset(f.clients))
    planner = plan["planner"] if isinstance(plan, dict) else plan.planner
    total = plan.get("total_resource") if isinstance(plan, dict) else plan.total_resource
    dep = Deployment(planner=planner, total_resource=total)
    for _gi, _li, _point, align, shared in _levels(plan):
        shared_idx = None
        if not shared.is_null:
            dep.stages.append(shared)
            shared_idx = len(dep.stages) - 1
        align_by_frag = {st.members[0]: st for st in align}
        for fid in shared.members:
            if fid not in table:
                raise ValidationError(f"plan member {fid!r} is not a known fragment; pass the merged fragments")
            start_layer, clients = table[fid]
            st = align_by_frag.get(fid)
            stages = []
            d_align = 0.0
            if st is not None and not st.is_null:
                dep.stages.append(st)
                stages.append(len(dep.stages) - 1)
                d_align = st.budget_ms
            if shared_idx is not None:
                stages.append(shared_idx)
            worst = 2.0 * (d_align + (shared.budget_ms if shared_idx is not None else 0.0))
            for cid in sorted(clients):
                dep.routes[cid] = RouteSpec(start_layer, tuple(stages), worst)
    return dep


def load_plan_json(path) -> dict:
    doc = json.loads(Path(path).read_text())
    if "groups" not in doc:
        raise ValidationError(f"{path}: not a plan document")
    return doc


def deploy_epochs(epoch_docs) -> list:
    """Plan transitions under churn (_Sim._plan_epoch, simulator.py:297-349): one entry per epoch,
    each {"kind": "deploy", "plan": plan JSON, "fragments": [...]} (a new plan is deployed at that
    epoch's REPLAN), {"kind": "keep"} (cut points unchanged: the previous plan stays) or
    {"kind": "infeasible"} (no routes).  Returns the `epochs` list `serving.serve` takes; stages of
    earlier deployments stay alive so in-flight requests drain on them."""
    out = []
    for e in epoch_docs:
        kind = e["kind"]
        if kind == "deploy":
            out.append(deploy(e["plan"], e["fragments"]))
        elif kind == "keep":
            out.append(None)
        elif kind == "infeasible":
            out.append("infeasible")
        else:
            raise ValidationError(f"unknown epoch kind {kind!r}")
    return out
