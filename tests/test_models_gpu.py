"""End-to-end unit-chain parity on the B200: libgx spans vs the fp32 CPU oracle.

Tolerance (north star): bf16 path within 2e-2 relative (L2 norm per request) of the fp32
forward, identical top-1 on inputs whose fp32 top-1 margin is decisive (> 2% of the logit
range; random-init networks produce near-ties that no bf16 path can be held to).
"""
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle.units import nchw_to_nhwc, run_span, units_for
from paper_2312_10636_b200 import _native as N
from paper_2312_10636_b200.models import build_chain, torch_model

RES = {"resnet18": 224, "resnet50": 224, "vgg16": 224, "inception_v3": 299}
_cache = {}


def _setup(name):
    if name not in _cache:
        from paper_2312_10636_b200.engine import DeviceModel
        m = torch_model(name)
        chain = build_chain(name, module=m)
        _cache[name] = (m, chain, DeviceModel(chain))
    return _cache[name]


def _inputs(x):
    return [nchw_to_nhwc(x[i:i + 1])[0].contiguous().cuda() for i in range(x.shape[0])]


def _check(got, ref, tol=2e-2):
    for i in range(ref.shape[0]):
        rel = ((got[i] - ref[i]).norm() / ref[i].norm()).item()
        assert rel < tol, (i, rel)
        top2 = ref[i].topk(2).values
        if (top2[0] - top2[1]) > 0.02 * (ref[i].max() - ref[i].min()):
            assert got[i].argmax() == ref[i].argmax(), i


@pytest.mark.parametrize("name", ["resnet18", "resnet50", "vgg16"])
def test_full_span_matches_fp32_oracle(name):
    from paper_2312_10636_b200.engine import StageInstance
    m, chain, dm = _setup(name)
    k = 4
    x = torch.randn(k, 3, RES[name], RES[name], generator=torch.Generator().manual_seed(1234))
    ref = run_span(units_for(name, m), 0, chain.n_units, x)
    st = StageInstance(dm, 0, chain.n_units, max_batch=8, sm_budget=148)
    got = torch.stack(st.run(_inputs(x), src_channels=3)).cpu().view(k, -1)
    _check(got, ref)


def test_client_cut_entry_activations_resnet50():
    """Requests entering at different boundaries (client ran the prefix in fp32)."""
    from paper_2312_10636_b200.engine import StageInstance
    m, chain, dm = _setup("resnet50")
    units = units_for("resnet50", m)
    x = torch.randn(3, 3, 224, 224, generator=torch.Generator().manual_seed(7))
    ref = run_span(units, 0, chain.n_units, x)
    for p in (1, 5, 9, 15, 17):
        act = run_span(units, 0, p, x)
        st = StageInstance(dm, p, chain.n_units, max_batch=4, sm_budget=60)
        got = torch.stack(st.run(_inputs(act))).cpu().view(3, -1)
        _check(got, ref)


def test_realignment_split_is_bit_exact():
    """[0,p) then [p,N) through the bf16 hand-off equals the single span bit for bit."""
    from paper_2312_10636_b200.engine import StageInstance
    m, chain, dm = _setup("resnet50")
    x = torch.randn(5, 3, 224, 224, generator=torch.Generator().manual_seed(3))
    inp = _inputs(x)
    full = StageInstance(dm, 0, 18, max_batch=8, sm_budget=148).run(inp, src_channels=3)
    for p, budgets in ((2, (30, 100)), (9, (148, 17)), (15, (8, 8))):
        a = StageInstance(dm, 0, p, max_batch=8, sm_budget=budgets[0])
        b = StageInstance(dm, p, 18, max_batch=8, sm_budget=budgets[1])
        mid = a.run(inp, src_channels=3)
        out = b.run(mid[:3]) + b.run(mid[3:])  # different batch compositions downstream
        for i in range(5):
            assert torch.equal(out[i], full[i]), (p, i)


@pytest.mark.parametrize("name", ["resnet50", "inception_v3", "vgg16"])
def test_every_unit_matches_fp32_oracle(name):
    """Each unit on the oracle's fp32 entry activation: strict 2e-2 per unit."""
    from paper_2312_10636_b200.engine import StageInstance
    m, chain, dm = _setup(name)
    units = units_for(name, m)
    x = torch.randn(2, 3, RES[name], RES[name], generator=torch.Generator().manual_seed(11))
    acts = [x]
    for u in range(chain.n_units):
        acts.append(run_span(units, u, u + 1, acts[-1]))
    for u in range(chain.n_units):
        st = StageInstance(dm, u, u + 1, max_batch=2, sm_budget=148)
        got = torch.stack(st.run(_inputs(acts[u]), out_dtype=torch.float32, src_channels=3 if u == 0 else 0)).cpu()
        ref = nchw_to_nhwc(acts[u + 1]).reshape(2, -1)
        rel = ((got.view(2, -1) - ref).norm() / ref.norm()).item()
        assert rel < 2e-2, (u, rel)


def test_inception_end_to_end_within_framework_bf16_error():
    """Random-init Inception-v3 amplifies bf16 rounding ~20x end to end (PyTorch's own bf16
    forward is ~20% off its fp32 forward on these weights): hold the executor to no worse than
    1.25x the framework's bf16 error, and identical top-1 on decisive inputs."""
    from paper_2312_10636_b200.engine import StageInstance
    m, chain, dm = _setup("inception_v3")
    x = torch.randn(2, 3, 299, 299, generator=torch.Generator().manual_seed(1234))
    ref = run_span(units_for("inception_v3", m), 0, chain.n_units, x)
    import copy
    with torch.no_grad():
        fb = copy.deepcopy(m).to(torch.bfloat16)(x.to(torch.bfloat16)).float()
    st = StageInstance(dm, 0, chain.n_units, max_batch=2, sm_budget=148)
    got = torch.stack(st.run(_inputs(x), src_channels=3)).cpu().view(2, -1)
    for i in range(2):
        fw = ((fb[i] - ref[i]).norm() / ref[i].norm()).item()
        rel = ((got[i] - ref[i]).norm() / ref[i].norm()).item()
        assert rel <= max(2e-2, 1.25 * fw), (i, rel, fw)
    _check(got, ref, tol=1.0)


@pytest.mark.parametrize("budget", [4, 148])
def test_span_kernel_matches_per_op_path(budget):
    """The single-launch persistent span kernel (gx_stage_set_exec(GX_EXEC_SPAN)) and the per-op
    graph path compute the same span.  The per-op path sums the wide 3x3 convs in halo order and
    adds the expand convs' residual inside the MMA, so the two agree to bf16 rounding, and both
    agree with the fp32 oracle."""
    from paper_2312_10636_b200.engine import DeviceModel, StageInstance
    m, _chain, _dm = _setup("resnet50")
    chain = build_chain("resnet50", module=m, fuse_downsample=False)  # the span kernel takes unfused ops
    dm = DeviceModel(chain)
    x = torch.randn(3, 3, 224, 224, generator=torch.Generator().manual_seed(5))
    inp = _inputs(x)
    ref = StageInstance(dm, 0, chain.n_units, max_batch=4, sm_budget=budget).run(inp, src_channels=3)
    got = StageInstance(dm, 0, chain.n_units, max_batch=4, sm_budget=budget,
                        exec_mode=N.GX_EXEC_SPAN).run(inp, src_channels=3)
    oracle = run_span(units_for("resnet50", m), 0, chain.n_units, x)
    for i, (a, b) in enumerate(zip(got, ref)):
        rel = ((a - b).norm() / b.norm()).item()
        assert rel < 1e-2, rel
        for t in (a, b):
            o = oracle[i].reshape(-1)
            assert ((t.cpu() - o).norm() / o.norm()).item() < 2e-2


def test_bert_full_span_matches_fp32_oracle():
    """configs[4]: the embeddings (K8) and 12 encoder layers from the requests' token ids."""
    from oracle.units import bert_token_ids
    from paper_2312_10636_b200.engine import StageInstance
    m, chain, dm = _setup("bert_base")
    k = 3
    x = bert_token_ids(k, 5)
    ref = run_span(units_for("bert_base", m), 0, chain.n_units, x)
    st = StageInstance(dm, 0, chain.n_units, max_batch=4, sm_budget=148)
    got = torch.stack(st.run([x[i].contiguous().cuda() for i in range(k)])).cpu().view(k, 128, 768)
    for i in range(k):
        rel = ((got[i] - ref[i]).norm() / ref[i].norm()).item()
        assert rel < 2e-2, (i, rel)


def test_bert_split_is_bit_exact():
    from paper_2312_10636_b200.engine import StageInstance
    from oracle.units import bert_token_ids
    m, chain, dm = _setup("bert_base")
    x = bert_token_ids(4, 6)
    inp = [x[i].contiguous().cuda() for i in range(4)]
    full = StageInstance(dm, 0, 12, max_batch=4, sm_budget=148).run(inp)
    a = StageInstance(dm, 0, 5, max_batch=4, sm_budget=37)
    b = StageInstance(dm, 5, 12, max_batch=4, sm_budget=100)
    mid = a.run(inp)
    out = b.run(mid[:1]) + b.run(mid[1:])
    for i in range(4):
        assert torch.equal(out[i], full[i]), i


def test_bert_embedding_unit_from_token_ids():
    """K8 alone: unit 0's embedding op vs transformers' BertEmbeddings on the same ids, and a
    fragment entering at boundary 1 (hidden state) after one that entered at 0 (token ids)."""
    from oracle.units import bert_token_ids
    from paper_2312_10636_b200.engine import StageInstance
    m, chain, dm = _setup("bert_base")
    ids = bert_token_ids(2, 9)
    ids[0, :4] = torch.tensor([0, 30521, 101, 102], dtype=torch.int32)  # table edges
    units = units_for("bert_base", m)
    ref1 = run_span(units, 0, 1, ids)
    st = StageInstance(dm, 0, 1, max_batch=2, sm_budget=8)
    got = torch.stack(st.run([ids[i].contiguous().cuda() for i in range(2)])).float().cpu().view(2, 128, 768)
    for i in range(2):
        assert ((got[i] - ref1[i]).norm() / ref1[i].norm()).item() < 2e-2
