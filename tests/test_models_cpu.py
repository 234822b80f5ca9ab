"""Host-side checks of the unit chains against the oracle (no GPU): boundary shapes, payload
bytes, unit counts as SURVEY App. B lists them, and BN folding arithmetic."""
import pytest
import torch

from oracle.units import run_span, units_for
from paper_2312_10636_b200.models import build_chain, torch_model

CASES = {"resnet18": (10, 224), "resnet50": (18, 224), "vgg16": (8, 224), "inception_v3": (19, 299)}


@pytest.mark.parametrize("name", list(CASES))
def test_chain_boundaries_match_oracle(name):
    n_units, res = CASES[name]
    m = torch_model(name)
    chain = build_chain(name, module=m)
    assert chain.n_units == n_units
    units = units_for(name, m)
    assert len(units) == n_units
    x = torch.randn(1, 3, res, res)
    for p in range(n_units):
        if p > 0:
            H, W, Cc, _ = chain.boundary_shape(p)
            if x.dim() == 4:
                assert tuple(x.shape[1:]) == (Cc, H, W), (p, x.shape, (H, W, Cc))
            else:
                assert x.shape[1] == H * W * Cc
        x = run_span(units, p, p + 1, x)
    assert x.shape == (1, 1000)
    assert chain.boundary_elems(n_units) == 1000


def test_resnet50_payloads_match_survey_appendix_b():
    chain = build_chain("resnet50")
    # SURVEY App. B lists bf16 bytes; the wire format is fp32 (PAPER.md:463, 588 KB input)
    bf16 = {1: 401_408, 2: 1_605_632, 5: 802_816, 9: 401_408, 15: 200_704}
    for p, b in bf16.items():
        assert chain.payload_bytes(p) == 2 * b
    assert chain.payload_bytes(0) == 3 * 224 * 224 * 4
    gflop = sum(chain.unit_flops) / 1e9
    assert abs(gflop - 8.18) < 0.05


def test_bn_folding_matches_module():
    from paper_2312_10636_b200.device import pack_conv_weight
    m = torch_model("resnet18")
    conv, bn = m.layer1[0].conv1, m.layer1[0].bn1
    x = torch.randn(2, 64, 9, 9)
    ref = bn(conv(x))
    scale = bn.weight / torch.sqrt(bn.running_var + bn.eps)
    w = conv.weight * scale[:, None, None, None]
    b = bn.bias - bn.running_mean * scale
    got = torch.nn.functional.conv2d(x, w, b, padding=1)
    assert torch.allclose(got, ref, atol=1e-4, rtol=1e-4)
    packed = pack_conv_weight(w.detach())
    assert packed.shape == (64, 576)


@pytest.mark.parametrize("name", list(CASES) + ["bert_base"])
def test_fp32_chain_mirrors_bf16_chain(name):
    """The fp32 execution mode is the same chain (units, boundaries, ops, payloads) with every
    tensor fp32 and weights stored fp32 (twice the bf16 bytes for conv / linear / FC weights)."""
    from paper_2312_10636_b200 import _native as N
    m = torch_model(name)
    # (bf16 ResNet-50 chains fuse each downsample into its expand GEMM; the fp32 mode keeps it apart)
    a = build_chain(name, module=m, fuse_downsample=False) if name in ("resnet18", "resnet50") else \
        build_chain(name, module=m)
    b = build_chain(name, module=m, dtype=N.GX_F32)
    assert b.dtype == N.GX_F32 and a.dtype == N.GX_BF16
    assert a.boundary == b.boundary and a.unit_first_op == b.unit_first_op
    # (bf16 Inception stores its 48 / 96 / 160-channel branch intermediates zero-padded to a multiple
    # of 64 channels, models._mid; never a boundary tensor)
    def padded(x, y):
        return x == y or x == -(-y // 64) * 64

    assert [t[:2] for t in a.tensors] == [t[:2] for t in b.tensors]
    assert all(padded(ta[2], tb[2]) for ta, tb in zip(a.tensors, b.tensors))
    assert all(a.tensors[t][2] == b.tensors[t][2] for t in a.boundary)
    # (BERT's boundary 0 holds int32 token ids in both modes: the K8 embedding's input)
    assert all(t[3] == N.GX_F32 or (t[3] == N.GX_I32 and i == b.boundary[0]) for i, t in enumerate(b.tensors))
    # bf16 chains: only the chain output may be fp32
    assert all(t[3] == N.GX_BF16 or i == a.boundary[-1] or (t[3] == N.GX_I32 and i == a.boundary[0])
               for i, t in enumerate(a.tensors))
    assert [a.payload_bytes(p) for p in range(a.n_units + 1)] == [b.payload_bytes(p) for p in range(b.n_units + 1)]
    assert [(o.kind, o.in_, o.out) for o in a.ops] == [(o.kind, o.in_, o.out) for o in b.ops]
    assert all(padded(oa.Cin, ob.Cin) and padded(oa.Cout, ob.Cout) for oa, ob in zip(a.ops, b.ops))
    assert b.blob.size > 1.8 * a.blob.size


def test_bert_boundary_zero_ships_token_ids():
    """K8: a BERT fragment entering at boundary 0 ships its 128 int32 token ids (512 B, the
    ModelSpec input bytes); unit 0 starts with the embedding op; inner boundaries stay the
    [128, 768] hidden state (393,216 B fp32)."""
    from paper_2312_10636_b200 import _native as N
    chain = build_chain("bert_base")
    assert chain.boundary_shape(0) == (128, 1, 1, N.GX_I32)
    assert chain.payload_bytes(0) == 512 and chain.payload_bytes(6) == 393216
    assert chain.ops[chain.unit_first_op[0]].kind == N.GX_OP_EMBED
    assert chain.model_spec_doc()["input_bytes"] == 512


def test_fused_downsample_chain_keeps_units():
    """The fused ResNet-50 chain (GX_OPF_DS) has the unfused chain's units, boundary shapes, payloads
    and FLOPs, with four ops fewer (one per stage's first bottleneck)."""
    from paper_2312_10636_b200 import _native as N
    m = torch_model("resnet50")
    a = build_chain("resnet50", module=m)
    b = build_chain("resnet50", module=m, fuse_downsample=False)
    assert a.n_units == b.n_units and len(a.ops) == len(b.ops) - 4
    assert [a.boundary_shape(p) for p in range(a.n_units + 1)] == [b.boundary_shape(p) for p in range(b.n_units + 1)]
    assert [round(f) for f in a.unit_flops] == [round(f) for f in b.unit_flops]
    ds = [o for o in a.ops if o.flags & N.GX_OPF_DS]
    assert [(o.Cin, a.tensors[o.in2][2], o.Cout, o.reserved) for o in ds] == [
        (64, 64, 256, 1), (128, 256, 512, 2), (256, 512, 1024, 2), (512, 1024, 2048, 2)]


@pytest.mark.parametrize("name", ["resnet50", "vgg16", "inception_v3"])
def test_padded_convs_count_logical_flops(name):
    """Convs run on zero-padded channels (stem 3 -> 8 / s2d, Inception's 48/96/160 -> 64/128/192
    intermediates) carry logical/executed FLOP ratios, so the executed conv/FC work scaled by them
    adds up to the chain's logical FLOPs (what the roofline tables divide by)."""
    from paper_2312_10636_b200 import _native as N
    c = build_chain(name, module=torch_model(name))
    total = 0.0
    for i, o in enumerate(c.ops):
        H, W, _, _ = c.tensors[o.out]
        if o.kind == N.GX_OP_CONV:
            k_ds = c.tensors[o.in2][2] if o.flags & N.GX_OPF_DS else 0
            executed = 2.0 * H * W * o.Cout * (o.Cin * o.R * o.S + k_ds)
        elif o.kind == N.GX_OP_FC:
            executed = 2.0 * o.Cin * o.Cout
        else:
            continue
        total += executed * c.op_flops_scale.get(i, 1.0)
    assert abs(total - sum(c.unit_flops)) <= 1e-9 * total
    if name == "inception_v3":
        padded = [i for i, v in c.op_flops_scale.items() if i > 0]
        assert len(padded) == 30 and all(0.69 < c.op_flops_scale[i] < 0.84 for i in padded)
