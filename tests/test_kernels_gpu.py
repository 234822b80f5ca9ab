"""Kernel parity on the B200: every libgx kernel vs a plain PyTorch fp32 reference of the same op.

bf16 in, fp32 accumulate, bf16 out: tolerance is bf16 output rounding plus input rounding
(relative 1.5e-2 on the max-norm, written per test).  Integer/byte work (gather/scatter) is
bit-exact.
"""
import pytest
import torch
import torch.nn.functional as F
from paper_2312_10636_b200.errors import ValidationError

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2312_10636_b200 import _native as N
    from paper_2312_10636_b200.device import WeightBlob, pack_conv_weight, run_op, tensor_desc


def _rel(a, b):
    return ((a.float() - b.float()).abs().max() / b.float().abs().max().clamp_min(1e-6)).item()


def _conv_case(k, H, W, Cin, Cout, R, S, stride, pad, residual, relu, cin_pad=None, sm_budget=0, out_coff=0,
               out_c=None, seed=0):
    g = torch.Generator().manual_seed(seed)
    dev = "cuda"
    cin_pad = cin_pad or Cin
    x = torch.randn(k, H, W, Cin, generator=g)
    w = torch.randn(Cout, Cin, R, S, generator=g) / (Cin * R * S) ** 0.5
    b = torch.randn(Cout, generator=g) * 0.1
    ph, pw = pad if isinstance(pad, tuple) else (pad, pad)
    Ho = (H + 2 * ph - R) // stride + 1
    Wo = (W + 2 * pw - S) // stride + 1
    xb = x.to(torch.bfloat16)
    ref = F.conv2d(xb.float().permute(0, 3, 1, 2), w.to(torch.bfloat16).float(), b, stride=stride, padding=(ph, pw))
    ref = ref.permute(0, 2, 3, 1)
    res = None
    if residual:
        res = torch.randn(k, Ho, Wo, Cout, generator=g).to(torch.bfloat16)
        ref = ref + res.float()
    if relu:
        ref = ref.clamp_min(0)
    blob = WeightBlob()
    w_off = blob.add_bf16(pack_conv_weight(w, cin_pad))
    b_off = blob.add_f32(b)
    wdev = torch.from_numpy(blob.bytes()).to(dev)
    xin = torch.zeros(k, H, W, cin_pad, dtype=torch.bfloat16)
    xin[..., :Cin] = xb
    xin = xin.to(dev)
    out_c = out_c or Cout
    y = torch.full((k, Ho, Wo, out_c), float("nan"), dtype=torch.bfloat16, device=dev)
    descs = [tensor_desc(H, W, cin_pad), tensor_desc(Ho, Wo, out_c), tensor_desc(Ho, Wo, Cout)]
    tensors = [xin, y, res.to(dev) if residual else y]
    op = N.make_op(N.GX_OP_CONV, 0, 1, in2=2 if residual else -1, out_coff=out_coff,
                   act=N.GX_ACT_RELU if relu else N.GX_ACT_NONE, R=R, S=S, sh=stride, sw=stride, ph=ph, pw=pw,
                   Cin=cin_pad, Cout=Cout, w_off=w_off, b_off=b_off)
    run_op(op, tensors, descs, wdev, k, sm_budget)
    torch.cuda.synchronize()
    got = y[..., out_coff:out_coff + Cout].float().cpu()
    assert torch.isfinite(got).all(), "conv left unwritten outputs"
    return got, ref


@pytest.mark.parametrize(
    "k,H,W,Cin,Cout,R,S,stride,pad,residual,relu",
    [
        (1, 8, 8, 64, 64, 1, 1, 1, 0, False, False),     # smallest 1x1
        (2, 14, 14, 64, 128, 3, 3, 1, 1, False, True),   # 3x3 s1 p1
        (3, 28, 28, 128, 256, 1, 1, 1, 0, True, True),   # bottleneck expand + residual
        (2, 56, 56, 64, 64, 3, 3, 1, 1, False, True),    # layer1 3x3
        (2, 28, 28, 128, 128, 3, 3, 2, 1, False, True),  # stride-2 3x3
        (2, 14, 14, 256, 512, 1, 1, 2, 0, False, False), # stride-2 downsample 1x1
        (1, 7, 7, 512, 2048, 1, 1, 1, 0, True, True),    # layer4 expand, many N tiles
        (5, 7, 7, 512, 512, 3, 3, 1, 1, False, True),    # M not a multiple of 128
        (1, 17, 17, 192, 160, 1, 7, 1, 0, False, True),  # 1x7 unpadded
        (2, 17, 17, 128, 192, 1, 7, 1, (0, 3), False, True),  # Inception 1x7, asymmetric pad
        (2, 17, 17, 128, 128, 7, 1, 1, (3, 0), False, True),  # Inception 7x1
        (3, 8, 8, 384, 384, 1, 3, 1, (0, 1), False, True),    # Inception E 1x3
        (2, 35, 35, 288, 64, 1, 1, 1, 0, False, True),        # Cin % 64 != 0 -> cp.async path
        (2, 35, 35, 288, 384, 3, 3, 2, 0, False, True),       # Mixed_6a 3x3 s2 on 288 ch
        (2, 35, 35, 64, 96, 5, 5, 1, 2, False, True),         # 5x5
        (16, 7, 7, 512, 512, 3, 3, 1, 1, True, True),         # tail tile + residual
        (3, 14, 14, 1024, 2048, 1, 1, 2, 0, False, False),    # downsample into layer4
        # halo path (conv_halo.cu): 3x3/s1/p1, Cin % 64 == 0, W >= 28
        (1, 56, 56, 64, 64, 3, 3, 1, 1, False, True),         # layer1 3x3 at k=1 (BH=2)
        (3, 28, 28, 128, 128, 3, 3, 1, 1, False, True),       # layer2 3x3 (BH=4)
        (2, 35, 35, 64, 96, 3, 3, 1, 1, False, True),         # Inception 35x35 (BH=3, last tile short)
        (2, 30, 30, 128, 192, 3, 3, 1, 1, False, False),      # W+2 = 32, BN not a power of two
        # wide halo (column tiles) and 32-channel halo rows
        (2, 147, 147, 32, 64, 3, 3, 1, 1, False, True),       # Inception Conv2d_2b (RB 64, column tiles)
        (1, 149, 149, 32, 32, 3, 3, 1, 0, False, True),       # Inception Conv2d_2a, unpadded
        (2, 112, 112, 128, 128, 3, 3, 1, 1, False, True),     # VGG-16 conv2 (RB 128, column tiles)
        (1, 224, 224, 64, 64, 3, 3, 1, 1, False, True),       # VGG-16 conv1_2
        (3, 40, 40, 32, 48, 3, 3, 1, 1, False, False),        # 32 channels, whole rows
    ],
)
def test_conv_matches_torch(k, H, W, Cin, Cout, R, S, stride, pad, residual, relu):
    got, ref = _conv_case(k, H, W, Cin, Cout, R, S, stride, pad, residual, relu)
    assert _rel(got, ref) < 1.5e-2


@pytest.mark.parametrize("k,H,Cout,path", [(2, 112, 64, "halo32"), (3, 56, 64, "halo32"), (1, 28, 32, "halo32"),
                                            (2, 112, 64, "im2col")])
def test_conv_s2d_stem(k, H, Cout, path):
    """The space-to-depth stem: 4x4 / stride 1 / pad (2, 2, 1, 1) over 16 channels, on the 32-byte
    halo path (conv_halo_kernel<32>: one halo tile, sixteen K=16 MMAs at row offsets) and on the
    im2col path (op flag GX_OPF_NO_HALO), vs torch on the same bf16 data."""
    g = torch.Generator().manual_seed(5)
    x = torch.randn(k, H, H, 16, generator=g).to(torch.bfloat16)
    w = torch.randn(Cout, 16, 4, 4, generator=g) / 16.0
    b = torch.randn(Cout, generator=g) * 0.1
    xp = F.pad(x.float().permute(0, 3, 1, 2), (2, 1, 2, 1))
    ref = F.conv2d(xp, w.to(torch.bfloat16).float(), b).clamp_min(0).permute(0, 2, 3, 1)
    blob = WeightBlob()
    w_off = blob.add_bf16(pack_conv_weight(w, 16))
    b_off = blob.add_f32(b)
    wdev = torch.from_numpy(blob.bytes()).cuda()
    y = torch.full((k, H, H, Cout), float("nan"), dtype=torch.bfloat16, device="cuda")
    op = N.make_op(N.GX_OP_CONV, 0, 1, act=N.GX_ACT_RELU, R=4, S=4, sh=1, sw=1, ph=2, pw=2, ph_hi=1, pw_hi=1,
                   Cin=16, Cout=Cout, w_off=w_off, b_off=b_off, flags=N.GX_OPF_NO_HALO if path == "im2col" else 0)
    run_op(op, [x.cuda(), y], [tensor_desc(H, H, 16), tensor_desc(H, H, Cout)], wdev, k, 3)
    torch.cuda.synchronize()
    got = y.float().cpu()
    assert torch.isfinite(got).all(), "conv left unwritten outputs"
    assert _rel(got, ref) < 1.5e-2


def test_conv_stem_channel_padded():
    # ResNet stem: 3-channel image zero-padded to 8 channels, 7x7 stride 2 pad 3
    got, ref = _conv_case(2, 64, 64, 3, 64, 7, 7, 2, 3, False, True, cin_pad=8)
    assert _rel(got, ref) < 1.5e-2


def test_conv_bounded_sm_budget_and_concat_offset():
    got, ref = _conv_case(4, 28, 28, 64, 96, 3, 3, 1, 1, False, True, sm_budget=5, out_coff=32, out_c=160)
    assert _rel(got, ref) < 1.5e-2


@pytest.mark.parametrize("k,residual", [(1, False), (1, True), (2, True), (3, False)])
def test_conv_1x1_single_short_tile(k, residual):
    """layer4 1x1 convs at batch 1-3 (M = 49k < 128): the A box holds only the live rows."""
    got, ref = _conv_case(k, 7, 7, 512, 2048, 1, 1, 1, 0, residual, True, sm_budget=6)
    assert _rel(got, ref) < 1.5e-2


def test_conv_large_m_persistent():
    got, ref = _conv_case(8, 56, 56, 256, 64, 1, 1, 1, 0, False, True, sm_budget=20)
    assert _rel(got, ref) < 1.5e-2


@pytest.mark.parametrize("mode,R,stride,pad", [("max", 3, 2, 1), ("max", 2, 2, 0), ("avg", 3, 1, 1),
                                                ("max", 3, 2, 0), ("max", 3, 1, 1), ("avg", 3, 1, 0),
                                                ("max", 3, 1, 0)])
def test_pool(mode, R, stride, pad):
    g = torch.Generator().manual_seed(1)
    k, H, W, Cc = 3, 15, 15, 64
    x = torch.randn(k, H, W, Cc, generator=g).to(torch.bfloat16)
    xn = x.float().permute(0, 3, 1, 2)
    if mode == "max":
        ref = F.max_pool2d(xn, R, stride, pad)
    else:
        ref = F.avg_pool2d(xn, R, stride, pad, count_include_pad=True)
    ref = ref.permute(0, 2, 3, 1)
    Ho, Wo = ref.shape[1], ref.shape[2]
    y = torch.empty(k, Ho, Wo, Cc, dtype=torch.bfloat16, device="cuda")
    op = N.make_op(N.GX_OP_MAXPOOL if mode == "max" else N.GX_OP_AVGPOOL, 0, 1, R=R, S=R, sh=stride, sw=stride,
                   ph=pad, pw=pad, flags=1)
    run_op(op, [x.cuda(), y], [tensor_desc(H, W, Cc), tensor_desc(Ho, Wo, Cc)], torch.zeros(256, device="cuda"), k)
    torch.cuda.synchronize()
    assert _rel(y.float().cpu(), ref) < 1e-2
    if mode == "max":  # a maximum is one of its inputs: bit-exact against the fp32 pool of the bf16 input
        assert torch.equal(y.float().cpu(), ref)


@pytest.mark.parametrize("k,H", [(5, 7), (700, 7), (3, 8)])  # few items (block per item) / many (warp per item)
def test_gap_and_fc(k, H):
    g = torch.Generator().manual_seed(2)
    HW, Cc, O = H * H, 2048, 1000
    x = torch.randn(k, H, H, Cc, generator=g).to(torch.bfloat16)
    w = torch.randn(O, Cc, generator=g) / Cc ** 0.5
    b = torch.randn(O, generator=g)
    pooled_ref = x.float().mean(dim=(1, 2))
    blob = WeightBlob()
    w_off = blob.add_bf16(w)
    b_off = blob.add_f32(b)
    wdev = torch.from_numpy(blob.bytes()).cuda()
    pooled = torch.empty(k, Cc, dtype=torch.bfloat16, device="cuda")
    run_op(N.make_op(N.GX_OP_GAP, 0, 1), [x.cuda(), pooled], [tensor_desc(H, H, Cc), tensor_desc(1, 1, Cc)], wdev, k)
    logits = torch.empty(k, O, dtype=torch.float32, device="cuda")
    run_op(N.make_op(N.GX_OP_FC, 0, 1, Cin=Cc, Cout=O, w_off=w_off, b_off=b_off), [pooled, logits],
           [tensor_desc(1, 1, Cc), tensor_desc(1, 1, O, N.GX_F32)], wdev, k)
    torch.cuda.synchronize()
    assert _rel(pooled.float().cpu(), pooled_ref) < 1e-2
    ref = pooled.float().cpu() @ w.to(torch.bfloat16).float().t() + b
    assert _rel(logits.cpu(), ref) < 1e-3


@pytest.mark.parametrize("path", ["tcgen05", "simt"])
@pytest.mark.parametrize("k,H,W,Cc,O,out_f32,relu", [
    (1, 1, 1, 2048, 1000, True, False),     # ResNet-50 head at batch 1 (Cout % 16 tail: 1000)
    (16, 1, 1, 2048, 1000, True, False),
    (3, 7, 7, 512, 4096, False, True),      # VGG-16 fc6: flattened 7x7x512 input, bf16 out + ReLU
    (130, 1, 1, 512, 1000, True, False),    # two 128-row M tiles
])
def test_fc_paths(path, k, H, W, Cc, O, out_f32, relu):
    """FC on the tcgen05 GEMM path (conv_tc_kernel with the flattened [k, K] input as A) and on the
    CUDA-core weight-streaming kernel (op flag GX_OPF_FC_SIMT): same results vs an fp32 matmul of
    the bf16 data."""
    g = torch.Generator().manual_seed(7)
    K = H * W * Cc
    x = torch.randn(k, H, W, Cc, generator=g).to(torch.bfloat16)
    w = torch.randn(O, K, generator=g) / K ** 0.5
    b = torch.randn(O, generator=g)
    blob = WeightBlob()
    w_off = blob.add_bf16(w)
    b_off = blob.add_f32(b)
    wdev = torch.from_numpy(blob.bytes()).cuda()
    y = torch.full((k, O), float("nan"), dtype=torch.float32 if out_f32 else torch.bfloat16, device="cuda")
    op = N.make_op(N.GX_OP_FC, 0, 1, Cin=K, Cout=O, w_off=w_off, b_off=b_off,
                   act=N.GX_ACT_RELU if relu else N.GX_ACT_NONE, flags=N.GX_OPF_FC_SIMT if path == "simt" else 0)
    run_op(op, [x.cuda(), y], [tensor_desc(H, W, Cc), tensor_desc(1, 1, O, N.GX_F32 if out_f32 else N.GX_BF16)],
           wdev, k, sm_budget=4)
    torch.cuda.synchronize()
    ref = x.reshape(k, K).float() @ w.to(torch.bfloat16).float().t() + b
    if relu:
        ref = ref.clamp_min(0)
    got = y.float().cpu()
    assert not got.isnan().any()
    assert _rel(got, ref) < (1e-3 if out_f32 else 1e-2)


def test_gather_scatter_bit_exact():
    import ctypes as C
    from paper_2312_10636_b200.device import context
    ctx = context(0)
    k, pix, Cc = 6, 56 * 56, 64
    srcs = []
    dts = []
    for i in range(k):
        if i % 2:
            srcs.append(torch.randn(pix * Cc, device="cuda"))
            dts.append(N.GX_F32)
        else:
            srcs.append(torch.randn(pix * Cc, device="cuda").to(torch.bfloat16))
            dts.append(N.GX_BF16)
    dst = torch.empty(k, pix * Cc, dtype=torch.bfloat16, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    N.check(N.lib().gx_gather(ctx.handle, k, N.ptr_array([t.data_ptr() for t in srcs]), N.i32_array(dts), pix, Cc,
                              Cc, C.c_void_p(dst.data_ptr()), 0, C.c_void_p(s)))
    outs = [torch.empty(pix * Cc, dtype=torch.float32, device="cuda") for _ in range(k)]
    N.check(N.lib().gx_scatter(ctx.handle, k, C.c_void_p(dst.data_ptr()), N.GX_BF16, pix * Cc,
                               N.ptr_array([o.data_ptr() for o in outs]), N.GX_F32, 0, C.c_void_p(s)))
    torch.cuda.synchronize()
    for i in range(k):
        exp = srcs[i].to(torch.bfloat16)
        assert torch.equal(dst[i], exp)
        assert torch.equal(outs[i], exp.float())
    # 3 -> 8 channel padding of the raw image (stem ingress)
    img = [torch.randn(224 * 224 * 3, device="cuda") for _ in range(2)]
    d8 = torch.empty(2, 224 * 224 * 8, dtype=torch.bfloat16, device="cuda")
    N.check(N.lib().gx_gather(ctx.handle, 2, N.ptr_array([t.data_ptr() for t in img]), N.i32_array([N.GX_F32] * 2),
                              224 * 224, 3, 8, C.c_void_p(d8.data_ptr()), 0, C.c_void_p(s)))
    torch.cuda.synchronize()
    for i in range(2):
        v = d8[i].view(224 * 224, 8)
        assert torch.equal(v[:, :3], img[i].view(-1, 3).to(torch.bfloat16))
        assert (v[:, 3:] == 0).all()


@pytest.mark.parametrize("k,S,K,O,act,residual", [(1, 128, 768, 2304, "none", False), (3, 128, 768, 768, "none", True),
                                                  (2, 128, 768, 3072, "gelu", False), (2, 128, 3072, 768, "none", True)])
def test_linear_matches_torch(k, S, K, O, act, residual):
    """BERT's four linears: [S, K] x W^T on the tcgen05 GEMM path (GX_OP_LINEAR, 1x1 over [S,1,K])."""
    g = torch.Generator().manual_seed(11)
    x = torch.randn(k, S, K, generator=g).to(torch.bfloat16)
    w = torch.randn(O, K, generator=g) / K ** 0.5
    b = torch.randn(O, generator=g) * 0.1
    ref = x.float() @ w.to(torch.bfloat16).float().t() + b
    res = torch.randn(k, S, O, generator=g).to(torch.bfloat16) if residual else None
    if residual:
        ref = ref + res.float()
    if act == "gelu":
        ref = F.gelu(ref)
    blob = WeightBlob()
    w_off = blob.add_bf16(pack_conv_weight(w.view(O, K, 1, 1)))
    b_off = blob.add_f32(b)
    wdev = torch.from_numpy(blob.bytes()).cuda()
    y = torch.full((k, S, O), float("nan"), dtype=torch.bfloat16, device="cuda")
    descs = [tensor_desc(S, 1, K), tensor_desc(S, 1, O), tensor_desc(S, 1, O)]
    op = N.make_op(N.GX_OP_LINEAR, 0, 1, in2=2 if residual else -1,
                   act=N.GX_ACT_GELU if act == "gelu" else N.GX_ACT_NONE, Cin=K, Cout=O, w_off=w_off, b_off=b_off)
    run_op(op, [x.cuda(), y, res.cuda() if residual else y], descs, wdev, k, 40)
    torch.cuda.synchronize()
    assert _rel(y.float().cpu(), ref) < 1.5e-2


@pytest.mark.parametrize("k,S,C", [(1, 128, 768), (5, 128, 768), (2, 33, 256), (1, 7, 1024)])
def test_layernorm_matches_torch(k, S, C):
    g = torch.Generator().manual_seed(12)
    x = (torch.randn(k, S, C, generator=g) * 3 + 1).to(torch.bfloat16)
    gamma = torch.randn(C, generator=g) * 0.2 + 1
    beta = torch.randn(C, generator=g) * 0.1
    ref = F.layer_norm(x.float(), (C,), gamma, beta, eps=1e-12)
    blob = WeightBlob()
    g_off, b_off = blob.add_f32(gamma), blob.add_f32(beta)
    wdev = torch.from_numpy(blob.bytes()).cuda()
    y = torch.full((k, S, C), float("nan"), dtype=torch.bfloat16, device="cuda")
    op = N.make_op(N.GX_OP_LAYERNORM, 0, 1, w_off=g_off, b_off=b_off, eps=1e-12)
    run_op(op, [x.cuda(), y], [tensor_desc(S, 1, C), tensor_desc(S, 1, C)], wdev, k, 16)
    torch.cuda.synchronize()
    assert _rel(y.float().cpu(), ref) < 1e-2


@pytest.mark.parametrize("k,S,heads", [(1, 128, 12), (3, 128, 12), (2, 77, 4), (1, 512, 2)])
def test_attention_matches_torch(k, S, heads):
    """Non-causal multi-head attention on a packed [q|k|v] row (BertSelfAttention, no mask)."""
    g = torch.Generator().manual_seed(13)
    D = 64
    hidden = heads * D
    qkv = (torch.randn(k, S, 3 * hidden, generator=g) * 1.5).to(torch.bfloat16)
    q, kk, v = qkv.float().split(hidden, dim=-1)
    sh = lambda t: t.view(k, S, heads, D).transpose(1, 2)
    ref = F.scaled_dot_product_attention(sh(q), sh(kk), sh(v)).transpose(1, 2).reshape(k, S, hidden)
    y = torch.full((k, S, hidden), float("nan"), dtype=torch.bfloat16, device="cuda")
    op = N.make_op(N.GX_OP_ATTENTION, 0, 1, heads=heads, Cout=hidden)
    run_op(op, [qkv.cuda(), y], [tensor_desc(S, 1, 3 * hidden), tensor_desc(S, 1, hidden)],
           torch.zeros(256, device="cuda"), k, 30)
    torch.cuda.synchronize()
    assert _rel(y.float().cpu(), ref) < 1.5e-2


def test_gather_scatter_max_batch_ragged():
    """The largest dispatched batch the ABI takes (64 rows), every row from its own buffer, fp32 and
    bf16 sources interleaved at odd sizes: bit-exact."""
    import ctypes as C
    from paper_2312_10636_b200.device import context
    ctx = context(0)
    k, pix, Cc = 64, 7 * 7, 2048
    srcs = [torch.randn(pix * Cc, device="cuda").to(torch.bfloat16 if i % 3 else torch.float32) for i in range(k)]
    dts = [N.GX_F32 if t.dtype == torch.float32 else N.GX_BF16 for t in srcs]
    dst = torch.empty(k, pix * Cc, dtype=torch.bfloat16, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    N.check(N.lib().gx_gather(ctx.handle, k, N.ptr_array([t.data_ptr() for t in srcs]), N.i32_array(dts), pix, Cc,
                              Cc, C.c_void_p(dst.data_ptr()), 3, C.c_void_p(s)))
    torch.cuda.synchronize()
    for i in range(k):
        assert torch.equal(dst[i], srcs[i].to(torch.bfloat16)), i
    with pytest.raises(ValidationError):
        N.check(N.lib().gx_gather(ctx.handle, 65, N.ptr_array([srcs[0].data_ptr()] * 65), N.i32_array(dts[:1] * 65),
                                  pix, Cc, Cc, C.c_void_p(dst.data_ptr()), 3, C.c_void_p(s)))


def test_stage_batch_sizes_share_one_instance():
    """One stage instance serves k = 1 .. max_batch (a CUDA graph per k, one workspace): each batch
    size gives the same per-request output, and k outside 1..max_batch is rejected."""
    from paper_2312_10636_b200.engine import DeviceModel, StageInstance
    from paper_2312_10636_b200.models import build_chain
    chain = build_chain("resnet18")
    dm = DeviceModel(chain, 0)
    st = StageInstance(dm, 6, chain.n_units, max_batch=8, sm_budget=3)
    x = [torch.rand(chain.boundary_elems(6), device="cuda") for _ in range(8)]
    full = st.run(x)
    for k in (1, 3, 8):
        part = st.run(x[:k])
        for i in range(k):
            assert torch.equal(part[i], full[i]), (k, i)
    with pytest.raises(ValidationError):
        st.run(x + x[:1])


@pytest.mark.parametrize("f,c_src,c_dst,H,dst_f32", [(2, 3, 16, 112, False), (2, 3, 16, 112, True),
                                                    (2, 3, 16, 56, False), (1, 3, 8, 37, False),
                                                    (1, 3, 8, 37, True), (2, 2, 12, 20, False)])
def test_gather_ex_space_to_depth_bit_exact(f, c_src, c_dst, H, dst_f32):
    """K1 gather into the stem's space-to-depth boundary (the vectorised one-pixel-per-thread path
    for 2x2 RGB blocks, the generic per-element path otherwise) and the plain channel-padded gather,
    into bf16 and into fp32 batches, for ragged fp32 / bf16 sources: bit-exact with torch's own
    rearrangement and cast."""
    import ctypes as C
    from paper_2312_10636_b200.device import context
    ctx = context(0)
    k = 5
    g = torch.Generator().manual_seed(9)
    imgs = [torch.randn(H * f, H * f, c_src, generator=g) for _ in range(k)]
    srcs = [im.cuda() if i % 2 == 0 else im.to(torch.bfloat16).cuda() for i, im in enumerate(imgs)]
    refs = []
    for im, s in zip(imgs, srcs):
        v = s.float().cpu()
        v = v.view(H, f, H, f, c_src).permute(0, 2, 1, 3, 4).reshape(H, H, f * f * c_src)
        refs.append(F.pad(v, (0, c_dst - f * f * c_src)))
    ref = torch.stack(refs)
    dt = torch.float32 if dst_f32 else torch.bfloat16
    out = torch.full((k, H, H, c_dst), float("nan"), dtype=dt, device="cuda")
    N.check(N.lib().gx_gather_ex(ctx.handle, k, N.ptr_array([s.data_ptr() for s in srcs]),
                                 N.i32_array([N.GX_F32 if s.dtype == torch.float32 else N.GX_BF16 for s in srcs]),
                                 H, H, f, c_src, c_dst, C.c_void_p(out.data_ptr()), N.GX_F32 if dst_f32 else N.GX_BF16,
                                 3, C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    torch.cuda.synchronize()
    assert torch.equal(out.cpu(), ref.to(dt))


@pytest.mark.parametrize("k,H,Ct,Cx,Cout,stride,budget", [
    (3, 56, 64, 64, 256, 1, 4),      # layer1 block 0 (downsample at stride 1)
    (2, 28, 128, 256, 512, 2, 6),    # layer2 block 0: block input 56x56x256 at stride 2
    (1, 7, 512, 1024, 2048, 2, 3),   # layer4 block 0 at batch 1
    (5, 14, 256, 512, 1024, 2, 148),
])
def test_conv_fused_downsample_matches_torch(k, H, Ct, Cx, Cout, stride, budget):
    """GX_OPF_DS: a bottleneck's expand 1x1 and its block's 1x1 downsample as one K-concatenated
    GEMM, y = relu(W3 t + Wd x[::s, ::s] + b3 + bd), against the two convs in fp32."""
    g = torch.Generator().manual_seed(11)
    t = torch.randn(k, H, H, Ct, generator=g).to(torch.bfloat16)
    x = torch.randn(k, H * stride, H * stride, Cx, generator=g).to(torch.bfloat16)
    w3 = torch.randn(Cout, Ct, 1, 1, generator=g) / Ct ** 0.5
    wd = torch.randn(Cout, Cx, 1, 1, generator=g) / Cx ** 0.5
    b = torch.randn(Cout, generator=g) * 0.1
    ref = (F.conv2d(t.float().permute(0, 3, 1, 2), w3.to(torch.bfloat16).float()) +
           F.conv2d(x.float().permute(0, 3, 1, 2), wd.to(torch.bfloat16).float(), stride=stride) +
           b.view(1, -1, 1, 1)).clamp_min(0).permute(0, 2, 3, 1)
    blob = WeightBlob()
    w_off = blob.add_bf16(torch.cat([pack_conv_weight(w3), pack_conv_weight(wd)], dim=1))
    b_off = blob.add_f32(b)
    wdev = torch.from_numpy(blob.bytes()).cuda()
    y = torch.full((k, H, H, Cout), float("nan"), dtype=torch.bfloat16, device="cuda")
    op = N.make_op(N.GX_OP_CONV, 0, 1, in2=2, act=N.GX_ACT_RELU, Cin=Ct, Cout=Cout, w_off=w_off, b_off=b_off,
                   flags=N.GX_OPF_DS, reserved=stride)
    run_op(op, [t.cuda(), y, x.cuda()],
           [tensor_desc(H, H, Ct), tensor_desc(H, H, Cout), tensor_desc(H * stride, H * stride, Cx)], wdev, k, budget)
    torch.cuda.synchronize()
    got = y.float().cpu()
    assert torch.isfinite(got).all()
    assert _rel(got, ref) < 1.5e-2
