"""Unit chains: the executor-side form of the reference's ModelSpec (profiles.py:31-87).

A model is a linear chain of N units; boundary p is the input of unit p (boundary 0 = the raw
input, boundary N = the output), exactly as ModelSpec.payload_bytes(p) counts them
(profiles.py:67-74).  Each unit lowers to a short run of libgx ops over per-sample NHWC bf16
tensors; BatchNorm is folded into the preceding conv at build time, ReLU / residual adds are
fused into the conv epilogue, Inception branch outputs are written straight into their concat
slice, and VGG's NCHW flatten is folded into fc1's column order.

Weights are random-initialised parameters of the named architecture (torchvision /
transformers definitions as the parameter source, seeded), so the CPU oracle can run the very
same parameters in fp32.  Only parameter tensors are taken from torch; nothing here computes.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch
import torch.nn as nn

from . import _native as N
from .device import WeightBlob, pack_conv_weight

BF16, F32 = N.GX_BF16, N.GX_F32


@dataclass
class UnitChain:
    model_id: str
    tensors: list = field(default_factory=list)  # (H, W, C, dtype)
    ops: list = field(default_factory=list)  # GxOp
    unit_first_op: list = field(default_factory=list)
    boundary: list = field(default_factory=list)
    blob: WeightBlob = field(default_factory=WeightBlob)
    input_channels: int = 3  # channels a client actually ships at boundary 0 (pre-padding)
    unit_flops: list = field(default_factory=list)  # per-sample FLOPs of each unit
    tensor_s2d: dict = field(default_factory=dict)  # tensor id -> space-to-depth factor (stride-2 stems)
    dtype: int = BF16  # compute element type (F32: the fp32 execution mode)
    # op index -> logical / executed FLOPs of a conv whose channels are zero-padded (the stem's
    # 3 -> 8 input, Inception's 48 / 96 / 160-channel intermediates stored at 64 / 128 / 192): the
    # roofline tables count the logical FLOPs only
    op_flops_scale: dict = field(default_factory=dict)

    @property
    def n_units(self) -> int:
        return len(self.boundary) - 1

    def boundary_shape(self, p: int):
        H, W, Cc, dt = self.tensors[self.boundary[p]]
        return H, W, Cc, dt

    def boundary_elems(self, p: int) -> int:
        H, W, Cc, _ = self.boundary_shape(p)
        return H * W * Cc

    def ingress_channels(self, p: int) -> int:
        """Channels per pixel a client ships at boundary p (the stem input is 3, padded to 8)."""
        return self.input_channels if p == 0 else self.boundary_shape(p)[2]

    def ingress_elems(self, p: int) -> int:
        """Elements of the client's wire tensor at boundary p (the raw image at a s2d stem)."""
        H, W, _, _ = self.boundary_shape(p)
        f = self.tensor_s2d.get(self.boundary[p], 1)
        return H * f * W * f * self.ingress_channels(p)

    def relu_boundary(self, p: int) -> bool:
        """Whether activations at inner boundary p are non-negative (CNN boundaries follow a ReLU /
        pool of ReLU outputs; BERT's hidden state is a LayerNorm output)."""
        return p > 0 and self.model_id != "bert_base"

    def payload_bytes(self, p: int) -> int:
        """fp32 wire bytes at boundary p (what ModelSpec.output_bytes records)."""
        return self.ingress_elems(p) * 4

    def model_spec_doc(self, compute_weight=None) -> dict:
        """A reference ModelSpec JSON document (profiles.py:89-101) for this chain."""
        cw = compute_weight or [f / 1e9 for f in self.unit_flops]
        return {
            "model_id": self.model_id,
            "input_bytes": self.payload_bytes(0),
            "layers": [{"compute_weight": round(float(cw[u]), 6), "output_bytes": self.payload_bytes(u + 1)}
                       for u in range(self.n_units)],
        }


class ChainBuilder:
    """dtype: BF16 (tensor-core path; only the chain output is fp32) or F32 (the fp32 execution
    mode: every tensor and weight fp32, graft_exec.h gx_model_dtype)."""

    def __init__(self, model_id: str, dtype: int = BF16):
        self.c = UnitChain(model_id)
        self.c.dtype = dtype
        self.dtype = dtype
        self._flops = 0.0

    # -- tensors / units --------------------------------------------------
    def tensor(self, H, W, Cc, dtype=None) -> int:
        self.c.tensors.append((H, W, Cc, self.dtype if dtype is None else dtype))
        return len(self.c.tensors) - 1

    def add_weight(self, t) -> int:
        """Weights in the chain's element type (biases and LayerNorm parameters are always fp32)."""
        return self.c.blob.add_f32(t) if self.dtype == F32 else self.c.blob.add_bf16(t)

    def shape(self, t):
        return self.c.tensors[t]

    def begin_unit(self, x: int):
        if self.c.unit_first_op:
            self.c.unit_flops.append(self._flops)
        self._flops = 0.0
        self.c.unit_first_op.append(len(self.c.ops))
        self.c.boundary.append(x)

    def finish(self, out: int) -> UnitChain:
        self.c.unit_flops.append(self._flops)
        self.c.unit_first_op.append(len(self.c.ops))
        self.c.boundary.append(out)
        return self.c

    def s2d_input(self, H, W, Cc, f) -> int:
        """A boundary tensor holding a [H*f, W*f, c] client image in space-to-depth form."""
        t = self.tensor(H, W, Cc)
        self.c.tensor_s2d[t] = f
        return t

    # -- ops ----------------------------------------------------------------
    @staticmethod
    def folded(conv: nn.Conv2d, bn: nn.BatchNorm2d | None):
        """Conv weight/bias with the following BatchNorm folded in (fp32)."""
        w = conv.weight.detach().float()
        b = conv.bias.detach().float() if conv.bias is not None else torch.zeros(w.shape[0])
        if bn is not None:
            scale = bn.weight.detach().float() / torch.sqrt(bn.running_var.detach().float() + bn.eps)
            w = w * scale[:, None, None, None]
            b = (b - bn.running_mean.detach().float()) * scale + bn.bias.detach().float()
        return w, b

    def conv(self, x, conv: nn.Conv2d, bn: nn.BatchNorm2d | None, relu=True, residual=-1, out=-1, out_coff=0,
             cin_pad=None, cout_pad=None):
        w, b = self.folded(conv, bn)
        sh, sw = conv.stride
        ph, pw = conv.padding
        return self.conv_w(x, w, b, (sh, sw), (ph, pw, ph, pw), relu, residual, out, out_coff, cin_pad,
                           cout_pad=cout_pad)

    def conv_w(self, x, w, b, stride, pad, relu=True, residual=-1, out=-1, out_coff=0, cin_pad=None, flops=None,
               cout_pad=None):
        """Conv from explicit (folded) weights; pad = (top, left, bottom, right).  cout_pad: the output
        tensor (a new one) stores cout_pad >= Cout channels, the extra ones zero (zero weights and
        bias); a conv reading a tensor with more channels than its weights have zero-pads its Cin."""
        H, W, Cx, _ = self.shape(x)
        cout, cin, R, S = w.shape
        sh, sw = stride
        ph, pw, ph_hi, pw_hi = pad
        Ho = (H + ph + ph_hi - R) // sh + 1
        Wo = (W + pw + pw_hi - S) // sw + 1
        logical = flops if flops is not None else 2.0 * Ho * Wo * cout * cin * R * S
        cin_pad = cin_pad or (Cx if Cx > cin else cin)
        assert cin_pad <= Cx, (cin_pad, Cx)
        if cout_pad and cout_pad > cout:
            assert out < 0
            w = torch.nn.functional.pad(w, (0, 0, 0, 0, 0, 0, 0, cout_pad - cout))
            b = torch.nn.functional.pad(b, (0, cout_pad - cout))
            cout = cout_pad
        if out < 0:
            out = self.tensor(Ho, Wo, cout)
        else:
            assert self.shape(out)[:2] == (Ho, Wo), (self.shape(out), Ho, Wo)
        executed = 2.0 * Ho * Wo * cout * cin_pad * R * S
        if executed != logical:
            self.c.op_flops_scale[len(self.c.ops)] = logical / executed
        w_off = self.add_weight(pack_conv_weight(w, cin_pad))
        b_off = self.c.blob.add_f32(b)
        self.c.ops.append(N.make_op(N.GX_OP_CONV, x, out, in2=residual, out_coff=out_coff,
                                    act=N.GX_ACT_RELU if relu else N.GX_ACT_NONE, R=R, S=S, sh=sh, sw=sw, ph=ph,
                                    pw=pw, Cin=cin_pad, Cout=cout, w_off=w_off, b_off=b_off,
                                    ph_hi=ph_hi if ph_hi != ph else -1, pw_hi=pw_hi if pw_hi != pw else -1))
        self._flops += logical
        return out

    def conv_ds(self, t, conv: nn.Conv2d, bn: nn.BatchNorm2d, x, ds_conv: nn.Conv2d, ds_bn: nn.BatchNorm2d,
                relu=True):
        """A bottleneck's expand 1x1 conv and its block's 1x1 downsample as ONE GEMM (GX_OPF_DS): K is
        [t's channels | x's channels at the downsample's stride], weights [W3 | Wds], bias b3 + bds; the
        downsample's output (the residual) is never written or read back."""
        w3, b3 = self.folded(conv, bn)
        wd, bd = self.folded(ds_conv, ds_bn)
        H, W, Ct, _ = self.shape(t)
        Hx, Wx, Cx, _ = self.shape(x)
        stride = ds_conv.stride[0]
        assert conv.kernel_size == (1, 1) and ds_conv.kernel_size == (1, 1) and conv.stride == (1, 1)
        assert (Hx + stride - 1) // stride == H and Ct % 64 == 0 and Cx % 64 == 0
        cout = w3.shape[0]
        out = self.tensor(H, W, cout)
        w = torch.cat([pack_conv_weight(w3), pack_conv_weight(wd)], dim=1)
        w_off = self.add_weight(w)
        b_off = self.c.blob.add_f32(b3 + bd)
        self.c.ops.append(N.make_op(N.GX_OP_CONV, t, out, in2=x, act=N.GX_ACT_RELU if relu else N.GX_ACT_NONE,
                                    Cin=Ct, Cout=cout, w_off=w_off, b_off=b_off, flags=N.GX_OPF_DS,
                                    reserved=stride))
        self._flops += 2.0 * H * W * cout * (Ct + Cx)
        return out

    def s2d_stem(self, conv: nn.Conv2d, bn: nn.BatchNorm2d | None, image_hw: int, relu=True):
        """A 7x7 stride-2 pad-3 stem as the equivalent 4x4 stride-1 conv over the 2x2
        space-to-depth image (channel (dy*2+dx)*3 + c), padding (2, 2, 1, 1).

        Output pixel ho reads image rows 2ho-3 .. 2ho+3; with j = r + 1 that is block row
        ho - 2 + j // 2, sub-row j % 2, so tap r maps to (R' = (r+1) // 2, dy = (r+1) % 2)."""
        w, b = self.folded(conv, bn)
        cout, cin, R, S = w.shape
        assert (R, S) == (7, 7) and conv.stride == (2, 2) and conv.padding == (3, 3)
        w2 = torch.zeros(cout, 16, 4, 4)
        for r in range(7):
            for s in range(7):
                Rp, dy = (r + 1) // 2, (r + 1) % 2
                Sp, dx = (s + 1) // 2, (s + 1) % 2
                for c in range(cin):
                    w2[:, (dy * 2 + dx) * cin + c, Rp, Sp] = w[:, c, r, s]
        x = self.s2d_input(image_hw // 2, image_hw // 2, 16, 2)
        self.begin_unit(x)
        Ho = image_hw // 2
        y = self.conv_w(x, w2, b, (1, 1), (2, 2, 1, 1), relu=relu, flops=2.0 * Ho * Ho * cout * cin * R * S)
        return y

    def pool(self, x, kind: str, k, s, p, out=-1, out_coff=0, count_include_pad=True):
        H, W, Cx, _ = self.shape(x)
        Ho = (H + 2 * p - k) // s + 1
        Wo = (W + 2 * p - k) // s + 1
        if out < 0:
            out = self.tensor(Ho, Wo, Cx)
        self.c.ops.append(N.make_op(N.GX_OP_MAXPOOL if kind == "max" else N.GX_OP_AVGPOOL, x, out, out_coff=out_coff,
                                    R=k, S=k, sh=s, sw=s, ph=p, pw=p, flags=1 if count_include_pad else 0))
        return out

    def gap(self, x):
        H, W, Cx, _ = self.shape(x)
        out = self.tensor(1, 1, Cx)
        self.c.ops.append(N.make_op(N.GX_OP_GAP, x, out))
        return out

    def fc(self, x, lin: nn.Linear, relu=False, out_dtype=None, weight=None):
        H, W, Cx, _ = self.shape(x)
        K = H * W * Cx
        w = (weight if weight is not None else lin.weight).detach().float()
        assert w.shape[1] == K, (w.shape, K)
        out = self.tensor(1, 1, w.shape[0], out_dtype)
        w_off = self.add_weight(w)
        b_off = self.c.blob.add_f32(lin.bias.detach().float())
        self.c.ops.append(N.make_op(N.GX_OP_FC, x, out, act=N.GX_ACT_RELU if relu else N.GX_ACT_NONE, Cin=K,
                                    Cout=w.shape[0], w_off=w_off, b_off=b_off))
        self._flops += 2.0 * K * w.shape[0]
        return out


# ---------------------------------------------------------------------------------------------
# deterministic random-init parameters (the architectures' own initialisers, seeded)
# ---------------------------------------------------------------------------------------------

def _calibrate_bn(model: nn.Module, example: torch.Tensor, seed: int):
    """Give every BatchNorm non-trivial, well-scaled statistics so folding is exercised.

    Running mean/var come from a seeded calibration batch (cumulative averaging), affine
    parameters are redrawn (gamma ~ U(0.5, 1.5), beta ~ N(0, 0.1)).  The BN closing each
    residual branch gets gamma ~ U(0.1, 0.3), as in trained ResNets: at plain random init a
    deep residual stack is chaotic (a 0.4% per-layer perturbation grows to ~10% at the logits
    of ResNet-50), which no finite-precision path could be held to 2e-2 against.
    """
    g = torch.Generator().manual_seed(seed + 7)
    last_bn = set()
    for m in model.modules():
        if hasattr(m, "bn3") and hasattr(m, "conv3"):
            last_bn.add(id(m.bn3))
        elif hasattr(m, "bn2") and hasattr(m, "conv2") and hasattr(m, "downsample"):
            last_bn.add(id(m.bn2))
    for m in model.modules():
        if isinstance(m, nn.BatchNorm2d):
            m.reset_running_stats()
            m.momentum = None
            with torch.no_grad():
                if id(m) in last_bn:
                    m.weight.copy_(torch.rand(m.num_features, generator=g) * 0.2 + 0.1)
                else:
                    m.weight.copy_(torch.rand(m.num_features, generator=g) + 0.5)
                m.bias.copy_(torch.randn(m.num_features, generator=g) * 0.1)
    model.train()
    with torch.no_grad():
        model(example)
    model.eval()


def torch_model(name: str, seed: int = 0) -> nn.Module:
    """The fp32 parameter source for `name` (also what the CPU oracle runs)."""
    import torchvision

    if name == "bert_base":
        from .bert import bert_model

        return bert_model(seed)
    torch.manual_seed(seed)
    if name == "resnet50":
        m = torchvision.models.resnet50(weights=None)
        ex = torch.randn(8, 3, 224, 224, generator=torch.Generator().manual_seed(seed + 1))
    elif name == "resnet18":
        m = torchvision.models.resnet18(weights=None)
        ex = torch.randn(8, 3, 224, 224, generator=torch.Generator().manual_seed(seed + 1))
    elif name == "vgg16":
        m = torchvision.models.vgg16(weights=None)
        ex = None
    elif name == "inception_v3":
        m = torchvision.models.inception_v3(weights=None, aux_logits=False, init_weights=True)
        ex = torch.randn(4, 3, 299, 299, generator=torch.Generator().manual_seed(seed + 1))
    else:
        raise KeyError(f"unknown model {name!r}")
    if ex is not None:
        _calibrate_bn(m, ex, seed)
    m.eval()
    return m


# ---------------------------------------------------------------------------------------------
# chain builders
# ---------------------------------------------------------------------------------------------

def _resnet_chain(name: str, m, dtype=BF16, fuse_downsample: bool | None = None) -> UnitChain:
    """fuse_downsample (default: bf16 chains): each bottleneck's downsample 1x1 is computed inside its
    expand conv's GEMM (GX_OPF_DS) instead of as an op whose output is the residual."""
    b = ChainBuilder(name, dtype)
    fuse = dtype == BF16 if fuse_downsample is None else fuse_downsample
    # boundary 0: the 3-channel 224x224 image, rearranged by the gather into 2x2 space-to-depth
    # blocks (112x112x16) so the 7x7/2 stem runs as a 4x4/1 conv with 32-byte im2col pixels
    y = b.s2d_stem(m.conv1, m.bn1, 224)
    y = b.pool(y, "max", 3, 2, 1)
    for layer in (m.layer1, m.layer2, m.layer3, m.layer4):
        for blk in layer:
            b.begin_unit(y)
            idn = y
            bottleneck = hasattr(blk, "conv3")
            if blk.downsample is not None and not (bottleneck and fuse):
                idn = b.conv(y, blk.downsample[0], blk.downsample[1], relu=False)
            if bottleneck:
                t = b.conv(y, blk.conv1, blk.bn1, relu=True)
                t = b.conv(t, blk.conv2, blk.bn2, relu=True)
                if blk.downsample is not None and fuse:
                    y = b.conv_ds(t, blk.conv3, blk.bn3, y, blk.downsample[0], blk.downsample[1])
                else:
                    y = b.conv(t, blk.conv3, blk.bn3, relu=True, residual=idn)
            else:  # basic block
                t = b.conv(y, blk.conv1, blk.bn1, relu=True)
                y = b.conv(t, blk.conv2, blk.bn2, relu=True, residual=idn)
    b.begin_unit(y)
    p = b.gap(y)
    out = b.fc(p, m.fc, out_dtype=F32)
    return b.finish(out)


def _vgg16_chain(m, dtype=BF16) -> UnitChain:
    b = ChainBuilder("vgg16", dtype)
    x = b.tensor(224, 224, 8)
    y = x
    first = True
    b.begin_unit(x)
    feats = list(m.features)
    i = 0
    while i < len(feats):
        layer = feats[i]
        if isinstance(layer, nn.Conv2d):
            y = b.conv(y, layer, None, relu=True, cin_pad=8 if first else None)
            first = False
            i += 2  # conv + relu
        elif isinstance(layer, nn.MaxPool2d):
            y = b.pool(y, "max", 2, 2, 0)
            i += 1
            if i < len(feats):
                b.begin_unit(y)
        else:
            i += 1
    # classifier: torch flattens NCHW (c, h, w); our activations are NHWC (h, w, c)
    fc1 = m.classifier[0]
    H, W, Cc, _ = b.shape(y)
    w1 = fc1.weight.detach().view(fc1.out_features, Cc, H, W).permute(0, 2, 3, 1).reshape(fc1.out_features, -1)
    b.begin_unit(y)
    y = b.fc(y, fc1, relu=True, weight=w1)
    b.begin_unit(y)
    y = b.fc(y, m.classifier[3], relu=True)
    b.begin_unit(y)
    y = b.fc(y, m.classifier[6], out_dtype=F32)
    return b.finish(y)


def _basic(b, x, bc, out=-1, out_coff=0):
    return b.conv(x, bc.conv, bc.bn, relu=True, out=out, out_coff=out_coff)


def _mid(b, x, bc):
    """A conv whose output only feeds the next conv of its branch (Inception's 48 / 96 / 160-channel
    intermediates): in the bf16 chain it is stored with its channels zero-padded to a multiple of 64,
    so the consumer's im2col TMA moves 128-byte pixel rows (64 channels per row) instead of 32 / 64-
    byte rows of 16 / 32 channels (the TMA row rate, not the tensor pipe, bounded those convs at
    0.18-0.29 of the budget-scaled peak), and 3x3/s1/p1 consumers qualify for the halo kernel.  The
    padding channels are exact zeros (zero weights and bias, ReLU(0) = 0), so results are unchanged
    up to the consumer's summation order."""
    c = bc.conv.out_channels
    pad = -(-c // 64) * 64 if b.dtype == BF16 and c % 64 else None
    return b.conv(x, bc.conv, bc.bn, relu=True, cout_pad=pad)


def _inception_chain(m, dtype=BF16) -> UnitChain:
    b = ChainBuilder("inception_v3", dtype)
    x = b.tensor(299, 299, 8)
    b.begin_unit(x)
    y = b.conv(x, m.Conv2d_1a_3x3.conv, m.Conv2d_1a_3x3.bn, relu=True, cin_pad=8)
    b.begin_unit(y)
    y = _basic(b, y, m.Conv2d_2a_3x3)
    b.begin_unit(y)
    y = _basic(b, y, m.Conv2d_2b_3x3)
    b.begin_unit(y)
    y = b.pool(y, "max", 3, 2, 0)
    b.begin_unit(y)
    y = _basic(b, y, m.Conv2d_3b_1x1)
    b.begin_unit(y)
    y = _basic(b, y, m.Conv2d_4a_3x3)
    b.begin_unit(y)
    y = b.pool(y, "max", 3, 2, 0)

    def cat(H, W, Cc):
        return b.tensor(H, W, Cc)

    for blk in (m.Mixed_5b, m.Mixed_5c, m.Mixed_5d):  # InceptionA
        b.begin_unit(y)
        H, W, _, _ = b.shape(y)
        pf = blk.branch_pool.conv.out_channels
        out = cat(H, W, 64 + 64 + 96 + pf)
        _basic(b, y, blk.branch1x1, out, 0)
        t = _mid(b, y, blk.branch5x5_1)
        _basic(b, t, blk.branch5x5_2, out, 64)
        t = _basic(b, y, blk.branch3x3dbl_1)
        t = _mid(b, t, blk.branch3x3dbl_2)
        _basic(b, t, blk.branch3x3dbl_3, out, 128)
        t = b.pool(y, "avg", 3, 1, 1)
        _basic(b, t, blk.branch_pool, out, 224)
        y = out
    blk = m.Mixed_6a  # InceptionB
    b.begin_unit(y)
    H, W, Cc, _ = b.shape(y)
    Ho, Wo = (H - 3) // 2 + 1, (W - 3) // 2 + 1
    out = cat(Ho, Wo, 384 + 96 + Cc)
    _basic(b, y, blk.branch3x3, out, 0)
    t = _basic(b, y, blk.branch3x3dbl_1)
    t = _mid(b, t, blk.branch3x3dbl_2)
    _basic(b, t, blk.branch3x3dbl_3, out, 384)
    b.pool(y, "max", 3, 2, 0, out=out, out_coff=480)
    y = out
    for blk in (m.Mixed_6b, m.Mixed_6c, m.Mixed_6d, m.Mixed_6e):  # InceptionC
        b.begin_unit(y)
        H, W, _, _ = b.shape(y)
        out = cat(H, W, 768)
        _basic(b, y, blk.branch1x1, out, 0)
        t = _mid(b, y, blk.branch7x7_1)
        t = _mid(b, t, blk.branch7x7_2)
        _basic(b, t, blk.branch7x7_3, out, 192)
        t = _mid(b, y, blk.branch7x7dbl_1)
        t = _mid(b, t, blk.branch7x7dbl_2)
        t = _mid(b, t, blk.branch7x7dbl_3)
        t = _mid(b, t, blk.branch7x7dbl_4)
        _basic(b, t, blk.branch7x7dbl_5, out, 384)
        t = b.pool(y, "avg", 3, 1, 1)
        _basic(b, t, blk.branch_pool, out, 576)
        y = out
    blk = m.Mixed_7a  # InceptionD
    b.begin_unit(y)
    H, W, Cc, _ = b.shape(y)
    Ho, Wo = (H - 3) // 2 + 1, (W - 3) // 2 + 1
    out = cat(Ho, Wo, 320 + 192 + Cc)
    t = _basic(b, y, blk.branch3x3_1)
    _basic(b, t, blk.branch3x3_2, out, 0)
    t = _basic(b, y, blk.branch7x7x3_1)
    t = _basic(b, t, blk.branch7x7x3_2)
    t = _basic(b, t, blk.branch7x7x3_3)
    _basic(b, t, blk.branch7x7x3_4, out, 320)
    b.pool(y, "max", 3, 2, 0, out=out, out_coff=512)
    y = out
    for blk in (m.Mixed_7b, m.Mixed_7c):  # InceptionE
        b.begin_unit(y)
        H, W, _, _ = b.shape(y)
        out = cat(H, W, 2048)
        _basic(b, y, blk.branch1x1, out, 0)
        t = _basic(b, y, blk.branch3x3_1)
        _basic(b, t, blk.branch3x3_2a, out, 320)
        _basic(b, t, blk.branch3x3_2b, out, 704)
        t = _basic(b, y, blk.branch3x3dbl_1)
        t = _basic(b, t, blk.branch3x3dbl_2)
        _basic(b, t, blk.branch3x3dbl_3a, out, 1088)
        _basic(b, t, blk.branch3x3dbl_3b, out, 1472)
        t = b.pool(y, "avg", 3, 1, 1)
        _basic(b, t, blk.branch_pool, out, 1856)
        y = out
    b.begin_unit(y)
    p = b.gap(y)
    out = b.fc(p, m.fc, out_dtype=F32)
    return b.finish(out)


def build_chain(name: str, seed: int = 0, module: nn.Module | None = None, dtype: int = BF16,
                fuse_downsample: bool | None = None) -> UnitChain:
    """The unit chain of `name` with its parameters; dtype F32 builds the fp32 execution mode (same
    units, boundaries and weights, every tensor fp32).  fuse_downsample: ResNet bottlenecks compute
    the downsample inside the expand GEMM (default for bf16 chains; the span kernel and the fp32
    kernels take the unfused form)."""
    m = module if module is not None else torch_model(name, seed)
    if name in ("resnet50", "resnet18"):
        return _resnet_chain(name, m, dtype, fuse_downsample)
    if name == "vgg16":
        return _vgg16_chain(m, dtype)
    if name == "inception_v3":
        return _inception_chain(m, dtype)
    if name == "bert_base":
        from .bert import bert_chain

        return bert_chain(m, dtype=dtype)
    raise KeyError(f"unknown model {name!r}")


MODELS = ("resnet18", "resnet50", "vgg16", "inception_v3", "bert_base")
