"""BERT-base as a unit chain (BASELINE.json configs[4]): 12 units = 12 encoder layers, unit 0
preceded by the embeddings ("N = 12 (+embed)").

Boundary 0 is the input: the request's 128 token ids (int32, 512 B on the wire); unit 0 starts
with the K8 embedding op (word + position + token-type 0, LayerNorm) that turns them into the
hidden state.  Boundary p >= 1 is the hidden state entering layer p, [S=128, hidden=768] per
request (393,216 B fp32 on the wire).  Per layer:
  QKV (fused 768 -> 2304)  -> attention (12 heads x 64, online softmax)
  -> output dense + residual -> LayerNorm -> FFN1 + GELU -> FFN2 + residual -> LayerNorm
The linears run on the tcgen05 GEMM path; the pre-LN residual adds are fused into the linear
epilogues.  Parameters come from transformers' BertModel(BertConfig()) (seeded, random init).
"""
from __future__ import annotations

import torch

from . import _native as N
from .device import pack_conv_weight
from .models import ChainBuilder, UnitChain


def _linear(b: ChainBuilder, x, weight, bias, act=N.GX_ACT_NONE, residual=-1):
    S, W, K, _ = b.shape(x)
    n_out = weight.shape[0]
    out = b.tensor(S, W, n_out)
    w_off = b.add_weight(pack_conv_weight(weight.detach().float().view(n_out, K, 1, 1)))
    b_off = b.c.blob.add_f32(bias.detach().float())
    b.c.ops.append(N.make_op(N.GX_OP_LINEAR, x, out, in2=residual, act=act, Cin=K, Cout=n_out, w_off=w_off,
                             b_off=b_off))
    b._flops += 2.0 * S * W * n_out * K
    return out


def _layernorm(b: ChainBuilder, x, ln):
    S, W, C, _ = b.shape(x)
    out = b.tensor(S, W, C)
    g_off = b.c.blob.add_f32(ln.weight.detach().float())
    be_off = b.c.blob.add_f32(ln.bias.detach().float())
    b.c.ops.append(N.make_op(N.GX_OP_LAYERNORM, x, out, w_off=g_off, b_off=be_off, eps=float(ln.eps)))
    return out


def _attention(b: ChainBuilder, qkv, heads: int):
    S, W, C3, _ = b.shape(qkv)
    hidden = C3 // 3
    out = b.tensor(S, W, hidden)
    b.c.ops.append(N.make_op(N.GX_OP_ATTENTION, qkv, out, heads=heads, Cout=hidden))
    b._flops += 4.0 * S * S * hidden
    return out


def _embed(b: ChainBuilder, ids, emb, hidden: int):
    """K8: LayerNorm(word[id] + token_type[0] + position[s]) (transformers BertEmbeddings with the
    default all-zero token types and absolute positions 0..S-1)."""
    S = b.shape(ids)[0]
    out = b.tensor(S, 1, hidden)
    w_off = b.add_weight(emb.word_embeddings.weight)
    p_off = b.add_weight(emb.position_embeddings.weight)
    t_off = b.add_weight(emb.token_type_embeddings.weight)
    ln = emb.LayerNorm
    g_off = b.c.blob.add_f32(torch.cat([ln.weight.detach().float(), ln.bias.detach().float()]))
    b.c.ops.append(N.make_op(N.GX_OP_EMBED, ids, out, Cin=emb.word_embeddings.weight.shape[0], Cout=hidden,
                             R=emb.position_embeddings.weight.shape[0], w_off=w_off, b_off=g_off, w2_off=p_off,
                             w3_off=t_off, eps=float(ln.eps)))
    b._flops += 10.0 * S * hidden
    return out


def bert_chain(m, seq_len: int = 128, dtype: int = N.GX_BF16) -> UnitChain:
    cfg = m.config
    hidden = cfg.hidden_size
    b = ChainBuilder("bert_base", dtype)
    b.c.input_channels = 1  # boundary 0: one int32 token id per position
    ids = b.tensor(seq_len, 1, 1, dtype=N.GX_I32)
    x = None
    for li, layer in enumerate(m.encoder.layer):
        if li == 0:
            b.begin_unit(ids)
            x = _embed(b, ids, m.embeddings, hidden)
        else:
            b.begin_unit(x)
        att = layer.attention
        sa = att.self
        w = torch.cat([sa.query.weight, sa.key.weight, sa.value.weight], 0)
        bias = torch.cat([sa.query.bias, sa.key.bias, sa.value.bias], 0)
        qkv = _linear(b, x, w, bias)
        ctx = _attention(b, qkv, cfg.num_attention_heads)
        h = _linear(b, ctx, att.output.dense.weight, att.output.dense.bias, residual=x)
        h = _layernorm(b, h, att.output.LayerNorm)
        f = _linear(b, h, layer.intermediate.dense.weight, layer.intermediate.dense.bias, act=N.GX_ACT_GELU)
        f = _linear(b, f, layer.output.dense.weight, layer.output.dense.bias, residual=h)
        x = _layernorm(b, f, layer.output.LayerNorm)
    return b.finish(x)


def bert_model(seed: int = 0):
    from transformers import BertConfig, BertModel

    torch.manual_seed(seed)
    return BertModel(BertConfig(), add_pooling_layer=False).eval()
