"""fp32 CPU forward of unit spans — the numerics oracle (test infrastructure only).

Unit boundaries follow paper_2312_10636_b200/models.py exactly: boundary p is the input of unit
p.  Each function takes / returns the torch (NCHW or [S, H]) layout the architecture defines.
"""
from __future__ import annotations

import torch
import torch.nn as nn
import torch.nn.functional as F


def resnet_units(m) -> list:
    units = [lambda x: m.maxpool(m.relu(m.bn1(m.conv1(x))))]
    for layer in (m.layer1, m.layer2, m.layer3, m.layer4):
        for blk in layer:
            units.append(blk)
    units.append(lambda x: m.fc(torch.flatten(m.avgpool(x), 1)))
    return units


def vgg16_units(m) -> list:
    feats = list(m.features)
    units, cur = [], []
    for layer in feats:
        cur.append(layer)
        if isinstance(layer, nn.MaxPool2d):
            units.append(nn.Sequential(*cur))
            cur = []
    c = m.classifier
    units.append(lambda x: F.relu(c[0](torch.flatten(m.avgpool(x), 1))))
    units.append(lambda x: F.relu(c[3](x)))
    units.append(lambda x: c[6](x))
    return units


def inception_units(m) -> list:
    return [m.Conv2d_1a_3x3, m.Conv2d_2a_3x3, m.Conv2d_2b_3x3, m.maxpool1, m.Conv2d_3b_1x1, m.Conv2d_4a_3x3,
            m.maxpool2, m.Mixed_5b, m.Mixed_5c, m.Mixed_5d, m.Mixed_6a, m.Mixed_6b, m.Mixed_6c, m.Mixed_6d,
            m.Mixed_6e, m.Mixed_7a, m.Mixed_7b, m.Mixed_7c,
            lambda x: m.fc(torch.flatten(m.avgpool(x), 1))]


def bert_units(m) -> list:
    """Unit u = encoder layer u on [k, S, hidden] (transformers BertLayer, no attention mask:
    the reference's profiled BERT runs full 128-token sequences); unit 0 starts
    from the token ids [k, S] through BertEmbeddings (token types 0, positions 0..S-1)."""
    out = []
    for i, layer in enumerate(m.encoder.layer):
        def f(x, layer=layer, first=i == 0):
            if first:
                x = m.embeddings(input_ids=x.long())
            r = layer(x)
            return r[0] if isinstance(r, tuple) else r
        out.append(f)
    return out


def bert_token_ids(n: int, seed: int, vocab: int = 30522, seq: int = 128) -> torch.Tensor:
    """A BERT client's input at boundary 0: token ids randint(0, 30522, (n, 128)) (SURVEY §8 inputs)."""
    return torch.randint(0, vocab, (n, seq), generator=torch.Generator().manual_seed(seed), dtype=torch.int32)


def units_for(name: str, m) -> list:
    if name in ("resnet50", "resnet18"):
        return resnet_units(m)
    if name == "vgg16":
        return vgg16_units(m)
    if name == "inception_v3":
        return inception_units(m)
    if name == "bert_base":
        return bert_units(m)
    raise KeyError(name)


@torch.no_grad()
def run_span(units: list, start: int, end: int, x: torch.Tensor) -> torch.Tensor:
    """fp32 forward of units [start, end) on a batch x (torch layout)."""
    for u in range(start, end):
        x = units[u](x)
    return x


def nchw_to_nhwc(x: torch.Tensor) -> torch.Tensor:
    return x.permute(0, 2, 3, 1).contiguous() if x.dim() == 4 else x


def nhwc_to_nchw(x: torch.Tensor) -> torch.Tensor:
    return x.permute(0, 3, 1, 2).contiguous() if x.dim() == 4 else x
