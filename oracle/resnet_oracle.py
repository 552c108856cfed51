"""TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

torch-CPU restatement of ``client_execute`` (fedsim/trainer.py:427-477) for
the ResNet-18 (GroupNorm) of BASELINE config 4.  The reference has no
ResNet, so this oracle is restatement-pinned: it reuses the LR oracle's
bit-exact minibatch orders (fedsim_oracle.minibatch_orders) and follows the
local loop exactly -- per-epoch permutation, partial last batch kept, mean
cross-entropy per batch, ``w -= lr * g`` (FedAvg), steps = E * ceil(n / bs).

Model (CIFAR variant, models.py resnet_spec): conv3x3(3->64)-GN-relu, four
stages of two BasicBlocks (64, 128, 256, 512 planes; stride 2 and a
conv1x1-GN shortcut entering stages 2-4), global average pool, fc(512->C).
GroupNorm has 2 groups, eps 1e-5.  Inputs are 3072 features read as a
32x32x3 NHWC image; conv weights are stored [co][kh][kw][ci].
"""

from __future__ import annotations

import numpy as np
import torch
import torch.nn.functional as F

from .cnn_oracle import _RoundGrad, _RoundValue
from .fedsim_oracle import minibatch_orders

GN_GROUPS, GN_EPS = 2, 1e-5


def layout(n_classes: int = 10):
    """[(name, shape)] in flat order -- must equal models.resnet_spec."""
    out = [("conv1_w", (64, 3, 3, 3)), ("gn1_w", (64,)), ("gn1_b", (64,))]
    cin = 64
    for li, planes in enumerate((64, 128, 256, 512), start=1):
        for bi in range(2):
            p = f"l{li}.{bi}."
            out += [(p + "conv1_w", (planes, 3, 3, cin)), (p + "gn1_w", (planes,)), (p + "gn1_b", (planes,)),
                    (p + "conv2_w", (planes, 3, 3, planes)), (p + "gn2_w", (planes,)),
                    (p + "gn2_b", (planes,))]
            if bi == 0 and li > 1:
                out += [(p + "down_w", (planes, 1, 1, cin)), (p + "down_gn_w", (planes,)),
                        (p + "down_gn_b", (planes,))]
            cin = planes
    out += [("fc_w", (n_classes, 512)), ("fc_b", (n_classes,))]
    return out


def unflatten(flat, n_classes: int = 10, dtype=torch.float64) -> dict:
    flat = torch.as_tensor(np.asarray(flat), dtype=dtype)
    out, pos = {}, 0
    for name, shp in layout(n_classes):
        size = int(np.prod(shp))
        out[name] = flat[pos:pos + size].reshape(shp).clone()
        pos += size
    assert pos == flat.numel()
    return out


def flatten(params: dict, n_classes: int = 10) -> np.ndarray:
    return torch.cat([params[n].detach().reshape(-1) for n, _ in layout(n_classes)]).numpy()


def _conv(x, w, stride, emulate):
    wt = w.permute(0, 3, 1, 2)
    pad = (w.shape[1] - 1) // 2
    if emulate:
        return _RoundGrad.apply(F.conv2d(_RoundValue.apply(x), _RoundValue.apply(wt), stride=stride, padding=pad))
    return F.conv2d(x, wt, stride=stride, padding=pad)


def _gn(z, g, b):
    return F.group_norm(z, GN_GROUPS, g, b, GN_EPS)


def _act(x, emulate):
    """Activations the device keeps in bf16 (conv inputs / residuals)."""
    return _RoundValue.apply(x) if emulate else x


def forward(p: dict, x: torch.Tensor, emulate_bf16: bool = False) -> torch.Tensor:
    """x [B, 3072] -> logits.  emulate_bf16 rounds exactly what the device
    stores as bf16: the input image, every activation (conv inputs and the
    residual stream), conv weights, and dL/dz at every conv output."""
    e = emulate_bf16
    h = x.reshape(-1, 32, 32, 3).permute(0, 3, 1, 2)
    h = _act(h, e)
    h = _act(F.relu(_gn(_conv(h, p["conv1_w"], 1, e), p["gn1_w"], p["gn1_b"])), e)
    for li in range(1, 5):
        for bi in range(2):
            q = f"l{li}.{bi}."
            stride = 2 if (bi == 0 and li > 1) else 1
            u = _act(F.relu(_gn(_conv(h, p[q + "conv1_w"], stride, e), p[q + "gn1_w"], p[q + "gn1_b"])), e)
            v = _gn(_conv(u, p[q + "conv2_w"], 1, e), p[q + "gn2_w"], p[q + "gn2_b"])
            sc = h
            if q + "down_w" in p:
                sc = _gn(_conv(h, p[q + "down_w"], stride, e), p[q + "down_gn_w"], p[q + "down_gn_b"])
            h = _act(F.relu(v + sc), e)
    pooled = h.mean(dim=(2, 3))
    return pooled @ p["fc_w"].t() + p["fc_b"]


def step(flat, X, y, lr: float, n_classes: int = 10, emulate_bf16: bool = False, dtype=torch.float64):
    """One SGD step on a batch: (new flat params, loss)."""
    p = {k: v.requires_grad_(True) for k, v in unflatten(flat, n_classes, dtype).items()}
    loss = F.cross_entropy(forward(p, torch.as_tensor(np.asarray(X), dtype=dtype), emulate_bf16),
                           torch.as_tensor(np.asarray(y), dtype=torch.long))
    names = [n for n, _ in layout(n_classes)]
    grads = torch.autograd.grad(loss, [p[n] for n in names])
    new = torch.cat([(p[n] - lr * g).detach().reshape(-1) for n, g in zip(names, grads)]).numpy()
    return new, float(loss.detach())


def client_train(flat_w0, X: np.ndarray, y: np.ndarray, client_id: int, seed: int, rnd: int,
                 epochs: int, batch_size: int, lr: float, n_classes: int = 10,
                 emulate_bf16: bool = False, dtype=torch.float64):
    """Returns (flat end parameters, steps, mean per-step loss)."""
    w = np.asarray(flat_w0, dtype=np.float64)
    n = len(y)
    bs = n if batch_size <= 0 else min(batch_size, n)
    steps, loss_sum = 0, 0.0
    for order in minibatch_orders(seed, client_id, rnd, n, epochs):
        for lo in range(0, n, bs):
            idx = order[lo:lo + bs]
            w, loss = step(w, X[idx], y[idx], lr, n_classes, emulate_bf16, dtype)
            loss_sum += loss
            steps += 1
    return w, steps, loss_sum / steps


def evaluate(flat, X: np.ndarray, y: np.ndarray, n_classes: int = 10, dtype=torch.float64):
    p = unflatten(flat, n_classes, dtype)
    with torch.no_grad():
        z = forward(p, torch.as_tensor(np.asarray(X), dtype=dtype))
        yt = torch.as_tensor(np.asarray(y), dtype=torch.long)
        return float((z.argmax(1) == yt).double().mean()), float(F.cross_entropy(z, yt))


def fedavg_round(flat_global, data: dict, selected, seed: int, rnd: int, epochs: int,
                 batch_size: int, lr: float, n_classes: int = 10, emulate_bf16: bool = False):
    """One SP FedAvg round: every selected client trains from the global
    model, the server adopts the sample-weighted average."""
    acc = np.zeros_like(np.asarray(flat_global, dtype=np.float64))
    wsum = 0.0
    for m in selected:
        X, y = data[m]
        w, _, _ = client_train(flat_global, X, y, m, seed, rnd, epochs, batch_size, lr, n_classes,
                               emulate_bf16)
        acc += len(y) * w
        wsum += len(y)
    return acc / wsum
