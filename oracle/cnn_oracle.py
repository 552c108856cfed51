"""TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

torch-CPU restatement of ``client_execute`` (fedsim/trainer.py:427-477) for
the 2-layer FEMNIST CNN of BASELINE config 2.  The reference has no CNN, so
this oracle is restatement-pinned: it reuses the LR oracle's bit-exact
minibatch orders (fedsim_oracle.minibatch_orders, pinned to the reference's
own permutations) and follows the loop exactly -- per-epoch permutation,
partial last batch kept, mean cross-entropy per batch, ``w -= lr * g`` with
the plain gradient (FedAvg), steps = E * ceil(n / bs), result weight = N_m.
The flat parameter layout is the product's (models.py cnn_spec, NHWC
conv weights and NHWC flatten order for fc1); this module converts.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.nn.functional as F

from .fedsim_oracle import minibatch_orders

NAMES = ("conv1_w", "conv1_b", "conv2_w", "conv2_b", "fc1_w", "fc1_b", "fc2_w", "fc2_b")


def shapes(n_classes: int):
    return ((32, 5, 5, 1), (32,), (64, 5, 5, 32), (64,), (512, 3136), (512,), (n_classes, 512),
            (n_classes,))


def unflatten(flat, n_classes: int, dtype=torch.float64) -> list[torch.Tensor]:
    flat = torch.as_tensor(np.asarray(flat), dtype=dtype)
    out, pos = [], 0
    for shp in shapes(n_classes):
        size = int(np.prod(shp))
        out.append(flat[pos:pos + size].reshape(shp).clone())
        pos += size
    return out


def flatten(params) -> np.ndarray:
    return torch.cat([p.detach().reshape(-1) for p in params]).numpy()


class _RoundValue(torch.autograd.Function):
    """bf16-round the value, pass the gradient through (device operand staging)."""

    @staticmethod
    def forward(ctx, x):
        return x.to(torch.bfloat16).to(x.dtype)

    @staticmethod
    def backward(ctx, g):
        return g


class _RoundGrad(torch.autograd.Function):
    """Identity forward; bf16-round the incoming gradient (the device stages
    dL/dz2 as bf16 for the conv2 dgrad and wgrad tensor-core GEMMs)."""

    @staticmethod
    def forward(ctx, x):
        return x.view_as(x)

    @staticmethod
    def backward(ctx, g):
        return g.to(torch.bfloat16).to(g.dtype)


class _Conv1Bf16(torch.autograd.Function):
    """conv1 as the device computes it (csrc/cnn.cu k_fwd): bf16 image and
    weights on the tensor cores, fp32 accumulation; the weight gradient is
    also a bf16 tensor-core product (k_bwd_conv: bf16 image windows x the
    bf16-rounded pre-pool gradient, which `forward` rounds with _RoundGrad)."""

    @staticmethod
    def forward(ctx, x, w):   # x [B, 1, 28, 28], w NHWC [32, 5, 5, 1]
        ctx.save_for_backward(x, w)
        xr = x.to(torch.bfloat16).to(x.dtype)
        wr = w.to(torch.bfloat16).to(w.dtype).permute(0, 3, 1, 2)
        return F.conv2d(xr, wr, padding=2)

    @staticmethod
    def backward(ctx, g):
        x, w = ctx.saved_tensors
        gw = torch.nn.grad.conv2d_weight(_bf16(x), (w.shape[0], w.shape[3], w.shape[1], w.shape[2]), _bf16(g),
                                         padding=2)
        return None, gw.permute(0, 2, 3, 1)


def _tf32(x: torch.Tensor) -> torch.Tensor:
    """fp32 -> tf32 by truncation (how tcgen05 kind::tf32 reads fp32 operands,
    measured in tests/test_gpu_umma.py)."""
    f = x.to(torch.float32).contiguous()
    return (f.view(torch.int32) & -8192).view(torch.float32).to(x.dtype)


def _bf16(x: torch.Tensor) -> torch.Tensor:
    """round to nearest bf16 (how the low-rank fc1 stores W0, X and dH)."""
    return x.to(torch.bfloat16).to(x.dtype)


def _tf32_rna(x: torch.Tensor) -> torch.Tensor:
    """fp32 -> tf32 rounded to nearest, ties away (cvt.rna.tf32.f32): how the
    low-rank fc1 stores X and dH."""
    f = x.to(torch.float32).contiguous()
    return ((f.view(torch.int32) + 4096) & -8192).view(torch.float32).to(x.dtype)


class _RnaValue(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x):
        return _tf32_rna(x)

    @staticmethod
    def backward(ctx, g):
        return g


class _RnaGrad(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x):
        return x.view_as(x)

    @staticmethod
    def backward(ctx, g):
        return _tf32_rna(g)


class _TruncValue(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x):
        return _tf32(x)

    @staticmethod
    def backward(ctx, g):
        return g


class _TruncGrad(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x):
        return x.view_as(x)

    @staticmethod
    def backward(ctx, g):
        return _tf32(g)


def forward(params, x: torch.Tensor, emulate_bf16: bool = False,
            fc1_base: torch.Tensor | None = None) -> torch.Tensor:
    """x [B, 784] -> logits; conv weights are NHWC ([co, ky, kx, ci]).

    emulate_bf16=True rounds exactly the operands the device feeds to its
    tensor cores -- bf16 for conv1 (the image and W1 in the forward, the image
    and dL/dz1 in its weight gradient), bf16 for conv2 (p1 and W2 in the forward, dL/dz2 in both
    backward GEMMs) and tf32 truncation for fc1 (X and W1 in the forward, dL/dz1
    in both backward GEMMs); everything else stays in the oracle's precision.
    Used to check the kernels' arithmetic separately from the effect of the
    reduced-precision operands on the trajectory.

    fc1_base (with emulate_bf16): the round-start fc1 weights W0 of a device
    run that used the low-rank fc1 (csrc/cnn_lazy.cu), whose tensor cores see
    bf16(W0) plus the client's accumulated update in (near) full precision
    instead of a rounded W_t: the emulated weight is bf16(W0) + (W_t - W0),
    and X and dL/dz1 (fc1 bias gradient included) are rounded to nearest
    bf16, as that path stores them (its Gram corrections carry high + low
    bf16 terms, i.e. are exact to ~2^-17)."""
    c1w, c1b, c2w, c2b, f1w, f1b, f2w, f2b = params
    h = x.reshape(-1, 1, 28, 28)
    if emulate_bf16:
        h = F.max_pool2d(F.relu(_RoundGrad.apply(_Conv1Bf16.apply(h, c1w) + c1b.view(1, -1, 1, 1))), 2)
    else:
        h = F.max_pool2d(F.relu(F.conv2d(h, c1w.permute(0, 3, 1, 2), c1b, padding=2)), 2)
    if emulate_bf16:
        z = F.conv2d(_RoundValue.apply(h), _RoundValue.apply(c2w).permute(0, 3, 1, 2), padding=2)
        h = F.max_pool2d(F.relu(_RoundGrad.apply(z) + c2b.view(1, -1, 1, 1)), 2)
    else:
        h = F.max_pool2d(F.relu(F.conv2d(h, c2w.permute(0, 3, 1, 2), c2b, padding=2)), 2)
    h = h.permute(0, 2, 3, 1).reshape(h.shape[0], -1)  # NHWC flatten
    if emulate_bf16:
        if fc1_base is None:
            h = F.relu(_TruncGrad.apply(_TruncValue.apply(h) @ _TruncValue.apply(f1w).t()) + f1b)
        else:
            w1 = f1w - fc1_base + _bf16(fc1_base)
            h = F.relu(_RoundGrad.apply(_RoundValue.apply(h) @ w1.t() + f1b))
    else:
        h = F.relu(h @ f1w.t() + f1b)
    return h @ f2w.t() + f2b


def decision_margins(params, x: torch.Tensor, fc1_base: torch.Tensor | None = None) -> dict:
    """How close one step's discrete decisions sit to flipping, under the
    emulating forward (emulate_bf16=True): for every ReLU the smallest
    |pre-activation|, for every 2x2 max-pool the smallest gap between the
    window's largest and second-largest input -- each divided by the RMS of
    that layer's pre-activations.  A decision whose margin is below the
    device-vs-oracle arithmetic noise (fp32 accumulation in another order,
    ~1e-6 relative) can legitimately go the other way on the device; a step
    without such a decision cannot flip anything, so its update must match
    tightly (tests/test_gpu_c2_headline.py)."""
    c1w, c1b, c2w, c2b, f1w, f1b, f2w, f2b = [p.detach() for p in params]

    def rms(z):
        return float(z.pow(2).mean().sqrt()) or 1.0

    def pool_gap(a, z):
        """[B, C, H, W] relu outputs -> smallest top1 - top2 over the 2x2
        windows with two positive candidates (a window with at most one
        positive input has a fixed argmax unless that input crosses zero,
        which the ReLU margin covers; zeros tie harmlessly)."""
        w = a.unfold(2, 2, 2).unfold(3, 2, 2).reshape(*a.shape[:2], a.shape[2] // 2, a.shape[3] // 2, 4)
        top = w.topk(2, dim=-1).values
        gap = torch.where(top[..., 1] > 0, top[..., 0] - top[..., 1], torch.full_like(top[..., 0], np.inf))
        return float(gap.min()) / rms(z)

    out = {}
    with torch.no_grad():
        h = x.reshape(-1, 1, 28, 28)
        z1 = F.conv2d(_RoundValue.apply(h), _RoundValue.apply(c1w).permute(0, 3, 1, 2), c1b, padding=2)
        out["relu1"] = float(z1.abs().min()) / rms(z1)
        a1 = F.relu(z1)
        out["pool1"] = pool_gap(a1, z1)
        h = F.max_pool2d(a1, 2)
        z2 = F.conv2d(_RoundValue.apply(h), _RoundValue.apply(c2w).permute(0, 3, 1, 2), padding=2) \
            + c2b.view(1, -1, 1, 1)
        out["relu2"] = float(z2.abs().min()) / rms(z2)
        a2 = F.relu(z2)
        out["pool2"] = pool_gap(a2, z2)
        h = F.max_pool2d(a2, 2).permute(0, 2, 3, 1).reshape(a2.shape[0], -1)
        if fc1_base is None:
            z3 = _tf32(h) @ _tf32(f1w).t() + f1b
        else:
            z3 = _bf16(h) @ (f1w - fc1_base + _bf16(fc1_base)).t() + f1b
        out["relu3"] = float(z3.abs().min()) / rms(z3)
    return out


def client_train(flat_w0, X: np.ndarray, y: np.ndarray, client_id: int, seed: int, rnd: int,
                 epochs: int, batch_size: int, lr: float, n_classes: int,
                 dtype=torch.float64, emulate_bf16: bool = False, mu: float = 0.0):
    """Returns (flat end parameters, steps, mean per-step loss).  mu > 0 adds
    FedProx's proximal gradient mu * (w - w0) (fedsim/trainer.py:249-257)."""
    params = [p.requires_grad_(True) for p in unflatten(flat_w0, n_classes, dtype)]
    anchor = [p.detach().clone() for p in params]
    Xt = torch.as_tensor(np.asarray(X), dtype=dtype)
    yt = torch.as_tensor(np.asarray(y), dtype=torch.long)
    n = len(y)
    bs = n if batch_size <= 0 else min(batch_size, n)
    steps, loss_sum = 0, 0.0
    for order in minibatch_orders(seed, client_id, rnd, n, epochs):
        for lo in range(0, n, bs):
            idx = torch.as_tensor(order[lo:lo + bs])
            loss = F.cross_entropy(forward(params, Xt[idx], emulate_bf16), yt[idx])
            grads = torch.autograd.grad(loss, params)
            with torch.no_grad():
                for p, g, p0 in zip(params, grads, anchor):
                    p -= lr * (g + mu * (p - p0)) if mu else lr * g
            loss_sum += float(loss.detach())
            steps += 1
    return flatten(params), steps, loss_sum / steps


def evaluate(flat, X: np.ndarray, y: np.ndarray, n_classes: int, dtype=torch.float64):
    params = unflatten(flat, n_classes, dtype)
    with torch.no_grad():
        z = forward(params, torch.as_tensor(np.asarray(X), dtype=dtype))
        yt = torch.as_tensor(np.asarray(y), dtype=torch.long)
        acc = float((z.argmax(1) == yt).double().mean())
        loss = float(F.cross_entropy(z, yt))
    return acc, loss


def fedavg_round(flat_global, data: dict, selected, seed: int, rnd: int, epochs: int,
                 batch_size: int, lr: float, n_classes: int, dtype=torch.float64,
                 emulate_bf16: bool = False):
    """One SP FedAvg round (fedsim/engine.py:748-812 semantics): every selected
    client trains from the global model, the server adopts the
    sample-weighted average."""
    acc = np.zeros_like(np.asarray(flat_global, dtype=np.float64))
    wsum = 0.0
    for m in selected:
        X, y = data[m]
        w, _, _ = client_train(flat_global, X, y, m, seed, rnd, epochs, batch_size, lr, n_classes,
                               dtype, emulate_bf16)
        acc += len(y) * np.asarray(w, dtype=np.float64)
        wsum += len(y)
    return acc / wsum
