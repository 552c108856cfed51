"""A CPU stand-in for the device layer, for multi-process (gloo) tests of the
round plumbing on a machine without a GPU.

``install()`` swaps the native kernels the host logic calls (fold, group
fold, lincomb, delta_affine, state gather/scatter) for torch CPU
equivalents and replaces batched training by a deterministic mock update
that depends on the client, the round, the start model and the client's
state.  Everything else -- selection, fits, schedule, device ownership, the
packed all-reduce, the owner-sharded state exchange, server rules, the state
store's bookkeeping -- is the product code under test.  Test infrastructure
only: nothing in the package imports it.
"""

from __future__ import annotations

import numpy as np
import torch

CPU = torch.device("cpu")


def _fold(acc, x, w):
    acc.add_(x.reshape(acc.shape), alpha=float(w))


def _fold_group(acc, xs, order, w):
    rows = range(xs.size(0)) if order is None else order.tolist()
    for j, r in enumerate(rows):
        acc.add_(xs[r].reshape(acc.shape), alpha=1.0 if w is None else float(w[j]))


def _lincomb(out, x, a=1.0, y=None, b=0.0, z=None, c=0.0):
    res = torch.zeros_like(out) if x is None else a * x.reshape(out.shape)
    if y is not None:
        res = res + b * y.reshape(out.shape)
    if z is not None:
        res = res + c * z.reshape(out.shape)
    out.copy_(res)
    return out


def _delta_affine(out, a, base, s, cvec=None, c=0.0, dmat=None, d=0.0):
    res = s.view(-1, 1) * (a - base.view(1, -1))
    if cvec is not None:
        res = res + c * cvec.view(1, -1)
    if dmat is not None:
        res = res + d * dmat
    out.copy_(res)
    return out


def _state_gather(work, store, slot):
    for j, s in enumerate(slot.tolist()):
        work[j].copy_(store[s] if s >= 0 else torch.zeros_like(work[j]))


def _state_scatter(store, work, slot):
    for j, s in enumerate(slot.tolist()):
        store[s].copy_(work[j])


def mock_train_group(plugin, spec, data, clients, w0, global_bundle, state_work, epochs,
                     batch_size, lr, seed, round_num, inputs=None, defer_fc1=False,
                     defer_check=False, timing=False):
    """A deterministic stand-in for a batched local run: client m's end
    model is w0 + 0.01*sin(1.7 m + 0.3 r + 0.1 i) - 0.05 * c_m."""
    from paper_2303_01778_b200.trainer import GroupOutcome
    clients = [int(c) for c in clients]
    n = data.sizes[clients].astype(np.int64)
    bs = n if batch_size <= 0 else np.minimum(batch_size, n)
    steps = (epochs * ((n + bs - 1) // bs)).astype(np.int64)
    i = torch.arange(spec.numel, dtype=torch.float64)
    rows = [0.01 * torch.sin(1.7 * m + 0.3 * round_num + 0.1 * i) for m in clients]
    w_out = (w0.double().view(1, -1) + torch.stack(rows)).float()
    if state_work is not None:
        w_out -= 0.05 * state_work
    return GroupOutcome(clients, n, steps, 0.1 * np.asarray(clients, dtype=np.float64), w_out, 1e-3)


def install() -> None:
    from paper_2303_01778_b200 import _kernels as K, aggregate, engine, trainer
    trainer.device = lambda: CPU
    engine.device = lambda: CPU
    K.fold, K.fold_group, K.lincomb = _fold, _fold_group, _lincomb
    K.delta_affine, K.state_gather, K.state_scatter = _delta_affine, _state_gather, _state_scatter
    aggregate.h2d = lambda a, d: torch.from_numpy(np.ascontiguousarray(a)).to(d)
    engine.train_group = mock_train_group
    engine.DeviceRuntime.prepare = lambda self, assignments, round_num: None
