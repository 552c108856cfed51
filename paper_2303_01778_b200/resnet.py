"""Host side of the ResNet-18 (GroupNorm) path (BASELINE config 4):
workspace management and argument marshalling for ``pb_resnet_train_group``
/ ``pb_resnet_eval`` (csrc/resnet.cu)."""

from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

from ._lib import ResnetTrainArgs, lib, ptr, stream_of
from .cnn import sweep_plan
from .models import ModelSpec

MAX_BATCH = 32


def workspace_sizes(BS: int, C: int) -> tuple[int, int, int, int]:
    """(arena bytes, bf16 row length, wgrad-partial floats, GN-partial floats)
    per slot, from the library's own network plan."""
    out = (ctypes.c_int64 * 4)()
    lib.check(lib.pb_resnet_workspace(BS, C, out))
    return int(out[0]), int(out[1]), int(out[2]), int(out[3])


class _Workspace:
    def __init__(self):
        self.key = None
        self.buf: dict[str, torch.Tensor] = {}

    def get(self, slots: int, BS: int, C: int, device) -> tuple[dict, tuple]:
        sizes = workspace_sizes(BS, C)
        key = (BS, C, device)
        if self.key != key or self.buf["slots"].numel() < slots * 16:
            self.buf = {}
            torch.cuda.empty_cache()
            arena, p16, part, gnp = sizes
            self.buf = {"slots": torch.empty(slots * 16, dtype=torch.uint8, device=device),
                        "w16": torch.empty(slots * p16, dtype=torch.bfloat16, device=device),
                        "arena": torch.empty(slots * arena, dtype=torch.uint8, device=device),
                        "part": torch.empty(slots * part, dtype=torch.float32, device=device),
                        "gnp": torch.empty(slots * gnp, dtype=torch.float32, device=device)}
            self.key = key
        return self.buf, sizes


_WS = _Workspace()


def _fill(a: ResnetTrainArgs, ws: dict, slots: int, BS: int, C: int) -> None:
    a.ws_slots, a.ws_w16, a.ws_arena = ptr(ws["slots"]), ptr(ws["w16"]), ptr(ws["arena"])
    a.ws_part, a.ws_gnp = ptr(ws["part"]), ptr(ws["gnp"])
    a.g, a.BS, a.C = slots, BS, C


def resnet_train_group(data, rows_d, off_d, n: np.ndarray, w0, w_out, loss, steps, bad, *,
                       spec: ModelSpec, epochs: int, batch_size: int, lr: float, terms: dict,
                       state_work=None, timeline=None) -> None:
    """Every client's local SGD run (pb_resnet_train_group); ``terms`` are the
    plugin's fused gradient terms (FedProx mu, SCAFFOLD controls with the
    clients' control rows in ``state_work``), as on the CNN path."""
    G = len(n)
    BS, _, rank, active = sweep_plan(n, batch_size, epochs)
    if BS > MAX_BATCH:
        raise ValueError(f"the ResNet path supports minibatches of up to {MAX_BATCH} samples, got {BS}")
    d = w_out.device
    w_out.copy_(w0.view(1, -1).expand(G, -1))
    loss.zero_()
    steps.zero_()
    bad.fill_(-1)
    rank_d = torch.from_numpy(rank).to(d)
    n_d = torch.from_numpy(n.astype(np.int32)).to(d)
    ws, _ = _WS.get(G, BS, spec.n_classes, d)
    a = ResnetTrainArgs()
    a.X, a.Y, a.order, a.order_off, a.n, a.rank = (ptr(data.X), ptr(data.Y), ptr(rows_d), ptr(off_d),
                                                    ptr(n_d), ptr(rank_d))
    limit = int(os.environ.get("PB_CNN_MAX_SWEEPS", "0"))  # debugging aid (shared with the CNN)
    if limit > 0:
        active = active[:limit].copy()
    a.active = active.ctypes.data
    a.sweeps = len(active)
    a.w, a.w_stride = ptr(w_out), w_out.stride(0)
    a.loss_sum, a.steps, a.bad = ptr(loss), ptr(steps), ptr(bad)
    _fill(a, ws, G, BS, spec.n_classes)
    a.batch_size, a.epochs, a.lr = batch_size, epochs, lr
    a.timeline = ptr(timeline)
    a.w0 = ptr(w0)
    a.mu = terms.get("mu", 0.0)
    a.ctrl_g, a.cg = ptr(terms.get("ctrl_g")), terms.get("cg", 0.0)
    ctrl_c = state_work if terms.get("ctrl_c") else None
    if terms.get("ctrl_c") and ctrl_c is None:
        raise ValueError("SCAFFOLD control terms need the clients' state rows")
    a.ctrl_c, a.ctrl_stride, a.cc = ptr(ctrl_c), (ctrl_c.stride(0) if ctrl_c is not None else 0), \
        terms.get("cc", 0.0)
    lib.check(lib.pb_resnet_train_group(ctypes.byref(a), stream_of(w_out)))


_EVAL_ORDER: dict = {}


def resnet_evaluate(model, X: torch.Tensor, Y: torch.Tensor) -> tuple[float, float]:
    spec = model.spec
    rows = int(Y.numel())
    P = spec.numel
    w = torch.zeros((P + 3) // 4 * 4, device=X.device)
    w[:P] = torch.cat([model.tensors[nm].reshape(-1) for nm in spec.names])
    key = (rows, X.device)
    order = _EVAL_ORDER.get(key)
    if order is None:
        order = torch.arange(rows, dtype=torch.int32, device=X.device)
        _EVAL_ORDER[key] = order
    BS = MAX_BATCH
    slots = min((rows + BS - 1) // BS, 64)
    ws, _ = _WS.get(slots, BS, spec.n_classes, X.device)
    a = ResnetTrainArgs()
    a.X, a.Y, a.order = ptr(X), ptr(Y), ptr(order)
    a.w, a.w_stride = ptr(w), w.numel()
    _fill(a, ws, slots, BS, spec.n_classes)
    a.batch_size, a.epochs = BS, 1
    out = torch.zeros(2, dtype=torch.float64, device=X.device)
    lib.check(lib.pb_resnet_eval(ctypes.byref(a), rows, ptr(out), stream_of(w)))
    correct, loss = out.cpu().tolist()
    return correct / rows, loss / rows
