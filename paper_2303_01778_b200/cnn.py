"""Host side of the CNN path: workspace management and argument marshalling
for ``pb_cnn_train_group`` / ``pb_cnn_eval`` (csrc/cnn.cu)."""

from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

from ._lib import CnnTrainArgs, LazyFoldArgs, h2d, lib, ptr, stream_of
from .models import ModelSpec

# bytes per sample of each workspace buffer (include/parrot_b200.h)
_PER_SAMPLE = {"p1": 4 * 337 * 16, "am1": 6272, "p2": 3136 * 4, "am2": 3136, "h": 512 * 4, "dh": 512 * 4,
               "dp2": 3136 * 4, "dz": 8 * 337 * 16, "dp1": 6272 * 4}
MAX_BATCH = 32


class _Workspace:
    def __init__(self):
        self.slots = 0
        self.bs = 0
        self.buf: dict[str, torch.Tensor] = {}

    def get(self, slots: int, bs: int, device) -> dict[str, torch.Tensor]:
        if slots > self.slots or bs > self.bs or (self.buf and self.buf["slots"].device != device):
            self.buf = {}
            torch.cuda.empty_cache()
            self.slots, self.bs = max(slots, self.slots), max(bs, self.bs)
            n = self.slots * self.bs
            # one plane (5392 B) of slack: the conv kernels' TMA views of
            # the p1 / dz2 planes may read a few rows past the last plane
            self.buf = {k: torch.empty(n * v + 5392, dtype=torch.uint8, device=device)
                        for k, v in _PER_SAMPLE.items()}
            self.buf["slots"] = torch.empty(self.slots * 32, dtype=torch.uint8, device=device)
            self.buf["w2b"] = torch.empty(self.slots * 102400, dtype=torch.uint8, device=device)
            self.buf["dht"] = torch.empty(self.slots * 512 * 32 * 4, dtype=torch.uint8, device=device)
        return self.buf


_WS = _Workspace()


class _LazyWorkspace:
    """Grow-only buffers of the low-rank fc1 (csrc/cnn_lazy.cu): the round's
    (X, dH) history per client plus the per-sweep partials."""

    HISTORY = ("hx", "hd")

    def __init__(self):
        self.buf: dict[str, torch.Tensor] = {}
        # True while the history buffers may hold non-finite values: fresh
        # allocations, or a round whose result read has not confirmed every
        # client finite (GroupOutcome.resolve clears it)
        self.dirty = True

    def _get(self, name: str, numel: int, device, dtype=torch.float32) -> torch.Tensor:
        t = self.buf.get(name)
        if t is None or t.numel() < numel or t.device != device or t.dtype != dtype:
            # 2x headroom: round sizes vary (the longest client sets the
            # history length), and a reallocation synchronises
            self.buf.pop(name, None)
            t = torch.empty(max(int(numel * 2.0), 8), dtype=dtype, device=device)
            self.buf[name] = t
            if name in self.HISTORY:
                self.dirty = True
        return t

    def get(self, rows: int, zp: int, gdt: int, slots: int, device) -> dict[str, torch.Tensor]:
        b16 = torch.bfloat16   # the history and the W0 copies are bf16 tensor-core operands
        out = {"hx": self._get("hx", rows * 3136, device, b16), "hd": self._get("hd", rows * 512, device, b16),
               "w0t": self._get("w0t", 2 * 3136 * 512, device, b16), "zp": self._get("zp", zp, device),
               "gdt": self._get("gdt", gdt, device, b16),
               "fpart": self._get("fpart", max(74, slots) * 512 * 32, device)}
        # The history GEMMs read whole 32-row chunks: rows a client has not
        # written this round are multiplied by exact zeros (dH^T pad columns
        # are zeroed by the head kernels, Gram rows past the live ones are
        # selected to 0), which needs every stale value to be finite.  Stale
        # values are the previous round's (finite) history, so the buffers
        # are only cleared when fresh or after a round with a diverged client.
        if self.dirty:
            for k in self.HISTORY:
                out[k].zero_()
        self.dirty = True   # until this round's result read confirms it
        return out


_LZ = _LazyWorkspace()


def lazy_enabled(terms: dict) -> bool:
    """The low-rank fc1 applies to plain SGD (FedAvg): no proximal or
    control-variate term in the local gradient.  PB_CNN_LAZY=0 forces the
    direct per-client fc1 (A/B testing)."""
    plain = not terms.get("mu") and terms.get("ctrl_g") is None and not terms.get("ctrl_c")
    return plain and os.environ.get("PB_CNN_LAZY", "1") != "0"


def lazy_plan(total: np.ndarray, active: np.ndarray, BS: int):
    """History layout: client row r owns hlen[r] = round_up(steps_r * BS, 64)
    rows from hoff[r] (64 bf16 = one 128-byte operand row of history
    columns); partial-buffer capacities over the sweeps (the Gram rows hold
    a high and a low bf16 term: 64 rows per slot)."""
    hlen = ((total * BS + 63) // 64 * 64).astype(np.int32)
    hoff = np.zeros(len(total), dtype=np.int64)
    if len(total) > 1:
        hoff[1:] = np.cumsum(hlen[:-1], dtype=np.int64)
    njt = (np.arange(len(active)) * BS + 127) // 128
    cap = int((active.astype(np.int64) * njt).max()) if len(active) else 0
    return hlen, hoff, int(hlen.sum()), cap * 512 * 32, cap * 64 * 128


class LazyFc1:
    """Deferred fc1 of a low-rank CNN round (csrc/cnn_lazy.cu): the clients'
    fc1_w end weights W0 - lr * HD_j^T HX_j are never written; a device
    partial folds them straight from the round's history with
    pb_cnn_lazy_fold (aggregate.fold_group).  Valid until the next CNN group
    reuses the history workspace."""

    entry = "fc1_w"
    SPLITS = 32

    def __init__(self, lz: dict, hoff: np.ndarray, hlen: np.ndarray, rows: int, BS: int, lr: float,
                 w0: torch.Tensor, switch: int = 0):
        self.lz, self.hoff, self.hlen, self.rows, self.BS, self.lr, self.w0 = lz, hoff, hlen, rows, BS, lr, w0
        self.switch = switch   # clients with more steps left the low-rank form (w rows hold fc1)
        self.steps = None

    def set_steps(self, steps: np.ndarray) -> None:
        self.steps = np.asarray(steps, dtype=np.int64)

    def fold(self, acc: torch.Tensor, rows: list[int], weights: np.ndarray, mat: torch.Tensor | None = None) -> None:
        """acc += sum_j w_j * fc1_w of client rows `rows` (contiguous); ``mat``
        (the group's fc1_w columns) holds the rows of switched clients."""
        if not rows:
            return
        if rows != list(range(rows[0], rows[0] + len(rows))):
            raise ValueError("lazy fc1 fold needs a contiguous run of group rows")
        d = acc.device
        r = np.asarray(rows)
        weights = np.asarray(weights, dtype=np.float32)
        nr = (self.steps[r] * self.BS).astype(np.int32)
        switched = self.steps[r] > self.switch if self.switch > 0 else np.zeros(len(r), dtype=bool)
        if switched.any():
            if mat is None:
                raise ValueError("switched clients fold from their materialised rows: pass mat")
            from . import _kernels as K
            sel = r[switched]
            K.fold_group(acc, mat, h2d(sel.astype(np.int32), d), h2d(weights[switched], d))
            if switched.all():
                return
            # their history columns (pads included) are scaled to exact zeros
            weights = np.where(switched, np.float32(0.0), weights)
            nr = np.where(switched, self.hlen[r], nr).astype(np.int32)
        lo = int(self.hoff[r[0]])
        hi = int(self.hoff[r[-1]] + self.hlen[r[-1]])
        hoff = h2d(self.hoff[r].astype(np.int64), d)
        nrows = h2d(nr, d)
        w = h2d(weights, d)
        part = _LZ._get("fold_part", self.SPLITS * 512 * 3136, d)
        lo_buf = _LZ._get("hd_lo", self.rows * 512, d, torch.bfloat16)
        f = LazyFoldArgs()
        f.acc, f.w0, f.hx, f.hd = ptr(acc), ptr(self.w0), ptr(self.lz["hx"]), ptr(self.lz["hd"])
        f.hrows, f.row_lo, f.row_hi = self.rows, lo, hi
        f.hoff, f.nrows, f.w, f.nclients = ptr(hoff), ptr(nrows), ptr(w), len(rows)
        f.part, f.splits = ptr(part), self.SPLITS
        f.wsum, f.lr = float(np.sum(weights.astype(np.float64))), self.lr
        f.hd_lo = ptr(lo_buf)
        lib.check(lib.pb_cnn_lazy_fold(ctypes.byref(f), stream_of(acc)))


def lz_switch_step(sweeps: int) -> int:
    """Sweep at which a low-rank round's remaining clients leave the
    low-rank form (0 = never): the history a step re-reads grows with the
    step count (2 x 250 KB per past step at bs 20) while the direct fc1
    streams a fixed 19 MB.  Off by default: measured on the C2 round, the
    direct kernels are slower than the low-rank ones in every sweep they
    would take over (switching at sweep 16 / 24 / 32 / 40 costs +15.9 /
    +7.0 / +3.4 / +2.1 ms per round; tools/sweep_times.py), because the
    sparse tail is latency-bound, not HBM-bound.  PB_LZ_SWITCH=s enables it."""
    s = int(os.environ.get("PB_LZ_SWITCH", "0"))
    return s if 0 < s < sweeps else 0


def _samples_per_cta() -> int:
    return int(os.environ.get("PB_CNN_SPB", "10"))


def _fill(args: CnnTrainArgs, ws: dict, slots: int, BS: int) -> None:
    args.ws_slots = ptr(ws["slots"])
    args.ws_w2b = ptr(ws["w2b"])
    for k in ("p1", "am1", "p2", "am2", "h", "dh", "dp2", "dz", "dp1", "dht"):
        setattr(args, "ws_" + k, ptr(ws[k]))
    args.g = slots
    args.BS = BS
    args.samples_per_cta = _samples_per_cta()


def sweep_plan(n: np.ndarray, batch_size: int, epochs: int):
    """Per-client step counts, slot order (most steps first) and the number
    of clients still stepping in each sweep."""
    bs = n.copy() if batch_size <= 0 else np.minimum(batch_size, n)
    total = epochs * ((n + bs - 1) // bs)
    rank = np.argsort(-total, kind="stable").astype(np.int32)
    sweeps = int(total.max()) if len(total) else 0
    active = np.array([(total > s).sum() for s in range(sweeps)], dtype=np.int32)
    return int(bs.max()) if len(bs) else 0, total, rank, active


def cnn_train_group(data, rows_d, off_d, n: np.ndarray, w0, w_out, loss, steps, bad, *,
                    spec: ModelSpec, epochs: int, batch_size: int, lr: float, terms: dict,
                    state_work, defer_fc1: bool = False, timeline=None) -> "LazyFc1 | None":
    G = len(n)
    BS, total, rank, active = sweep_plan(n, batch_size, epochs)
    if BS > MAX_BATCH:
        raise ValueError(f"the CNN path supports minibatches of up to {MAX_BATCH} samples, got {BS}")
    d = w_out.device
    lazy = lazy_enabled(terms)
    defer = defer_fc1 and lazy
    if defer:  # the fc1_w columns stay unwritten: the fold reads the history
        f_off, f_size = [(o, sz) for nm, o, sz, _ in spec.columns() if nm == "fc1_w"][0]
        w_out[:, :f_off].copy_(w0[:f_off].view(1, -1).expand(G, -1))
        w_out[:, f_off + f_size:].copy_(w0[f_off + f_size:].view(1, -1).expand(G, -1))
    else:
        w_out.copy_(w0.view(1, -1).expand(G, -1))
    loss.zero_()
    steps.zero_()
    bad.fill_(-1)
    rank_d = h2d(rank, d)
    n_d = h2d(n.astype(np.int32), d)
    ws = _WS.get(G, BS, d)
    a = CnnTrainArgs()
    a.X, a.Y, a.order, a.order_off, a.n, a.rank = (ptr(data.X), ptr(data.Y), ptr(rows_d),
                                                    ptr(off_d), ptr(n_d), ptr(rank_d))
    limit = int(os.environ.get("PB_CNN_MAX_SWEEPS", "0"))  # debugging aid
    if limit > 0:
        active = active[:limit].copy()
    a.active = active.ctypes.data
    a.sweeps = len(active)
    a.w, a.w0 = ptr(w_out), ptr(w0)
    a.w_stride = w_out.stride(0)
    a.ctrl_g = ptr(terms.get("ctrl_g"))
    ctrl_c = state_work if terms.get("ctrl_c") else None
    a.ctrl_c = ptr(ctrl_c)
    a.ctrl_stride = ctrl_c.stride(0) if ctrl_c is not None else 0
    a.loss_sum, a.steps, a.bad = ptr(loss), ptr(steps), ptr(bad)
    _fill(a, ws, G, BS)
    handle = None
    if lazy:
        hlen, hoff, rows, zp, gdt = lazy_plan(total, active, BS)
        if limit > 0:
            _LZ.dirty = True   # truncated clients never reach the step that zeroes their pad columns
        lz = _LZ.get(rows, zp, gdt, G, d)
        hlen_d = h2d(hlen, d)
        hoff_d = h2d(hoff, d)
        a.lz_hx, a.lz_hxt, a.lz_hd, a.lz_hdt = ptr(lz["hx"]), None, ptr(lz["hd"]), None
        a.lz_hoff, a.lz_hlen, a.lz_w0t = ptr(hoff_d), ptr(hlen_d), ptr(lz["w0t"])
        a.lz_zp, a.lz_gdt, a.lz_fpart = ptr(lz["zp"]), ptr(lz["gdt"]), ptr(lz["fpart"])
        a.lz_rows = rows
        a.lz_defer = 1 if defer else 0
        a.lz_switch = lz_switch_step(len(active))
        if defer:
            handle = LazyFc1(lz, hoff, hlen, rows, BS, lr, w0, a.lz_switch)
    a.C, a.batch_size, a.epochs = spec.n_classes, batch_size, epochs
    a.lr, a.mu = lr, terms.get("mu", 0.0)
    a.cg, a.cc = terms.get("cg", 0.0), terms.get("cc", 0.0)
    a.timeline = ptr(timeline)
    lib.check(lib.pb_cnn_train_group(ctypes.byref(a), stream_of(w_out)))
    return handle


_EVAL_ORDER: dict = {}


def cnn_evaluate(model, X: torch.Tensor, Y: torch.Tensor) -> tuple[float, float]:
    spec = model.spec
    rows = int(Y.numel())
    w = torch.cat([model.tensors[n].reshape(-1) for n in spec.names]).contiguous()
    key = (rows, X.device)
    order = _EVAL_ORDER.get(key)
    if order is None:
        order = torch.arange(rows, dtype=torch.int32, device=X.device)
        _EVAL_ORDER[key] = order
    BS = MAX_BATCH
    slots = min((rows + BS - 1) // BS, 1024)
    ws = _WS.get(slots, BS, X.device)
    a = CnnTrainArgs()
    a.X, a.Y, a.order = ptr(X), ptr(Y), ptr(order)
    a.w = a.w0 = ptr(w)
    a.w_stride = (w.numel() + 3) // 4 * 4
    _fill(a, ws, slots, BS)
    a.C, a.batch_size, a.epochs = spec.n_classes, BS, 1
    out = torch.zeros(2, dtype=torch.float64, device=X.device)
    lib.check(lib.pb_cnn_eval(ctypes.byref(a), rows, ptr(out), stream_of(w)))
    correct, loss = out.cpu().tolist()
    return correct / rows, loss / rows
