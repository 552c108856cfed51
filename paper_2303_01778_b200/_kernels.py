"""Thin torch-tensor wrappers over the C ABI (argument marshalling only; all
arithmetic happens in libparrot_b200.so on the current CUDA stream)."""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from ._lib import LrTrainArgs, lib, ptr, stream_of

F32 = torch.float32


def _f32_dev(t: torch.Tensor) -> None:
    if t.dtype != F32 or not t.is_cuda:
        raise TypeError(f"expected a CUDA float32 tensor, got {t.dtype} on {t.device}")


def _rowmat(t: torch.Tensor) -> tuple[int, int, int]:
    """(base address, row stride in elements, width) of a 2-D row-major view
    whose rows are contiguous."""
    if t.dim() != 2 or (t.size(1) > 1 and t.stride(1) != 1):
        raise ValueError("expected a 2-D view with contiguous rows")
    return t.data_ptr(), t.stride(0), t.size(1)


def fold(acc: torch.Tensor, x: torch.Tensor, w: float) -> None:
    """acc += w * x  (one client into a running sum)."""
    _f32_dev(acc)
    _f32_dev(x)
    if acc.numel() != x.numel() or not acc.is_contiguous() or not x.is_contiguous():
        raise ValueError("fold: acc and x must be contiguous and equal-sized")
    lib.check(lib.pb_fold_f32(ptr(acc), ptr(x), float(w), acc.numel(), stream_of(acc)))


def fold_group(acc: torch.Tensor, xs: torch.Tensor, order: torch.Tensor | None,
               w: torch.Tensor | None) -> None:
    """acc += sum_j w[j] * xs[order[j]] in j order; xs is [rows, n] (a column
    slice of a wider matrix is fine)."""
    _f32_dev(acc)
    base, stride, n = _rowmat(xs)
    if acc.numel() != n or not acc.is_contiguous():
        raise ValueError("fold_group: accumulator/row size mismatch")
    g = int(order.numel()) if order is not None else xs.size(0)
    lib.check(lib.pb_fold_group_f32(ptr(acc), base, stride, ptr(order), ptr(w), g, n,
                                    stream_of(acc)))


def lincomb(out: torch.Tensor, x: torch.Tensor | None, a: float = 1.0,
            y: torch.Tensor | None = None, b: float = 0.0,
            z: torch.Tensor | None = None, c: float = 0.0) -> torch.Tensor:
    """out = a*x + b*y + c*z (None terms skipped)."""
    n = out.numel()
    for t in (out, x, y, z):
        if t is not None:
            _f32_dev(t)
            if t.numel() != n or not t.is_contiguous():
                raise ValueError("lincomb: operands must be contiguous and equal-sized")
    lib.check(lib.pb_lincomb_f32(ptr(out), ptr(x), float(a), ptr(y), float(b), ptr(z), float(c),
                                 n, stream_of(out)))
    return out


def delta_affine(out: torch.Tensor, a: torch.Tensor, base: torch.Tensor, s: torch.Tensor,
                 cvec: torch.Tensor | None = None, c: float = 0.0,
                 dmat: torch.Tensor | None = None, d: float = 0.0) -> torch.Tensor:
    """out[j] = s[j]*(a[j] - base) + c*cvec + d*dmat[j]   for a group."""
    ob, os_, n = _rowmat(out)
    ab, as_, na = _rowmat(a)
    g = out.size(0)
    if na != n or base.numel() != n or s.numel() != g:
        raise ValueError("delta_affine: shape mismatch")
    db, ds_ = (0, 0)
    if dmat is not None:
        db, ds_, nd = _rowmat(dmat)
        if nd != n:
            raise ValueError("delta_affine: dmat width mismatch")
    lib.check(lib.pb_delta_affine_group(ob, os_, ab, as_, ptr(base), ptr(s), ptr(cvec), float(c),
                                        db or None, ds_, float(d), g, n, stream_of(out)))
    return out


def state_gather(work: torch.Tensor, store: torch.Tensor, slot: torch.Tensor) -> None:
    wb, ws, width = _rowmat(work)
    sb, ss, sw = _rowmat(store)
    if sw < width:
        raise ValueError("state_gather: store narrower than work rows")
    lib.check(lib.pb_state_gather(wb, ws, sb, ss, ptr(slot), slot.numel(), width,
                                  stream_of(work)))


def state_scatter(store: torch.Tensor, work: torch.Tensor, slot: torch.Tensor) -> None:
    wb, ws, width = _rowmat(work)
    sb, ss, sw = _rowmat(store)
    if sw < width:
        raise ValueError("state_scatter: store narrower than work rows")
    lib.check(lib.pb_state_scatter(sb, ss, wb, ws, ptr(slot), slot.numel(), width,
                                   stream_of(work)))


def lr_train(X, Y, order, order_off, n, w0, w_out, loss_sum, steps, nonfinite, *, F, C, epochs,
             batch_size, lr, mu=0.0, prox_loss=0.0, ctrl_g=None, cg=0.0, ctrl_c=None,
             cc=0.0, client_ns=None) -> None:
    a = LrTrainArgs()
    a.X, a.Y, a.order, a.order_off, a.n = ptr(X), ptr(Y), ptr(order), ptr(order_off), ptr(n)
    a.w0, a.w_out = ptr(w0), ptr(w_out)
    a.ctrl_g, a.ctrl_c = ptr(ctrl_g), ptr(ctrl_c)
    a.ctrl_stride = ctrl_c.stride(0) if ctrl_c is not None else 0
    a.loss_sum, a.steps, a.nonfinite = ptr(loss_sum), ptr(steps), ptr(nonfinite)
    a.g = w_out.size(0)
    a.F, a.C, a.epochs, a.batch_size = F, C, epochs, batch_size
    a.lr, a.mu, a.prox_loss, a.cg, a.cc = lr, mu, prox_loss, cg, cc
    a.client_ns = ptr(client_ns)
    lib.check(lib.pb_lr_train_group(ctypes.byref(a), stream_of(w_out)))


def lr_eval(X, Y, w, F: int, C: int) -> tuple[float, float]:
    rows = Y.numel()
    out = torch.zeros(2, dtype=torch.float64, device=w.device)
    lib.check(lib.pb_lr_eval(ptr(X), ptr(Y), rows, F, C, ptr(w), ptr(out), stream_of(w)))
    correct, loss = out.cpu().tolist()
    return correct / rows, loss / rows


def minibatch_rows(keys: np.ndarray, n: np.ndarray, row_base: np.ndarray, epochs: int,
                   threads: int = 4) -> tuple[np.ndarray, np.ndarray]:
    """Host (native) minibatch orders: returns (rows int32, per-client offsets)."""
    n = np.ascontiguousarray(n, dtype=np.int64)
    off = np.zeros(len(n), dtype=np.int64)
    if len(n) > 1:
        off[1:] = np.cumsum(n * epochs)[:-1]
    out = np.empty(int((n * epochs).sum()), dtype=np.int32)
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    base = np.ascontiguousarray(row_base, dtype=np.int64)
    P64 = ctypes.POINTER(ctypes.c_int64)
    lib.check(lib.pb_minibatch_rows(keys.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                                    n.ctypes.data_as(P64), off.ctypes.data_as(P64),
                                    base.ctypes.data_as(P64), len(n), int(epochs),
                                    out.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                    int(threads)))
    return out, off
