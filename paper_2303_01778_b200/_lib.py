"""ctypes binding of libparrot_b200.so (declared in include/parrot_b200.h).

There is no fallback: if the library is missing the import fails loudly, and
every non-zero return code becomes ``NativeError`` carrying pb_last_error().
"""

from __future__ import annotations

import ctypes
import os

import numpy as np
from ctypes import POINTER, c_double, c_float, c_int, c_int32, c_int64, c_uint32, c_uint64, c_void_p
from pathlib import Path

# PB_LIB: an alternative build of the same library (A/B comparisons, tools/ab_round.py)
_PATH = Path(os.environ.get("PB_LIB") or Path(__file__).resolve().parent / "libparrot_b200.so")


class NativeError(RuntimeError):
    """A libparrot_b200 entry point returned an error code."""


class LrTrainArgs(ctypes.Structure):
    _fields_ = [
        ("X", c_void_p), ("Y", c_void_p), ("order", c_void_p), ("order_off", c_void_p),
        ("n", c_void_p), ("w0", c_void_p), ("w_out", c_void_p), ("ctrl_g", c_void_p),
        ("ctrl_c", c_void_p), ("ctrl_stride", c_int64), ("loss_sum", c_void_p),
        ("steps", c_void_p), ("nonfinite", c_void_p), ("g", c_int64),
        ("F", c_int32), ("C", c_int32), ("epochs", c_int32), ("batch_size", c_int32),
        ("lr", c_float), ("mu", c_float), ("prox_loss", c_float), ("cg", c_float),
        ("cc", c_float), ("client_ns", c_void_p),
    ]


class CnnTrainArgs(ctypes.Structure):
    _fields_ = [
        ("X", c_void_p), ("Y", c_void_p), ("order", c_void_p), ("order_off", c_void_p),
        ("n", c_void_p), ("rank", c_void_p), ("active", c_void_p), ("sweeps", c_int32),
        ("w", c_void_p), ("w_stride", c_int64), ("w0", c_void_p), ("ctrl_g", c_void_p),
        ("ctrl_c", c_void_p),
        ("ctrl_stride", c_int64), ("loss_sum", c_void_p), ("steps", c_void_p), ("bad", c_void_p),
        ("ws_slots", c_void_p), ("ws_p1", c_void_p), ("ws_am1", c_void_p), ("ws_p2", c_void_p),
        ("ws_am2", c_void_p), ("ws_h", c_void_p), ("ws_dh", c_void_p), ("ws_dp2", c_void_p),
        ("ws_dz", c_void_p), ("ws_dp1", c_void_p), ("ws_dht", c_void_p),
        ("lz_hx", c_void_p), ("lz_hxt", c_void_p), ("lz_hd", c_void_p), ("lz_hdt", c_void_p),
        ("lz_hoff", c_void_p), ("lz_hlen", c_void_p), ("lz_w0t", c_void_p), ("lz_zp", c_void_p),
        ("lz_gdt", c_void_p), ("lz_fpart", c_void_p), ("lz_rows", c_int64), ("lz_defer", c_int32),
        ("lz_switch", c_int32),
        ("g", c_int64),
        ("C", c_int32), ("BS", c_int32), ("batch_size", c_int32), ("epochs", c_int32),
        ("samples_per_cta", c_int32),
        ("lr", c_float), ("mu", c_float), ("cg", c_float), ("cc", c_float),
        ("timeline", c_void_p), ("ws_w2b", c_void_p),
    ]


class LazyFoldArgs(ctypes.Structure):
    _fields_ = [
        ("acc", c_void_p), ("w0", c_void_p), ("hx", c_void_p), ("hd", c_void_p),
        ("hrows", c_int64), ("row_lo", c_int64), ("row_hi", c_int64), ("hoff", c_void_p),
        ("nrows", c_void_p), ("w", c_void_p), ("nclients", c_int64), ("part", c_void_p),
        ("splits", c_int32), ("wsum", c_float), ("lr", c_float), ("hd_lo", c_void_p),
    ]


class ResnetTrainArgs(ctypes.Structure):
    _fields_ = [
        ("X", c_void_p), ("Y", c_void_p), ("order", c_void_p), ("order_off", c_void_p),
        ("n", c_void_p), ("rank", c_void_p), ("active", c_void_p), ("sweeps", c_int32),
        ("w", c_void_p), ("w_stride", c_int64), ("loss_sum", c_void_p), ("steps", c_void_p),
        ("bad", c_void_p), ("ws_slots", c_void_p), ("ws_w16", c_void_p), ("ws_arena", c_void_p),
        ("ws_part", c_void_p), ("ws_gnp", c_void_p), ("g", c_int64),
        ("C", c_int32), ("BS", c_int32), ("batch_size", c_int32), ("epochs", c_int32),
        ("lr", c_float), ("timeline", c_void_p),
        ("w0", c_void_p), ("ctrl_g", c_void_p), ("ctrl_c", c_void_p), ("ctrl_stride", c_int64),
        ("mu", c_float), ("cg", c_float), ("cc", c_float),
    ]


_SIGS = {
    "pb_last_error": (ctypes.c_char_p, []),
    "pb_version": (c_int, []),
    "pb_abi_sizes": (c_int, [POINTER(c_int64), c_int]),
    "pb_device_sm_count": (c_int, [c_int]),
    "pb_prof_enable": (c_int, [c_int]),
    "pb_prof_select": (c_int, [c_uint64]),
    "pb_launch_count": (c_int64, []),
    "pb_prof_collect": (c_int, [POINTER(c_double), POINTER(c_int64), c_int]),
    "pb_greedy_assign": (c_int, [POINTER(c_double), c_int64, POINTER(c_double), POINTER(c_double),
                                 c_int64, POINTER(c_int64), POINTER(c_double)]),
    "pb_minibatch_rows": (c_int, [POINTER(c_uint64), POINTER(c_int64), POINTER(c_int64),
                                  POINTER(c_int64), c_int64, c_int, POINTER(c_int32), c_int]),
    "pb_fold_f32": (c_int, [c_void_p, c_void_p, c_float, c_int64, c_void_p]),
    "pb_fold_group_f32": (c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_int64,
                                  c_int64, c_void_p]),
    "pb_lincomb_f32": (c_int, [c_void_p, c_void_p, c_float, c_void_p, c_float, c_void_p, c_float,
                               c_int64, c_void_p]),
    "pb_delta_affine_group": (c_int, [c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_void_p,
                                      c_void_p, c_float, c_void_p, c_int64, c_float, c_int64,
                                      c_int64, c_void_p]),
    "pb_state_gather": (c_int, [c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_int64, c_int64,
                                c_void_p]),
    "pb_state_scatter": (c_int, [c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_int64,
                                 c_int64, c_void_p]),
    "pb_lr_train_group": (c_int, [POINTER(LrTrainArgs), c_void_p]),
    "pb_lr_eval": (c_int, [c_void_p, c_void_p, c_int64, c_int, c_int, c_void_p, c_void_p,
                           c_void_p]),
    "pb_umma_tf32_selftest": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_int,
                                      c_void_p]),
    "pb_umma_tf32_probe": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "pb_umma_bench": (c_int, [c_int, c_int, c_int, c_int, c_int, c_int, c_void_p, c_void_p]),
    "pb_cnn_train_group": (c_int, [POINTER(CnnTrainArgs), c_void_p]),
    "pb_cnn_lazy_fold": (c_int, [POINTER(LazyFoldArgs), c_void_p]),
    "pb_resnet_workspace": (c_int, [c_int, c_int, POINTER(c_int64)]),
    "pb_umma_bench_multi": (c_int, [c_int, c_int, c_int, c_int, c_void_p, c_void_p, c_void_p]),
    "pb_tmem_ld_bench": (c_int, [c_int, c_int, c_int, c_void_p, c_void_p, c_void_p]),
    "pb_umma_bench2": (c_int, [c_int, c_int, c_int, c_int, c_uint32, c_uint32, c_uint32, c_uint32, c_uint32, c_int,
                               c_uint32, c_int, c_int, c_void_p, c_uint32, c_void_p]),
    "pb_tma_tf32_selftest": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_int, c_void_p]),
    "pb_tma_bw_probe": (c_int, [c_void_p, c_int, c_int64, c_int64, c_int, c_int, c_void_p, c_void_p]),
    "pb_tma_bf16_mn_selftest": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_int,
                                        c_void_p]),
    "pb_rn_conv_selftest": (c_int, [c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_void_p,
                                    c_void_p, c_void_p, c_void_p, c_void_p]),
    "pb_resnet_train_group": (c_int, [POINTER(ResnetTrainArgs), c_void_p]),
    "pb_resnet_eval": (c_int, [POINTER(ResnetTrainArgs), c_int64, c_void_p, c_void_p]),
    "pb_cnn_eval": (c_int, [POINTER(CnnTrainArgs), c_int64, c_void_p, c_void_p]),
    "pb_umma_selftest": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_int,
                                 c_int, c_void_p]),
}


class _Lib:
    def __init__(self, path: Path):
        if not path.exists():
            raise ImportError(
                f"{path} is missing: build it with `python -m paper_2303_01778_b200.build` "
                "(there is no CPU fallback for the device path)")
        self._dll = ctypes.CDLL(str(path))
        self.path = path
        for name, (res, args) in _SIGS.items():
            fn = getattr(self._dll, name)
            fn.restype = res
            fn.argtypes = args
            setattr(self, name, fn)

    def exported(self) -> list[str]:
        return sorted(_SIGS)

    def check(self, rc: int) -> None:
        if rc != 0:
            raise NativeError(self.pb_last_error().decode("utf-8", "replace"))


lib = _Lib(_PATH)


KERNEL_CLASSES = ("fold1", "fold_group", "lincomb", "delta_affine", "state_gather",
                  "state_scatter", "lr_train", "lr_eval", "cnn_slots", "cnn_fwd", "cnn_fc1_fwd",
                  "cnn_head", "cnn_fc1_bwd", "cnn_bwd_conv", "cnn_wgrad", "cnn_lz_xt",
                  "cnn_lz_gram_fwd", "cnn_lz_fwd", "cnn_lz_gram_bwd", "cnn_lz_bwd", "cnn_lz_mat",
                  "rn_conv_fwd", "rn_conv_dgrad", "rn_conv_wgrad", "rn_norm", "rn_head", "rn_sgd")


def prof_collect() -> dict[str, tuple[float, int]]:
    """{kernel class: (total ms, launches)} since the last collect."""
    n = len(KERNEL_CLASSES)
    ms = (c_double * n)()
    cnt = (c_int64 * n)()
    lib.check(lib.pb_prof_collect(ms, cnt, n))
    return {k: (ms[i], cnt[i]) for i, k in enumerate(KERNEL_CLASSES) if cnt[i]}


def h2d(a, device):
    """Small host array -> device without a host stall: pinned staging and an
    asynchronous copy on the current stream (a pageable copy would wait for
    all queued device work first)."""
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).pin_memory().to(device, non_blocking=True)


def ptr(t) -> int | None:
    """Raw device/host address of a torch tensor (None for None)."""
    return None if t is None else t.data_ptr()


def stream_of(t=None) -> int:
    """The current CUDA stream handle of the tensor's device, as void*."""
    import torch
    dev = t.device if t is not None else torch.device("cuda")
    return torch.cuda.current_stream(dev).cuda_stream
