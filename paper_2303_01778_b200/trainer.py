"""Client training, parameter bundles and the algorithm plugins -- device path.

API mirrors ``fedsim/trainer.py`` (AggOp, ParamBundle, ModelParams,
TrainReport, AlgorithmPlugin + FedAvg/FedProx/FedNova/Scaffold/FedDyn,
make_plugin, client_execute, evaluate).  Differences, all deliberate:

* bundle tensors live on the GPU in fp32 (``ParamBundle.numpy(name)`` gives a
  float64 host copy); the reference keeps float64 NumPy arrays;
* the built-in plugins run their ``local_gradient``/``finalize`` as fused
  device terms (``grad_terms``) and a group finalizer (``finalize_group``),
  because the whole local run of a client happens inside one kernel
  (SURVEY.md §8(a) a4-a6).  They also expose the reference's per-minibatch
  hooks (``local_gradient(model, xb, yb, ctx)``, ``finalize(...)``) on device
  tensors; a reference-style plugin that overrides those hooks (and not the
  fused ones) is executed client by client through them on the GPU
  (``uses_hooks``, ``hook_client_execute``) -- the drop-in path for custom
  algorithms, not the batched hot path;
* training is batched: ``train_group`` runs G clients concurrently, one CTA
  (LR) per client, with bit-identical minibatch orders
  (``default_rng([seed, 6, client, round]).permutation`` per epoch,
  restated natively in csrc/host_sched.cpp).
"""

from __future__ import annotations

import abc
import enum
import time
import weakref
from dataclasses import dataclass, field
from typing import Mapping, Sequence

import numpy as np
import torch

from . import _kernels as K
from .core import STREAM_MINIBATCH, ClientProfile
from .models import ModelSpec, cnn_spec, lr_spec, resnet_spec
from .statestore import ClientState


class NonFiniteLossError(RuntimeError):
    """Local training diverged (fedsim/trainer.py:31-32)."""


class AggOp(enum.Enum):
    WEIGHTED_AVERAGE = "WeightedAverage"
    SUM = "Sum"
    SIMPLE_AVERAGE = "SimpleAverage"
    COLLECT = "Collect"


AVERAGING_OPS = (AggOp.WEIGHTED_AVERAGE, AggOp.SUM, AggOp.SIMPLE_AVERAGE)


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2303_01778_b200 runs on a CUDA device (sm_100a); none is visible")
    return torch.device("cuda", torch.cuda.current_device())


def to_device(t) -> torch.Tensor:
    """Own an fp32, contiguous device copy of an ndarray / tensor / scalar."""
    if isinstance(t, torch.Tensor):
        return t.detach().to(device=device(), dtype=torch.float32).contiguous().clone()
    return torch.from_numpy(np.array(t, dtype=np.float32, copy=True)).to(device())


def _all_finite(*ts: torch.Tensor) -> bool:
    return bool(all(torch.isfinite(t).all().item() for t in ts))


@dataclass(frozen=True)
class ModelParams:
    """The reference's LR model: weights [C, F], bias [C] (device fp32)."""

    weights: torch.Tensor
    bias: torch.Tensor

    def __post_init__(self) -> None:
        object.__setattr__(self, "weights", _as_dev(self.weights))
        object.__setattr__(self, "bias", _as_dev(self.bias))
        if not _all_finite(self.weights, self.bias):
            raise ValueError("model parameters must be finite")

    def copy(self) -> "ModelParams":
        return ModelParams(self.weights.clone(), self.bias.clone())

    @staticmethod
    def zeros(n_classes: int, n_features: int) -> "ModelParams":
        d = device()
        return ModelParams(torch.zeros(n_classes, n_features, device=d),
                           torch.zeros(n_classes, device=d))

    @property
    def spec(self) -> ModelSpec:
        return lr_spec(self.weights.shape[0], self.weights.shape[1])

    def named(self) -> dict[str, torch.Tensor]:
        return {"weights": self.weights, "bias": self.bias}


@dataclass(frozen=True)
class NamedParams:
    """A model given as named device tensors in a ModelSpec layout (CNN)."""

    spec: ModelSpec
    tensors: dict

    @staticmethod
    def from_flat(spec: ModelSpec, flat) -> "NamedParams":
        flat = to_device(flat).reshape(-1)
        if flat.numel() != spec.numel:
            raise ValueError(f"flat vector has {flat.numel()} values, spec needs {spec.numel}")
        return NamedParams(spec, {n: flat[o:o + s].view(sh) for n, o, s, sh in spec.columns()})

    def named(self) -> dict[str, torch.Tensor]:
        return dict(self.tensors)


def _as_dev(t) -> torch.Tensor:
    if isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float32:
        return t
    return to_device(t)


@dataclass(frozen=True)
class BundleEntry:
    tensor: torch.Tensor
    op: AggOp
    weight: float = 1.0
    client_id: int | None = None

    def __post_init__(self) -> None:
        if self.op is AggOp.WEIGHTED_AVERAGE and not self.weight > 0:
            raise ValueError("WeightedAverage entries require weight > 0")
        if self.op is AggOp.COLLECT and self.client_id is None:
            raise ValueError("Collect entries must carry the originating client_id")


@dataclass
class ParamBundle:
    """Named device tensors annotated with how the server combines them
    (fedsim/trainer.py:76-109).  Tensors are immutable once added."""

    entries: dict[str, BundleEntry] = field(default_factory=dict)

    def add(self, name: str, tensor, op: AggOp, weight: float = 1.0,
            client_id: int | None = None) -> "ParamBundle":
        if name in self.entries:
            raise ValueError(f"duplicate bundle entry {name!r}")
        self.entries[name] = BundleEntry(to_device(tensor), op, weight, client_id)
        return self

    def _put(self, name: str, tensor: torch.Tensor, op: AggOp, weight: float = 1.0,
             client_id: int | None = None) -> "ParamBundle":
        """Add an existing device tensor without copying (internal)."""
        if name in self.entries:
            raise ValueError(f"duplicate bundle entry {name!r}")
        self.entries[name] = BundleEntry(tensor, op, weight, client_id)
        return self

    def tensor(self, name: str) -> torch.Tensor:
        return self.entries[name].tensor

    def numpy(self, name: str) -> np.ndarray:
        return self.entries[name].tensor.detach().cpu().double().numpy()

    def model(self) -> ModelParams:
        return ModelParams(self.tensor("weights"), self.tensor("bias"))

    def named_model(self, spec: ModelSpec, prefix: str = "") -> dict[str, torch.Tensor]:
        return {n: self.tensor(prefix + n) for n in spec.names}

    def flat(self, spec: ModelSpec, prefix: str = "") -> torch.Tensor:
        """Model-shaped entries packed into one flat [P] device vector."""
        return torch.cat([self.tensor(prefix + n).reshape(-1) for n in spec.names])

    def replaced(self, **tensors) -> "ParamBundle":
        out = ParamBundle()
        for name, e in self.entries.items():
            t = tensors.pop(name, e.tensor)
            out.entries[name] = BundleEntry(_as_dev(t), e.op, e.weight, e.client_id)
        if tensors:
            raise KeyError(f"no such bundle entries: {sorted(tensors)}")
        return out


@dataclass(frozen=True)
class TrainReport:
    client_result: ParamBundle
    new_state: ClientState | None
    samples_processed: int
    measured_seconds: float

    def __post_init__(self) -> None:
        if self.samples_processed > 0 and not self.measured_seconds > 0:
            raise ValueError("measured_seconds must be > 0 when samples were processed")


@dataclass
class LocalContext:
    """Everything a plugin's gradient hook may read during one client task
    (fedsim/trainer.py:161-170); tensors are fp32 device tensors."""

    start_model: ModelParams
    global_bundle: ParamBundle
    state: dict | None
    lr: float
    n_samples: int


def _model_unchecked(w: torch.Tensor, b: torch.Tensor) -> ModelParams:
    """A ModelParams without the per-construction finiteness sync (the hook
    loop checks the accumulated loss once at the end instead)."""
    m = object.__new__(ModelParams)
    object.__setattr__(m, "weights", w)
    object.__setattr__(m, "bias", b)
    return m


def _softmax_terms(model: ModelParams, x: torch.Tensor):
    z = x @ model.weights.T + model.bias
    z = z - z.max(dim=1, keepdim=True).values
    return z, torch.log(torch.exp(z).sum(dim=1))


def loss_value(model: ModelParams, x: torch.Tensor, y: torch.Tensor) -> torch.Tensor:
    """Mean cross-entropy (fedsim/trainer.py:131-133), a 0-d device tensor."""
    z, lse = _softmax_terms(model, x)
    return (lse - z[torch.arange(len(y), device=z.device), y]).mean()


def loss_and_grad(model: ModelParams, x: torch.Tensor, y: torch.Tensor):
    """Mean CE and its gradient for multinomial LR (fedsim/trainer.py:136-145):
    P = softmax(XW^T + b), grad_W = (P - Y)^T X / B, grad_b = sum(P - Y) / B.
    Returns (loss as a 0-d device tensor, grad_W, grad_b)."""
    z, lse = _softmax_terms(model, x)
    p = torch.exp(z - lse[:, None])
    rows = torch.arange(len(y), device=z.device)
    loss = (lse - z[rows, y]).mean()
    p[rows, y] -= 1.0
    p /= len(y)
    return loss, p.T @ x, p.sum(dim=0)


# ---------------------------------------------------------------------------
# device-resident client data
# ---------------------------------------------------------------------------

@dataclass
class ClientData:
    """All clients' samples packed on the device: X [rows, F] fp32, Y [rows]
    int32, client m owning rows [row_base[m], row_base[m] + sizes[m])."""

    X: torch.Tensor
    Y: torch.Tensor
    row_base: np.ndarray
    sizes: np.ndarray
    n_features: int
    n_classes: int

    @staticmethod
    def from_profiles(profiles: Sequence[ClientProfile], n_classes: int | None = None) -> "ClientData":
        d = device()
        ids = [p.client_id for p in profiles]
        m = max(ids) + 1 if ids else 0
        sizes = np.zeros(m, dtype=np.int64)
        base = np.zeros(m, dtype=np.int64)
        feats, labels, pos = [], [], 0
        for p in profiles:
            sizes[p.client_id] = p.sample_count
            base[p.client_id] = pos
            pos += p.sample_count
            feats.append(np.asarray(p.data_partition.features, dtype=np.float32))
            labels.append(np.asarray(p.data_partition.labels, dtype=np.int32))
        X = torch.from_numpy(np.concatenate(feats) if feats else np.zeros((0, 1), np.float32)).to(d)
        Y = torch.from_numpy(np.concatenate(labels) if labels else np.zeros(0, np.int32)).to(d)
        if n_classes is None:
            n_classes = 1 + max(int(np.max(p.data_partition.labels)) for p in profiles)
        return ClientData(X, Y, base, sizes, int(X.shape[1]), int(n_classes))


# ---------------------------------------------------------------------------
# group training
# ---------------------------------------------------------------------------

@dataclass
class GroupOutcome:
    clients: list[int]
    n: np.ndarray           # samples per client
    steps: np.ndarray       # local steps taken
    loss_mean: np.ndarray   # mean per-step loss (Collect local_loss)
    w_out: torch.Tensor     # [G, P] end models
    seconds: float          # device time of the training launch
    lazy: object | None = None  # deferred low-rank fc1 (cnn.LazyFc1): fc1_w rows unmaterialised
    pending: object | None = None  # deferred result read (train_group(defer_check=True))
    client_seconds: np.ndarray | None = None  # [G] device-measured task time (timing=True)
    timing: object | None = None  # (stamps tensor, decoder) until the result read
    lazy_history: bool = False  # trained on the low-rank fc1 history workspace (cnn._LZ)

    def resolve(self) -> None:
        """Finish a deferred result read: wait for the group's [bad | steps |
        loss] copy, raise on a diverged client, fill loss_mean / seconds."""
        if self.pending is None:
            return
        res_h, done, t0, t1, round_num = self.pending
        self.pending = None
        done.synchronize()
        res = res_h.numpy()
        _IO["d2h"] += res.size * 8
        G = len(self.clients)
        bad_h, steps_h, loss_h = res[:G], res[G:2 * G].astype(np.int64), res[2 * G:]
        self.seconds = max(t0.elapsed_time(t1) / 1e3, 1e-9)
        for j in range(G):
            if bad_h[j] >= 0:
                raise NonFiniteLossError(f"client {self.clients[j]} round {round_num}: loss diverged")
        if not np.array_equal(steps_h, self.steps):
            raise RuntimeError(f"round {round_num}: device step counts differ from the plan")
        if self.lazy_history:
            from .cnn import _LZ
            _LZ.dirty = False   # every client finite: the history may stay as stale operands
        self.loss_mean = loss_h / np.maximum(steps_h, 1)
        self._decode_timing()

    def _decode_timing(self) -> None:
        if self.timing is not None:
            stamps, decode = self.timing
            self.timing = None
            self.client_seconds = decode(stamps.cpu().numpy())


@dataclass
class ResultGroup:
    """Per-client result entries of one aggregation op, stored as the rows of
    one [G, width] device matrix (entry k = columns cols[k])."""

    names: list[str]
    cols: list[tuple[int, int, tuple]]
    mat: torch.Tensor
    op: AggOp
    weights: np.ndarray
    lazy: object | None = None  # cnn.LazyFc1 when the fc1_w columns are deferred


def spec_groups(spec: ModelSpec, mat: torch.Tensor, op: AggOp, weights, prefix: str = ""):
    return ResultGroup([prefix + n for n in spec.names],
                       [(o, s, sh) for _, o, s, sh in spec.columns()], mat, op,
                       np.asarray(weights, dtype=np.float64))


def client_bundle(groups: Sequence[ResultGroup], j: int, client_id: int) -> ParamBundle:
    out = ParamBundle()
    for g in groups:
        for name, (off, size, shape) in zip(g.names, g.cols):
            view = g.mat[j, off:off + size].view(shape)
            out._put(name, view, g.op, float(g.weights[j]),
                     client_id if g.op is AggOp.COLLECT else None)
    return out


_IO = {"h2d": 0, "d2h": 0}


def io_bytes() -> tuple[int, int]:
    """Host<->device bytes moved by the training path so far (inputs / results)."""
    return _IO["h2d"], _IO["d2h"]


class GroupInputs:
    """Host-prepared per-round inputs of one training group: the clients'
    minibatch row ids (native NumPy-PCG64 permutations), offsets and sizes,
    in pinned memory, plus their device copies once uploaded."""

    def __init__(self, data: "ClientData", clients: Sequence[int], epochs: int, seed: int,
                 round_num: int):
        self.clients = [int(c) for c in clients]
        G = len(self.clients)
        self.n = data.sizes[self.clients].astype(np.int64)
        keys = np.zeros((G, 4), dtype=np.uint64)
        keys[:, 0] = np.uint64(seed)
        keys[:, 1] = STREAM_MINIBATCH
        keys[:, 2] = np.asarray(self.clients, dtype=np.uint64)
        keys[:, 3] = round_num
        rows, off = K.minibatch_rows(keys, self.n, data.row_base[self.clients], epochs)
        self.rows_h = torch.from_numpy(rows).pin_memory()
        self.off_h = torch.from_numpy(off).pin_memory()
        self.n_h = torch.from_numpy(self.n.astype(np.int32)).pin_memory()
        self.rows_d = self.off_d = self.n_d = None

    def upload(self) -> "GroupInputs":
        if self.rows_d is None:
            d = device()
            self.rows_d = self.rows_h.to(d, non_blocking=True)
            self.off_d = self.off_h.to(d, non_blocking=True)
            self.n_d = self.n_h.to(d, non_blocking=True)
            _IO["h2d"] += (self.rows_h.numel() * 4 + self.off_h.numel() * 8 + self.n_h.numel() * 4)
        return self


def train_group(plugin: "AlgorithmPlugin", spec: ModelSpec, data: ClientData,
                clients: Sequence[int], w0: torch.Tensor, global_bundle: ParamBundle,
                state_work: torch.Tensor | None, epochs: int, batch_size: int, lr: float,
                seed: int, round_num: int, inputs: GroupInputs | None = None,
                defer_fc1: bool = False, defer_check: bool = False,
                timing: bool = False) -> GroupOutcome:
    """Run every listed client's full local schedule concurrently on the GPU.

    timing (real clock): per-client device task times from %globaltimer
    stamps taken by the kernels (``GroupOutcome.client_seconds``): for the LR
    model each client's own CTA span; for the sweep models (CNN, ResNet) the
    duration of every sweep divided among the clients active in it, summed
    over the client's sweeps (the clients' times add up to the group's).

    defer_fc1 (CNN, plain SGD): leave the clients' fc1_w columns of w_out
    unmaterialised and return the round's low-rank history instead
    (``GroupOutcome.lazy``); only valid when the caller folds the group with
    aggregate.fold_group and reads no per-client fc1 weights."""
    d = device()
    lazy = None
    if inputs is None:
        inputs = GroupInputs(data, clients, epochs, seed, round_num)
    if [int(c) for c in clients] != inputs.clients:
        raise ValueError("prepared inputs belong to a different client group")
    inputs.upload()
    clients, n = inputs.clients, inputs.n
    G = len(clients)
    P = spec.numel
    # CNN rows padded to 32 floats: 16-byte aligned vector / cp.async access
    P_pad = (P + 31) // 32 * 32 if spec.kind in ("cnn", "resnet") else P
    w_out = torch.empty(G, P_pad, device=d)[:, :P]
    loss = torch.empty(G, dtype=torch.float64, device=d)
    steps = torch.empty(G, dtype=torch.int32, device=d)
    bad = torch.empty(G, dtype=torch.int32, device=d)
    terms = plugin.grad_terms(spec, global_bundle)
    if terms.get("ctrl_c") and state_work is None:
        raise ValueError(f"{plugin.name} needs client state for training")
    bs_c = n if batch_size <= 0 else np.minimum(batch_size, n)
    steps_plan = (epochs * ((n + bs_c - 1) // bs_c)).astype(np.int64)
    stamps = decode = None
    if timing and spec.kind == "lr":
        stamps = torch.zeros(G, 2, dtype=torch.int64, device=d)

        def decode(ns):
            return np.maximum((ns[:, 1] - ns[:, 0]) * 1e-9, 1e-9)
    elif timing:
        sweeps = int(steps_plan.max())
        active = np.array([(steps_plan > s).sum() for s in range(sweeps)], dtype=np.float64)
        stamps = torch.zeros(sweeps + 1, dtype=torch.int64, device=d)

        def decode(ts):
            share = np.diff(ts.astype(np.float64)) * 1e-9 / active   # per active client, per sweep
            cum = np.concatenate([[0.0], np.cumsum(share)])
            return np.maximum(cum[steps_plan], 1e-9)
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    lz_used = False
    if spec.kind == "lr":
        K.lr_train(data.X, data.Y, inputs.rows_d, inputs.off_d, inputs.n_d, w0, w_out, loss,
                   steps, bad, F=spec.n_features, C=spec.n_classes, epochs=epochs,
                   batch_size=batch_size, lr=lr, mu=terms.get("mu", 0.0),
                   prox_loss=terms.get("prox_loss", 0.0), ctrl_g=terms.get("ctrl_g"),
                   cg=terms.get("cg", 0.0), ctrl_c=state_work if terms.get("ctrl_c") else None,
                   cc=terms.get("cc", 0.0), client_ns=stamps)
    elif spec.kind == "cnn":
        from .cnn import cnn_train_group, lazy_enabled
        lz_used = lazy_enabled(terms)
        lazy = cnn_train_group(data, inputs.rows_d, inputs.off_d, n, w0, w_out, loss, steps, bad,
                               spec=spec, epochs=epochs, batch_size=batch_size, lr=lr, terms=terms,
                               state_work=state_work, defer_fc1=defer_fc1, timeline=stamps)
    elif spec.kind == "resnet":
        from .resnet import resnet_train_group
        resnet_train_group(data, inputs.rows_d, inputs.off_d, n, w0, w_out, loss, steps, bad,
                           spec=spec, epochs=epochs, batch_size=batch_size, lr=lr, terms=terms,
                           state_work=state_work, timeline=stamps)
    else:
        raise ValueError(f"unknown model kind {spec.kind!r}")
    t1.record()
    if defer_check:
        # the step counts are the plan's (a diverged client raises when the
        # read completes, GroupOutcome.resolve); the read itself is queued
        # behind the training without blocking the host
        res_h = torch.empty(3 * G, dtype=torch.float64, pin_memory=True)
        res_h.copy_(torch.cat([bad.double(), steps.double(), loss]), non_blocking=True)
        done = torch.cuda.Event()
        done.record()
        if lazy is not None:
            lazy.set_steps(steps_plan)
        return GroupOutcome(clients, n, steps_plan, np.full(G, np.nan), w_out, float("nan"), lazy,
                            pending=(res_h, done, t0, t1, round_num),
                            timing=(stamps, decode) if stamps is not None else None,
                            lazy_history=lz_used)
    # one device->host read per group: failures, step counts, losses
    res = torch.cat([bad.double(), steps.double(), loss]).cpu().numpy()
    _IO["d2h"] += res.size * 8
    bad_h, steps_h, loss_h = res[:G], res[G:2 * G].astype(np.int64), res[2 * G:]
    seconds = max(t0.elapsed_time(t1) / 1e3, 1e-9)
    for j in range(G):
        if bad_h[j] >= 0:
            raise NonFiniteLossError(f"client {clients[j]} round {round_num}: loss diverged")
    if lazy is not None:
        lazy.set_steps(steps_h)
    if lz_used:
        from .cnn import _LZ
        _LZ.dirty = False   # every client finite: the history may stay as stale operands
    go = GroupOutcome(clients, n, steps_h, loss_h / np.maximum(steps_h, 1), w_out, seconds, lazy,
                      timing=(stamps, decode) if stamps is not None else None)
    go._decode_timing()
    return go


# ---------------------------------------------------------------------------
# algorithm plugins
# ---------------------------------------------------------------------------

def _spec_of_model(model) -> ModelSpec:
    if isinstance(model, ModelParams):
        return model.spec
    if isinstance(model, NamedParams):
        return model.spec
    raise TypeError(f"unsupported model type {type(model).__name__}")


class AlgorithmPlugin(abc.ABC):
    """One federated optimisation algorithm (fedsim/trainer.py:172-215), with
    its hooks expressed as fused device terms."""

    name: str
    is_stateful: bool = False
    state_prefix: str | None = None

    def __init__(self, lr: float = 0.1, batch_size: int = 0, collect_local_loss: bool = False):
        if not lr > 0:
            raise ValueError("lr must be > 0")
        self.lr = float(lr)
        self.batch_size = int(batch_size)
        self.collect_local_loss = bool(collect_local_loss)
        self.spec: ModelSpec | None = None

    # -- naming -------------------------------------------------------------
    def _names(self) -> tuple[str, ...]:
        return self.spec.names if self.spec is not None else ("weights", "bias")

    @property
    def required_result_entries(self) -> tuple[str, ...]:
        return self._names()

    # -- global / state -----------------------------------------------------
    def init_global(self, model) -> ParamBundle:
        self.spec = _spec_of_model(model)
        out = ParamBundle()
        for name, t in model.named().items():
            out.add(name, t, AggOp.WEIGHTED_AVERAGE)
        return out

    def default_state(self, model) -> dict[str, torch.Tensor] | None:
        if self.state_prefix is None:
            return None
        return {self.state_prefix + n: torch.zeros_like(_as_dev(t))
                for n, t in model.named().items()}

    def state_names(self, spec: ModelSpec) -> list[str]:
        return [self.state_prefix + n for n in spec.names] if self.state_prefix else []

    # -- fused hooks (the batched kernels) -----------------------------------
    def grad_terms(self, spec: ModelSpec, glob: ParamBundle) -> dict:
        """Extra gradient terms: g + mu*(w - w0) + cg*ctrl_g + cc*state."""
        return {}

    def finalize_group(self, spec: ModelSpec, go: GroupOutcome, w0: torch.Tensor,
                       glob: ParamBundle, state_work: torch.Tensor | None):
        """-> (list[ResultGroup], new state rows [G, P] or None)."""
        raise NotImplementedError(f"plugin {self.name!r} has no fused group finalizer")

    # -- reference hooks (fedsim/trainer.py:199-207), on device tensors --------
    def local_gradient(self, model: ModelParams, xb: torch.Tensor, yb: torch.Tensor,
                       ctx: LocalContext):
        """Return (loss, grad_weights, grad_bias) on one minibatch."""
        raise NotImplementedError(f"plugin {self.name!r} defines no local_gradient hook")

    def finalize(self, end_model: ModelParams, steps: int, ctx: LocalContext, n_samples: int):
        """Build the uploaded result bundle and the new state payload."""
        raise NotImplementedError(f"plugin {self.name!r} defines no finalize hook")

    @abc.abstractmethod
    def server_update(self, old_global: ParamBundle, agg) -> ParamBundle:
        """Apply the server rule to the folded aggregate."""


def _model_bundle(model: ModelParams, op: AggOp, weight: float = 1.0, prefix: str = "",
                  weights=None, bias=None) -> ParamBundle:
    out = ParamBundle()
    out._put(prefix + "weights", model.weights if weights is None else weights, op, weight)
    out._put(prefix + "bias", model.bias if bias is None else bias, op, weight)
    return out


def _per_client(values, d=None) -> torch.Tensor:
    return torch.from_numpy(np.asarray(values, dtype=np.float32)).to(d or device())


class FedAvg(AlgorithmPlugin):
    """fedsim/trainer.py:218-234."""

    name = "fedavg"

    def finalize_group(self, spec, go, w0, glob, state_work):
        return [spec_groups(spec, go.w_out, AggOp.WEIGHTED_AVERAGE, go.n)], None

    def local_gradient(self, model, xb, yb, ctx):
        return loss_and_grad(model, xb, yb)

    def finalize(self, end_model, steps, ctx, n_samples):
        return _model_bundle(end_model, AggOp.WEIGHTED_AVERAGE, n_samples), None

    def server_update(self, old_global, agg):
        return old_global.replaced(**{n: agg.bundle.tensor(n) for n in self._names()})


class FedProx(FedAvg):
    """fedsim/trainer.py:237-257: g + mu*(w - w0); loss + mu/2*||w - w0||^2."""

    name = "fedprox"

    def __init__(self, mu: float = 0.01, **kw):
        super().__init__(**kw)
        if mu < 0:
            raise ValueError("mu must be >= 0")
        self.mu = float(mu)

    def grad_terms(self, spec, glob):
        return {"mu": self.mu, "prox_loss": 0.5 * self.mu} if self.mu != 0.0 else {}

    def local_gradient(self, model, xb, yb, ctx):
        loss, gw, gb = loss_and_grad(model, xb, yb)
        if self.mu != 0.0:
            dw = model.weights - ctx.start_model.weights
            db = model.bias - ctx.start_model.bias
            loss = loss + 0.5 * self.mu * ((dw * dw).sum() + (db * db).sum())
            gw = gw + self.mu * dw
            gb = gb + self.mu * db
        return loss, gw, gb


class FedNova(FedAvg):
    """fedsim/trainer.py:260-285: upload (w0 - w)/(lr*steps) and n*lr*steps."""

    name = "fednova"

    @property
    def required_result_entries(self):
        return tuple("direction_" + n for n in self._names()) + ("step_scale",)

    def finalize_group(self, spec, go, w0, glob, state_work):
        d = go.w_out.device
        scale = self.lr * go.steps.astype(np.float64)
        direction = torch.empty_like(go.w_out)
        K.delta_affine(direction, go.w_out, w0, _per_client(-1.0 / scale, d))
        step = _per_client(go.n * scale, d).view(-1, 1)
        return [spec_groups(spec, direction, AggOp.WEIGHTED_AVERAGE, go.n, "direction_"),
                ResultGroup(["step_scale"], [(0, 1, (1,))], step, AggOp.SUM,
                            np.ones(len(go.n)))], None

    def finalize(self, end_model, steps, ctx, n_samples):
        scale = self.lr * steps
        x = ctx.start_model
        out = _model_bundle(end_model, AggOp.WEIGHTED_AVERAGE, n_samples, "direction_",
                            (x.weights - end_model.weights) / scale, (x.bias - end_model.bias) / scale)
        out._put("step_scale", torch.tensor([n_samples * scale], dtype=torch.float32,
                                            device=x.weights.device), AggOp.SUM)
        return out, None

    def server_update(self, old_global, agg):
        first = "direction_" + self._names()[0]
        eff = float(agg.bundle.tensor("step_scale").double().sum().item()) / agg.weights[first]
        out = {}
        for n in self._names():
            x = old_global.tensor(n)
            out[n] = K.lincomb(torch.empty_like(x), x, 1.0,
                               agg.bundle.tensor("direction_" + n), -eff)
        return old_global.replaced(**out)


class Scaffold(AlgorithmPlugin):
    """fedsim/trainer.py:288-348: local steps use g + (c - c_m); uploads the
    model delta (WA) and control delta (SA); c_m+ = c_m - c + (x - y)/(steps lr)."""

    name = "scaffold"
    is_stateful = True
    state_prefix = "ctrl_"

    def __init__(self, client_fraction: float = 1.0, **kw):
        super().__init__(**kw)
        if not 0 < client_fraction <= 1:
            raise ValueError("client_fraction must be in (0, 1]")
        self.client_fraction = float(client_fraction)

    @property
    def required_result_entries(self):
        names = self._names()
        return tuple("delta_" + n for n in names) + tuple("ctrl_delta_" + n for n in names)

    def init_global(self, model):
        out = super().init_global(model)
        for n, t in model.named().items():
            out._put("server_ctrl_" + n, torch.zeros_like(_as_dev(t)), AggOp.SUM)
        return out

    def grad_terms(self, spec, glob):
        return {"ctrl_g": glob.flat(spec, "server_ctrl_"), "cg": 1.0, "ctrl_c": True, "cc": -1.0}

    def finalize_group(self, spec, go, w0, glob, state_work):
        d = go.w_out.device
        G = len(go.n)
        c = glob.flat(spec, "server_ctrl_")
        inv = 1.0 / (go.steps.astype(np.float64) * self.lr)
        delta = torch.empty_like(go.w_out)
        K.delta_affine(delta, go.w_out, w0, _per_client(np.ones(G), d))
        ctrl_delta = torch.empty_like(go.w_out)
        K.delta_affine(ctrl_delta, go.w_out, w0, _per_client(-inv, d), cvec=c, c=-1.0)
        new_c = torch.empty_like(go.w_out)
        K.delta_affine(new_c, go.w_out, w0, _per_client(-inv, d), cvec=c, c=-1.0,
                       dmat=state_work, d=1.0)
        return [spec_groups(spec, delta, AggOp.WEIGHTED_AVERAGE, go.n, "delta_"),
                spec_groups(spec, ctrl_delta, AggOp.SIMPLE_AVERAGE, np.ones(G), "ctrl_delta_")], new_c

    def local_gradient(self, model, xb, yb, ctx):
        loss, gw, gb = loss_and_grad(model, xb, yb)
        g = ctx.global_bundle
        gw = gw + (g.tensor("server_ctrl_weights") - _as_dev(ctx.state["ctrl_weights"]))
        gb = gb + (g.tensor("server_ctrl_bias") - _as_dev(ctx.state["ctrl_bias"]))
        return loss, gw, gb

    def finalize(self, end_model, steps, ctx, n_samples):
        x, y, g = ctx.start_model, end_model, ctx.global_bundle
        inv = 1.0 / (steps * self.lr)
        cw, cb = _as_dev(ctx.state["ctrl_weights"]), _as_dev(ctx.state["ctrl_bias"])
        new_cw = cw - g.tensor("server_ctrl_weights") + (x.weights - y.weights) * inv
        new_cb = cb - g.tensor("server_ctrl_bias") + (x.bias - y.bias) * inv
        out = _model_bundle(y, AggOp.WEIGHTED_AVERAGE, n_samples, "delta_",
                            y.weights - x.weights, y.bias - x.bias)
        out._put("ctrl_delta_weights", new_cw - cw, AggOp.SIMPLE_AVERAGE)
        out._put("ctrl_delta_bias", new_cb - cb, AggOp.SIMPLE_AVERAGE)
        return out, {"ctrl_weights": new_cw, "ctrl_bias": new_cb}

    def server_update(self, old_global, agg):
        out = {}
        for n in self._names():
            x = old_global.tensor(n)
            out[n] = K.lincomb(torch.empty_like(x), x, 1.0, agg.bundle.tensor("delta_" + n), 1.0)
            c = old_global.tensor("server_ctrl_" + n)
            out["server_ctrl_" + n] = K.lincomb(torch.empty_like(c), c, 1.0,
                                                agg.bundle.tensor("ctrl_delta_" + n),
                                                self.client_fraction)
        return old_global.replaced(**out)


class FedDyn(AlgorithmPlugin):
    """fedsim/trainer.py:351-407: g - h_m + alpha*(w - w0); h_m+ = h_m - alpha*(y - x);
    server keeps h and recentres the simple average by -h/alpha."""

    name = "feddyn"
    is_stateful = True
    state_prefix = "grad_corr_"

    def __init__(self, alpha: float = 0.1, client_fraction: float = 1.0, **kw):
        super().__init__(**kw)
        if not alpha > 0:
            raise ValueError("alpha must be > 0")
        if not 0 < client_fraction <= 1:
            raise ValueError("client_fraction must be in (0, 1]")
        self.alpha = float(alpha)
        self.client_fraction = float(client_fraction)

    def init_global(self, model):
        self.spec = _spec_of_model(model)
        out = ParamBundle()
        for n, t in model.named().items():
            out.add(n, t, AggOp.SIMPLE_AVERAGE)
        for n, t in model.named().items():
            out._put("server_h_" + n, torch.zeros_like(_as_dev(t)), AggOp.SUM)
        return out

    def grad_terms(self, spec, glob):
        return {"mu": self.alpha, "ctrl_c": True, "cc": -1.0}

    def finalize_group(self, spec, go, w0, glob, state_work):
        G = len(go.n)
        new_h = torch.empty_like(go.w_out)
        K.delta_affine(new_h, go.w_out, w0, _per_client(np.full(G, -self.alpha), go.w_out.device),
                       dmat=state_work, d=1.0)
        return [spec_groups(spec, go.w_out, AggOp.SIMPLE_AVERAGE, np.ones(G))], new_h

    def local_gradient(self, model, xb, yb, ctx):
        loss, gw, gb = loss_and_grad(model, xb, yb)
        x = ctx.start_model
        gw = gw - _as_dev(ctx.state["grad_corr_weights"]) + self.alpha * (model.weights - x.weights)
        gb = gb - _as_dev(ctx.state["grad_corr_bias"]) + self.alpha * (model.bias - x.bias)
        return loss, gw, gb

    def finalize(self, end_model, steps, ctx, n_samples):
        x, y = ctx.start_model, end_model
        new_hw = _as_dev(ctx.state["grad_corr_weights"]) - self.alpha * (y.weights - x.weights)
        new_hb = _as_dev(ctx.state["grad_corr_bias"]) - self.alpha * (y.bias - x.bias)
        return (_model_bundle(y, AggOp.SIMPLE_AVERAGE),
                {"grad_corr_weights": new_hw, "grad_corr_bias": new_hb})

    def server_update(self, old_global, agg):
        out = {}
        af = self.alpha * self.client_fraction
        for n in self._names():
            x = old_global.tensor(n)
            avg = agg.bundle.tensor(n)
            h = old_global.tensor("server_h_" + n)
            new_h = K.lincomb(torch.empty_like(h), h, 1.0, avg, -af, x, af)
            out["server_h_" + n] = new_h
            out[n] = K.lincomb(torch.empty_like(x), avg, 1.0, new_h, -1.0 / self.alpha)
        return old_global.replaced(**out)


PLUGINS: dict[str, type[AlgorithmPlugin]] = {
    cls.name: cls for cls in (FedAvg, FedProx, FedNova, Scaffold, FedDyn)}


def make_plugin(name: str, **hyper) -> AlgorithmPlugin:
    cls = PLUGINS.get(name.lower())
    if cls is None:
        raise ValueError(f"unknown algorithm {name!r}; available: {sorted(PLUGINS)}")
    return cls(**hyper)


def uses_hooks(plugin: AlgorithmPlugin) -> bool:
    """True for a reference-style plugin: it customises the per-minibatch
    hooks (``local_gradient`` / ``finalize``) rather than the fused device
    terms, so its clients run one by one through those hooks.  A plugin with
    neither raises a ConfigError naming what is missing."""
    cls = type(plugin)
    builtin = next((b for b in cls.__mro__ if b in _BUILTIN), None)
    if builtin is not None:
        return (cls.local_gradient is not builtin.local_gradient
                or cls.finalize is not builtin.finalize)
    fused = cls.finalize_group is not AlgorithmPlugin.finalize_group
    hooks = (cls.local_gradient is not AlgorithmPlugin.local_gradient
             and cls.finalize is not AlgorithmPlugin.finalize)
    if not fused and not hooks:
        from .core import ConfigError
        raise ConfigError(f"plugin {getattr(plugin, 'name', cls.__name__)!r} implements neither the "
                          "reference hooks (local_gradient + finalize) nor the fused device hooks "
                          "(grad_terms + finalize_group)")
    return not fused


_BUILTIN = frozenset(PLUGINS.values())


def hook_client_execute(plugin: AlgorithmPlugin, client_id: int, X: torch.Tensor, Y: torch.Tensor,
                        global_bundle: ParamBundle, state: ClientState | None, epochs: int,
                        batch_size: int, lr: float, seed: int, round_num: int) -> TrainReport:
    """client_execute (fedsim/trainer.py:427-477) through the plugin's own
    per-minibatch hooks, on the GPU: the same stream-6 permutations, partial
    last batch, ``w -= lr * g`` steps and finalize; X [n, F] fp32 and Y [n]
    are the client's device rows.  The loss is accumulated on the device and
    checked once at the end (a diverged step makes the sum non-finite)."""
    if epochs < 1:
        raise ValueError("epochs must be >= 1")
    from .core import stream_rng
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    n = int(X.shape[0])
    start = global_bundle.model()
    ctx = LocalContext(start_model=start, global_bundle=global_bundle,
                       state=state.payload if state is not None else None, lr=lr, n_samples=n)
    rng = stream_rng(seed, STREAM_MINIBATCH, client_id, round_num)
    bs = n if batch_size <= 0 else min(batch_size, n)
    Y = Y.long()
    w, b = start.weights.clone(), start.bias.clone()
    steps = 0
    loss_total = torch.zeros((), dtype=torch.float64, device=w.device)
    for _ in range(epochs):
        order = torch.from_numpy(rng.permutation(n)).to(w.device)
        for lo in range(0, n, bs):
            batch = order[lo:lo + bs]
            loss, gw, gb = plugin.local_gradient(_model_unchecked(w, b), X[batch], Y[batch], ctx)
            w = w - lr * _as_dev(gw)
            b = b - lr * _as_dev(gb)
            loss_total = loss_total + loss
            steps += 1
    mean_loss = float(loss_total.item()) / steps
    if not np.isfinite(mean_loss):
        raise NonFiniteLossError(f"client {client_id} round {round_num}: loss diverged")
    result, payload = plugin.finalize(ModelParams(w, b), steps, ctx, n)
    if plugin.collect_local_loss:
        result._put("local_loss", torch.tensor([mean_loss], dtype=torch.float32, device=w.device),
                    AggOp.COLLECT, client_id=client_id)
    new_state = None
    if payload is not None:
        new_state = ClientState(client_id, round_num, payload)
    torch.cuda.synchronize()
    return TrainReport(client_result=result, new_state=new_state, samples_processed=epochs * n,
                       measured_seconds=max(time.perf_counter() - t0, 1e-9))


def spec_of_bundle(bundle: ParamBundle, plugin: AlgorithmPlugin | None = None) -> ModelSpec:
    if plugin is not None and plugin.spec is not None:
        return plugin.spec
    if "weights" in bundle.entries and "bias" in bundle.entries:
        w = bundle.tensor("weights")
        return lr_spec(w.shape[0], w.shape[1])
    if "fc2_w" in bundle.entries:
        return cnn_spec(bundle.tensor("fc2_w").shape[0])
    if "fc_w" in bundle.entries and "l4.1.conv2_w" in bundle.entries:
        return resnet_spec(bundle.tensor("fc_w").shape[0])
    raise ValueError("cannot infer the model layout from the bundle")


def finalize_results(plugin: AlgorithmPlugin, spec: ModelSpec, go: GroupOutcome, w0: torch.Tensor,
                     glob: ParamBundle, state_work):
    groups, new_state = plugin.finalize_group(spec, go, w0, glob, state_work)
    if plugin.collect_local_loss:
        loss = _per_client(go.loss_mean, go.w_out.device).view(-1, 1)
        groups.append(ResultGroup(["local_loss"], [(0, 1, (1,))], loss, AggOp.COLLECT,
                                  np.ones(len(go.n))))
    return groups, new_state


def client_execute(plugin: AlgorithmPlugin, client: ClientProfile, global_bundle: ParamBundle,
                   state: ClientState | None, epochs: int, batch_size: int, lr: float,
                   seed: int, round_num: int) -> TrainReport:
    """One client's E local epochs (fedsim/trainer.py:427-477) on the GPU."""
    if epochs < 1:
        raise ValueError("epochs must be >= 1")
    if uses_hooks(plugin):
        d = device()
        part = client.data_partition
        return hook_client_execute(
            plugin, client.client_id,
            torch.from_numpy(np.asarray(part.features, dtype=np.float32)).to(d),
            torch.from_numpy(np.asarray(part.labels, dtype=np.int64)).to(d),
            global_bundle, state, epochs, batch_size, lr, seed, round_num)
    spec = spec_of_bundle(global_bundle, plugin)
    data = ClientData.from_profiles([client], n_classes=spec.n_classes)
    w0 = global_bundle.flat(spec)
    work = None
    if plugin.is_stateful and state is not None:
        work = torch.cat([_as_dev(state.payload[n]).reshape(-1)
                          for n in plugin.state_names(spec)]).view(1, -1)
    go = train_group(plugin, spec, data, [client.client_id], w0, global_bundle, work, epochs,
                     batch_size, lr, seed, round_num)
    groups, new_rows = finalize_results(plugin, spec, go, w0, global_bundle, work)
    bundle = client_bundle(groups, 0, client.client_id)
    new_state = None
    if new_rows is not None:
        payload = {plugin.state_prefix + n: new_rows[0, o:o + s].view(sh)
                   for n, o, s, sh in spec.columns()}
        new_state = ClientState(client.client_id, round_num, payload)
    return TrainReport(client_result=bundle, new_state=new_state,
                       samples_processed=epochs * client.sample_count,
                       measured_seconds=go.seconds)


# ---------------------------------------------------------------------------
# evaluation
# ---------------------------------------------------------------------------

_EVAL_CACHE: dict = {}


def _eval_tensors(ds):
    """Device copy of an eval set, uploaded once per dataset object."""
    hit = _EVAL_CACHE.get(id(ds))
    if hit is None or hit[0]() is not ds:
        d = device()
        hit = (weakref.ref(ds),
               torch.from_numpy(np.asarray(ds.features, dtype=np.float32)).to(d),
               torch.from_numpy(np.asarray(ds.labels, dtype=np.int32)).to(d))
        _EVAL_CACHE[id(ds)] = hit
        weakref.finalize(ds, _EVAL_CACHE.pop, id(ds), None)
    return hit[1], hit[2]


def evaluate(model, ds) -> tuple[float, float]:
    """Held-out accuracy and mean cross-entropy (fedsim/trainer.py:148-158)."""
    if isinstance(model, ModelParams):
        C, F = model.weights.shape
        if ds.features.shape[1] != F or ds.n_classes != C:
            raise ValueError(f"model ({tuple(model.weights.shape)}) does not match dataset "
                             f"({ds.features.shape[1]} features, {ds.n_classes} classes)")
        X, Y = _eval_tensors(ds)
        w = torch.cat([model.weights.reshape(-1), model.bias.reshape(-1)])
        return K.lr_eval(X, Y, w, F, C)
    if isinstance(model, NamedParams) and model.spec.kind == "cnn":
        from .cnn import cnn_evaluate
        X, Y = _eval_tensors(ds)
        return cnn_evaluate(model, X, Y)
    if isinstance(model, NamedParams) and model.spec.kind == "resnet":
        from .resnet import resnet_evaluate
        X, Y = _eval_tensors(ds)
        return resnet_evaluate(model, X, Y)
    raise TypeError(f"cannot evaluate {type(model).__name__}")
