"""Round driver: select -> fit -> schedule (host, bit-exact) -> batched device
execution -> hierarchical fold -> server rule -> evaluate.

Reference: ``fedsim/engine.py`` (PARROT branch of ``SimulationEngine.run_round``
at :748-812 and ``DeviceWorker.execute_clients`` at :470-503, the device seam).
What changes is the device side:

* the K simulated devices of a process share the GPU; all their clients of a
  round train in ONE batched launch (``train_group``), then each device's
  clients are folded into that device's partial in plan order
  (``fold_group``), which is exactly the reference's sequential
  load-train-save-fold loop reordered -- legal because a round never places
  a client on two devices and minibatch order depends only on
  (seed, client, round);
* stateful algorithms gather/scatter client state through the HBM store;
* with ``torch.distributed`` initialised (one process per GPU, NCCL), rank r
  executes the devices k with k % world == r and the per-device partials are
  combined with ONE all-reduce of the packed partial (kernel (d)); every rank
  then applies the same server rule, so the global model stays replicated.

Timing under the virtual clock (default) is the reference's synthetic model
(``virtual_task_seconds`` + ``report_time``), so fits, plans and device loads
are bit-identical to the reference's.  The in-process byte channel and wire
codec of the reference are not rebuilt (NCCL replaces them).
"""

from __future__ import annotations

import math
import os
import sys
import threading
import time
from dataclasses import dataclass
from pathlib import Path
from typing import Sequence

import numpy as np
import torch

from .aggregate import (DevicePartial, PartialEntry, fold_group, global_fold, local_fold,
                        partial_byte_roles, server_update)
from .core import (STREAM_NOISE, ClientProfile, ConfigError, SimConfig, select_clients,
                   stream_rng)
from .estimate import (InsufficientDataError, TimingHistory, TimingRecord, WorkloadFit,
                       estimation_error, fit_device, record)
from .metrics import CostLedger, ReplicaGauge
from .models import ModelSpec, init_params, spec_for
from .schedule import MODE_GREEDY, RoundPlan, schedule, uniform_division, warm_jit
from .statestore import StateStore
from .trainer import (AggOp, AlgorithmPlugin, ClientData, FedAvg, GroupInputs, ModelParams, NamedParams,
                      NonFiniteLossError, ParamBundle, device, evaluate, finalize_results, hook_client_execute, io_bytes,
                      spec_of_bundle, train_group, uses_hooks)

RESULTS_HEADER = ("round\tscheme\tscheduling\tsim_seconds\twall_seconds\t"
                  "device_loads\ttrips_up\ttrips_down\tbytes_avg\tbytes_special\t"
                  "accuracy\tloss\test_error")


class DeviceFailureError(RuntimeError):
    """A device's client execution raised; the round aborts with the cause."""


_TRACE = os.environ.get("PB_TRACE_ROUND") == "1"   # per-round host timeline on stderr (diagnostics)


_PREWARMED = False


def _prewarm_small_pool(blocks: int = 96) -> None:
    """Reserve small-block segments of torch's caching allocator once: the
    per-round input uploads (< 1 MB each) then never hit a fresh cudaMalloc,
    which was measured to stall a round's launch by up to ~100 ms."""
    global _PREWARMED
    if _PREWARMED or not torch.cuda.is_available():
        return
    _PREWARMED = True
    d = device()
    # small pool (<= 1 MB requests, 2 MB segments) and the 1-10 MB class of
    # the large pool (20 MB segments): per-round inputs / partials live there
    keep = [torch.empty(1 << 20, dtype=torch.uint8, device=d) for _ in range(blocks)]
    keep += [torch.empty(4 << 20, dtype=torch.uint8, device=d) for _ in range(blocks // 2)]
    del keep

@dataclass(frozen=True)
class DeviceModel:
    """fedsim/engine.py:380-403: identity plus injected timing behaviour."""

    device_id: int
    hetero_ratio: float = 0.0
    dynamic: bool = False
    t_true: float = 1e-4
    b_true: float = 0.0
    noise: float = 0.0

    def __post_init__(self) -> None:
        if self.device_id < 0:
            raise ConfigError("device_id must be >= 0")
        if self.hetero_ratio < 0:
            raise ConfigError(f"device {self.device_id}: hetero_ratio must be >= 0")
        if self.t_true <= 0 or self.b_true < 0 or self.noise < 0:
            raise ConfigError(f"device {self.device_id}: bad ground-truth timing")


def make_device_models(k: int, hetero=0.0, dynamic: bool = False, t_true=1e-4, b_true=0.0,
                       noise: float = 0.0) -> list[DeviceModel]:
    def per_device(v, label):
        if np.isscalar(v):
            return [float(v)] * k
        vals = [float(x) for x in v]
        if len(vals) != k:
            raise ConfigError(f"{label} needs {k} values, got {len(vals)}")
        return vals

    het, ts, bs = per_device(hetero, "hetero"), per_device(t_true, "t_true"), per_device(b_true, "b_true")
    return [DeviceModel(i, het[i], dynamic, ts[i], bs[i], noise) for i in range(k)]


def report_time(measured_seconds: float, device: DeviceModel, round_num: int,
                total_rounds: int) -> float:
    """measured*(1+eta_k), times (1+cos(3.14 r/R + k)) for dynamic devices, floor 1e-9."""
    if measured_seconds <= 0:
        raise ValueError("measured_seconds must be > 0")
    out = measured_seconds * (1.0 + device.hetero_ratio)
    if device.dynamic:
        out *= 1.0 + math.cos(3.14 * round_num / total_rounds + device.device_id)
    return max(out, 1e-9)


def virtual_task_seconds(device: DeviceModel, sample_count: int, seed: int, round_num: int,
                         client_id: int) -> float:
    """N*t_true + b_true with optional relative noise from stream 4."""
    base = sample_count * device.t_true + device.b_true
    if device.noise > 0:
        eps = stream_rng(seed, STREAM_NOISE, round_num, device.device_id, client_id).standard_normal()
        base *= 1.0 + device.noise * eps
    return max(base, 1e-9)


@dataclass
class RoundInputs:
    """Everything the host decides for one round before the device runs it."""

    round: int
    selection: object
    sizes: dict
    fits: dict | None
    fit_seconds: float
    schedule_seconds: float
    plan: RoundPlan
    fa_tasks: list | None
    assign: dict
    group: GroupInputs | None
    wall0: float
    records: list | None = None   # virtual-clock timing records, committed at hand-out
    executed: list | None = None  # multi-process: every rank's clients (state exchange)

    def upload(self) -> "RoundInputs":
        if self.group is not None:
            self.group.upload()
        return self


@dataclass
class RoundOutcome:
    round: int
    scheme: str
    scheduling_mode: str
    simulated_round_seconds: float
    wall_seconds: float
    device_loads: dict
    costs: CostLedger
    accuracy: float
    loss: float
    estimation_error: float
    fit_seconds: float
    schedule_seconds: float
    new_global: ParamBundle
    device_seconds: float = 0.0     # GPU time of the round's training launch(es)


def append_results(path: str | Path, outcome: RoundOutcome) -> None:
    path = Path(path)
    fresh = not path.exists() or path.stat().st_size == 0
    loads = ",".join(f"{outcome.device_loads[k]:.9g}" for k in sorted(outcome.device_loads))
    row = "\t".join([str(outcome.round), outcome.scheme, outcome.scheduling_mode,
                     f"{outcome.simulated_round_seconds:.9g}", f"{outcome.wall_seconds:.9g}",
                     loads, str(outcome.costs.trips_up), str(outcome.costs.trips_down),
                     str(outcome.costs.bytes_avg_params), str(outcome.costs.bytes_special_params),
                     f"{outcome.accuracy:.9g}", f"{outcome.loss:.9g}",
                     f"{outcome.estimation_error:.9g}"])
    with open(path, "a", encoding="utf-8") as fh:
        if fresh:
            fh.write(RESULTS_HEADER + "\n")
        fh.write(row + "\n")


# ---------------------------------------------------------------------------
# device runtime (the GPU-resident side of a process)
# ---------------------------------------------------------------------------

class DeviceRuntime:
    """Client data, state store and model layout shared by the local devices."""

    def __init__(self, cfg: SimConfig, plugin: AlgorithmPlugin, spec: ModelSpec, data: ClientData,
                 store: StateStore | None, gauge: ReplicaGauge):
        self.cfg, self.plugin, self.spec, self.data = cfg, plugin, spec, data
        self.store, self.gauge = store, gauge
        self.last_device_seconds = 0.0
        self.client_seconds: dict[int, float] = {}   # device-measured task time per client (real clock)
        self.batch_peak = 0   # most clients trained in one batched launch
        self.pending: GroupOutcome | None = None   # group whose result read is outstanding
        self.hooks = uses_hooks(plugin)
        self.shard = None   # distributed.ShardedState: stateful clients owned across ranks

    def resolve(self) -> None:
        """Complete the outstanding result read of the last group (raises on a
        diverged client)."""
        go, self.pending = self.pending, None
        if go is not None:
            go.resolve()
            self.last_device_seconds = go.seconds

    def prepare(self, assignments: dict[int, list[int]], round_num: int) -> GroupInputs | None:
        """Host side of a round for the local devices: minibatch row ids of all
        their clients (device order, then plan order)."""
        clients = [m for dev in sorted(assignments) for m in assignments[dev]]
        if not clients or self.hooks:
            return None
        return GroupInputs(self.data, clients, self.cfg.local_epochs, self.cfg.seed, round_num)

    def execute(self, assignments: dict[int, list[int]], bundle: ParamBundle,
                round_num: int, inputs: GroupInputs | None = None,
                executed: list[list[int]] | None = None) -> dict[int, DevicePartial]:
        """Train every assigned client of the local devices in one batched
        launch, then fold each device's clients in its plan order.
        ``executed`` (multi-process stateful rounds): every rank's clients,
        for the owner-sharded state exchange."""
        t_in = time.perf_counter()
        order = [(dev, m) for dev in sorted(assignments) for m in assignments[dev]]
        partials = {dev: DevicePartial(device_id=dev) for dev in assignments}
        self.last_device_seconds = 0.0
        if not order:
            if self.shard is not None:   # an idle rank still takes part in the state exchange
                width = self.spec.numel
                self.shard.gather(executed, torch.empty(0, width, device=device()))
                self._failure_vote(None, round_num)
                self.shard.scatter(executed, round_num, torch.empty(0, width, device=device()))
            return partials
        clients = [m for _, m in order]
        if len(set(clients)) != len(clients):
            raise ValueError(f"round {round_num}: a client is assigned twice")
        plugin, spec = self.plugin, self.spec
        if plugin.is_stateful and self.store is None:
            raise ConfigError(f"{plugin.name} is stateful and needs a state store")
        if self.hooks:
            return self._execute_hooks(assignments, bundle, round_num)
        w0 = bundle.flat(spec)
        work = None
        if plugin.is_stateful:
            if not self.store.configured:   # a fresh store behind a bare DeviceWorker
                self.store.configure(plugin.state_names(spec), [sh for *_, sh in spec.columns()],
                                     capacity=self.cfg.total_clients)
            work = torch.empty(len(clients), (spec.numel + 3) // 4 * 4, device=w0.device)[:, :spec.numel]
            if self.shard is not None:
                self.shard.gather(executed, work)
            else:
                self.store.gather(clients, work)
        # one live model replica per busy simulated device (the reference's
        # Table-1 quantity); the batch itself is the GPU's real concurrency
        busy = sum(1 for dev in assignments if assignments[dev])
        self.batch_peak = max(self.batch_peak, len(clients))
        self.gauge.acquire(busy)
        try:
            # FedAvg folds exactly the end models: the CNN's low-rank fc1 can be
            # folded from the round's history without materialising them
            defer = spec.kind == "cnn" and type(plugin) is FedAvg
            # the group's result read (failures, losses, device time) can wait
            # for the end of the round unless something needs it now; a
            # stateful round reads it before its states are committed, so a
            # diverged client leaves the store untouched
            late = (self.cfg.clock == "virtual" and not plugin.collect_local_loss
                    and not plugin.is_stateful)
            err = None
            try:
                go = train_group(plugin, spec, self.data, clients, w0, bundle, work,
                                 self.cfg.local_epochs, plugin.batch_size, plugin.lr, self.cfg.seed,
                                 round_num, inputs=inputs, defer_fc1=defer, defer_check=late,
                                 timing=self.cfg.clock == "real")
            except Exception as exc:
                err = exc
            if self.shard is not None:
                self._failure_vote(err, round_num)
            elif err is not None:
                raise err
        finally:
            self.gauge.release(busy)
        t_tr = time.perf_counter()
        self.pending = go if go.pending is not None else None
        self.last_device_seconds = go.seconds
        self.client_seconds = ({} if go.client_seconds is None else
                               dict(zip(clients, go.client_seconds.tolist())))
        groups, new_state = finalize_results(plugin, spec, go, w0, bundle, work)
        t_fin = time.perf_counter()
        if go.lazy is not None:
            for g in groups:
                if g.op is AggOp.WEIGHTED_AVERAGE:
                    g.lazy = go.lazy
        if plugin.is_stateful and new_state is not None:
            if self.shard is not None:
                self.shard.scatter(executed, round_num, new_state)
            else:
                self.store.scatter(clients, round_num, new_state)
        pos = 0
        for dev in sorted(assignments):
            k = len(assignments[dev])
            fold_group(partials[dev], groups, list(range(pos, pos + k)), assignments[dev])
            pos += k
        if _TRACE:
            t_end = time.perf_counter()
            print(f"  execute: train_group {1e3 * (t_tr - t_in):.1f} finalize {1e3 * (t_fin - t_tr):.1f} "
                  f"fold {1e3 * (t_end - t_fin):.1f} ms", file=sys.stderr, flush=True)
        return partials

    def _failure_vote(self, err: Exception | None, round_num: int) -> None:
        """Multi-process stateful rounds: every rank learns whether any rank's
        clients diverged before a state is committed (one small all-reduce),
        so all ranks abort together instead of one hanging in the exchange."""
        import torch.distributed as dist
        flag = torch.tensor([0.0 if err is None else 1.0], device=device())
        dist.all_reduce(flag)
        if err is not None:
            raise err
        if flag.item() > 0:
            raise NonFiniteLossError(f"round {round_num}: a client on another rank diverged")

    def _execute_hooks(self, assignments: dict[int, list[int]], bundle: ParamBundle,
                       round_num: int) -> dict[int, DevicePartial]:
        """A reference-style plugin (``uses_hooks``): Algorithm 2's
        Device_Executes loop of fedsim/engine.py:470-503 -- load state, train
        through the plugin's hooks, save, fold -- one client at a time."""
        plugin, data, store = self.plugin, self.data, self.store
        partials = {dev: DevicePartial(device_id=dev) for dev in assignments}
        self.client_seconds = {}
        total = 0.0
        for dev in sorted(assignments):
            for m in assignments[dev]:
                state = None
                if plugin.is_stateful:
                    base = bundle.model()
                    state = store.load(m, default_factory=lambda: plugin.default_state(base))
                lo, n = int(data.row_base[m]), int(data.sizes[m])
                self.gauge.acquire()
                try:
                    rep = hook_client_execute(plugin, m, data.X[lo:lo + n], data.Y[lo:lo + n], bundle,
                                              state, self.cfg.local_epochs, plugin.batch_size,
                                              plugin.lr, self.cfg.seed, round_num)
                finally:
                    self.gauge.release()
                if plugin.is_stateful and rep.new_state is not None and rep.new_state.payload:
                    store.save(m, round_num, rep.new_state.payload)
                local_fold(partials[dev], rep.client_result, m)
                self.client_seconds[m] = rep.measured_seconds
                total += rep.measured_seconds
        self.last_device_seconds = total
        return partials


class DeviceWorker:
    """One simulated device (fedsim/engine.py:453-503): ``execute_clients``
    trains its clients (batched on the GPU) and folds them in order."""

    def __init__(self, device_model: DeviceModel, cfg: SimConfig, plugin: AlgorithmPlugin,
                 profiles: Sequence[ClientProfile], store: StateStore | None,
                 gauge: ReplicaGauge, channel=None, *, runtime: DeviceRuntime | None = None):
        self.device = device_model
        self.cfg, self.plugin, self.profiles, self.store, self.gauge = cfg, plugin, profiles, store, gauge
        self.channel = channel
        self._runtime = runtime

    def _rt(self, bundle: ParamBundle) -> DeviceRuntime:
        if self._runtime is None:
            spec = spec_of_bundle(bundle, self.plugin)
            data = ClientData.from_profiles(self.profiles, n_classes=spec.n_classes)
            self._runtime = DeviceRuntime(self.cfg, self.plugin, spec, data, self.store, self.gauge)
        return self._runtime

    def execute_clients(self, bundle: ParamBundle, clients: Sequence[int],
                        round_num: int) -> tuple[DevicePartial, list[TimingRecord]]:
        """fedsim/engine.py:470-503: the device's clients in plan order ->
        (partial, timing records).  Works on a fresh StateStore: the store's
        layout is declared from the plugin's state schema on first use."""
        rt = self._rt(bundle)
        partial = rt.execute({self.device.device_id: list(clients)}, bundle, round_num)[
            self.device.device_id]
        rt.resolve()
        timings = [TimingRecord(self.device.device_id, m, round_num,
                                int(rt.data.sizes[m]),
                                self._reported(rt, m, round_num, len(clients)))
                   for m in clients]
        return partial, timings

    def _reported(self, rt: DeviceRuntime, m: int, round_num: int, g: int) -> float:
        if self.cfg.clock == "virtual":
            measured = virtual_task_seconds(self.device, int(rt.data.sizes[m]), self.cfg.seed,
                                            round_num, m)
        else:   # device-measured per-client task time (kernel %globaltimer stamps)
            measured = rt.client_seconds[m]
        return report_time(measured, self.device, round_num, self.cfg.total_rounds)


# ---------------------------------------------------------------------------
# server loop
# ---------------------------------------------------------------------------

def result_schema(plugin: AlgorithmPlugin, spec: ModelSpec) -> list[tuple[str, AggOp, tuple]]:
    """The (name, op, shape) entries every client result carries."""
    cols = [(n, sh) for n, _, _, sh in spec.columns()]
    name = plugin.name
    if name in ("fedavg", "fedprox"):
        out = [(n, AggOp.WEIGHTED_AVERAGE, sh) for n, sh in cols]
    elif name == "fednova":
        out = [("direction_" + n, AggOp.WEIGHTED_AVERAGE, sh) for n, sh in cols]
        out.append(("step_scale", AggOp.SUM, (1,)))
    elif name == "scaffold":
        out = [("delta_" + n, AggOp.WEIGHTED_AVERAGE, sh) for n, sh in cols]
        out += [("ctrl_delta_" + n, AggOp.SIMPLE_AVERAGE, sh) for n, sh in cols]
    elif name == "feddyn":
        out = [(n, AggOp.SIMPLE_AVERAGE, sh) for n, sh in cols]
    else:
        raise ValueError(f"no result schema for plugin {name!r}")
    if plugin.collect_local_loss:
        out.append(("local_loss", AggOp.COLLECT, (1,)))
    return out


def _schema_of(partials) -> list[tuple[str, AggOp, tuple]]:
    """(name, op, shape) of the entries a hook plugin's results carried."""
    for p in partials:
        if p.entries:
            return [(n, pe.op, tuple(pe.acc.shape) if pe.acc is not None else
                     tuple(pe.collected[0][1].shape)) for n, pe in p.entries.items()]
    return []


class SimulationEngine:
    """Server loop with the reference's constructor and outputs
    (fedsim/engine.py:563-828), executing on the GPU.

    Extra keyword arguments: ``model`` ("lr" default, "cnn" or "resnet"),
    ``client_data`` (a prebuilt device ClientData), ``init_seed`` (CNN/ResNet init),
    ``eval_batch`` (unused for LR)."""

    def __init__(self, cfg: SimConfig, plugin: AlgorithmPlugin, profiles: Sequence[ClientProfile],
                 device_models: Sequence[DeviceModel], store: StateStore | None = None,
                 eval_data=None, results_path: str | Path | None = None, start_round: int = 0,
                 initial_global: ParamBundle | None = None, history: TimingHistory | None = None,
                 eval_every: int = 1, *, model: str | None = None,
                 client_data: ClientData | None = None, init_seed: int = 0):
        if len(profiles) != cfg.total_clients:
            raise ConfigError(f"need {cfg.total_clients} client profiles, got {len(profiles)}")
        if len(device_models) != cfg.num_devices:
            raise ConfigError(f"scheme {cfg.scheme} with K={cfg.num_devices} needs "
                              f"{cfg.num_devices} device models, got {len(device_models)}")
        if [d.device_id for d in device_models] != list(range(cfg.num_devices)):
            raise ConfigError("device ids must be 0..K-1 in order")
        if plugin.is_stateful and store is None:
            raise ConfigError(f"{plugin.name} is stateful and needs a state store")
        if not 0 <= start_round <= cfg.total_rounds:
            raise ConfigError(f"start_round {start_round} outside [0, {cfg.total_rounds}]")
        if cfg.scheme == "FA_DIST" and cfg.clock == "real":
            raise ConfigError("FA_DIST under the real clock is not supported on the device path")
        self.cfg, self.plugin = cfg, plugin
        self.profiles = list(profiles)
        self.devices = list(device_models)
        self.store, self.eval_data, self.results_path = store, eval_data, results_path
        self.eval_every = max(1, eval_every)
        self.history = history if history is not None else TimingHistory()
        self._prefetch = None       # (round, thread, result box) of a round prepared ahead
        self._after_enqueue = None  # run_round's hook: start that preparation
        self.gauge = ReplicaGauge()
        self.next_round = start_round
        self.sizes = np.array([p.sample_count for p in self.profiles], dtype=np.int64)
        self.data = client_data if client_data is not None else ClientData.from_profiles(self.profiles)
        if initial_global is not None:
            self.global_bundle = initial_global
            self.spec = spec_of_bundle(initial_global, plugin if plugin.spec else None)
            plugin.spec = self.spec
        else:
            self.spec = spec_for(model or "lr", self.data.n_features, self.data.n_classes)
            if self.spec.kind == "lr":
                start = ModelParams.zeros(self.spec.n_classes, self.spec.n_features)
            else:
                start = NamedParams.from_flat(self.spec, init_params(self.spec, init_seed))
            self.global_bundle = plugin.init_global(start)
        if plugin.is_stateful and not uses_hooks(plugin) and not store.configured:
            names = plugin.state_names(self.spec)
            store.configure(names, [sh for _, _, _, sh in self.spec.columns()], capacity=cfg.total_clients)
        self._world, self._rank = 1, 0
        if torch.distributed.is_available() and torch.distributed.is_initialized():
            self._world = torch.distributed.get_world_size()
            self._rank = torch.distributed.get_rank()
            if cfg.clock == "real":
                raise ConfigError("multi-process runs need the virtual clock (shared histories)")
            if uses_hooks(plugin) and self._world > 1:
                raise ConfigError(f"reference-style plugin {plugin.name!r} (per-minibatch hooks) runs "
                                  "single-process; multi-GPU rounds need a fused plugin")

        from .distributed import local_devices
        self.local_devices = local_devices(cfg.num_devices, self._world, self._rank)
        self.runtime = DeviceRuntime(cfg, plugin, self.spec, self.data, store, self.gauge)
        if plugin.is_stateful and self._world > 1:
            # the plan moves clients between ranks every round: each client's
            # state lives with its owner rank and travels around the round
            from .distributed import ShardedState
            self.runtime.shard = ShardedState(store, self._world, self._rank)
        _prewarm_small_pool()
        if cfg.scheme == "PARROT" and cfg.scheduling in ("full-history", "time-window"):
            warm_jit()

    # -- per-round pieces -------------------------------------------------------
    def _fit_all(self, round_num: int):
        if self.cfg.scheduling not in ("full-history", "time-window") \
                or round_num <= self.cfg.warmup_rounds:
            return None, 0.0
        window = self.cfg.time_window if self.cfg.scheduling == "time-window" else "all-history"
        t0 = time.perf_counter()
        fits: dict[int, WorkloadFit | None] = {}
        for k in range(self.cfg.num_devices):
            try:
                fits[k] = fit_device(self.history, k, window, round_num)
            except InsufficientDataError:
                fits[k] = None
        return fits, time.perf_counter() - t0

    def _reported(self, dev: int, m: int, round_num: int, measured: float | None = None) -> float:
        d = self.devices[dev]
        if measured is None:
            measured = virtual_task_seconds(d, int(self.sizes[m]), self.cfg.seed, round_num, m)
        return report_time(measured, d, round_num, self.cfg.total_rounds)

    def _fa_tasks(self, round_num: int, selected: Sequence[int]):
        """FA_DIST work pulling under the virtual clock (fedsim/engine.py:699-746):
        returns [(device, client)] in completion (= fold) order."""
        k = self.cfg.num_devices
        pending = list(selected)
        clocks = {d: 0.0 for d in range(k)}
        busy: dict[int, tuple[float, int]] = {}
        done = []
        idx = 0
        for d in range(min(k, len(pending))):
            busy[d] = (clocks[d] + self._reported(d, pending[idx], round_num), pending[idx])
            idx += 1
        while busy:
            d = min(busy, key=lambda x: (busy[x][0], x))
            t_end, m = busy.pop(d)
            clocks[d] = t_end
            done.append((d, m))
            if idx < len(pending):
                busy[d] = (clocks[d] + self._reported(d, pending[idx], round_num), pending[idx])
                idx += 1
        return done

    def _reduce_partials(self, partials: list[DevicePartial], schema,
                         inp: "RoundInputs") -> list[DevicePartial]:
        """Multi-process: ONE all-reduce of this rank's packed partials (NCCL);
        weight sums, counts and fold order come from the plan every rank holds
        (built-in plugins weight a client by its sample count)."""
        from . import _kernels as K
        from .distributed import allreduce_partials
        if inp.fa_tasks is not None:
            assign = {i: [m] for i, (_, m) in enumerate(inp.fa_tasks)}
        else:
            assign = {k: list(inp.plan.assignments.get(k, [])) for k in range(self.cfg.num_devices)}
        return [allreduce_partials(partials, schema, device=device(),
                                   fold=lambda acc, x: K.fold(acc, x, 1.0),
                                   assign=assign, weights=inp.sizes)]

    # -- the round ----------------------------------------------------------------
    def prepare_round(self, round_num: int) -> "RoundInputs":
        """Host half of a round: selection, workload fits, schedule, the
        virtual-clock timing records (added to the history now, exactly the
        records the reference's devices report) and the local clients'
        minibatch orders.  Deterministic in (seed, round, history).  A round
        already prepared ahead by run_round is handed out, never re-prepared
        (its timing records are in the history exactly once)."""
        inp = self._take_prefetch(round_num)
        if inp is None:
            inp = self._prepare(round_num)
        if self.cfg.clock == "virtual":
            self.history.add_many(inp.records)
        return inp

    # -- host/device overlap ---------------------------------------------------
    def _take_prefetch(self, round_num: int) -> "RoundInputs | None":
        pf = self._prefetch
        if pf is None:
            return None
        self._prefetch = None
        pf[1].join()
        if pf[0] != round_num:      # another round was asked for: drop it (no side effects)
            return None
        if "exc" in pf[2]:
            raise pf[2]["exc"]
        return pf[2]["inp"]

    def _start_prefetch(self, round_num: int) -> None:
        """Prepare ``round_num`` on a helper thread (virtual clock only: its
        plan and minibatch orders depend on the history up to the previous
        round, whose records are already in; its own records are added when
        the round is handed out, so an unconsumed prefetch leaves no trace)."""
        if self._prefetch is not None:
            return
        box: dict = {}

        def work():
            try:
                box["inp"] = self._prepare(round_num)
            except BaseException as exc:  # re-raised by the consumer
                box["exc"] = exc

        t = threading.Thread(target=work, name=f"prepare-round-{round_num}", daemon=True)
        self._prefetch = (round_num, t, box)
        t.start()

    def _prepare(self, round_num: int) -> "RoundInputs":
        cfg = self.cfg
        wall0 = time.perf_counter()
        selection = select_clients(cfg, round_num)
        sizes = {m: int(self.sizes[m]) for m in selection.selected}
        fits, fit_seconds = self._fit_all(round_num)
        t0 = time.perf_counter()
        fa_tasks = None
        if cfg.scheme in ("SP", "SD_DIST"):
            plan = uniform_division(round_num, selection, cfg.num_devices)
        elif cfg.scheme == "PARROT":
            plan = schedule(round_num, selection, fits, sizes, cfg)
        else:
            plan = RoundPlan(round=round_num, assignments={}, predicted_loads={},
                             mode="work-pulling")
            fa_tasks = self._fa_tasks(round_num, selection.selected)
        schedule_seconds = time.perf_counter() - t0
        if fa_tasks is not None:
            mine = [(i, dev, m) for i, (dev, m) in enumerate(fa_tasks)
                    if dev % self._world == self._rank]
            assign = {i: [m] for i, _, m in mine}
        else:
            assign = {k: list(plan.assignments.get(k, [])) for k in self.local_devices}
        inp = RoundInputs(round_num, selection, sizes, fits, fit_seconds, schedule_seconds, plan,
                          fa_tasks, assign, self.runtime.prepare(assign, round_num), wall0)
        if self._world > 1 and self.plugin.is_stateful:
            from .distributed import rank_clients
            if fa_tasks is not None:
                raise ConfigError("FA_DIST with a stateful plugin runs single-process")
            inp.executed = rank_clients(plan.assignments, cfg.num_devices, self._world)
        if cfg.clock == "virtual":   # built here (possibly on the helper thread), added at hand-out
            inp.records = self._records(inp, None)
        return inp

    def _records(self, inp: "RoundInputs", measured: dict | None) -> list:
        """Timing records in the reference's order: device order, plan order
        (fedsim/engine.py:689-697), or completion order for FA_DIST.
        ``measured`` (real clock): client -> device-measured task seconds."""
        r = inp.round
        if inp.fa_tasks is not None:
            tasks = list(inp.fa_tasks)
        else:
            tasks = [(dev, m) for dev in range(self.cfg.num_devices)
                     for m in inp.plan.assignments.get(dev, [])]
        return [TimingRecord(dev, m, r, inp.sizes[m],
                             self._reported(dev, m, r, None if measured is None else measured[m]))
                for dev, m in tasks]

    def _record(self, inp: "RoundInputs", measured: dict | None) -> None:
        for rec in self._records(inp, measured):
            record(self.history, rec)

    def _measured_seconds(self, inp: "RoundInputs") -> dict:
        """Real clock: each client's task time as measured on the device
        (DeviceRuntime.client_seconds; FA_DIST runs virtual-only)."""
        got = self.runtime.client_seconds
        missing = [m for m in inp.selection.selected if m not in got]
        if missing:
            raise DeviceFailureError(f"no device timing for clients {missing[:5]}")
        return got

    def execute_round(self, inp: "RoundInputs", sync: bool = True) -> RoundOutcome:
        """Device half of a round: batched training, hierarchical fold,
        (multi-GPU) partial all-reduce, server rule, evaluation.

        A device failure (e.g. a diverged client) raises DeviceFailureError
        and leaves the engine as it was before the round, as the reference
        does (it raises before any aggregation, fedsim/engine.py:684-687): the
        global model is only replaced once the round's result read succeeded,
        client states are committed only after it (stateful rounds read their
        results before the scatter), and the round's timing records and any
        prefetched next round are dropped."""
        cfg, round_num = self.cfg, inp.round
        trace = _TRACE and [(time.perf_counter(), "start")]
        ledger = CostLedger(round=round_num, scheme=cfg.scheme)
        try:
            got = self.runtime.execute(inp.assign, self.global_bundle, round_num, inp.group,
                                       inp.executed)
        except Exception as exc:
            self._abort_round(round_num)
            raise DeviceFailureError(f"device {self._rank} failed: {exc!r}") from exc
        if trace:
            trace.append((time.perf_counter(), "train+fold enqueued"))
        partials = [got[k] for k in sorted(inp.assign)]
        schema = (result_schema(self.plugin, self.spec) if not self.runtime.hooks
                  else _schema_of(partials))
        if cfg.clock == "real":
            self._record(inp, self._measured_seconds(inp))
        if self._world > 1:
            partials = self._reduce_partials(partials, schema, inp)
        agg = global_fold(partials)
        new_global = server_update(self.plugin, self.global_bundle, agg)

        # communication ledger at the reference's 8 B/element convention
        if cfg.scheme != "SP":
            avg_elems = sum(int(np.prod(sh)) for _, op, sh in schema if op is not AggOp.COLLECT)
            coll_elems = sum(int(np.prod(sh)) for _, op, sh in schema if op is AggOp.COLLECT)
            if inp.fa_tasks is not None:
                uploads = [[m] for _, m in inp.fa_tasks]
            else:
                uploads = [inp.plan.assignments.get(k, []) for k in range(cfg.num_devices)]
            for clients in uploads:
                ledger.add_downlink()
                ledger.add_uplink(8 * avg_elems if clients else 0, 8 * coll_elems * len(clients))

        loads = {dev: 0.0 for dev in range(cfg.num_devices)}
        for rec in self.history.round_records(round_num):
            loads[rec.device_id] += rec.reported_seconds
        sim_seconds = max(loads.values()) + cfg.trip_overhead_seconds * (
            ledger.trips_up + ledger.trips_down)
        est_err = float("nan")
        if inp.fits is not None and inp.plan.mode == MODE_GREEDY:
            est_err = estimation_error(self.history, inp.fits, round_num)
        accuracy = loss = float("nan")
        if self.eval_data is not None and (round_num % self.eval_every == 0
                                           or round_num == cfg.total_rounds - 1):
            accuracy, loss = evaluate(self.global_model(new_global), self.eval_data)
        ledger.peak_live_model_replicas = self.gauge.peak
        ledger.peak_device_batch = self.runtime.batch_peak
        if self.store is not None:
            ledger.state_bytes_disk = self.store.stats().bytes_on_disk
        # all of the round's device work is queued: the next round's host
        # preparation may start now (it then overlaps the wait below instead
        # of competing with this thread for the interpreter while enqueueing)
        cb, self._after_enqueue = self._after_enqueue, None
        if cb is not None:
            cb()
        if trace:
            trace.append((time.perf_counter(), "all enqueued"))
        try:
            self.runtime.resolve()   # the round's result read (queued after training)
        except Exception as exc:
            self._abort_round(round_num)
            raise DeviceFailureError(f"device {self._rank} failed: {exc!r}") from exc
        self.global_bundle = new_global
        if trace:
            trace.append((time.perf_counter(), "result read"))
        if sync and torch.cuda.is_available():
            torch.cuda.synchronize()
        if trace:
            trace.append((time.perf_counter(), "synced"))
            print("round", round_num, " ".join(f"{n}@{1e3 * (t - trace[0][0]):.1f}" for t, n in trace[1:]),
                  file=sys.stderr, flush=True)
        outcome = RoundOutcome(round=round_num, scheme=cfg.scheme, scheduling_mode=inp.plan.mode,
                               simulated_round_seconds=sim_seconds,
                               wall_seconds=time.perf_counter() - inp.wall0, device_loads=loads,
                               costs=ledger, accuracy=accuracy, loss=loss,
                               estimation_error=est_err, fit_seconds=inp.fit_seconds,
                               schedule_seconds=inp.schedule_seconds, new_global=new_global,
                               device_seconds=self.runtime.last_device_seconds)
        if self.results_path is not None and self._rank == 0:
            append_results(self.results_path, outcome)
        return outcome

    def _abort_round(self, round_num: int) -> None:
        """Undo a failed round's host-side traces: its timing records and a
        next round prepared ahead from them."""
        self._after_enqueue = None
        pf, self._prefetch = self._prefetch, None
        if pf is not None:
            pf[1].join()
        self.history.discard_round(round_num)
        self.runtime.pending = None

    def run_round(self, round_num: int) -> RoundOutcome:
        """One round through the public API.  Under the virtual clock the
        next round's host half (selection, fits, schedule, minibatch orders)
        runs on a helper thread while this round's kernels execute (started
        once the round's device work is queued)."""
        inp = self.prepare_round(round_num)
        if self.cfg.clock == "virtual" and round_num + 1 < self.cfg.total_rounds:
            self._after_enqueue = lambda: self._start_prefetch(round_num + 1)
        return self.execute_round(inp)

    @staticmethod
    def io_bytes() -> tuple[int, int]:
        """(host->device, device->host) bytes of round inputs/results so far."""
        return io_bytes()

    def global_model(self, bundle: ParamBundle | None = None):
        bundle = self.global_bundle if bundle is None else bundle
        if self.spec.kind == "lr":
            return bundle.model()
        return NamedParams(self.spec, bundle.named_model(self.spec))

    def run(self, rounds: int | None = None) -> list[RoundOutcome]:
        remaining = self.cfg.total_rounds - self.next_round
        count = remaining if rounds is None else min(rounds, remaining)
        out = []
        for _ in range(count):
            out.append(self.run_round(self.next_round))
            self.next_round += 1
        if self.store is not None:
            self.store.flush()
        return out
