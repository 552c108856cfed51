"""paper_2303_01778_b200 -- a B200-native device-side hot path for FedML
Parrot's federated-learning simulator (arXiv 2303.01778).

Drop-in for the reference package ``fedsim`` on the Parrot path: the same
public names (``fedsim/__init__.py:85-140``), with client training, local and
global aggregation and the client-state store executed by hand-written
sm_100a kernels in ``libparrot_b200.so`` (C ABI: include/parrot_b200.h).
Selection, workload fits and the greedy schedule stay on the host and are
bit-identical to the reference.

Host-only modules (core, data, estimate, schedule, metrics) import without a
GPU; the device modules need CUDA and the built library and fail loudly
otherwise -- there is no CPU fallback.
"""

from .core import (ALL_HISTORY, CLOCK_MODES, SCHEDULING_MODES, SCHEMES, ClientProfile,
                   ClientSelection, ConfigError, DataSlice, SimConfig, select_clients, stream_rng)
from .data import PartitionSpec, SyntheticDataset, export_partitions, generate, partition
from .estimate import TimingHistory, TimingRecord, WorkloadFit, estimation_error, fit_device
from .metrics import CostLedger, expected_costs, reconcile, scheme_formulas
from .schedule import RoundPlan, greedy_assign, makespan, schedule, uniform_division

__version__ = "0.1.0"

_DEVICE_NAMES = {
    "aggregate": ("AggregateResult", "DevicePartial", "flat_aggregate", "global_fold",
                  "local_fold", "server_update"),
    "engine": ("DeviceModel", "RoundOutcome", "SimulationEngine", "make_device_models"),
    "statestore": ("ClientState", "StateStore"),
    "trainer": ("PLUGINS", "AggOp", "FedAvg", "FedDyn", "FedNova", "FedProx", "ModelParams",
                "ParamBundle", "Scaffold", "client_execute", "evaluate", "make_plugin"),
}


def __getattr__(name):
    """Device-side names load lazily (they import torch and the native lib)."""
    import importlib
    for mod, names in _DEVICE_NAMES.items():
        if name in names:
            return getattr(importlib.import_module(f".{mod}", __name__), name)
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")


__all__ = sorted([
    "ALL_HISTORY", "CLOCK_MODES", "SCHEDULING_MODES", "SCHEMES", "ClientProfile",
    "ClientSelection", "ConfigError", "CostLedger", "DataSlice", "PartitionSpec", "RoundPlan",
    "SimConfig", "SyntheticDataset", "TimingHistory", "TimingRecord", "WorkloadFit",
    "estimation_error", "expected_costs", "export_partitions", "fit_device", "generate",
    "greedy_assign", "makespan", "partition", "reconcile", "scheme_formulas", "schedule",
    "select_clients", "stream_rng", "uniform_division",
    *[n for names in _DEVICE_NAMES.values() for n in names],
])
