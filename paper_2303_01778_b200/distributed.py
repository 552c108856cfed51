"""Multi-GPU plumbing for the round: which simulated devices a rank executes,
and the one collective of a round -- the all-reduce of the packed per-device
partial sums (kernel (d) of the north star).

One process per GPU (``torch.distributed``, NCCL over NVLink 5 / NVSwitch).
Every rank computes the same selection, fits and plan (host-side, bit-exact),
executes the devices ``k`` with ``k % world == rank`` and folds them locally
in device order.  Everything else a device partial carries besides the sums
is host-known on every rank: the weight sums (the clients' sample counts),
the counts and the fold order follow from the plan.  So a round exchanges
exactly ONE buffer, with ONE ``all_reduce`` and no host synchronisation:

    [acc of every averaged entry | Collect values at their global plan slots]

(the Collect slots are zero except where this rank wrote its own clients'
values, so the sum is the gather).  Every rank then applies the same server
rule, so the global model stays replicated without a broadcast (the
reference's downlink, ``fedsim/engine.py:680-697``).  NCCL's reduction order
differs from the reference's device-order sum (``fedsim/aggregate.py:130-132``),
so cross-world parity is tolerance-based.

The functions take the device and the fold as parameters so the packing logic
is exercised by world-size-2 ``gloo`` tests on CPU (tests/test_distributed_cpu.py).
"""

from __future__ import annotations

from typing import Callable, Mapping, Sequence

import numpy as np
import torch


def local_devices(num_devices: int, world: int, rank: int) -> list[int]:
    """Simulated devices executed by ``rank`` (round-robin over ranks)."""
    return [k for k in range(num_devices) if k % world == rank]


def allreduce_partials(partials: Sequence, schema, *, device, fold: Callable,
                       assign: Mapping[int, Sequence[int]], weights: Mapping[int, float],
                       group=None):
    """Combine this rank's device partials with every other rank's.

    ``schema`` is [(name, AggOp, shape)] (every client result carries these);
    ``fold(acc, x)`` accumulates ``x`` into ``acc`` (the fold kernel on the GPU,
    ``Tensor.add_`` in CPU tests); ``assign`` is the round's whole plan
    {device: clients in plan order} (all ranks, all devices) and ``weights``
    each client's WeightedAverage weight (its sample count).  Returns one
    DevicePartial with the global sums, weight sums, counts, Collect items and
    fold order, identical on every rank."""
    import torch.distributed as dist

    from .aggregate import DevicePartial, PartialEntry
    from .trainer import AggOp

    order = [m for dev in sorted(assign) for m in assign[dev]]   # global fold order
    slot = {m: i for i, m in enumerate(order)}
    live = [p for p in partials if p.entries]
    sizes = [int(np.prod(sh)) for _, _, sh in schema]
    width = sum(sz if op is not AggOp.COLLECT else sz * len(order)
                for (_, op, _), sz in zip(schema, sizes))
    packed = torch.zeros(width, dtype=torch.float32, device=device)
    views, pos = [], 0
    for (name, op, shape), size in zip(schema, sizes):
        n = size if op is not AggOp.COLLECT else size * len(order)
        view = packed[pos:pos + n]
        pos += n
        views.append(view)
        if op is AggOp.COLLECT:
            items = [(c, t) for p in live if name in p.entries for c, t in p.entries[name].collected]
            if items:
                idx = torch.tensor([slot[c] for c, _ in items], dtype=torch.int64, device=device)
                vals = torch.stack([t.reshape(-1).to(device, torch.float32) for _, t in items])
                view.view(len(order), size).index_copy_(0, idx, vals)
            continue
        for p in live:   # this rank's devices, in device order
            pe = p.entries.get(name)
            if pe is not None:
                fold(view, pe.acc.reshape(-1))
    dist.all_reduce(packed, group=group)     # the round's one collective

    out = DevicePartial(device_id=dist.get_rank(group))
    wsum = 0.0
    for dev in sorted(assign):          # per-device sums in device order, as global_fold adds them
        wsum += float(sum(float(weights[m]) for m in assign[dev]))
    for (name, op, shape), size, view in zip(schema, sizes, views):
        if op is AggOp.COLLECT:
            vals = view.view(len(order), *shape)
            out.entries[name] = PartialEntry(op=op, collected=[(m, vals[i]) for i, m in enumerate(order)],
                                             count=len(order))
            continue
        out.entries[name] = PartialEntry(op=op, acc=view.view(shape),
                                         weight_sum=wsum if op is AggOp.WEIGHTED_AVERAGE else 0.0,
                                         count=len(order))
    out.clients_folded = list(order)
    return out


def rank_clients(assign: Mapping[int, Sequence[int]], num_devices: int, world: int) -> list[list[int]]:
    """The clients each rank trains in a round, in its work-row order (its
    devices in device order, each in plan order -- DeviceRuntime.execute)."""
    return [[m for dev in local_devices(num_devices, world, r) for m in assign.get(dev, [])]
            for r in range(world)]


class ShardedState:
    """Stateful clients across ranks: client m's state lives in the store of
    its owner rank ``m % world`` (HBM, optionally FSST files -- owners write
    disjoint files), while the plan may train it on any rank.  Around a round
    the rows travel by two ``all_to_all`` exchanges whose split sizes every
    rank knows from the plan (no size handshake, no host sync):

    * gather:  owners -> executing ranks, into the work rows;
    * scatter: executing ranks -> owners, then the owners' scatter kernels
      commit them (stale-write guard and file writes at the owner).

    A client trained on its own owner rank still goes through its own split
    of the exchange (a self copy)."""

    def __init__(self, store, world: int, rank: int, group=None):
        self.store, self.world, self.rank, self.group = store, world, rank, group

    def owner(self, m: int) -> int:
        return int(m) % self.world

    def _plan(self, executed: Sequence[Sequence[int]]):
        me, W = self.rank, self.world
        outgoing = [[m for m in executed[r] if self.owner(m) == me] for r in range(W)]
        incoming = [[m for m in executed[me] if self.owner(m) == o] for o in range(W)]
        return outgoing, incoming

    def gather(self, executed: Sequence[Sequence[int]], work: torch.Tensor) -> None:
        """work rows [G, width] <- the states of this rank's clients
        (executed[rank] order), zeros for never-saved clients."""
        import torch.distributed as dist
        outgoing, incoming = self._plan(executed)
        width, dev = work.size(1), work.device
        send_ids = [m for lst in outgoing for m in lst]
        send = torch.empty(len(send_ids), width, dtype=work.dtype, device=dev)
        if send_ids:
            self.store.gather(send_ids, send)
        recv_ids = [m for lst in incoming for m in lst]
        recv = torch.empty(len(recv_ids), width, dtype=work.dtype, device=dev)
        dist.all_to_all_single(recv, send, [len(x) for x in incoming], [len(x) for x in outgoing],
                               group=self.group)
        at = {m: i for i, m in enumerate(recv_ids)}
        perm = torch.tensor([at[m] for m in executed[self.rank]], dtype=torch.int64, device=dev)
        work.copy_(recv.index_select(0, perm))

    def scatter(self, executed: Sequence[Sequence[int]], round_num: int, rows: torch.Tensor) -> None:
        """The new states ``rows`` (executed[rank] order) go home and are
        committed by their owners for ``round_num``."""
        import torch.distributed as dist
        outgoing, incoming = self._plan(executed)
        width, dev = rows.size(1), rows.device
        at = {m: i for i, m in enumerate(executed[self.rank])}
        send_ids = [m for lst in incoming for m in lst]      # grouped by owner
        perm = torch.tensor([at[m] for m in send_ids], dtype=torch.int64, device=dev)
        send = rows.index_select(0, perm) if send_ids else torch.empty(0, width, device=dev)
        recv_ids = [m for lst in outgoing for m in lst]      # grouped by executing rank
        recv = torch.empty(len(recv_ids), width, dtype=rows.dtype, device=dev)
        dist.all_to_all_single(recv, send.contiguous(), [len(x) for x in outgoing],
                               [len(x) for x in incoming], group=self.group)
        if recv_ids:
            self.store.scatter(recv_ids, round_num, recv)
