"""Multi-GPU plumbing for the round: which simulated devices a rank executes,
and the one collective of a round -- the all-reduce of the packed per-device
partial sums (kernel (d) of the north star).

One process per GPU (``torch.distributed``, NCCL over NVLink 5 / NVSwitch).
Every rank computes the same selection, fits and plan (host-side, bit-exact),
executes the devices ``k`` with ``k % world == rank``, folds them locally in
device order, and then ONE all-reduce of a flat fp32 buffer
[acc of every averaged entry] plus one of a float64 buffer [weight sums,
counts] combines the ranks; Collect entries (per-client scalars) travel by
``all_gather_object``.  Every rank then applies the same server rule, so the
global model stays replicated without a broadcast.  NCCL's reduction order
differs from the reference's device-order sum, so cross-world parity is
tolerance-based.

The functions take the device and the fold as parameters so the packing logic
is exercised by world-size-2 ``gloo`` tests on CPU (tests/test_distributed_cpu.py).
"""

from __future__ import annotations

from typing import Callable, Sequence

import numpy as np
import torch


def local_devices(num_devices: int, world: int, rank: int) -> list[int]:
    """Simulated devices executed by ``rank`` (round-robin over ranks)."""
    return [k for k in range(num_devices) if k % world == rank]


def allreduce_partials(partials: Sequence, schema, *, device, fold: Callable,
                       group=None):
    """Combine this rank's device partials with every other rank's.

    ``schema`` is [(name, AggOp, shape)] (every client result carries these);
    ``fold(acc, x)`` accumulates ``x`` into ``acc`` (the fold kernel on the GPU,
    ``Tensor.add_`` in CPU tests).  Returns one DevicePartial holding the
    global sums, weight sums, counts, Collect items and folded client ids."""
    import torch.distributed as dist

    from .aggregate import DevicePartial, PartialEntry
    from .trainer import AggOp

    live = [p for p in partials if p.entries]
    accs, meta = [], []
    for name, op, shape in schema:
        if op is AggOp.COLLECT:
            continue
        acc = torch.zeros(int(np.prod(shape)), dtype=torch.float32, device=device)
        wsum, cnt = 0.0, 0
        for p in live:  # this rank's devices, in device order
            pe = p.entries.get(name)
            if pe is not None:
                fold(acc, pe.acc.reshape(-1))
                wsum += pe.weight_sum
                cnt += pe.count
        accs.append(acc)
        meta += [wsum, float(cnt)]
    packed = torch.cat(accs) if accs else torch.zeros(0, device=device)
    meta_t = torch.tensor(meta, dtype=torch.float64, device=device)
    dist.all_reduce(packed, group=group)
    dist.all_reduce(meta_t, group=group)
    meta_h = meta_t.cpu().numpy()
    out = DevicePartial(device_id=dist.get_rank(group))
    pos = mi = 0
    for name, op, shape in schema:
        if op is AggOp.COLLECT:
            continue
        size = int(np.prod(shape))
        out.entries[name] = PartialEntry(op=op, acc=packed[pos:pos + size].view(shape),
                                         weight_sum=float(meta_h[mi]),
                                         count=int(round(meta_h[mi + 1])))
        pos += size
        mi += 2
    mine = {name: [(c, t.detach().cpu()) for p in live if name in p.entries
                   for c, t in p.entries[name].collected]
            for name, op, _ in schema if op is AggOp.COLLECT}
    gathered = [None] * dist.get_world_size(group)
    dist.all_gather_object(gathered, (mine, [c for p in live for c in p.clients_folded]),
                           group=group)
    for name, op, _ in schema:
        if op is not AggOp.COLLECT:
            continue
        items = [(c, t.to(device)) for g in gathered for c, t in g[0].get(name, [])]
        out.entries[name] = PartialEntry(op=op, collected=items, count=len(items))
    out.clients_folded = [c for g in gathered for c in g[1]]
    return out
