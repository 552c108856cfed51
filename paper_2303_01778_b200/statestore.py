"""Client state manager: an HBM-resident per-client store with an optional
FSST on-disk tier.

Reference: ``fedsim/statestore.py`` (one fsynced file per client, loaded
before and saved after each task).  Here the primary copy of every client's
state is a row of a device matrix ``[slots, width]`` (fp32), moved to and
from a group's working rows by the gather/scatter kernels
(``pb_state_gather`` / ``pb_state_scatter``, csrc/state.cu) -- kernel (c) of
the north star.  The disk tier keeps the reference's byte format
(``client_%08d.state``: 28-byte little-endian header, magic ``FSST``,
version 1, client, round, payload length, CRC-32; tensor-map payload of
float64 data), so stores written by either implementation are readable by
the other.  Semantics kept: never-saved clients load the default (all-zero)
state at round -1, saves must strictly increase the round (StaleWriteError),
CRC/magic failures raise CorruptRecordError, peak checked-out states are
tracked.

persist="sync"  -- every save also writes + fsyncs the file (reference
                   durability; slow: one file per client per round);
persist="async" -- files are written by a background thread, ``flush()``
                   waits for them;
persist="none"  -- HBM only (the bench's mode); ``flush_to_disk()`` can still
                   spill everything on demand.

Capacity tiers (``hbm_bytes``): when M x width exceeds the HBM budget, the
first clients to save fill the HBM matrix and the rest live in a pinned
(device-mapped) host tier of fixed-size chunks; the same gather/scatter
kernels move both tiers, the host tier over the host link (one launch per
tier and chunk, no staging copy).  ``configure(..., capacity=M)`` sizes the
HBM matrix once, so a store never grows by reallocating and copying it.
"""


from __future__ import annotations

import os
import queue
import struct
import threading
import zlib
from dataclasses import dataclass
from pathlib import Path
from typing import Callable, Mapping, Sequence

import numpy as np
import torch

MAGIC = b"FSST"
VERSION = 1
_HEADER = struct.Struct("<4sHHIIQI")


class StaleWriteError(RuntimeError):
    """A save went backwards (or sideways) in rounds."""


class CorruptRecordError(RuntimeError):
    """Magic/version/checksum mismatch on a state file."""


@dataclass(frozen=True)
class ClientState:
    client_id: int
    round_written: int
    payload: dict


@dataclass(frozen=True)
class StateStoreStats:
    bytes_on_disk: int
    live_cache_entries: int
    loads: int
    saves: int
    peak_live_entries: int


def encode_tensor_map(payload: Mapping[str, object]) -> bytes:
    """u32 count; per entry u16 name len, name, u8 ndim, u64 dims, f64 data."""
    out = bytearray(struct.pack("<I", len(payload)))
    for name, t in payload.items():
        arr = _host_f64(t)
        raw = name.encode("utf-8")
        out += struct.pack("<H", len(raw)) + raw + struct.pack("<B", arr.ndim)
        out += struct.pack(f"<{arr.ndim}Q", *arr.shape) + arr.tobytes()
    return bytes(out)


def decode_tensor_map(blob: bytes, offset: int = 0) -> tuple[dict[str, np.ndarray], int]:
    (count,) = struct.unpack_from("<I", blob, offset)
    pos = offset + 4
    out: dict[str, np.ndarray] = {}
    for _ in range(count):
        (ln,) = struct.unpack_from("<H", blob, pos)
        name = blob[pos + 2: pos + 2 + ln].decode("utf-8")
        pos += 2 + ln
        ndim = blob[pos]
        pos += 1
        shape = struct.unpack_from(f"<{ndim}Q", blob, pos)
        pos += 8 * ndim
        size = int(np.prod(shape, dtype=np.int64)) if ndim else 1
        out[name] = np.frombuffer(blob, dtype="<f8", count=size, offset=pos).reshape(shape).copy()
        pos += 8 * size
    return out, pos


def tensor_map_data_bytes(payload: Mapping[str, object]) -> int:
    return sum(8 * int(np.asarray(_host_f64(t)).size) for t in payload.values())


def _host_f64(t) -> np.ndarray:
    if isinstance(t, torch.Tensor):
        return t.detach().cpu().double().numpy()
    return np.asarray(t, dtype="<f8")


class StateStore:
    """Per-client state, HBM-resident, optionally mirrored to FSST files."""

    def __init__(self, root: str | Path | None = None, persist: str | None = None,
                 device: torch.device | None = None, hbm_bytes: int | None = None,
                 host_chunk_bytes: int = 256 << 20):
        if persist is None:
            persist = "sync" if root is not None else "none"
        if persist not in ("sync", "async", "none"):
            raise ValueError(f"persist must be sync|async|none, got {persist!r}")
        if persist != "none" and root is None:
            raise ValueError("a persisting store needs a root directory")
        self.root = Path(root) if root is not None else None
        self.persist = persist
        self._device = device
        self._lock = threading.Lock()
        self._last_round: dict[int, int] = {}
        self._loads = 0
        self._saves = 0
        self._live: set[int] = set()
        self._peak_live = 0
        self._slot: dict[int, int] = {}            # HBM tier: client -> row of _rows
        self._rows: torch.Tensor | None = None
        self._hbm_budget = hbm_bytes               # None: no HBM limit
        self._capacity: int | None = None          # expected clients (configure)
        self._hslot: dict[int, tuple[int, int]] = {}   # host tier: client -> (chunk, row)
        self._hchunks: list[torch.Tensor] = []     # pinned [chunk_rows, width] views
        self._host_chunk_bytes = int(host_chunk_bytes)
        self._chunk_rows = 0
        self._schema: list[tuple[str, tuple[int, ...]]] | None = None
        self._width = 0
        self._queue: "queue.Queue | None" = None
        self._writer: threading.Thread | None = None
        self._writer_error: BaseException | None = None
        if self.root is not None:
            self.root.mkdir(parents=True, exist_ok=True)
            for path in self.root.glob("client_*.state"):
                cid, rnd, _, _ = self._read_header(path)
                self._last_round[cid] = rnd

    # -- helpers --------------------------------------------------------------
    def _dev(self) -> torch.device:
        if self._device is None:
            self._device = torch.device("cuda", torch.cuda.current_device())
        return self._device

    def _path(self, client_id: int) -> Path:
        return self.root / f"client_{client_id:08d}.state"

    @staticmethod
    def _read_header(path: Path) -> tuple[int, int, int, int]:
        with open(path, "rb") as fh:
            head = fh.read(_HEADER.size)
        if len(head) != _HEADER.size:
            raise CorruptRecordError(f"{path}: truncated header")
        magic, version, _, cid, rnd, length, crc = _HEADER.unpack(head)
        if magic != MAGIC or version != VERSION:
            raise CorruptRecordError(f"{path}: bad magic or version")
        return cid, rnd, length, crc

    def _read_file(self, client_id: int) -> tuple[int, dict[str, np.ndarray]]:
        path = self._path(client_id)
        cid, rnd, length, crc = self._read_header(path)
        if cid != client_id:
            raise CorruptRecordError(f"{path}: header claims client {cid}")
        with open(path, "rb") as fh:
            fh.seek(_HEADER.size)
            blob = fh.read(length)
        if len(blob) != length or zlib.crc32(blob) != crc:
            raise CorruptRecordError(f"{path}: payload checksum mismatch")
        return rnd, decode_tensor_map(blob)[0]

    def _has_file(self, client_id: int) -> bool:
        return self.root is not None and self._path(client_id).exists()

    def _set_schema(self, payload: Mapping[str, object]) -> None:
        schema = [(n, tuple(np.shape(t) if not isinstance(t, torch.Tensor) else t.shape))
                  for n, t in payload.items()]
        if self._schema is None:
            self._schema = schema
            self._width = int(sum(int(np.prod(s, dtype=np.int64)) if s else 1 for _, s in schema))
        elif [n for n, _ in schema] != [n for n, _ in self._schema]:
            raise ValueError("state payload schema changed between saves")

    @property
    def configured(self) -> bool:
        """True once the payload layout is known (configure() or a first save)."""
        return self._schema is not None

    def configure(self, names: Sequence[str], shapes: Sequence[tuple[int, ...]],
                  capacity: int | None = None) -> None:
        """Declare the payload layout up front (the engine does this, with
        capacity = the number of clients, so the HBM matrix is allocated once)."""
        self._set_schema({n: np.zeros(s, dtype=np.float32) for n, s in zip(names, shapes)})
        if capacity is not None:
            self._capacity = int(capacity)
            if self._rows is None:
                self._ensure_rows(min(self._capacity, self._hbm_cap()))

    def _pad(self) -> int:
        # row stride padded to 16 bytes: the gather/scatter kernels move rows
        # with 16-byte vectors
        return (self._width + 3) // 4 * 4

    def _hbm_cap(self) -> int:
        """Most rows the HBM tier may hold (the budget over the padded row)."""
        if self._hbm_budget is None:
            return 1 << 62
        return int(self._hbm_budget) // (4 * self._pad())

    def _ensure_rows(self, need: int) -> None:
        cap = 0 if self._rows is None else self._rows.shape[0]
        if need <= cap or need <= 0:
            return
        if self._capacity is not None:   # sized once for every client the HBM tier can hold
            new_cap = max(need, min(self._capacity, self._hbm_cap()))
        else:
            new_cap = min(max(need, 2 * cap, 64), self._hbm_cap())
        rows = torch.zeros(new_cap, self._pad(), device=self._dev())[:, :self._width]
        if self._rows is not None:
            rows[:cap].copy_(self._rows)
        self._rows = rows

    def _slot_for(self, client_id: int) -> int:
        """The client's HBM row, or -2 when it lives in the host tier (a home
        is assigned at the first save and never changes)."""
        s = self._slot.get(client_id)
        if s is not None:
            return s
        if client_id in self._hslot:
            return -2
        if len(self._slot) < self._hbm_cap():
            s = len(self._slot)
            self._slot[client_id] = s
            self._ensure_rows(s + 1)
            return s
        n = len(self._hslot)
        if self._chunk_rows == 0:
            self._chunk_rows = max(1, self._host_chunk_bytes // (4 * self._pad()))
        k, r = divmod(n, self._chunk_rows)
        if k == len(self._hchunks):
            self._hchunks.append(torch.zeros(self._chunk_rows, self._pad(),
                                             pin_memory=True)[:, :self._width])
        self._hslot[client_id] = (k, r)
        return -2

    def _row(self, client_id: int) -> torch.Tensor:
        """The client's stored row (an HBM or pinned-host view)."""
        s = self._slot_for(client_id)
        if s >= 0:
            return self._rows[s]
        k, r = self._hslot[client_id]
        return self._hchunks[k][r]

    def _has_row(self, client_id: int) -> bool:
        return client_id in self._slot or client_id in self._hslot

    def _flat(self, payload: Mapping[str, object]) -> torch.Tensor:
        parts = []
        for n, shape in self._schema:
            t = payload[n]
            t = t if isinstance(t, torch.Tensor) else torch.from_numpy(np.asarray(t, np.float32))
            parts.append(t.to(self._dev(), torch.float32).reshape(-1))
        return torch.cat(parts)

    def _unflat(self, row: torch.Tensor) -> dict[str, torch.Tensor]:
        out, pos = {}, 0
        for n, shape in self._schema:
            size = int(np.prod(shape, dtype=np.int64)) if shape else 1
            out[n] = row[pos:pos + size].view(shape)
            pos += size
        return out

    def _track_checkout(self, client_id: int) -> None:
        self._live.add(client_id)
        self._peak_live = max(self._peak_live, len(self._live))

    def _page_in(self, client_id: int) -> None:
        """Disk tier -> HBM row (CRC-checked); the file's round becomes the
        client's last-written round (a file another process wrote after this
        store was opened is picked up with its own round)."""
        rnd, payload = self._read_file(client_id)
        self._set_schema(payload)
        self._row(client_id).copy_(self._flat(payload))
        with self._lock:
            self._last_round[client_id] = rnd

    # -- reference API ----------------------------------------------------------
    def load(self, client_id: int,
             default_factory: Callable[[], Mapping[str, object]] | None = None) -> ClientState | None:
        if not self._has_row(client_id) and self._has_file(client_id):
            self._page_in(client_id)
        if not self._has_row(client_id):
            if default_factory is None:
                return None
            with self._lock:
                self._track_checkout(client_id)
            return ClientState(client_id, -1, dict(default_factory()))
        row = self._row(client_id).to(self._dev(), copy=True)
        with self._lock:
            self._loads += 1
            self._track_checkout(client_id)
        return ClientState(client_id, self._last_round[client_id], self._unflat(row))

    def save(self, client_id: int, round_num: int, payload: Mapping[str, object]) -> None:
        self._check_rounds([client_id], round_num)
        self._set_schema(payload)
        row = self._row(client_id)
        row.copy_(self._flat(payload))
        self._commit([client_id], round_num, rows=row.view(1, -1))

    def stats(self) -> StateStoreStats:
        self.flush()
        with self._lock:
            disk = sum(p.stat().st_size for p in self.root.glob("client_*.state")) \
                if self.root is not None else 0
            return StateStoreStats(bytes_on_disk=disk, live_cache_entries=len(self._live),
                                   loads=self._loads, saves=self._saves,
                                   peak_live_entries=self._peak_live)

    # -- device fast path -------------------------------------------------------
    def gather(self, client_ids: Sequence[int], work: torch.Tensor) -> None:
        """Load the listed clients' states into work rows [G, width] (zeros for
        never-saved clients) with one gather kernel."""
        from . import _kernels as K
        ids = [int(c) for c in client_ids]
        for c in ids:
            if not self._has_row(c) and self._has_file(c):
                self._page_in(c)
        # -1: never saved (default zeros), -2: the row lives in another tier
        slots = np.array([self._slot.get(c, -2 if c in self._hslot else -1) for c in ids], dtype=np.int32)
        with self._lock:
            self._loads += sum(1 for c in ids if self._has_row(c))
            for c in ids:
                self._track_checkout(c)
        if self._rows is not None:
            K.state_gather(work, self._rows, torch.from_numpy(slots).to(work.device))
        elif (slots == -1).any():
            work[torch.from_numpy(np.flatnonzero(slots == -1)).to(work.device)] = 0.0
        for k, chunk in enumerate(self._hchunks):   # host tier: read over the host link
            hs = np.array([self._hslot[c][1] if self._hslot.get(c, (-1, 0))[0] == k else -2 for c in ids],
                          dtype=np.int32)
            if (hs >= 0).any():
                K.state_gather(work, chunk, torch.from_numpy(hs).to(work.device))

    def scatter(self, client_ids: Sequence[int], round_num: int, work: torch.Tensor) -> None:
        """Persist the group's new states (rows of ``work``) for ``round_num``."""
        from . import _kernels as K
        ids = [int(c) for c in client_ids]
        if len(set(ids)) != len(ids):
            raise ValueError("a client appears twice in one scatter (disjoint-client contract)")
        self._check_rounds(ids, round_num)
        if self._schema is None:
            raise ValueError("state store schema unknown; call configure() first")
        slots = np.array([self._slot_for(c) for c in ids], dtype=np.int32)
        if self._rows is not None and (slots >= 0).any():
            K.state_scatter(self._rows, work, torch.from_numpy(slots).to(work.device))
        for k, chunk in enumerate(self._hchunks):   # host tier: written over the host link
            hs = np.array([self._hslot[c][1] if self._hslot.get(c, (-1, 0))[0] == k else -1 for c in ids],
                          dtype=np.int32)
            if (hs >= 0).any():
                K.state_scatter(chunk, work, torch.from_numpy(hs).to(work.device))
        self._commit(ids, round_num, rows=work)

    # -- commit / persistence -----------------------------------------------------
    def _check_rounds(self, ids: Sequence[int], round_num: int) -> None:
        with self._lock:
            for c in ids:
                prev = self._last_round.get(c, -1)
                if round_num <= prev:
                    raise StaleWriteError(
                        f"client {c}: save at round {round_num} after round {prev}")

    def _commit(self, ids: Sequence[int], round_num: int, rows: torch.Tensor) -> None:
        if self.persist != "none":
            host = rows.detach().to("cpu", torch.float64).numpy()
            jobs = [(c, round_num, host[j]) for j, c in enumerate(ids)]
            if self.persist == "sync":
                for job in jobs:
                    self._write_file(*job)
            else:
                self._start_writer()
                for job in jobs:
                    self._queue.put(job)
        with self._lock:
            for c in ids:
                self._last_round[c] = round_num
                self._live.discard(c)
            self._saves += len(ids)

    def _write_file(self, client_id: int, round_num: int, row: np.ndarray) -> None:
        payload, pos = {}, 0
        for n, shape in self._schema:
            size = int(np.prod(shape, dtype=np.int64)) if shape else 1
            payload[n] = row[pos:pos + size].reshape(shape)
            pos += size
        blob = encode_tensor_map(payload)
        head = _HEADER.pack(MAGIC, VERSION, 0, client_id, round_num, len(blob), zlib.crc32(blob))
        path = self._path(client_id)
        tmp = path.with_suffix(".tmp")
        fd = os.open(tmp, os.O_WRONLY | os.O_CREAT | os.O_TRUNC, 0o644)
        try:
            os.write(fd, head + blob)
            os.fsync(fd)
        finally:
            os.close(fd)
        os.replace(tmp, path)
        dfd = os.open(self.root, os.O_RDONLY)
        try:
            os.fsync(dfd)
        finally:
            os.close(dfd)

    def _start_writer(self) -> None:
        if self._writer is not None:
            return
        self._queue = queue.Queue()

        def run():
            while True:
                job = self._queue.get()
                try:
                    if job is None:
                        return
                    self._write_file(*job)
                except BaseException as exc:  # surfaced by flush()
                    self._writer_error = exc
                finally:
                    self._queue.task_done()

        self._writer = threading.Thread(target=run, name="fsst-writer", daemon=True)
        self._writer.start()

    def flush(self) -> None:
        """Wait for write-behind files (persist='async')."""
        if self._queue is not None:
            self._queue.join()
        if self._writer_error is not None:
            err, self._writer_error = self._writer_error, None
            raise err

    def flush_to_disk(self, root: str | Path | None = None) -> None:
        """Spill every HBM-resident state to FSST files (any persist mode)."""
        if root is not None:
            self.root = Path(root)
            self.root.mkdir(parents=True, exist_ok=True)
        if self.root is None:
            raise ValueError("no root directory to flush to")
        if self._rows is not None:
            host = self._rows.detach().to("cpu", torch.float64).numpy()
            for c, s in self._slot.items():
                self._write_file(c, self._last_round[c], host[s])
        torch.cuda.synchronize(self._dev())   # host-tier rows written by kernels
        for c, (k, r) in self._hslot.items():
            self._write_file(c, self._last_round[c], self._hchunks[k][r].double().numpy())

    def hbm_bytes(self) -> int:
        return 0 if self._rows is None else self._rows.shape[0] * self._pad() * 4

    def host_bytes(self) -> int:
        """Pinned host-tier bytes (clients beyond the HBM budget)."""
        return sum(c.shape[0] * self._pad() * 4 for c in self._hchunks)

    def tier_of(self, client_id: int) -> str | None:
        """'hbm', 'host' or None (never saved in this process)."""
        return "hbm" if client_id in self._slot else ("host" if client_id in self._hslot else None)

    def close(self) -> None:
        self.flush()
        if self._writer is not None:
            self._queue.put(None)
            self._writer.join()
            self._writer = None
