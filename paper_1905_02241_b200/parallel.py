"""Multi-GPU plumbing: cell sharding, process groups and validation checksums.

Mechanism instances are independent (modlc/codegen.py:59 "independent
iterations"; permutation invariance, modlc/interp.py:706-723) and the voltage
is exogenous per step, so the hot path shards with NO per-step
exchange.  One process per GPU owns a contiguous range of cells -- all
mechanism instances of a cell and its node_index targets live on one GPU --
balanced by the bytes each cell moves per timestep (the HBM-bound cost), not
by cell count (the paper runs one rank per core the same way).

The only collectives are at the end of a run (and the bench's barrier /
max-time reduction): every rank reduces its slots to deterministic (sum,
sum|x|) checksums on the device and the ranks all-gather them, so a
multi-GPU run can be validated against a single-GPU or oracle run shard by
shard.  No PyTorch: `NcclGroup` calls NCCL through the runtime library
(libnmodl_b200_rt: nmodl_nccl_*), one rank per GPU; `FileGroup` is the
same interface over files in a directory, for ranks that share one GPU
(NCCL refuses two ranks on one device) and for the CPU tests.
"""

from __future__ import annotations

import ctypes as C
import os
import time
from pathlib import Path

import numpy as np


def partition_cells(cell_cost: np.ndarray, world: int) -> np.ndarray:
    """Contiguous cell ranges with balanced total cost.

    Returns bounds[world+1]: rank r owns cells [bounds[r], bounds[r+1]).
    Greedy split of the cost prefix sum at multiples of total/world; every
    rank gets at least one cell when there are enough cells.
    """
    cost = np.asarray(cell_cost, dtype=np.float64)
    n = len(cost)
    if world < 1:
        raise ValueError("world must be >= 1")
    if n == 0:
        return np.zeros(world + 1, dtype=np.int64)
    prefix = np.concatenate([[0.0], np.cumsum(cost)])
    targets = prefix[-1] * np.arange(1, world) / world
    cuts = np.searchsorted(prefix, targets, side="left")
    bounds = np.concatenate([[0], cuts, [n]]).astype(np.int64)
    # keep ranges non-empty and monotone when possible
    for r in range(1, world):
        lo = bounds[r - 1] + (1 if n >= world else 0)
        bounds[r] = min(max(bounds[r], lo), n - (world - r if n >= world else 0))
    return bounds


def shard_instances(instances_per_cell: np.ndarray, bounds: np.ndarray, rank: int) -> tuple[int, int]:
    """[lo, hi) instance range of `rank` given per-cell instance counts."""
    offs = np.concatenate([[0], np.cumsum(np.asarray(instances_per_cell, dtype=np.int64))])
    return int(offs[bounds[rank]]), int(offs[bounds[rank + 1]])


# ---------------------------------------------------------------------------
# process groups


class LocalGroup:
    """world = 1: every collective is the identity."""

    rank, world, backend = 0, 1, "local"

    def barrier(self) -> None:
        pass

    def allreduce(self, values, op: str = "sum") -> list:
        return [float(v) for v in values]

    def allgather(self, local: np.ndarray) -> np.ndarray:
        return np.asarray(local)[None]

    def close(self) -> None:
        pass


class FileGroup:
    """Collectives through files in a directory shared by the ranks of one
    node: rank r writes `<seq>.<r>.npy` atomically (write + rename), then
    waits for the others.  Deterministic (every rank reduces the gathered
    table in rank order).  Used when ranks share a GPU and in CPU tests."""

    backend = "file"

    def __init__(self, directory, rank: int, world: int, timeout_s: float = 600.0):
        self.dir = Path(directory)
        self.dir.mkdir(parents=True, exist_ok=True)
        self.rank, self.world = int(rank), int(world)
        self.timeout = timeout_s
        self.seq = 0

    def _path(self, seq: int, rank: int) -> Path:
        return self.dir / f"{seq}.{rank}.npy"

    def allgather(self, local: np.ndarray) -> np.ndarray:
        local = np.ascontiguousarray(local)
        seq = self.seq
        self.seq += 1
        tmp = self.dir / f".{seq}.{self.rank}.{os.getpid()}.tmp"
        with open(tmp, "wb") as fh:
            np.save(fh, local)
        os.replace(tmp, self._path(seq, self.rank))
        out = []
        deadline = time.monotonic() + self.timeout
        for r in range(self.world):
            p = self._path(seq, r)
            while not p.is_file():
                if time.monotonic() > deadline:
                    raise TimeoutError(f"FileGroup: rank {r} never wrote {p}")
                time.sleep(0.002)
            for _ in range(1000):  # a complete file was renamed in; read it
                try:
                    out.append(np.load(p))
                    break
                except (EOFError, ValueError, OSError):
                    time.sleep(0.002)
        # the previous round's files are no longer needed by anyone who reached this one
        if seq >= 1:
            self._path(seq - 1, self.rank).unlink(missing_ok=True)
        return np.stack(out)

    def allreduce(self, values, op: str = "sum") -> list:
        table = self.allgather(np.asarray(values, dtype=np.float64))
        red = table.max(axis=0) if op == "max" else table.sum(axis=0)
        return [float(x) for x in red]

    def barrier(self) -> None:
        self.allgather(np.zeros(1))

    def close(self) -> None:
        # after this barrier every rank has read every earlier round; the
        # barrier's own (tiny) files stay -- a slow rank may still read them
        self.barrier()


class NcclGroup:
    """One rank per GPU over NCCL (NVLink/NVSwitch within the node), bound
    through the runtime library.  The unique id is bootstrapped through a
    file in `bootstrap_dir` (single node: the ranks share /tmp)."""

    backend = "nccl"

    def __init__(self, rank: int, world: int, device: int, bootstrap_dir, timeout_s: float = 600.0):
        from . import runtime as rt

        self.rank, self.world, self.device = int(rank), int(world), int(device)
        rt.set_device(self.device)
        self.rt = rt
        self.L = rt.lib()
        d = Path(bootstrap_dir)
        d.mkdir(parents=True, exist_ok=True)
        idf = d / "nccl.id"
        uid = (C.c_ubyte * 128)()
        if self.rank == 0:
            rt.check(self.L.nmodl_nccl_unique_id(uid), "ncclGetUniqueId")
            tmp = d / f".nccl.id.{os.getpid()}"
            tmp.write_bytes(bytes(uid))
            os.replace(tmp, idf)
        else:
            deadline = time.monotonic() + timeout_s
            while not (idf.is_file() and idf.stat().st_size == 128):
                if time.monotonic() > deadline:
                    raise TimeoutError(f"NcclGroup: no unique id at {idf}")
                time.sleep(0.01)
            C.memmove(uid, idf.read_bytes(), 128)
        comm = C.c_void_p()
        rt.check(self.L.nmodl_nccl_init(C.byref(comm), self.world, uid, self.rank), "ncclCommInitRank")
        self.comm = comm
        self.stream = rt.Stream()
        self.barrier()
        if self.rank == 0:
            idf.unlink(missing_ok=True)

    def _device_copy(self, arr: np.ndarray):
        buf = self.rt.DeviceBuffer(max(arr.nbytes, 8))
        self.rt.h2d(buf.ptr, arr.ctypes.data, arr.nbytes, self.stream)
        return buf

    def allreduce(self, values, op: str = "sum") -> list:
        a = np.ascontiguousarray(values, dtype=np.float64)
        src = self._device_copy(a)
        dst = self.rt.DeviceBuffer(max(a.nbytes, 8))
        self.rt.check(self.L.nmodl_nccl_allreduce_f64(self.comm, C.c_void_p(src.ptr), C.c_void_p(dst.ptr), a.size,
                                                      1 if op == "max" else 0, C.c_void_p(self.stream.handle)),
                      "ncclAllReduce")
        out = np.empty_like(a)
        self.rt.d2h(out.ctypes.data, dst.ptr, a.nbytes, self.stream)
        self.stream.sync()
        return [float(x) for x in out]

    def allgather(self, local: np.ndarray) -> np.ndarray:
        a = np.ascontiguousarray(local, dtype=np.float64)
        src = self._device_copy(a)
        dst = self.rt.DeviceBuffer(max(a.nbytes * self.world, 8))
        self.rt.check(self.L.nmodl_nccl_allgather_f64(self.comm, C.c_void_p(src.ptr), C.c_void_p(dst.ptr), a.size,
                                                      C.c_void_p(self.stream.handle)), "ncclAllGather")
        out = np.empty((self.world,) + a.shape)
        self.rt.d2h(out.ctypes.data, dst.ptr, out.nbytes, self.stream)
        self.stream.sync()
        return out

    def barrier(self) -> None:
        self.allreduce([0.0])

    def close(self) -> None:
        if self.comm:
            self.rt.check(self.L.nmodl_nccl_destroy(self.comm), "ncclCommDestroy")
            self.comm = None


def bootstrap_dir() -> Path:
    """Rendezvous directory shared by the ranks of one launch on one node:
    NMODL_BOOTSTRAP_DIR, else keyed by the launcher (torchrun's agent is
    every worker's parent) and its master port."""
    explicit = os.environ.get("NMODL_BOOTSTRAP_DIR")
    if explicit:
        return Path(explicit)
    key = f"{os.getppid()}_{os.environ.get('MASTER_PORT', '0')}_{os.environ.get('TORCHELASTIC_RUN_ID', 'x')}"
    return Path("/tmp") / f"nmodl_b200_{key}"


def init_group(device_count: int | None = None):
    """The process group of this launch, from the launcher's environment
    (RANK / WORLD_SIZE / LOCAL_RANK): LocalGroup for one rank; NcclGroup
    when every rank has its own GPU; FileGroup when ranks share GPUs (a
    multi-rank run on a one-GPU box).  Returns (group, device)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world <= 1:
        return LocalGroup(), 0
    if device_count is None:
        from . import runtime as rt

        device_count = rt.device_count()
    ndev = max(device_count, 1)
    device = local % ndev
    if ndev >= world and os.environ.get("NMODL_GROUP", "nccl") == "nccl":
        try:
            return NcclGroup(rank, world, device, bootstrap_dir()), device
        except Exception as exc:  # noqa: BLE001 -- validation collectives only: keep going
            import sys

            print(f"[parallel] rank {rank}: NCCL group unavailable ({exc}); using the file group", file=sys.stderr)
            return FileGroup(bootstrap_dir() / "file_fallback", rank, world), device
    return FileGroup(bootstrap_dir() / "file", rank, world), device


# ---------------------------------------------------------------------------
# checksums


def device_checksums(runner, dev, names=None) -> np.ndarray:
    """(sum, sum|x|) per array of a device store, computed on the device with a
    fixed reduction tree (nmodl_checksum) -- identical bits run to run."""
    from . import runtime as rt

    names = names or list(dev.names) + ["i_acc", "g_acc"]
    scratch = rt.DeviceBuffer(8 * 2 * 1024)
    out = rt.DeviceBuffer(16 * len(names))
    L = rt.lib()
    for i, name in enumerate(names):
        rt.check(L.nmodl_checksum(C.c_void_p(dev.ptr[name]), dev.n, C.c_void_p(scratch.ptr),
                                  C.c_void_p(out.ptr + 16 * i), C.c_void_p(runner.stream.handle)), "checksum")
    host = np.empty(2 * len(names))
    rt.d2h(host.ctypes.data, out.ptr, host.nbytes, runner.stream)
    runner.stream.sync()
    return host.reshape(len(names), 2)


def host_checksums(arrays: dict, names) -> np.ndarray:
    """Same quantity on host arrays (for CPU-side comparison; tree differs)."""
    return np.array([[float(np.sum(arrays[n])), float(np.sum(np.abs(arrays[n])))] for n in names])


def gather_checksums(local: np.ndarray, group=None) -> np.ndarray:
    """All-gather per-rank checksum tables -> array[world, ...] (the local
    table alone without a group)."""
    if group is None:
        return np.asarray(local)[None]
    return group.allgather(local)
