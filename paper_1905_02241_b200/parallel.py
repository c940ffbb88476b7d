"""Multi-GPU plumbing: cell sharding and validation checksums.

Mechanism instances are independent (modlc/codegen.py:59 "independent
iterations"; permutation invariance, modlc/interp.py:706-723) and the voltage
is exogenous per step, so the hot path shards with NO per-step
exchange.  One process per GPU owns a contiguous range of cells -- all
mechanism instances of a cell and its node_index targets live on one GPU --
balanced by the bytes each cell moves per timestep (the HBM-bound cost), not
by cell count.

The only collective is at the end of a run: every rank reduces its slots to
deterministic (sum, sum|x|) checksums on the device and the ranks all-gather
them (NCCL over NVLink on GPUs; gloo in the CPU tests), so a multi-GPU run can
be validated against a single-GPU or oracle run shard by shard.
"""

from __future__ import annotations

import ctypes as C

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


def gather_checksums(local: np.ndarray, group=None, device=None) -> np.ndarray:
    """All-gather per-rank checksum tables -> array[world, ...].

    Uses torch.distributed (NCCL when `device` is a CUDA device, gloo on CPU);
    with no initialised process group it returns the local table only."""
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        return local[None]
    world = dist.get_world_size(group)
    t = torch.as_tensor(np.ascontiguousarray(local), dtype=torch.float64)
    if device is not None:
        t = t.to(device)
    out = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(out, t, group=group)
    return np.stack([o.cpu().numpy() for o in out])
