"""Multi-process (world_size 2, CPU) coverage of the sharding path.

The GPU hot path has no per-step collective; what crosses ranks is (1) the
cell partition every rank computes identically and (2) the end-of-run
checksum all-gather.  Both are exercised here with two real processes
through the product's torch-free FileGroup (parallel.py), and the same
all-gather is cross-checked against torch.distributed's gloo backend (test
only: the product never imports torch).
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1905_02241_b200.parallel import (FileGroup, gather_checksums, host_checksums, init_group,
                                            partition_cells, shard_instances)


def test_partition_balances_cost_and_covers_all_cells():
    rng = np.random.default_rng(0)
    cost = rng.integers(1, 100, 10_000).astype(float)
    for world in (1, 2, 4, 8):
        b = partition_cells(cost, world)
        assert b[0] == 0 and b[-1] == len(cost)
        assert np.all(np.diff(b) > 0)
        loads = np.array([cost[b[r]:b[r + 1]].sum() for r in range(world)])
        assert loads.max() <= cost.sum() / world + cost.max()


def test_partition_degenerate():
    assert partition_cells(np.ones(3), 8)[-1] == 3
    assert partition_cells(np.array([]), 2).tolist() == [0, 0, 0]


def test_shard_instances_contiguous():
    per_cell = np.array([3, 0, 5, 2, 7])
    b = partition_cells(per_cell.astype(float) + 1, 2)
    lo0, hi0 = shard_instances(per_cell, b, 0)
    lo1, hi1 = shard_instances(per_cell, b, 1)
    assert lo0 == 0 and hi0 == lo1 and hi1 == per_cell.sum()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q, boot):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    group = FileGroup(boot, rank, world)
    try:
        from conftest import load_ir
        from oracle import interp_np as O

        # every rank derives the same partition, then simulates only its shard
        n_cells, per_cell = 40, np.full(40, 25)
        bounds = partition_cells(per_cell.astype(float), world)
        lo, hi = shard_instances(per_cell, bounds, rank)
        ir = load_ir("hh_subset")
        full = O.init(ir, int(per_cell.sum()), 42)
        shard = O.InstanceData(hi - lo, {k: v[lo:hi].copy() for k, v in full.arrays.items()},
                               {k: v[lo:hi].copy() for k, v in full.acc.items()}, dict(full.scalars))
        O.simulate(ir, shard, 5)
        names = list(ir.slot_names())
        local = host_checksums(shard.arrays, names)
        table = gather_checksums(local, group)
        # cross-check: gloo's all_gather delivers the same table
        import torch

        parts = [torch.empty(local.shape, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, torch.as_tensor(local))
        assert np.array_equal(np.stack([p.numpy() for p in parts]), table)
        assert group.allreduce([float(rank + 1)], "max") == [float(world)]
        assert group.allreduce([1.0, 2.0], "sum") == [float(world), 2.0 * world]
        q.put((rank, table.tolist(), (lo, hi)))
    finally:
        group.close()
        dist.destroy_process_group()


def test_two_rank_shards_reassemble_to_single_run(tmp_path):
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parent))
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, str(tmp_path / "grp"))) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    results.sort()
    t0, t1 = np.array(results[0][1]), np.array(results[1][1])
    np.testing.assert_array_equal(t0, t1)  # all-gather delivered identical tables
    # instance independence: shard checksums sum to the single-process run's
    from conftest import load_ir
    from oracle import interp_np as O

    ir = load_ir("hh_subset")
    full = O.simulate(ir, O.init(ir, 1000, 42), 5)
    for name_i, name in enumerate(ir.slot_names()):
        lo0, hi0 = results[0][2]
        lo1, hi1 = results[1][2]
        a = full.arrays[name]
        assert np.isclose(t0[0][name_i][0] + t0[1][name_i][0], a[lo0:hi0].sum() + a[lo1:hi1].sum(), rtol=1e-12)
        assert hi0 == lo1


def test_init_group_single_rank_and_file_fallback(monkeypatch, tmp_path):
    """WORLD_SIZE=1 -> LocalGroup; more ranks than GPUs -> FileGroup (ranks
    sharing a device; NCCL needs one GPU per rank)."""
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    g, dev = init_group(device_count=0)
    assert g.world == 1 and g.backend == "local" and dev == 0
    assert gather_checksums(np.ones((2, 2)), g).shape == (1, 2, 2)
    monkeypatch.setenv("WORLD_SIZE", "1")
    monkeypatch.setenv("NMODL_BOOTSTRAP_DIR", str(tmp_path))
    g, _ = init_group(device_count=1)
    assert g.backend == "local"
    monkeypatch.setenv("WORLD_SIZE", "2")
    monkeypatch.setenv("RANK", "1")
    monkeypatch.setenv("LOCAL_RANK", "1")
    g, dev = init_group(device_count=1)
    assert g.backend == "file" and g.rank == 1 and dev == 0


def test_product_modules_do_not_import_torch():
    """The package and bench.py's product arm run without PyTorch."""
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    code = ("import sys; sys.path.insert(0, %r); import paper_1905_02241_b200, paper_1905_02241_b200.parallel, "
            "paper_1905_02241_b200.runner, paper_1905_02241_b200.column, bench; "
            "assert 'torch' not in sys.modules, 'torch imported'" % str(root))
    subprocess.run([sys.executable, "-c", code], check=True, timeout=300)
