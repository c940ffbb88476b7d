"""The product's NCCL process group (parallel.NcclGroup: ncclGetUniqueId /
ncclCommInitRank / ncclAllReduce / ncclAllGather bound through the runtime
library, no PyTorch) on the one GPU this run has: a one-rank communicator
exercises the same bootstrap, device copies and collectives a multi-GPU
launch uses (NCCL refuses two ranks on one device, so the two-process test
in test_gpu_column.py goes through the file group instead)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_nccl_group_one_rank(tmp_path):
    from paper_1905_02241_b200.parallel import NcclGroup, gather_checksums

    g = NcclGroup(0, 1, 0, tmp_path / "boot")
    try:
        assert g.allreduce([1.5, -2.0, 3.25], "sum") == [1.5, -2.0, 3.25]
        assert g.allreduce([7.0, 1.0], "max") == [7.0, 1.0]
        table = np.arange(12, dtype=np.float64).reshape(6, 2)
        out = gather_checksums(table, g)
        assert out.shape == (1, 6, 2)
        np.testing.assert_array_equal(out[0], table)
        g.barrier()
    finally:
        g.close()
    assert not (tmp_path / "boot" / "nccl.id").exists()  # rank 0 removes the bootstrap id


def test_device_checksums_gather_through_nccl(tmp_path):
    """A device store's fixed-tree checksums, all-gathered over NCCL, equal
    the local table bit for bit."""
    from conftest import load_ir
    from paper_1905_02241_b200.instance import init
    from paper_1905_02241_b200.parallel import NcclGroup, device_checksums, gather_checksums
    from paper_1905_02241_b200.runner import CudaRunner

    ir = load_ir("hh_subset")
    r = CudaRunner(ir)
    dev = r.to_device(init(ir, 100_000, 42))
    r.run_kernel(dev, "initialize", 1)
    r.run_kernel(dev, "step", 10)
    local = device_checksums(r, dev)
    g = NcclGroup(0, 1, 0, tmp_path / "boot")
    try:
        table = gather_checksums(local, g)
    finally:
        g.close()
    np.testing.assert_array_equal(table[0].view(np.int64), local.view(np.int64))
