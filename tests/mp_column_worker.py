"""Worker of tests/test_gpu_column.py::test_two_process_column_shards: one
rank of a multi-process column run.  RANK / WORLD_SIZE / LOCAL_RANK /
NMODL_BOOTSTRAP_DIR come from the environment (as under torchrun); the
process builds its CudaRunner shard of the cells, steps it, reduces its
device checksums and all-gathers them through the product's process group
(parallel.init_group: FileGroup when the ranks share one GPU)."""

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main(out_path: str, n_cells: int, steps: int) -> None:
    from paper_1905_02241_b200.column import ColumnShard, ColumnSpec
    from paper_1905_02241_b200.parallel import gather_checksums, init_group, partition_cells

    group, device = init_group()
    from paper_1905_02241_b200 import runtime as rt

    rt.require_device(device)
    spec = ColumnSpec(n_cells=n_cells, dend_per_cell=4, syn_per_cell=10, seed=3)
    bounds = partition_cells(np.full(spec.n_cells, spec.cell_cost()), group.world)
    shard = ColumnShard(spec, int(bounds[group.rank]), int(bounds[group.rank + 1]))
    shard.launch(steps)
    shard.check()
    table = gather_checksums(shard.checksums(), group)
    if group.rank == 0:
        np.save(out_path, table)
        np.save(out_path + ".bounds.npy", bounds)
    group.close()


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]))
