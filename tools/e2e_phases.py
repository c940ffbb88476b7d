"""Where the column's public call (column.simulate_column) spends its time:
construction (upload, node layout, nrn_init), the timesteps, the checks and
the download, each bracketed by a stream sync (GPU box).

    python tools/e2e_phases.py [CELLS] [TIMESTEPS]
"""

import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import bench
    from paper_1905_02241_b200 import runtime as rt
    from paper_1905_02241_b200.column import LAUNCH_ORDER, ColumnShard, ColumnSpec, host_stores, shard_layout, simulate_column

    cells = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
    spec = ColumnSpec(n_cells=cells)
    host = host_stores(spec, 0, cells)
    lay = shard_layout(spec, 0, cells)  # inputs, generated before the clock (as bench.e2e_column)
    _, _, shard = simulate_column(spec, 10, 0, cells, host=host, options_for=bench.options_for, schedule="grouped",
                                  layout=lay)
    runners = shard.runners
    del shard
    host = host_stores(spec, 0, cells)
    pins = [rt.PinnedRegistration(a) for h in host.values() for a in list(h.arrays.values()) + list(h.acc.values())]
    for r in runners.values():
        r.trace = []
    out = {}
    t0 = time.perf_counter()
    shard = ColumnShard(spec, 0, cells, bench.options_for, host=host, runners=runners, schedule="grouped", layout=lay)
    shard.stream.sync()
    t1 = time.perf_counter()
    shard.launch(steps)
    shard.stream.sync()
    t2 = time.perf_counter()
    shard.check()
    t3 = time.perf_counter()
    for m in LAUNCH_ORDER:
        shard.runners[m].to_host(shard.devs[m], host[m], only_dirty=True)
    t4 = time.perf_counter()
    shard.nodes.download(shard.stream)
    t5 = time.perf_counter()
    out["ms"] = {"construct": 1e3 * (t1 - t0), "steps": 1e3 * (t2 - t1), "check": 1e3 * (t3 - t2),
                 "download": 1e3 * (t4 - t3), "nodes": 1e3 * (t5 - t4), "total": 1e3 * (t5 - t0)}
    stages = {}
    for m, r in runners.items():
        prev = None
        for stage, t in r.trace:
            if prev is not None:
                stages[f"{m}:{stage}"] = round(1e3 * (t - prev), 3)
            prev = t
    out["stages_ms"] = stages
    del pins
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
