"""Diagnostic (GPU box): what the column step's critical path is made of.

    NMODL_COLUMN_CELLS=12500 python tools/diag_column_path.py

Builds the bench column shard (grouped schedule, bench.options_for) and
times, each as one CUDA graph of 200 repetitions on the shard's stream, the
full step and partial launch sequences of it.  The partial sequences are
for timing only (they skip work the step needs, e.g. the combine then folds
stale soma currents); nothing here is a benchmark number.
"""

import ctypes as C
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
from paper_1905_02241_b200 import runtime as rt  # noqa: E402
from paper_1905_02241_b200.column import ColumnShard  # noqa: E402

REPS = 200


def main():
    rt.require_device(0)
    spec = bench._column_spec()
    shard = ColumnShard(spec, 0, spec.n_cells, bench.options_for, **bench._column_mode())
    s = shard.stream
    L = rt.lib()
    syn, ih = "ProbAMPANMDA_EMS", "Ih"

    def synapse(late=False):
        shard.runners[syn].launch(shard.devs[syn], "step_nodes", 1, late_wait=late)

    def ih_():
        shard.runners[ih].launch(shard.devs[ih], "step_nodes", 1)

    def soma_main():
        shard.group.launch(s, 1)

    def combine():
        shard._combine_soma(L, C)

    seqs = {
        "full step (shard.launch)": lambda: shard.launch(1),
        "synapse": lambda: synapse(),
        "Ih": ih_,
        "soma group": soma_main,
        "Ih + synapse": lambda: (ih_(), synapse()),
        "Ih + combine + synapse(late)": lambda: (ih_(), combine(), synapse(True)),
        "soma group + Ih + combine + synapse(late), one stream": lambda: (soma_main(), ih_(), combine(), synapse(True)),
    }
    shard.launch(10)
    s.sync()
    out = {"cells": spec.n_cells}
    a, b = rt.Event(), rt.Event()
    for name, fn in seqs.items():
        g = rt.capture(s, lambda: [fn() for _ in range(REPS)])
        g.upload(s)
        g.launch(s)  # warm
        s.sync()
        best = None
        for _ in range(3):
            a.record(s)
            g.launch(s)
            b.record(s)
            b.sync()
            t = a.elapsed_ms(b) / REPS * 1e3
            best = t if best is None else min(best, t)
        out[name] = round(best, 2)
        print(json.dumps({name: out[name]}), flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
