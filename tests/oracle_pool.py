"""Test helper: the numpy oracle on a large instance prefix, split across
host processes.

Instances never interact (modlc/interp.py:706-723) and `init_range` draws
exactly instances [lo, hi) of the seeded store, so the oracle run of
[0, k) is the concatenation of independent runs of its chunks.  That makes a
65,536-instance x 1000-step oracle run of the kinetic schemes (numpy LU at
~3e5 instance-steps/s) take seconds on the box's host
cores instead of minutes.  Test infrastructure only.
"""

from __future__ import annotations

import multiprocessing as mp
import os
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent


def _chunk(args):
    stems, lo, hi, steps, seed, couplings = args
    import sys

    if str(ROOT) not in sys.path:
        sys.path.insert(0, str(ROOT))
    from oracle import interp_np as O
    from paper_1905_02241_b200.instance import init_range
    from paper_1905_02241_b200.ir import MechIR

    irs = {m: MechIR.load(ROOT / "fixtures" / "ir" / f"{m}.json") for m in stems}
    datas = {}
    for m in stems:
        x = init_range(irs[m], lo, hi, seed)
        datas[m] = O.InstanceData(x.n, x.arrays, x.acc, x.scalars)
    runners = {m: O.OracleRunner(irs[m]) for m in stems}
    for m in stems:  # nrn_init per population, before any coupling (as bench.py sets up)
        runners[m].run_kernel(datas[m], "initialize", 1)
    for _ in range(steps):
        for m in stems:  # launch order
            for dst, dslot, src, sslot in couplings:
                if dst == m:  # the consumer reads the producer's value of this step
                    datas[m].arrays[dslot][:] = datas[src].arrays[sslot]
            runners[m].run_kernel(datas[m], "state_update", 1)
            runners[m].run_kernel(datas[m], "current_update", 1)
    return {m: (d.arrays, d.acc, d.newton_iters) for m, d in datas.items()}


def oracle_prefix(stems, k, steps, seed=42, couplings=(), chunk=4096, procs=None):
    """{stem: InstanceData} of the oracle on instances [0, k) of each
    population, stepped together in `stems` order with `couplings`
    ((dst, dst_slot, src, src_slot): dst's slot holds src's value)."""
    from oracle import interp_np as O

    bounds = list(range(0, k, chunk)) + [k]
    jobs = [(list(stems), lo, hi, steps, seed, list(couplings)) for lo, hi in zip(bounds[:-1], bounds[1:])]
    procs = procs or max(1, min(len(jobs), os.cpu_count() or 1))
    with mp.get_context("fork").Pool(procs) as pool:
        parts = pool.map(_chunk, jobs)
    out = {}
    for m in stems:
        arrays = {a: np.concatenate([p[m][0][a] for p in parts]) for a in parts[0][m][0]}
        acc = {a: np.concatenate([p[m][1][a] for p in parts]) for a in parts[0][m][1]}
        iters = [max(col) for col in zip(*[p[m][2] for p in parts])] if parts[0][m][2] else []
        out[m] = O.InstanceData(k, arrays, acc, {}, iters)
    return out
