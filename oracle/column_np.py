"""ORACLE (test infrastructure only) -- several mechanism populations stepped
over shared nodes with ion coupling (paper_1905_02241_b200/column.py).

Builder-defined semantics (parity unpinned by the reference, which has one
store per mechanism and no nodes): per timestep, for each population in
launch order: v <- node_v[node_index]; consumer ion slots <- the producer's
current values; state_update; current_update; node_rhs -= i_acc and
node_d += g_acc in instance order (np.subtract.at / np.add.at).  The node
rhs/d arrays are reset to zero at the start of every timestep (reset=True,
a cable solver's per-step matrix setup) or accumulate across steps.
"""

from __future__ import annotations

import numpy as np

from .interp_np import OracleRunner
from .nodes_np import abs_terms, numeric_h, scatter


def simulate_column(irs, datas, node_index, node_v, order, couplings, steps, reset=True, terms=None):
    """`terms` (optional dict) receives per-node sums of |contributions| held
    by the returned rhs/d (scale for metrics.node_dev)."""
    n_nodes = len(node_v)
    rhs, d = np.zeros(n_nodes), np.zeros(n_nodes)
    si, sg = np.zeros(n_nodes), np.zeros(n_nodes)
    runners = {m: OracleRunner(irs[m]) for m in order}

    def couple(m):
        for dst, dslot, src, sslot in couplings:
            if dst == m:
                datas[m].arrays[dslot][:] = datas[src].arrays[sslot]

    for m in order:
        datas[m].arrays["v"][:] = node_v[node_index[m]]
        couple(m)
        runners[m].run_kernel(datas[m], "initialize", 1)
    for _ in range(steps):
        if reset:
            rhs[:] = 0.0
            d[:] = 0.0
            si[:] = 0.0
            sg[:] = 0.0
        for m in order:
            datas[m].arrays["v"][:] = node_v[node_index[m]]
            couple(m)
            runners[m].run_kernel(datas[m], "state_update", 1)
            runners[m].run_kernel(datas[m], "current_update", 1)
            scatter(rhs, d, node_index[m], datas[m].acc["i_acc"], datas[m].acc["g_acc"])
            a, b = abs_terms(node_index[m], n_nodes, datas[m].acc["i_acc"], datas[m].acc["g_acc"], numeric_h(irs[m]))
            si += a
            sg += b
    if terms is not None:
        terms["rhs"], terms["d"] = si, sg
    return datas, rhs, d
