"""ORACLE (test infrastructure only) -- several mechanism populations stepped
over shared nodes with ion coupling (paper_1905_02241_b200/column.py).

Builder-defined semantics (parity unpinned by the reference, which has one
store per mechanism and no nodes): per timestep, for each population in
launch order: v <- node_v[node_index]; consumer ion slots <- the producer's
current values; state_update; current_update; node_rhs -= i_acc and
node_d += g_acc in instance order (np.subtract.at / np.add.at).
"""

from __future__ import annotations

import numpy as np

from .interp_np import OracleRunner
from .nodes_np import scatter


def simulate_column(irs, datas, node_index, node_v, order, couplings, steps):
    n_nodes = len(node_v)
    rhs, d = np.zeros(n_nodes), np.zeros(n_nodes)
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
        for m in order:
            datas[m].arrays["v"][:] = node_v[node_index[m]]
            couple(m)
            runners[m].run_kernel(datas[m], "state_update", 1)
            runners[m].run_kernel(datas[m], "current_update", 1)
            scatter(rhs, d, node_index[m], datas[m].acc["i_acc"], datas[m].acc["g_acc"])
    return datas, rhs, d
