"""ORACLE (test infrastructure only) -- node_index gather/scatter restatement.

The reference has no node arrays: voltage is a per-instance exogenous array
and currents accumulate per instance (modlc/interp.py:80-81,
475-514).  The node_index extension required by the north star is therefore
BUILDER-DEFINED, following the CoreNEURON convention the reference's SIMD
backend gestures at with ATOMIC_ADD (modlc/codegen.py:77-78) and SPEC.md:603
models as ordered addition:

    v[i]              = node_v[node_index[i]]          (gather, before each step)
    node_rhs[k]      -= i_acc[i]   for i with node_index[i] == k, ascending i
    node_d[k]        += g_acc[i]   likewise

np.subtract.at / np.add.at apply the updates unbuffered in index order, which
is the sequential-in-instance-order semantics.  The scatter layout is a
stable sort by node: perm = argsort(node_index, kind="stable"),
offsets = exclusive prefix sum of per-node counts.  Parity unpinned by the
reference (no reference golden vectors exist for this path).
"""

from __future__ import annotations

import numpy as np

from .interp_np import OracleRunner


def scatter_layout(node_index: np.ndarray, n_nodes: int):
    perm = np.argsort(node_index, kind="stable")
    counts = np.bincount(node_index, minlength=n_nodes)
    offsets = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    rank = np.empty_like(perm)
    rank[perm] = np.arange(len(perm))
    return perm.astype(np.int64), offsets, rank.astype(np.int64)


def scatter(node_rhs, node_d, node_index, i_acc, g_acc):
    np.subtract.at(node_rhs, node_index, i_acc)
    np.add.at(node_d, node_index, g_acc)


def simulate_nodes(ir, data, steps, node_index, node_v, node_rhs=None, node_d=None, jac_mode="exact"):
    n_nodes = len(node_v)
    node_rhs = np.zeros(n_nodes) if node_rhs is None else node_rhs.copy()
    node_d = np.zeros(n_nodes) if node_d is None else node_d.copy()
    runner = OracleRunner(ir, jac_mode)
    data.arrays["v"][:] = node_v[node_index]
    runner.run_kernel(data, "initialize", 1)
    for _ in range(steps):
        data.arrays["v"][:] = node_v[node_index]
        runner.run_kernel(data, "state_update", 1)
        runner.run_kernel(data, "current_update", 1)
        scatter(node_rhs, node_d, node_index, data.acc["i_acc"], data.acc["g_acc"])
    return data, node_rhs, node_d
