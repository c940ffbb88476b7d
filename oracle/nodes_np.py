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
is the sequential-in-instance-order semantics.

Per timestep the node arrays are reset first (``reset=True``, the default):
a cable solver rebuilds its matrix every step, so rhs[k] = 0 - sum_i i_acc[i]
and d[k] = 0 + sum_i g_acc[i] over that step's instances only (nodes without
instances hold 0).  ``reset=False`` keeps the accumulate-across-steps form
(node_rhs/node_d initial values, then every step's contributions).  The scatter layout is a
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


def simulate_nodes(ir, data, steps, node_index, node_v, node_rhs=None, node_d=None, jac_mode="exact", reset=True,
                   terms=None):
    """`terms` (optional dict) receives "rhs"/"d": per node, the sum of |i_acc|
    / |g_acc| of every contribution the returned arrays hold (the scale for
    metrics.node_dev)."""
    n_nodes = len(node_v)
    si, sg = np.zeros(n_nodes), np.zeros(n_nodes)
    node_rhs = np.zeros(n_nodes) if (node_rhs is None or reset) else node_rhs.copy()
    node_d = np.zeros(n_nodes) if (node_d is None or reset) else node_d.copy()
    runner = OracleRunner(ir, jac_mode)
    data.arrays["v"][:] = node_v[node_index]
    runner.run_kernel(data, "initialize", 1)
    for _ in range(steps):
        data.arrays["v"][:] = node_v[node_index]
        runner.run_kernel(data, "state_update", 1)
        runner.run_kernel(data, "current_update", 1)
        if reset:
            node_rhs[:] = 0.0
            node_d[:] = 0.0
            si[:] = 0.0
            sg[:] = 0.0
        scatter(node_rhs, node_d, node_index, data.acc["i_acc"], data.acc["g_acc"])
        a, b = abs_terms(node_index, n_nodes, data.acc["i_acc"], data.acc["g_acc"], numeric_h(ir))
        si += a
        sg += b
    if terms is not None:
        terms["rhs"], terms["d"] = si, sg
    return data, node_rhs, node_d


def numeric_h(ir):
    """The conductance perturbation when `ir`'s g_acc is the two-point
    difference quotient (modlc/interp.py:495-514), else None."""
    return 0.001 if (ir.currents and not ir.analytic_conductance) else None


def abs_terms(node_index, n_nodes, i_acc, g_acc, h=None):
    """Per node: sum |i_acc| and sum |g_acc| of its instances (the scale of a
    one-step node sum, for the |delta| <= tol * sum|terms| bound).  For a
    difference-quotient g_acc (h given) a term's scale is max(|g|, |i|/h),
    the unit metrics.g_acc_dev holds each instance's g_acc to."""
    si = np.zeros(n_nodes)
    sg = np.zeros(n_nodes)
    np.add.at(si, node_index, np.abs(i_acc))
    g = np.abs(g_acc) if h is None else np.maximum(np.abs(g_acc), np.abs(i_acc) / h)
    np.add.at(sg, node_index, g)
    return si, sg
