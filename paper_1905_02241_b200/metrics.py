"""Parity metrics (used by the GPU tests and the CLI `verify`).

`rel_dev` is the reference's diff_trajectories metric (modlc/interp.py:658-672):
max |a-b| / max(|a|, |b|, 1e-30).  `rel_dev_floor` adds the per-slot scale
floor BASELINE.md §4 motivates for CONSERVE/LU schemes: the denominator is
at least floor * max|slot|, so 1e-14-magnitude occupancies do not turn ulp
noise of the exp() implementations into large relative errors.
"""

import numpy as np

TOL = 1e-10  # north star: 1e-10 relative in fp64 after 1000 timesteps


def _pair(a, b, name):
    xa = a.acc[name] if name in a.acc else a.arrays[name]
    xb = b.acc[name] if name in b.acc else b.arrays[name]
    return np.asarray(xa), np.asarray(xb)


def rel_dev(a, b, names):
    worst, where = 0.0, None
    for name in names:
        xa, xb = _pair(a, b, name)
        d = np.abs(xa - xb) / np.maximum(np.maximum(np.abs(xa), np.abs(xb)), 1e-30)
        m = float(np.max(d)) if d.size else 0.0
        if m > worst:
            worst, where = m, name
    return worst, where


def rel_dev_floor(a, b, names, floor=1e-6):
    worst, where = 0.0, None
    for name in names:
        xa, xb = _pair(a, b, name)
        scale = max(float(np.max(np.abs(xa))) if xa.size else 0.0, float(np.max(np.abs(xb))) if xb.size else 0.0)
        den = np.maximum(np.maximum(np.maximum(np.abs(xa), np.abs(xb)), floor * scale), 1e-30)
        m = float(np.max(np.abs(xa - xb) / den)) if xa.size else 0.0
        if m > worst:
            worst, where = m, name
    return worst, where


def compared_names(ir):
    """States, ion variables, every other slot, and the accumulators."""
    from .ir import from_layout

    return list(from_layout(ir).slot_names()) + ["v", "i_acc", "g_acc"]


H = 0.001  # CONDUCTANCE_PERTURBATION, modlc/odes.py:45


def g_acc_dev(ir, a, b):
    """Numeric-conductance g_acc is a difference quotient (i(v+h) - i(v))/h
    (modlc/interp.py:495-514): its rounding error scales with |i|/h, not |g|.
    The reference's own two CPU paths (numpy oracle vs emitted C) disagree by
    8.6e-10 pure-relative on it (ProbAMPANMDA_EMS, 1000 steps).  We therefore
    hold it to the north-star 1e-10 relative to the currents it is built from:
    |dg| <= 1e-10 * max(|g|, |i_acc|/h)."""
    ga, gb = np.asarray(a.acc["g_acc"]), np.asarray(b.acc["g_acc"])
    ia = np.abs(np.asarray(a.acc["i_acc"]))
    den = np.maximum(np.maximum(np.maximum(np.abs(ga), np.abs(gb)), ia / H), 1e-30)
    return float(np.max(np.abs(ga - gb) / den)) if ga.size else 0.0


def solve_groups(ir):
    """State groups solved together by one LinearSolveNode / NewtonSolveNode
    (or the k<=3 symbolic sparse solve, recognised by its `*_new` unknowns)."""
    from .ir import iter_nodes

    groups = []
    for stmts in ir.kernels.values():
        for s in stmts:
            for node in iter_nodes(s):
                if node.kind in ("LinearSolveNode", "NewtonSolveNode") and len(node.attrs["states"]) > 1:
                    groups.append([x for x in node.attrs["states"] if x in ir.slot_names()])
        news = [s.children[0].attrs["name"] for s in stmts
                if s.kind == "Assign" and s.children[1].kind == "Identifier"
                and s.children[1].attrs["name"].endswith("_new") and s.children[0].kind == "Identifier"]
        if len(news) > 1:
            groups.append([x for x in news if x in ir.slot_names()])
    out = []
    for g in groups:
        if len(g) > 1 and g not in out:
            out.append(g)
    return out


def group_dev(a, b, group):
    """Normwise-per-instance relative error over a jointly solved state
    vector: |dx_j| / max_k |x_k| (the backward-stability bound an LU/Newton
    solve actually guarantees; tiny occupancies inherit the absolute error of
    the whole vector -- the reference's own C and numpy paths differ by
    1.9e-10 pure-relative on na6 for exactly this reason)."""
    xa = np.stack([np.asarray(a.arrays[s]) for s in group])
    xb = np.stack([np.asarray(b.arrays[s]) for s in group])
    den = np.maximum(np.maximum(np.abs(xa).max(axis=0), np.abs(xb).max(axis=0)), 1e-30)
    return float(np.max(np.abs(xa - xb) / den[None, :])) if xa.size else 0.0


def parity(ir, a, b, floored=False):
    from .ir import from_layout

    ir = from_layout(ir)
    """(worst deviation, slot) using the metric appropriate to each slot:
    pure relative (diff_trajectories) everywhere, except numeric-conductance
    g_acc (g_acc_dev) and jointly solved state vectors (group_dev)."""
    names = compared_names(ir)
    numeric_g = bool(ir.currents) and not ir.analytic_conductance
    grouped = {s for g in solve_groups(ir) for s in g}
    plain = [x for x in names if not (numeric_g and x == "g_acc") and x not in grouped]
    worst, where = (rel_dev_floor(a, b, plain) if floored else rel_dev(a, b, plain))
    if numeric_g:
        g = g_acc_dev(ir, a, b)
        if g > worst:
            worst, where = g, "g_acc"
    for grp in solve_groups(ir):
        g = group_dev(a, b, grp)
        if g > worst:
            worst, where = g, "+".join(grp)
    return worst, where


def node_dev(got, want, scale) -> float:
    """Node rhs/d deviation: max |got - want| / max(|got|, |want|, scale) with
    `scale` = the per-node sum of |terms| folded into it (oracle/nodes_np.
    abs_terms).  A node sum of same-sign terms is held to the pure relative
    bar; one whose terms cancel is held to it relative to the terms' size,
    the bound a sum of individually-rounded terms can honour."""
    got, want, scale = (np.asarray(x, dtype=np.float64) for x in (got, want, scale))
    den = np.maximum(np.maximum(np.abs(got), np.abs(want)), np.maximum(scale, 1e-30))
    return float(np.max(np.abs(got - want) / den)) if got.size else 0.0
