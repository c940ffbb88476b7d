"""Synthetic instance stores in the reference's data format.

`init` produces exactly what modlc/interp.py:61-84 `init(layout, n, seed, dt)`
produces -- one named, seeded substream per slot (`_slot_rng`,
interp.py:55-58), parameters at their defaults, ion currents zero,
concentrations/reversals/states/other assigned uniform in the documented
ranges (interp.py:26-30), v uniform in [-80, 40] -- so benchmark inputs are
the same synthetic populations the reference's own tests and CLI use, and a
prefix of a large store equals a small store (prefix stability).

`node_layout` draws the node_index extension inputs (SURVEY §8(d) workload
2): a random compartment per instance and a voltage per compartment.
"""

from __future__ import annotations

import zlib

import numpy as np

from .ir import from_layout
from .runner import HostInstanceData

V_RANGE = (-80.0, 40.0)
STATE_RANGE = (0.0, 1.0)
CONC_RANGE = (1e-9, 1e-3)
REVERSAL_RANGE = (-100.0, 100.0)
ASSIGNED_RANGE = (0.0, 1.0)


def _slot_rng(seed: int, name: str) -> np.random.Generator:
    return np.random.default_rng([seed, zlib.crc32(name.encode())])


def init(layout, n: int, seed: int, dt: float = 0.025) -> HostInstanceData:
    ir = from_layout(layout)
    if n < 1:
        raise ValueError("need at least one instance")
    arrays = {}
    for slot in ir.slots:
        rng = _slot_rng(seed, slot.name)
        if slot.role == "parameter":
            arrays[slot.name] = np.full(n, slot.default if slot.default is not None else 0.0)
        elif slot.ion_kind == "current":
            arrays[slot.name] = np.zeros(n)
        elif slot.ion_kind == "conc":
            arrays[slot.name] = rng.uniform(*CONC_RANGE, n)
        elif slot.ion_kind == "reversal":
            arrays[slot.name] = rng.uniform(*REVERSAL_RANGE, n)
        elif slot.role == "state":
            arrays[slot.name] = rng.uniform(*STATE_RANGE, n)
        else:
            arrays[slot.name] = rng.uniform(*ASSIGNED_RANGE, n)
    arrays["v"] = _slot_rng(seed, "v").uniform(*V_RANGE, n)
    scalars = dict(ir.global_scalars)
    scalars["dt"] = dt
    return HostInstanceData(n, arrays, {"i_acc": np.zeros(n), "g_acc": np.zeros(n)}, scalars)


def _range_rng(seed: int, name: str, lo: int) -> np.random.Generator:
    """The `_slot_rng` stream advanced to draw `lo` (one 64-bit draw per double)."""
    bg = np.random.PCG64(np.random.SeedSequence([seed, zlib.crc32(name.encode())]))
    bg.advance(lo)
    return np.random.Generator(bg)


def init_range(layout, lo: int, hi: int, seed: int, dt: float = 0.025) -> HostInstanceData:
    """Instances [lo, hi) of `init(layout, N, seed)` for any N >= hi, without
    materialising the prefix -- so each rank of a sharded run draws exactly
    the instances it owns and the union over ranks is the single-GPU store."""
    ir = from_layout(layout)
    n = hi - lo
    if n < 1:
        raise ValueError("need at least one instance")
    arrays = {}
    for slot in ir.slots:
        if slot.role == "parameter":
            arrays[slot.name] = np.full(n, slot.default if slot.default is not None else 0.0)
            continue
        if slot.ion_kind == "current":
            arrays[slot.name] = np.zeros(n)
            continue
        rng = _range_rng(seed, slot.name, lo)
        if slot.ion_kind == "conc":
            arrays[slot.name] = rng.uniform(*CONC_RANGE, n)
        elif slot.ion_kind == "reversal":
            arrays[slot.name] = rng.uniform(*REVERSAL_RANGE, n)
        elif slot.role == "state":
            arrays[slot.name] = rng.uniform(*STATE_RANGE, n)
        else:
            arrays[slot.name] = rng.uniform(*ASSIGNED_RANGE, n)
    arrays["v"] = _range_rng(seed, "v", lo).uniform(*V_RANGE, n)
    scalars = dict(ir.global_scalars)
    scalars["dt"] = dt
    return HostInstanceData(n, arrays, {"i_acc": np.zeros(n), "g_acc": np.zeros(n)}, scalars)


def node_layout(n: int, n_nodes: int, seed: int):
    """(node_index int32[n], node_v float64[n_nodes]) for the scatter workload."""
    rng = np.random.default_rng([seed, zlib.crc32(b"node_index")])
    node_index = rng.integers(0, n_nodes, n, dtype=np.int32)
    node_v = np.random.default_rng([seed, zlib.crc32(b"node_v")]).uniform(*V_RANGE, n_nodes)
    return node_index, node_v
