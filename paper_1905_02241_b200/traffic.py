"""Algorithmic HBM traffic of one launch (the roofline numerator).

The reference's measurement model (modlc/analysis.py:158-265, `_Traffic` /
`profile_kernel`) counts 8 bytes per distinct per-instance slot read plus 8
per distinct slot written, per kernel.  For the fused nrn_state+nrn_cur launch
SURVEY.md §8(d) fixes the unit: distinct slots over the *pair*, with v,
parameters, ion reads and the accumulators counted once each (hh: 10 reads +
8 writes = 144 B/instance-step).  The generated kernel's own load/store sets
(`MechAbi.kernels`) are exactly those distinct slots, so the model reads them
from the ABI instead of re-deriving them.

node_index variant (§8(d) workload 2): v is not a per-instance slot; each
instance reads its 4-byte node index and an 8-byte gathered node voltage, and
each node's rhs and d are read and written once per launch (32 B per node).
"""

from __future__ import annotations


def bytes_per_instance(abi, kernel: str = "step") -> int:
    k = abi.kernels[kernel]
    acc = 2 if kernel in ("step", "current_update", "step_nodes") else 0
    return 8 * (len(k["loads"]) + len(k["stores"]) + acc)


def launch_bytes(abi, n: int, kernel: str = "step", n_nodes: int = 0) -> int:
    """`n_nodes`: nodes that own at least one instance (the ones touched)."""
    if kernel == "step_nodes":
        per = bytes_per_instance(abi, "step_nodes") + 4 + 8
        return n * per + 32 * n_nodes
    return n * bytes_per_instance(abi, kernel)


def describe(abi, kernel: str = "step") -> dict:
    k = abi.kernels[kernel]
    return {
        "reads": list(k["loads"]) + (["node_index(4B)", "node_v(gather)"] if kernel == "step_nodes" else []),
        "writes": list(k["stores"]) + ["i_acc", "g_acc"],
        "bytes_per_instance": bytes_per_instance(abi, kernel) + (12 if kernel == "step_nodes" else 0),
    }
