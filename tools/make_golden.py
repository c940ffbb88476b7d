"""Generate tests/golden/*.npz from the REFERENCE runtime (modlc.interp).

Each fixture mechanism is compiled by the reference front-end and simulated by
the reference's own `interp.simulate` (modlc/interp.py:640-655) on
`interp.init(layout, n, seed)` inputs.  The final instance store (arrays,
accumulators, scalars, Newton iteration record) is saved, together with the
store right after `initialize`.  tests/test_oracle_golden.py then requires
oracle/interp_np.py to reproduce these trajectories bit-for-bit from the
committed IR JSON, which pins the oracle to the reference.

Run here (the reference tree is needed):  python tools/make_golden.py
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_1905_02241_b200.frontend import _import_modlc  # noqa: E402
from paper_1905_02241_b200.ir import MechIR  # noqa: E402

OUT = ROOT / "tests" / "golden"
N = 64
SEED = 42
STEPS = 40


def _layout_for(ir: MechIR):
    """Recompile the IR's source with the recorded options via the reference."""
    from modlc.corpus import corpus_path
    from modlc.pipeline import compile_file

    fname = ir.meta["file"]
    opts = dict(ir.meta.get("options", {}))
    if "passes" in opts:
        opts["passes"] = tuple(opts["passes"])
    local = ROOT / "fixtures" / "mod" / fname
    path = local if local.is_file() else corpus_path(fname)
    return compile_file(path, **opts).layout


def _pack(prefix, data, out):
    for k, v in data.arrays.items():
        out[f"{prefix}a:{k}"] = v.copy()
    for k, v in data.acc.items():
        out[f"{prefix}c:{k}"] = v.copy()
    out[f"{prefix}scalars"] = np.array(json.dumps(data.scalars))
    out[f"{prefix}newton_iters"] = np.array(data.newton_iters, dtype=np.int64)


def main() -> int:
    _import_modlc()
    from modlc import interp

    OUT.mkdir(parents=True, exist_ok=True)
    index = {}
    for path in sorted((ROOT / "fixtures" / "ir").glob("*.json")):
        ir = MechIR.load(path)
        stem = path.stem
        layout = _layout_for(ir)
        out = {}
        try:
            data = interp.init(layout, N, SEED)
            runner = interp.Runner(layout)
            runner.run_kernel(data, "initialize", 1)
            _pack("init/", data, out)
            for _ in range(STEPS):
                runner.run_kernel(data, "state_update", 1)
                runner.run_kernel(data, "current_update", 1)
            _pack("final/", data, out)
            status = "ok"
        except interp.InterpError as exc:
            status = f"InterpError: {exc}"
        if any(node_kind == "NewtonSolveNode" for node_kind in _kinds(ir)):
            data = interp.init(layout, N, SEED)
            interp.simulate(layout, data, 10, jac_mode="fd")
            _pack("fd/", data, out)
        np.savez_compressed(OUT / f"{stem}.npz", **out)
        index[stem] = {"status": status, "n": N, "seed": SEED, "steps": STEPS}
        print(stem, status)
    # reference known-answer constants (pkg/tests/test_interp.py:18, test_odes.py:38-41)
    index["_constants"] = {
        "CNEXP_ONE_STEP_TRUE": 0.024690087971667333,
        "PADE_ONE_STEP_TRUE": 0.024691358024691357,
        "NEWTON_QUAD_ROOT": 0.9160797830996161,
    }
    # reference differential checks on the corpus: passes vs none (SPEC: deviation 0 / <=1e-12)
    diffs = {}
    for path in sorted((ROOT / "fixtures" / "ir").glob("*.nopass.json")):
        stem = path.stem[: -len(".nopass")]
        if not (ROOT / "fixtures" / "ir" / f"{stem}.json").is_file():
            continue
        try:
            a = _layout_for(MechIR.load(path))
            b = _layout_for(MechIR.load(ROOT / "fixtures" / "ir" / f"{stem}.json"))
            diffs[stem] = interp.compare_pipelines(a, b, 32, SEED, 20)
        except interp.InterpError as exc:
            diffs[stem] = f"InterpError: {exc}"
    index["_compare_pipelines"] = diffs
    (OUT / "index.json").write_text(json.dumps(index, indent=1, sort_keys=True) + "\n")
    return 0


def _kinds(ir):
    from paper_1905_02241_b200.ir import iter_nodes

    for stmts in ir.kernels.values():
        for s in stmts:
            for node in iter_nodes(s):
                yield node.kind


if __name__ == "__main__":
    raise SystemExit(main())
