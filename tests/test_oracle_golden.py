"""Pin the oracle (oracle/interp_np.py) to the reference runtime.

The golden trajectories were produced by the reference's own
modlc.interp.simulate (tools/make_golden.py); the oracle must reproduce them
bit-for-bit from the committed IR.  Known-answer constants are the
reference's (pkg/tests/test_interp.py:18, pkg/tests/test_odes.py:38-41).
"""

import json

import numpy as np
import pytest

from conftest import GOLDEN_DIR, all_ir_stems, load_ir
from oracle import interp_np as O

INDEX = json.loads((GOLDEN_DIR / "index.json").read_text())


def _unpack(z, prefix):
    arrays = {k[len(prefix) + 2:]: z[k] for k in z.files if k.startswith(prefix + "a:")}
    acc = {k[len(prefix) + 2:]: z[k] for k in z.files if k.startswith(prefix + "c:")}
    return arrays, acc, json.loads(str(z[prefix + "scalars"])), list(z[prefix + "newton_iters"])


def _assert_same(data, z, prefix):
    arrays, acc, scalars, iters = _unpack(z, prefix)
    assert list(data.arrays) == list(arrays)
    for k, v in arrays.items():
        np.testing.assert_array_equal(data.arrays[k], v, err_msg=k)
    for k, v in acc.items():
        np.testing.assert_array_equal(data.acc[k], v, err_msg=k)
    assert data.scalars == scalars
    assert data.newton_iters == iters


@pytest.mark.parametrize("stem", all_ir_stems())
def test_oracle_reproduces_reference_bit_exact(stem):
    meta = INDEX[stem]
    assert meta["status"] == "ok"
    z = np.load(GOLDEN_DIR / f"{stem}.npz")
    ir = load_ir(stem)
    data = O.init(ir, meta["n"], meta["seed"])
    runner = O.OracleRunner(ir)
    runner.run_kernel(data, "initialize", 1)
    _assert_same(data, z, "init/")
    for _ in range(meta["steps"]):
        runner.run_kernel(data, "state_update", 1)
        runner.run_kernel(data, "current_update", 1)
    _assert_same(data, z, "final/")
    if "fd/scalars" in z.files:
        fd = O.init(ir, meta["n"], meta["seed"])
        O.simulate(ir, fd, 10, jac_mode="fd")
        _assert_same(fd, z, "fd/")


@pytest.mark.parametrize("stem", sorted(INDEX["_compare_pipelines"]))
def test_oracle_compare_pipelines_matches_reference(stem):
    a = load_ir(f"{stem}.nopass")
    b = load_ir(stem)
    assert O.compare_pipelines(a, b, 32, 42, 20) == INDEX["_compare_pipelines"][stem]


GATE = {"format": "nmodl-b200-ir/1"}


def test_cnexp_one_step_known_answer():
    """1 - exp(-0.025) (pkg/tests/test_interp.py:18,77-84) via cat-free gate."""
    from paper_1905_02241_b200.ir import MechIR, Node, Slot

    num = lambda x: Node("Number", (), {"value": float(x)})
    ident = lambda n: Node("Identifier", (), {"name": n})
    b = lambda op, l, r: Node("Binary", (l, r), {"op": op})
    # y = -(1) + (y + 1)*exp(-dt)  is what cnexp emits for y' = (1 - y)/1
    upd = Node("Assign", (ident("y"), b("+", num(1.0), b("*", Node("Call", (Node("Unary", (ident("dt"),), {"op": "-"}),), {"name": "exp"}), b("-", ident("y"), num(1.0))))))
    ir = MechIR("gate", [Slot("y", "state", 0)], {"dt": 0.025, "celsius": 6.3},
                {"initialize": (Node("Assign", (ident("y"), num(0.0))),), "state_update": (upd,), "current_update": ()},
                {}, [], {})
    data = O.init(ir, 4, 0)
    r = O.OracleRunner(ir)
    r.run_kernel(data, "initialize", 1)
    r.run_kernel(data, "state_update", 1)
    assert np.allclose(data.arrays["y"], INDEX["_constants"]["CNEXP_ONE_STEP_TRUE"], rtol=1e-13, atol=0)


def test_two_state_equilibrium_and_conservation():
    """pkg/tests/test_interp.py:87-98 on the corpus twostate scheme."""
    ir = load_ir("corpus_twostate")
    data = O.init(ir, 8, 0)
    r = O.OracleRunner(ir)
    r.run_kernel(data, "initialize", 1)
    for _ in range(2000):
        r.run_kernel(data, "state_update", 1)
        assert np.max(np.abs(data.arrays["A"] + data.arrays["B"] - 1.0)) <= 1e-12
    assert np.allclose(data.arrays["A"], 1.0 / 3.0, atol=1e-9)
    assert np.allclose(data.arrays["B"], 2.0 / 3.0, atol=1e-9)


def test_lu_solve_batched_against_numpy():
    """pkg/tests/test_interp.py:189-195."""
    rng = np.random.default_rng(0)
    a = rng.normal(size=(32, 5, 5))
    b = rng.normal(size=(32, 5))
    expected = np.linalg.solve(a, b[..., None])[..., 0]
    assert np.allclose(O.lu_solve_batched(a, b), expected, rtol=1e-10, atol=1e-12)


def test_permutation_invariance_corpus():
    """pkg/tests/test_interp.py:198-200, widened to several mechanisms."""
    for stem in ("corpus_cat", "hh_subset", "corpus_fourstate", "corpus_cacum"):
        assert O.permutation_invariant(load_ir(stem), 64, 11, 10) == 0.0


def test_newton_nonconvergence_message():
    ir = load_ir("corpus_cacum")
    data = O.init(ir, 4, 0)
    r = O.OracleRunner(ir)
    r.run_kernel(data, "initialize", 1)
    data.scalars["dt"] = 1e12
    data.arrays["ica"][:] = 1e30
    with pytest.raises(O.InterpError, match="Newton failed to converge for instance 0"):
        r.run_kernel(data, "state_update", 1)


def test_nonfinite_reports_first_instance():
    ir = load_ir("hh_subset")
    data = O.init(ir, 8, 0)
    data.arrays["v"][5] = np.nan
    with pytest.raises(O.InterpError, match="at instance 5 after kernel initialize"):
        O.OracleRunner(ir).run_kernel(data, "initialize", 1)
