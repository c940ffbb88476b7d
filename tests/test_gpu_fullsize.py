"""Parity at the BASELINE.json sizes through size-independent properties.

The oracle cannot run 10M instances x 1000 steps in test time, but the
domain gives exact size-independent checks:

* prefix stability -- `init` draws one seeded stream per slot, so the first k
  instances of an n-instance store equal a k-instance store, and instances
  never interact (modlc/interp.py:55-84, 706-723): the first 65,536 results
  of the full-size GPU run must match the oracle run on 65,536 instances;
* node sums -- node rhs/d are rebuilt every step, so after the full-size
  run they must be bit-identical to sequential np.subtract.at / np.add.at
  applied to the GPU's own final per-instance currents;
* determinism / permutation invariance -- two full-size runs, one of them on
  a permuted store, give bit-identical per-instance results.

The full-size runs use the builds bench.py measures (bench.options_for) and
its population set-up (bbp20m's Ca_HVA -> CaDynamics_E2 shared ica slot);
the oracle side of the 65,536-instance prefixes runs chunked over the host
cores (tests/oracle_pool.py).  The default builds are covered at small sizes
by test_gpu_parity.py.
"""

import numpy as np
import pytest

from conftest import load_ir
from oracle import interp_np as O
from oracle import nodes_np as N
from oracle_pool import oracle_prefix
from parity import TOL, parity

pytestmark = pytest.mark.gpu
PREFIX = 65536


def _runner(stem, ir):
    from bench import options_for
    from paper_1905_02241_b200.runner import CudaRunner

    return CudaRunner(ir, options=options_for(stem))


def _prefix(data, k):
    return O.InstanceData(k, {n: a[:k].copy() for n, a in data.arrays.items()},
                          {n: a[:k].copy() for n, a in data.acc.items()}, dict(data.scalars), list(data.newton_iters))


def test_hh_1m_1000_steps_prefix_matches_oracle():
    from paper_1905_02241_b200.instance import init
    from paper_1905_02241_b200.runner import CudaRunner, simulate

    ir = load_ir("hh_subset")
    n, steps = 1_000_000, 1000
    gpu = simulate(ir, init(ir, n, 42), steps, runner=_runner("hh_subset", ir))
    ref = O.simulate(ir, O.init(ir, PREFIX, 42), steps)
    dev, where = parity(ir, ref, _prefix(gpu, PREFIX))
    assert dev <= TOL, (dev, where)


def test_synapse_10m_nodes_1000_steps():
    from paper_1905_02241_b200.instance import init, node_layout
    from paper_1905_02241_b200.runner import CudaRunner, simulate_nodes

    ir = load_ir("ProbAMPANMDA_EMS")
    n, n_nodes, steps = 10_000_000, 1_000_000, 1000
    idx, nv = node_layout(n, n_nodes, 42)
    gpu, rhs, d = simulate_nodes(ir, init(ir, n, 42), steps, idx, nv, runner=_runner("ProbAMPANMDA_EMS", ir))
    # per-instance prefix vs the oracle driven by the same gathered voltages
    ref = O.init(ir, PREFIX, 42)
    ref, _, _ = N.simulate_nodes(ir, ref, steps, idx[:PREFIX], nv)
    dev, where = parity(ir, ref, _prefix(gpu, PREFIX))
    assert dev <= TOL, (dev, where)
    # node rhs/d hold the last step's reduction (per-step reset): bit-exact
    # against the in-order scatter of the GPU's own final currents
    rhs_ref, d_ref = np.zeros(n_nodes), np.zeros(n_nodes)
    N.scatter(rhs_ref, d_ref, idx, gpu.acc["i_acc"], gpu.acc["g_acc"])
    np.testing.assert_array_equal(rhs, rhs_ref)
    np.testing.assert_array_equal(d, d_ref)
    assert np.all(np.isfinite(rhs)) and np.all(np.isfinite(d))


def test_bbp20m_coupled_as_bench_runs_it():
    """bench.py's bbp20m step exactly: six populations of 3,333,333 instances,
    its builds, one stream in launch order, CaDynamics_E2 reading Ca_HVA's ica
    array (share_slot), nrn_init then 1000 steps; the first 65,536 instances
    of every population vs the coupled oracle (same order, same coupling)."""
    from bench import WORKLOADS
    from paper_1905_02241_b200.instance import init

    w = WORKLOADS["bbp20m"]
    stems = [m for m, _ in w["mechs"]]
    n, steps = w["mechs"][0][1], 1000
    runners, devs = {}, {}
    for m in stems:
        ir = load_ir(m)
        r = _runner(m, ir)
        devs[m] = r.to_device(init(ir, n, 42))
        r.run_kernel(devs[m], "initialize", 1)
        runners[m] = r
    for dst, dslot, src, sslot in w["couplings"]:
        runners[dst].share_slot(devs[dst], dslot, devs[src], sslot)
    s0 = runners[stems[0]].stream
    for m in stems:
        runners[m].stream = s0
    for _ in range(steps):
        for m in stems:
            runners[m].launch(devs[m], "step", 1)
    s0.sync()
    ref = oracle_prefix(stems, PREFIX, steps, 42, w["couplings"])
    for m in stems:
        runners[m].check(devs[m])
        got = init(load_ir(m), n, 0)
        runners[m].to_host(devs[m], got)
        dev, where = parity(load_ir(m), ref[m], _prefix(got, PREFIX))
        assert dev <= TOL, (m, dev, where)
        del got


def test_bbp_set_permutation_invariance():
    from paper_1905_02241_b200.instance import init
    from paper_1905_02241_b200.runner import CudaRunner, simulate

    n, steps = 3_333_333, 300
    for stem in ("NaTs2_t", "K_Pst", "Ca_HVA", "SKv3_1", "Ih", "cadyn"):
        ir = load_ir(stem)
        runner = _runner(stem, ir)
        base = init(ir, n, 42)
        gpu = simulate(ir, base.copy(), steps, runner=runner)
        # permuted store -> identical per-instance bits after un-permuting
        perm = np.random.default_rng(1).permutation(n)
        shuffled = base.copy()
        for k in shuffled.arrays:
            shuffled.arrays[k] = shuffled.arrays[k][perm].copy()
        out = simulate(ir, shuffled, steps, runner=runner)
        inv = np.argsort(perm)
        for k in gpu.arrays:
            np.testing.assert_array_equal(out.arrays[k][inv], gpu.arrays[k], err_msg=f"{stem}:{k}")


_KINETIC_REF = {}


@pytest.mark.parametrize("n", [1_000_000, 10_000_000])
def test_kinetic_prefix(n):
    """kinetic1m and kinetic10m as bench.py runs them (1000 steps, bench
    builds): the first 65,536 instances vs the oracle (computed once)."""
    from paper_1905_02241_b200.instance import init
    from paper_1905_02241_b200.runner import CudaRunner, simulate

    for stem in ("na6", "cdp5ish"):
        ir = load_ir(stem)
        gpu = simulate(ir, init(ir, n, 42), 1000, runner=_runner(stem, ir))
        if stem not in _KINETIC_REF:
            _KINETIC_REF[stem] = oracle_prefix([stem], PREFIX, 1000, 42)[stem]
        ref = _KINETIC_REF[stem]
        dev, where = parity(ir, ref, _prefix(gpu, PREFIX))
        assert dev <= TOL, (stem, n, dev, where)
        if stem == "cdp5ish":
            assert gpu.newton_iters and max(gpu.newton_iters) <= 50
        del gpu


def test_column_100k_as_bench_runs_it_prefix_matches_oracle():
    """configs[4] exactly as bench.py runs it (100,000 cells, bench builds,
    the grouped soma schedule, 1000 steps): cells never interact and every
    cell's instances, synapse compartments and node voltages are drawn from
    global ids (column.shard_layout), so the first 150 cells of the full
    column must equal the 150-cell column -- states, currents and the node
    rhs/d of those cells' compartments -- against oracle/column_np.py."""
    from bench import _column_mode, options_for
    from oracle import column_np as CN
    from paper_1905_02241_b200.column import (COUPLINGS, LAUNCH_ORDER, ColumnShard, ColumnSpec, load_irs,
                                              shard_layout)
    from paper_1905_02241_b200.instance import init_range
    from parity import node_dev

    full = ColumnSpec(n_cells=100_000)
    k_cells, steps = 150, 1000
    shard = ColumnShard(full, 0, full.n_cells, options_for, **_column_mode())
    shard.launch(steps)
    shard.check()
    irs = load_irs()
    small = ColumnSpec(n_cells=k_cells, dend_per_cell=full.dend_per_cell, syn_per_cell=full.syn_per_cell,
                       seed=full.seed)
    lay = shard_layout(small, 0, k_cells)
    datas = {m: init_range(irs[m], lay["mechs"][m][0], lay["mechs"][m][1], small.seed) for m in LAUNCH_ORDER}
    datas = {m: O.InstanceData(x.n, x.arrays, x.acc, x.scalars) for m, x in datas.items()}
    idx = {m: lay["mechs"][m][2] for m in LAUNCH_ORDER}
    terms = {}
    ref, rhs, d = CN.simulate_column(irs, datas, idx, lay["node_v"], LAUNCH_ORDER, COUPLINGS, steps, terms=terms)
    for m in LAUNCH_ORDER:
        lo, hi, _ = shard.layout["mechs"][m]
        got = init_range(irs[m], lo, hi, full.seed)
        shard.runners[m].to_host(shard.devs[m], got)
        k = lay["mechs"][m][1]  # the small column's instance count of m
        dev, where = parity(irs[m], ref[m], _prefix(got, k))
        assert dev <= TOL, (m, dev, where)
        del got
    nodes = shard.nodes.download(shard.stream)
    nn = k_cells * full.nodes_per_cell
    for name, want, scale in (("node_rhs", rhs, terms["rhs"]), ("node_d", d, terms["d"])):
        assert node_dev(nodes[name][:nn], want, scale) <= 1e-10, name
