"""Synthetic column (BASELINE configs[4]): seven populations over shared nodes,
Ca_HVA -> CaDynamics_E2 ion coupling, vs oracle/column_np.py; and shard
additivity (cells split across "ranks" = the single-shard checksums)."""

import numpy as np
import pytest

from oracle import column_np as CN
from oracle import interp_np as O
from parity import TOL, node_dev, parity

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("bench_options", [False, True])
@pytest.mark.parametrize("schedule", ["sequential", "concurrent", "grouped"])
def test_small_column_matches_oracle(bench_options, schedule):
    """Default builds, and the builds bench.py measures (bench.options_for:
    relaxed rate arithmetic, fast_redo, ... -- here in node_index mode with
    shared nodes and the one-instance-per-node path); every launch schedule
    (one stream, concurrent soma populations, the soma populations as one
    grouped launch)."""
    from paper_1905_02241_b200.column import COUPLINGS, LAUNCH_ORDER, ColumnShard, ColumnSpec, load_irs, shard_layout
    from paper_1905_02241_b200.instance import init_range

    spec = ColumnSpec(n_cells=300, dend_per_cell=5, syn_per_cell=12, seed=7)
    steps = 100
    opts = None
    if bench_options:
        from bench import options_for as opts
    shard = ColumnShard(spec, 0, spec.n_cells, opts, schedule=schedule)
    assert shard.schedule == schedule
    shard.launch(steps)
    shard.check()
    irs = load_irs()
    lay = shard_layout(spec, 0, spec.n_cells)
    datas = {m: init_range(irs[m], lay["mechs"][m][0], lay["mechs"][m][1], spec.seed) for m in LAUNCH_ORDER}
    datas = {m: O.InstanceData(x.n, x.arrays, x.acc, x.scalars) for m, x in datas.items()}
    idx = {m: lay["mechs"][m][2] for m in LAUNCH_ORDER}
    terms = {}
    ref, rhs, d = CN.simulate_column(irs, datas, idx, lay["node_v"], LAUNCH_ORDER, COUPLINGS, steps, terms=terms)
    for m in LAUNCH_ORDER:
        got = init_range(irs[m], lay["mechs"][m][0], lay["mechs"][m][1], spec.seed)
        shard.runners[m].to_host(shard.devs[m], got)
        dev, where = parity(irs[m], ref[m], got)
        assert dev <= TOL, (m, dev, where)
    nodes = shard.nodes.download(shard.stream)
    for name, want, scale in (("node_rhs", rhs, terms["rhs"]), ("node_d", d, terms["d"])):
        assert node_dev(nodes[name], want, scale) <= 1e-10, name


def test_column_shards_add_up():
    """Two shards of cells hold exactly the single-shard instances: per-array
    sums (checksums) of the two shards add to the whole column's."""
    from paper_1905_02241_b200.column import ColumnShard, ColumnSpec

    spec = ColumnSpec(n_cells=500, dend_per_cell=4, syn_per_cell=10, seed=3)
    whole = ColumnShard(spec, 0, 500)
    a, b = ColumnShard(spec, 0, 230), ColumnShard(spec, 230, 500)
    for s in (whole, a, b):
        s.launch(20)
        s.check()
    cw, ca, cb = whole.checksums(), a.checksums(), b.checksums()
    np.testing.assert_allclose(ca[:, 1] + cb[:, 1], cw[:, 1], rtol=1e-12)


def test_concurrent_soma_is_bit_identical_and_graph_capturable():
    """Every concurrent schedule (side streams + in-order combine; one
    grouped soma launch + combine) gives the sequential schedule's node
    rhs/d and states BIT FOR BIT, also when the step is captured into a CUDA
    graph (as bench.py does)."""
    from paper_1905_02241_b200 import runtime as rt
    from paper_1905_02241_b200.column import LAUNCH_ORDER, ColumnShard, ColumnSpec

    spec = ColumnSpec(n_cells=700, dend_per_cell=6, syn_per_cell=9, seed=5)
    seq = ColumnShard(spec, 0, spec.n_cells)
    seq.launch(30)
    seq.check()
    a = seq.nodes.download(seq.stream)
    for mode in ("concurrent", "grouped"):
        con = ColumnShard(spec, 0, spec.n_cells, schedule=mode)
        assert con.schedule == mode
        g = rt.capture(con.stream, lambda: con.launch(30))
        g.launch(con.stream)
        con.check()
        b = con.nodes.download(con.stream)
        for k in ("node_rhs", "node_d"):
            np.testing.assert_array_equal(a[k].view(np.int64), b[k].view(np.int64), err_msg=f"{mode}: {k}")
        np.testing.assert_array_equal(seq.checksums(), con.checksums(), err_msg=mode)
    assert set(LAUNCH_ORDER)


def test_two_process_column_shards(tmp_path):
    """Two real processes, each owning a CudaRunner shard of the column's cells
    (parallel.partition_cells), all-gather their device checksums through the
    product's process group (ranks sharing this one GPU -> FileGroup; NCCL
    needs a GPU per rank).  The gathered table equals, bit for bit, the
    tables of the same two shards built in this process, and the shards add
    up to the whole column."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    from paper_1905_02241_b200.column import ColumnShard, ColumnSpec

    n_cells, steps, world = 500, 20, 2
    out = str(tmp_path / "table.npy")
    worker = Path(__file__).resolve().parent / "mp_column_worker.py"
    procs = []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), LOCAL_RANK=str(r),
                   NMODL_BOOTSTRAP_DIR=str(tmp_path / "boot"))
        procs.append(subprocess.Popen([sys.executable, str(worker), out, str(n_cells), str(steps)], env=env))
    for p in procs:
        assert p.wait(timeout=600) == 0
    table = np.load(out)
    bounds = np.load(out + ".bounds.npy")
    spec = ColumnSpec(n_cells=n_cells, dend_per_cell=4, syn_per_cell=10, seed=3)
    for r in range(world):
        s = ColumnShard(spec, int(bounds[r]), int(bounds[r + 1]))
        s.launch(steps)
        s.check()
        np.testing.assert_array_equal(table[r], s.checksums())
    whole = ColumnShard(spec, 0, n_cells)
    whole.launch(steps)
    np.testing.assert_allclose(table[0][:, 1] + table[1][:, 1], whole.checksums()[:, 1], rtol=1e-12)


@pytest.mark.parametrize("bench_options", [False, True])
def test_errors_inside_the_soma_group_match_the_sequential_schedule(bench_options):
    """A soma population that fails inside the grouped launch (conductances
    so large that its current overflows for two cells) reports exactly the
    error the one-stream schedule reports (member status words, instance in
    caller order)."""
    from paper_1905_02241_b200.column import ColumnShard, ColumnSpec, host_stores
    from paper_1905_02241_b200.runner import InterpError

    spec = ColumnSpec(n_cells=400, dend_per_cell=3, syn_per_cell=5, seed=11)
    opts = None
    if bench_options:
        from bench import options_for as opts
    msgs = {}
    for schedule in ("sequential", "grouped"):
        host = host_stores(spec, 0, spec.n_cells)
        host["NaTs2_t"].arrays["gNaTs2_tbar"][[123, 45]] = 1e308
        host["NaTs2_t"].arrays["ena"][[123, 45]] = -1e300  # ina = g m^3 h (v - ena) overflows
        shard = ColumnShard(spec, 0, spec.n_cells, opts, schedule=schedule, host=host)
        assert shard.schedule == schedule
        shard.launch(3)
        with pytest.raises(InterpError) as e:
            shard.check()
        msgs[schedule] = str(e.value)
    assert msgs["grouped"] == msgs["sequential"]
    assert "instance 45 " in msgs["sequential"], msgs


def test_direct_population_group_is_bit_identical():
    """kind="direct" population group: the BBP set (NaTs2_t | K_Pst |
    Ca_HVA -> CaDynamics_E2 on the shared ica | SKv3_1 | Ih) stepped by ONE
    launch per timestep gives exactly the six separate launches' results."""
    import dataclasses

    from bench import options_for
    from paper_1905_02241_b200.instance import init
    from paper_1905_02241_b200.runner import CudaRunner, PopulationGroup
    from conftest import load_ir

    stems = ["NaTs2_t", "K_Pst", "Ca_HVA", "SKv3_1", "Ih", "cadyn"]
    n, steps = 50_001, 40
    outs = []
    for grouped in (False, True):
        rs, ds = {}, {}
        for m in stems:
            ir = load_ir(m)
            rs[m] = CudaRunner(ir, options=options_for(m))
            ds[m] = rs[m].to_device(init(ir, n, 7))
            rs[m].run_kernel(ds[m], "initialize", 1)
        rs["cadyn"].share_slot(ds["cadyn"], "ica", ds["Ca_HVA"], "ica")
        s = rs[stems[0]].stream
        for m in stems:
            rs[m].stream = s
        if grouped:
            cad = dataclasses.replace(rs["cadyn"].options, ilp=rs["Ca_HVA"].options.ilp)
            g = PopulationGroup("bbp_t", [[(rs["NaTs2_t"], ds["NaTs2_t"])], [(rs["K_Pst"], ds["K_Pst"])],
                                          [(rs["Ca_HVA"], ds["Ca_HVA"]), (rs["cadyn"], ds["cadyn"], cad)],
                                          [(rs["SKv3_1"], ds["SKv3_1"])], [(rs["Ih"], ds["Ih"])]], kind="direct")
            g.launch(s, steps)
        else:
            for _ in range(steps):
                for m in stems:
                    rs[m].launch(ds[m], "step", 1)
        s.sync()
        res = {}
        for m in stems:
            rs[m].check(ds[m])
            got = init(load_ir(m), n, 0)
            rs[m].to_host(ds[m], got)
            res[m] = got
        outs.append(res)
    for m in stems:
        for k in outs[0][m].arrays:
            np.testing.assert_array_equal(outs[0][m].arrays[k].view(np.int64), outs[1][m].arrays[k].view(np.int64),
                                          err_msg=f"{m}:{k}")
        for k in outs[0][m].acc:
            np.testing.assert_array_equal(outs[0][m].acc[k].view(np.int64), outs[1][m].acc[k].view(np.int64),
                                          err_msg=f"{m}:{k}")


def test_direct_group_with_newton_members_is_bit_identical():
    """The kinetic pair (register LU; Newton with an LU per iteration) as one
    direct group launch: states and currents equal the separate launches."""
    from bench import options_for
    from paper_1905_02241_b200.instance import init
    from paper_1905_02241_b200.runner import CudaRunner, PopulationGroup
    from conftest import load_ir

    stems = ["na6", "cdp5ish"]
    n, steps = 30_011, 60
    outs = []
    for grouped in (False, True):
        rs, ds = {}, {}
        for m in stems:
            ir = load_ir(m)
            rs[m] = CudaRunner(ir, options=options_for(m))
            ds[m] = rs[m].to_device(init(ir, n, 9))
            rs[m].run_kernel(ds[m], "initialize", 1)
        s = rs[stems[0]].stream
        for m in stems:
            rs[m].stream = s
        if grouped:
            PopulationGroup("kin_t", [[(rs[m], ds[m])] for m in stems], kind="direct").launch(s, steps)
        else:
            for _ in range(steps):
                for m in stems:
                    rs[m].launch(ds[m], "step", 1)
        s.sync()
        res = {}
        for m in stems:
            rs[m].check(ds[m])
            got = init(load_ir(m), n, 0)
            rs[m].to_host(ds[m], got)
            res[m] = got
        outs.append(res)
    for m in stems:
        for k in list(outs[0][m].arrays) + ["i_acc", "g_acc"]:
            a = outs[0][m].acc[k] if k in ("i_acc", "g_acc") else outs[0][m].arrays[k]
            b = outs[1][m].acc[k] if k in ("i_acc", "g_acc") else outs[1][m].arrays[k]
            np.testing.assert_array_equal(a.view(np.int64), b.view(np.int64), err_msg=f"{m}:{k}")
