"""node_index gather / deterministic segmented scatter vs oracle/nodes_np.py."""

import numpy as np
import pytest

from conftest import load_ir
from oracle import interp_np as O
from oracle import nodes_np as N
from parity import TOL, node_dev, parity

NODE_TOL = 1e-10  # node rhs/d, relative to max(|value|, sum of |terms|) (metrics.node_dev)


def _check_nodes(rhs_gpu, d_gpu, rhs_ref, d_ref, terms):
    assert node_dev(rhs_gpu, rhs_ref, terms["rhs"]) <= NODE_TOL
    assert node_dev(d_gpu, d_ref, terms["d"]) <= NODE_TOL

pytestmark = pytest.mark.gpu


def _inputs(n, n_nodes, seed):
    from paper_1905_02241_b200.instance import node_layout

    return node_layout(n, n_nodes, seed)


@pytest.mark.parametrize("n,n_nodes", [(5000, 500), (3000, 7), (4096, 4096), (2000, 1)])
def test_scatter_layout_bit_exact(n, n_nodes):
    """Stable sort permutation, its inverse and node offsets are bit-exact."""
    from paper_1905_02241_b200.runner import CudaRunner

    ir = load_ir("ProbAMPANMDA_EMS")
    idx, nv = _inputs(n, n_nodes, 3)
    r = CudaRunner(ir)
    dev = r.to_device(O.init(ir, n, 1))
    r.bind_nodes(dev, idx, nv)
    got = r.node_arrays(dev)
    perm, offsets, rank = N.scatter_layout(idx, n_nodes)
    np.testing.assert_array_equal(got["perm"], perm)
    np.testing.assert_array_equal(got["rank"], rank)
    np.testing.assert_array_equal(got["offsets"], offsets)
    np.testing.assert_array_equal(got["node_index_sorted"], idx[perm])


@pytest.mark.parametrize("stem,n,n_nodes,steps", [
    ("ProbAMPANMDA_EMS", 20000, 2000, 200),
    ("ProbAMPANMDA_EMS", 6000, 3, 50),       # huge segments: global-memory reduction path
    ("hh_subset", 8192, 8192, 100),
    ("corpus_exp2syn", 10000, 999, 100),
    ("na6", 4000, 400, 50),
])
@pytest.mark.parametrize("reset", [True, False])
def test_simulate_nodes_matches_oracle(stem, n, n_nodes, steps, reset):
    """Per-step node reset (default: rhs/d rebuilt every timestep, as a cable
    solver does) and the accumulate-across-steps form; node rhs/d at 1e-10."""
    from paper_1905_02241_b200.runner import simulate_nodes

    ir = load_ir(stem)
    idx, nv = _inputs(n, n_nodes, 11)
    rhs0 = np.linspace(-1.0, 1.0, n_nodes)
    d0 = np.linspace(0.5, 2.0, n_nodes)
    terms = {}
    ref, rhs_ref, d_ref = N.simulate_nodes(ir, O.init(ir, n, 5), steps, idx, nv, rhs0, d0, reset=reset, terms=terms)
    gpu, rhs_gpu, d_gpu = simulate_nodes(ir, O.init(ir, n, 5), steps, idx, nv, rhs0.copy(), d0.copy(), reset=reset)
    dev, where = parity(ir, ref, gpu)
    assert dev <= TOL, (where, dev)
    if not reset:  # the initial values are part of the sums
        terms = {"rhs": terms["rhs"] + np.abs(rhs0), "d": terms["d"] + np.abs(d0)}
    _check_nodes(rhs_gpu, d_gpu, rhs_ref, d_ref, terms)


@pytest.mark.parametrize("pipe", [False, True])
def test_scatter_arithmetic_bit_exact(pipe):
    """Given the GPU's own per-instance i_acc/g_acc, the node sums are
    bit-identical to sequential np.subtract.at / np.add.at (shared-memory
    staged currents, and the pipelined kernel's L2 read-back)."""
    from paper_1905_02241_b200.codegen_cuda import CudaOptions
    from paper_1905_02241_b200.runner import CudaRunner, simulate_nodes

    ir = load_ir("ProbAMPANMDA_EMS")
    n, n_nodes = 30000, 1234
    idx, nv = _inputs(n, n_nodes, 2)
    rhs0 = np.zeros(n_nodes)
    d0 = np.zeros(n_nodes)
    runner = CudaRunner(ir, options=CudaOptions(fast_path=False, pipe=pipe))
    gpu, rhs_gpu, d_gpu = simulate_nodes(ir, O.init(ir, n, 9), 1, idx, nv, rhs0.copy(), d0.copy(), runner=runner)
    rhs_ref, d_ref = rhs0.copy(), d0.copy()
    N.scatter(rhs_ref, d_ref, idx, gpu.acc["i_acc"], gpu.acc["g_acc"])
    np.testing.assert_array_equal(rhs_gpu, rhs_ref)
    np.testing.assert_array_equal(d_gpu, d_ref)


@pytest.mark.parametrize("stem", ["Ih", "hh_subset", "ProbAMPANMDA_EMS"])
def test_one_instance_per_node_path(stem):
    """node_index a permutation (density mechanisms: <= 1 instance per
    compartment): the conflict-free direct-update path, same results."""
    from paper_1905_02241_b200.runner import CudaRunner, simulate_nodes

    ir = load_ir(stem)
    n = 7001
    idx = np.random.default_rng(5).permutation(n).astype(np.int32)
    nv = np.random.default_rng(6).uniform(-80, 40, n)
    terms = {}
    ref, rhs_ref, d_ref = N.simulate_nodes(ir, O.init(ir, n, 2), 40, idx, nv, terms=terms)
    runner = CudaRunner(ir)
    gpu, rhs_gpu, d_gpu = simulate_nodes(ir, O.init(ir, n, 2), 40, idx, nv, runner=runner)
    dev, where = parity(ir, ref, gpu)
    assert dev <= TOL, (where, dev)
    _check_nodes(rhs_gpu, d_gpu, rhs_ref, d_ref, terms)


@pytest.mark.parametrize("n,n_nodes,tile", [(5000, 500, 64), (5000, 500, 1536), (3000, 7, 100), (4096, 4096, 256),
                                           (2000, 1, 64), (100000, 250000, 700), (1, 3, 64)])
def test_device_segments_and_tiles_match_host_restatement(n, n_nodes, tile):
    """nmodl_node_segments (device) == the numpy restatement in runner.py."""
    from paper_1905_02241_b200.runner import CudaRunner, tile_nodes_for

    ir = load_ir("ProbAMPANMDA_EMS")
    idx, nv = _inputs(n, n_nodes, 4)
    r = CudaRunner(ir)
    dev = r.to_device(O.init(ir, n, 1))
    nb = r.bind_nodes(dev, idx, nv, tile=tile)
    _, offsets, _ = N.scatter_layout(idx, n_nodes)
    seg_node = np.flatnonzero(np.diff(offsets))
    seg_off = np.concatenate([offsets[seg_node], [n]]).astype(np.int64)
    assert nb.n_segs == len(seg_node)
    np.testing.assert_array_equal(nb.seg_offsets_host, seg_off)
    np.testing.assert_array_equal(nb.tile_segs_host, tile_nodes_for(seg_off, tile))
    assert nb.seg_unique == (1 if len(seg_node) == n else 0)


def test_write_back_covers_every_array():
    """simulate_nodes copies back only what the device may have changed; the
    result must still equal the oracle's whole store (parameters untouched,
    v = gathered node voltage, accumulators, states)."""
    from paper_1905_02241_b200.runner import simulate_nodes

    ir = load_ir("ProbAMPANMDA_EMS")
    n, n_nodes = 7000, 900
    idx, nv = _inputs(n, n_nodes, 2)
    base = O.init(ir, n, 8)
    base.arrays["v"][:] = 1e300  # never read: the voltage comes from the nodes
    ref, _, _ = N.simulate_nodes(ir, base.copy(), 20, idx, nv)
    gpu, _, _ = simulate_nodes(ir, base.copy(), 20, idx, nv)
    for name in ref.arrays:
        if name not in ir_states_and_assigned(ir):
            np.testing.assert_array_equal(gpu.arrays[name], ref.arrays[name], err_msg=name)
    dev, where = parity(ir, ref, gpu)
    assert dev <= TOL, (where, dev)


def ir_states_and_assigned(ir):
    from paper_1905_02241_b200.codegen_cuda import CudaPrinter

    p = CudaPrinter(ir)
    p.emit_unit()
    out = set()
    for k in p._abi.kernels.values():
        out |= set(k["stores"])
    return out


def test_nonfinite_node_voltage_reports_like_oracle():
    from paper_1905_02241_b200.runner import InterpError, simulate_nodes

    ir = load_ir("hh_subset")
    n, n_nodes = 3000, 300
    idx, nv = _inputs(n, n_nodes, 5)
    nv = nv.copy()
    nv[idx[1234]] = np.nan
    with pytest.raises(O.InterpError) as e_ref:
        N.simulate_nodes(ir, O.init(ir, n, 1), 5, idx, nv)
    with pytest.raises(InterpError) as e_gpu:
        simulate_nodes(ir, O.init(ir, n, 1), 5, idx, nv)
    assert str(e_gpu.value) == str(e_ref.value)


@pytest.mark.parametrize("waves,tile", [(0, 2048), (0, 256), (2, 1024)])
def test_node_kernel_grid_waves_matches_oracle(waves, tile):
    """Node kernel with one CTA per tile (grid_waves=0) or two resident
    waves: same trajectories, node rhs/d as the in-order oracle."""
    from paper_1905_02241_b200.codegen_cuda import CudaOptions
    from paper_1905_02241_b200.runner import CudaRunner, simulate_nodes

    ir = load_ir("ProbAMPANMDA_EMS")
    n, n_nodes = 30000, 3000
    idx, nv = _inputs(n, n_nodes, 5)
    terms = {}
    ref, rhs_ref, d_ref = N.simulate_nodes(ir, O.init(ir, n, 9), 40, idx, nv, terms=terms)
    runner = CudaRunner(ir, options=CudaOptions(fast_path=False, tile=tile, grid_waves=waves))
    gpu, rhs_gpu, d_gpu = simulate_nodes(ir, O.init(ir, n, 9), 40, idx, nv, runner=runner)
    dev, where = parity(ir, ref, gpu)
    assert dev <= TOL, (where, dev)
    _check_nodes(rhs_gpu, d_gpu, rhs_ref, d_ref, terms)


NODE_PIPE = [dict(fast_path=False, pipe=True), dict(fast_path=True, fast_redo=True, pipe=True)]


@pytest.mark.parametrize("variant", range(len(NODE_PIPE)))
@pytest.mark.parametrize("n,n_nodes,tile", [(20000, 2000, 512), (6000, 3, 512), (9000, 4000, 128), (777, 50, 64),
                                           (30000, 30000, 2048)])
def test_node_kernel_cp_async_pipeline_matches_oracle(variant, n, n_nodes, tile):
    """Node kernel with the per-thread cp.async pipeline (CudaOptions.pipe):
    the next instance -- possibly the first of the next tile -- is in flight
    while the current one computes; tiles smaller than the block leave
    threads without instances; huge segments exceed the tile.  Same
    trajectories, node rhs/d as the in-order oracle."""
    from paper_1905_02241_b200.codegen_cuda import CudaOptions
    from paper_1905_02241_b200.runner import CudaRunner, simulate_nodes

    ir = load_ir("ProbAMPANMDA_EMS")
    idx, nv = _inputs(n, n_nodes, 6)
    terms = {}
    ref, rhs_ref, d_ref = N.simulate_nodes(ir, O.init(ir, n, 10), 50, idx, nv, terms=terms)
    kw = NODE_PIPE[variant]
    runner = CudaRunner(ir, options=CudaOptions(tile=tile, **kw))
    gpu, rhs_gpu, d_gpu = simulate_nodes(ir, O.init(ir, n, 10), 50, idx, nv, runner=runner)
    dev, where = parity(ir, ref, gpu)
    assert dev <= TOL, (where, dev)
    _check_nodes(rhs_gpu, d_gpu, rhs_ref, d_ref, terms)



@pytest.mark.parametrize("stem", ["Ih", "hh_subset", "NaTs2_t", "cadyn", "K_Pst"])
@pytest.mark.parametrize("sparse", [False, True])
def test_step_unique_kernel(stem, sparse):
    """One instance per node with a pipelined build (bench.options_for): the
    `step_unique` kernel (direct kernels' cp.async pipeline and ILP, v
    gathered from the node, each instance folding into its own node) gives
    the tiled step_nodes path's states, currents and node rhs/d BIT FOR BIT,
    and matches the oracle.  `sparse`: fewer instances than nodes (somas)."""
    from bench import options_for
    from paper_1905_02241_b200.runner import CudaRunner, simulate_nodes

    ir = load_ir(stem)
    n, n_nodes = 9001, (3 * 9001 if sparse else 9001)
    idx = np.random.default_rng(5).permutation(n_nodes)[:n].astype(np.int32)
    nv = np.random.default_rng(6).uniform(-80, 40, n_nodes)
    terms = {}
    ref, rhs_ref, d_ref = N.simulate_nodes(ir, O.init(ir, n, 2), 60, idx, nv, terms=terms)
    fast = CudaRunner(ir, options=options_for(stem))
    assert "step_unique" in fast.entry
    a, rhs_a, d_a = simulate_nodes(ir, O.init(ir, n, 2), 60, idx, nv, runner=fast)
    tiled = CudaRunner(ir, options=options_for(stem))
    del tiled.entry["step_unique"]  # force the tiled node kernel
    b, rhs_b, d_b = simulate_nodes(ir, O.init(ir, n, 2), 60, idx, nv, runner=tiled)
    for k in a.arrays:
        np.testing.assert_array_equal(a.arrays[k].view(np.int64), b.arrays[k].view(np.int64), err_msg=k)
    for k in a.acc:
        np.testing.assert_array_equal(a.acc[k].view(np.int64), b.acc[k].view(np.int64), err_msg=k)
    np.testing.assert_array_equal(rhs_a.view(np.int64), rhs_b.view(np.int64))
    np.testing.assert_array_equal(d_a.view(np.int64), d_b.view(np.int64))
    dev, where = parity(ir, ref, a)
    assert dev <= TOL, (where, dev)
    _check_nodes(rhs_a, d_a, rhs_ref, d_ref, terms)


def test_unused_arrays_are_not_uploaded_but_still_checked():
    """simulate_nodes leaves arrays no kernel reads or writes (the synapse's
    Use, Dep, Fac, u0, Nrrp) on the host -- same results bit for bit as the
    whole-store upload -- and a non-finite value in one of them still raises
    the oracle's error (found by the host scan, the call is redone with the
    whole store)."""
    from paper_1905_02241_b200.runner import CudaRunner, InterpError, _unread_arrays, simulate_nodes

    ir = load_ir("ProbAMPANMDA_EMS")
    n, n_nodes = 20_000, 3_000
    idx, nv = _inputs(n, n_nodes, 12)
    r = CudaRunner(ir)
    assert set(_unread_arrays(r, O.init(ir, 8, 1), ("initialize", "step_nodes"))) == {"Use", "Dep", "Fac", "u0", "Nrrp"}
    a, rhs_a, d_a = simulate_nodes(ir, O.init(ir, n, 2), 50, idx, nv, runner=r)
    b, rhs_b, d_b = simulate_nodes(ir, O.init(ir, n, 2), 50, idx, nv, runner=r, _skip_unread=False)
    for k in a.arrays:
        np.testing.assert_array_equal(a.arrays[k].view(np.int64), b.arrays[k].view(np.int64), err_msg=k)
    np.testing.assert_array_equal(rhs_a.view(np.int64), rhs_b.view(np.int64))
    np.testing.assert_array_equal(d_a.view(np.int64), d_b.view(np.int64))
    bad = O.init(ir, n, 2)
    bad.arrays["Dep"][777] = np.inf
    with pytest.raises(Exception) as want:
        N.simulate_nodes(ir, bad.copy(), 5, idx, nv)
    with pytest.raises(InterpError) as got:
        simulate_nodes(ir, bad.copy(), 5, idx, nv, runner=r)
    assert str(got.value) == str(want.value)
    assert "'Dep'" in str(got.value)


def test_simulate_skips_unused_arrays_the_same_way():
    from paper_1905_02241_b200.runner import CudaRunner, InterpError, simulate

    ir = load_ir("ProbAMPANMDA_EMS")
    r = CudaRunner(ir)
    a = simulate(ir, O.init(ir, 5000, 3), 40, runner=r)
    b = simulate(ir, O.init(ir, 5000, 3), 40, runner=r, _skip_unread=False)
    for k in a.arrays:
        np.testing.assert_array_equal(a.arrays[k].view(np.int64), b.arrays[k].view(np.int64), err_msg=k)
    bad = O.init(ir, 5000, 3)
    bad.arrays["u0"][4321] = np.nan
    with pytest.raises(Exception) as want:
        O.simulate(ir, bad.copy(), 5)
    with pytest.raises(InterpError) as got:
        simulate(ir, bad.copy(), 5, runner=r)
    assert str(got.value) == str(want.value)


@pytest.mark.parametrize("flags", [0, 1])
@pytest.mark.parametrize("n_pops", [1, 2, 5, 8])
def test_combine_unique_in_population_order(n_pops, flags):
    """nmodl_combine_unique_ex (plain and programmatic launch) folds the
    populations' currents into node rhs/d in population order: bit-identical
    to rhs -= i_0; rhs -= i_1; ... on the host; nodes without an instance
    are left alone."""
    import ctypes as C

    from paper_1905_02241_b200 import runtime as rt

    rng = np.random.default_rng(7 + n_pops)
    n, n_nodes = 3001, 4000
    node_index = rng.permutation(n_nodes)[:n].astype(np.int32)  # one instance per node
    rhs0, d0 = rng.standard_normal(n_nodes), rng.standard_normal(n_nodes)
    cur_i = [rng.standard_normal(n) * 10.0 ** rng.integers(-6, 6) for _ in range(n_pops)]
    cur_g = [rng.random(n) * 10.0 ** rng.integers(-6, 6) for _ in range(n_pops)]
    s = rt.Stream()

    def up(a):
        a = np.ascontiguousarray(a)
        b = rt.DeviceBuffer(a.nbytes)
        rt.h2d(b.ptr, a.ctypes.data, a.nbytes, s)
        return b

    bufs = [up(rhs0), up(d0), up(node_index)] + [up(a) for a in cur_i] + [up(a) for a in cur_g]
    ip = (C.c_void_p * n_pops)(*[b.ptr for b in bufs[3:3 + n_pops]])
    gp = (C.c_void_p * n_pops)(*[b.ptr for b in bufs[3 + n_pops:]])
    L = rt.lib()
    rt.check(L.nmodl_combine_unique_ex(C.c_void_p(bufs[0].ptr), C.c_void_p(bufs[1].ptr), C.c_void_p(bufs[2].ptr), n,
                                       ip, gp, n_pops, flags, C.c_void_p(s.handle)), "combine_unique_ex")
    rhs, d = np.empty(n_nodes), np.empty(n_nodes)
    rt.d2h(rhs.ctypes.data, bufs[0].ptr, rhs.nbytes, s)
    rt.d2h(d.ctypes.data, bufs[1].ptr, d.nbytes, s)
    s.sync()
    er, ed = rhs0.copy(), d0.copy()
    for p in range(n_pops):
        er[node_index] = er[node_index] - cur_i[p]
        ed[node_index] = ed[node_index] + cur_g[p]
    assert np.array_equal(rhs, er) and np.array_equal(d, ed)
