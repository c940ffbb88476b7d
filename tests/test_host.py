"""CPU-side tests of the product: printer, IR, ABI, C-ABI exports, host logic.

No CUDA device needed: libraries are loaded with ctypes and only host-side
functions (ABI descriptors) are called.
"""

import ctypes
import json
import re
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT, all_ir_stems, load_ir
from paper_1905_02241_b200.codegen_cuda import (
    CudaOptions,
    CudaPrinter,
    UnsupportedConstruct,
    emit_cuda,
    emit_cuda_header,
)
from paper_1905_02241_b200.ir import MechIR, Node, Slot


def test_emission_deterministic_and_named():
    """Same contract as the reference emitters (pkg/tests/test_codegen.py:9-23)."""
    ir = load_ir("corpus_cat")
    a, b = emit_cuda(ir), emit_cuda(load_ir("corpus_cat"))
    assert a.text == b.text
    assert a.backend == "cuda" and a.filename == "cat.cu"
    assert "__global__" in a.text and "cat_k_step" in a.text
    assert 'extern "C"' in a.text


@pytest.mark.parametrize("stem", all_ir_stems())
def test_every_fixture_prints(stem):
    text = emit_cuda(load_ir(stem)).text
    assert text.endswith("\n")


def test_abi_field_order_mirrors_reference_struct():
    """count, scalars (sorted), v, i_acc, g_acc, slots in layout order
    (modlc/codegen.py:425-437), count renamed, extension fields appended."""
    ir = load_ir("hh_subset")
    p = CudaPrinter(ir)
    p.emit_unit()
    names = [f.name for f in p._abi.fields]
    assert names[0] == "n_instances"
    scal = [f.name for f in p._abi.fields if f.role == "scalar"]
    assert scal == sorted(ir.global_scalars)
    i_v = names.index("v")
    assert names[i_v : i_v + 3] == ["v", "i_acc", "g_acc"]
    slots = [f.key for f in p._abi.fields if f.role == "slot"]
    assert slots == ir.slot_names()
    assert "n" in slots  # STATE n no longer collides with the count field


def test_traffic_model_hh_is_144_bytes():
    """hh fused unique traffic = 10 reads + 8 writes = 144 B."""
    from paper_1905_02241_b200.traffic import bytes_per_instance

    p = CudaPrinter(load_ir("hh_subset"))
    p.emit_unit()
    k = p._abi.kernels["step"]
    assert sorted(k["loads"]) == sorted(["gnabar", "gkbar", "gl", "el", "m", "h", "n", "ena", "ek", "v"])
    assert sorted(k["stores"]) == sorted(["ina", "ik", "il", "m", "h", "n"])
    assert bytes_per_instance(p._abi, "step") == 144


def test_verbatim_in_kernel_is_rejected():
    ir = load_ir("corpus_leak")
    ir.kernels["state_update"] = (Node("Verbatim", (), {"text": "x = 1;"}),)
    with pytest.raises(UnsupportedConstruct):
        emit_cuda(ir)


def test_per_lane_global_write_is_rejected():
    """Last-active-lane GLOBAL writes (modlc/interp.py:361-367) are not lowered."""
    ir = load_ir("corpus_globals2")
    ident = lambda n: Node("Identifier", (), {"name": n})
    ir.kernels["state_update"] = ir.kernels["state_update"] + (Node("Assign", (ident("tadj"), ident("v"))),)
    with pytest.raises(UnsupportedConstruct):
        emit_cuda(ir)


def test_uniform_global_write_is_lowered():
    text = emit_cuda(load_ir("corpus_globals2")).text
    assert "scalars_rw" in text and "g_tadj" in text


def test_ir_json_round_trip():
    ir = load_ir("cdp5ish")
    again = MechIR.from_json(ir.to_json())
    assert again.to_json() == ir.to_json()
    assert emit_cuda(again).text == emit_cuda(ir).text


def test_ir_matches_reference_front_end_when_available():
    from paper_1905_02241_b200 import frontend

    if not frontend.modlc_available():
        pytest.skip("reference front-end not importable here")
    fresh = frontend.compile_mod(ROOT / "fixtures" / "mod" / "hh_subset.mod")
    fresh.meta = load_ir("hh_subset").meta
    assert fresh.to_obj()["kernels"] == load_ir("hh_subset").to_obj()["kernels"]


def test_headers_up_to_date():
    for h in sorted((ROOT / "include" / "mechanisms").glob("*.h")):
        mech = h.stem
        stem = next(s for s in all_ir_stems() if load_ir(s).mechanism == mech and "." not in s)
        assert emit_cuda_header(load_ir(stem)).text == h.read_text(), h.name


# ---- C-ABI exports ---------------------------------------------------------------


def _declared(header: Path):
    text = header.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    text = re.sub(r"#define NMODL_B200_MECHANISM.*?\n\n", "\n", text, flags=re.S)
    return sorted(set(re.findall(r"\b(nmodl_\w+)\s*\(", text)))


def test_runtime_library_exports_every_declared_symbol():
    from paper_1905_02241_b200.build import build_runtime
    from paper_1905_02241_b200.runtime import RUNTIME_SYMBOLS

    lib = ctypes.CDLL(str(build_runtime()))
    declared = _declared(ROOT / "include" / "nmodl_b200.h")
    assert declared, "no declarations parsed"
    for sym in declared:
        assert hasattr(lib, sym), sym
    assert set(RUNTIME_SYMBOLS) <= set(declared)
    lib.nmodl_abi_version.restype = ctypes.c_int
    assert lib.nmodl_abi_version() == 1
    lib.nmodl_status_size.restype = ctypes.c_int
    assert lib.nmodl_status_size() == 32


@pytest.mark.parametrize("stem", ["hh_subset", "ProbAMPANMDA_EMS", "na6", "cdp5ish", "corpus_cat"])
def test_mechanism_library_exports_and_abi(stem):
    from paper_1905_02241_b200.build import build_mechanism

    ir = load_ir(stem)
    mb = build_mechanism(ir)
    lib = ctypes.CDLL(str(mb.so_path))
    for k in ("initialize", "state_update", "current_update", "step", "step_nodes", "abi", "abi_size",
              "step_nodes_ctas"):
        assert hasattr(lib, f"{mb.symbol}_{k}")
    f = getattr(lib, f"{mb.symbol}_abi")
    f.restype = ctypes.c_char_p
    assert json.loads(f().decode()) == json.loads(mb.abi.to_json())
    size = getattr(lib, f"{mb.symbol}_abi_size")
    size.restype = ctypes.c_longlong
    fields = [(x.name, {"i64": ctypes.c_longlong, "f64": ctypes.c_double}.get(x.ctype, ctypes.c_void_p))
              for x in mb.abi.fields]
    assert size() == ctypes.sizeof(type("S", (ctypes.Structure,), {"_fields_": fields}))


def test_population_group_builds_and_mirrors_member_structs():
    """emit_group: one library whose args struct is the members' C-ABI
    stores back to back plus the chain CTA ranges (mirrored by
    runner.PopulationGroup); the member code is the standalone node
    kernel's, namespaced; members with Newton solves are rejected."""
    from paper_1905_02241_b200.build import build_group
    from paper_1905_02241_b200.codegen_cuda import UnsupportedConstruct, emit_group

    def struct_of(abi):
        fields = [(x.name, {"i64": ctypes.c_longlong, "f64": ctypes.c_double}.get(x.ctype, ctypes.c_void_p))
                  for x in abi.fields]
        return type("S", (ctypes.Structure,), {"_fields_": fields})

    chains = [[(load_ir("NaTs2_t"), None)], [(load_ir("Ca_HVA"), None), (load_ir("cadyn"), None)]]
    gb = build_group("t_grp", chains)
    assert gb.text == emit_group("t_grp", chains)[0].text  # deterministic
    assert "t_grp_m1_1::CaDynamics_E2_k_step_nodes_unique" in gb.text
    lib = ctypes.CDLL(str(gb.so_path))
    assert hasattr(lib, "t_grp_step_unique")
    size = lib.t_grp_args_size
    size.restype = ctypes.c_longlong
    fields = [(f"md{ci}_{mi}", struct_of(a)) for ci, row in enumerate(gb.abis) for mi, a in enumerate(row)]
    fields.append(("cta", ctypes.c_longlong * 3))
    assert size() == ctypes.sizeof(type("A", (ctypes.Structure,), {"_fields_": fields}))
    with pytest.raises(UnsupportedConstruct):
        emit_group("bad", [[(load_ir("cdp5ish"), None)]])


def test_runner_fails_loudly_without_device():
    from paper_1905_02241_b200 import runtime as rt

    if rt.device_count() > 0:
        pytest.skip("a device is visible")
    from paper_1905_02241_b200.runner import CudaRunner

    with pytest.raises(rt.CudaError, match="no CPU fallback"):
        CudaRunner(load_ir("corpus_cat"))


# ---- host logic --------------------------------------------------------------------


def test_tile_nodes_cover_all_nodes():
    from paper_1905_02241_b200.runner import tile_nodes_for

    rng = np.random.default_rng(0)
    for n, n_nodes, t in [(10000, 1000, 512), (100, 3, 16), (5000, 5000, 1536), (7, 1, 2)]:
        idx = rng.integers(0, n_nodes, n)
        offsets = np.concatenate([[0], np.cumsum(np.bincount(idx, minlength=n_nodes))])
        tiles = tile_nodes_for(offsets, t)
        assert tiles[0] == 0 and tiles[-1] == n_nodes
        assert np.all(np.diff(tiles) > 0)
        sizes = offsets[tiles[1:]] - offsets[tiles[:-1]]
        assert sizes.sum() == n
        maxseg = np.max(np.diff(offsets))
        assert np.all(sizes <= t + maxseg)


def test_product_init_matches_oracle_init():
    """Synthetic inputs are the reference's init format (interp.py:61-84)."""
    from oracle import interp_np as O
    from paper_1905_02241_b200.instance import init

    for stem in ("hh_subset", "ProbAMPANMDA_EMS", "cdp5ish"):
        ir = load_ir(stem)
        a, b = init(ir, 100, 42), O.init(ir, 100, 42)
        assert list(a.arrays) == list(b.arrays)
        for k in a.arrays:
            np.testing.assert_array_equal(a.arrays[k], b.arrays[k])
        assert a.scalars == b.scalars


def test_node_oracle_layout_is_stable_sort():
    from oracle.nodes_np import scatter_layout

    idx = np.array([3, 1, 3, 0, 1, 3], dtype=np.int32)
    perm, offsets, rank = scatter_layout(idx, 5)
    assert perm.tolist() == [3, 1, 4, 0, 2, 5]
    assert offsets.tolist() == [0, 1, 3, 3, 6, 6]
    assert np.all(perm[rank] == np.arange(6))


def test_constant_division_is_correctly_rounded():
    """nmodl::div_c's Markstein sequence equals IEEE a/c (checked with exact
    rational arithmetic, including near-power-of-two adversarial numerators),
    for the divisor literals that appear in the fixtures."""
    import math
    import random
    from fractions import Fraction as Fr

    from paper_1905_02241_b200.ir import iter_nodes

    rn = lambda x: float(x)
    fma = lambda a, b, c: rn(Fr(a) * Fr(b) + Fr(c))
    consts = set()
    for stem in all_ir_stems():
        ir = load_ir(stem)
        for stmts in list(ir.kernels.values()) + [(f,) for f in ir.functions.values()]:
            for s in stmts:
                for n in iter_nodes(s):
                    if n.kind == "Binary" and n.attrs["op"] == "/" and n.children[1].kind == "Number":
                        c = n.children[1].attrs["value"]
                        if c != 0 and abs(math.frexp(c)[0]) != 0.5:
                            consts.add(c)
    assert consts
    rng = random.Random(3)
    for c in sorted(consts):
        y = rn(Fr(1) / Fr(c))
        for _ in range(300):
            e = rng.randint(-900, 900)
            a = math.ldexp(rng.random() + 1.0, e) * rng.choice((1, -1))
            if rng.random() < 0.3:
                a = math.nextafter(math.ldexp(1.0, e), math.inf if rng.random() < 0.5 else 0.0)
            q = rn(Fr(a) * Fr(y))
            q1 = fma(fma(-c, q, a), y, q)
            assert q1 == rn(Fr(a) / Fr(c)), (c, a)


def test_cli_compile_from_ir_and_mod(tmp_path):
    from paper_1905_02241_b200 import frontend
    from paper_1905_02241_b200.cli import main

    assert main(["compile", str(ROOT / "fixtures" / "ir" / "na6.json"), "-o", str(tmp_path)]) == 0
    assert (tmp_path / "na6.cu").is_file() and (tmp_path / "na6.h").is_file()
    if frontend.modlc_available():
        assert main(["compile", str(ROOT / "fixtures" / "mod" / "hh_subset.mod"), "-o", str(tmp_path)]) == 0
        assert (tmp_path / "hh.cu").read_text() == emit_cuda(load_ir("hh_subset")).text


def test_cli_rejects_unsupported(tmp_path):
    from paper_1905_02241_b200.cli import main

    ir = load_ir("corpus_leak")
    ir.kernels["state_update"] = (Node("Verbatim", (), {"text": "x = 1;"}),)
    p = tmp_path / "bad.json"
    p.write_text(ir.to_json())
    assert main(["compile", str(p), "-o", str(tmp_path)]) == 1


def test_census_counts_match_the_mechanism():
    """hh: 9 exp per instance-step (6 rates + 3 cnexp), x^3/x^4 as products,
    numeric-conductance bodies counted twice (modlc/analysis.py:243-250)."""
    from paper_1905_02241_b200.analysis import census, roofline

    c = census(load_ir("hh_subset"))
    assert c["exp"] == 9 and c["pow"] == 1 and c["ipow"] == 2  # q10 stays a (hoisted) pow
    syn = census(load_ir("ProbAMPANMDA_EMS"))
    assert syn["exp"] == 4 + 2  # 4 cnexp decays + Mg block at v and v+h
    r = roofline(load_ir("ProbAMPANMDA_EMS"))
    assert r["bound"] == "hbm" and r["bytes_per_instance"] == 152


OPTION_SETS = [
    ("hh_subset", dict(pipe=True, recip=True, div_approx=True, fast_redo=True, fast_path=True)),
    ("hh_subset", dict(exp_share=True, recip=True, fast_path=True)),
    ("NaTs2_t", dict(exp_share=True, fast_path=False)),
    ("NaTs2_t", dict(ilp=2, pipe=True, recip=True, div_approx=True, fast_redo=True, fast_path=True, min_blocks=2)),
    ("K_Pst", dict(ilp=2, recip=True, quot=True, exp_smem=True, pipe=True, fast_path=True, fast_redo=True)),
    ("na6", dict(lu_spec=True, pipe=True, fast_path=True, fast_redo=True)),
    ("cdp5ish", dict(lu_spec=True, div_approx=True, fast_path=True)),
    ("ProbAMPANMDA_EMS", dict(ilp=2, fast_path=False)),
    ("ProbAMPANMDA_EMS", dict(pipe=True, fast_path=True, fast_redo=True, grid_waves=0)),
]


@pytest.mark.parametrize("stem,kw", OPTION_SETS)
def test_option_builds_are_deterministic_and_keep_the_abi(stem, kw):
    """Every code-generation option is a pure function of (layout, options),
    and none of them changes the C ABI (struct layout, entry points)."""
    from paper_1905_02241_b200.codegen_cuda import cuda_abi

    ir = load_ir(stem)
    a, abi_a = cuda_abi(ir, CudaOptions(**kw))
    b, _ = cuda_abi(load_ir(stem), CudaOptions(**kw))
    assert a.text == b.text
    _, abi0 = cuda_abi(ir, CudaOptions())
    assert abi_a.to_json() == abi0.to_json()
    assert emit_cuda_header(ir, CudaOptions(**kw)).text == emit_cuda_header(ir).text


def test_reciprocal_shadows_remove_the_tau_divisions():
    """recip: hh's three `dt/tau` with tau = 1/(q10*sum) become products and
    the 1/(q10*sum) quotients are never formed; quot: K_Pst's
    `dt/((...)/qt)` become one division each."""
    base = emit_cuda(load_ir("hh_subset"), CudaOptions(fast_path=True)).text
    rec = emit_cuda(load_ir("hh_subset"), CudaOptions(fast_path=True, recip=True)).text
    assert rec.count("NM_DIV(") < base.count("NM_DIV(")
    assert "md.dt) * l_mtau_rd" in rec and "l_mtau = NM_DIV" not in rec.split("hh_body_state_update")[1].split("hh_body_current_update")[0]
    kp = emit_cuda(load_ir("K_Pst"), CudaOptions(recip=True, quot=True)).text
    assert "l_mTau_rn = nm_n" in kp and "NM_DIV((double)(md.dt) * l_mTau_rd, l_mTau_rn)" in kp


def test_speculative_lu_keeps_a_pivoted_fallback():
    """lu_spec emits the swap-free elimination guarded by the first-max test
    and the full pivoted LU behind `!ok` (na6: runtime LU, k=6)."""
    text = emit_cuda(load_ir("na6"), CudaOptions(lu_spec=True)).text
    assert "bool ok_" in text and "a row swap is due" in text
    assert "const bool sw = (piv ==" in text  # the pivoted path is still there
    plain = emit_cuda(load_ir("na6"), CudaOptions()).text
    assert "bool ok_" not in plain


def test_solver_cores_keep_ieee_division_under_div_approx():
    """div_approx relaxes rate-code division only: LU pivots / back
    substitution and Newton updates use NM_DIVX (always the IEEE quotient)."""
    text = emit_cuda(load_ir("cdp5ish"), CudaOptions(div_approx=True, fast_path=True)).text
    assert "#define NM_DIVX(a, b) (FAST ? nmodl::div_f((a), (b), dfl) : ((a) / (b)))" in text
    assert "nmodl::div_af" in text
    assert "= NM_DIVX(" in text


@pytest.mark.parametrize("stem,kw", [OPTION_SETS[0], OPTION_SETS[2], OPTION_SETS[3], OPTION_SETS[5]])
def test_option_builds_compile_for_sm100a(stem, kw, tmp_path):
    """nvcc cross-compiles the emitted TU for sm_100a (no GPU needed)."""
    import subprocess

    from paper_1905_02241_b200.build import ARCH, INCLUDE, nvcc_path

    src = tmp_path / "m.cu"
    src.write_text(emit_cuda(load_ir(stem), CudaOptions(**kw)).text)
    proc = subprocess.run([nvcc_path(), ARCH, "-O3", "-std=c++17", "-cubin", f"-I{INCLUDE}", "-diag-suppress", "177,550",
                           str(src), "-o", str(tmp_path / "m.cubin")], capture_output=True, text=True)
    assert proc.returncode == 0, proc.stderr[-2000:]


def test_exp_sharing_reuses_affine_exponentials():
    """exp_share: hh's three exp(-(v+c)/10) (two vtrap, one beta_h) become
    one exp and two constant multiples; NaTs2_t's exp(-(u+32)/6) /
    exp((u+32)/6) pairs become one exp and one quotient each."""
    hh = emit_cuda(load_ir("hh_subset"), CudaOptions(exp_share=True))
    body = hh.text.split("hh_body_state_update")[1].split("hh_body_current_update")[0]
    assert body.count("NM_EXP(") == 7  # 9 exps, two of the three /10 ones now constant multiples
    assert len(re.findall(r"t_xs\d+ \* hh_K\[\d+\]", body)) == 2
    nat = emit_cuda(load_ir("NaTs2_t"), CudaOptions(exp_share=True)).text
    body = nat.split("NaTs2_t_body_state_update")[1].split("NaTs2_t_body_current_update")[0]
    assert body.count("NM_EXP(") == 4 and len(re.findall(r"NM_DIV\(1\.0, t_xs\d+\)", body)) == 2


def test_census_next_to_measured_ncu_counters():
    """analysis.measured: the reference-style census beside one committed ncu
    capture (profiles/r01j): kernel time, DRAM bytes and FP64 instructions
    per instance, roof fractions in (0, 1]."""
    import json

    from bench import options_for
    from paper_1905_02241_b200.analysis import measured

    summ = json.loads((ROOT / "profiles" / "r01j" / "r1j_hh.json").read_text())[0]
    r = measured(load_ir("hh_subset"), summ, 1_000_000, options_for("hh_subset"))
    assert r["algorithmic_bytes"] == 144
    assert 0 < r["hbm_fraction_algorithmic"] <= 1 and 0 < r["fp64_pipe_fraction"] <= 1
    assert r["measured_fp64_instr"] < r["census_fp64_ops"]  # relaxed build: fewer than the census prices
    assert 80 < r["measured_dram_bytes"] < 150


def test_codegen_hazards_rwglobal():
    """Text-level guards for two code-generation hazards (fixtures/mod/rwglobal.mod):
    kernel-written GLOBALs are read from one buffer and written to the other
    (no in-launch read-after-write between instance 0 and later blocks), the
    v+h pass's GLOBAL write is carried into the base pass, and an exp of a
    slot is recomputed after the slot is reassigned (exp_share)."""
    import re

    from paper_1905_02241_b200.codegen_cuda import CudaOptions, emit_cuda

    ir = load_ir("rwglobal")
    text = emit_cuda(ir, CudaOptions(exp_share=True, fast_redo=True, pipe=True)).text
    assert "md.scalars_rw_out[0] = " in text
    assert not re.search(r"md\.scalars_rw\[\d+\] =", text)
    assert "local.scalars_rw_out = md->scalars_rw + ((step + 1) & 1) * 1;" in text
    assert "I.g_cnt = S.g_cnt;" in text
    body = text[text.index("rwglobal_body_state_update"):text.index("rwglobal_body_current_update")]
    first, second = body.index("I.s = I.v;"), body.rindex("NM_EXP")
    exps_of_s = re.findall(r"const double (t_xs\d+) = NM_EXP\(\(double\)\(\(rwglobal_K\[\d+\] \* I\.s\)\)\);", body)
    assert len(exps_of_s) == 2 and first < second


def test_prune_stale_keeps_what_a_build_touched(tmp_path, monkeypatch):
    """build.prune_stale: a cached library reused (touched) since the stamp
    stays with its source and log; one nobody built or reused goes."""
    import os
    import time

    from paper_1905_02241_b200 import build as B

    mech = tmp_path / "mech"
    mech.mkdir()
    monkeypatch.setattr(B, "BUILD", tmp_path)
    old = time.time() - 100
    for stem in ("hh-aaaa", "hh-bbbb", "group_soma-cccc"):
        for name in (f"lib{stem}.so", f"{stem}.cu", f"{stem}.log"):
            (mech / name).write_text("x")
            os.utime(mech / name, (old, old))
    stamp = time.time()
    B._touch(mech / "libhh-aaaa.so")
    B._touch(mech / "libgroup_soma-cccc.so")
    assert B.prune_stale(stamp) == 3
    assert sorted(p.name for p in mech.iterdir()) == sorted(
        ["libhh-aaaa.so", "hh-aaaa.cu", "hh-aaaa.log", "libgroup_soma-cccc.so", "group_soma-cccc.cu",
         "group_soma-cccc.log"])


def test_direct_population_group_text():
    """emit_group(kind="direct"): every member's fused step code as a device
    function, called in member order by every CTA with a barrier between
    members (their cp.async pipelines share the dynamic shared memory), a
    resident-CTA query; chained members must share ilp."""
    import dataclasses

    from paper_1905_02241_b200.codegen_cuda import CudaOptions, emit_group

    ca = CudaOptions(ilp=2, pipe=True)
    unit, _ = emit_group("d_grp", [[(load_ir("NaTs2_t"), CudaOptions(ilp=2, pipe=True))],
                                   [(load_ir("Ca_HVA"), ca), (load_ir("cadyn"), dataclasses.replace(ca))]],
                         kind="direct")
    t = unit.text
    k = t.index("d_grp_k_step_group(const d_grp_args a)")
    body = t[k:t.index("\n}\n", k)]
    calls = [ln.strip() for ln in body.splitlines() if "_k_step_dev<JAC_FD>" in ln]
    assert [c.split("::")[1].split("_k_step_dev")[0] for c in calls] == ["NaTs2_t", "Ca_HVA", "CaDynamics_E2"]
    assert body.count("__syncthreads();") == 2
    assert "int d_grp_group_ctas(void)" in t and "int d_grp_step_group(" in t
    with pytest.raises(ValueError):
        emit_group("bad", [[(load_ir("Ca_HVA"), CudaOptions(ilp=2)), (load_ir("cadyn"), CudaOptions(ilp=1))]],
                   kind="direct")


def test_lu_approx_modes_touch_only_the_solver_quotients():
    """CudaOptions.lu_approx: 0 leaves the emitted text of every solver as
    before (no NM_DIVM; build keys and ncu records stay valid); 2 routes only
    the LU multipliers through NM_DIVM (relaxed in the fast pass, IEEE in the
    exact redo) and keeps the back-substitution on NM_DIVX; 1 relaxes
    NM_DIVX itself in the fast pass."""
    from paper_1905_02241_b200.codegen_cuda import CudaOptions, emit_cuda

    ir = load_ir("na6")
    text = {m: emit_cuda(ir, CudaOptions(fast_path=True, lu_approx=m)).text for m in (0, 1, 2)}
    assert "NM_DIVM" not in text[0] and "NM_DIVM" not in text[1]
    mult = re.findall(r"const double f = (NM_DIV\w)\(", text[2])
    assert mult and set(mult) == {"NM_DIVM"}
    assert re.search(r"= NM_DIVX\(", text[2])  # back-substitution keeps the IEEE-capable macro
    assert "#define NM_DIVM(a, b) (FAST ? nmodl::div_af" in text[2]
    assert "#define NM_DIVX(a, b) (FAST ? nmodl::div_f(" in text[2]
    assert "#define NM_DIVX(a, b) (FAST ? nmodl::div_af" in text[1]
    assert text[0] == emit_cuda(ir, CudaOptions(fast_path=True)).text
