"""Per-kernel operation census and roofline classification for B200.

Restates the reference's static analysis (modlc/analysis.py:77-147 `_Census`,
:158-265 `_Traffic`/`profile_kernel`) for the fused CUDA step and prices it
on B200: the census counts the per-instance operations of nrn_state +
nrn_cur as generated (numeric conductance doubles the current body,
modlc/analysis.py:243-250; solver nodes count one Newton iteration / one LU),
the traffic is the generated kernel's own load/store set (traffic.py), and
the FP64 cost uses the instruction counts of the sequences actually emitted
(SASS-derived: exp 16 FP64 ops, IEEE division 8 + MUFU, literal division 3).

`roofline(ir)` returns both times for one instance-step and which one binds:
    t_hbm  = bytes / HBM bandwidth        (MEASURED_PEAKS.json hbm_gbs)
    t_fp64 = FP64 ops / FP64 rate         (the measured DFMA rate of
             tools/micro/fp64_peak.cu, profiles/fp64_peak.json; nominal
             148 SM x 64 FP64 lanes x clock when that file is absent)
"""

from __future__ import annotations

import math
from collections import Counter

from .codegen_cuda import CudaPrinter
from .ir import from_layout, iter_nodes, newton_parts
from .traffic import bytes_per_instance

# FP64 pipe operations per emitted operation (from the sm_100a SASS of the
# generated code: tools/ncu_opcodes.py on profiles/r01/prof_r1f_*).
FP64_COST = {"exp": 16, "log": 22, "sqrt": 10, "pow": 60, "div": 8, "div_const": 3, "rcp": 6,
             "add": 1, "sub": 1, "mul": 1, "neg": 0, "cmp": 1, "fabs": 0, "ipow": 2}
FP64_LANES_PER_SM = 64
SM_COUNT = 148
_ROOT = __import__("pathlib").Path(__file__).resolve().parent.parent


def fp64_rate(clock_ghz: float = 1.965) -> float:
    """FP64 pipe instructions per second: measured (profiles/fp64_peak.json,
    1.705e13 DFMA/s on B200 = 58.7 per SM per clock), else nominal."""
    import json

    p = _ROOT / "profiles" / "fp64_peak.json"
    if p.is_file():
        return float(json.loads(p.read_text())["dfma_per_s"])
    return SM_COUNT * FP64_LANES_PER_SM * clock_ghz * 1e9


def _census_expr(node, out: Counter, fns) -> None:
    for n in iter_nodes(node):
        k = n.kind
        if k == "Binary":
            op = n.attrs["op"]
            if op == "/":
                lhs, rhs = n.children
                if rhs.kind == "Number":
                    out["div_const"] += 1
                elif lhs.kind == "Number" and lhs.attrs["value"] == 1.0:
                    out["rcp"] += 1
                else:
                    out["div"] += 1
            elif op == "^":
                r = n.children[1]
                if r.kind == "Number" and r.attrs["value"] in (2.0, 3.0, 4.0):
                    out["ipow"] += 1
                else:
                    out["pow"] += 1
            elif op in ("+",):
                out["add"] += 1
            elif op == "-":
                out["sub"] += 1
            elif op == "*":
                out["mul"] += 1
            elif op in ("<", "<=", ">", ">=", "==", "!="):
                out["cmp"] += 1
        elif k == "Unary" and n.attrs["op"] == "-":
            out["neg"] += 1
        elif k == "Call":
            name = n.attrs["name"]
            if name in ("exp", "log", "sqrt", "pow", "fabs"):
                out[name] += 1
            elif name in fns:
                for s in fns[name].children[-1].children:
                    _census_expr(s, out, fns)


def census(layout) -> Counter:
    """Operations per instance-step of the fused state + current kernel."""
    ir = from_layout(layout)
    out: Counter = Counter()
    for kname in ("state_update", "current_update"):
        mult = 2 if (kname == "current_update" and ir.currents and not ir.analytic_conductance) else 1
        c: Counter = Counter()
        for s in ir.kernels.get(kname, ()):
            if s.kind == "NewtonSolveNode":
                res, jac = newton_parts(s)
                for e in res + [x for row in jac for x in row]:
                    _census_expr(e, c, ir.functions)
                k = s.attrs["n"]
                c["div"] += k  # one LU / adjugate division per unknown
                c["mul"] += k ** 3 // 3
                c["sub"] += k ** 3 // 3
            elif s.kind == "LinearSolveNode":
                _census_expr(s, c, ir.functions)
                k = s.attrs["n"]
                c["div"] += k * (k + 1) // 2
                c["mul"] += k ** 3 // 3
                c["sub"] += k ** 3 // 3
            else:
                _census_expr(s, c, ir.functions)
        for key, v in c.items():
            out[key] += v * mult
    return out


def fp64_ops(layout) -> int:
    return sum(FP64_COST.get(k, 1) * v for k, v in census(layout).items())


def hbm_peak_gbs() -> float:
    """MEASURED_PEAKS.json hbm_gbs (driver-written copy bandwidth), else the
    value recorded on this pool's B200s."""
    import json

    p = _ROOT / "MEASURED_PEAKS.json"
    if p.is_file():
        return float(json.loads(p.read_text())["hbm_gbs"])
    return 6548.5


def roofline(layout, hbm_gbs: float | None = None, clock_ghz: float = 1.965, kernel: str = "step") -> dict:
    """Per instance-step: bytes, FP64 ops, time at the HBM and FP64 roofs."""
    ir = from_layout(layout)
    p = CudaPrinter(ir)
    p.emit_unit()
    b = bytes_per_instance(p._abi, kernel)
    f = fp64_ops(ir)
    hbm_gbs = hbm_peak_gbs() if hbm_gbs is None else hbm_gbs
    rate = fp64_rate(clock_ghz)
    t_hbm = b / (hbm_gbs * 1e9)
    t_fp = f / rate
    return {
        "mechanism": ir.mechanism,
        "bytes_per_instance": b,
        "fp64_ops_per_instance": f,
        "ops": dict(census(ir)),
        "t_hbm_ns": t_hbm * 1e9 * 1e3 / 1e3,
        "t_fp64_ns": t_fp * 1e9,
        "bound": "hbm" if t_hbm >= t_fp else "fp64",
        "fp64_per_byte": f / max(b, 1),
        "ridge_fp64_per_byte": rate / (hbm_gbs * 1e9),
        "max_hbm_fraction_at_fp64_roof": min(1.0, t_hbm / t_fp) if t_fp > 0 else 1.0,
    }


def table(stems_and_layouts) -> str:
    rows = ["| mechanism | B/inst-step | FP64 ops/inst-step | FP64 ops/B | bound | max HBM fraction |",
            "|---|---|---|---|---|---|"]
    for name, lay in stems_and_layouts:
        r = roofline(lay)
        rows.append(f"| {name} | {r['bytes_per_instance']} | {r['fp64_ops_per_instance']} | "
                    f"{r['fp64_per_byte']:.2f} | {r['bound']} | {min(1.0, r['max_hbm_fraction_at_fp64_roof']):.0%} |")
    return "\n".join(rows)


FP64_OPCODES = ("DFMA", "DMUL", "DADD", "DSETP", "DMNMX")


def measured(layout, ncu_summary: dict, n_instances: int, options=None) -> dict:
    """The census next to what one ncu capture of the same kernel measured
    (tools/ncu_summary.py output, e.g. profiles/r01j/r1j_hh.json): FP64
    thread-instructions and DRAM bytes per instance-step, the kernel time,
    and the fraction of the HBM / FP64 roofs the capture reached.
    `options`: the CudaOptions of the captured build (the traffic model
    reads the emitted kernel's load/store set)."""
    ir = from_layout(layout)
    p = CudaPrinter(ir, options)
    p.emit_unit()
    m = ncu_summary["metrics"]

    def num(prefix):
        key = next(k for k in m if k.startswith(prefix))
        return float(str(m[key]).replace(",", ""))

    us = num("gpu__time_duration")
    dram = (num("dram__bytes_read") + num("dram__bytes_write")) * 1e6  # ncu reports MB
    ops = ncu_summary.get("instructions", {}).get("by_opcode_per_instance", {})
    fp64_meas = sum(v for k, v in ops.items() if k in FP64_OPCODES)
    clock = num("sm__cycles_elapsed.avg.per_second") * 1e9
    fp64_rate = SM_COUNT * FP64_LANES_PER_SM * clock
    b = bytes_per_instance(p._abi, "step_nodes" if "step_nodes" in ncu_summary["kernel"] else "step")
    return {
        "mechanism": ir.mechanism,
        "census_fp64_ops": fp64_ops(ir),
        "measured_fp64_instr": fp64_meas,
        "algorithmic_bytes": b,
        "measured_dram_bytes": dram / n_instances,
        "kernel_us": us,
        "hbm_fraction_algorithmic": b * n_instances / (us * 1e-6) / (hbm_peak_gbs() * 1e9),
        "fp64_pipe_fraction": fp64_meas * n_instances / (us * 1e-6) / fp64_rate,
    }


if __name__ == "__main__":  # pragma: no cover
    import sys
    from pathlib import Path

    from .ir import MechIR

    root = Path(__file__).resolve().parent.parent / "fixtures" / "ir"
    if sys.argv[1:2] == ["--ncu"]:
        # --ncu REPORT.json:STEM:N ...  census vs one ncu capture per kernel
        import json

        sys.path.insert(0, str(root.parent.parent))
        from bench import options_for

        print("| mechanism | census FP64 ops | measured FP64 instr | algorithmic B | DRAM B (ncu) | µs | "
              "HBM (alg.) | FP64 pipe |")
        print("|---|---|---|---|---|---|---|---|")
        for spec in sys.argv[2:]:
            path, stem, n = spec.rsplit(":", 2)
            r = measured(MechIR.load(root / f"{stem}.json"), json.load(open(path))[0], int(n), options_for(stem))
            print(f"| {stem} | {r['census_fp64_ops']} | {r['measured_fp64_instr']:.0f} | {r['algorithmic_bytes']} | "
                  f"{r['measured_dram_bytes']:.0f} | {r['kernel_us']:.1f} | {r['hbm_fraction_algorithmic']:.0%} | "
                  f"{r['fp64_pipe_fraction']:.0%} |")
        sys.exit(0)
    stems = sys.argv[1:] or ["ProbAMPANMDA_EMS", "hh_subset", "NaTs2_t", "K_Pst", "Ca_HVA", "SKv3_1", "Ih",
                             "cadyn", "na6", "cdp5ish"]
    print(table([(s, MechIR.load(root / f"{s}.json")) for s in stems]))
    _ = math
