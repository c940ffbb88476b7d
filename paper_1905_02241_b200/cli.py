"""Command line: `python -m paper_1905_02241_b200 {compile,verify,bench} FILE.mod`.

The reference CLI (modlc/cli.py) is left untouched -- its tests require
`--backend cuda` to stay rejected (pkg/tests/test_cli.py:26-29) -- so the CUDA
backend ships its own entry point with the same conventions: the front-end is
the reference's `compile_file` (modlc/pipeline.py:62-65), exit codes are
0 ok / 1 diagnostics / 2 verify failure (modlc/cli.py:21-23), and `verify`
differentially runs the reference runtime (`modlc.interp`) against the GPU on
identical seeded inputs (the shape of `cmd_verify`, modlc/cli.py:233-266).

A MechIR JSON file (fixtures/ir/*.json) may be given instead of a .mod file;
then no reference front-end is needed for `compile` and `bench`.
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

EXIT_OK, EXIT_DIAG, EXIT_VERIFY = 0, 1, 2
VERIFY_TOLERANCE = 1e-10  # GPU vs CPU: the north-star parity bound


def _load(path: str, passes=None):
    from .ir import MechIR

    p = Path(path)
    if p.suffix == ".json":
        return MechIR.load(p)
    from .frontend import compile_mod

    kwargs = {} if passes is None else {"passes": tuple(passes)}
    return compile_mod(p, **kwargs)


def cmd_compile(args) -> int:
    from .build import build_mechanism
    from .codegen_cuda import CudaOptions, UnsupportedConstruct, emit_cuda, emit_cuda_header

    ir = _load(args.file, args.passes)
    opts = CudaOptions(ilp=args.ilp, fast_path=not args.no_fast_path)
    try:
        unit = emit_cuda(ir, opts)
        header = emit_cuda_header(ir, opts)
    except UnsupportedConstruct as exc:
        print(f"{args.file}: error: {exc}", file=sys.stderr)
        return EXIT_DIAG
    out = Path(args.output or ".")
    out.mkdir(parents=True, exist_ok=True)
    (out / unit.filename).write_text(unit.text)
    (out / header.filename).write_text(header.text)
    print(f"wrote {out / unit.filename} and {out / header.filename}")
    if args.build:
        mb = build_mechanism(ir, opts)
        print(f"built {mb.so_path}")
    return EXIT_OK


def cmd_verify(args) -> int:
    """Reference runtime vs CUDA on `init(layout, n, seed)`, `steps` steps."""
    from .frontend import reference_layout
    from .runner import CudaRunner, simulate

    try:
        layout = reference_layout(args.file, **({} if args.passes is None else {"passes": tuple(args.passes)}))
    except ImportError as exc:
        print(f"verify needs the reference front-end/runtime: {exc}", file=sys.stderr)
        return EXIT_DIAG
    from modlc import interp

    ref = interp.init(layout, args.instances, args.seed)
    gpu = interp.init(layout, args.instances, args.seed)
    interp.simulate(layout, ref, args.steps)
    simulate(layout, gpu, args.steps, runner=CudaRunner(layout))
    from .metrics import parity

    worst_pure = interp.diff_trajectories(ref, gpu, [s.name for s in layout.slots] + ["v", "i_acc", "g_acc"])
    worst, where = parity(layout, ref, gpu)
    report = {"file": args.file, "instances": args.instances, "steps": args.steps,
              "deviation": worst, "worst_slot": where, "deviation_pure_relative": worst_pure,
              "metric": "diff_trajectories; jointly solved states normwise per instance; numeric-conductance "
                        "g_acc relative to |i|/h (paper_1905_02241_b200/metrics.py)",
              "tolerance": VERIFY_TOLERANCE, "ok": bool(worst <= VERIFY_TOLERANCE)}
    print(json.dumps(report))
    return EXIT_OK if report["ok"] else EXIT_VERIFY


def cmd_bench(args) -> int:
    from . import runtime as rt
    from .instance import init
    from .runner import CudaRunner
    from .traffic import launch_bytes

    ir = _load(args.file, args.passes)
    runner = CudaRunner(ir)
    dev = runner.to_device(init(ir, args.instances, args.seed))
    runner.run_kernel(dev, "initialize", 1)
    runner.launch(dev, "step", 5)
    a, b = rt.Event(), rt.Event()
    a.record(runner.stream)
    runner.launch(dev, "step", args.steps)
    b.record(runner.stream)
    b.sync()
    runner.check(dev)
    ms = a.elapsed_ms(b) / args.steps
    gbs = launch_bytes(runner.abi, args.instances, "step") / (ms / 1e3) / 1e9
    print(json.dumps({"mechanism": ir.mechanism, "instances": args.instances, "ms_per_step": ms,
                      "instance_steps_per_s": args.instances / (ms / 1e3), "GBps": gbs}))
    return EXIT_OK


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="paper_1905_02241_b200", description=__doc__.split("\n")[0])
    sub = ap.add_subparsers(dest="cmd", required=True)
    for name in ("compile", "verify", "bench"):
        p = sub.add_parser(name)
        p.add_argument("file", help="NMODL .mod (reference front-end) or MechIR .json")
        p.add_argument("--passes", nargs="*", default=None, help="reference DSL passes (default: all)")
        if name == "compile":
            p.add_argument("-o", "--output", default=None)
            p.add_argument("--build", action="store_true", help="also nvcc the .so (sm_100a)")
            p.add_argument("--ilp", type=int, default=1)
            p.add_argument("--no-fast-path", action="store_true")
        else:
            p.add_argument("--instances", type=int, default=256 if name == "verify" else 1_000_000)
            p.add_argument("--steps", type=int, default=100)
            p.add_argument("--seed", type=int, default=42)
    return ap


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return {"compile": cmd_compile, "verify": cmd_verify, "bench": cmd_bench}[args.cmd](args)
    except Exception as exc:  # diagnostics from the front-end (CompileError etc.)
        if type(exc).__name__ in ("CompileError", "SemanticError", "ParseError", "SolverError", "LexError"):
            print(f"{args.file}: error: {exc}", file=sys.stderr)
            return EXIT_DIAG
        raise


if __name__ == "__main__":
    raise SystemExit(main())
