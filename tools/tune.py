"""Kernel tuning sweep (GPU): launch-shape options per mechanism.

    python tools/tune.py [stem ...]

Prints one JSON line per (mechanism, options): launch time from CUDA events
(L2 flushed between launches when the working set is L2-sized), achieved
algorithmic GB/s and instance-steps/s.  Used to pick bench.py's options.
"""

import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_1905_02241_b200 import runtime as rt  # noqa: E402
from paper_1905_02241_b200.codegen_cuda import CudaOptions  # noqa: E402
from paper_1905_02241_b200.instance import init, node_layout  # noqa: E402
from paper_1905_02241_b200.ir import MechIR  # noqa: E402
from paper_1905_02241_b200.runner import CudaRunner  # noqa: E402
from paper_1905_02241_b200.traffic import launch_bytes  # noqa: E402

SIZES = {"hh_subset": 1_000_000, "ProbAMPANMDA_EMS": 10_000_000, "na6": 1_000_000, "cdp5ish": 1_000_000, "cadyn": 3_333_333, "SKv3_1": 3_333_333, "Ih": 3_333_333,
         "NaTs2_t": 3_333_333, "K_Pst": 3_333_333, "Ca_HVA": 3_333_333}
SHAPES = [dict(ilp=1), dict(ilp=2), dict(ilp=1, min_blocks=4), dict(ilp=1, min_blocks=3), dict(ilp=2, min_blocks=3)]
CODEGEN = [dict(fast_path=False), dict()]
VARIANTS = [CudaOptions(**a, **b) for b in CODEGEN for a in SHAPES]


def run(stem, opts, nodes=0, steps=30):
    ir = MechIR.load(ROOT / "fixtures" / "ir" / f"{stem}.json")
    n = int(os.environ.get("TUNE_N", SIZES.get(stem, 1_000_000)))
    r = CudaRunner(ir, options=opts)
    dev = r.to_device(init(ir, n, 42))
    kernel = "step"
    if nodes:
        idx, nv = node_layout(n, nodes, 42)
        r.bind_nodes(dev, idx, nv)
        kernel = "step_nodes"
    r.run_kernel(dev, "initialize", 1)
    info = rt.device_info(0)
    lb = launch_bytes(r.abi, n, kernel, dev.nodes.n_segs if dev.nodes is not None else 0)
    # bench.py's timing: one graph of `steps` launches, external events around
    # each launch, the clean L2 flush between them for L2-sized stores
    from bench import L2Flush

    flush = L2Flush(info["l2_bytes"]) if lb < 3 * info["l2_bytes"] else None
    for _ in range(int(os.environ.get("TUNE_WARMUP", "10"))):
        r.launch(dev, kernel, 1)
    r.stream.sync()
    evs = [(rt.Event(), rt.Event()) for _ in range(steps)]

    def body():
        for a, b in evs:
            if flush is not None:
                flush(r.stream)
            a.record_external(r.stream)
            r.launch(dev, kernel, 1)
            b.record_external(r.stream)

    g = rt.capture(r.stream, body)
    g.upload(r.stream)
    g.launch(r.stream)
    r.stream.sync()
    total = sum(a.elapsed_ms(b) for a, b in evs)
    r.check(dev)
    ms = total / steps
    return {"stem": stem, "opts": opts.__dict__ if hasattr(opts, "__dict__") else str(opts), "kernel": kernel, "n": n,
            "ms": ms, "GBps": lb / (ms / 1e3) / 1e9, "inst_steps_per_s": n / (ms / 1e3), "flush": bool(flush)}


BOOL_OPTS = tuple(f.name for f in __import__("dataclasses").fields(CudaOptions) if f.type in (bool, "bool"))


def grid(spec: str):
    """'ilp=1,2 fast_path=0,1' -> the CudaOptions cross product."""
    import itertools

    keys, values = [], []
    for part in spec.split():
        k, vs = part.split("=")
        keys.append(k)
        values.append([bool(int(v)) if k in BOOL_OPTS else int(v)
                       for v in vs.split(",")])
    return [CudaOptions(**dict(zip(keys, combo))) for combo in itertools.product(*values)]


def main():
    global VARIANTS
    args = sys.argv[1:]
    if args and args[0] == "--grid":
        VARIANTS = grid(args[1])
        args = args[2:]
    if args and args[0] == "--around":
        # bench.options_for(stem) with the listed fields varied: --around "exp_smem=0,1 fast_path=0,1" stems...
        import dataclasses

        sys.path.insert(0, str(ROOT))
        from bench import options_for

        spec, stems_ = args[1], args[2:]
        deltas = grid(spec)
        keys = [p.split("=")[0] for p in spec.split()]
        for stem in stems_:
            for d in deltas:
                opts = dataclasses.replace(options_for(stem), **{k: getattr(d, k) for k in keys})
                nodes = int(os.environ.get("TUNE_NODES", 1_000_000)) if stem == "ProbAMPANMDA_EMS" else 0
                try:
                    res = run(stem, opts, nodes)
                except Exception as exc:  # noqa: BLE001
                    res = {"stem": stem, "opts": str(opts), "error": repr(exc)[:300]}
                print(json.dumps(res), flush=True)
        return
    if args and args[0] == "--synapse":
        VARIANTS = [CudaOptions(fast_path=False, tile=t, block=b, min_blocks=m)
                    for t in (1024, 2048, 4096) for b in (256, 512) for m in (0, 2, 3, 5) if not (b == 512 and m > 2)]
        args = ["ProbAMPANMDA_EMS"]
    if args and args[0] == "--hh":
        VARIANTS = [CudaOptions(ilp=i, fast_path=f, min_blocks=m) for f in (False, True) for i in (1, 2) for m in (0, 3, 4)]
        args = ["hh_subset"]
    if args and args[0] == "--kinetic":
        VARIANTS = [CudaOptions(ilp=1, fast_path=f, min_blocks=m) for f in (False, True) for m in (0, 2, 3)]
        args = ["na6", "cdp5ish"]
    if args and args[0] == "--quick":
        VARIANTS = [CudaOptions(ilp=i, fast_path=f) for f in (False, True) for i in (1, 2)]
        args = args[1:]
    stems = args or ["hh_subset", "NaTs2_t", "na6", "cdp5ish", "ProbAMPANMDA_EMS"]
    rt.require_device(0)
    for stem in stems:
        for opts in VARIANTS:
            nodes = int(os.environ.get("TUNE_NODES", 1_000_000)) if stem == "ProbAMPANMDA_EMS" else 0
            try:
                res = run(stem, opts, nodes)
            except Exception as exc:  # noqa: BLE001
                res = {"stem": stem, "opts": str(opts), "error": repr(exc)[:300]}
            print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
