"""Stream-launched steps (the public run_kernel path) with and without
programmatic dependent launch, against the same steps replayed from a graph:
    python tools/stream_pdl.py          (GPU box)"""
import dataclasses
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from bench import options_for  # noqa: E402
from paper_1905_02241_b200 import runtime as rt  # noqa: E402
from paper_1905_02241_b200.instance import init, node_layout  # noqa: E402
from paper_1905_02241_b200.ir import MechIR  # noqa: E402
from paper_1905_02241_b200.runner import CudaRunner  # noqa: E402

K = 200
ir = MechIR.load(ROOT / "fixtures" / "ir" / "ProbAMPANMDA_EMS.json")
idx, nv = node_layout(10_000_000, 1_000_000, 42)
data = init(ir, 10_000_000, 42)
for pdl in (False, True):
    r = CudaRunner(ir, options=dataclasses.replace(options_for("ProbAMPANMDA_EMS"), pdl=pdl))
    dev = r.to_device(data, skip=("v",))
    r.bind_nodes(dev, idx, nv)
    r.gather_voltage(dev)
    r.run_kernel(dev, "initialize", 1)
    r.launch(dev, "step_nodes", 20)
    r.stream.sync()
    a, b = rt.Event(), rt.Event()
    a.record(r.stream)
    r.launch(dev, "step_nodes", K)
    b.record(r.stream)
    b.sync()
    stream_us = a.elapsed_ms(b) / K * 1e3
    g = rt.capture(r.stream, lambda: r.launch(dev, "step_nodes", K))
    g.upload(r.stream)
    a.record(r.stream)
    g.launch(r.stream)
    b.record(r.stream)
    b.sync()
    graph_us = a.elapsed_ms(b) / K * 1e3
    r.check(dev)
    print(json.dumps({"pdl": pdl, "stream_us_per_step": round(stream_us, 2), "graph_us_per_step": round(graph_us, 2)}),
          flush=True)
    del dev
