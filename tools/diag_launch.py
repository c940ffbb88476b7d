"""Diagnostic: per-step time of 1000 stream launches (launch_steps loop) vs
the same 1000 launches replayed from a CUDA graph (synapse10m)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from bench import Population, options_for  # noqa: E402
from paper_1905_02241_b200 import runtime as rt  # noqa: E402

p = Population("ProbAMPANMDA_EMS", 10_000_000, 1_000_000, 42, options_for("ProbAMPANMDA_EMS"))
p.setup_device()
s = p.runner.stream
a, b = rt.Event(), rt.Event()
for _ in range(20):
    p.launch(1)
s.sync()
for rep in range(2):
    a.record(s)
    p.launch(1000)
    b.record(s)
    b.sync()
    print("stream loop 1000:", round(a.elapsed_ms(b) / 1000, 4), "ms/step")
g = rt.capture(s, lambda: p.launch(1000))
for rep in range(2):
    a.record(s)
    g.launch(s)
    b.record(s)
    b.sync()
    print("graph 1000:", round(a.elapsed_ms(b) / 1000, 4), "ms/step")
g2 = rt.capture(s, lambda: [p.launch(1) for _ in range(200)])
a.record(s)
g2.launch(s)
b.record(s)
b.sync()
print("graph 200 x launch(1):", round(a.elapsed_ms(b) / 200, 4), "ms/step")
