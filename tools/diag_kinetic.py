"""Diagnostic: cdp5ish launch time alone vs after na6 (bench kinetic1m order)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import ctypes as C  # noqa: E402

from bench import Population, options_for  # noqa: E402
from paper_1905_02241_b200 import runtime as rt  # noqa: E402

pops = [Population(s, 1_000_000, 0, 42, options_for(s)) for s in ("na6", "cdp5ish")]
for p in pops:
    p.setup_device()
s0 = pops[0].runner.stream
for p in pops:
    p.runner.stream = s0
info = rt.device_info(0)
fb = rt.DeviceBuffer(2 * info["l2_bytes"])
for _ in range(20):
    for p in pops:
        p.launch(1)
s0.sync()


def timed(seq, reps=30):
    evs = [(rt.Event(), rt.Event()) for _ in seq]
    tot = [0.0] * len(seq)
    for _ in range(reps):
        rt.check(rt.lib().nmodl_spin(2_000_000, C.c_void_p(s0.handle)), "spin")
        rt.check(rt.lib().nmodl_l2_flush(C.c_void_p(fb.ptr), fb.nbytes // 8, C.c_void_p(s0.handle)), "f")
        for j, p in enumerate(seq):
            evs[j][0].record(s0)
            p.launch(1)
            evs[j][1].record(s0)
        s0.sync()
        for j in range(len(seq)):
            tot[j] += evs[j][0].elapsed_ms(evs[j][1])
    return [round(t / reps, 4) for t in tot]


print("na6, cdp5:", timed(pops))
print("cdp5 alone:", timed([pops[1]]))
print("cdp5, na6:", timed(pops[::-1]))
print("na6 alone:", timed([pops[0]]))
print("cdp5 x3:", timed([pops[1]] * 3))

from bench import ClockSampler  # noqa: E402

with ClockSampler(0) as clk:
    print("with NVML sampler, na6, cdp5:", timed(pops))
print(clk.summary())
with ClockSampler(0, period_s=0.02) as clk:
    print("with NVML sampler @20ms, na6, cdp5:", timed(pops))
