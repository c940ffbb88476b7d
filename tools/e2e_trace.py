"""Stage timings of one public-API node_index call (simulate_nodes).

    python tools/e2e_trace.py [n] [n_nodes] [steps]
"""

import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from bench import options_for  # noqa: E402
from paper_1905_02241_b200 import runtime as rt  # noqa: E402
from paper_1905_02241_b200.instance import init, node_layout  # noqa: E402
from paper_1905_02241_b200.ir import MechIR  # noqa: E402
from paper_1905_02241_b200.runner import CudaRunner, simulate_nodes  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
    n_nodes = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 1000
    ir = MechIR.load(ROOT / "fixtures" / "ir" / "ProbAMPANMDA_EMS.json")
    r = CudaRunner(ir, options=options_for("ProbAMPANMDA_EMS"))
    data = init(ir, n, 42)
    idx, nv = node_layout(n, n_nodes, 42)
    pins = [rt.PinnedRegistration(a) for a in list(data.arrays.values()) + list(data.acc.values()) + [idx, nv]]
    for rep in range(3):
        r.trace = []
        t0 = time.perf_counter()
        simulate_nodes(ir, data, steps, idx, nv, runner=r)
        total = time.perf_counter() - t0
        marks = r.trace
        prev = t0
        out = []
        for stage, t in marks:
            out.append(f"{stage}={1e3 * (t - prev):.1f}ms")
            prev = t
        print(f"rep {rep}: total {1e3 * total:.1f} ms | " + " ".join(out), flush=True)
    del pins


if __name__ == "__main__":
    main()
