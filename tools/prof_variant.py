"""Run a few launches of one mechanism variant (for ncu captures).

    python tools/prof_variant.py STEM N key=value ...   (CudaOptions fields)
"""

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_1905_02241_b200.codegen_cuda import CudaOptions  # noqa: E402
from paper_1905_02241_b200.instance import init  # noqa: E402
from paper_1905_02241_b200.ir import MechIR  # noqa: E402
from paper_1905_02241_b200.runner import CudaRunner  # noqa: E402


def main():
    stem, n = sys.argv[1], int(sys.argv[2])
    kw = {}
    for a in sys.argv[3:]:
        k, v = a.split("=")
        kw[k] = int(v) if v.isdigit() else (v == "True")
    ir = MechIR.load(ROOT / "fixtures" / "ir" / f"{stem}.json")
    r = CudaRunner(ir, options=CudaOptions(**kw))
    dev = r.to_device(init(ir, n, 42))
    r.run_kernel(dev, "initialize", 1)
    r.launch(dev, "step", 4)
    r.stream.sync()
    r.check(dev)


if __name__ == "__main__":
    main()
