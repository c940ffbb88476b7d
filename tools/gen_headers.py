"""Write include/mechanisms/<mech>.h for the benchmarked mechanisms.

    python tools/gen_headers.py
"""

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from bench import WORKLOADS  # noqa: E402
from paper_1905_02241_b200.codegen_cuda import emit_cuda_header  # noqa: E402
from paper_1905_02241_b200.ir import MechIR  # noqa: E402

stems = sorted({stem for w in WORKLOADS.values() for stem, _ in w["mechs"]} | {"corpus_cat"})
out = ROOT / "include" / "mechanisms"
out.mkdir(parents=True, exist_ok=True)
for stem in stems:
    unit = emit_cuda_header(MechIR.load(ROOT / "fixtures" / "ir" / f"{stem}.json"))
    (out / unit.filename).write_text(unit.text)
    print("wrote", unit.filename)
