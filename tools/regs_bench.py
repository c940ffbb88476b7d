"""Registers / stack of the k_step kernels of bench.py's builds (or of the
stems given): python tools/regs_bench.py [stem ...]"""
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from bench import options_for  # noqa: E402
from paper_1905_02241_b200.build import build_mechanism  # noqa: E402
from paper_1905_02241_b200.ir import MechIR  # noqa: E402

stems = sys.argv[1:] or ["ProbAMPANMDA_EMS", "hh_subset", "NaTs2_t", "K_Pst", "Ca_HVA", "SKv3_1", "Ih", "cadyn",
                         "na6", "cdp5ish"]
for stem in stems:
    mb = build_mechanism(MechIR.load(ROOT / "fixtures" / "ir" / f"{stem}.json"), options_for(stem))
    out = subprocess.run(["cuobjdump", "--dump-resource-usage", str(mb.so_path)], capture_output=True, text=True).stdout
    for m in re.finditer(r"Function (\S+):\s*\n\s*(REG:\d+ STACK:\d+ SHARED:\d+ LOCAL:\d+)", out):
        if "k_step" in m.group(1) and "ILb0E" in m.group(1):
            print(f"{stem:18s} {m.group(1)[:44]:44s} {m.group(2)}")
