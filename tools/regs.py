"""Registers / stack / local memory of the k_step kernels in built libraries:
python tools/regs.py lib1.so [lib2.so ...]"""
import re
import subprocess
import sys

for so in sys.argv[1:]:
    out = subprocess.run(["cuobjdump", "--dump-resource-usage", so], capture_output=True, text=True).stdout
    for m in re.finditer(r"Function (\S+):\s*\n\s*(REG:\d+ STACK:\d+ SHARED:\d+ LOCAL:\d+)", out):
        name = m.group(1)
        if "k_step" in name and "Lb0E" in name or ("k_step" in name and "ILb0E" in name):
            print(so.split("/")[-1], name[:60], m.group(2))
