"""Per-opcode dynamic instruction counts and stall samples from an ncu report.

    python tools/ncu_opcodes.py gpurun_out/prof.ncu-rep [instances]

Reads the SASS source page (`ncu -i ... --page source --csv --print-source
sass`), sums "Instructions Executed" (warp-level) per opcode and prints them
per instance when the instance count is given.
"""

import collections
import csv
import io
import subprocess
import sys


def opcode_table(report: str):
    out = subprocess.run(["ncu", "-i", report, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True, check=True).stdout
    tables = []
    cur = None
    for line in out.splitlines():
        if line.startswith('"Kernel Name"'):
            cur = {"kernel": next(csv.reader([line]))[1], "lines": []}
            tables.append(cur)
        elif cur is not None:
            cur["lines"].append(line)
    result = []
    for t in tables:
        rows = list(csv.reader(io.StringIO("\n".join(t["lines"]))))
        hdr = rows[0]
        ie, src = hdr.index("Instructions Executed"), hdr.index("Source")
        st = hdr.index("Warp Stall Sampling (All Samples)")
        cnt, stall = collections.Counter(), collections.Counter()
        for r in rows[1:]:
            if len(r) <= ie or not r[ie].strip().isdigit():
                continue
            toks = r[src].split()
            if not toks:
                continue
            op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
            op = op.split(".")[0]
            cnt[op] += int(r[ie])
            stall[op] += int(r[st]) if r[st].strip().isdigit() else 0
        result.append((t["kernel"], cnt, stall))
    return result


def main():
    report = sys.argv[1]
    n = float(sys.argv[2]) if len(sys.argv) > 2 else None
    for kernel, cnt, stall in opcode_table(report):
        tot = sum(cnt.values())
        print(f"== {kernel}: {tot} warp instructions" + (f" = {tot * 32 / n:.1f} thread-instr per instance" if n else ""))
        for op, c in cnt.most_common(25):
            per = f"{c * 32 / n:8.1f}/inst" if n else ""
            print(f"  {op:8s} {c:11d} {per}  stall_samples={stall[op]}")


if __name__ == "__main__":
    main()
