"""Summarise ncu reports into small text/JSON files under profiles/.

    python tools/ncu_summary.py OUT_DIR report.ncu-rep[:instances] ...

For each kernel in each report: duration, DRAM bytes (read/write), DRAM
throughput %, FP64 pipe %, issue %, occupancy, registers, top stall reasons
and the per-opcode dynamic instruction mix (tools/ncu_opcodes.py).
"""

import csv
import io
import json
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
from ncu_opcodes import opcode_table  # noqa: E402

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "sm__cycles_elapsed.avg.per_second",
    "lts__t_sector_hit_rate.pct", "smsp__inst_executed.sum", "launch__grid_size", "launch__block_size",
]


def raw_metrics(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    kernels = []
    for row in rows[2:]:
        d = dict(zip(hdr, row))
        m = {k: d[k] for k in KEYS if k in d}
        m["units"] = {k: units[hdr.index(k)] for k in KEYS if k in d}
        stalls = {k.split("stalled_")[1].split("_per_issue")[0]: float(v) for k, v in d.items()
                  if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")
                  and v not in ("", "n/a")}
        m["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:6])
        kernels.append((d["Kernel Name"], m))
    return kernels


def main():
    out_dir = Path(sys.argv[1])
    out_dir.mkdir(parents=True, exist_ok=True)
    for arg in sys.argv[2:]:
        report, _, inst = arg.partition(":")
        n = float(inst) if inst else None
        metrics = raw_metrics(report)
        ops = {k: (c, st) for k, c, st in opcode_table(report)}
        result = []
        for name, m in metrics:
            key = next((k for k in ops if k.split("(")[0].replace("(bool)", "") in name or name.split("(")[0] in k), None)
            entry = {"kernel": name, "metrics": m}
            if key:
                c, st = ops[key]
                tot = sum(c.values())
                entry["instructions"] = {"warp_total": tot, "thread_per_instance": tot * 32 / n if n else None,
                                         "by_opcode_per_instance": {op: round(v * 32 / n, 1) if n else v
                                                                    for op, v in c.most_common(20)}}
            result.append(entry)
        dst = out_dir / (Path(report).stem + ".json")
        dst.write_text(json.dumps(result, indent=1) + "\n")
        print("wrote", dst)


if __name__ == "__main__":
    main()
