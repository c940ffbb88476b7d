"""ncu evidence for every kernel bench.py times, keyed by the exact build.

    python tools/profile_bench.py OUT_DIR [WORKLOAD ...]      (on the GPU box)

For each workload (default: all of bench.WORKLOADS) this runs, under
`ncu --set full --import-source on --clock-control none`, a child process
that sets the workload up exactly as bench.py does (same builds from
bench.options_for, same population sizes, same couplings / column shard),
warms up 3 steps and launches ONE more step; ncu captures only that step's
kernels (launch-skip over the warm-up).  The parent then

  * writes OUT_DIR/<workload>.ncu-rep and the summary OUT_DIR/<workload>.json
    (tools/ncu_summary.py: time, DRAM bytes, pipes, occupancy, stalls, opcode
    mix per kernel), and
  * records every captured kernel's DRAM bytes (read + write, one launch)
    under "<build key>@<instances>" (the content-addressed library stem and
    the population size) in OUT_DIR/ncu_traffic.json, which bench.py reads as `roofline.traffic`
    when the build it times has the same key (copy it to profiles/).
"""

from __future__ import annotations

import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))

WARM = 3
# bench.py warms the secondary workloads 100 steps (cdp5ish's Newton iteration
# counts fall over the first ~100 steps after nrn_init): profile the same state
WARM_FOR = {"kinetic1m": 100, "kinetic10m": 100, "kinetic1m_grouped": 100}
FP64_OPCODES = ("DFMA", "DMUL", "DADD", "DSETP", "DMNMX")  # the FP64 pipe (paper_1905_02241_b200.analysis)


def child(workload: str, out: str) -> None:
    import argparse

    import bench
    from paper_1905_02241_b200 import runtime as rt

    rt.require_device(0)
    rows = []
    if workload == "column":
        from paper_1905_02241_b200.column import LAUNCH_ORDER, ColumnShard

        spec = bench._column_spec()
        shard = ColumnShard(spec, 0, spec.n_cells, bench.options_for, **bench._column_mode())
        shard.launch(WARM)
        shard.stream.sync()
        shard.launch(1)
        shard.stream.sync()
        shard.check()
        per_step = shard.kernels_per_step()
        from paper_1905_02241_b200.column import SOMA_MECHS

        for m in LAUNCH_ORDER:
            if m in shard.group_members:
                continue
            r, d = shard.runners[m], shard.devs[m]
            rows.append({"kernel": f"{r.mb.symbol}_k_{r.node_kernel(d)}", "build": r.mb.so_path.stem[3:], "n": d.n})
        if shard.grouped:
            gb = shard.group.gb
            rows.append({"kernel": f"{gb.symbol}_k_step_unique", "build": gb.so_path.stem[3:],
                         "n": sum(shard.devs[m].n for m in shard.group_members)})
    else:
        w = bench.WORKLOADS[workload]
        dist = argparse.Namespace(rank=0)
        pops = [bench.Population(s, n, w["nodes"], 42, bench.options_for(s)) for s, n in w["mechs"]]
        for p in pops:
            p.setup_device()
        by = {p.stem: p for p in pops}
        for dst, dslot, src, sslot in w.get("couplings", ()):
            by[dst].runner.share_slot(by[dst].dev, dslot, by[src].dev, sslot)
        s0 = pops[0].runner.stream
        for p in pops:
            p.runner.stream = s0
        members = list(pops)
        if w.get("grouped"):
            pops = [bench._DirectGroup(pops, w.get("couplings", ()), s0, w["grouped"])]
        for _ in range(WARM_FOR.get(workload, WARM) + 1):
            for p in pops:
                p.launch(1)
        s0.sync()
        for p in members:
            p.runner.check(p.dev)
        per_step = len(pops)
        for p in pops:
            rows.append({"kernel": p.kernel_name, "build": p.build_key, "n": p.n, "bytes_per_launch": p.launch_bytes()})
        del dist
    Path(out).write_text(json.dumps({"workload": workload, "per_step": per_step, "kernels": rows}))


def _raw(report: Path) -> list[dict]:
    txt = subprocess.run(["ncu", "-i", str(report), "--page", "raw", "--csv", "--print-units", "base"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = rows[0]
    return [dict(zip(hdr, r)) for r in rows[2:]]


def _num(v: str) -> float:
    return float(str(v).replace(",", ""))


def parent(out_dir: Path, workloads: list[str]) -> None:
    import bench

    import os

    tag = os.environ.get("PROFILE_TAG", out_dir.name)  # where the summaries get committed under profiles/
    out_dir.mkdir(parents=True, exist_ok=True)
    traffic_path = out_dir / "ncu_traffic.json"
    record = json.loads(traffic_path.read_text()) if traffic_path.is_file() else {"by_build": {}}
    for wl in workloads:
        meta = out_dir / f"{wl}.meta.json"
        # the per-step kernel count is known after setup; a dry child run is
        # cheap compared to the capture, so read it from bench's own tables
        if wl == "column":
            per_step = {"sequential": 7, "concurrent": 8, "grouped": 4}[bench._column_mode()["schedule"]]
            regex = "regex:_k_step|combine"
        else:
            per_step = 1 if bench.WORKLOADS[wl].get("grouped") else len(bench.WORKLOADS[wl]["mechs"])
            regex = "regex:_k_step"
        rep = out_dir / f"{wl}"
        cmd = ["ncu", "--set", "full", "--import-source", "on", "--clock-control", "none", "-k", regex,
               "--launch-skip", str(WARM_FOR.get(wl, WARM) * per_step), "--launch-count", str(per_step), "-f", "-o", str(rep),
               sys.executable, __file__, "--child", wl, str(meta)]
        print(" ".join(cmd), flush=True)
        proc = subprocess.run(cmd, capture_output=True, text=True)
        (out_dir / f"{wl}.ncu.log").write_text(proc.stdout[-20000:] + proc.stderr[-20000:])
        if proc.returncode != 0:
            print(f"[profile] {wl}: ncu rc={proc.returncode}", flush=True)
            continue
        info = json.loads(meta.read_text())
        by_kernel = {k["kernel"]: k for k in info["kernels"]}
        for r in _raw(Path(str(rep) + ".ncu-rep")):
            name = r["Kernel Name"].split("(")[0].split("<")[0].replace("void ", "").strip()
            k = by_kernel.get(name)
            if k is None:
                continue
            dram = _num(r["dram__bytes_read.sum"]) + _num(r["dram__bytes_write.sum"])
            record["by_build"][f"{k['build']}@{k['n']}"] = {
                "kernel": name, "workload": wl, "instances": k["n"], "dram_bytes": dram,
                "dram_read": _num(r["dram__bytes_read.sum"]), "dram_write": _num(r["dram__bytes_write.sum"]),
                "us": _num(r["gpu__time_duration.sum"]) / 1e3, "bytes_per_launch": k.get("bytes_per_launch"),
                "capture": f"ncu --set full, one launch after {WARM_FOR.get(wl, WARM)} warm-up steps; summary "
                           f"profiles/{tag}/{wl}.json",
            }
        subprocess.run([sys.executable, str(ROOT / "tools" / "ncu_summary.py"), str(out_dir),
                        f"{rep}.ncu-rep"], check=False)
        # measured FP64 pipe instructions per instance (opcode mix x 32 lanes / n)
        summ = out_dir / f"{wl}.json"
        if summ.is_file():
            for e in json.loads(summ.read_text()):
                name = e["kernel"].split("(")[0].split("<")[0].replace("void ", "").strip()
                k = by_kernel.get(name)
                ops = (e.get("instructions") or {}).get("by_opcode_per_instance") or {}
                key = f"{k['build']}@{k['n']}" if k else None
                if key in record["by_build"] and ops:
                    fp = sum(v for op, v in ops.items() if op in FP64_OPCODES)
                    record["by_build"][key]["fp64_instr_per_instance"] = 32.0 * fp / k["n"]
        traffic_path.write_text(json.dumps(record, indent=1, sort_keys=True) + "\n")
    print("wrote", traffic_path)


if __name__ == "__main__":
    if sys.argv[1] == "--child":
        child(sys.argv[2], sys.argv[3])
    else:
        import bench

        parent(Path(sys.argv[1]), sys.argv[2:] or [w for w in bench.WORKLOADS])
