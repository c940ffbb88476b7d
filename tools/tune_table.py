"""Summarise tools/tune.py JSON lines: best variant per mechanism, and a
per-line table.   python tools/tune_table.py gpurun_out/tune_*.jsonl"""
import json
import sys

KEYS = ("ilp", "fast_path", "min_blocks", "pipe", "grid_waves", "tile", "exp_table", "recip", "div_approx", "exp_smem", "fast_redo", "lu_spec", "warp_tiles", "idx_ahead", "quot", "exp_estrin", "exp_share", "block")
best = {}
for path in sys.argv[1:]:
    for line in open(path):
        d = json.loads(line)
        if "error" in d:
            print("ERR", d["stem"], d["error"][:160])
            continue
        o = d["opts"]
        tag = " ".join(f"{k}={int(o[k]) if isinstance(o[k], bool) else o[k]}" for k in KEYS if k in o)
        print(f"{d['stem']:17s} {tag:70s} {d['ms']:.4f} ms {d['GBps']:6.0f} GB/s")
        if d["stem"] not in best or d["ms"] < best[d["stem"]][0]:
            best[d["stem"]] = (d["ms"], tag, d["GBps"])
print()
for s, (ms, tag, g) in best.items():
    print(f"BEST {s:17s} {ms:.4f} ms {g:6.0f} GB/s  {tag}")
