"""Build (here, without a GPU) the kernel libraries a tools/tune.py sweep will
load, so the GPU box only runs them:  python tools/prebuild.py --around SPEC stems...
(same arguments as tools/tune.py --around / --grid)."""

import dataclasses
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))

from bench import options_for  # noqa: E402
from paper_1905_02241_b200.build import build_mechanism  # noqa: E402
from paper_1905_02241_b200.ir import MechIR  # noqa: E402
from tune import grid  # noqa: E402


def main():
    args = sys.argv[1:]
    jobs = []
    while args:
        mode, spec = args[0], args[1]
        stems = []
        args = args[2:]
        while args and not args[0].startswith("--"):
            stems.append(args.pop(0))
        deltas = grid(spec)
        keys = [p.split("=")[0] for p in spec.split()]
        for stem in stems:
            for d in deltas:
                opts = d if mode == "--grid" else dataclasses.replace(
                    options_for(stem), **{k: getattr(d, k) for k in keys})
                jobs.append((stem, opts))
    print(f"{len(jobs)} builds")

    def one(job):
        stem, opts = job
        try:
            build_mechanism(MechIR.load(ROOT / "fixtures" / "ir" / f"{stem}.json"), opts)
        except Exception as exc:  # noqa: BLE001
            print(stem, opts, exc)

    with ThreadPoolExecutor(8) as pool:
        list(pool.map(one, jobs))


if __name__ == "__main__":
    main()
