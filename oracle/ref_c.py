"""ORACLE (test/bench infrastructure only) -- ctypes binding of oracle/_ref.

Runs the reference-emitted scalar C (built by oracle/build_ref.py) on numpy
instance stores: `ref_steps(md, steps, nthreads)` performs `steps` x
(state_update, zero accumulators, current_update) with the instances split
into contiguous per-thread shards.  Used as the CPU baseline ("kind":
"reference") by bench.py and as a second CPU cross-check in tests.
"""

from __future__ import annotations

import ctypes as C
import json
import os
import subprocess
import tempfile
from pathlib import Path

import numpy as np

REF_DIR = Path(__file__).resolve().parent / "_ref"


def available(stem: str) -> bool:
    return (REF_DIR / f"{stem}.c").is_file() and (REF_DIR / f"{stem}.json").is_file()


def native_build(stem: str) -> Path:
    """Compile the shipped C with -O3 -march=native for the host it runs on."""
    out = REF_DIR / "native"
    out.mkdir(parents=True, exist_ok=True)
    so = out / f"lib{stem}.so"
    src = REF_DIR / f"{stem}.c"
    if not so.is_file() or so.stat().st_mtime < src.stat().st_mtime:
        tmp = Path(tempfile.mkdtemp(dir=out)) / f"lib{stem}.so"
        subprocess.run(["gcc", "-O3", "-march=native", "-fPIC", "-shared", "-pthread", str(src), "-o", str(tmp), "-lm"],
                       check=True, capture_output=True)
        os.replace(tmp, so)
    return so


class RefC:
    def __init__(self, stem: str, so_path: Path | None = None):
        meta = json.loads((REF_DIR / f"{stem}.json").read_text())
        self.meta = meta
        self.so = so_path or (REF_DIR / f"lib{stem}.so")
        self.lib = C.CDLL(str(self.so))
        fields = [("n_instances", C.c_long), ("solver_failures", C.c_long)]
        fields += [(s, C.c_double) for s in meta["scalars"]]
        fields += [(f, C.POINTER(C.c_double)) for f in meta["fields"][2 + len(meta["scalars"]):]]
        self.Struct = type("ref_data", (C.Structure,), {"_fields_": fields})
        self.lib.ref_steps.argtypes = [C.POINTER(self.Struct), C.c_long, C.c_int]
        self.lib.ref_initialize.argtypes = [C.POINTER(self.Struct)]

    def _bind(self, data):
        """Struct pointing at the numpy arrays of `data` (kept alive by `data`)."""
        md = self.Struct()
        md.n_instances = data.n
        md.solver_failures = 0
        for s in self.meta["scalars"]:
            setattr(md, s, float(data.scalars[s]))
        ptr = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))
        md.v = ptr(data.arrays["v"])
        md.i_acc = ptr(data.acc["i_acc"])
        md.g_acc = ptr(data.acc["g_acc"])
        for name in self.meta["slots"]:
            setattr(md, name.replace("[", "_").replace("]", ""), ptr(data.arrays[name]))
        return md

    def initialize(self, data):
        md = self._bind(data)
        self.lib.ref_initialize(C.byref(md))
        return data

    def steps(self, data, steps: int, nthreads: int = 1):
        md = self._bind(data)
        self.lib.ref_steps(C.byref(md), int(steps), int(nthreads))
        return md.solver_failures
