"""ORACLE (test/bench infrastructure only) -- build the reference's own CPU path.

The reference's compiled CPU implementation of nrn_state/nrn_cur is the C its
codegen emits (`modlc.codegen.emit_scalar`, modlc/codegen.py:568-570).  The
reference never compiles it; here it is compiled unchanged
except for the one edit SURVEY.md §0 documents: the struct's `long n` count
field is renamed because a STATE named `n` collides with it
(modlc/codegen.py:427).  A small pthread driver (ours, appended) shards the
instances by pointer offset, one contiguous range per thread, and zeroes the
accumulators before every current_update because the emitted C adds into them
(modlc/codegen.py:326,331).

Outputs go to oracle/_ref/ (git-ignored, travels to the GPU box):
  <stem>.c      generated source (reference C + driver)
  <stem>.json   struct layout for the ctypes binding (oracle/ref_c.py)
  lib<stem>.so  gcc -O3 build (portable -march=x86-64-v3; bench.py rebuilds
                with -march=native on the box it runs on)

Needs the reference front-end, so it runs where /root/reference (or
baseline/_ref) is importable.  `python oracle/build_ref.py`
"""

from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
REF_DIR = ROOT / "oracle" / "_ref"
sys.path.insert(0, str(ROOT))

# mechanisms the benchmark and the CPU-baseline leg use
REF_MECHS = {
    "hh_subset": "fixtures/mod/hh_subset.mod",
    "ProbAMPANMDA_EMS": "fixtures/mod/ProbAMPANMDA_EMS.mod",
    "NaTs2_t": "fixtures/mod/NaTs2_t.mod",
    "K_Pst": "fixtures/mod/K_Pst.mod",
    "Ca_HVA": "fixtures/mod/Ca_HVA.mod",
    "SKv3_1": "fixtures/mod/SKv3_1.mod",
    "Ih": "fixtures/mod/Ih.mod",
    "cadyn": "fixtures/mod/cadyn.mod",
    "na6": "fixtures/mod/na6.mod",
    "cdp5ish": "fixtures/mod/cdp5ish.mod",
    "corpus_cat": "corpus:cat.mod",
}

PORTABLE_FLAGS = ["-O3", "-march=x86-64-v3"]


def _driver(mech: str, layout) -> str:
    from modlc.codegen import mangle

    ptrs = ["v", "i_acc", "g_acc"] + [mangle(s.name) for s in layout.slots]
    shift = "\n".join(f"        j->md.{p} += lo;" for p in ptrs)
    return f"""
/* ---- multi-threaded driver (nmodl-b200 oracle/_ref, not reference code) ---- */
#include <pthread.h>
#include <string.h>
typedef struct {{ {mech}_data md; long steps; }} ref_job;
static void *ref_worker(void *p) {{
    ref_job *j = (ref_job *)p;
    for (long s = 0; s < j->steps; s++) {{
        {mech}_state_update(&j->md);
        memset(j->md.i_acc, 0, sizeof(double) * (size_t)j->md.n_instances);
        memset(j->md.g_acc, 0, sizeof(double) * (size_t)j->md.n_instances);
        {mech}_current_update(&j->md);
    }}
    return 0;
}}
int ref_steps({mech}_data *md, long steps, int nthreads) {{
    if (nthreads < 1) nthreads = 1;
    pthread_t th[512];
    ref_job jobs[512];
    if (nthreads > 512) nthreads = 512;
    long n = md->n_instances;
    for (int t = 0; t < nthreads; t++) {{
        long lo = n * t / nthreads, hi = n * (t + 1) / nthreads;
        ref_job *j = &jobs[t];
        j->md = *md;
        j->steps = steps;
        j->md.n_instances = hi - lo;
{shift}
        pthread_create(&th[t], 0, ref_worker, j);
    }}
    long failures = 0;
    for (int t = 0; t < nthreads; t++) {{
        pthread_join(th[t], 0);
        failures += jobs[t].md.solver_failures;
    }}
    md->solver_failures += failures;
    return 0;
}}
int ref_initialize({mech}_data *md) {{ {mech}_initialize(md); return 0; }}
"""


def generate(stem: str, src: str) -> dict:
    from modlc.codegen import emit_scalar, mangle
    from modlc.corpus import corpus_path
    from modlc.pipeline import compile_file

    path = corpus_path(src.split(":", 1)[1]) if src.startswith("corpus:") else ROOT / src
    layout = compile_file(path).layout
    text = emit_scalar(layout).text
    if "    long n;\n" not in text or "id < md->n;" not in text:
        raise RuntimeError("unexpected emitted C shape")
    text = text.replace("    long n;\n", "    long n_instances;\n").replace("id < md->n;", "id < md->n_instances;")
    mech = layout.mechanism
    text += _driver(mech, layout)
    REF_DIR.mkdir(parents=True, exist_ok=True)
    (REF_DIR / f"{stem}.c").write_text(text)
    meta = {
        "mechanism": mech,
        "scalars": sorted(layout.global_scalars),
        "slots": [s.name for s in layout.slots],
        "fields": ["n_instances", "solver_failures"]
        + sorted(layout.global_scalars)
        + ["v", "i_acc", "g_acc"]
        + [mangle(s.name) for s in layout.slots],
    }
    (REF_DIR / f"{stem}.json").write_text(json.dumps(meta, indent=1))
    return meta


def compile_c(stem: str, out_dir: Path = REF_DIR, flags=None, suffix: str = "") -> Path:
    flags = flags or PORTABLE_FLAGS
    out_dir.mkdir(parents=True, exist_ok=True)
    so = out_dir / f"lib{stem}{suffix}.so"
    cmd = ["gcc", *flags, "-fPIC", "-shared", "-pthread", str(REF_DIR / f"{stem}.c"), "-o", str(so), "-lm"]
    subprocess.run(cmd, check=True, capture_output=True)
    return so


def build_all(quiet: bool = False) -> None:
    from paper_1905_02241_b200.frontend import _import_modlc

    _import_modlc()
    for stem, src in REF_MECHS.items():
        generate(stem, src)
        compile_c(stem)
        compile_c(stem, flags=["-O2", "-ffp-contract=off"], suffix=".parity")
        if not quiet:
            print("built", stem)


if __name__ == "__main__":
    build_all()
