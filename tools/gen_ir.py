"""Regenerate fixtures/ir/*.json from the reference front-end.

Runs only where the reference compiler is importable (this container, or any
box with baseline/_ref).  Inputs: our restated mechanisms in fixtures/mod and
the reference corpus (modlc/corpus/*.mod).  Each mechanism is compiled with
the default pass order (modlc/passes.py:32) and, for the corpus, also with
passes=() so the un-inlined FUNCTION/PROCEDURE path is covered.

    python tools/gen_ir.py
"""

from __future__ import annotations

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_1905_02241_b200.frontend import _import_modlc, compile_mod  # noqa: E402

OUT = ROOT / "fixtures" / "ir"


def main() -> int:
    _import_modlc()
    from modlc.corpus import corpus_files

    OUT.mkdir(parents=True, exist_ok=True)
    jobs = []
    for path in sorted((ROOT / "fixtures" / "mod").glob("*.mod")):
        jobs.append((path, path.stem, {}))
    for path in corpus_files():
        jobs.append((path, f"corpus_{path.stem}", {}))
        jobs.append((path, f"corpus_{path.stem}.nopass", {"passes": ()}))
    # solver-shape variants the default build does not reach
    cat = next(p for p in corpus_files() if p.stem == "cat")
    jobs.append((cat, "corpus_cat.pade", {"pade": True}))
    hh = ROOT / "fixtures" / "mod" / "hh_subset.mod"
    jobs.append((hh, "hh_subset.nopass", {"passes": ()}))
    # Pade (2+x)/(2-x) cnexp update (modlc/odes.py:414-434): the exp-cost lever
    jobs.append((hh, "hh_subset.pade", {"pade": True}))
    jobs.append((ROOT / "fixtures" / "mod" / "NaTs2_t.mod", "NaTs2_t.pade", {"pade": True}))
    three = next(p for p in corpus_files() if p.stem == "threestate")
    jobs.append((three, "corpus_threestate.nocse", {"use_cse": False}))
    written = 0
    for path, stem, kw in jobs:
        try:
            ir = compile_mod(path, **kw)
        except Exception as exc:  # unsupported constructs stay out of the fixture set
            print(f"skip {stem}: {type(exc).__name__}: {exc}")
            continue
        ir.meta = {"file": path.name, "options": {k: list(v) if isinstance(v, tuple) else v for k, v in kw.items()}}
        (OUT / f"{stem}.json").write_text(ir.to_json())
        written += 1
    print(f"wrote {written} IR files to {OUT}")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
