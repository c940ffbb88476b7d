"""Access to the reference compiler front-end (kept as-is, not rebuilt).

The north star keeps `modlc`'s parser, DSL passes, symbolic solver lowering
and `MechanismLayout` unchanged (/root/reference/pkg/src/modlc/pipeline.py:35-65).
This module only locates an importable copy of it -- the offline install in
``baseline/_ref`` (travels to the GPU box), ``$MODLC_SRC``, or the read-only
reference tree when it exists -- and converts its layouts into `MechIR`.
Nothing on the kernel path needs it: printing, building and running kernels
work from `MechIR` JSON alone.
"""

from __future__ import annotations

import importlib
import os
import sys
from pathlib import Path

from .ir import MechIR, from_layout

REPO_ROOT = Path(__file__).resolve().parent.parent
_CANDIDATES = (
    REPO_ROOT / "baseline" / "_ref",
    Path(os.environ.get("MODLC_SRC", "/nonexistent")),
    Path("/root/reference/pkg/src"),
)


def modlc_available() -> bool:
    try:
        _import_modlc()
        return True
    except ImportError:
        return False


def _import_modlc():
    try:
        return importlib.import_module("modlc.pipeline")
    except ImportError:
        pass
    for cand in _CANDIDATES:
        if (cand / "modlc" / "pipeline.py").is_file():
            sys.dont_write_bytecode = True  # the reference tree is read-only
            sys.path.insert(0, str(cand))
            return importlib.import_module("modlc.pipeline")
    raise ImportError(
        "reference front-end `modlc` not importable; install it into baseline/_ref "
        "or set MODLC_SRC, or load a pre-compiled MechIR JSON instead"
    )


def compile_mod(path, **kwargs) -> MechIR:
    """`modlc.pipeline.compile_file(path, **kwargs).layout` as `MechIR`."""
    pipeline = _import_modlc()
    result = pipeline.compile_file(str(path), **kwargs)
    passes = kwargs.get("passes", "default")
    ir = from_layout(result.layout, source=f"{Path(path).name} passes={passes}")
    return ir


def compile_text(text: str, filename: str = "<input>", **kwargs) -> MechIR:
    pipeline = _import_modlc()
    result = pipeline.compile_source(text, filename=filename, **kwargs)
    return from_layout(result.layout, source=filename)


def reference_layout(path, **kwargs):
    """The live reference `MechanismLayout` (for tests that drive both sides)."""
    pipeline = _import_modlc()
    return pipeline.compile_file(str(path), **kwargs).layout
