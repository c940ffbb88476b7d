"""Shared test configuration.

`-m "not gpu"` runs everywhere (oracle vs golden vectors, IR, printer, host
logic, C-ABI symbol exports, gloo multi-process).  `-m gpu` tests are the CUDA
parity tests proper; they need a B200 and the in-tree built libraries.
"""

import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

IR_DIR = ROOT / "fixtures" / "ir"
GOLDEN_DIR = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def load_ir(stem):
    from paper_1905_02241_b200.ir import MechIR

    return MechIR.load(IR_DIR / f"{stem}.json")


def all_ir_stems():
    return sorted(p.stem for p in IR_DIR.glob("*.json"))


@pytest.fixture(scope="session")
def ir_stems():
    return all_ir_stems()
