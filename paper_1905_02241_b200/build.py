"""nvcc driver: builds the runtime library and per-mechanism kernel libraries.

Everything is built in-tree under ``paper_1905_02241_b200/_build`` so the
shared objects travel to the GPU box with the repository snapshot.  Mechanism
libraries are content-addressed (hash of the generated text, the device
headers and the flags), so a rebuild happens only when something changed and
stale objects can never be picked up.
"""

from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
import threading
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

from .codegen_cuda import CudaOptions, CudaPrinter, MechAbi

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
INCLUDE = CSRC / "include"
BUILD = PKG / "_build"
RUNTIME_SO = BUILD / "libnmodl_b200_rt.so"
ARCH = "-gencode=arch=compute_100a,code=sm_100a"

_lock = threading.Lock()
_key_locks: dict[str, threading.Lock] = {}


def nvcc_path() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).is_file():
            return cand
    raise RuntimeError("nvcc not found; the CUDA backend needs nvcc 12.9 (sm_100a)")


def base_flags(fmad: bool = False) -> list[str]:
    return [
        ARCH,
        "-O3",
        "-lineinfo",
        "-std=c++17",
        f"-fmad={'true' if fmad else 'false'}",
        "-Xcompiler",
        "-fPIC",
        "-shared",
        "-cudart",
        "shared",
        "-diag-suppress",
        "177,550",
        f"-I{INCLUDE}",
    ]


def _headers_digest() -> str:
    h = hashlib.sha256()
    for p in sorted(INCLUDE.rglob("*")):
        if p.is_file():
            h.update(p.name.encode())
            h.update(p.read_bytes())
    return h.hexdigest()


def _run(cmd: list[str], log: Path) -> None:
    proc = subprocess.run(cmd, capture_output=True, text=True)
    log.write_text(" ".join(cmd) + "\n" + proc.stdout + proc.stderr)
    if proc.returncode != 0:
        raise RuntimeError(f"nvcc failed ({log}):\n{proc.stderr[-4000:]}")


def build_runtime(force: bool = False) -> Path:
    """libnmodl_b200_rt.so from csrc/nmodl_rt.cu."""
    src = CSRC / "nmodl_rt.cu"
    stamp = BUILD / "libnmodl_b200_rt.stamp"
    digest = hashlib.sha256(src.read_bytes() + _headers_digest().encode()).hexdigest()
    with _lock:
        if not force and RUNTIME_SO.is_file() and stamp.is_file() and stamp.read_text() == digest:
            return RUNTIME_SO
        BUILD.mkdir(parents=True, exist_ok=True)
        tmp = RUNTIME_SO.with_suffix(".so.tmp")
        _run([nvcc_path(), *base_flags(), str(src), "-o", str(tmp)], BUILD / "libnmodl_b200_rt.log")
        tmp.replace(RUNTIME_SO)
        stamp.write_text(digest)
    return RUNTIME_SO


class MechBuild:
    """Generated source + built library + ABI for one mechanism/options pair."""

    def __init__(self, so_path: Path, cu_path: Path, abi: MechAbi, symbol: str, text: str):
        self.so_path = so_path
        self.cu_path = cu_path
        self.abi = abi
        self.symbol = symbol  # C prefix of the entry points
        self.text = text


def build_mechanism(layout, options: CudaOptions | None = None, fmad: bool | None = None,
                    force: bool = False) -> MechBuild:
    """emit_cuda + nvcc -> content-addressed shared object."""
    options = options or CudaOptions()
    fmad = options.fmad if fmad is None else fmad
    printer = CudaPrinter(layout, options)
    text = printer.emit_unit()
    abi = printer._abi
    flags = base_flags(fmad)
    # the key must not depend on where the repo lives (the GPU box runs it
    # from another path): the include directory enters through its content
    portable = [f for f in flags if not f.startswith("-I")]
    key = hashlib.sha256(
        (text + "\0" + " ".join(portable) + "\0" + _headers_digest()).encode()
    ).hexdigest()[:20]
    out_dir = BUILD / "mech"
    stem = f"{printer.mech}-{key}"
    so = out_dir / f"lib{stem}.so"
    cu = out_dir / f"{stem}.cu"
    with _lock:
        key_lock = _key_locks.setdefault(key, threading.Lock())
    with key_lock:
        out_dir.mkdir(parents=True, exist_ok=True)
        if force or not so.is_file():
            cu.write_text(text)
            tmp = so.with_suffix(f".so.tmp{os.getpid()}.{threading.get_ident()}")
            _run([nvcc_path(), *flags, str(cu), "-o", str(tmp)], out_dir / f"{stem}.log")
            tmp.replace(so)
        else:
            _touch(so)
    return MechBuild(so, cu, abi, printer.mech, text)


def _touch(path: Path) -> None:
    """Mark a cached library as in use (prune_stale keeps what a build touched)."""
    try:
        os.utime(path)
    except OSError:
        pass


def prune_stale(since: float) -> int:
    """Remove the generated sources / logs / libraries in _build/mech that no
    build since `since` (a time.time() stamp) produced or reused -- the
    content-addressed cache otherwise keeps every variant ever built, and the
    tree travels to the GPU box.  Returns the number of files removed."""
    out_dir = BUILD / "mech"
    if not out_dir.is_dir():
        return 0
    keep = {p.name[3:-3] for p in out_dir.glob("lib*.so") if p.stat().st_mtime >= since - 1.0}
    removed = 0
    for p in out_dir.iterdir():
        stem = p.name[3:-3] if p.name.startswith("lib") and p.name.endswith(".so") else p.name.rsplit(".", 1)[0]
        if stem not in keep:
            p.unlink()
            removed += 1
    return removed


def build_many(layouts, options: CudaOptions | None = None, fmad: bool | None = None,
               jobs: int | None = None) -> list[MechBuild]:
    jobs = jobs or min(8, os.cpu_count() or 4)
    with ThreadPoolExecutor(jobs) as pool:
        return list(pool.map(lambda l: build_mechanism(l, options, fmad), layouts))


class GroupBuild:
    """Built population group (codegen_cuda.emit_group): library + member ABIs."""

    def __init__(self, so_path: Path, cu_path: Path, symbol: str, abis, text: str):
        self.so_path = so_path
        self.cu_path = cu_path
        self.symbol = symbol
        self.abis = abis
        self.text = text


_GROUP_MEMO: dict = {}


def build_group(name: str, chains, fmad: bool = False, force: bool = False, kind: str = "unique") -> GroupBuild:
    """emit_group + nvcc -> content-addressed shared object (same keying as
    build_mechanism: generated text, portable flags, header digest)."""
    from .codegen_cuda import _cname, emit_group

    # in-process memo: a caller that rebuilds the same group from the same
    # layout objects (a column call reusing its runners) skips the emission
    memo = (name, kind, fmad, tuple(tuple((id(lay), repr(o)) for lay, o in ch) for ch in chains))
    hit = _GROUP_MEMO.get(memo)
    if hit is not None and not force and hit[1].so_path.is_file():
        return hit[1]
    unit, abis = emit_group(name, chains, kind)
    flags = base_flags(fmad)
    portable = [f for f in flags if not f.startswith("-I")]
    key = hashlib.sha256((unit.text + "\0" + " ".join(portable) + "\0" + _headers_digest()).encode()).hexdigest()[:20]
    out_dir = BUILD / "mech"
    stem = f"group_{_cname(name)}-{key}"
    so = out_dir / f"lib{stem}.so"
    cu = out_dir / f"{stem}.cu"
    with _lock:
        key_lock = _key_locks.setdefault(key, threading.Lock())
    with key_lock:
        out_dir.mkdir(parents=True, exist_ok=True)
        if force or not so.is_file():
            cu.write_text(unit.text)
            tmp = so.with_suffix(f".so.tmp{os.getpid()}.{threading.get_ident()}")
            _run([nvcc_path(), *flags, str(cu), "-o", str(tmp)], out_dir / f"{stem}.log")
            tmp.replace(so)
        else:
            _touch(so)
    gb = GroupBuild(so, cu, _cname(name), abis, unit.text)
    # the layouts stay referenced by the memo, so their ids are not reused
    _GROUP_MEMO[memo] = ([lay for ch in chains for lay, _ in ch], gb)
    return gb
