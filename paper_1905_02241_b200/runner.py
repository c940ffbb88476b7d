"""`CudaRunner`: the GPU drop-in for the reference's `interp.Runner`.

Same constructor and `run_kernel(data, kernel_name, steps) -> data` contract
as modlc/interp.py:124-131,456-471, operating in place on an `InstanceData`
(the reference's, or any object with ``n/arrays/acc/scalars/newton_iters``),
so `simulate`, `compare_pipelines` and `diff_trajectories`-style callers work
unchanged.  Errors surface as `InterpError` with the reference's messages.

Two ways to drive it:

* host data (drop-in): every call uploads the store, runs the kernel(s) on the
  device and writes the results back into the numpy arrays;
* device-resident (`to_device` / `DeviceInstanceData`): the SoA store lives in
  HBM across calls; `run_kernel` then only launches.  This is the production
  path (and what `simulate` uses between its single upload and download).

Kernel names are the reference's three plus ``"step"`` (fused
state_update+current_update per timestep) and ``"step_nodes"`` (the
node_index gather/scatter variant, see `bind_nodes`).
"""

from __future__ import annotations

import ctypes as C
import sys

import numpy as np

from . import runtime as rt
from .build import build_mechanism
from .codegen_cuda import CudaOptions
from .ir import NEWTON_MAX_ITER, from_layout, iter_nodes

KERNELS = ("initialize", "state_update", "current_update", "step", "step_nodes")
_PARTS = {
    "initialize": ("initialize",),
    "state_update": ("state_update",),
    "current_update": ("current_update",),
    "step": ("state_update", "current_update"),
    "step_nodes": ("state_update", "current_update"),
}
_KNAME = {0: "initialize", 1: "state_update", 2: "current_update"}
ALIGN = 256


class InterpError(RuntimeError):
    """Raised like the reference's modlc.interp.InterpError (interp.py:33-34)."""


def _interp_error(msg: str) -> Exception:
    """Return an exception that is also a modlc.interp.InterpError when the
    reference runtime is loaded, so reference callers catch it unchanged."""
    ref = sys.modules.get("modlc.interp")
    if ref is not None and hasattr(ref, "InterpError"):
        cls = type("InterpError", (InterpError, ref.InterpError), {})
        return cls(msg)
    return InterpError(msg)


class HostInstanceData:
    """Minimal InstanceData (modlc/interp.py:37-52) for callers without modlc."""

    def __init__(self, n, arrays, acc, scalars, newton_iters=None):
        self.n = n
        self.arrays = arrays
        self.acc = acc
        self.scalars = scalars
        self.newton_iters = list(newton_iters or [])

    def copy(self):
        return HostInstanceData(
            self.n,
            {k: v.copy() for k, v in self.arrays.items()},
            {k: v.copy() for k, v in self.acc.items()},
            dict(self.scalars),
            list(self.newton_iters),
        )


class NodeBinding:
    """node_index scatter layout resident on the device (builder extension).

    perm/rank: node-stable sort of instances (np.argsort(node_index,
    kind="stable") and its inverse); offsets: per-node instance segments in
    sorted order; seg_node/seg_offsets: the nodes that own instances and their
    instance ranges; tile_segs: CTA tiles made of whole segments.
    """

    def __init__(self, n, n_nodes):
        self.n = n
        self.n_nodes = n_nodes
        self.buffers = []
        # 1: this population's launch starts each touched node's rhs/d from 0
        # (it is the first to fold into them in a timestep); 0: accumulate
        self.assign = 0

    def alloc(self, nbytes):
        b = rt.DeviceBuffer(nbytes)
        self.buffers.append(b)
        return b.ptr

    def host_array(self, name: str, stream) -> np.ndarray:
        """Host copy of the int64 perm/rank arrays, fetched on first use
        (error remapping, tests) -- never on the stepping path."""
        cache = self.__dict__.setdefault("_host", {})
        if name not in cache:
            arr = np.empty(self.n, dtype=np.int64)
            rt.d2h(arr.ctypes.data, getattr(self, name), arr.nbytes, stream)
            stream.sync()
            cache[name] = arr
        return cache[name]

    @property
    def perm_host(self):
        return self.host_array("perm", self.stream)

    def _host_i64(self, name, ptr, count):
        cache = self.__dict__.setdefault("_host", {})
        if name not in cache:
            arr = np.empty(count, dtype=np.int64)
            rt.d2h(arr.ctypes.data, ptr, arr.nbytes, self.stream)
            self.stream.sync()
            cache[name] = arr
        return cache[name]

    @property
    def offsets_host(self):
        return self._host_i64("offsets", self.node_offsets_full, self.n_nodes + 1)

    @property
    def tile_segs_host(self):
        return self._host_i64("tile_segs", self.tile_segs, self.n_tiles + 1)

    @property
    def seg_offsets_host(self):
        return self._host_i64("seg_offsets", self.seg_offsets, self.n_segs + 1)


class NodeArrays:
    """Device node arrays (voltage, rhs, d) shared by several mechanism
    populations of one cell set (a compartment is one node)."""

    def __init__(self, node_v, node_rhs=None, node_d=None, stream=None):
        node_v = np.ascontiguousarray(node_v, dtype=np.float64)
        self.n_nodes = int(node_v.shape[0])
        nb = self.n_nodes * 8
        self.buffers = [rt.DeviceBuffer(nb) for _ in range(3)]
        self.node_v, self.node_rhs, self.node_d = (b.ptr for b in self.buffers)
        s = stream or rt.Stream()
        rt.h2d(self.node_v, node_v.ctypes.data, nb, s)
        for ptr, host in ((self.node_rhs, node_rhs), (self.node_d, node_d)):
            if host is None:
                rt.memset(ptr, 0, nb, s)
            else:
                h = np.ascontiguousarray(host, dtype=np.float64)
                rt.h2d(ptr, h.ctypes.data, nb, s)
        s.sync()

    def download(self, stream) -> dict:
        out = {}
        for name in ("node_v", "node_rhs", "node_d"):
            arr = np.empty(self.n_nodes)
            rt.d2h(arr.ctypes.data, getattr(self, name), arr.nbytes, stream)
            out[name] = arr
        stream.sync()
        return out


class DeviceInstanceData:
    """Device-resident SoA store: one arena, 256-byte aligned arrays."""

    def __init__(self, runner: "CudaRunner", n: int, names: list[str], scalars: dict):
        self.runner = runner
        self.n = n
        self.names = list(names)  # data.arrays order (slots ..., v)
        self.scalars = dict(scalars)
        self.newton_iters: list[int] = []
        stride = ((n * 8 + ALIGN - 1) // ALIGN) * ALIGN
        self.stride = stride
        count = len(self.names) + 2
        self.arena = rt.DeviceBuffer(stride * count)
        self.ptr = {name: self.arena.ptr + i * stride for i, name in enumerate(self.names)}
        self.ptr["i_acc"] = self.arena.ptr + len(self.names) * stride
        self.ptr["g_acc"] = self.arena.ptr + (len(self.names) + 1) * stride
        # kernel-written GLOBALs: two buffers (read / write) swapped per step
        # by the generated launch_steps; between calls buffer 0 is current
        self.nrw = max(1, len(runner.abi.rw_scalars))
        self.scalars_rw = rt.DeviceBuffer(16 * self.nrw)
        self.prebad: dict[str, int] = {}
        self.nodes: NodeBinding | None = None
        # arrays a launch (or the voltage gather) may have changed since the
        # upload: the only ones a write-back has to bring home
        self.dirty: set[str] = set()
        # arrays holding no value yet (not uploaded, not written by a launch):
        # never permuted, never downloaded
        self.unset: set[str] = set()

    def reorder(self, perm_ptr: int, stream) -> None:
        """new[k] = old[perm[k]] for every array, into a fresh arena."""
        names = list(self.names) + ["i_acc", "g_acc"]
        arena = rt.DeviceBuffer(self.stride * len(names))
        L = rt.lib()
        new_ptr = {}
        for i, name in enumerate(names):
            dst = arena.ptr + i * self.stride
            if name not in self.unset:
                rt.check(L.nmodl_permute(C.c_void_p(self.ptr[name]), C.c_void_p(dst), C.c_void_p(perm_ptr), self.n,
                                         0, C.c_void_p(stream.handle)), "permute")
            new_ptr[name] = dst
        stream.sync()
        self.arena = arena  # the old arena returns to the allocator cache
        self.ptr = new_ptr

    # ---- host <-> device ------------------------------------------------------
    def upload_from(self, data, stream, skip=()) -> None:
        self.unset |= set(skip)
        for name in self.names:
            if name in skip:
                continue
            arr = np.ascontiguousarray(data.arrays[name], dtype=np.float64)
            if arr.shape != (self.n,):
                raise ValueError(f"array {name!r} has shape {arr.shape}, expected ({self.n},)")
            rt.h2d(self.ptr[name], arr.ctypes.data, arr.nbytes, stream)
            stream.sync() if arr is not data.arrays[name] else None
        for name in ("i_acc", "g_acc"):
            if name in skip:
                continue
            arr = np.ascontiguousarray(data.acc[name], dtype=np.float64)
            rt.h2d(self.ptr[name], arr.ctypes.data, arr.nbytes, stream)
        stream.sync()

    def download_into(self, data, stream, names=None, acc=True) -> None:
        names = self.names if names is None else names
        for name in names:
            dst = data.arrays[name]
            if not (dst.flags.c_contiguous and dst.dtype == np.float64):
                tmp = np.empty(self.n)
                rt.d2h(tmp.ctypes.data, self.ptr[name], tmp.nbytes, stream)
                stream.sync()
                dst[:] = tmp
            else:
                rt.d2h(dst.ctypes.data, self.ptr[name], dst.nbytes, stream)
        for name in ("i_acc", "g_acc") if acc else ():
            dst = data.acc[name]
            rt.d2h(dst.ctypes.data, self.ptr[name], dst.nbytes, stream)
        stream.sync()

    def array(self, name) -> np.ndarray:
        out = np.empty(self.n)
        s = self.runner.stream
        rt.d2h(out.ctypes.data, self.ptr[name], out.nbytes, s)
        s.sync()
        return out


class CudaRunner:
    """Compiles one mechanism for sm_100a and executes its kernels."""

    def __init__(self, layout, jac_mode: str = "exact", *, options: CudaOptions | None = None,
                 fmad: bool | None = None, device: int | None = None):
        if jac_mode not in ("exact", "fd"):
            raise ValueError("jac_mode must be 'exact' or 'fd'")
        self.layout = layout
        self.ir = from_layout(layout)
        self.jac_mode = jac_mode
        self.flags = 1 if jac_mode == "fd" else 0
        self.device = rt.require_device(device)
        self.options = options or CudaOptions()
        self.mb = build_mechanism(self.ir, self.options, fmad)
        self.abi = self.mb.abi
        self.lib = C.CDLL(str(self.mb.so_path))
        sym = self.mb.symbol
        self.entry = {}
        for k in KERNELS + ("step_unique",):
            fn = getattr(self.lib, f"{sym}_{k}", None)
            if fn is None and k == "step_unique":
                continue  # emitted for pipelined builds only
            fn.restype = C.c_int
            fn.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int]
            self.entry[k] = fn
        fields = []
        for f in self.abi.fields:
            ct = {"i64": C.c_longlong, "f64": C.c_double}.get(f.ctype, C.c_void_p)
            fields.append((f.name, ct))
        self.Struct = type(f"{sym}_data", (C.Structure,), {"_fields_": fields})
        size_fn = getattr(self.lib, f"{sym}_abi_size")
        size_fn.restype = C.c_longlong
        if size_fn() != C.sizeof(self.Struct):
            raise RuntimeError(f"ABI mismatch for {sym}: C {size_fn()} vs ctypes {C.sizeof(self.Struct)}")
        self.stream = rt.Stream()
        self.status = rt.DeviceBuffer(C.sizeof(rt.Status))
        self._reset_status()
        self._writes = {}
        for k in KERNELS:
            w = set(self.abi.kernels.get(k, {}).get("stores", ()))
            if k in ("current_update", "step", "step_nodes"):
                w |= {"i_acc", "g_acc"}
            self._writes[k] = w
        self.n_newton = len(self.abi.newton_nodes)
        self._newton_kernel = [s.split(":")[0] for s in self.abi.newton_nodes]
        self._max_iter = {}
        for kname, stmts in self.ir.kernels.items():
            for s in stmts:
                for node in iter_nodes(s):
                    if node.kind == "NewtonSolveNode":
                        self._max_iter.setdefault(kname, int(node.attrs.get("max_iter", NEWTON_MAX_ITER)))

    # ---- helpers ----------------------------------------------------------------
    trace: list | None = None  # set to [] to record (stage, seconds) wall-clock marks

    def _mark(self, stage: str) -> None:
        if self.trace is not None:
            import time

            self.stream.sync()
            self.trace.append((stage, time.perf_counter()))

    def _reset_status(self) -> None:
        rt.check(rt.lib().nmodl_status_reset(C.c_void_p(self.status.ptr), C.c_void_p(self.stream.handle)),
                 "status_reset")

    def _read_status(self) -> rt.Status:
        st = rt.Status()
        rt.d2h(C.addressof(st), self.status.ptr, C.sizeof(st), self.stream)
        self.stream.sync()
        return st

    def to_device(self, data, skip=()) -> DeviceInstanceData:
        """Upload an InstanceData into a device-resident store.  Arrays named
        in `skip` are left unset on the device (the caller overwrites them
        before any kernel reads them, e.g. v from the node voltage gather)."""
        names = list(data.arrays)
        missing = [s for s in self.abi.slots if s not in data.arrays]
        if missing or "v" not in data.arrays:
            raise _interp_error(f"layout mismatch: instance data lacks {missing or ['v']}")
        self._mark("upload:start")
        dev = DeviceInstanceData(self, int(data.n), names, data.scalars)
        dev.newton_iters = list(data.newton_iters)
        self._mark("upload:alloc")
        dev.upload_from(data, self.stream, skip)
        self._mark("upload:h2d")
        self._prescan(dev, skip)
        self._mark("upload:prescan")
        return dev

    def _prescan(self, dev: DeviceInstanceData, skip=()) -> None:
        """First non-finite index per array, once per upload (interp.py:538-545)."""
        buf = rt.DeviceBuffer(8 * len(dev.names))
        rt.memset(buf.ptr, 0xFF, 8 * len(dev.names), self.stream)
        L = rt.lib()
        for i, name in enumerate(dev.names):
            if name in skip:
                continue
            rt.check(L.nmodl_first_nonfinite(C.c_void_p(dev.ptr[name]), dev.n, C.c_void_p(buf.ptr + 8 * i),
                                             C.c_void_p(self.stream.handle)), "first_nonfinite")
        out = np.empty(len(dev.names), dtype=np.uint64)
        rt.d2h(out.ctypes.data, buf.ptr, out.nbytes, self.stream)
        self.stream.sync()
        dev.prebad = {name: int(v) for name, v in zip(dev.names, out) if v != np.uint64(rt.NO_ERROR)}

    def to_host(self, dev: DeviceInstanceData, data, only_dirty: bool = False) -> None:
        """Download a device store into `data` (arrays, acc, scalars, newton record).

        `only_dirty`: `data` is the very object the store was uploaded from,
        so arrays no launch could have written (parameters, ion reversal
        potentials, ...) already hold the device values and are not copied."""
        self._mark("download:start")
        names = list(dev.names)
        acc = True
        if only_dirty:
            names = [n for n in names if n in dev.dirty]
            acc = "i_acc" in dev.dirty
        names = [n for n in names if n not in dev.unset or n in dev.dirty]
        acc = acc and ("i_acc" not in dev.unset or "i_acc" in dev.dirty)
        if dev.nodes is not None:
            self._unpermute_into(dev, data, names, acc)
        else:
            dev.download_into(data, self.stream, names, acc)
        self._mark("download:arrays")
        data.scalars.update(dev.scalars)
        data.newton_iters[:] = dev.newton_iters

    def _struct(self, dev: DeviceInstanceData, newton_rec=0):
        """The `<mech>_data` argument block for `dev` (positional build: this
        runs once per launch call on the host)."""
        nb = dev.nodes
        vals = []
        for f in self.abi.fields:
            role = f.role
            if role == "slot" or role == "v" or role == "acc":
                vals.append(dev.ptr[f.key])
            elif role == "scalar":
                if f.key not in dev.scalars:
                    raise _interp_error(f"unbound name {f.key!r}")
                vals.append(float(dev.scalars[f.key]))
            elif role == "count":
                vals.append(dev.n)
            elif role == "status":
                vals.append(self.status.ptr)
            elif role == "newton":
                vals.append(newton_rec or None)
            elif role == "scalars_rw":
                vals.append(dev.scalars_rw.ptr)
            elif role == "scalars_rw_out":
                vals.append(dev.scalars_rw.ptr + 8 * dev.nrw)
            elif role == "node":
                vals.append((0 if f.ctype == "i64" else None) if nb is None else getattr(nb, f.key))
        return self.Struct(*vals)

    def _sync_scalars_in(self, dev) -> None:
        rw = self.abi.rw_scalars
        if rw:
            vals = np.array([float(dev.scalars.get(s, 0.0)) for s in rw])
            rt.h2d(dev.scalars_rw.ptr, vals.ctypes.data, vals.nbytes, self.stream)
            self.stream.sync()

    def _sync_scalars_out(self, dev) -> None:
        rw = self.abi.rw_scalars
        if rw:
            vals = np.empty(len(rw))
            rt.d2h(vals.ctypes.data, dev.scalars_rw.ptr, vals.nbytes, self.stream)
            self.stream.sync()
            for s, v in zip(rw, vals):
                dev.scalars[s] = float(v)

    # ---- execution -----------------------------------------------------------------
    def node_kernel(self, dev: DeviceInstanceData) -> str:
        """The kernel a `step_nodes` launch of `dev` runs: `step_unique` (the
        direct kernels' cp.async pipeline, one instance per node) when the
        build has it and every occupied node holds one instance, else the
        tiled `step_nodes` with its in-order segment reduction."""
        if dev.nodes is not None and dev.nodes.seg_unique in (1, 2) and "step_unique" in self.entry:
            return "step_unique"
        return "step_nodes"

    def launch(self, dev: DeviceInstanceData, kernel_name: str, steps: int = 1, newton_rec: int = 0,
               late_wait: bool = False) -> None:
        """Enqueue `steps` launches on the runner's stream (no sync, no checks).
        `late_wait` (tiled node kernel of a pdl build): the kernel's programmatic
        wait moves from its start to its node fold -- only for a launch whose
        predecessor in the stream writes nothing this population reads but the
        node arrays (ColumnShard: the synapses after the soma combine)."""
        if kernel_name == "step_nodes" and dev.nodes is None:
            raise ValueError("step_nodes needs bind_nodes() first")
        md = self._struct(dev, newton_rec)
        dev.dirty |= self._writes[kernel_name]
        rt.set_device(self.device)
        entry = self.entry[self.node_kernel(dev) if kernel_name == "step_nodes" else kernel_name]
        flags = self.flags | (2 if (late_wait and kernel_name == "step_nodes") else 0)
        rc = entry(C.byref(md), int(steps), C.c_void_p(self.stream.handle), flags)
        rt.check(rc, f"launch {self.mb.symbol}_{kernel_name}")

    def run_kernel(self, data, kernel_name: str, steps: int = 1):
        """modlc/interp.py:456-471 on the device."""
        if kernel_name not in KERNELS:
            raise KeyError(kernel_name)
        host = not isinstance(data, DeviceInstanceData)
        dev = self.to_device(data) if host else data
        if steps > 0 and dev.n > 0:
            self._run(dev, kernel_name, steps, host_data=data if host else None)
        if host:
            self.to_host(dev, data, only_dirty=True)
        return data

    def _run(self, dev, kernel_name, steps, host_data=None):
        parts = _PARTS[kernel_name]
        nn = self.n_newton
        rec = None
        if nn:
            rec = rt.DeviceBuffer(4 * nn * steps)
            rt.memset(rec.ptr, 0xFF, 4 * nn * steps, self.stream)
        self._sync_scalars_in(dev)
        self.launch(dev, kernel_name, steps, rec.ptr if rec else 0)
        st = self._read_status()
        self._sync_scalars_out(dev)
        if rec is not None:
            raw = np.empty(nn * steps, dtype=np.int32)
            rt.d2h(raw.ctypes.data, rec.ptr, raw.nbytes, self.stream)
            self.stream.sync()
            raw = raw.reshape(steps, nn)
            for step in range(steps):
                for p in parts:
                    for q in range(nn):
                        if self._newton_kernel[q] == p and raw[step, q] >= 0:
                            dev.newton_iters.append(int(raw[step, q]))
        key = st.err_key
        # pre-existing non-finite values in arrays this launch never rewrites
        # (prebad holds caller-order instance indices, like the error keys)
        written = set(self.abi.kernels["step" if kernel_name == "step_nodes" else kernel_name]["stores"])
        order = self.abi.array_order
        kcode = {"initialize": 0, "state_update": 1, "current_update": 2}[parts[0]]
        for name, idx in dev.prebad.items():
            if name not in written and name in order:
                cand = (kcode << 62) | (1 << 61) | (order.index(name) << 48) | idx
                key = min(key, cand)
        if key != rt.NO_ERROR:
            self._reset_status()
            if host_data is not None:
                self.to_host(dev, host_data, only_dirty=True)
            raise _interp_error(self._message(key, st, dev))
        # a completed launch rewrote (or checked) every array it stores: a
        # non-finite value seen at upload is gone from those
        for name in written:
            dev.prebad.pop(name, None)

    def _message(self, key, st, dev) -> str:
        kernel = _KNAME[(key >> 62) & 3]
        phase = (key >> 61) & 1
        ordinal = (key >> 48) & 0x1FFF
        kind = (key >> 46) & 3
        inst = key & ((1 << 40) - 1)  # caller order (node kernels map through perm)
        if phase == 1:
            name = self.abi.array_order[ordinal]
            return f"non-finite value in {name!r} at instance {inst} after kernel {kernel}"
        if kind == 0:
            return "WHILE loop exceeded 10000 iterations"
        if kind == 1:
            max_iter = self._max_iter.get(kernel, NEWTON_MAX_ITER)
            return (f"Newton failed to converge for instance {inst} "
                    f"(residual {st.payload:.3e} after {max_iter} iterations)")
        return f"singular matrix in runtime linear solve (instance {inst})"

    # ---- CUDA graphs -------------------------------------------------------------------
    def capture(self, dev: DeviceInstanceData, kernel_name: str, steps: int) -> rt.Graph:
        """Capture `steps` launches into a replayable graph (no Newton record)."""
        self._sync_scalars_in(dev)
        return rt.capture(self.stream, lambda: self.launch(dev, kernel_name, steps))

    def check(self, dev: DeviceInstanceData, kernel_name: str = "step") -> None:
        """Raise if any launch since the last check reported an error."""
        st = self._read_status()
        if st.err_key != rt.NO_ERROR:
            self._reset_status()
            raise _interp_error(self._message(st.err_key, st, dev))

    # ---- node_index extension ----------------------------------------------------------
    def bind_nodes(self, dev: DeviceInstanceData, node_index, node_v=None, node_rhs=None, node_d=None,
                   tile: int | None = None, shared: "NodeArrays | None" = None,
                   prepared: "NodeBinding | None" = None) -> NodeBinding:
        """Attach node arrays and reorder the store node-stably on the device.

        With `shared`, the node voltage/rhs/d arrays are the given device
        arrays (all mechanisms of a cell population fold into the same nodes,
        in launch order); otherwise they are allocated from the host arrays.
        `prepared`: the result of prepare_nodes() for this population (its
        node layout was built on another stream while the store uploaded)."""
        if dev.nodes is not None:
            raise ValueError("nodes already bound")
        if prepared is None:
            nb = self.prepare_nodes(dev.n, node_index, node_v, node_rhs, node_d, tile, shared)
        else:
            nb = prepared
            if nb.n != dev.n:
                raise ValueError("prepared node layout is for another population size")
        return self._finish_nodes(dev, nb)

    def node_tile(self, n: int) -> int:
        """Target instances per node tile: whole waves of the node kernel's
        persistent grid (G resident CTAs, each looping over tiles) with at
        most ~94% of the shared-memory tile, so every CTA gets the same
        number of equal tiles (an unbalanced last wave costs up to a tile's
        time; 1.25M synapses: 724 tiles on 592 CTAs took 1.6x as long)."""
        if getattr(self, "_node_ctas", None) is None:
            fn = getattr(self.lib, f"{self.mb.symbol}_step_nodes_ctas")
            fn.restype = C.c_int
            rt.set_device(self.device)
            self._node_ctas = max(1, int(fn()))
        G = self._node_ctas
        cap = max(64, (15 * self.options.tile) // 16)
        waves = max(1, -(-n // (G * cap)))
        return max(64, -(-n // (G * waves)))

    def aux_stream(self) -> "rt.Stream":
        """A second stream of this runner (node layout built beside the upload)."""
        if getattr(self, "_aux", None) is None:
            self._aux = rt.Stream()
        return self._aux

    def prepare_nodes(self, n: int, node_index, node_v=None, node_rhs=None, node_d=None, tile: int | None = None,
                      shared: "NodeArrays | None" = None, stream: "rt.Stream | None" = None) -> NodeBinding:
        """Enqueue the node layout of an n-instance population (node_index
        upload, stable sort, segments, tiles, node arrays) on `stream`
        without waiting for it; bind_nodes(prepared=...) completes it."""
        self._mark("bind:start")
        node_index = np.ascontiguousarray(node_index, dtype=np.int32)
        if shared is None:
            node_v = np.ascontiguousarray(node_v, dtype=np.float64)
            n_nodes = int(node_v.shape[0])
        else:
            n_nodes = shared.n_nodes
        if node_index.shape != (n,):
            raise ValueError("node_index must have one entry per instance")
        nb = NodeBinding(n, n_nodes)
        s = stream or self.stream
        nb.stream = s
        nb._host_keep = (node_index, node_v, node_rhs, node_d)  # sources of the async copies
        L = rt.lib()
        idx_in = nb.alloc(4 * n)
        rt.h2d(idx_in, node_index.ctypes.data, 4 * n, s)
        counts = nb.alloc(4 * n_nodes)
        nb.node_offsets_full = nb.alloc(8 * (n_nodes + 1))
        scratch = nb.alloc(8 * n)
        nb.perm = nb.alloc(8 * n)
        nb.rank = nb.alloc(8 * n)
        bad = nb.alloc(4)
        rt.check(L.nmodl_scatter_layout(C.c_void_p(idx_in), n, n_nodes, C.c_void_p(counts),
                                        C.c_void_p(nb.node_offsets_full), C.c_void_p(scratch), C.c_void_p(nb.perm),
                                        C.c_void_p(nb.rank), C.c_void_p(bad), C.c_void_p(s.handle)),
                 "scatter_layout")
        self._mark("bind:sort")
        nb.node_index = nb.alloc(4 * n)
        rt.check(L.nmodl_permute_i32(C.c_void_p(idx_in), C.c_void_p(nb.node_index), C.c_void_p(nb.perm), n,
                                     C.c_void_p(s.handle)), "permute_i32")
        if shared is not None:
            nb.node_v, nb.node_rhs, nb.node_d = shared.node_v, shared.node_rhs, shared.node_d
            nb.shared = shared
        else:
            nb.node_v = nb.alloc(8 * n_nodes)
            rt.h2d(nb.node_v, node_v.ctypes.data, 8 * n_nodes, s)
            nb.node_rhs = nb.alloc(8 * n_nodes)
            nb.node_d = nb.alloc(8 * n_nodes)
            for ptr, host in ((nb.node_rhs, node_rhs), (nb.node_d, node_d)):
                if host is None:
                    rt.memset(ptr, 0, 8 * n_nodes, s)
                else:
                    h = np.ascontiguousarray(host, dtype=np.float64)
                    rt.h2d(ptr, h.ctypes.data, 8 * n_nodes, s)
        # segments: the nodes that own at least one instance, in node order;
        # the reduction touches only those (sparse populations such as one
        # channel per soma leave most compartments alone).  Tiles: target 3/4
        # of the shared-memory capacity so a tile rarely spills to the
        # global-memory reduction path when a segment straddles a boundary,
        # but keep >= 4 tiles per SM so small populations still fill the GPU.
        # Both are built on the device (nmodl_node_segments; host
        # restatement: tile_nodes_for) -- only two counts come back.
        if tile is None:
            T = self.node_tile(n)
        else:
            T = int(tile)
        n_marks = -(-max(n, 1) // T)
        nb.seg_node = nb.alloc(4 * max(1, n_nodes))
        nb.seg_offsets = nb.alloc(8 * (n_nodes + 1))
        nb.tile_segs = nb.alloc(8 * (n_marks + 1))
        counts = nb.alloc(16)
        rt.check(L.nmodl_node_segments(C.c_void_p(nb.node_offsets_full), n_nodes, n, T, C.c_void_p(nb.seg_node),
                                       C.c_void_p(nb.seg_offsets), C.c_void_p(nb.tile_segs), C.c_void_p(counts),
                                       C.c_void_p(s.handle)), "node_segments")
        nb._pending = (counts, bad)
        return nb

    @staticmethod
    def _enqueue_counts(nb: NodeBinding) -> None:
        """Copy the layout's two counts and the range flag to the host (async)."""
        counts, bad = nb._pending
        nb._cnt = np.empty(2, dtype=np.int64)
        nb._bad = np.empty(1, dtype=np.int32)
        rt.d2h(nb._cnt.ctypes.data, counts, 16, nb.stream)
        rt.d2h(nb._bad.ctypes.data, bad, 4, nb.stream)

    def _apply_counts(self, nb: NodeBinding) -> None:
        """After the counts landed: segment / tile counts, one-per-node flag."""
        nb._host_keep = None
        nb.stream = self.stream
        if nb._bad[0] != 0x7FFFFFFF:
            raise ValueError(f"node_index out of range at instance {int(nb._bad[0])}")
        nb.n_segs = int(nb._cnt[0])
        nb.n_tiles = int(nb._cnt[1]) - 1
        nb.seg_unique = 1 if nb.n_segs == nb.n else 0  # every occupied node holds exactly one instance

    def _finish_nodes(self, dev: DeviceInstanceData, nb: NodeBinding) -> NodeBinding:
        self._enqueue_counts(nb)
        nb.stream.sync()
        self._apply_counts(nb)
        s = nb.stream
        self._mark("bind:segments_tiles")
        # reorder every instance array into node-sorted order (on the device):
        # gather into a fresh arena, then retire the old one (no copy back)
        dev.reorder(nb.perm, s)
        self._mark("bind:reorder")
        dev.nodes = nb
        return nb

    def gather_voltage(self, dev: DeviceInstanceData) -> None:
        """v[i] = node_v[node_index[i]] in the (node-sorted) device store."""
        nb = dev.nodes
        rt.check(rt.lib().nmodl_gather_v(C.c_void_p(nb.node_v), C.c_void_p(nb.node_index), C.c_void_p(dev.ptr["v"]),
                                         dev.n, C.c_void_p(self.stream.handle)), "gather_v")
        dev.dirty.add("v")

    @staticmethod
    def share_slot(dst: DeviceInstanceData, dst_slot: str, src: DeviceInstanceData, src_slot: str) -> None:
        """Ion coupling: make `dst`'s slot the very array `src` writes (e.g.
        Ca_HVA's ica read by CaDynamics_E2).  Both stores must hold the same
        instances in the same order (same node_index, hence same sort); the
        producer's launch must precede the consumer's in each timestep.  The
        reference keeps one store per mechanism (modlc/layout.py:124-128);
        sharing is the device-side equivalent of NEURON's ion arrays."""
        if dst.n != src.n:
            raise ValueError("shared ion slots need equal instance counts")
        if (dst.nodes is None) != (src.nodes is None) or (
            dst.nodes is not None and not np.array_equal(dst.nodes.perm_host, src.nodes.perm_host)
        ):
            raise ValueError("shared ion slots need identical instance order")
        dst.ptr[dst_slot] = src.ptr[src_slot]
        dst.shared_slots = getattr(dst, "shared_slots", set()) | {dst_slot}
        dst.dirty.add(dst_slot)  # holds the producer's values now: download it

    def node_arrays(self, dev: DeviceInstanceData) -> dict:
        nb = dev.nodes
        out = {}
        for name in ("node_rhs", "node_d", "node_v"):
            arr = np.empty(nb.n_nodes)
            rt.d2h(arr.ctypes.data, getattr(nb, name), arr.nbytes, self.stream)
            out[name] = arr
        for name, ptr, dt in (("perm", nb.perm, np.int64), ("rank", nb.rank, np.int64),
                              ("node_index_sorted", nb.node_index, np.int32)):
            arr = np.empty(nb.n, dtype=dt)
            rt.d2h(arr.ctypes.data, ptr, arr.nbytes, self.stream)
            out[name] = arr
        offs = np.empty(nb.n_nodes + 1, dtype=np.int64)
        rt.d2h(offs.ctypes.data, nb.node_offsets_full, offs.nbytes, self.stream)
        out["offsets"] = offs
        self.stream.sync()
        return out

    def _unpermute_into(self, dev, data, names=None, acc=True) -> None:
        nb = dev.nodes
        L = rt.lib()
        s = self.stream
        tmp = rt.DeviceBuffer(8 * dev.n)
        # per-instance voltage is the gathered node voltage
        rt.check(L.nmodl_gather_v(C.c_void_p(nb.node_v), C.c_void_p(nb.node_index), C.c_void_p(dev.ptr["v"]),
                                  dev.n, C.c_void_p(s.handle)), "gather_v")
        # one stream: each permute waits for the previous copy out of `tmp`,
        # the host waits once at the end
        names = list(dev.names) if names is None else list(names)
        for name in names + (["i_acc", "g_acc"] if acc else []):
            rt.check(L.nmodl_permute(C.c_void_p(dev.ptr[name]), C.c_void_p(tmp.ptr), C.c_void_p(nb.perm), dev.n, 1,
                                     C.c_void_p(s.handle)), "unpermute")
            dst = data.acc[name] if name in ("i_acc", "g_acc") else data.arrays[name]
            rt.d2h(dst.ctypes.data, tmp.ptr, 8 * dev.n, s)
        s.sync()


def tile_nodes_for(offsets: np.ndarray, tile: int) -> np.ndarray:
    """CTA tiles of whole segments (`offsets` = segment start offsets plus the
    total), ~`tile` instances each.

    Boundary nodes are the first node whose segment starts at or after each
    multiple of `tile`; a segment larger than a tile becomes its own tile
    (the kernel then reduces it from global memory instead of shared).
    """
    n = int(offsets[-1])
    n_nodes = len(offsets) - 1
    if n_nodes == 0:
        return np.zeros(1, dtype=np.int64)
    marks = np.arange(0, max(n, 1), tile, dtype=np.int64)
    starts = np.searchsorted(offsets[:-1], marks, side="left")
    bounds = np.unique(np.concatenate([[0], starts, [n_nodes]])).astype(np.int64)
    return bounds


class PopulationGroup:
    """Several node_index populations stepped by ONE launch (a population
    group, codegen_cuda.emit_group): `chains` is a list of chains of
    (CudaRunner, DeviceInstanceData); each chain owns a contiguous CTA range,
    its members run in order over the same instance-to-thread map (a later
    member reads what an earlier one wrote for the same instance: the
    Ca_HVA ica -> CaDynamics_E2 coupling).  Members must be one-instance-
    per-node populations (their node binding has seg_unique 1 or 2); each
    keeps its own store, status word and build options, and runs the same
    generated code as its standalone kernel, so results are bit-identical.
    Errors are reported through the members' runners (`check`)."""

    def __init__(self, name: str, chains, kind: str = "unique"):
        """kind="direct": direct (no node_index) populations, each running its
        fused step kernel's code; members may be (runner, dev, options) to
        build a member with other launch options than its runner (chained
        direct members need one ilp).  Every CTA of the resident grid runs
        every member in turn."""
        from .build import build_group

        self.name = name
        self.kind = kind
        self.chains = [[tuple(m[:2]) for m in ch] for ch in chains]
        member_opts = [[(m[0].ir, m[2] if len(m) > 2 else m[0].options) for m in ch] for ch in chains]
        runners = [r for ch in self.chains for r, _ in ch]
        if not runners:
            raise ValueError("empty population group")
        flags = {r.flags for r in runners}
        if len(flags) != 1:
            raise ValueError("population group members need one Jacobian mode")
        self.flags = flags.pop()
        self.device = runners[0].device
        self.gb = build_group(name, member_opts, kind=kind)
        self.lib = C.CDLL(str(self.gb.so_path))
        g = self.gb.symbol
        self.ilp = {ci: (ch[0][2].ilp if len(ch[0]) > 2 else ch[0][0].options.ilp) for ci, ch in enumerate(chains)}
        fields = [(f"md{ci}_{mi}", r.Struct) for ci, ch in enumerate(self.chains) for mi, (r, _) in enumerate(ch)]
        fields.append(("cta", C.c_longlong * (len(self.chains) + 1)))
        self.Args = type(f"{g}_args", (C.Structure,), {"_fields_": fields})
        size_fn = getattr(self.lib, f"{g}_args_size")
        size_fn.restype = C.c_longlong
        if size_fn() != C.sizeof(self.Args):
            raise RuntimeError(f"ABI mismatch for group {g}: C {size_fn()} vs ctypes {C.sizeof(self.Args)}")
        self.fn = getattr(self.lib, f"{g}_step_unique" if kind == "unique" else f"{g}_step_group")
        self.fn.restype = C.c_int
        self.fn.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int]
        self.block = runners[0].options.block
        self.ctas = None
        if kind == "direct":
            f = getattr(self.lib, f"{g}_group_ctas")
            f.restype = C.c_int
            rt.set_device(self.device)
            self.ctas = max(1, int(f()))

    def _chain_ctas(self) -> list[int]:
        if self.kind == "unique":  # one instance per thread, as many CTAs as that takes
            return [(max(dev.n for _, dev in ch) + self.block - 1) // self.block for ch in self.chains]
        # direct: every CTA of the persistent grid runs every member in turn
        need = max((max(dev.n for _, dev in ch) + self.ilp[ci] * self.block - 1) // (self.ilp[ci] * self.block)
                   for ci, ch in enumerate(self.chains))
        return [0] * (len(self.chains) - 1) + [max(1, min(self.ctas, need))]

    def args(self):
        vals = []
        for ch in self.chains:
            for r, dev in ch:
                if self.kind == "unique" and (dev.nodes is None or dev.nodes.seg_unique not in (1, 2)):
                    raise ValueError(f"{r.mb.symbol}: group members need a one-instance-per-node binding")
                if self.kind == "direct" and dev.nodes is not None:
                    raise ValueError(f"{r.mb.symbol}: direct group members must not be node-bound")
                vals.append(r._struct(dev))
        cta = [0]
        for c in self._chain_ctas():
            cta.append(cta[-1] + c)
        return self.Args(*vals, (C.c_longlong * len(cta))(*cta))

    def launch(self, stream: "rt.Stream", steps: int = 1) -> None:
        """Enqueue `steps` group launches on `stream` (no sync, no checks)."""
        a = self.args()
        for ch in self.chains:
            for r, dev in ch:
                dev.dirty |= r._writes["step_nodes" if self.kind == "unique" else "step"]
        rt.set_device(self.device)
        rt.check(self.fn(C.byref(a), int(steps), C.c_void_p(stream.handle), self.flags), f"launch group {self.name}")

    def check(self) -> None:
        for ch in self.chains:
            for r, dev in ch:
                r.check(dev)


def _unread_arrays(runner: "CudaRunner", data, kernels) -> list[str]:
    """Arrays of `data` that none of `kernels` reads or writes (parameters the
    mechanism declares but never uses): their values never reach the device
    and never come back, so a call need not upload them -- only their
    finiteness matters (the reference scans every array after every kernel,
    interp.py:538-545).  Written arrays are always uploaded: a conditional
    write must leave the other instances' values as they were."""
    touched = set()
    for k in kernels:
        touched |= set(runner.abi.kernels[k]["loads"]) | set(runner.abi.kernels[k]["stores"])
    return [n for n in data.arrays if n not in touched and n != "v"]


class _HostScan:
    """First non-finite index of host arrays, on a worker thread (numpy
    releases the GIL) while the device steps."""

    def __init__(self, arrays: dict):
        import threading

        self.arrays = arrays
        self.bad: dict[str, int] = {}
        self.thread = threading.Thread(target=self._run, daemon=True)
        self.thread.start()

    def _run(self) -> None:
        for name, a in self.arrays.items():
            if not np.isfinite(a).all():
                self.bad[name] = int(np.flatnonzero(~np.isfinite(a))[0])

    def join(self) -> dict:
        self.thread.join()
        return self.bad


def simulate(layout, data, steps: int, jac_mode: str = "exact", on_step=None, runner: CudaRunner | None = None,
             _skip_unread: bool = True):
    """GPU twin of modlc.interp.simulate (interp.py:640-655): one upload,
    initialize, `steps` fused state+current launches, one download."""
    runner = runner or CudaRunner(layout, jac_mode=jac_mode)
    # i_acc / g_acc are outputs only (written with `=` by nrn_cur, read by
    # nothing): not uploaded; downloaded once a launch has written them.
    # Arrays no kernel reads are not uploaded either; a host thread checks
    # them for non-finite values while the device steps, and if it finds one
    # the call is redone with the whole store (the reference reports it after
    # the first kernel).
    unread = _unread_arrays(runner, data, ("initialize", "step")) if (_skip_unread and on_step is None) else []
    scan = _HostScan({n: data.arrays[n] for n in unread}) if unread else None
    dev = runner.to_device(data, skip=("i_acc", "g_acc") + tuple(unread))
    err = None
    try:
        runner.run_kernel(dev, "initialize", 1)
        if on_step is None:
            runner.run_kernel(dev, "step", steps)
        else:
            for step in range(steps):
                runner.run_kernel(dev, "step", 1)
                runner.to_host(dev, data, only_dirty=True)
                on_step(step, data)
    except InterpError as exc:
        err = exc
    if scan is not None and scan.join():
        return simulate(layout, data, steps, jac_mode, on_step, runner, _skip_unread=False)
    runner.to_host(dev, data, only_dirty=True)
    if err is not None:
        raise err
    return data


def simulate_nodes(layout, data, steps: int, node_index, node_v, node_rhs=None, node_d=None,
                   jac_mode: str = "exact", runner: CudaRunner | None = None, timings: dict | None = None,
                   reset: bool = True, _skip_unread: bool = True):
    """node_index run of one mechanism population (builder extension).

    Per timestep: v_i = node_v[node_index[i]]; nrn_state; nrn_cur; then
    node_rhs[k] = 0 - sum_i i_acc[i] and node_d[k] = 0 + sum_i g_acc[i] over
    the instances i of node k in ascending instance order (deterministic; the
    oracle restatement is oracle/nodes_np.py): the node arrays are rebuilt
    every step, as a cable solver's matrix is.  With ``reset=False`` they
    start from node_rhs/node_d and accumulate across steps instead.
    Instances are initialised with the gathered voltage.  Returns (data,
    node_rhs, node_d); `data` is updated in place in instance order.
    `timings` (optional dict) receives wall-clock seconds per phase.
    """
    import time

    clock = time.perf_counter
    t = {}
    t0 = clock()
    runner = runner or CudaRunner(layout, jac_mode=jac_mode)
    node_v = np.ascontiguousarray(node_v, dtype=np.float64)
    # the node layout (node_index upload, stable sort, segments, tiles) is
    # built on a second stream while the instance store uploads
    aux = runner.aux_stream()
    if reset:  # nodes without instances hold 0; the others are assigned every step
        node_rhs = node_d = None
    prep = runner.prepare_nodes(int(data.n), node_index, node_v, node_rhs, node_d, stream=aux)
    # v is never uploaded (every instance's voltage is its node's); i_acc /
    # g_acc are outputs only; arrays no kernel reads are scanned on the host
    # instead (see simulate)
    unread = _unread_arrays(runner, data, ("initialize", "step_nodes")) if _skip_unread else []
    scan = _HostScan({n: data.arrays[n] for n in unread}) if unread else None
    dev = runner.to_device(data, skip=("v", "i_acc", "g_acc") + tuple(unread))
    t["upload"] = clock() - t0
    t0 = clock()
    nb = runner.bind_nodes(dev, node_index, prepared=prep)
    nb.assign = 1 if reset else 0
    runner.gather_voltage(dev)
    if not np.isfinite(node_v).all():
        # a non-finite node voltage is a pre-existing non-finite v for the
        # first instance (in caller order) that reads it
        dev.prebad["v"] = int(np.flatnonzero(~np.isfinite(node_v[np.asarray(node_index)]))[0])
    t["bind_nodes"] = clock() - t0
    err = None
    try:
        t0 = clock()
        runner.run_kernel(dev, "initialize", 1)
        t["initialize"] = clock() - t0
        t0 = clock()
        runner.run_kernel(dev, "step_nodes", steps)
        t["steps"] = clock() - t0
    except InterpError as exc:
        err = exc
    if scan is not None and scan.join():
        return simulate_nodes(layout, data, steps, node_index, node_v, node_rhs, node_d, jac_mode, runner, timings,
                              reset, _skip_unread=False)
    t0 = clock()
    runner.to_host(dev, data, only_dirty=True)
    out = {}
    for name in ("node_rhs", "node_d"):
        arr = np.empty(nb.n_nodes)
        rt.d2h(arr.ctypes.data, getattr(nb, name), arr.nbytes, runner.stream)
        out[name] = arr
    runner.stream.sync()
    t["download"] = clock() - t0
    if err is not None:
        raise err
    if timings is not None:
        timings.update(t)
    return data, out["node_rhs"], out["node_d"]
