"""Synthetic cortical column (BASELINE configs[4]): every mechanism of a cell
population stepped together, sharded by cell.

Builder-defined workload (the reference has no cells, nodes or ion sharing;
SPEC.md:441, modlc/layout.py:124-128).  Cell c owns compartments (nodes)
[c*(1+D), (c+1)*(1+D)); node 0 of a cell is the soma.

  soma, one instance per cell:  NaTs2_t, K_Pst, Ca_HVA, CaDynamics_E2, SKv3_1
  soma + every dendrite:        Ih
  S synapses per cell:          ProbAMPANMDA_EMS on random compartments of the cell

Per timestep every population runs one fused kernel that gathers v from the
shared node voltage and runs nrn_state + nrn_cur; the currents are folded
into the shared node rhs/d in LAUNCH_ORDER (Ih, the soma populations, the
synapses), each population in instance order.  The node rhs/d are rebuilt
every timestep (a cable solver's matrix setup): Ih, which has one instance
on every compartment, goes first and assigns them (rhs = 0 - i, d = 0 + g);
the other populations accumulate.  ColumnShard's schedules arrange the
launches differently (one stream, side streams, one grouped launch) but
perform the same operations per node in the same order.
CaDynamics_E2 reads Ca_HVA's `ica` array directly (ion coupling; Ca_HVA runs
first), which is what NEURON's shared ion arrays do.  Instance data are drawn with
`init_range`, so a shard of cells [lo, hi) holds exactly the instances the
single-GPU column holds for those cells: shard checksums add up across ranks.
"""

from __future__ import annotations

import os

import zlib
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .instance import V_RANGE, init_range
from .ir import MechIR

FIXTURES = Path(__file__).resolve().parent.parent / "fixtures" / "ir"
SOMA_MECHS = ("NaTs2_t", "K_Pst", "Ca_HVA", "cadyn", "SKv3_1")
LAUNCH_ORDER = ("Ih", "NaTs2_t", "K_Pst", "Ca_HVA", "cadyn", "SKv3_1", "ProbAMPANMDA_EMS")
COUPLINGS = (("cadyn", "ica", "Ca_HVA", "ica"),)  # consumer slot <- producer slot


@dataclass(frozen=True)
class ColumnSpec:
    n_cells: int = 100_000
    dend_per_cell: int = 20
    syn_per_cell: int = 100
    seed: int = 42

    @property
    def nodes_per_cell(self) -> int:
        return 1 + self.dend_per_cell

    def instances_per_cell(self, stem: str) -> int:
        if stem in SOMA_MECHS:
            return 1
        if stem == "Ih":
            return self.nodes_per_cell
        if stem == "ProbAMPANMDA_EMS":
            return self.syn_per_cell
        raise KeyError(stem)

    def cell_cost(self) -> float:
        """Bytes one cell moves per timestep (for cost-balanced sharding)."""
        per_inst = {"ProbAMPANMDA_EMS": 171.0, "Ih": 56.0, "SKv3_1": 64.0, "cadyn": 72.0}
        return sum(self.instances_per_cell(m) * per_inst.get(m, 80.0) for m in LAUNCH_ORDER)


def shard_layout(spec: ColumnSpec, cell_lo: int, cell_hi: int) -> dict:
    """Per mechanism: (global instance range, node_index local to the shard);
    plus the shard's node voltages."""
    npc = spec.nodes_per_cell
    ncell = cell_hi - cell_lo
    cells = np.arange(cell_lo, cell_hi, dtype=np.int64)
    out = {}
    for stem in LAUNCH_ORDER:
        k = spec.instances_per_cell(stem)
        lo, hi = cell_lo * k, cell_hi * k
        local_cell = np.repeat(np.arange(ncell, dtype=np.int64), k)
        if stem in SOMA_MECHS:
            comp = np.zeros(ncell * k, dtype=np.int64)
        elif stem == "Ih":
            comp = np.tile(np.arange(npc, dtype=np.int64), ncell)
        else:  # synapses: compartment drawn per global synapse id (shard-independent)
            bg = np.random.PCG64(np.random.SeedSequence([spec.seed, zlib.crc32(b"syn_comp")]))
            bg.advance(lo)
            u = np.random.Generator(bg).random(hi - lo)  # one 64-bit draw per synapse
            comp = np.minimum((u * npc).astype(np.int64), npc - 1)
        out[stem] = (lo, hi, (local_cell * npc + comp).astype(np.int32))
    bg = np.random.PCG64(np.random.SeedSequence([spec.seed, zlib.crc32(b"node_v")]))
    bg.advance(cell_lo * npc)
    node_v = np.random.Generator(bg).uniform(*V_RANGE, ncell * npc)
    return {"mechs": out, "node_v": node_v, "n_nodes": ncell * npc}


def host_stores(spec: ColumnSpec, cell_lo: int, cell_hi: int) -> dict:
    """{stem: HostInstanceData} of cells [cell_lo, cell_hi) (init_range: the
    single-GPU column's instances for exactly those cells)."""
    lay = shard_layout(spec, cell_lo, cell_hi)
    irs = load_irs()
    return {stem: init_range(irs[stem], lay["mechs"][stem][0], lay["mechs"][stem][1], spec.seed)
            for stem in LAUNCH_ORDER}


def load_irs() -> dict:
    return {stem: MechIR.load(FIXTURES / f"{stem}.json") for stem in LAUNCH_ORDER}


SCHEDULES = ("sequential", "concurrent", "grouped")


class ColumnShard:
    """All populations of cells [cell_lo, cell_hi) resident on one GPU.

    Per timestep every population runs once and folds its currents into the
    shared node rhs/d in LAUNCH_ORDER (Ih, the soma populations -- Ca_HVA
    before CaDynamics_E2, which reads its ica -- then the synapses).  The
    `schedule` only changes how the launches are arranged -- every schedule
    performs the same operations on every node in the same order, so all
    give bit-identical results (tests/test_gpu_column.py):

    * "sequential": one launch per population on one stream;
    * "concurrent": the one-per-cell soma populations on side streams,
      leaving their currents in i_acc/g_acc (seg_unique 2); one combine
      kernel folds them into the soma nodes in order;
    * "grouped": the soma populations as ONE launch (runner.PopulationGroup,
      chains NaTs2_t | K_Pst | Ca_HVA -> CaDynamics_E2 | SKv3_1) on a side
      stream beside Ih, then the combine and the synapses: 4 launches per
      timestep instead of 8 -- what matters when a rank holds few cells
      (strong scaling)."""

    def __init__(self, spec: ColumnSpec, cell_lo: int, cell_hi: int, options_for=None,
                 concurrent_soma: bool = False, reset: bool = True, host: dict | None = None,
                 runners: dict | None = None, grouped_soma: bool = False, schedule: str | None = None,
                 layout: dict | None = None):
        from . import runtime as rt
        from .runner import CudaRunner, NodeArrays

        if schedule is None:
            schedule = "grouped" if grouped_soma else ("concurrent" if concurrent_soma else "sequential")
        if schedule not in SCHEDULES:
            raise ValueError(f"schedule must be one of {SCHEDULES}")
        self.spec = spec
        self.reset = reset
        self.cells = (cell_lo, cell_hi)
        # `layout`: shard_layout(spec, cell_lo, cell_hi) computed by the caller
        # (the node_index / node_v inputs, like `host` for the stores)
        lay = shard_layout(spec, cell_lo, cell_hi) if layout is None else layout
        if lay["n_nodes"] != (cell_hi - cell_lo) * spec.nodes_per_cell:
            raise ValueError("layout is for another shard")
        self.layout = lay
        irs = load_irs()
        self.runners, self.devs, self.node_index = {}, {}, {}
        first = None
        for stem in LAUNCH_ORDER:
            opts = options_for(stem) if options_for else None
            r = runners[stem] if runners is not None else CudaRunner(irs[stem], options=opts)
            if first is None:
                first = r
            else:
                r.stream = first.stream  # one stream: launch order == step order
            self.runners[stem] = r
        self.stream = first.stream
        self.nodes = NodeArrays(lay["node_v"], stream=self.stream)
        for stem in LAUNCH_ORDER:
            lo, hi, idx = lay["mechs"][stem]
            r = self.runners[stem]
            data = host[stem] if host is not None else init_range(irs[stem], lo, hi, spec.seed)
            dev = r.to_device(data)
            r.bind_nodes(dev, idx, shared=self.nodes)
            r.gather_voltage(dev)
            self.devs[stem] = dev
            self.node_index[stem] = idx
        for dst, dslot, src, sslot in COUPLINGS:
            self.runners[dst].share_slot(self.devs[dst], dslot, self.devs[src], sslot)
        for stem in LAUNCH_ORDER:
            self.runners[stem].run_kernel(self.devs[stem], "initialize", 1)
        # per-step node reset: the first population assigns rhs/d when it has
        # one instance on every node; otherwise a memset starts each step
        fb = self.devs[LAUNCH_ORDER[0]].nodes
        self._assign_first = bool(reset) and fb.seg_unique == 1 and fb.n == self.nodes.n_nodes
        fb.assign = 1 if self._assign_first else 0
        unique = all(self.devs[m].nodes.seg_unique == 1 for m in SOMA_MECHS)
        if schedule != "sequential" and not unique:
            schedule = "sequential"
        self.schedule = schedule
        self.grouped = schedule == "grouped"
        self.concurrent = schedule != "sequential"
        self._soma_order = [m for m in LAUNCH_ORDER if m in SOMA_MECHS]
        # the combine rides programmatic dependent launch when the kernels do
        # and no memset sits between it and the kernel before it on the stream
        self._combine_pdl = (all(r.options.pdl for r in self.runners.values()) and self._assign_first
                             and os.environ.get("NMODL_COMBINE_PDL", "1") == "1")
        import ctypes as C

        if self.concurrent:
            self._fork = rt.Event()
            for m in SOMA_MECHS:
                self.devs[m].nodes.seg_unique = 2  # currents stay in i_acc/g_acc
            k = len(self._soma_order)
            self._iptr = (C.c_void_p * k)(*[self.devs[m].ptr["i_acc"] for m in self._soma_order])
            self._gptr = (C.c_void_p * k)(*[self.devs[m].ptr["g_acc"] for m in self._soma_order])
        if schedule == "concurrent":
            self._side = {m: rt.Stream() for m in SOMA_MECHS}
            self._ca = rt.Event()
            self._join = {m: rt.Event() for m in SOMA_MECHS}
        if self.grouped:
            from .runner import PopulationGroup

            def member(m):
                return (self.runners[m], self.devs[m])

            chains = [[member(m)] for m in self._soma_order if m not in ("Ca_HVA", "cadyn")]
            chains.insert(self._soma_order.index("Ca_HVA"), [member("Ca_HVA"), member("cadyn")])
            self.group = PopulationGroup("soma", chains)
            self._group_stream = rt.Stream()
            self._group_done = rt.Event()

    @property
    def group_members(self) -> list[str]:
        """Populations stepped inside the population-group launch."""
        if not self.grouped:
            return []
        return [m for m in LAUNCH_ORDER if m in SOMA_MECHS]

    @property
    def n_instances(self) -> int:
        return sum(d.n for d in self.devs.values())

    def _reset_nodes(self) -> None:
        """Start of a timestep: node rhs/d rebuilt from zero (cable-solver
        matrix setup; oracle/column_np.py reset=True)."""
        if self.reset and not self._assign_first:
            from . import runtime as rt

            nbytes = 8 * self.nodes.n_nodes
            rt.memset(self.nodes.node_rhs, 0, nbytes, self.stream)
            rt.memset(self.nodes.node_d, 0, nbytes, self.stream)

    def _combine_soma(self, L, C) -> None:
        from . import runtime as rt

        first = self.devs[self._soma_order[0]]
        nb = first.nodes
        # programmatic dependent launch behind the kernel before it on the main
        # stream (Ih, or the previous step's synapses), which writes none of the
        # soma currents: their loads overlap its tail, the fold waits for it
        flags = 1 if self._combine_pdl else 0
        rt.check(L.nmodl_combine_unique_ex(C.c_void_p(nb.node_rhs), C.c_void_p(nb.node_d), C.c_void_p(nb.node_index),
                                           first.n, self._iptr, self._gptr, len(self._soma_order), flags,
                                           C.c_void_p(self.stream.handle)), "combine_unique")

    def launch(self, steps: int = 1) -> None:
        import ctypes as C

        from . import runtime as rt

        L = rt.lib()
        main = self.stream
        soma_at = min(LAUNCH_ORDER.index(m) for m in SOMA_MECHS)
        before = [m for m in LAUNCH_ORDER[:soma_at]]
        after = [m for m in LAUNCH_ORDER[soma_at:] if m not in SOMA_MECHS]
        for _ in range(steps):
            if self.schedule == "sequential":
                self._reset_nodes()
                for stem in LAUNCH_ORDER:
                    self.runners[stem].launch(self.devs[stem], "step_nodes", 1)
                continue
            self._reset_nodes()
            self._fork.record(main)
            if self.schedule == "grouped":
                side = self._group_stream
                rt.stream_wait(side, self._fork)
                self.group.launch(side, 1)
                self._group_done.record(side)
                joins = [self._group_done]
            else:
                for m in self._soma_order:
                    side = self._side[m]
                    rt.stream_wait(side, self._fork)
                    if m == "cadyn":
                        rt.stream_wait(side, self._ca)  # reads this step's Ca_HVA ica
                    r = self.runners[m]
                    r.stream = side
                    r.launch(self.devs[m], "step_nodes", 1)
                    r.stream = main
                    if m == "Ca_HVA":
                        self._ca.record(side)
                    self._join[m].record(side)
                joins = [self._join[m] for m in self._soma_order]
            # folds in LAUNCH_ORDER: the populations before the soma group,
            # the soma group (combine, in order), the populations after it
            for stem in before:
                self.runners[stem].launch(self.devs[stem], "step_nodes", 1)
            for e in joins:
                rt.stream_wait(main, e)
            self._combine_soma(L, C)
            for k, stem in enumerate(after):
                # the first population after the combine reads nothing the combine
                # writes except the node rhs/d it folds into: its loads and maths
                # may start while the combine runs (programmatic late wait)
                self.runners[stem].launch(self.devs[stem], "step_nodes", 1, late_wait=(k == 0))

    def kernels_per_step(self) -> int:
        """Our kernels per timestep (memsets not counted)."""
        return {"sequential": len(LAUNCH_ORDER), "concurrent": len(LAUNCH_ORDER) + 1,
                "grouped": len(LAUNCH_ORDER) - len(SOMA_MECHS) + 2}[self.schedule]

    def check(self) -> None:
        for stem in LAUNCH_ORDER:
            self.runners[stem].check(self.devs[stem])

    def launch_bytes(self) -> int:
        from .traffic import launch_bytes

        total = 0
        for stem in LAUNCH_ORDER:
            d = self.devs[stem]
            total += launch_bytes(self.runners[stem].abi, d.n, "step_nodes", d.nodes.n_segs)
        return total

    def checksums(self) -> np.ndarray:
        from .parallel import device_checksums

        rows = []
        for stem in LAUNCH_ORDER:
            r, d = self.runners[stem], self.devs[stem]
            rows.append(device_checksums(r, d, [s for s in r.abi.slots if s in d.ptr] + ["i_acc", "g_acc"]))
        return np.concatenate(rows)


def simulate_column(spec: ColumnSpec, steps: int, cell_lo: int = 0, cell_hi: int | None = None,
                    host: dict | None = None, options_for=None, runners: dict | None = None,
                    reset: bool = True, concurrent_soma: bool = False, grouped_soma: bool = False,
                    schedule: str | None = None, layout: dict | None = None):
    """Public column call (configs[4]): upload the stores of cells
    [cell_lo, cell_hi) (`host`, e.g. from host_stores(), ideally pinned),
    build the shared node layout on the device, nrn_init, `steps` timesteps
    of all populations, then download every store (in place, instance order)
    and the node arrays.  Returns (host, {"node_rhs", "node_d", "node_v"},
    shard).  Pass the previous call's `shard.runners` to reuse the loaded
    kernels, and `layout` (shard_layout(spec, cell_lo, cell_hi): the node_index
    and node_v inputs) to skip generating it."""
    cell_hi = spec.n_cells if cell_hi is None else cell_hi
    if host is None:
        host = host_stores(spec, cell_lo, cell_hi)
    shard = ColumnShard(spec, cell_lo, cell_hi, options_for, concurrent_soma=concurrent_soma, reset=reset,
                        host=host, runners=runners, grouped_soma=grouped_soma, schedule=schedule, layout=layout)
    shard.launch(steps)
    shard.check()
    for stem in LAUNCH_ORDER:
        shard.runners[stem].to_host(shard.devs[stem], host[stem], only_dirty=True)
    nodes = shard.nodes.download(shard.stream)
    return host, nodes, shard
