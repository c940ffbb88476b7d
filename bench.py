"""Benchmark: nrn_state + nrn_cur instance-steps/s (fp64) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload synapse10m|hh1m|hh10m|bbp20m|kinetic1m|column]
                    [--no-also] [--no-e2e] [--no-cpu] [--no-sustained]

One JSON line on rank 0.  A "step" is one timestep of the hot path over the
whole synthetic population on every rank: one fused nrn_state+nrn_cur launch
per mechanism (for node_index workloads also the voltage gather and the
in-order rhs/d reduction, inside the same kernel).  Workloads are the
BASELINE.json configs:

  synapse10m  configs[1]  ProbAMPANMDA_EMS restated (4 cnexp states, Mg block,
                          numeric conductance), 10M instances / GPU, random
                          node_index onto 1M nodes (default; inputs >> L2)
  hh1m        configs[0]  hh (cnexp, analytic conductance), 1M instances / GPU
                          (working set ~ L2: L2 flushed between timed steps)
  hh10m       configs[0]'s mechanism at 10M instances (inputs >> L2): the
                          same kernel where the 1M size floor does not bind
  bbp20m      configs[2]  NaTs2_t, K_Pst, Ca_HVA, SKv3_1, Ih, CaDynamics_E2;
                          20M instances / GPU split evenly (6 launches / step)
  bbp20m_grouped          the same step as ONE population-group launch
  kinetic1m   configs[3]  6-state KINETIC Na (runtime LU k=6) + cdp5-style
                          Newton k=5 with LU, 1M instances each
  kinetic1m_grouped       the kinetic pair as ONE population-group launch
  kinetic10m  the same kernels at 10M instances each (inputs >> L2): where
                          the 1M launch-size floor does not bind
  column      configs[4]  100k-cell synthetic column, cells split over ranks
                          (strong scaling)

Timing: W untimed warm-up steps, then K steps replayed from one CUDA graph
bracketed by a barrier and a synchronize on both sides; CUDA events recorded
INSIDE the graph (external event-record nodes) around every population's
launch give each kernel's launch duration within the same timed replay.
Multi-GPU (torchrun): one process per GPU, each rank owns its own shard of
cells, max-over-ranks time; collectives (barrier, max time, checksum
all-gather) go through paper_1905_02241_b200.parallel (NCCL bound by the
runtime library; no PyTorch anywhere).  `--impl reference` times the
reference's own CPU implementation (its emitted scalar C, oracle/_ref,
compiled -O3 -march=native, all host threads) on a bounded sample of the
same workload, rank 0 only; the ours-arm `cpu_baseline` is the same
measurement with a smaller step count.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

BASELINE = json.loads((ROOT / "BASELINE.json").read_text())
METRIC = BASELINE["metric"]
UNIT = "instance-steps/s"

WORKLOADS = {
    "synapse10m": {
        "config": BASELINE["configs"][1],
        "mechs": [("ProbAMPANMDA_EMS", 10_000_000)],
        "nodes": 1_000_000,
    },
    "hh1m": {"config": BASELINE["configs"][0], "mechs": [("hh_subset", 1_000_000)], "nodes": 0},
    "hh10m": {"config": BASELINE["configs"][0] + " -- at 10M instances (inputs >> L2)",
              "mechs": [("hh_subset", 10_000_000)], "nodes": 0},
    "bbp20m": {
        "config": BASELINE["configs"][2],
        "mechs": [(m, 20_000_000 // 6) for m in ("NaTs2_t", "K_Pst", "Ca_HVA", "SKv3_1", "Ih", "cadyn")],
        "nodes": 0,
        # CaDynamics_E2 accumulates the calcium current Ca_HVA writes (same
        # compartments, same order): its `ica` slot is Ca_HVA's array
        "couplings": [("cadyn", "ica", "Ca_HVA", "ica")],
    },
    # the same six populations stepped by ONE population-group launch per
    # timestep (codegen_cuda.emit_group kind="direct"; bit-identical)
    "bbp20m_grouped": {
        "config": BASELINE["configs"][2] + " -- all six populations in one launch per step",
        "mechs": [(m, 20_000_000 // 6) for m in ("NaTs2_t", "K_Pst", "Ca_HVA", "SKv3_1", "Ih", "cadyn")],
        "nodes": 0,
        "couplings": [("cadyn", "ica", "Ca_HVA", "ica")],
        "grouped": "bbp",
    },
    "kinetic1m": {"config": BASELINE["configs"][3], "mechs": [("na6", 1_000_000), ("cdp5ish", 1_000_000)], "nodes": 0},
    "kinetic1m_grouped": {"config": BASELINE["configs"][3] + " -- both populations in one launch per step",
                          "mechs": [("na6", 1_000_000), ("cdp5ish", 1_000_000)], "nodes": 0, "grouped": "kinetic"},
    "kinetic10m": {"config": BASELINE["configs"][3] + " -- at 10M instances each (inputs >> L2)",
                   "mechs": [("na6", 10_000_000), ("cdp5ish", 10_000_000)], "nodes": 0},
    # configs[4]: strong scaling -- the column is fixed, cells are split over ranks
    "column": {"config": BASELINE["configs"][4], "mechs": [], "nodes": 0, "cells": 100_000},
}
DEFAULT_WORKLOAD = "synapse10m"


def options_for(stem: str):
    """Launch shapes / codegen picked with tools/tune.py on B200
    (profiles/tune_r01.md).  `pipe` = per-thread cp.async double buffering;
    `recip` / `div_approx` = relaxed arithmetic (reciprocal shadows, 2-ulp
    rate-code division), parity-tested at 1e-10 after 1000 steps
    (tests/test_gpu_parity.py::test_relaxed_arithmetic_within_tolerance)."""
    from paper_1905_02241_b200.codegen_cuda import CudaOptions

    tuned = {
        "ProbAMPANMDA_EMS": CudaOptions(ilp=1, fast_path=False, tile=2304, min_blocks=4),  # 2048: 0.2823, 2304: 0.2807 ms (3 reps); min_blocks=4 keeps it at <= 64 registers (4 CTAs/SM)
        "hh_subset": CudaOptions(ilp=1, pipe=True, recip=True, div_approx=True, exp_share=True,
                                 fast_redo=True),  # 0.0412 -> 0.0329 ms
        "NaTs2_t": CudaOptions(ilp=2, min_blocks=2, pipe=True, recip=True, div_approx=True, exp_share=True,
                               fast_redo=True),  # 0.0788 -> 0.0557 ms
        "K_Pst": CudaOptions(ilp=2, min_blocks=2, pipe=True, recip=True, quot=True, div_approx=True, exp_smem=True,
                             exp_share=True, fast_redo=True),  # 0.0717 -> 0.0574 ms
        "Ca_HVA": CudaOptions(ilp=2, min_blocks=2, pipe=True, recip=True, div_approx=True, fast_redo=True),  # 0.0707 -> 0.0561
        "SKv3_1": CudaOptions(ilp=2, grid_waves=4, div_approx=True, fast_redo=True),  # 0.0500 -> 0.0426 -> 0.0388 ms (r02 ilp=2)
        "Ih": CudaOptions(ilp=2, pipe=True, grid_waves=4, recip=True, div_approx=True, fast_redo=True,
                          min_blocks=4),  # 0.0474 -> 0.0392 ms; min_blocks=4: step_unique at 64 registers (column Ih 7.5 -> 6.5 us at 12.5k cells)
        "cadyn": CudaOptions(pipe=True, min_blocks=2),  # 0.0471 -> 0.0462 ms (profiles/r02/tune_small.jsonl)
        "na6": CudaOptions(ilp=1, min_blocks=2, pipe=True, fast_redo=True, lu_spec=True,
                           lu_approx=2),  # 0.0485 -> 0.0369 ms; lu_approx=2 (LU multipliers): 1M 34.8 -> 32.8 us, 10M 252 -> 240 us
        "cdp5ish": CudaOptions(ilp=1, min_blocks=2, pipe=True, div_approx=True, fast_redo=True, lu_spec=True,
                               lu_approx=1),  # 0.0583 -> 0.0390; lu_approx: 1M 41.9 -> 38.5 us, 10M 331 -> 292 us
    }
    import dataclasses

    # programmatic dependent launch for every kernel: the next step's CTAs are
    # scheduled while the previous grid drains (column 357 -> 352 us, 12.5k
    # cells 56.3 -> 54.3 us; profiles/r02/pdl_*.json); NMODL_PDL=0 turns it off
    opts = dataclasses.replace(tuned.get(stem, CudaOptions()), pdl=os.environ.get("NMODL_PDL", "1") == "1")
    # experiments: NMODL_OPT_<stem>="min_blocks=4,ilp=1" overrides fields of one mechanism's build
    extra = os.environ.get(f"NMODL_OPT_{stem}")
    if extra:
        kw = {}
        for part in extra.split(","):
            k, v = part.split("=")
            kw[k] = (v in ("1", "True", "true")) if isinstance(getattr(opts, k), bool) else int(v)
        opts = dataclasses.replace(opts, **kw)
    return opts


RELAXED_NOTE = ("fp64 throughout; rate code uses reciprocal/quotient shadows (X/(1/E) -> X*E), <=2-ulp division, "
                "shared affine exponentials (exp(aX+b) = exp(aX+b0)*exp(b-b0)) and (K_Pst) a 1-ulp shared-table exp "
                "where tuned (bench.options_for); solver cores IEEE except the kinetic LUs' quotients (<=2-ulp, one refined "
                "reciprocal per pivot: cdp5ish all, na6 the multipliers); parity 1e-10 after 1000 steps is tested for every flag")


def bench_irs():
    """(IR, options) pairs bench.py launches -- prebuilt by __graft_entry__.build()."""
    from paper_1905_02241_b200.ir import MechIR

    out = []
    for w in WORKLOADS.values():
        for stem, _ in w["mechs"]:
            ir = MechIR.load(ROOT / "fixtures" / "ir" / f"{stem}.json")
            out.append((ir, options_for(stem)))
    return out


# ---------------------------------------------------------------------------
# clocks


class ClockSampler:
    """SM clock and clock-event reasons sampled DURING the timed region
    (B200_PROFILING.md clocks line).  NVML is polled every ~1 ms from a
    thread, so even a few-millisecond timed region gets samples."""

    REASONS = {
        "hw_slowdown": 0x8,
        "sw_thermal_slowdown": 0x20,
        "hw_thermal_slowdown": 0x40,
        "hw_power_brake_slowdown": 0x80,
        "sw_power_cap": 0x4,
    }

    def __init__(self, gpu_index: int, period_s: float = 0.001):
        self.gpu = gpu_index
        self.period = period_s
        self.rows = []
        self.stop = threading.Event()
        self.thread = None

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
        except Exception as exc:  # noqa: BLE001 -- report, never fail the bench
            self.error = repr(exc)
        return self

    def _poll(self):
        nv, h = self.nv, self.h
        while not self.stop.is_set():
            try:
                self.rows.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM),
                                  nv.nvmlDeviceGetCurrentClocksEventReasons(h)))
            except Exception:  # noqa: BLE001
                pass
            time.sleep(self.period)

    def __exit__(self, *exc):
        self.stop.set()
        if self.thread is not None:
            self.thread.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": getattr(self, "max_mhz", None),
                    "reasons": ["unsampled"], "samples": 0, "error": getattr(self, "error", None)}
        reasons = set()
        for _, mask in self.rows:
            for name, bit in self.REASONS.items():
                if mask & bit:
                    reasons.add(name)
        return {
            "sm_mhz": statistics.median(r[0] for r in self.rows),
            "sm_max_mhz": self.max_mhz,
            "reasons": sorted(reasons),
            "samples": len(self.rows),
            "source": "NVML, 1 ms polling during the timed region",
        }


# ---------------------------------------------------------------------------
# distributed plumbing


class Dist:
    """One process per GPU (torchrun env: RANK / WORLD_SIZE / LOCAL_RANK).
    The process group is paper_1905_02241_b200.parallel.init_group: NCCL
    through the runtime library when every rank has its own GPU, a file
    group when ranks share one (a multi-rank smoke run on a one-GPU box),
    the identity for one rank.  No PyTorch."""

    def __init__(self, need_group: bool = True):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.device = 0
        self.group = None
        if need_group:
            from paper_1905_02241_b200.parallel import init_group

            self.group, self.device = init_group()

    @property
    def backend(self):
        return getattr(self.group, "backend", "none")

    def barrier(self):
        if self.group is not None:
            self.group.barrier()

    def allreduce(self, values, op="max"):
        if self.group is None:
            return [float(v) for v in values]
        return self.group.allreduce(values, op)

    def allgather(self, local):
        from paper_1905_02241_b200.parallel import gather_checksums

        return gather_checksums(local, self.group)

    def close(self):
        if self.group is not None:
            self.group.close()


# ---------------------------------------------------------------------------
# roofline denominators and the ncu traffic record


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.is_file():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def _fp64_peak(sm_mhz=None):
    """FP64 pipe instructions/s: the DFMA microbenchmark's measured rate
    (tools/micro/fp64_peak.cu -> profiles/fp64_peak.json), else 148 SMs x 64
    lanes x the sampled SM clock."""
    p = ROOT / "profiles" / "fp64_peak.json"
    if p.is_file():
        d = json.loads(p.read_text())
        return float(d["dfma_per_s"]), f"measured ({d.get('source', 'profiles/fp64_peak.json')})"
    mhz = sm_mhz or 1965.0
    return 148 * 64 * mhz * 1e6, f"nominal 148 SM x 64 FP64 lanes x {mhz:.0f} MHz"


def _traffic_record():
    p = ROOT / "profiles" / "ncu_traffic.json"
    return json.loads(p.read_text()) if p.is_file() else {}


def _traffic(build_keys):
    """ncu DRAM bytes (read + write) per launch of these exact builds at these
    population sizes ("<content-addressed library stem>@<instances>": the
    generated text + flags + headers), from `ncu --set full` captures of the
    same bench configuration (tools/profile_bench.py); None unless every
    build was captured."""
    rec = _traffic_record().get("by_build", {})
    total = 0.0
    for k in build_keys:
        e = rec.get(k)
        if e is None:
            return None, f"no ncu capture of build {k}"
        total += e["dram_bytes"]
    return total, "ncu --set full capture of the same build(s): " + ", ".join(
        rec[k].get("capture", "?") for k in build_keys)


def _fp64_instr(ir, n, key):
    """FP64 pipe instructions of one launch: the ncu-measured per-instance
    count of this exact build (DFMA+DMUL+DADD+DSETP+DMNMX, profiles/
    ncu_traffic.json), else the static census (analysis.fp64_ops: the
    reference census priced with the library-exact instruction sequences)."""
    e = _traffic_record().get("by_build", {}).get(key, {})
    if "fp64_instr_per_instance" in e:
        return e["fp64_instr_per_instance"] * n, "ncu-measured FP64 instructions of this build"
    from paper_1905_02241_b200.analysis import fp64_ops

    return fp64_ops(ir) * n, "static census (analysis.fp64_ops)"


def _roofline(kernel_name, bytes_per_launch, fp64, launch_ms, build_keys, sm_mhz):
    """roofline object of one kernel launch: algorithmic bytes of one launch /
    its measured duration against the measured HBM copy peak, and FP64 pipe
    instructions of one launch / duration against the measured DFMA rate.
    `fp64` = (instructions, how counted).  `bound` is the static
    classification: the roof the kernel would reach first."""
    fp64_per_launch, fp64_src = fp64
    peak, peak_src = _peaks()
    fpeak, fpeak_src = _fp64_peak(sm_mhz)
    s = launch_ms / 1e3
    achieved = bytes_per_launch / s / 1e9
    t_hbm = bytes_per_launch / (peak * 1e9)
    t_fp = fp64_per_launch / fpeak
    traffic, tnote = _traffic(build_keys)
    return {
        "bound": "hbm" if t_hbm >= t_fp else "fp64",
        "kernel": kernel_name,
        "achieved": achieved,
        "peak": peak,
        "unit": "GB/s",
        "frac": achieved / peak,
        "traffic": traffic,
        "traffic_source": tnote,
        "peak_source": peak_src,
        "bytes_per_launch": bytes_per_launch,
        "launch_ms": launch_ms,
        "fp64": {"achieved": fp64_per_launch / s / 1e9, "peak": fpeak / 1e9, "unit": "G FP64-pipe instr/s",
                 "frac": fp64_per_launch / s / fpeak, "instr_per_launch": fp64_per_launch,
                 "peak_source": fpeak_src, "count": fp64_src},
        "max_hbm_frac_at_fp64_roof": min(1.0, t_hbm / t_fp) if t_fp > 0 else 1.0,
    }


# ---------------------------------------------------------------------------
# our implementation


class Population:
    """One mechanism population resident on this GPU."""

    def __init__(self, stem, n, n_nodes, seed, options):
        from paper_1905_02241_b200.instance import init, node_layout
        from paper_1905_02241_b200.ir import MechIR
        from paper_1905_02241_b200.runner import CudaRunner

        self.stem = stem
        self.ir = MechIR.load(ROOT / "fixtures" / "ir" / f"{stem}.json")
        self.n = n
        self.n_nodes = n_nodes
        self.runner = CudaRunner(self.ir, options=options)
        self.build_key = self.runner.mb.so_path.stem[3:]  # lib<mech>-<hash>
        self.data = init(self.ir, n, seed)
        self.kernel = "step_nodes" if n_nodes else "step"
        if n_nodes:
            self.node_index, self.node_v = node_layout(n, n_nodes, seed)
        self.dev = None

    @property
    def kernel_name(self):
        k = self.runner.node_kernel(self.dev) if (self.kernel == "step_nodes" and self.dev is not None) else self.kernel
        return f"{self.runner.mb.symbol}_k_{k}"

    def setup_device(self):
        r = self.runner
        if self.n_nodes:
            self.dev = r.to_device(self.data, skip=("v",))
            r.bind_nodes(self.dev, self.node_index, self.node_v)
            r.gather_voltage(self.dev)
        else:
            self.dev = r.to_device(self.data)
        r.run_kernel(self.dev, "initialize", 1)
        # the store is resident now: drop the host copy (8 ranks x GBs of numpy otherwise)
        self.data = None
        if self.n_nodes:
            self.node_index = self.node_v = None

    def launch(self, steps=1):
        self.runner.launch(self.dev, self.kernel, steps)

    def launch_bytes(self):
        from paper_1905_02241_b200.traffic import launch_bytes

        touched = self.dev.nodes.n_segs if (self.dev is not None and self.dev.nodes is not None) else 0
        return launch_bytes(self.runner.abi, self.n, self.kernel, touched)


class L2Flush:
    """Between timed steps of an L2-sized workload: write a 2 x L2 buffer
    (evicts every line the previous step left in L2), then read a second
    2 x L2 buffer so the flush's own dirty lines are written back before
    the next step starts instead of during it (tools/micro/flush_modes.cu)."""

    def __init__(self, l2_bytes):
        from paper_1905_02241_b200 import runtime as rt

        self.rt = rt
        self.w = rt.DeviceBuffer(2 * l2_bytes)
        self.r = rt.DeviceBuffer(2 * l2_bytes)
        rt.memset(self.r.ptr, 0, self.r.nbytes, rt.Stream())
        rt.lib().nmodl_device_sync()

    def __call__(self, stream):
        L = self.rt.lib()
        self.rt.check(L.nmodl_l2_flush(C_void(self.w.ptr), self.w.nbytes // 8, C_void(stream.handle)), "l2_flush")
        self.rt.check(L.nmodl_l2_clean(C_void(self.r.ptr), self.r.nbytes // 8, C_void(stream.handle)), "l2_clean")


SUSTAINED_S = 0.6


def run_workload(name, args, dist, sustained=True):
    from paper_1905_02241_b200 import runtime as rt

    w = WORKLOADS[name]
    seed = 42 + dist.rank
    pops = [Population(stem, n, w["nodes"], seed, options_for(stem)) for stem, n in w["mechs"]]
    for p in pops:
        p.setup_device()
    by_stem = {p.stem: p for p in pops}
    for dst, dslot, src, sslot in w.get("couplings", ()):
        by_stem[dst].runner.share_slot(by_stem[dst].dev, dslot, by_stem[src].dev, sslot)
    info = rt.device_info(dist.device)
    working = sum(p.launch_bytes() for p in pops)
    flush = L2Flush(info["l2_bytes"]) if working < 3 * info["l2_bytes"] else None
    s0 = pops[0].runner.stream
    for p in pops:  # one stream: launch order == step order (bbp20m's coupling)
        p.runner.stream = s0
    members = list(pops)
    if w.get("grouped"):
        pops = [_DirectGroup(pops, w.get("couplings", ()), s0, w["grouped"])]
    K, W = args.steps, args.warmup
    for _ in range(W):
        for p in pops:
            p.launch(1)
    s0.sync()
    for p in members:
        p.runner.check(p.dev)
    # the timed graph: K steps.  External event records before a step and
    # after every population's launch time each kernel inside this replay:
    # every step when an L2 flush runs between steps (the flush is excluded
    # from the step time), else the first min(K, 20) steps of a multi-
    # population step (an event node between two kernels also cuts their
    # programmatic-dependent-launch edge, so the other steps run without
    # them); a single-population step needs none (its kernel IS the step).
    P = len(pops)
    E = K if flush is not None else (0 if P == 1 else min(K, 20))
    evs = [[rt.Event() for _ in range(P + 1)] for _ in range(E)]

    def body():
        for k in range(K):
            if flush is not None:
                flush(s0)
            if k < E:
                evs[k][0].record_external(s0)
            for j, p in enumerate(pops):
                p.launch(1)
                if k < E:
                    evs[k][j + 1].record_external(s0)

    graph = rt.capture(s0, body)
    graph.upload(s0)
    ev_a, ev_b = rt.Event(), rt.Event()
    dist.barrier()
    s0.sync()
    phys = _physical_gpu(dist.device)
    with ClockSampler(phys) as clk:
        ev_a.record(s0)
        graph.launch(s0)
        ev_b.record(s0)
        ev_b.sync()
    graph_ms = ev_a.elapsed_ms(ev_b)
    # with a flush the timed region is the steps only (flush kernels excluded)
    total_ms = sum(evs[k][0].elapsed_ms(evs[k][P]) for k in range(K)) if flush is not None else graph_ms
    if E:  # per-population launch durations, scaled from the evented steps to K
        per_pop_ms = [sum(evs[k][j].elapsed_ms(evs[k][j + 1]) for k in range(E)) * K / E for j in range(P)]
    else:
        per_pop_ms = [total_ms]
    del graph
    for p in members:
        p.runner.check(p.dev)
    clocks = clk.summary()
    sus = None
    if sustained and flush is None:
        S = int(min(20000, max(K, SUSTAINED_S / max(total_ms / K / 1e3, 1e-9))))
        g2 = rt.capture(s0, lambda: [p.launch(1) for _ in range(S) for p in pops])
        g2.upload(s0)
        dist.barrier()
        s0.sync()
        with ClockSampler(phys) as clk2:
            ev_a.record(s0)
            g2.launch(s0)
            ev_b.record(s0)
            ev_b.sync()
        sms = ev_a.elapsed_ms(ev_b)
        del g2
        for p in members:
            p.runner.check(p.dev)
        smax = dist.allreduce([sms], "max")[0]
        n_all_s = dist.allreduce([float(sum(p.n for p in pops))], "sum")[0]
        sus = {"value": n_all_s * S / (smax / 1e3), "ms_per_step": smax / S, "steps": S, "seconds": smax / 1e3,
               "clocks": clk2.summary(),
               "note": f"one graph of {S} steps (>= {SUSTAINED_S} s) right after the timed burst"}
    dist.barrier()
    max_ms = dist.allreduce([total_ms], "max")[0]
    n_rank = sum(p.n for p in pops)
    n_all = dist.allreduce([float(n_rank)], "sum")[0]
    value = n_all * K / (max_ms / 1e3)
    j = int(np.argmax(per_pop_ms))
    dom = pops[j]
    sm_mhz = clocks.get("sm_mhz")
    key = f"{dom.build_key}@{dom.n}"
    roof = _roofline(dom.kernel_name, dom.launch_bytes(), _pop_fp64(dom), per_pop_ms[j] / K, [key], sm_mhz)
    roof["share_of_step"] = per_pop_ms[j] / max(total_ms, 1e-30)
    roof["model"] = _describe(dom)
    from paper_1905_02241_b200.parallel import device_checksums

    local = np.concatenate([device_checksums(p.runner, p.dev) for p in members])
    table = dist.allgather(local)
    per_mech = {}
    for i, p in enumerate(pops):
        ms = per_pop_ms[i] / K
        key = f"{p.build_key}@{p.n}"
        r = _roofline(p.kernel_name, p.launch_bytes(), _pop_fp64(p), ms, [key], sm_mhz)
        per_mech[p.stem] = {"instances": p.n, "ms_per_launch": ms, "GBps": r["achieved"], "hbm_frac": r["frac"],
                            "fp64_frac": r["fp64"]["frac"], "bound": r["bound"], "traffic": r["traffic"],
                            "bytes_per_instance_step": p.launch_bytes() / p.n, "build": p.build_key}
    return {
        "value": value,
        "checksum_of_checksums": float(np.sum(table[..., 1])),
        "ms_per_step": max_ms / K,
        "n_rank": n_rank,
        "clocks": clocks,
        "sustained": sus,
        "gpu_launches": K * P,
        "l2": ("L2 flushed between timed steps (write 2xL2, then read 2xL2 clean; flush kernels outside the "
               "event-timed steps)") if flush is not None else "inputs larger than L2 (no flush)",
        "roofline": roof,
        "per_mechanism": per_mech,
    }


def _pop_fp64(p):
    """FP64 instructions of one launch of a population (or of a direct group:
    the sum over its members, each counted with its own build's ncu count)."""
    if isinstance(p, _DirectGroup):
        parts = [_pop_fp64(m) for m in p.pops]
        return sum(x for x, _ in parts), "; ".join(sorted({c for _, c in parts}))
    return _fp64_instr(p.ir, p.n, f"{p.build_key}@{p.n}")


class _DirectGroup:
    """Every population of a direct workload as ONE population-group launch
    per step (runner.PopulationGroup kind="direct": every CTA runs every
    population in turn; an ion consumer follows its producer with the
    producer's ilp, so each thread reads the ica it just wrote)."""

    def __init__(self, pops, couplings, stream, name):
        import dataclasses

        from paper_1905_02241_b200.runner import PopulationGroup

        by = {p.stem: p for p in pops}
        chained = {dst: src for dst, _, src, _ in couplings}
        chains = []
        for p in pops:
            if p.stem in chained:
                continue
            chain = [(p.runner, p.dev)]
            for dst, src in chained.items():
                if src == p.stem:
                    q = by[dst]
                    chain.append((q.runner, q.dev, dataclasses.replace(q.runner.options, ilp=p.runner.options.ilp)))
            chains.append(chain)
        self.group = PopulationGroup(name, chains, kind="direct")
        self.pops = pops
        self.stream = stream
        self.n = sum(p.n for p in pops)
        self.stem = "group(" + "+".join(p.stem for p in pops) + ")"
        self.kernel = "step"
        self.ir = pops[0].ir
        self.build_key = self.group.gb.so_path.stem[3:]
        self.runner = pops[0].runner
        self.dev = pops[0].dev

    @property
    def kernel_name(self):
        return f"{self.group.gb.symbol}_k_step_group"

    def launch(self, steps=1):
        self.group.launch(self.stream, steps)

    def launch_bytes(self):
        return sum(p.launch_bytes() for p in self.pops)


def _describe(pop):
    from paper_1905_02241_b200.traffic import describe

    if isinstance(pop, _DirectGroup):
        return {m.stem: describe(m.runner.abi, m.kernel) for m in pop.pops}
    return describe(pop.runner.abi, pop.kernel)


def _physical_gpu(device):
    visible = os.environ.get("CUDA_VISIBLE_DEVICES")
    if visible and visible.split(",")[0].isdigit():
        return int(visible.split(",")[device])
    return device


def _column_mode():
    """Launch schedule of the column step (NMODL_COLUMN_MODE, column.SCHEDULES):
    "grouped" (default: the soma populations as one population-group launch
    beside Ih, then the in-order combine), "concurrent" or "sequential" --
    all bit-identical (tests/test_gpu_column.py)."""
    return {"schedule": os.environ.get("NMODL_COLUMN_MODE", "grouped")}


def _column_spec():
    from paper_1905_02241_b200.column import ColumnSpec

    return ColumnSpec(n_cells=int(os.environ.get("NMODL_COLUMN_CELLS", WORKLOADS["column"]["cells"])))


def run_column(args, dist, sustained=True):
    """configs[4]: 100k-cell synthetic column, cells partitioned over ranks by
    per-cell bytes/step (parallel.partition_cells); strong scaling."""
    from paper_1905_02241_b200 import runtime as rt
    from paper_1905_02241_b200.column import LAUNCH_ORDER, ColumnShard
    from paper_1905_02241_b200.parallel import partition_cells

    spec = _column_spec()
    bounds = partition_cells(np.full(spec.n_cells, spec.cell_cost()), dist.world)
    shard = ColumnShard(spec, int(bounds[dist.rank]), int(bounds[dist.rank + 1]), options_for, **_column_mode())
    s0 = shard.stream
    K, W = args.steps, args.warmup
    shard.launch(W)
    s0.sync()
    shard.check()
    ev_a, ev_b = rt.Event(), rt.Event()
    graph = rt.capture(s0, lambda: shard.launch(K))
    graph.upload(s0)
    dist.barrier()
    s0.sync()
    phys = _physical_gpu(dist.device)
    with ClockSampler(phys) as clk:
        ev_a.record(s0)
        graph.launch(s0)
        ev_b.record(s0)
        ev_b.sync()
    ms = ev_a.elapsed_ms(ev_b)
    del graph
    shard.check()
    clocks = clk.summary()
    sus = None
    if sustained:
        S = int(min(20000, max(K, SUSTAINED_S / max(ms / K / 1e3, 1e-9))))
        g2 = rt.capture(s0, lambda: shard.launch(S))
        g2.upload(s0)
        dist.barrier()
        s0.sync()
        with ClockSampler(phys) as clk2:
            ev_a.record(s0)
            g2.launch(s0)
            ev_b.record(s0)
            ev_b.sync()
        sms = ev_a.elapsed_ms(ev_b)
        del g2
        shard.check()
        smax = dist.allreduce([sms], "max")[0]
        n_all_s = dist.allreduce([float(shard.n_instances)], "sum")[0]
        sus = {"value": n_all_s * S / (smax / 1e3), "ms_per_step": smax / S, "steps": S, "seconds": smax / 1e3,
               "clocks": clk2.summary()}
    # per-population launch durations: each population's launches alone in
    # their own graph (the soma populations overlap inside the real step)
    per_pop = {}
    reps = 10
    for m in LAUNCH_ORDER:
        g = rt.capture(s0, lambda m=m: shard.runners[m].launch(shard.devs[m], "step_nodes", reps))
        g.upload(s0)
        a, b = rt.Event(), rt.Event()
        a.record(s0)
        g.launch(s0)
        b.record(s0)
        b.sync()
        per_pop[m] = a.elapsed_ms(b) / reps
    shard.check()
    dist.barrier()
    max_ms = dist.allreduce([ms], "max")[0]
    n_all = dist.allreduce([float(shard.n_instances)], "sum")[0]
    table = dist.allgather(shard.checksums())
    from paper_1905_02241_b200.traffic import launch_bytes

    keys, parts = _column_keys(shard)
    fp64 = (sum(p[0] for p in parts), "; ".join(sorted({p[1] for p in parts})))
    roof = _roofline(f"whole step: {shard.kernels_per_step()} launches ({shard.schedule} schedule)",
                     shard.launch_bytes(), fp64, ms / K, keys,
                     clocks.get("sm_mhz"))
    roof["share_of_step"] = 1.0
    per_mech = {}
    for m in LAUNCH_ORDER:
        d, r = shard.devs[m], shard.runners[m]
        b = launch_bytes(r.abi, d.n, "step_nodes", d.nodes.n_segs)
        per_mech[m] = {"instances": d.n, "ms_per_launch_alone": per_pop[m], "GBps_alone": b / (per_pop[m] / 1e3) / 1e9,
                       "segments": d.nodes.n_segs, "build": r.mb.so_path.stem[3:]}
    return {
        "value": n_all * K / (max_ms / 1e3),
        "ms_per_step": max_ms / K,
        "n_rank": shard.n_instances,
        "clocks": clocks,
        "sustained": sus,
        "gpu_launches": K * shard.kernels_per_step(),
        "l2": "inputs larger than L2 (no flush)",
        "roofline": roof,
        "checksum_of_checksums": float(np.sum(table[..., 1])),
        "cells_per_rank": [int(b) for b in np.diff(bounds)],
        "per_mechanism": per_mech,
    }


def _column_keys(shard):
    """Build keys ("<library stem>@<instances>") of the kernels one column step
    launches, and their FP64 instruction counts: the standalone population
    kernels, or -- grouped soma mode -- Ih, the synapses and the soma group
    (whose instance count is the sum of its members')."""
    from paper_1905_02241_b200.column import LAUNCH_ORDER, SOMA_MECHS

    keys, parts = [], []
    for m in LAUNCH_ORDER:
        if m in shard.group_members:
            continue
        k = f"{shard.runners[m].mb.so_path.stem[3:]}@{shard.devs[m].n}"
        keys.append(k)
        parts.append(_fp64_instr(shard.runners[m].ir, shard.devs[m].n, k))
    if shard.grouped:
        n = sum(shard.devs[m].n for m in shard.group_members)
        k = f"{shard.group.gb.so_path.stem[3:]}@{n}"
        keys.append(k)
        e = _traffic_record().get("by_build", {}).get(k, {})
        if "fp64_instr_per_instance" in e:
            parts.append((e["fp64_instr_per_instance"] * n, "ncu-measured FP64 instructions of this build"))
        else:
            for m in shard.group_members:
                parts.append(_fp64_instr(shard.runners[m].ir, shard.devs[m].n, "?"))
    return keys, parts


def C_void(x):
    import ctypes

    return ctypes.c_void_p(x)


def e2e_measure(name, dist, calls=2, timesteps=1000):
    """Same metric through the public API with host buffers: each call uploads
    the population from pinned host memory, binds nodes, runs nrn_init and
    `timesteps` fused steps, and downloads the full store (and node arrays)."""
    from paper_1905_02241_b200 import runtime as rt
    from paper_1905_02241_b200.instance import init, node_layout
    from paper_1905_02241_b200.ir import MechIR
    from paper_1905_02241_b200.runner import CudaRunner, simulate, simulate_nodes

    w = WORKLOADS[name]
    seed = 42 + dist.rank
    jobs = []
    for stem, n in w["mechs"]:
        ir = MechIR.load(ROOT / "fixtures" / "ir" / f"{stem}.json")
        runner = CudaRunner(ir, options=options_for(stem))
        data = init(ir, n, seed)
        pins = [rt.PinnedRegistration(a) for a in list(data.arrays.values()) + list(data.acc.values())]
        extra = None
        if w["nodes"]:
            idx, nv = node_layout(n, w["nodes"], seed)
            extra = (idx, nv)
            pins += [rt.PinnedRegistration(idx), rt.PinnedRegistration(nv)]
        jobs.append((ir, runner, data, extra, pins, n))

    phases = {}

    def one_call():
        for ir, runner, data, extra, _, n in jobs:
            if extra is None:
                simulate(ir, data, timesteps, runner=runner)
            else:
                t = {}
                simulate_nodes(ir, data, timesteps, extra[0], extra[1], runner=runner, timings=t)
                for k, v in t.items():
                    if isinstance(v, float):
                        phases[k] = phases.get(k, 0.0) + v
                    else:
                        phases[k] = v

    one_call()  # warm-up (also primes graph/occupancy caches)
    phases.clear()
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(calls):
        one_call()
    dt = time.perf_counter() - t0
    phases["unaccounted"] = dt - sum(v for v in phases.values() if isinstance(v, float))
    dt = dist.allreduce([dt], "max")[0]
    n_all = dist.allreduce([float(sum(j[5] for j in jobs))], "sum")[0]
    h2d = int(sum(_h2d(j) for j in jobs))
    d2h = int(sum(_d2h(j) for j in jobs))
    return _e2e_line(n_all * timesteps * calls / dt, h2d, d2h, timesteps, calls,
                     f"one public-API call (runner.simulate{'_nodes' if w['nodes'] else ''}): pinned H2D of the store "
                     "(arrays no kernel touches stay on the host, scanned for non-finite values there)"
                     + (", node_index + node_v upload, device sort" if w["nodes"] else "")
                     + f", nrn_init, {timesteps} timesteps, D2H of the written arrays"
                     + (" and node rhs/d" if w["nodes"] else ""),
                     {k: (v / calls if isinstance(v, float) else v) for k, v in phases.items()})


def _e2e_line(value, h2d_call, d2h_call, timesteps, calls, step, phases=None):
    """The e2e object: the copy fields of the contract are per timestep (one
    public call = `timesteps` steps, one upload and one download); the
    per-call bytes are stated beside them."""
    out = {"value": value, "unit": UNIT,
           "h2d_bytes_per_step": h2d_call / timesteps, "d2h_bytes_per_step": d2h_call / timesteps,
           "h2d_bytes_per_call": h2d_call, "d2h_bytes_per_call": d2h_call,
           "timesteps_per_call": timesteps, "calls": calls, "call": step}
    if phases is not None:
        out["phase_seconds_per_call"] = phases
    return out


def _h2d(job):
    """Bytes the public call copies host->device: the store (v excepted in
    node mode: it is gathered from the node voltages; i_acc/g_acc are
    outputs only; arrays no kernel reads or writes stay on the host,
    runner._unread_arrays), node_index, node_v."""
    from paper_1905_02241_b200.runner import _unread_arrays

    ir, runner, data, extra, _, n = job
    unread = set(_unread_arrays(runner, data, ("initialize", "step_nodes" if extra is not None else "step")))
    b = sum(a.nbytes for k, a in data.arrays.items()
            if not (extra is not None and k == "v") and k not in unread)
    if extra is not None:
        b += extra[0].nbytes + extra[1].nbytes
    return b


def _d2h(job):
    """Bytes copied back: the arrays a launch may write (states, assigned,
    currents, accumulators; v in node mode) and the node rhs/d arrays."""
    ir, runner, data, extra, _, n = job
    written = runner._writes["initialize"] | runner._writes["step_nodes" if extra is not None else "step"]
    if extra is not None:
        written = written | {"v"}
    b = sum(8 * n for k in list(data.arrays) + ["i_acc", "g_acc"] if k in written)
    if extra is not None:
        b += 2 * extra[1].nbytes
    return b


def e2e_column(dist, calls=1, timesteps=1000):
    """configs[4] through the public column call (column.simulate_column):
    pinned H2D of this rank's seven stores, the node voltages and node_index
    arrays, the device-side node layout, nrn_init, `timesteps` steps of all
    populations, D2H of every written array and the node arrays.  The
    inputs (stores, node_index, node_v) are generated before the clock
    starts."""
    from paper_1905_02241_b200 import runtime as rt
    from paper_1905_02241_b200.column import LAUNCH_ORDER, host_stores, shard_layout, simulate_column
    from paper_1905_02241_b200.parallel import partition_cells

    spec = _column_spec()
    bounds = partition_cells(np.full(spec.n_cells, spec.cell_cost()), dist.world)
    lo, hi = int(bounds[dist.rank]), int(bounds[dist.rank + 1])
    host = host_stores(spec, lo, hi)
    pins = [rt.PinnedRegistration(a) for h in host.values() for a in list(h.arrays.values()) + list(h.acc.values())]
    lay = shard_layout(spec, lo, hi)
    mode = _column_mode()
    # warm-up call: loads the kernels (reused below), primes the caches
    _, _, shard = simulate_column(spec, 10, lo, hi, host=host, options_for=options_for, layout=lay, **mode)
    runners = shard.runners
    writes = {m: runners[m]._writes["initialize"] | runners[m]._writes["step_nodes"] | {"v"} for m in LAUNCH_ORDER}
    del shard
    host = host_stores(spec, lo, hi)  # fresh inputs (the warm-up advanced them)
    pins = [rt.PinnedRegistration(a) for h in host.values() for a in list(h.arrays.values()) + list(h.acc.values())]
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(calls):
        _, nodes, shard = simulate_column(spec, timesteps, lo, hi, host=host, options_for=options_for,
                                          runners=runners, layout=lay, **mode)
    dt = time.perf_counter() - t0
    dt = dist.allreduce([dt], "max")[0]
    n_rank = sum(h.n for h in host.values())
    n_all = dist.allreduce([float(n_rank)], "sum")[0]
    h2d = sum(a.nbytes for h in host.values() for a in h.arrays.values())
    h2d += sum(idx.nbytes for _, _, idx in lay["mechs"].values()) + lay["node_v"].nbytes
    d2h = sum(8 * host[m].n for m in LAUNCH_ORDER for k in list(host[m].arrays) + ["i_acc", "g_acc"] if k in writes[m])
    d2h += 3 * 8 * lay["n_nodes"]
    del pins
    return _e2e_line(n_all * timesteps * calls / dt, h2d, d2h, timesteps, calls,
                     "one public column call (column.simulate_column): pinned H2D of the 7 stores, node_v and "
                     f"node_index, device node layout, nrn_init, {timesteps} timesteps, D2H of the written arrays "
                     "and node v/rhs/d")


# ---------------------------------------------------------------------------
# CPU reference (the reference's emitted C, all host threads)


def numpy_oracle_rate(name, n=65536, budget_s=4.0):
    """SURVEY.md §8(d) CPU leg 2: the reference's numpy runtime semantics
    (`modlc.interp.Runner`, restated bit-exactly in oracle/interp_np.py),
    single-threaded by design, on a 65,536-instance prefix of each mechanism;
    the population step is the n-weighted sum of the per-mechanism times."""
    from oracle import interp_np as O
    from paper_1905_02241_b200.ir import MechIR

    mechs = _reference_mechs(name)
    total_s, total_n, parts = 0.0, 0, []
    for stem, n_full in mechs:
        ir = MechIR.load(ROOT / "fixtures" / "ir" / f"{stem}.json")
        data = O.init(ir, n, 42)
        runner = O.OracleRunner(ir)
        runner.run_kernel(data, "initialize", 1)
        steps, dt = 0, 0.0
        t0 = time.perf_counter()
        while dt < budget_s / len(mechs) or steps < 2:
            runner.run_kernel(data, "state_update", 1)
            runner.run_kernel(data, "current_update", 1)
            steps += 1
            dt = time.perf_counter() - t0
        total_s += dt / steps * (n_full / n)
        total_n += n_full
        parts.append(f"{stem}: {n} x {steps} steps in {dt:.2f}s")
    return {"value": total_n / total_s, "unit": UNIT, "cores": 1,
            "sample": "oracle/interp_np.py (numpy restatement of modlc.interp.Runner), single thread; " + "; ".join(parts)}


def _reference_mechs(name):
    if name == "column":
        from paper_1905_02241_b200.column import LAUNCH_ORDER

        spec = _column_spec()
        return [(m, spec.n_cells * spec.instances_per_cell(m)) for m in LAUNCH_ORDER]
    return WORKLOADS[name]["mechs"]


def reference_arm(name, K, W, budget_s=60.0):
    """The reference's CPU path: W untimed + K timed steps of its emitted
    scalar C (all host threads).  Each step advances one timestep of a
    bounded instance sample per mechanism, sized so the whole run takes about
    `budget_s`; the full-population step time is the sample's time scaled by
    n / sample (the C loop is per-instance independent).  Used by
    `--impl reference` and, with a smaller K, as the ours-arm cpu_baseline."""
    from oracle import ref_c
    from paper_1905_02241_b200.instance import init
    from paper_1905_02241_b200.ir import MechIR

    threads = os.cpu_count() or 1
    mechs = _reference_mechs(name)
    jobs = []
    for stem, n in mechs:
        if not ref_c.available(stem):
            return None
        r = ref_c.RefC(stem, ref_c.native_build(stem))
        ir = MechIR.load(ROOT / "fixtures" / "ir" / f"{stem}.json")
        probe = min(n, 200_000)
        data = init(ir, probe, 42)
        r.initialize(data)
        t0 = time.perf_counter()
        r.steps(data, 1, threads)
        per_inst = max((time.perf_counter() - t0) / probe, 1e-12)
        per_step_budget = budget_s / max(K + W, 1) / len(mechs)
        ns = int(min(n, max(10_000, per_step_budget / per_inst)))
        data = init(ir, ns, 42)
        r.initialize(data)
        jobs.append((stem, n, ns, r, data))
    for _ in range(W):
        for stem, n, ns, r, data in jobs:
            r.steps(data, 1, threads)
    step_s = 0.0
    for _ in range(K):
        for stem, n, ns, r, data in jobs:
            t0 = time.perf_counter()
            r.steps(data, 1, threads)
            step_s += (time.perf_counter() - t0) * (n / ns)
    total = sum(n for _, n, _, _, _ in jobs)
    return {
        "value": total * K / step_s,
        "ms_per_step": step_s / K * 1e3,
        "unit": UNIT,
        "cores": threads,
        "kind": "reference",
        "sample": "reference-emitted scalar C (modlc.codegen.emit_scalar, count field renamed), gcc -O3 -march=native, "
                  f"{threads} threads, {K} timed steps after {W}, each step: "
                  + ", ".join(f"{stem} {ns} of {n} instances" for stem, n, ns, _, _ in jobs)
                  + (" (full-population time = sample time x n/sample)")
                  + ("; no node_index scatter (the reference has none)" if WORKLOADS[name]["nodes"] else ""),
        "cpu": _cpu_model(),
    }


def _cpu_model():
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ---------------------------------------------------------------------------


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=list(WORKLOADS), default=DEFAULT_WORKLOAD)
    ap.add_argument("--no-also", action="store_true", help="skip the secondary workloads")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-sustained", action="store_true")
    ap.add_argument("--cells", type=int, default=None,
                    help="column only: cells of the whole column (default 100,000); e.g. 12,500 = one rank's "
                         "share at 8 GPUs, timed on one GPU as the strong-scaling proxy")
    args = ap.parse_args()
    if args.cells is not None:
        os.environ["NMODL_COLUMN_CELLS"] = str(args.cells)
    w = WORKLOADS[args.workload]
    column = args.workload == "column"
    config = {
        "workload": args.workload,
        "baseline_config": w["config"],
        "mechanisms": {stem: n for stem, n in _reference_mechs(args.workload)},
        "instances_per_gpu": None if column else sum(n for _, n in w["mechs"]),
        "n_nodes_per_gpu": w["nodes"],
        "dt_ms": 0.025,
        "parallelism": (f"{args.gpus} x cell shard (strong scaling, no per-step collective)" if column else
                        f"{args.gpus} x instance shard by cell (weak scaling, no per-step collective)"),
    }
    if column:
        config["cells"] = _column_spec().n_cells
        config["schedule"] = _column_mode()["schedule"]
    line = {"metric": METRIC, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "higher_is_better": True, "scaling": "strong" if column else "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (modlc.interp.init-format seeded instance store; random node_index)",
            "config": config}
    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        if rank == 0:
            ref = reference_arm(args.workload, args.steps, args.warmup)
            line["impl"] = "reference"
            if ref is None:
                line["unavailable"] = "oracle/_ref not built (needs the reference front-end)"
            else:
                line.update({"value": ref["value"], "ms_per_step": ref["ms_per_step"],
                             "cpu_baseline": {k: ref[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu")},
                             "e2e": {"value": ref["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                                     "d2h_bytes_per_step": 0}})
            print(json.dumps(line), flush=True)
        return
    dist = Dist()
    from paper_1905_02241_b200 import runtime as rt

    rt.require_device(dist.device)
    if column:
        res = run_column(args, dist, sustained=not args.no_sustained)
        e2e = None if args.no_e2e else e2e_column(dist)
    else:
        res = run_workload(args.workload, args, dist, sustained=not args.no_sustained)
        e2e = None if args.no_e2e else e2e_measure(args.workload, dist)
    also = {}
    if not args.no_also and not column:
        for other in ("hh1m", "hh10m", "bbp20m", "bbp20m_grouped", "kinetic1m", "kinetic1m_grouped", "kinetic10m"):
            if other == args.workload:
                continue
            # warm-up past the initial transient: Newton iteration counts
            # (cdp5ish) fall over the first ~100 steps after nrn_init
            a = argparse.Namespace(steps=min(args.steps, 50), warmup=max(args.warmup, 100))
            r = run_workload(other, a, dist, sustained=False)
            also[other] = {"value": r["value"], "ms_per_step": r["ms_per_step"], "l2": r["l2"],
                           "roofline": r["roofline"], "per_mechanism": r["per_mechanism"]}
            del r
    cpu = None
    if dist.rank == 0 and args.gpus == 1 and not args.no_cpu:
        cpu = reference_arm(args.workload, K=20, W=5, budget_s=30.0)
        if cpu is not None and not column:
            cpu["numpy_oracle"] = numpy_oracle_rate(args.workload)
    if dist.rank == 0:
        line.update({
            "value": res["value"],
            "ms_per_step": res["ms_per_step"],
            "roofline": res["roofline"],
            "cpu_baseline": None if cpu is None else {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample",
                                                                          "cpu", "numpy_oracle") if k in cpu},
            "e2e": e2e,
            "gpu_launches": res["gpu_launches"],
            "clocks": res["clocks"],
            "sustained": res["sustained"],
            "l2": res["l2"],
            "arithmetic": RELAXED_NOTE,
            "per_mechanism": res["per_mechanism"],
            "validation": {"checksum_of_checksums": res.get("checksum_of_checksums"),
                           "how": f"per-array sum|x| on each GPU (fixed-tree device reduction), all-gathered "
                                  f"({dist.backend} process group)"},
            "also": also,
        })
        if column:
            line["cells_per_rank"] = res["cells_per_rank"]
        print(json.dumps(line), flush=True)
    dist.close()


if __name__ == "__main__":
    main()
