"""Benchmark: nrn_state + nrn_cur instance-steps/s (fp64) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload synapse10m|hh1m|bbp20m|kinetic1m] [--no-also]

One JSON line on rank 0.  A "step" is one timestep of the hot path over the
whole synthetic population on every rank: one fused nrn_state+nrn_cur launch
per mechanism (for the default workload also the node_index gather and the
in-order rhs/d reduction, inside the same kernel).  Workloads are the
BASELINE.json configs:

  synapse10m  configs[1]  ProbAMPANMDA_EMS restated (4 cnexp states, Mg block,
                          numeric conductance), 10M instances / GPU, random
                          node_index onto 1M nodes (default; inputs >> L2)
  hh1m        configs[0]  hh (cnexp, analytic conductance), 1M instances / GPU
                          (working set ~ L2: L2 flushed between timed steps)
  bbp20m      configs[2]  NaTs2_t, K_Pst, Ca_HVA, SKv3_1, Ih, CaDynamics_E2;
                          20M instances / GPU split evenly (6 launches / step)
  kinetic1m   configs[3]  6-state KINETIC Na (runtime LU k=6) + cdp5-style
                          Newton k=5 with LU, 1M instances each

Multi-GPU (torchrun): one process per GPU, each rank owns its own shard of
cells (weak scaling, no per-step collective); timings are CUDA events on the
launching stream, max over ranks; NCCL only all-reduces validation checksums.
`--impl reference` times the reference's own CPU implementation (its emitted
scalar C, oracle/_ref, compiled -O3 -march=native, all host threads) on a
bounded sample of the same workload, rank 0 only.
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
    "bbp20m": {
        "config": BASELINE["configs"][2],
        "mechs": [(m, 20_000_000 // 6) for m in ("NaTs2_t", "K_Pst", "Ca_HVA", "SKv3_1", "Ih", "cadyn")],
        "nodes": 0,
        # CaDynamics_E2 accumulates the calcium current Ca_HVA writes (same
        # compartments, same order): its `ica` slot is Ca_HVA's array
        "couplings": [("cadyn", "ica", "Ca_HVA", "ica")],
    },
    "kinetic1m": {"config": BASELINE["configs"][3], "mechs": [("na6", 1_000_000), ("cdp5ish", 1_000_000)], "nodes": 0},
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
        "ProbAMPANMDA_EMS": CudaOptions(ilp=1, fast_path=False, tile=2304),  # 2048: 0.2823, 2304: 0.2807 ms (3 reps)
        "hh_subset": CudaOptions(ilp=1, pipe=True, recip=True, div_approx=True, exp_share=True,
                                 fast_redo=True),  # 0.0412 -> 0.0329 ms
        "NaTs2_t": CudaOptions(ilp=2, min_blocks=2, pipe=True, recip=True, div_approx=True, exp_share=True,
                               fast_redo=True),  # 0.0788 -> 0.0557 ms
        "K_Pst": CudaOptions(ilp=2, min_blocks=2, pipe=True, recip=True, quot=True, div_approx=True, exp_smem=True,
                             exp_share=True, fast_redo=True),  # 0.0717 -> 0.0574 ms
        "Ca_HVA": CudaOptions(ilp=2, min_blocks=2, pipe=True, recip=True, div_approx=True, fast_redo=True),  # 0.0707 -> 0.0561
        "SKv3_1": CudaOptions(ilp=1, pipe=True, grid_waves=4, div_approx=True, fast_redo=True),  # 0.0500 -> 0.0426 ms
        "Ih": CudaOptions(ilp=2, pipe=True, grid_waves=4, recip=True, div_approx=True, fast_redo=True),  # 0.0474 -> 0.0392 ms
        "na6": CudaOptions(ilp=1, min_blocks=2, pipe=True, fast_redo=True, lu_spec=True),  # 0.0485 -> 0.0369 ms
        "cdp5ish": CudaOptions(ilp=1, min_blocks=2, pipe=True, div_approx=True, fast_redo=True, lu_spec=True),  # 0.0583 -> 0.0390
    }
    return tuned.get(stem, CudaOptions())


RELAXED_NOTE = ("fp64 throughout; rate code uses reciprocal/quotient shadows (X/(1/E) -> X*E), <=2-ulp division, "
                "shared affine exponentials (exp(aX+b) = exp(aX+b0)*exp(b-b0)) and (K_Pst) a 1-ulp shared-table exp "
                "where tuned (bench.options_for); solver cores IEEE; parity 1e-10 after 1000 steps is tested for every flag")


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
    """torchrun plumbing: one process per GPU; NCCL for the (tiny) barrier /
    max-time / checksum collectives.  When fewer GPUs than ranks are visible
    (a multi-rank smoke test on one GPU) ranks share devices and the
    collectives fall back to gloo."""

    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.device = self.local
        self.pg = None
        self.backend = None
        if self.world > 1 or os.environ.get("TORCHELASTIC_RUN_ID"):
            import torch
            import torch.distributed as dist

            ndev = max(torch.cuda.device_count(), 1)
            self.device = self.local % ndev
            torch.cuda.set_device(self.device)
            if ndev >= self.world:
                self.backend = "nccl"
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.device))
            else:
                self.backend = "gloo"
                dist.init_process_group("gloo")
            self.pg = dist

    @property
    def tensor_device(self):
        return f"cuda:{self.device}" if self.backend == "nccl" else None

    def barrier(self):
        if self.pg:
            self.pg.barrier()

    def allreduce(self, values, op="max"):
        if not self.pg:
            return list(values)
        import torch

        t = torch.tensor(list(values), dtype=torch.float64, device=self.tensor_device or "cpu")
        self.pg.all_reduce(t, op={"max": self.pg.ReduceOp.MAX, "sum": self.pg.ReduceOp.SUM}[op])
        return t.cpu().tolist()

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()


# ---------------------------------------------------------------------------
# our implementation


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.is_file():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def _ncu_traffic(workload):
    p = ROOT / "profiles" / "ncu_traffic.json"
    if p.is_file():
        d = json.loads(p.read_text())
        return d.get(workload)
    return None


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
        self.data = init(self.ir, n, seed)
        self.kernel = "step_nodes" if n_nodes else "step"
        if n_nodes:
            self.node_index, self.node_v = node_layout(n, n_nodes, seed)
        self.dev = None

    def setup_device(self):
        import ctypes as C

        from paper_1905_02241_b200 import runtime as rt

        r = self.runner
        self.dev = r.to_device(self.data)
        if self.n_nodes:
            nb = r.bind_nodes(self.dev, self.node_index, self.node_v)
            rt.check(rt.lib().nmodl_gather_v(C.c_void_p(nb.node_v), C.c_void_p(nb.node_index),
                                             C.c_void_p(self.dev.ptr["v"]), self.n, C.c_void_p(r.stream.handle)),
                     "gather_v")
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


# device-side head start (nmodl_spin) before host-issued timed launches: the
# per-launch ctypes overhead -- and a GIL hand-off to the NVML clock sampler
# thread (5 ms switch interval) -- must not show up as GPU idle time between
# the events
HEAD_START_NS = 12_000_000


def run_workload(name, args, dist, stream_timing=True):
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
    streams = [p.runner.stream for p in pops]
    working = sum(p.launch_bytes() for p in pops)
    flush = working < 3 * info["l2_bytes"]
    flush_buf = rt.DeviceBuffer(2 * info["l2_bytes"]) if flush else None
    s0 = streams[0]
    # all populations on one stream so the step sequence is ordered
    for p in pops:
        p.runner.stream = s0
    ev_a, ev_b = rt.Event(), rt.Event()
    K, W = args.steps, args.warmup
    for _ in range(W):
        for p in pops:
            p.launch(1)
    s0.sync()
    for p in pops:
        p.runner.check(p.dev)
    # per-kernel timing (launch duration of the dominant kernel) + step time
    per_pop_ms = [0.0] * len(pops)
    evs = [(rt.Event(), rt.Event()) for _ in pops]
    dist.barrier()
    s0.sync()
    total_ms = 0.0
    visible = os.environ.get("CUDA_VISIBLE_DEVICES")
    phys = int(visible.split(",")[dist.device]) if visible and visible.split(",")[0].isdigit() else dist.device
    with ClockSampler(phys) as clk:
        if flush:
            for _ in range(K):
                # head start so the host enqueues the whole step before the GPU reaches it
                rt.check(rt.lib().nmodl_spin(HEAD_START_NS, C_void(s0.handle)), "spin")
                rt.check(rt.lib().nmodl_l2_flush(C_void(flush_buf.ptr), flush_buf.nbytes // 8, C_void(s0.handle)), "flush")
                ev_a.record(s0)
                if len(pops) == 1:  # no inner events: the step IS the launch
                    pops[0].launch(1)
                else:
                    for j, p in enumerate(pops):
                        evs[j][0].record(s0)
                        p.launch(1)
                        evs[j][1].record(s0)
                ev_b.record(s0)
                ev_b.sync()
                step_ms = ev_a.elapsed_ms(ev_b)
                total_ms += step_ms
                for j in range(len(pops)):
                    per_pop_ms[j] += step_ms if len(pops) == 1 else evs[j][0].elapsed_ms(evs[j][1])
        else:
            graph = rt.capture(s0, lambda: [p.launch(1) for _ in range(K) for p in pops])
            ev_a.record(s0)
            graph.launch(s0)
            ev_b.record(s0)
            ev_b.sync()
            total_ms = ev_a.elapsed_ms(ev_b)
            # separate pass: per-population launch durations (same stream, events between kernels)
            for _ in range(min(K, 10)):
                rt.check(rt.lib().nmodl_spin(HEAD_START_NS, C_void(s0.handle)), "spin")
                for j, p in enumerate(pops):
                    evs[j][0].record(s0)
                    p.launch(1)
                    evs[j][1].record(s0)
                s0.sync()
                for j in range(len(pops)):
                    per_pop_ms[j] += evs[j][0].elapsed_ms(evs[j][1]) * (K / min(K, 10))
    s0.sync()
    for p in pops:
        p.runner.check(p.dev)
    clocks = clk.summary()
    dist.barrier()
    max_ms = dist.allreduce([total_ms], "max")[0]
    n_rank = sum(p.n for p in pops)
    n_all = dist.allreduce([float(n_rank)], "sum")[0]
    value = n_all * K / (max_ms / 1e3)
    # roofline of the dominant kernel (largest share of the step)
    j = int(np.argmax(per_pop_ms))
    dom = pops[j]
    dom_ms = per_pop_ms[j] / K
    peak, peak_src = _peaks()
    achieved = dom.launch_bytes() / (dom_ms / 1e3) / 1e9
    from paper_1905_02241_b200.traffic import describe

    from paper_1905_02241_b200.parallel import device_checksums, gather_checksums

    local = np.concatenate([device_checksums(p.runner, p.dev) for p in pops])
    table = gather_checksums(local, device=dist.tensor_device)
    res = {
        "value": value,
        "checksum_of_checksums": float(np.sum(table[..., 1])),
        "ms_per_step": max_ms / K,
        "n_rank": n_rank,
        "clocks": clocks,
        "gpu_launches": K * len(pops),
        "l2": "L2 flushed between timed steps" if flush else "inputs larger than L2 (no flush)",
        "roofline": {
            "bound": "hbm",
            "kernel": f"{dom.runner.mb.symbol}_k_{dom.kernel}",
            "achieved": achieved,
            "peak": peak,
            "unit": "GB/s",
            "frac": achieved / peak,
            "traffic": _ncu_traffic(name),
            "peak_source": peak_src,
            "bytes_per_launch": dom.launch_bytes(),
            "model": describe(dom.runner.abi, dom.kernel),
            "share_of_step": per_pop_ms[j] / max(sum(per_pop_ms), 1e-30),
            "launch_ms": dom_ms,
        },
        "per_mechanism": {
            p.stem: {"instances": p.n, "ms_per_launch": per_pop_ms[i] / K,
                     "GBps": p.launch_bytes() / (per_pop_ms[i] / K / 1e3) / 1e9,
                     "bytes_per_instance_step": p.launch_bytes() / p.n}
            for i, p in enumerate(pops)
        },
        "pops": pops,
    }
    return res


def run_column(args, dist):
    """configs[4]: 100k-cell synthetic column, cells partitioned over ranks by
    per-cell bytes/step (parallel.partition_cells); strong scaling."""
    from paper_1905_02241_b200 import runtime as rt
    from paper_1905_02241_b200.column import ColumnShard, ColumnSpec
    from paper_1905_02241_b200.parallel import gather_checksums, partition_cells

    spec = ColumnSpec(n_cells=WORKLOADS["column"]["cells"])
    bounds = partition_cells(np.full(spec.n_cells, spec.cell_cost()), dist.world)
    shard = ColumnShard(spec, int(bounds[dist.rank]), int(bounds[dist.rank + 1]), options_for,
                        concurrent_soma=os.environ.get("NMODL_COLUMN_SEQUENTIAL") is None)
    s0 = shard.stream
    K, W = args.steps, args.warmup
    shard.launch(W)
    s0.sync()
    shard.check()
    ev_a, ev_b = rt.Event(), rt.Event()
    graph = rt.capture(s0, lambda: shard.launch(K))
    dist.barrier()
    visible = os.environ.get("CUDA_VISIBLE_DEVICES")
    phys = int(visible.split(",")[dist.device]) if visible and visible.split(",")[0].isdigit() else dist.device
    with ClockSampler(phys) as clk:
        ev_a.record(s0)
        graph.launch(s0)
        ev_b.record(s0)
        ev_b.sync()
    ms = ev_a.elapsed_ms(ev_b)
    shard.check()
    # per-population launch durations (separate pass, events between kernels)
    from paper_1905_02241_b200.column import LAUNCH_ORDER

    # (each population's launches captured in its own graph, so host launch
    # latency does not pollute the small populations' times)
    per_pop = {}
    reps = 10
    for m in LAUNCH_ORDER:
        g = rt.capture(s0, lambda m=m: shard.runners[m].launch(shard.devs[m], "step_nodes", reps))
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
    table = gather_checksums(shard.checksums(), device=dist.tensor_device)
    peak, peak_src = _peaks()
    achieved = shard.launch_bytes() / (ms / K / 1e3) / 1e9
    return {
        "value": n_all * K / (max_ms / 1e3),
        "ms_per_step": max_ms / K,
        "n_rank": shard.n_instances,
        "clocks": clk.summary(),
        "gpu_launches": K * 7,
        "l2": "inputs larger than L2 (no flush)",
        "roofline": {"bound": "hbm", "kernel": "7 x <mech>_k_step_nodes (whole step)", "achieved": achieved,
                     "peak": peak, "unit": "GB/s", "frac": achieved / peak, "traffic": None, "peak_source": peak_src,
                     "bytes_per_launch": shard.launch_bytes()},
        "checksum_of_checksums": float(np.sum(table[..., 1])),
        "cells_per_rank": [int(b) for b in np.diff(bounds)],
        "per_mechanism": {m: {"instances": shard.devs[m].n, "ms_per_launch": per_pop[m],
                              "segments": shard.devs[m].nodes.n_segs} for m in shard.devs},
    }


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
                    phases[k] = phases.get(k, 0.0) + v

    one_call()  # warm-up (also primes graph/occupancy caches)
    phases.clear()
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(calls):
        one_call()
    dt = time.perf_counter() - t0
    phases["unaccounted"] = dt - sum(phases.values())
    dt = dist.allreduce([dt], "max")[0]
    n_all = dist.allreduce([float(sum(j[5] for j in jobs))], "sum")[0]
    return {
        "value": n_all * timesteps * calls / dt,
        "unit": UNIT,
        "h2d_bytes_per_step": int(sum(_h2d(j) for j in jobs)),
        "d2h_bytes_per_step": int(sum(_d2h(j) for j in jobs)),
        "step": f"one public-API call: pinned H2D of the store, nrn_init, {timesteps} timesteps, D2H of the store"
                + (", node_index upload + device sort, node rhs/d download" if w["nodes"] else ""),
        "timesteps_per_call": timesteps,
        "calls": calls,
        "phase_seconds_per_call": {k: v / calls for k, v in phases.items()},
    }


def _h2d(job):
    """Bytes the public call copies host->device: the whole store (v excepted
    in node mode: it is gathered from the node voltages; i_acc/g_acc are
    outputs only), node_index, node_v."""
    ir, runner, data, extra, _, n = job
    b = sum(a.nbytes for k, a in data.arrays.items() if not (extra is not None and k == "v"))
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


# ---------------------------------------------------------------------------
# CPU reference (the reference's emitted C, all host threads)


def cpu_reference(name, target_s=10.0, max_n=2_000_000, steps_cap=200):
    from oracle import ref_c
    from paper_1905_02241_b200.instance import init
    from paper_1905_02241_b200.ir import MechIR

    w = WORKLOADS[name]
    threads = os.cpu_count() or 1
    per_mech = []
    total_inst_steps = 0.0
    total_s = 0.0
    for stem, n in w["mechs"]:
        if not ref_c.available(stem):
            return None
        so = ref_c.native_build(stem)
        r = ref_c.RefC(stem, so)
        ir = MechIR.load(ROOT / "fixtures" / "ir" / f"{stem}.json")
        ns = min(n, max_n)
        data = init(ir, ns, 42)
        r.initialize(data)
        t0 = time.perf_counter()
        r.steps(data, 2, threads)
        dt1 = (time.perf_counter() - t0) / 2
        steps = int(max(2, min(steps_cap, (target_s / len(w["mechs"])) / max(dt1, 1e-6))))
        t0 = time.perf_counter()
        r.steps(data, steps, threads)
        dt = time.perf_counter() - t0
        per_mech.append(f"{stem}: {ns} instances x {steps} steps in {dt:.2f}s")
        # time-weighted combination: the population's full step is the sum of its mechanisms
        total_s += dt * (n / ns) / steps
        total_inst_steps += n
    value = total_inst_steps / total_s
    return {
        "value": value,
        "unit": UNIT,
        "cores": threads,
        "kind": "reference",
        "numpy_oracle": numpy_oracle_rate(name),
        "sample": "reference-emitted scalar C (modlc.codegen.emit_scalar, count field renamed), gcc -O3 "
                  "-march=native, contiguous shards per thread, accumulators zeroed per step; "
                  + "; ".join(per_mech)
                  + ("; no node_index scatter (the reference has none)" if w["nodes"] else ""),
        "cpu": _cpu_model(),
    }


def numpy_oracle_rate(name, n=65536, budget_s=4.0):
    """SURVEY.md §8(d) CPU leg 2: the reference's numpy runtime semantics
    (`modlc.interp.Runner`, restated bit-exactly in oracle/interp_np.py),
    single-threaded by design, on a 65,536-instance prefix of each mechanism;
    the population step is the n-weighted sum of the per-mechanism times."""
    from oracle import interp_np as O
    from paper_1905_02241_b200.ir import MechIR

    w = WORKLOADS[name]
    if not w["mechs"]:
        return None
    total_s, total_n, parts = 0.0, 0, []
    for stem, n_full in w["mechs"]:
        ir = MechIR.load(ROOT / "fixtures" / "ir" / f"{stem}.json")
        data = O.init(ir, n, 42)
        runner = O.OracleRunner(ir)
        runner.run_kernel(data, "initialize", 1)
        steps, dt = 0, 0.0
        t0 = time.perf_counter()
        while dt < budget_s / len(w["mechs"]) or steps < 2:
            runner.run_kernel(data, "state_update", 1)
            runner.run_kernel(data, "current_update", 1)
            steps += 1
            dt = time.perf_counter() - t0
        total_s += dt / steps * (n_full / n)
        total_n += n_full
        parts.append(f"{stem}: {n} x {steps} steps in {dt:.2f}s")
    return {"value": total_n / total_s, "unit": UNIT, "cores": 1,
            "sample": "oracle/interp_np.py (numpy restatement of modlc.interp.Runner), single thread; " + "; ".join(parts)}


def reference_arm(name, K, W, budget_s=60.0):
    """`--impl reference`: W untimed + K timed steps of the reference CPU path
    (emitted scalar C, all host threads).  Each step advances one timestep of
    a bounded instance sample per mechanism, sized so the whole run takes
    about `budget_s`; the full-population step time is extrapolated linearly
    in the instance count (the C loop is per-instance independent)."""
    from oracle import ref_c
    from paper_1905_02241_b200.instance import init
    from paper_1905_02241_b200.ir import MechIR

    w = WORKLOADS[name]
    threads = os.cpu_count() or 1
    mechs = w["mechs"]
    if name == "column":
        from paper_1905_02241_b200.column import LAUNCH_ORDER, ColumnSpec

        spec = ColumnSpec(n_cells=w["cells"])
        mechs = [(m, spec.n_cells * spec.instances_per_cell(m)) for m in LAUNCH_ORDER]
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
                  f"{threads} threads, per step: " + ", ".join(f"{stem} {ns} of {n} instances" for stem, n, ns, _, _ in jobs)
                  + ("; no node_index scatter (the reference has none)" if w["nodes"] else ""),
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
    args = ap.parse_args()
    dist = Dist()
    w = WORKLOADS[args.workload]
    config = {
        "workload": args.workload,
        "baseline_config": w["config"],
        "mechanisms": {stem: n for stem, n in w["mechs"]},
        "instances_per_gpu": sum(n for _, n in w["mechs"]),
        "n_nodes_per_gpu": w["nodes"],
        "dt_ms": 0.025,
        "parallelism": f"{args.gpus} x instance shard by cell (weak scaling, no per-step collective)",
    }
    if args.impl == "reference":
        if dist.rank == 0:
            K, W = args.steps, args.warmup
            ref = reference_arm(args.workload, K, W)
            line = {"impl": "reference", "metric": METRIC, "unit": UNIT, "n_gpus": args.gpus, "steps": K,
                    "warmup": W, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                    "data": "synthetic (modlc.interp.init-format seeded instance store)", "config": config}
            if ref is None:
                line.update({"unavailable": "oracle/_ref not built (needs the reference front-end)"})
            else:
                line.update({"value": ref["value"], "ms_per_step": ref["ms_per_step"],
                             "cpu_baseline": {k: ref[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu")},
                             "e2e": {"value": ref["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}})
            print(json.dumps(line), flush=True)
        dist.close()
        return
    from paper_1905_02241_b200 import runtime as rt

    rt.require_device(dist.device)
    if args.workload == "column":
        res = run_column(args, dist)
        e2e = None
        config["cells"] = WORKLOADS["column"]["cells"]
        config["instances_per_gpu"] = None
        config["parallelism"] = f"{args.gpus} x cell shard (strong scaling, no per-step collective; NCCL checksum gather)"
    else:
        res = run_workload(args.workload, args, dist)
        e2e = None if args.no_e2e else e2e_measure(args.workload, dist)
    also = {}
    if not args.no_also and args.workload != "column":
        for other in ("hh1m", "bbp20m", "kinetic1m"):
            if other == args.workload:
                continue
            # warm-up past the initial transient: Newton iteration counts
            # (cdp5ish) fall over the first ~100 steps after nrn_init
            a = argparse.Namespace(steps=min(args.steps, 50), warmup=max(args.warmup, 100))
            r = run_workload(other, a, dist)
            also[other] = {"value": r["value"], "ms_per_step": r["ms_per_step"], "l2": r["l2"],
                           "roofline": {k: r["roofline"][k] for k in ("kernel", "achieved", "peak", "frac", "bytes_per_launch", "launch_ms")},
                           "per_mechanism": r["per_mechanism"]}
            del r
    cpu = None
    if dist.rank == 0 and args.gpus == 1 and args.workload != "column":
        cpu = cpu_reference(args.workload)
    if dist.rank == 0:
        config["l2_policy"] = res["l2"]
        config["arithmetic"] = RELAXED_NOTE
        line = {
            "metric": METRIC,
            "value": res["value"],
            "unit": UNIT,
            "n_gpus": args.gpus,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": res["ms_per_step"],
            "higher_is_better": True,
            "scaling": "strong" if args.workload == "column" else "weak",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (modlc.interp.init-format seeded instance store; random node_index)",
            "config": config,
            "roofline": res["roofline"],
            "cpu_baseline": None if cpu is None else {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu", "numpy_oracle")},
            "e2e": e2e,
            "gpu_launches": res["gpu_launches"],
            "clocks": res["clocks"],
            "per_mechanism": res["per_mechanism"],
            "validation": {"checksum_of_checksums": res.get("checksum_of_checksums"),
                           "how": "per-array sum|x| on each GPU (fixed-tree device reduction), all-gathered with NCCL"},
            "also": also,
        }
        print(json.dumps(line), flush=True)
    dist.close()


if __name__ == "__main__":
    main()
