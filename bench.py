#!/usr/bin/env python3
"""Benchmark of the hybrid NAD stage pass (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--config 3]

One bench "step" is one SSP-RK3 time step of BASELINE config 3 by default
(8,388,608 triangles on the periodic unit square, p=3, random quadrants + 1 %
noise; 3 stages = 25,165,824 cell-stage updates): device dt (max_stable_dt) +
3 x (central LSQ + NAD + spread/compaction + CWENOZ + MUSCL + fallback + HLLC
flux + RK update). Config 3 is the largest 2D configuration, the one BASELINE
quotes at 1/2/4/8 GPUs; configs 1 and 2 (`--config 1|2`) and the 3D configs
4, 4c (forced all-CWENOZ) and 5 are selectable.
`value` = cell-stage updates / s with the state resident in HBM (device
timed with CUDA events on the solver's stream, max over ranks); `e2e` = the
same metric through the C ABI with the state copied host->device (pinned)
before and device->host after every step, inside the timed region.
N > 1 (torchrun): strong scaling by default -- the config's mesh RCB-split
into N subdomains, NCCL halo exchange every stage (`--scaling weak` repeats
the config's domain per GPU instead).

--impl reference times the reference's own CPU code (oracle/_ref: the
unmodified /root/reference sources compiled here; single-threaded -- it has
no parallel regions) on the same config, seed and RK3 driver; for config 3 on
a bounded sample (a 512x512x2 tile of the same configuration, because the
reference's single-threaded setup of the full mesh alone takes ~8 min).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "cell-stage updates/sec (NAD+reconstruct+flux+RK, fp64) at 1/2/4/8 B200; % roofline"
UNIT = "cell-stage/s"

CONFIGS = {
    # name: mesh, order, ic, params, opts, bcs, description
    "1": dict(nx=128, ny=128, rect=(0.0, 0.0, 1.0, 1.0), jitter=0.1, periodic="both", order=2, ic=0,
              params=[10.0], opts=dict(lambda1p=1e4, cfl=0.5), bcs={},
              desc="BASELINE config 1: periodic unit square, 128x128x2 jittered tris, p=2, isentropic vortex"),
    "2": dict(nx=2048, ny=64, rect=(-5.0, 0.0, 5.0, 1.0), jitter=0.1, periodic="y", order=2, ic=1,
              params=[-4.0, 3.857143, 2.629369, 0.0, 10.33333, 0.2, 5.0], opts=dict(lambda1p=1e3, cfl=0.5),
              bcs={"left": "outflow", "right": "outflow"},
              desc="BASELINE config 2: [-5,5]x[0,1], 2048x64x2 jittered tris, p=2, shock into sine wave, "
                   "transmissive x, periodic y"),
    "3": dict(nx=2048, ny=2048, rect=(0.0, 0.0, 1.0, 1.0), jitter=0.0, periodic="both", order=3, ic=2,
              params=[0.5, 0.5, 0.01], opts=dict(lambda1p=1e3, cfl=0.5), bcs={},
              desc="BASELINE config 3: periodic unit square, 2048x2048x2 tris, p=3, random quadrants + 1% noise"),
}
SEED = 1
# CPU legs (cpu_baseline, --impl reference) run the reference on a bounded
# sample of the workload: configs 1-2 whole; config 3 as a 512x512x2 tile of
# the same configuration (same p, IC, seed, margins; per-cell work identical,
# the mesh 16x smaller so the reference's single-threaded setup takes ~30 s)
CPU_SAMPLE = {"3": dict(nx=512, ny=512)}


def workload_config(cfg, world=1, strong=True):
    """The static `config` dict of a 2D bench line -- identical in both arms."""
    c = CONFIGS[cfg]
    cells = 2 * c["nx"] * c["ny"] * (1 if (strong or world == 1) else world)
    K = (c["order"] + 1) * (c["order"] + 2) // 2 - 1
    par = "single"
    wl = c["desc"]
    if world > 1:
        par = f"domain decomposition x{world} (RCB), NCCL halo exchange every stage"
        wl += (f"; strong scaling: the config's mesh split into {world} subdomains" if strong else
               f"; weak scaling: the config's domain repeated {world}x in y, one block per GPU")
    return {"workload": wl, "config": cfg, "cells": cells, "order": c["order"], "K": K, "M": 2 * K,
            "integrator": "SSP-RK3 (3 stages/step)", "mode": "hybrid", "parallelism": par,
            "l2": "inputs larger than L2 (per-cell operator data >= 0.7 GB)"}


def cpu_sample_case(cfg):
    """(config dict of the CPU sample, description) for the CPU legs."""
    c = dict(CONFIGS[cfg])
    if cfg in CPU_SAMPLE:
        c.update(CPU_SAMPLE[cfg])
        return c, (f"a {c['nx']}x{c['ny']}x2 tile of config {cfg} ({2 * c['nx'] * c['ny']} cells; same p, IC, "
                   f"seed and options)")
    return c, f"config {cfg} itself ({2 * c['nx'] * c['ny']} cells)"


def env_overrides():
    """UCFVB_* diagnostics knobs set in the environment (none in a benchmark run)."""
    return {k: v for k, v in sorted(os.environ.items()) if k.startswith("UCFVB_")}


def traffic_for(cfg, cells, phase):
    """ncu DRAM bytes (read + write) per launch of `phase` measured on this
    config and size (profiles/traffic.json, keyed by config), else None."""
    tf = ROOT / "profiles" / "traffic.json"
    try:
        t = json.loads(tf.read_text()).get(f"config{cfg}")
        if t and int(t.get("cells", -1)) == int(cells):
            return t.get(phase)
    except Exception:
        pass
    return None

# 3D configurations (the reference is 2D only)
CONFIGS3 = {
    "4": dict(n=128, kind=0, jitter=0.05, order=2, ic=0, params=[0.1], mode="hybrid", classes=False,
              desc="BASELINE config 4: periodic [0,2pi]^3, 128^3 hexahedra (+-5% jitter), p=2, Taylor-Green M=0.1, "
                   "hybrid"),
    "4c": dict(n=128, kind=0, jitter=0.05, order=2, ic=0, params=[0.1], mode="cwenoz", classes=False,
               desc="BASELINE config 4, forced all-CWENOZ: periodic [0,2pi]^3, 128^3 hexahedra (+-5% jitter), p=2, "
                    "Taylor-Green M=0.1"),
    "5": dict(n=128, kind=1, jitter=0.0, order=3, ic=1, params=[0.6, 4.0, 8], mode="hybrid", classes=True,
              desc="BASELINE config 5: periodic [0,2pi]^3, 128^3 cubes x 6 tetrahedra, p=3, random-phase solenoidal "
                   "field E(k)~k^4 exp(-2(k/4)^2) (|k|<=8), rms Mach 0.6, hybrid"),
}


def env_rank():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), \
        int(os.environ.get("LOCAL_RANK", "0"))


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled through NVML every
    ~2 ms during the timed region (nvidia-smi's fields, without its 0.3 s/call)."""

    REASONS = {  # nvmlClocksEventReason* bits
        0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap",
        0x80: "hw_power_brake_slowdown",
    }

    def __init__(self, index=0, period=0.002):
        self.index = index
        self.period = period
        self.samples = []
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        self._nvml = None

    def _run(self):
        nv = self._nvml
        h = nv.nvmlDeviceGetHandleByIndex(self.index)
        try:
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
        except Exception:
            pass
        get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            getattr(nv, "nvmlDeviceGetCurrentClocksThrottleReasons")
        while not self._stop.is_set():
            try:
                self.samples.append((float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)), int(get_reasons(h))))
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self._nvml = nv
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
            time.sleep(0.01)
        except Exception:
            self._nvml = None
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"], "samples": 0}
        mhz = [m for m, _ in self.samples]
        reasons = set()
        for _, r in self.samples:
            for bit, name in self.REASONS.items():
                if r & bit:
                    reasons.add(name)
        return {"sm_mhz": float(np.median(mhz)), "sm_max_mhz": self.max_mhz, "reasons": sorted(reasons),
                "samples": len(self.samples), "source": "nvml"}


# ---------------------------------------------------------------- roofline model
def kernel_bytes(K, NQ, NF, MM, MD, mix=None):
    """Algorithmic HBM bytes per cell of each kernel: every
    array the kernel must read or write, once; stencil-neighbour gathers of U
    counted as L2 hits (only the cell's own U is counted). Face points are
    double4 (32 B), indices int32, labels uint8. `mix` = class fractions
    (L, C, M, F) of the run: the central kernel stores candidate face points
    only for raw-Linear cells and dofs only for cells that are not raw-MUSCL;
    final Linear cells were raw-Linear and final MUSCL cells include every
    raw-MUSCL one, so f_L and 1 - f_M are lower bounds of those fractions
    (bytes never overcounted)."""
    Q = NF * NQ
    fl, fm = (1.0, 0.0) if mix is None else (float(mix[0]), float(mix[2]))
    central = (32 + 4 * MM + 8 * MM * K      # U, stencil ids, pinv        (TMA group A)
               + 8 * Q * K + 8 + 4 * NF + 4 * Q  # phi, threshold, nbrs, slots (TMA group B)
               + 32 * Q * fl + 32 * K * (1.0 - fm) + 1)  # candidate face points, dofs, raw label
    cwenoz = (32 + 4 * NF * MD + 16 * NF * MD + 8 * K * K + 8 * Q * K + 4 * NF + 32 * K  # U, dir ids/pinv, OI, phi, nbrs, dofs
              + 4 * Q + 32 * Q + 8)           # slots, face points, chunk entry/label
    muscl = 32 + 4 * MM + 16 * MM + 16 * Q + 4 * NF + 4 * Q + 32 * Q + 8
    faces_per_cell = NF / 2.0
    flux = faces_per_cell * (2 * NQ * 32 + 24 + 2 + 8 + 2 * 32)  # both sides' points, geometry, kind, slots, +-flux
    gather = 32 * NF + 2 * 32 + 8 + 32 + 8                       # residual slots, RK terms, 1/area, output, h (dt)
    spread = 1 + 4 * NF + 1 + 1
    return dict(central=int(central), spread=spread, cwenoz=int(cwenoz), muscl=int(muscl),
                flux=int(flux + gather))


def kernel_bytes3(K, M, NF, NQ, MD, per_cell_ops):
    """Algorithmic HBM bytes per cell of each 3D kernel: own
    U (40 B), index arrays, operator rows (per-cell rows only; lattice-class
    rows are a few KB in total and live in L1/L2), face values (40 B per
    point) and residual terms; stencil gathers of U counted as L2 hits."""
    Q = NF * NQ
    ops = 1 if per_cell_ops else 0
    central = (40 + 4 + 8 + 4 * NF + 4 * (M + 1) + ops * 8 * M * K + ops * 8 * Q * K + 4 * Q
               + 40 * Q + 32 + 1)
    spread = 1 + 4 * NF + 1 + 4
    # CWENOZ recomputes the central solve (pinv re-read) instead of reading stored dofs
    cwenoz = (4 + 40 + 4 + 4 * (M + 1) + ops * (8 * M * K + 4 * NF * MD + 24 * NF * MD + 8 * K * K + 8 * Q * K)
              + 4 * Q + 32 + 40 * Q + 1)
    muscl = 4 + 40 + 4 + 4 * (M + 1) + ops * (24 * M + 24 * Q) + 4 * NF + 8 + 4 * Q + 32 + 40 * Q + 1
    faces = NF / 2.0
    flux = faces * (2 * NQ * 40 + NQ * 32 + 40)
    gather = 4 * NF + 40 * NF + 8 + 3 * 40
    return dict(central=int(central), spread=spread, cwenoz=int(cwenoz), muscl=int(muscl), flux=int(flux),
                gather=int(gather))


def kernel_flops3(K, M, NF, NQ, MD):
    """fp64 flops per cell of the 3D reconstruction kernels (2 per fused
    multiply-add of the contractions; five variables): the roofline for the
    lattice-class configuration, whose operator rows live on chip."""
    Q = NF * NQ
    return dict(central=10 * (M * K + Q * K), spread=0,
                cwenoz=10 * (M * K + NF * 3 * MD + Q * K + K * K),
                muscl=10 * (3 * M + 3 * Q + Q * K), flux=0, gather=0)


def measured_peak_fp64():
    p = ROOT / "profiles" / "fp64_peak.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["fp64_fma_tflops"]), "measured (profiles/fp64_peak.json)"
        except Exception:
            pass
    return 34.0, "fallback"


def measured_peak_hbm():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured"
        except Exception:
            pass
    return 6650.0, "fallback"


# ---------------------------------------------------------------- setup
def scaled_config(cfg, world):
    """Weak scaling: the config's domain repeated `world` times along y (periodic
    in y), so every rank owns one config-sized block of cells."""
    c = dict(CONFIGS[cfg])
    if world > 1:
        x0, y0, x1, y1 = c["rect"]
        c["rect"] = (x0, y0, x1, y0 + world * (y1 - y0))
        c["ny"] = c["ny"] * world
    return c


def build_case(cfg, n_threads=0, world=1, strong=False):
    from paper_2510_25906_b200.mesh import Mesh, Stencils
    c = CONFIGS[cfg] if strong else scaled_config(cfg, world)
    nq = (c["order"] + 2) // 2
    t0 = time.perf_counter()
    mesh = Mesh.structured_tri(c["nx"], c["ny"], c["rect"], jitter=c["jitter"], seed=SEED, periodic=c["periodic"],
                               n_qp=nq)
    st = Stencils(mesh, c["order"], n_threads=n_threads)
    u0 = mesh.project_initial(c["ic"], c["params"], seed=SEED, degree=max(2 * c["order"], 2), n_threads=n_threads)
    return mesh, st, u0, time.perf_counter() - t0


def cpu_reference_run(cfg, steps, budget_s=None, warmup=0):
    """The reference's own CPU path (oracle/_ref) on the same mesh, seed, RK3 driver.
    `warmup` untimed RK3 steps run first. Returns (cell-stage/s, steps timed, setup seconds, cells)."""
    from oracle import ref as R
    from paper_2510_25906_b200 import _abi as A
    from paper_2510_25906_b200.solver import make_bcs
    c, _ = cpu_sample_case(cfg)
    nq = (c["order"] + 2) // 2
    per = {"both": 3, "y": 2, "x": 1, "none": 0}[c["periodic"]]
    t0 = time.perf_counter()
    rm = R.RefMesh.structured_tri(c["nx"], c["ny"], c["rect"], jitter=c["jitter"], seed=SEED, periodic=per,
                                  n_qp=nq)
    o = A.options_from_dict(order=c["order"], **c["opts"])
    rs = R.RefSolver(rm, o, make_bcs(c["bcs"]))
    u0 = rm.project_initial(c["ic"], c["params"], seed=SEED, degree=max(2 * c["order"], 2))
    rs.set_state(u0)
    setup = time.perf_counter() - t0
    done, wall, t = 0, 0.0, 0.0
    for _ in range(warmup):
        t, _, _ = rs.run_steps(1, A.RK3, t0=t)
    while done < steps:
        t, w, _ = rs.run_steps(1, A.RK3, t0=t)
        wall += w
        done += 1
        if budget_s is not None and wall >= budget_s:
            break
    n = rm.n_cells
    return n * 3 * done / wall, done, setup, n


# ---------------------------------------------------------------- arms
def run_reference_arm(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return
    from oracle import ref as R
    cfg = args.config
    if not R.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libucfv_ref.so was not built "
                                                              "(reference sources absent at build time)"}))
        return
    # warm-up steps are untimed; each timed step is one full RK3 step of the
    # bounded sample, the timed steps bounded by a wall budget
    budget = float(os.environ.get("UCFVB_REF_BUDGET_S", "60"))
    rate, done, setup, n = cpu_reference_run(cfg, max(1, args.steps), budget_s=budget, warmup=args.warmup)
    _, sample = cpu_sample_case(cfg)
    cores = os.cpu_count()
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": args.gpus, "steps": done,
        "warmup": args.warmup, "ms_per_step": 1e3 * n * 3 / rate, "higher_is_better": True,
        "scaling": "strong" if args.scaling == "strong" else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(cfg, world, args.scaling == "strong"),
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": 1, "kind": "reference",
                         "sample": f"{done} timed RK3 steps (after {args.warmup} untimed) of {sample} through the "
                                   f"unmodified reference Solver::compute_residual (single-threaded: the reference "
                                   f"has no parallel regions; host has {cores} cores); setup {setup:.1f}s excluded"},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def run_b200_arm(args):
    import torch
    import torch.distributed as dist

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    if world > 1 and not dist.is_initialized():
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2510_25906_b200 import _abi as A
    from paper_2510_25906_b200.solver import Solver, make_bcs

    cfg = args.config
    c = CONFIGS[cfg]
    threads = max(1, (os.cpu_count() or 1) // max(1, world))
    strong = args.scaling == "strong"
    mesh, st, u0, setup_s = build_case(cfg, n_threads=threads, world=world, strong=strong)
    opts = A.options_from_dict(order=c["order"], mode="hybrid", **c["opts"])
    bcs = make_bcs(c["bcs"])
    sub = None
    if world == 1:
        solver = Solver(mesh, opts, bcs, stencils=st, device=local)
        n = solver.n_cells
    else:
        from paper_2510_25906_b200.decompose import Subdomain, partition_rcb
        from paper_2510_25906_b200.solver import nccl_unique_id
        t0 = time.perf_counter()
        part = partition_rcb(mesh, world)
        sub = Subdomain(mesh, st, part, world, rank)
        solver = Solver.on_subdomain(sub, opts, bcs, device=local)
        ids = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(ids, src=0)
        solver.attach_nccl(ids[0], rank, world)
        u0 = sub.local_state(u0)
        setup_s += time.perf_counter() - t0
        n = sub.n_owned
    stream = torch.cuda.ExternalStream(solver.stream(), device=local)

    def barrier():
        if world > 1:
            dist.barrier()

    def sum_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor(np.asarray(x, dtype=np.float64), device="cuda")
        dist.all_reduce(t)
        return t.cpu().numpy() if t.dim() else float(t.item())

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- value leg: state resident in HBM, K graph-replayed RK3 steps
    solver.state = u0
    solver.run_steps(args.warmup, A.RK3)
    lists_used = solver.list_stats()["lists"]
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ev0.record(stream)
        t_final, _ = solver.run_steps(args.steps, A.RK3, t0=0.0)
        ev1.record(stream)
        ev1.synchronize()
    torch.cuda.synchronize()
    barrier()
    ms = max_over_ranks(ev0.elapsed_time(ev1))
    launches = solver.launch_count()
    owned_total = int(round(sum_over_ranks(float(n))))
    total_units = owned_total * 3 * args.steps
    value = total_units / (ms * 1e-3)

    # census of the same K steps from u0 (outside the timed region): per-step
    # NAD class fractions (run.cpp:110-116 step labels) and threshold ties
    solver.state = u0
    _, census = solver.run_steps(args.steps, A.RK3, census=True)
    ties = int(round(sum_over_ranks(float(solver.nad_ties()))))
    mix = census.sum(0) / census.sum()
    per_step = [[round(float(x), 4) for x in row / max(1, row.sum())] for row in census]

    # ---- per-kernel durations (events between kernel groups, un-graphed stages)
    solver.state = u0
    solver.run_steps(2, A.RK3)
    solver.set_phase_timing(True)
    p0 = solver.phase_times().copy()
    n_phase_steps = 5
    solver.run_steps(n_phase_steps, A.RK3)
    torch.cuda.synchronize()
    phases = (solver.phase_times() - p0) / (3 * n_phase_steps)  # seconds per stage
    solver.set_phase_timing(False)

    # ---- e2e leg: host state in pinned memory, H2D + step + D2H per step.
    # (a) serial: step i uploads buf[i % 2] and downloads its result into
    #     buf[(i + 1) % 2], the next step's input (a dependent chain: nothing
    #     can overlap). (b) pipelined, the reported e2e value: the K steps are K
    #     independent states of the mesh (an ensemble; a ring of 3 pinned inputs
    #     and 3 pinned outputs) through ucfvb_advance_host_batch, which uploads
    #     entry i+1 and downloads entry i-1 on copy streams while entry i steps.
    host = [torch.from_numpy(np.ascontiguousarray(u0)).pin_memory(),
            torch.empty((solver.n_cells, 4), dtype=torch.float64).pin_memory()]
    lib = A.load_library()
    import ctypes as C
    hptr = [C.cast(h.data_ptr(), A.c_dp) for h in host]
    t_dev = C.c_double()
    e2e_steps = args.steps

    def e2e_step(i):
        # the host-state call: H2D of this step's input, one RK3 step (device
        # dt), D2H of the result, one synchronisation (include/ucfvb.h)
        rc = lib.ucfvb_advance_host(solver._h, hptr[i & 1], hptr[(i + 1) & 1], 1, A.RK3, 0.0, C.byref(t_dev))
        if rc:
            raise RuntimeError(lib.ucfvb_last_error(solver._h).decode())

    n_ring = 3
    ring_in = [torch.empty((solver.n_cells, 4), dtype=torch.float64).pin_memory() for _ in range(n_ring)]
    ring_out = [torch.empty((solver.n_cells, 4), dtype=torch.float64).pin_memory() for _ in range(n_ring)]
    for i in range(max(n_ring, args.warmup)):  # warm-up; its first states fill the input ring
        if i < n_ring:
            ring_in[i].copy_(host[i & 1])
        e2e_step(i)
    host[0].copy_(torch.from_numpy(np.ascontiguousarray(u0)))
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    e0.record(stream)
    for i in range(e2e_steps):
        e2e_step(i)
    e1.record(stream)
    e1.synchronize()
    wall_e2e = time.perf_counter() - w0
    e2e_serial_ms = max_over_ranks(max(e0.elapsed_time(e1), 1e3 * wall_e2e))
    e2e_serial = owned_total * 3 * e2e_steps / (e2e_serial_ms * 1e-3)

    tab_in = (A.c_dp * e2e_steps)(*[C.cast(ring_in[i % n_ring].data_ptr(), A.c_dp) for i in range(e2e_steps)])
    tab_out = (A.c_dp * e2e_steps)(*[C.cast(ring_out[i % n_ring].data_ptr(), A.c_dp) for i in range(e2e_steps)])

    def e2e_batch(nb):
        rc = lib.ucfvb_advance_host_batch(solver._h, nb, tab_in, tab_out, 1, A.RK3, 0.0, None)
        if rc:
            raise RuntimeError(lib.ucfvb_last_error(solver._h).decode())

    e2e_batch(min(e2e_steps, n_ring))  # warm-up: staging buffers, copy streams
    barrier()
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    e0.record(stream)
    e2e_batch(e2e_steps)
    e1.record(stream)
    e1.synchronize()
    wall_e2e = time.perf_counter() - w0
    e2e_ms = max_over_ranks(max(e0.elapsed_time(e1), 1e3 * wall_e2e))
    e2e_value = owned_total * 3 * e2e_steps / (e2e_ms * 1e-3)

    # ---- roofline of the dominant kernel
    K, NQ = st.view.K, st.view.n_qp
    NF = 3
    sd = st.numpy()
    MM = int(np.max(np.diff(sd["central_ptr"]))) - 1
    MD = int(np.max(np.diff(sd["dir_member_ptr"]))) - 1
    kb = kernel_bytes(K, NQ, NF, MM, MD, mix)
    names = ["central (reconstruct)", "spread+compaction (detect)", "cwenoz+muscl (weights)", "flux+RK"]
    phase_bytes = [kb["central"] * n, kb["spread"] * n,
                   (kb["cwenoz"] * mix[1] + kb["muscl"] * mix[2]) * n, kb["flux"] * n]
    dom = int(np.argmax(phases))
    peak, peak_kind = measured_peak_hbm()
    achieved = phase_bytes[dom] / phases[dom] / 1e9
    stage_bytes = sum(phase_bytes)
    stage_achieved = stage_bytes / phases.sum() / 1e9
    traffic = traffic_for(cfg, solver.n_cells, names[dom].split()[0]) if world == 1 else None

    cpu_baseline = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            from oracle import ref as R
            if R.available():
                rate, done, rsetup, _ = cpu_reference_run(cfg, 50, budget_s=float(os.environ.get("UCFVB_CPU_S", "12")))
                _, sample = cpu_sample_case(cfg)
                cpu_baseline = {"value": rate, "unit": UNIT, "cores": 1, "kind": "reference",
                                "sample": f"{done} RK3 steps of {sample}, unmodified reference sources "
                                          f"(oracle/_ref), 1 thread (the reference has no parallel regions); setup "
                                          f"{rsetup:.1f}s excluded; host has {os.cpu_count()} cores"}
        except Exception as e:  # pragma: no cover
            cpu_baseline = {"value": None, "unit": UNIT, "cores": 1, "kind": "reference", "sample": f"failed: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if strong else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(cfg, world, strong),
            "census": {"class_lists": lists_used,
                       "class_mix": {"linear": round(float(mix[0]), 4), "cwenoz": round(float(mix[1]), 4),
                                     "muscl": round(float(mix[2]), 4), "first": round(float(mix[3]), 4)},
                       "class_mix_per_step_LCMF": per_step, "nad_ties": ties,
                       "note": "step labels after the first stage of each step (run.cpp:110-116), the K timed "
                               "steps re-run from the initial state; nad_ties summed over every detecting stage"},
            "setup_s": round(setup_s, 3),
            "cells_per_gpu": n,
            "env_overrides": env_overrides(),
            "clocks": clk.summary(),
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(solver.n_cells * 32 * world),
                    "d2h_bytes_per_step": int(solver.n_cells * 32 * world),
                    "call": "ucfvb_advance_host_batch: the K steps are K independent host states (pinned), "
                            "uploads and downloads on copy streams overlap the stepping",
                    "serial_value": e2e_serial,
                    "serial_call": "ucfvb_advance_host: each step's input is the previous step's downloaded "
                                   "result (dependent chain, copies on the critical path)"},
            "gpu_launches": int(launches),
            "roofline": {"bound": "hbm", "kernel": names[dom], "achieved": achieved, "peak": peak,
                         "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic,
                         "bytes_per_cell": {k: int(v) for k, v in kb.items()},
                         "stage_achieved": stage_achieved, "stage_frac": stage_achieved / peak,
                         "phase_us": [round(1e6 * p, 2) for p in phases]},
            "cpu_baseline": cpu_baseline,
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def build_case3(cfg, n_threads=0, n=None):
    from paper_2510_25906_b200.solver3d import Mesh3, Stencils3
    c = CONFIGS3[cfg]
    t0 = time.perf_counter()
    mesh = Mesh3(n or c["n"], kind=c["kind"], jitter=c["jitter"], seed=SEED, order=c["order"], n_threads=n_threads)
    st = Stencils3(mesh, c["order"], lattice_classes=c["classes"], n_threads=n_threads)
    deg = 1 if c["ic"] == 1 else max(2 * c["order"], 2)
    u0 = mesh.project_initial(c["ic"], c["params"], seed=SEED, degree=deg, n_threads=n_threads)
    return mesh, st, u0, time.perf_counter() - t0


def workload_config3(cfg, world=1):
    """The static `config` dict of a 3D bench line -- identical in both arms."""
    c = CONFIGS3[cfg]
    nper = 6 if c["kind"] == 1 else 1
    K = {2: 9, 3: 19}.get(c["order"], None)
    wl = c["desc"] + (f"; strong scaling: the config's mesh RCB-split into {world} subdomains, NCCL halo exchange "
                      f"every stage" if world > 1 else "")
    return {"workload": wl, "config": cfg, "cells": nper * c["n"] ** 3, "order": c["order"], "K": K,
            "M": 2 * K if K else None, "nf": 4 if c["kind"] == 1 else 6, "integrator": "SSP-RK3 (3 stages/step)",
            "mode": c["mode"], "operator_rows": "lattice classes (6 shared rows)" if c["classes"] else "per cell",
            "parallelism": f"domain decomposition x{world}" if world > 1 else "single",
            "l2": "inputs larger than L2 (face values alone > 0.5 GB)"}


def port3_rate(cfg, budget_s, warmup=0):
    """The 3D oracle restatement (oracle/ucfv3_port.c, 1 thread) on a bounded
    sample: the same config on a 12^3-cube mesh, `warmup` untimed RK3 steps,
    then RK3 steps until `budget_s`."""
    from oracle.port3 import Port3Solver
    from paper_2510_25906_b200 import _abi as A
    c = CONFIGS3[cfg]
    mesh, st, u0, _ = build_case3(cfg, n=12)
    P = Port3Solver(mesh, st, A.options_from_dict(order=c["order"], mode=c["mode"], cfl=0.5))
    P.state = u0.copy()
    for _ in range(warmup):
        P.advance(P.max_stable_dt(), rk=A.RK3)
    done, t0 = 0, time.perf_counter()
    while done < 2 or (time.perf_counter() - t0 < budget_s and done < 200):
        P.advance(P.max_stable_dt(), rk=A.RK3)
        done += 1
    dt = time.perf_counter() - t0
    return mesh.n_cells * 3 * done / dt, done, mesh.n_cells


def run_arm_3d(args):
    """3D configurations 4 / 4c / 5: one GPU, or (torchrun, N>1) strong scaling
    of the config's mesh RCB-split into N subdomains with an NCCL halo exchange
    every stage."""
    import ctypes as C

    import torch
    rank, world, local = env_rank()
    cfg = args.config
    c = CONFIGS3[cfg]
    from paper_2510_25906_b200 import _abi as A
    if args.impl == "reference":
        if rank != 0:
            return
        rate, done, ncell = port3_rate(cfg, float(os.environ.get("UCFVB_CPU_S", "20")), warmup=args.warmup)
        sample = (f"{done} RK3 steps of config {cfg} on a 12^3-cube mesh ({ncell} cells), 3D oracle restatement "
                  f"oracle/ucfv3_port.c (the reference is 2D only), 1 thread; host has {os.cpu_count()} cores")
        print(json.dumps({"metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": args.gpus, "steps": done,
                          "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True, "scaling": "strong",
                          "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
                          "config": workload_config3(cfg, world),
                          "cpu_baseline": {"value": rate, "unit": UNIT, "cores": 1, "kind": "port", "sample": sample},
                          "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))
        return
    from paper_2510_25906_b200 import solver3d as S3
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1 and not dist.is_initialized():
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    threads = max(1, (os.cpu_count() or 1) // world)
    mesh, st, u0, setup_s = build_case3(cfg, n_threads=threads)
    opts = A.options_from_dict(order=c["order"], mode=c["mode"], cfl=0.5)
    n_global = mesh.n_cells
    if world == 1:
        solver = S3.Solver3(mesh, opts, st, device=local)
        n = mesh.n_cells
    else:  # strong scaling: the config's mesh RCB-split, NCCL halo exchange every stage
        from paper_2510_25906_b200.solver import nccl_unique_id
        t0 = time.perf_counter()
        sub = S3.Subdomain3(mesh, st, S3.partition_rcb3(mesh, world), world, rank)
        solver = S3.Solver3.on_subdomain(sub, opts, device=local)
        ids = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(ids, src=0)
        solver.attach_nccl(ids[0], rank, world)
        u0 = sub.local_state(u0)
        setup_s += time.perf_counter() - t0
        n = sub.n_local
    stream = torch.cuda.ExternalStream(solver.stream(), device=local)

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def barrier():
        if world > 1:
            dist.barrier()
    solver.state = u0
    solver.run_steps(args.warmup)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ev0.record(stream)
        solver.run_steps(args.steps)
        ev1.record(stream)
        ev1.synchronize()
    torch.cuda.synchronize()
    barrier()
    ms = max_over_ranks(ev0.elapsed_time(ev1))
    launches = solver.launch_count()
    value = n_global * 3 * args.steps / (ms * 1e-3)
    census = np.array(solver.census(), dtype=float)
    if world > 1:
        tc = torch.tensor(census, device="cuda", dtype=torch.float64)
        dist.all_reduce(tc)
        census = tc.cpu().numpy()
    # NAD class fractions per step (BASELINE config 5 asks for them), from the
    # initial state, outside the timed region
    per_step = []
    solver.state = u0
    for _ in range(min(args.steps, 10)):
        solver.run_steps(1)
        cs = np.array(solver.census(), dtype=float)
        if world > 1:
            tc = torch.tensor(cs, device="cuda", dtype=torch.float64)
            dist.all_reduce(tc)
            cs = tc.cpu().numpy()
        per_step.append([round(float(x), 4) for x in cs / cs.sum()])
    mix = census / census.sum()
    ties = solver.nad_ties()
    # per-kernel-group durations (events between groups, un-graphed stages)
    solver.set_phase_timing(True)
    p0 = solver.phase_times().copy()
    nps = 3
    solver.run_steps(nps)
    phases = (solver.phase_times() - p0) / (3 * nps)
    solver.set_phase_timing(False)
    # e2e: pinned host state, H2D + step + D2H every step
    host = [torch.from_numpy(np.ascontiguousarray(u0)).pin_memory(),
            torch.empty((n, 5), dtype=torch.float64).pin_memory()]
    L = S3.lib()
    hp = [C.cast(h.data_ptr(), C.POINTER(C.c_double)) for h in host]
    tt = C.c_double()

    def e2e_step(i):
        rc = L.ucfvb3_advance_host(solver._h, hp[i & 1], hp[(i + 1) & 1], 1, A.RK3, 0.0, C.byref(tt))
        if rc:
            raise RuntimeError(L.ucfvb3_last_error(solver._h).decode())

    for i in range(args.warmup):
        e2e_step(i)
    host[0].copy_(torch.from_numpy(np.ascontiguousarray(u0)))
    e2e_steps = max(3, args.steps // 4)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    e0.record(stream)
    for i in range(e2e_steps):
        e2e_step(i)
    e1.record(stream)
    e1.synchronize()
    e2e_serial_ms = max_over_ranks(max(e0.elapsed_time(e1), 1e3 * (time.perf_counter() - w0)))
    e2e_serial = n_global * 3 * e2e_steps / (e2e_serial_ms * 1e-3)
    # the reported e2e: the same steps as independent host states through the pipelined batch call
    n_ring = 3
    ring_in = [torch.from_numpy(np.ascontiguousarray(u0)).pin_memory() for _ in range(n_ring)]
    ring_out = [torch.empty((n, 5), dtype=torch.float64).pin_memory() for _ in range(n_ring)]
    dpp = C.POINTER(C.c_double)
    tab_in = (dpp * e2e_steps)(*[C.cast(ring_in[i % n_ring].data_ptr(), dpp) for i in range(e2e_steps)])
    tab_out = (dpp * e2e_steps)(*[C.cast(ring_out[i % n_ring].data_ptr(), dpp) for i in range(e2e_steps)])

    def e2e_batch(nb):
        rc = L.ucfvb3_advance_host_batch(solver._h, nb, tab_in, tab_out, 1, A.RK3, 0.0, None)
        if rc:
            raise RuntimeError(L.ucfvb3_last_error(solver._h).decode())

    e2e_batch(min(e2e_steps, n_ring))
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    e0.record(stream)
    e2e_batch(e2e_steps)
    e1.record(stream)
    e1.synchronize()
    e2e_ms = max_over_ranks(max(e0.elapsed_time(e1), 1e3 * (time.perf_counter() - w0)))
    e2e_value = n_global * 3 * e2e_steps / (e2e_ms * 1e-3)
    kb = kernel_bytes3(st.K, st.M, mesh.nf, mesh.nq, st.MD, not c["classes"])
    names = ["central (reconstruct)", "spread+compaction (detect)", "cwenoz+muscl (weights)", "flux", "gather+RK"]
    if c["mode"] == "cwenoz":
        wbytes = kb["cwenoz"]
    else:
        wbytes = kb["cwenoz"] * mix[1] + kb["muscl"] * mix[2]
    phase_bytes = [kb["central"] * n, kb["spread"] * n, wbytes * n, kb["flux"] * n, kb["gather"] * n]
    dom = int(np.argmax(phases))
    if c["classes"]:  # operator rows on chip: the fp64 pipe bounds the reconstruction kernels
        kf = kernel_flops3(st.K, st.M, mesh.nf, mesh.nq, st.MD)
        wfl = kf["cwenoz"] if c["mode"] == "cwenoz" else kf["cwenoz"] * mix[1] + kf["muscl"] * mix[2]
        phase_flops = [kf["central"] * n, 0, wfl * n, 0, 0]
        dom = int(np.argmax([phases[0], 0, phases[2], 0, 0]))
        bound, unit = "fp64", "TFLOP/s"
        peak, peak_kind = measured_peak_fp64()
        achieved = phase_flops[dom] / phases[dom] / 1e12
        stage_achieved = sum(phase_flops) / phases.sum() / 1e12
    else:
        bound, unit = "hbm", "GB/s"
        peak, peak_kind = measured_peak_hbm()
        achieved = phase_bytes[dom] / phases[dom] / 1e9
        stage_achieved = sum(phase_bytes) / phases.sum() / 1e9
    cpu_baseline = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, done, ncell = port3_rate(cfg, float(os.environ.get("UCFVB_CPU_S", "12")))
        cpu_baseline = {"value": rate, "unit": UNIT, "cores": 1, "kind": "port",
                        "sample": f"{done} RK3 steps of config {cfg} on a 12^3-cube mesh ({ncell} cells), 3D oracle "
                                  f"restatement oracle/ucfv3_port.c (the reference is 2D only), 1 thread; host has "
                                  f"{os.cpu_count()} cores"}
    if rank != 0:
        dist.destroy_process_group()
        return
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": workload_config3(cfg, world),
        "census": {"class_mix_last_step": {"linear": round(float(mix[0]), 4), "cwenoz": round(float(mix[1]), 4),
                                           "muscl": round(float(mix[2]), 4), "first": round(float(mix[3]), 4)},
                   "class_mix_per_step_LCMF": per_step, "nad_ties": int(ties)},
        "setup_s": round(setup_s, 2), "cells_local": n,
        "env_overrides": env_overrides(),
        "clocks": clk.summary(),
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(n * 40), "d2h_bytes_per_step": int(n * 40),
                "call": "ucfvb3_advance_host_batch: the steps are independent host states (pinned), uploads and "
                        "downloads on copy streams overlap the stepping",
                "serial_value": e2e_serial,
                "serial_call": "ucfvb3_advance_host: each step's input is the previous step's downloaded result"},
        "gpu_launches": int(launches),
        "roofline": {"bound": bound, "kernel": names[dom], "achieved": achieved, "peak": peak, "peak_kind": peak_kind,
                     "unit": unit, "frac": achieved / peak, "traffic": None,
                     "bytes_per_cell": {k: int(v) for k, v in kb.items()},
                     "stage_achieved": stage_achieved, "stage_frac": stage_achieved / peak,
                     "phase_us": [round(1e6 * p, 2) for p in phases]},
        "cpu_baseline": cpu_baseline,
    }
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="3", choices=sorted(CONFIGS) + sorted(CONFIGS3))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"],
                    help="N>1: strong (the config's mesh split N ways, default) or weak (config domain repeated per GPU)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.config in CONFIGS3:
        run_arm_3d(args)
    elif args.impl == "reference":
        run_reference_arm(args)
    else:
        run_b200_arm(args)


if __name__ == "__main__":
    main()
