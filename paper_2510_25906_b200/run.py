"""run_simulation's outer loop and outputs over the device solver
(/root/reference/proj/src/run.cpp:60-213).

    res = run_simulation(solver, mesh, t_end, out_dir="out", output_every=50)

Steps `dt = min(max_stable_dt, t_end - t); advance` while t < t_end - 1e-14
t_end entirely on the device (ucfvb_run_until; the loop condition, dt and t
never leave the GPU between snapshots), records a CensusRow per step (first-
stage label counts, run.cpp:109-116), and writes the reference's files:
fields_<step>.vtk every `output_every` steps and at the end, census.csv and
timing.csv (run.cpp:128-150). The writers are the native ones in
libucfvb.so, byte-identical to the reference's.

Timing rows (run.cpp:118-127) carry per-step PhaseTimes deltas only when
`phase_timing=True`; that mode runs one un-graphed step per call with
per-phase CUDA events (slower), otherwise timing.csv is not written.
"""
from __future__ import annotations

import ctypes as C
import os
import time
from dataclasses import dataclass, field

import numpy as np

from . import _abi as A


@dataclass
class RunResult:
    """RunResult (run.hpp:27-38) minus mesh/errors."""
    state: np.ndarray
    final_labels: np.ndarray
    census: list = field(default_factory=list)   # [(step, t, dt, counts[4])]
    timing: list = field(default_factory=list)   # [(step, wall, reconstruct, detect, weights, flux)]
    wall_seconds: float = 0.0
    steps: int = 0
    t: float = 0.0
    t_end: float = 0.0


def _ck(lib, rc):
    if rc != A.OK:
        raise A.error_for(rc, lib.ucfvb_last_error(None).decode())


def write_field_snapshot(mesh, state, labels, gamma, path):
    """write_field_snapshot (run.cpp:160-190)."""
    lib = A.load_library()
    u = np.ascontiguousarray(state, dtype=np.float64)
    lab = np.ascontiguousarray(labels, dtype=np.uint8)
    _ck(lib, lib.ucfvb_write_field_snapshot(C.byref(mesh.view), u.ctypes.data_as(A.c_dp),
                                            lab.ctypes.data_as(C.POINTER(C.c_uint8)), float(gamma),
                                            os.fsencode(path)))


def write_census_csv(rows, n_cells, path):
    """write_census_csv (run.cpp:192-202); rows = [(step, t, dt, counts[4])]."""
    lib = A.load_library()
    arr = (A.CensusRow * max(1, len(rows)))()
    for i, (step, t, dt, counts) in enumerate(rows):
        arr[i].step, arr[i].t, arr[i].dt = int(step), float(t), float(dt)
        for k in range(4):
            arr[i].counts[k] = int(counts[k])
    _ck(lib, lib.ucfvb_write_census_csv(arr, len(rows), int(n_cells), os.fsencode(path)))


def write_timing_csv(rows, path):
    """write_timing_csv (run.cpp:204-213); rows = [(step, wall, reconstruct, detect, weights, flux)]."""
    lib = A.load_library()
    arr = (A.TimingRow * max(1, len(rows)))()
    for i, r in enumerate(rows):
        arr[i].step = int(r[0])
        arr[i].wall, arr[i].reconstruct, arr[i].detect, arr[i].weights, arr[i].flux = map(float, r[1:6])
    _ck(lib, lib.ucfvb_write_timing_csv(arr, len(rows), os.fsencode(path)))


def run_simulation(solver, mesh, t_end: float, rk: int = A.RK3, t0: float = 0.0, out_dir: str | None = None,
                   output_every: int = 0, phase_timing: bool = False, max_steps: int = 1 << 20) -> RunResult:
    """The stepping loop of run_simulation (run.cpp:92-150) from the solver's current state."""
    writing = bool(out_dir)
    if writing:
        os.makedirs(out_dir, exist_ok=True)
    gamma = solver.options.gamma
    wall0 = time.perf_counter()
    t, step = float(t0), 0
    census, timing = [], []
    if phase_timing:
        solver.set_phase_timing(True)
        prev = solver.phase_times().copy()
    try:
        while step < max_steps:
            if phase_timing:
                chunk = 1
            elif output_every > 0:
                chunk = output_every - step % output_every
            else:
                chunk = max_steps - step
            chunk = min(chunk, max_steps - step)
            t_new, n, cen, dts = solver.run_until(t_end, rk, t, max_steps=chunk)
            for k in range(n):
                t = t + dts[k]  # run.cpp:107, the device accumulated the same sum
                step += 1
                census.append((step, t, dts[k], cen[k].tolist()))
            if n and t != t_new:
                raise RuntimeError(f"run_simulation: host t {t!r} != device t {t_new!r}")
            if phase_timing and n:
                now = solver.phase_times().copy()
                d = now - prev
                prev = now
                timing.append((step, time.perf_counter() - wall0, d[0], d[1], d[2], d[3]))
            if writing and output_every > 0 and n and step % output_every == 0:
                write_field_snapshot(mesh, solver.state, solver.step_labels(), gamma,
                                     os.path.join(out_dir, f"fields_{step}.vtk"))
            if n < chunk:
                break  # the loop condition ended the run
    finally:
        if phase_timing:
            solver.set_phase_timing(False)
    res = RunResult(state=solver.state, final_labels=solver.step_labels(), census=census, timing=timing,
                    wall_seconds=time.perf_counter() - wall0, steps=step, t=t, t_end=t_end)
    if writing:
        write_field_snapshot(mesh, res.state, res.final_labels, gamma, os.path.join(out_dir, f"fields_{step}.vtk"))
        write_census_csv(census, solver.n_cells, os.path.join(out_dir, "census.csv"))
        if phase_timing:
            write_timing_csv(timing, os.path.join(out_dir, "timing.csv"))
    return res
