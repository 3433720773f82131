"""The evolve pipeline around the propagator, on the B200:
transverse ground state of the occupied guide by imaginary time, the initial
state, one CTAP run, and the current sweep as independent replicas over the
GPUs of a job.

Drop-in for the compute part of ctapsim.runner (runner.py:125-251): the
potential, its minima and partition, the imaginary-time relaxation, the
real-time evolution and every observable run on the device through libctap.
Configuration objects and chip geometry stay the reference's (an
ExperimentConfig with .to_layout(i_middle) / .to_grid(), or any object with
the same attributes); manifests, CSV export and the CLI are out of scope.
"""

from __future__ import annotations

import copy
import dataclasses
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _device
from .constants import hbar
from .magfield import MinimumAbsentError, assemble_potential
from .observables import EdgeMonitor, PopulationRecorder, build_partition, transfer_fidelity
from .propagator import REAL_TIME, evolve_real, ground_state_imaginary, make_plan
from .qgrid import Wavefunction, make_grid

MASK_POTENTIAL = 1e-18  # J, the wall of the windowed relaxation (runner.py:37)


@dataclass(frozen=True)
class TransverseSpectrum:
    """magfield.TransverseSpectrum (magfield.py:252-258)."""

    omega_x: float
    omega_y: float
    v_min: float
    energies: tuple


def transverse_spectrum(potential, z_index: int, guide_index: int) -> TransverseSpectrum:
    """Harmonic estimate of one guide's two lowest transverse energies from
    3-point curvatures at the node nearest the refined minimum
    (magfield.py:262-286).  Reads five values of V from the device."""
    x0, y0, vmin = potential.guide_minimum(z_index, guide_index)
    grid = potential.grid
    xs, ys = np.asarray(grid.x), np.asarray(grid.y)
    i = int(np.clip(np.argmin(np.abs(xs - x0)), 1, grid.n[0] - 2))
    j = int(np.clip(np.argmin(np.abs(ys - y0)), 1, grid.n[1] - 2))
    vals = potential.values
    if isinstance(vals, torch.Tensor):
        idx = torch.tensor([[i, j], [i + 1, j], [i - 1, j], [i, j + 1], [i, j - 1]], device=vals.device)
        st = _device.to_host(vals[idx[:, 0], idx[:, 1], z_index])
    else:
        st = np.array([vals[i, j, z_index], vals[i + 1, j, z_index], vals[i - 1, j, z_index],
                       vals[i, j + 1, z_index], vals[i, j - 1, z_index]])
    v0, vxp, vxm, vyp, vym = st
    dx, dy, _ = grid.spacing
    vxx = (vxp - 2 * v0 + vxm) / dx ** 2
    vyy = (vyp - 2 * v0 + vym) / dy ** 2
    if vxx <= 0 or vyy <= 0:
        raise MinimumAbsentError(f"non-positive curvature at slice {z_index}, guide {guide_index}")
    m = potential.layout.mass
    wx, wy = np.sqrt(vxx / m), np.sqrt(vyy / m)
    e0 = hbar * (wx / 2 + wy / 2)
    e1 = hbar * (1.5 * min(wx, wy) + 0.5 * max(wx, wy))
    return TransverseSpectrum(float(wx), float(wy), float(vmin), (float(e0), float(e1)))


def transverse_ground_state(potential, partition, z_index: int, guide_index: int = 0,
                            tau: float = 1e-7, tol: float = 1e-10, threads: int = 1) -> np.ndarray:
    """2D transverse ground state of one guide at slice z_index
    (runner.py:125-165): the slice potential walled off outside the guide's x
    window, replicated on a thin 8-slice grid and relaxed in imaginary time
    on the device.  Returns phi(x, y) normalised to int |phi|^2 dx dy = 1."""
    grid = potential.grid
    xs = np.asarray(grid.x)
    vals = _device.to_device_f64(potential.values)
    v_slice = vals[:, :, z_index].clone()
    if guide_index == 0:
        window = xs < partition.xb1[z_index]
    elif guide_index == 1:
        window = (xs >= partition.xb1[z_index]) & (xs < partition.xb2[z_index])
    else:
        window = xs >= partition.xb2[z_index]
    v_slice[torch.from_numpy(~window).to(v_slice.device), :] = MASK_POTENTIAL
    x0, y0, _ = potential.guide_minimum(z_index, guide_index)
    spec = transverse_spectrum(potential, z_index, guide_index)
    mass = potential.layout.mass
    sx = np.sqrt(hbar / (mass * spec.omega_x))
    sy = np.sqrt(hbar / (mass * spec.omega_y))
    nz_thin = 8
    thin = make_grid(grid.n[0], grid.n[1], nz_thin,
                     (grid.extents[0], grid.extents[1], nz_thin * grid.spacing[2]),
                     origin=(grid.origin[0], grid.origin[1], 0.0))
    seed2d = np.exp(-((xs[:, None] - x0) ** 2) / (2 * sx ** 2)
                    - ((np.asarray(grid.y)[None, :] - y0) ** 2) / (2 * sy ** 2))
    seed = np.repeat(seed2d[:, :, None], nz_thin, axis=2).astype(complex)
    v_thin = v_slice[:, :, None].expand(-1, -1, nz_thin).contiguous()
    gs = ground_state_imaginary(thin, v_thin, seed, tol=tol, tau=tau, mass=mass, threads=threads)
    phi = gs.amplitudes[:, :, 0]
    dx, dy, _ = grid.spacing
    return phi / np.sqrt(np.sum(np.abs(phi) ** 2) * dx * dy)


def initial_state(cfg, potential, partition, threads: int = 1) -> Wavefunction:
    """Transverse ground state of the left guide times a Gaussian along z
    (runner.py:168-181), normalised on the device."""
    grid = potential.grid
    z0 = cfg.z_start_eff
    zs = np.asarray(grid.z)
    iz0 = int(np.argmin(np.abs(zs - z0)))
    phi = transverse_ground_state(potential, partition, iz0, guide_index=0,
                                  tau=cfg.gs_tau, tol=cfg.gs_tol, threads=threads)
    envelope = np.exp(-((zs - z0) ** 2) / (2 * cfg.sigma_z_eff ** 2))
    amps = phi[:, :, None] * envelope[None, None, :]
    return Wavefunction(amps.astype(np.complex128), grid, time=0.0).normalize()


def prepare_potential(cfg, i_middle: float | None = None, layout=None):
    """Layout, grid, device potential (with minima) and partition
    (runner.py:114-122).  `layout` overrides cfg.to_layout(i_middle)."""
    layout = cfg.to_layout(i_middle=i_middle) if layout is None else layout
    grid = cfg.to_grid()
    potential = assemble_potential(layout, grid)
    partition = build_partition(potential)
    return layout, grid, potential, partition


def evolve_point(cfg, i_middle: float | None = None, layout=None, observers=()) -> dict:
    """One CTAP run (the compute of run_evolve, runner.py:184-229): potential,
    partition, initial state, real-time evolution with the population
    recorder and edge monitor.  Returns run_evolve's `results` plus the
    trace and the device wavefunction."""
    layout, grid, potential, partition = prepare_potential(cfg, i_middle, layout)
    psi = initial_state(cfg, potential, partition)
    plan = make_plan(grid, potential.values, cfg.mass, cfg.dt, mode=REAL_TIME)
    recorder = PopulationRecorder(partition, stride=cfg.trace_stride, margin_cells=cfg.edge_margin_cells)
    monitor = EdgeMonitor(stride=cfg.edge_stride, margin_cells=cfg.edge_margin_cells,
                          threshold=cfg.edge_threshold)
    psi, stats = evolve_real(psi, plan, cfg.n_steps, [recorder, monitor, *observers])
    tr = recorder.trace
    return {
        "i_middle_effective": cfg.i_middle if i_middle is None else i_middle,
        "final_p_l": tr.p_l[-1], "final_p_m": tr.p_m[-1], "final_p_r": transfer_fidelity(tr),
        "max_p_m": tr.max_middle(), "final_norm": tr.norm[-1], "max_edge": max(tr.edge),
        "steps_per_second": stats.steps_per_second, "trace": tr, "psi": psi,
    }


ORDERINGS = ("counter_intuitive", "intuitive")


def sweep_points(values) -> list:
    """(ordering, i_m) in run_sweep's order (runner.py:238-242)."""
    return [(o, float(v)) for o in ORDERINGS for v in values]


def rank_share(n_points: int, rank: int, world: int) -> list:
    """Indices of the sweep points replica `rank` of `world` runs
    (round-robin: the runs are equally long)."""
    return list(range(rank, n_points, world))


def run_sweep(cfg, out_dir=None, group=None, run_point=None) -> list:
    """run_sweep (runner.py:232-251) as independent replicas: with
    torch.distributed initialised, rank r of W runs points r, r + W, ... on
    its own GPU, the rows are gathered in the reference's order and rank 0
    writes sweep.csv.  `run_point(cfg_point, i_m) -> final_p_r` defaults to
    evolve_point.  Returns the rows (i_m, ordering, final_p_r)."""
    import torch.distributed as dist

    points = sweep_points(cfg.sweep_values())
    dist_on = dist.is_available() and dist.is_initialized()
    rank = dist.get_rank(group) if dist_on else 0
    world = dist.get_world_size(group) if dist_on else 1
    if run_point is None:
        def run_point(c, i_m):
            return evolve_point(c, i_middle=i_m)["final_p_r"]
    mine = {}
    for k in rank_share(len(points), rank, world):
        ordering, i_m = points[k]
        if dataclasses.is_dataclass(cfg):
            cfg_point = dataclasses.replace(cfg, ordering=ordering)
        else:  # any object with the same attributes: a copy with this point's ordering
            cfg_point = copy.copy(cfg)
            setattr(cfg_point, "ordering", ordering)
        mine[k] = float(run_point(cfg_point, i_m))
    if dist_on:
        parts = [None] * world
        dist.all_gather_object(parts, mine, group=group)
        merged = {}
        for p in parts:
            merged.update(p)
    else:
        merged = mine
    rows = [(points[k][1], points[k][0], merged[k]) for k in range(len(points))]
    if out_dir is not None and rank == 0:
        os.makedirs(out_dir, exist_ok=True)
        with open(os.path.join(out_dir, "sweep.csv"), "w") as fh:
            fh.write("i_m,ordering,final_p_r\n")
            for i_m, ordering, pr in rows:
                fh.write(f"{i_m:.17g},{ordering},{pr:.17g}\n")
    return rows


# ---------------------------------------------------------------------------
# the measurement harness (runner.py:260-325)
# ---------------------------------------------------------------------------

def bench_thread_counts(max_threads: int | None = None) -> list:
    """Powers of two up to the host thread count, plus the count itself
    (runner.py:260-268).  The device path ignores the count (make_plan's
    `threads` is accepted for signature compatibility), so every row of a
    run_bench report times the same B200 kernels."""
    hw = max_threads or (os.cpu_count() or 1)
    counts, c = [], 1
    while c < hw:
        counts.append(c)
        c *= 2
    counts.append(hw)
    return sorted(set(counts))


def run_bench(cfg, out_dir, thread_counts=None, warm_steps: int | None = None,
              timed_steps: int | None = None, chunks: int = 10) -> dict:
    """Split-step steps/sec on the configured grid (runner.py:271-325) on the
    device: the reference's synthetic harmonic trap and Gaussian packet, warm
    steps discarded, the timed steps in `chunks` evolve_real calls, median
    chunk rate (spread min..max), written to bench.csv / bench.txt in the
    reference's format.  One row per entry of `thread_counts` (default
    [1]: the device does not depend on the host thread count)."""
    from .qgrid import gaussian_packet

    os.makedirs(out_dir, exist_ok=True)
    warm = cfg.bench_warm_steps if warm_steps is None else warm_steps
    timed = cfg.bench_timed_steps if timed_steps is None else timed_steps
    grid = cfg.to_grid()
    x, y, z = grid.meshgrid()
    center = [o + e / 2 for o, e in zip(grid.origin, grid.extents)]
    v = 0.5 * cfg.mass * cfg.omega_z ** 2 * ((x - center[0]) ** 2 + (y - center[1]) ** 2
                                             + (z - center[2]) ** 2)
    psi0 = gaussian_packet(grid, center, [e / 16 for e in grid.extents])
    report = {"grid": grid.n, "warm_steps": warm, "timed_steps": timed, "rates": {}}
    for nt in (thread_counts or [1]):
        plan = make_plan(grid, v, cfg.mass, cfg.dt, mode=REAL_TIME, threads=nt)
        psi = psi0.copy()
        evolve_real(psi, plan, warm)
        per_chunk = max(1, timed // chunks)
        rates = []
        for _ in range(chunks):
            psi, stats = evolve_real(psi, plan, per_chunk)
            rates.append(stats.steps_per_second)
        rates = np.array(rates)
        report["rates"][nt] = {"median": float(np.median(rates)), "min": float(rates.min()),
                               "max": float(rates.max())}
    csv_path = os.path.join(out_dir, "bench.csv")
    with open(csv_path, "w") as fh:
        fh.write("threads,steps_per_sec\n")
        for nt, r in report["rates"].items():
            fh.write(f"{nt},{r['median']:.17g}\n")
    ref_steps = 100_000  # reference-chip full run at dt = 1 us
    txt_path = os.path.join(out_dir, "bench.txt")
    with open(txt_path, "w") as fh:
        fh.write(f"split-operator kernel benchmark, grid {grid.n} (B200, libctap)\n")
        fh.write(f"warm {warm} steps discarded, {timed} timed steps in {chunks} chunks\n")
        for nt, r in report["rates"].items():
            fh.write(f"threads={nt}: median {r['median']:.3f} steps/s "
                     f"(spread {r['min']:.3f}..{r['max']:.3f}); projected "
                     f"{ref_steps}-step run: {ref_steps / r['median'] / 3600:.4f} h\n")
    report["csv"] = csv_path
    report["txt"] = txt_path
    return report
