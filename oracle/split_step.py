"""numpy/scipy restatement of the reference split-step path (TEST ORACLE ONLY).

Every function cites the reference file:line it restates; paths are relative
to /root/reference/pkg/src/ctapsim/.  The arithmetic is written operation for
operation like the reference so that results are bit-identical to it (pinned
by tests/test_oracle_golden.py against fixtures produced by the reference).
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np
import scipy.constants as _sc
import scipy.fft as sfft

# constants.py:3-14 -- CODATA values from scipy at run time, masses as literals
HBAR = _sc.hbar
MU0 = _sc.mu_0
MUB = _sc.physical_constants["Bohr magneton"][0]
MASSES = {"li6": 9.9883e-27, "na23": 3.8175e-26, "rb87": 1.44316e-25}
MU0_4PI = MU0 / (4.0 * np.pi)  # magfield.py:31


def unit_time(mass: float) -> float:
    """UnitSystem.time (qgrid.py:37-39) with length 1e-6 m."""
    return mass * 1e-6 ** 2 / HBAR


def unit_energy(mass: float) -> float:
    """UnitSystem.energy (qgrid.py:41-43)."""
    return HBAR ** 2 / (mass * 1e-6 ** 2)


@dataclass(frozen=True)
class Grid:
    """SimGrid (qgrid.py:66-120): n, extents (m), origin (m)."""

    n: tuple
    extents: tuple
    origin: tuple

    @property
    def spacing(self):
        return tuple(L / n for L, n in zip(self.extents, self.n))  # qgrid.py:72-74

    @property
    def dvol(self):
        dx, dy, dz = self.spacing  # qgrid.py:77-79
        return dx * dy * dz

    def axis(self, i):
        return self.origin[i] + np.arange(self.n[i]) * self.spacing[i]  # qgrid.py:81-82

    def k_axis(self, i):
        return 2.0 * np.pi * np.fft.fftfreq(self.n[i], d=self.spacing[i])  # qgrid.py:96-98

    def k_squared(self):
        kx, ky, kz = (self.k_axis(i) for i in range(3))  # qgrid.py:112-115
        return kx[:, None, None] ** 2 + ky[None, :, None] ** 2 + kz[None, None, :] ** 2

    def meshgrid(self):
        return np.meshgrid(self.axis(0), self.axis(1), self.axis(2), indexing="ij")


def as_grid(g) -> Grid:
    return Grid(tuple(int(v) for v in g.n), tuple(float(v) for v in g.extents),
                tuple(float(v) for v in g.origin))


@dataclass
class Factors:
    """StepPlan phase fields (propagator.py:37-52)."""

    exp_v_half: np.ndarray
    exp_v_full: np.ndarray
    exp_k: np.ndarray
    dt: float
    imaginary: bool


def make_factors(grid: Grid, potential: np.ndarray, mass: float, dt: float,
                 imaginary: bool = False) -> Factors:
    """make_plan (propagator.py:55-81)."""
    dt_i = dt / unit_time(mass)
    k2_i = grid.k_squared() * 1e-6 ** 2
    if not imaginary:
        v_i = potential / unit_energy(mass)
        evh = np.exp(-0.5j * v_i * dt_i)
        evf = np.exp(-1.0j * v_i * dt_i)
        ek = np.exp(-0.5j * k2_i * dt_i)
    else:
        v_i = (potential - potential.min()) / unit_energy(mass)
        evh = np.exp(-0.5 * v_i * dt_i)
        evf = np.exp(-1.0 * v_i * dt_i)
        ek = np.exp(-0.5 * k2_i * dt_i)
    return Factors(evh, evf, ek, dt, imaginary)


_PARALLEL_MIN_SIZE = 1 << 18  # propagator.py:30


def _mul_inplace(a: np.ndarray, b: np.ndarray, pool):
    """_mul_inplace (propagator.py:84-95): a *= b, chunked over axis 0 across
    the pool (numpy releases the GIL); elementwise, so bit-identical either way."""
    if pool is None or a.size < _PARALLEL_MIN_SIZE:
        np.multiply(a, b, out=a)
        return
    nchunks = pool._max_workers
    bounds = np.linspace(0, a.shape[0], nchunks + 1).astype(int)
    futs = [pool.submit(np.multiply, a[lo:hi], b[lo:hi], a[lo:hi])
            for lo, hi in zip(bounds[:-1], bounds[1:]) if hi > lo]
    for fu in futs:
        fu.result()


def advance(amps: np.ndarray, f: Factors, n: int, workers: int | None = None) -> np.ndarray:
    """_advance (propagator.py:98-107): n merged Strang steps, with the
    thread pool evolve_real creates when threads > 1 (propagator.py:156)
    driving the pointwise multiplies and scipy.fft's workers the FFTs."""
    from concurrent.futures import ThreadPoolExecutor

    w = workers or os.cpu_count()
    pool = ThreadPoolExecutor(w) if w > 1 else None
    try:
        _mul_inplace(amps, f.exp_v_half, pool)
        for j in range(n):
            amps = sfft.fftn(amps, workers=w, overwrite_x=True)
            _mul_inplace(amps, f.exp_k, pool)
            amps = sfft.ifftn(amps, workers=w, overwrite_x=True)
            _mul_inplace(amps, f.exp_v_full if j < n - 1 else f.exp_v_half, pool)
    finally:
        if pool is not None:
            pool.shutdown()
    return amps


def event_schedule(n_steps: int, strides) -> list:
    """evolve_real's schedule (propagator.py:150-155)."""
    events = {0, n_steps}
    for s in strides:
        if s <= 0:
            raise ValueError("observer stride must be positive")
        events.update(range(0, n_steps + 1, s))
    return sorted(e for e in events if e <= n_steps)


def evolve(amps: np.ndarray, f: Factors, n_steps: int, stride: int | None = None,
           on_event=None, workers: int | None = None, t0: float = 0.0) -> np.ndarray:
    """evolve_real (propagator.py:134-173) with one observer of `stride`;
    on_event(step, t, amps) fires at step 0, every stride and at n_steps, with
    the time stamp accumulated per segment as psi.time is (:163)."""
    current = 0
    t = t0
    for ev in event_schedule(n_steps, [stride] if stride else []):
        if ev > current:
            amps = advance(amps, f, ev - current, workers)
            t += (ev - current) * f.dt
            current = ev
        if on_event is not None and stride and (ev % stride == 0 or ev == n_steps):
            on_event(ev, t, amps)
    return amps


# ------------------------------------------------------------ observables

def norm(amps, grid: Grid) -> float:
    return float(np.sum(np.abs(amps) ** 2) * grid.dvol)  # qgrid.py:150-154


def populations(amps, grid: Grid, xb1, xb2):
    """observables.populations (observables.py:74-88)."""
    dx, dy, dz = grid.spacing
    w = (np.abs(amps) ** 2).sum(axis=1) * dy
    xs = grid.axis(0)
    in_l = xs[:, None] < np.asarray(xb1)[None, :]
    in_r = xs[:, None] >= np.asarray(xb2)[None, :]
    p_l = float(np.sum(w, where=in_l) * dx * dz)
    p_r = float(np.sum(w, where=in_r) * dx * dz)
    p_m = float(np.sum(w, where=~(in_l | in_r)) * dx * dz)
    return p_l, p_m, p_r


def density_xz(amps, grid: Grid):
    return (np.abs(amps) ** 2).sum(axis=1) * grid.spacing[1]  # observables.py:91-94


def edge_density(amps, grid: Grid, margin_cells: int = 2) -> float:
    """observables.edge_density (observables.py:97-110)."""
    if margin_cells < 1:
        raise ValueError("margin_cells must be >= 1")
    rho = np.abs(amps) ** 2
    m = margin_cells
    mask = np.zeros(grid.n, dtype=bool)
    mask[:m, :, :] = True
    mask[-m:, :, :] = True
    mask[:, :m, :] = True
    mask[:, -m:, :] = True
    mask[:, :, :m] = True
    mask[:, :, -m:] = True
    return float(np.sum(rho, where=mask) * grid.dvol)


def trace_row(t, amps, grid: Grid, xb1, xb2, margin=2):
    """PopulationRecorder.notify (observables.py:173-176)."""
    pl, pm, pr = populations(amps, grid, xb1, xb2)
    return (t, pl, pm, pr, norm(amps, grid), edge_density(amps, grid, margin))


def evolve_with_trace(amps, grid: Grid, f: Factors, n_steps: int, stride: int,
                      xb1, xb2, margin=2, t0=0.0, workers=None):
    """run_evolve's evolve stage (runner.py:192-209) with a PopulationRecorder."""
    rows = []

    def on_event(ev, t, a):
        rows.append(trace_row(t, a, grid, xb1, xb2, margin))

    amps = evolve(amps, f, n_steps, stride, on_event, workers, t0)
    return amps, np.array(rows)


# --------------------------------------------------------------- energies

def kinetic_expectation(amps, grid: Grid, mass: float) -> float:
    """propagator.kinetic_expectation (propagator.py:176-185)."""
    phi = sfft.fftn(amps, workers=os.cpu_count())
    k2 = grid.k_squared()
    w = float(np.sum(np.abs(phi) ** 2))
    t = float(np.sum((HBAR ** 2 * k2 / (2 * mass)) * np.abs(phi) ** 2))
    return t / w


def potential_expectation(amps, potential) -> float:
    rho = np.abs(amps) ** 2  # propagator.py:188-190
    return float(np.sum(potential * rho) / np.sum(rho))


def energy_expectation(amps, grid: Grid, potential, mass) -> float:
    return kinetic_expectation(amps, grid, mass) + potential_expectation(amps, potential)


def normalize(amps, grid: Grid):
    amps /= np.sqrt(norm(amps, grid))  # qgrid.py:159-162
    return amps


def ground_state_imaginary(grid: Grid, potential, seed, tol=1e-10, tau=1e-7, mass=None,
                           check_every=100, max_steps=400_000):
    """propagator.ground_state_imaginary (propagator.py:198-241)."""
    mass = MASSES["li6"] if mass is None else mass
    amps = np.asarray(seed, complex).copy()
    normalize(amps, grid)
    f = make_factors(grid, potential, mass, tau, imaginary=True)
    e_prev = energy_expectation(amps, grid, potential, mass)
    done = 0
    while done < max_steps:
        n = min(check_every, max_steps - done)
        amps = advance(amps, f, n)
        normalize(amps, grid)
        done += n
        e_now = energy_expectation(amps, grid, potential, mass)
        if abs(e_now - e_prev) < tol * max(abs(e_now), 1e-300):
            return amps, done
        e_prev = e_now
    raise RuntimeError("imaginary-time relaxation did not converge")


# ----------------------------------------------------------- initial data

def gaussian_packet(grid: Grid, center, widths, momentum=(0.0, 0.0, 0.0)):
    """qgrid.gaussian_packet (qgrid.py:171-196) -> normalized amplitudes."""
    center = np.asarray(center, float)
    widths = np.asarray(widths, float)
    momentum = np.asarray(momentum, float)
    x, y, z = grid.axis(0), grid.axis(1), grid.axis(2)
    fx = np.exp(-((x - center[0]) ** 2) / (2 * widths[0] ** 2) + 1j * momentum[0] * x)
    fy = np.exp(-((y - center[1]) ** 2) / (2 * widths[1] ** 2) + 1j * momentum[1] * y)
    fz = np.exp(-((z - center[2]) ** 2) / (2 * widths[2] ** 2) + 1j * momentum[2] * z)
    amp = (fx[:, None, None] * fy[None, :, None] * fz[None, None, :]).astype(np.complex128)
    return normalize(amp, grid)


def harmonic_potential(grid: Grid, mass, omegas, center):
    """ho_potential of the reference tests (tests/test_propagator.py:13-18)."""
    x, y, z = grid.meshgrid()
    wx, wy, wz = omegas
    return 0.5 * mass * (wx ** 2 * (x - center[0]) ** 2
                         + wy ** 2 * (y - center[1]) ** 2
                         + wz ** 2 * (z - center[2]) ** 2)


def bench_potential(grid: Grid, mass, f_z=5.0):
    """run_bench's synthetic potential (runner.py:284-288): 1/2 m w_z^2 |r-c|^2."""
    omega = 2 * np.pi * f_z
    c = [grid.origin[i] + grid.extents[i] / 2 for i in range(3)]
    x, y, z = grid.meshgrid()
    return 0.5 * mass * omega ** 2 * ((x - c[0]) ** 2 + (y - c[1]) ** 2 + (z - c[2]) ** 2)
