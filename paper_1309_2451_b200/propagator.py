"""Split-step propagation on the B200: drop-in for ctapsim.propagator.

Same public surface as the reference (propagator.py:1-294): REAL_TIME /
IMAGINARY_TIME, StepPlan, make_plan, step, evolve_real (+ EvolveStats and the
observer protocol), kinetic/potential/energy_expectation,
ground_state_imaginary (+ ConvergenceError), SnapshotObserver,
ProgressObserver, imaginary_step_count_estimate.  Same argument meaning,
return values, exception types and messages.

What changes is where the work happens: the plan holds no phase fields (the
kernels recompute exp(-i V dt/2), exp(-i V dt), exp(-i k^2 dt/2) per point
with the reference's exact operation order), the wavefunction stays in HBM,
and every telescoped segment is one ctap_advance call (libctap.so) that runs
four fused axis passes per step.
"""

from __future__ import annotations

import ctypes
from collections import OrderedDict
import os
import sys
import time as _time
import weakref
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device, _lib
from .qgrid import UnitSystem, Wavefunction, as_simgrid, grid_key, same_grid, write_snapshot

REAL_TIME = "real_time"
IMAGINARY_TIME = "imaginary_time"

# wavefunction precision of a plan: complex128 (the reference's) or the
# optional complex64 mode (phases still exact in FP64; gate <= 1e-4)
PRECISIONS = {"complex128": torch.complex128, "complex64": torch.complex64}

# phase-table mask of make_plan (bit 0: exp(-iV dt) table, bit 1: exp(-ik^2 dt/2)
# table); the environment variable is for A/B
# measurements
PHASE_TABLE_V = 1
PHASE_TABLE_K = 2
DEFAULT_PHASE_TABLES = int(os.environ.get("CTAP_PHASE_TABLES", "0"))


class ConvergenceError(RuntimeError):
    """Imaginary-time relaxation failed to reach the tolerance."""


# ---------------------------------------------------------------------------
# native plan
# ---------------------------------------------------------------------------

class NativePlan:
    """Owns one ctap_plan (include/ctap.h) and the device buffers it points at."""

    def __init__(self, grid, v_dev: torch.Tensor | None, mass: float, dt: float,
                 mode: str = REAL_TIME, v_shift: float = 0.0, slab_p: int = 1, slab_r: int = 0,
                 phase_tables: int = 0, precision: str = "complex128", pencil_c: int = 0):
        lib = _lib.load()
        dev = _device.require_cuda()
        self.grid = as_simgrid(grid)
        units = UnitSystem(length=1e-6, mass=mass)
        desc = _lib.CtapPlanDesc()
        for i in range(3):
            desc.n[i] = int(self.grid.n[i])
        desc.e0 = units.energy
        desc.dt_i = dt / units.time
        desc.len2 = units.length ** 2
        desc.v_shift = float(v_shift)
        desc.mode = _lib.REAL_TIME_MODE if mode == REAL_TIME else _lib.IMAGINARY_TIME_MODE
        desc.slab_p = int(slab_p)
        desc.slab_r = int(slab_r)
        desc.phase_tables = int(phase_tables)
        desc.pencil_c = int(pencil_c)
        if precision not in PRECISIONS:
            raise ValueError(f"unknown precision {precision!r}; known: {sorted(PRECISIONS)}")
        desc.dtype = _lib.DTYPE_C64 if precision == "complex64" else _lib.DTYPE_C128
        self.precision = precision
        self.torch_dtype = PRECISIONS[precision]
        self.desc = desc
        # squared wavenumbers exactly as k_squared() forms them (qgrid.py:112-115)
        self._k2 = [np.ascontiguousarray(self.grid.k_axis(i) ** 2) for i in range(3)]
        self._v = v_dev  # None: FFT/reduction-only plan
        handle = ctypes.c_void_p()
        _lib.check(lib.ctap_plan_create(ctypes.byref(desc), self._k2[0].ctypes.data,
                                        self._k2[1].ctypes.data, self._k2[2].ctypes.data,
                                        None if v_dev is None else v_dev.data_ptr(),
                                        ctypes.byref(handle)))
        self.handle = handle
        self._fin = weakref.finalize(self, lib.ctap_plan_destroy, handle)
        self._out = torch.zeros(8, dtype=torch.float64, device=dev)

    def advance(self, psi: torch.Tensor, n: int):
        _lib.call("ctap_advance", self.handle, psi.data_ptr(), int(n), _device.stream_handle())

    def step_schedule(self) -> tuple[int, int]:
        """(slab planes, streams) of ctap_advance's step schedule; (0, 1) is
        plane order (ctap_step_schedule)."""
        planes, streams = ctypes.c_int64(), ctypes.c_int32()
        _lib.call("ctap_step_schedule", self.handle, ctypes.byref(planes), ctypes.byref(streams))
        return planes.value, streams.value

    def launches(self, n: int) -> int:
        """Kernel launches of ctap_advance(n) under its step schedule."""
        if n <= 0:
            return 0
        planes, _ = self.step_schedule()
        if planes == 0:
            return 4 * n + 1
        s = self.grid.n[0] // planes
        return 2 * s + (n - 1) * (1 + 3 * s) + 1 + 2 * s

    def advance_observe(self, psi: torch.Tensor, n: int, xs: torch.Tensor, xb1, xb2, margin: int) -> torch.Tensor:
        """n steps, then the observer sums fused into the segment-end pass
        (ctap_advance_observe): [sum rho, left, middle, right, edge]."""
        out = torch.empty(5, dtype=torch.float64, device=psi.device)
        _lib.call("ctap_advance_observe", self.handle, psi.data_ptr(), int(n), xs.data_ptr(),
                  None if xb1 is None else xb1.data_ptr(), None if xb2 is None else xb2.data_ptr(),
                  int(margin), out.data_ptr(), _device.stream_handle())
        return out

    def run_pass(self, kind: int, src: torch.Tensor, dst: torch.Tensor):
        _lib.call("ctap_pass", self.handle, int(kind), src.data_ptr(), dst.data_ptr(),
                  _device.stream_handle())

    def run_pass_zchunk(self, kind: int, src: torch.Tensor, dst: torch.Tensor, z0: int, zn: int):
        """A slab pass on z columns [z0, z0 + zn) with chunk-major transpose
        buffers (ctap_pass_zchunk)."""
        _lib.call("ctap_pass_zchunk", self.handle, int(kind), src.data_ptr(), dst.data_ptr(), int(z0), int(zn),
                  _device.stream_handle())

    def run_pass_ptr(self, kind: int, src: int, dst: int):
        """A pass on raw device addresses (plan-external buffers)."""
        _lib.call("ctap_pass", self.handle, int(kind), src, dst, _device.stream_handle())

    def set_peer_buffers(self, which: int, ptrs):
        arr = (ctypes.c_void_p * len(ptrs))(*ptrs)
        _lib.call("ctap_set_peer_buffers", self.handle, int(which), arr, len(ptrs))

    def clear_peer_buffers(self):
        """Unregister both peer tables (count 0): the fused passes then fail
        with EINVAL instead of storing through stale mappings."""
        for which in (0, 1):
            _lib.call("ctap_set_peer_buffers", self.handle, which, None, 0)

    def fft3d(self, data: torch.Tensor, direction: int = -1):
        _lib.call("ctap_fft3d", self.handle, data.data_ptr(), int(direction), _device.stream_handle())

    def scale(self, psi: torch.Tensor, divisor: float):
        _lib.call("ctap_scale", self.handle, psi.data_ptr(), float(divisor), _device.stream_handle())

    def observe(self, psi: torch.Tensor, xs: torch.Tensor, xb1, xb2, margin: int) -> torch.Tensor:
        out = torch.empty(5, dtype=torch.float64, device=psi.device)
        _lib.call("ctap_observe", self.handle, psi.data_ptr(), xs.data_ptr(),
                  None if xb1 is None else xb1.data_ptr(), None if xb2 is None else xb2.data_ptr(),
                  int(margin), out.data_ptr(), _device.stream_handle())
        return out

    def k2_sums(self, phi: torch.Tensor) -> torch.Tensor:
        out = torch.empty(2, dtype=torch.float64, device=phi.device)
        _lib.call("ctap_k2_sums", self.handle, phi.data_ptr(), out.data_ptr(), _device.stream_handle())
        return out

    def v_sums(self, psi: torch.Tensor) -> torch.Tensor:
        out = torch.empty(2, dtype=torch.float64, device=psi.device)
        _lib.call("ctap_v_sums", self.handle, psi.data_ptr(), out.data_ptr(), _device.stream_handle())
        return out

    def density_xz(self, psi: torch.Tensor) -> torch.Tensor:
        nxl = self.grid.n[0] // self.desc.slab_p
        out = torch.empty((nxl, self.grid.n[2]), dtype=torch.float64, device=psi.device)
        _lib.call("ctap_density_xz", self.handle, psi.data_ptr(), out.data_ptr(), _device.stream_handle())
        return out

    def phase_field(self, which: int) -> torch.Tensor:
        nxl = self.grid.n[0] // self.desc.slab_p
        out = torch.empty((nxl, self.grid.n[1], self.grid.n[2]), dtype=torch.complex128,
                          device=self._out.device)  # inspection is always complex128
        _lib.call("ctap_phase_field", self.handle, int(which), out.data_ptr(), _device.stream_handle())
        return out


_AUX = OrderedDict()
_AUX_MAX = 8  # potential-free plans kept (least recently used evicted)


def _aux_plan(grid, dtype=torch.complex128) -> NativePlan:
    """A potential-free plan for FFTs and reductions on `grid` (LRU-cached)."""
    key = (grid_key(grid), torch.cuda.current_device() if torch.cuda.is_available() else -1, dtype)
    p = _AUX.get(key)
    if p is None:
        from .constants import species_mass

        prec = "complex64" if dtype == torch.complex64 else "complex128"
        p = NativePlan(grid, None, species_mass("li6"), 1e-6, precision=prec)
        _AUX[key] = p
        while len(_AUX) > _AUX_MAX:
            _AUX.popitem(last=False)
    else:
        _AUX.move_to_end(key)
    return p


# ---------------------------------------------------------------------------
# plan
# ---------------------------------------------------------------------------

@dataclass
class StepPlan:
    """Plan for one (grid, potential, dt) triple (propagator.py:37-52).

    `exp_v_half`, `exp_v_full`, `exp_k` are materialised lazily (on the device,
    then copied to the host) only if someone inspects them."""

    grid: object
    dt: float
    mode: str
    mass: float
    potential: object
    threads: int = 1
    native: NativePlan = field(default=None, repr=False)
    _fields: dict = field(default_factory=dict, repr=False)

    def matches(self, psi) -> bool:
        return same_grid(psi.grid, self.grid)

    def _field(self, which: int) -> np.ndarray:
        if which not in self._fields:
            self._fields[which] = _device.to_host(self.native.phase_field(which))
        return self._fields[which]

    @property
    def exp_v_half(self) -> np.ndarray:
        return self._field(0)

    @property
    def exp_v_full(self) -> np.ndarray:
        return self._field(1)

    @property
    def exp_k(self) -> np.ndarray:
        return self._field(2)


def make_plan(grid, potential, mass: float, dt: float, mode: str = REAL_TIME,
              threads: int = 1, *, phase_tables: int | None = None,
              precision: str = "complex128") -> StepPlan:
    """make_plan (propagator.py:55-81).

    `threads` is accepted for signature compatibility (the device decides its
    own parallelism).  `phase_tables` (B200 extension) is a mask choosing
    which of exp(-i V dt) (PHASE_TABLE_V) and exp(-i k^2 dt/2)
    (PHASE_TABLE_K) are kept as HBM tables instead of being recomputed per
    point every step; the phases are bit-identical either way.  None picks
    the measured-fastest default.  `precision="complex64"` selects the
    optional complex64 mode (complex64 storage and transforms, exact FP64
    phases; held to <= 1e-4 against the complex128 oracle)."""
    if mode not in (REAL_TIME, IMAGINARY_TIME):
        raise ValueError(f"unknown mode {mode!r}")
    if tuple(potential.shape) != tuple(grid.n):
        raise ValueError("potential shape does not match the grid")
    v_dev = _device.to_device_f64(potential)
    if mode == REAL_TIME:
        # the reference asserts |exp(-i V dt/2)| == 1 to 1e-14, which fails
        # exactly when V (hence the phase) is not finite
        if not bool(torch.isfinite(v_dev).all()):
            raise AssertionError("real-time potential factor is not unit modulus")
        shift = 0.0
    else:
        shift = float(v_dev.min().item())
    if phase_tables is None:
        phase_tables = DEFAULT_PHASE_TABLES
    native = NativePlan(grid, v_dev, mass, dt, mode, v_shift=shift, phase_tables=phase_tables,
                        precision=precision)
    return StepPlan(grid=grid, dt=dt, mode=mode, mass=mass, potential=potential,
                    threads=threads, native=native)


# ---------------------------------------------------------------------------
# stepping
# ---------------------------------------------------------------------------

def _resident(psi):
    """(wavefunction used for device work, writeback) for our or foreign psi."""
    if isinstance(psi, Wavefunction):
        return psi, None
    w = Wavefunction(np.asarray(psi.amplitudes), psi.grid, getattr(psi, "time", 0.0))
    return w, psi


def _writeback(w: Wavefunction, foreign):
    if foreign is not None:
        foreign.amplitudes = np.array(w.amplitudes)
        foreign.time = w.time
        if hasattr(foreign, "invalidate_norm"):
            foreign.invalidate_norm()


def step(psi, plan: StepPlan):
    """Advance by one dt (propagator.py:110-121)."""
    if not plan.matches(psi):
        raise ValueError("plan was built for a different grid")
    w, foreign = _resident(psi)
    plan.native.advance(w.device_amplitudes(plan.native.torch_dtype), 1)
    w.invalidate_norm()
    if plan.mode == IMAGINARY_TIME:
        w.normalize()
    else:
        w.time += plan.dt
    _writeback(w, foreign)
    return psi


@dataclass
class EvolveStats:
    n_steps: int = 0
    wall_seconds: float = 0.0

    @property
    def steps_per_second(self) -> float:
        return self.n_steps / self.wall_seconds if self.wall_seconds > 0 else float("inf")


def event_schedule(n_steps: int, observers) -> list:
    """Observer event steps (propagator.py:150-155)."""
    events = {0, n_steps}
    for obs in observers:
        if obs.stride <= 0:
            raise ValueError("observer stride must be positive")
        events.update(range(0, n_steps + 1, obs.stride))
    return sorted(e for e in events if e <= n_steps)


class _FusedObservation:
    """Which observer event sums evolve_real asks the segment-end pass for:
    the (partition, margin) of the first PopulationRecorder firing at the
    event, else the margin of an EdgeMonitor (no partition).  Other observers
    of the event hit the same cached sums or make their own reduction."""

    def __init__(self, grid):
        self.grid = grid
        self._xs = None
        self._bounds = {}

    @property
    def xs(self):
        if self._xs is None:
            self._xs = _device.to_device_f64(self.grid.x)
        return self._xs

    def bounds(self, part):
        if part is None:
            return None, None
        key = id(part)
        if key not in self._bounds:
            self._bounds[key] = (part, _device.to_device_f64(part.xb1), _device.to_device_f64(part.xb2))
        return self._bounds[key][1:]

    @staticmethod
    def request(firing):
        from .observables import EdgeMonitor, PopulationRecorder

        for obs in firing:
            if isinstance(obs, PopulationRecorder):
                return obs.partition, int(obs.margin_cells)
        for obs in firing:
            if isinstance(obs, EdgeMonitor):
                return None, int(obs.margin_cells)
        return None


def evolve_real(psi, plan: StepPlan, n_steps: int, observers=()):
    """Propagate n_steps of real time with observers (propagator.py:134-173).

    Observers fire at step 0, at multiples of their stride and at the last
    step, on this thread; between events the half steps are telescoped and
    each segment is a single ctap_advance launch sequence on the current
    CUDA stream.  `stats.wall_seconds` includes a final device synchronize.
    """
    if plan.mode != REAL_TIME:
        raise ValueError("evolve_real requires a real-time plan")
    if not plan.matches(psi):
        raise ValueError("plan was built for a different grid")
    if n_steps < 0:
        raise ValueError("n_steps must be >= 0")
    stats = EvolveStats(n_steps=n_steps)
    schedule = event_schedule(n_steps, observers)
    w, foreign = _resident(psi)
    fused = _FusedObservation(w.grid)
    t0 = _time.perf_counter()
    try:
        current = 0
        for ev in schedule:
            firing = [obs for obs in observers if ev % obs.stride == 0 or ev == n_steps]
            if ev > current:
                d = w.device_amplitudes(plan.native.torch_dtype)
                req = fused.request(firing)
                if req is None:
                    plan.native.advance(d, ev - current)
                else:  # the event's sums come out of the segment-end pass
                    part, margin = req
                    sums = plan.native.advance_observe(d, ev - current, fused.xs, *fused.bounds(part), margin)
                w.time += (ev - current) * plan.dt
                w.invalidate_norm()
                if req is not None:
                    w._obs_cache[int(margin)] = (part, sums.tolist())
                current = ev
            for obs in firing:
                obs.notify(ev, w)
    finally:
        if torch.cuda.is_available():
            torch.cuda.synchronize()
        stats.wall_seconds = _time.perf_counter() - t0
        _writeback(w, foreign)
    return psi, stats


# ---------------------------------------------------------------------------
# energies and imaginary time
# ---------------------------------------------------------------------------

def _kinetic_sums(w: Wavefunction) -> tuple:
    d = w.device_amplitudes(None)
    plan = _aux_plan(w.grid, d.dtype)
    phi = d.clone()
    plan.fft3d(phi, -1)
    s = plan.k2_sums(phi).tolist()
    return s[0], s[1]


def kinetic_expectation(psi, mass: float, workers: int = 1) -> float:
    """<T> in joules (propagator.py:176-185)."""
    from .constants import hbar

    w, _ = _resident(psi)
    sk, s = _kinetic_sums(w)
    return (hbar ** 2 / (2 * mass)) * sk / s


def _potential_from(w: Wavefunction, potential) -> float:
    v_dev = _device.to_device_f64(potential)
    if tuple(v_dev.shape) != tuple(w.grid.n):
        raise ValueError(f"potential shape {tuple(v_dev.shape)} does not match the grid {tuple(w.grid.n)}")
    d = w.device_amplitudes(None)
    # the cached potential-free plan of the grid, V passed to the reduction
    # (no per-call plan with its v_i buffer and device synchronize)
    plan = _aux_plan(w.grid, d.dtype)
    out = torch.empty(2, dtype=torch.float64, device=d.device)
    _lib.call("ctap_v_sums_with", plan.handle, d.data_ptr(), v_dev.data_ptr(), out.data_ptr(), _device.stream_handle())
    s = out.tolist()
    return s[0] / s[1]


def potential_expectation(psi, potential) -> float:
    """<V> = sum V |psi|^2 / sum |psi|^2 (propagator.py:188-190)."""
    w, _ = _resident(psi)
    return _potential_from(w, potential)


def energy_expectation(psi, potential, mass: float, workers: int = 1) -> float:
    return kinetic_expectation(psi, mass, workers) + potential_expectation(psi, potential)


def _energy_on_plan(w: Wavefunction, plan: StepPlan) -> float:
    from .constants import hbar

    sk, s = _kinetic_sums(w)
    sv = plan.native.v_sums(w.device_amplitudes(plan.native.torch_dtype)).tolist()
    return (hbar ** 2 / (2 * plan.mass)) * sk / s + sv[0] / sv[1]


def ground_state_imaginary(grid, potential, seed, tol: float = 1e-10, tau: float = 1e-7,
                           mass: float | None = None, threads: int = 1, check_every: int = 100,
                           max_steps: int = 400_000) -> Wavefunction:
    """Imaginary-time relaxation (propagator.py:198-241), all on the device."""
    if mass is None:
        from .constants import species_mass

        mass = species_mass("li6")
    if tol <= 0:
        raise ValueError("tol must be positive")
    v_dev = _device.to_device_f64(potential)
    if not bool(torch.isfinite(v_dev).all()):
        raise ValueError("potential must be bounded")
    if isinstance(seed, Wavefunction):
        psi = seed
    elif hasattr(seed, "amplitudes") and hasattr(seed, "grid"):
        psi = Wavefunction(np.asarray(seed.amplitudes), grid, getattr(seed, "time", 0.0))
    elif isinstance(seed, torch.Tensor):
        psi = Wavefunction(seed.to(torch.complex128).clone(), grid)
    else:
        psi = Wavefunction(np.asarray(seed, complex).copy(), grid)
    psi.normalize()
    plan = make_plan(grid, v_dev, mass, tau, mode=IMAGINARY_TIME, threads=threads)
    e_prev = _energy_on_plan(psi, plan)
    e_now = e_prev
    done = 0
    while done < max_steps:
        n = min(check_every, max_steps - done)
        plan.native.advance(psi.device_amplitudes(plan.native.torch_dtype), n)
        psi.invalidate_norm()
        psi.normalize()
        done += n
        e_now = _energy_on_plan(psi, plan)
        if abs(e_now - e_prev) < tol * max(abs(e_now), 1e-300):
            return psi
        e_prev = e_now
    raise ConvergenceError(
        f"imaginary-time relaxation did not converge within {max_steps} steps "
        f"(last relative change {abs(e_now - e_prev) / max(abs(e_now), 1e-300):.3e})")


# ---------------------------------------------------------------------------
# observers
# ---------------------------------------------------------------------------

@dataclass
class SnapshotObserver:
    """QWF1 snapshot every `stride` steps (propagator.py:244-257)."""

    out_dir: object
    stride: int = 1
    written: list = field(default_factory=list)

    def notify(self, step_index: int, psi):
        import os

        path = os.path.join(str(self.out_dir), f"psi_{step_index:07d}.qwf")
        write_snapshot(path, psi.amplitudes, psi.grid, time=psi.time)
        self.written.append(path)


class AsyncSnapshotObserver:
    """QWF1 snapshots without stalling the step loop.

    At each event psi is copied device-to-device into a snapshot buffer (one
    HBM read + write), the device-to-host copy of that buffer runs on a side
    stream into pinned memory while the propagation continues, and a writer
    thread produces the same files as SnapshotObserver
    (psi_<step:07d>.qwf, qgrid.write_snapshot).  Call close() (or use it as a
    context manager) to wait for the last file."""

    def __init__(self, out_dir, stride: int = 1):
        import queue
        import threading

        self.out_dir = out_dir
        self.stride = stride
        self.written = []
        self._q = queue.Queue()
        self._free = queue.Queue()  # indices of snapshot buffers not in flight
        for i in range(3):
            self._free.put(i)
        self._bufs = {}
        self._stream = None
        self._err = None
        self._thread = threading.Thread(target=self._writer, daemon=True)
        self._thread.start()

    def _writer(self):
        while True:
            item = self._q.get()
            if item is None:
                return
            path, event, host, grid, t, idx = item
            try:
                event.synchronize()
                write_snapshot(path, host.numpy(), grid, time=t)
                self.written.append(path)
            except BaseException as exc:  # surfaced by close()
                self._err = exc
            finally:
                self._free.put(idx)  # the buffer pair may be refilled now

    def notify(self, step_index: int, psi):
        import os

        d = psi.device_amplitudes(None) if isinstance(psi, Wavefunction) else _device.to_device_c128(psi.amplitudes)
        if self._stream is None:
            self._stream = torch.cuda.Stream(device=d.device)
        key = (tuple(d.shape), d.dtype)
        if key not in self._bufs:
            self._bufs[key] = [(torch.empty_like(d), torch.empty(d.shape, dtype=d.dtype, pin_memory=True))
                               for _ in range(3)]
        idx = self._free.get()  # blocks while all three snapshots are still in flight
        dev_buf, host = self._bufs[key][idx]
        dev_buf.copy_(d)                                # on the propagation stream
        ready = torch.cuda.Event()
        ready.record()
        self._stream.wait_event(ready)
        with torch.cuda.stream(self._stream):
            host.copy_(dev_buf, non_blocking=True)      # overlaps the next steps
            done = torch.cuda.Event()
            done.record(self._stream)
        path = os.path.join(str(self.out_dir), f"psi_{step_index:07d}.qwf")
        self._q.put((path, done, host, psi.grid, psi.time, idx))

    def close(self):
        self._q.put(None)
        self._thread.join()
        if self._err is not None:
            raise self._err

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
        return False


@dataclass
class ProgressObserver:
    """Progress line on stderr (propagator.py:260-285); norm from the device."""

    stride: int = 1000
    stream: object = None
    _t0: float = field(default=None, repr=False)
    _last: tuple = field(default=None, repr=False)

    def notify(self, step_index: int, psi):
        now = _time.perf_counter()
        stream = self.stream if self.stream is not None else sys.stderr
        if self._t0 is None:
            self._t0 = now
            self._last = (step_index, now)
            rate = 0.0
        else:
            s0, t0 = self._last
            rate = (step_index - s0) / (now - t0) if now > t0 else 0.0
            self._last = (step_index, now)
        print(f"step {step_index}  t = {psi.time:.6e} s  norm = {psi.norm():.12f}  "
              f"{rate:.2f} steps/s", file=stream, flush=True)

    @property
    def elapsed(self) -> float:
        return 0.0 if self._t0 is None else _time.perf_counter() - self._t0


def imaginary_step_count_estimate(gap_energy: float, tau: float, decades: float = 10) -> int:
    """Steps for an excited admixture to decay `decades` decades (propagator.py:288-294)."""
    from .constants import hbar

    rate = gap_energy * tau / hbar
    return int(np.ceil(decades * np.log(10.0) / max(rate, 1e-300)))
