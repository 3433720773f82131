"""Benchmark of the B200 split-step propagator (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--grid 512x512x512] [--decomp slab|pencil] [--pencil-c C]
                    [--transport nccl|fused] [--share-device]

Workload (default: BASELINE config 4, the configuration the metric is quoted
on): 512^3 complex128 split-step propagation of the 3D TDSE in the paper-chip
CTAP potential (V from the bit-exact device Biot-Savart kernel on the
product-side chip geometry, paper_1309_2451_b200/chip.py), dt = 1 us, Li-6.
A "step" is one Strang split step; K steps are timed as one telescoped
segment (what evolve_real runs between observer events), after W warm-up
segments of the same length (CUDA-graph capture happens there).

N > 1: one process per GPU (the driver's torchrun, or -- with WORLD_SIZE
unset -- this script re-launches itself under torch.distributed.run), x-slab
decomposition with NCCL all-to-all transposes (--transport fused: CUDA-IPC
peer stores inside the passes) or, with --decomp pencil, a Pr x Pc pencil
grid (config 5).  Strong scaling: the grid is fixed.  Rank 0 prints one JSON
line; the time is the max over ranks of the CUDA-event time.

--share-device: every rank on cuda:0 over gloo (a launch/correctness test of
the N-rank path on a one-GPU box; ranks time-share the GPU, so the number is
not a measurement and says so).

--impl reference times the reference's own CPU path on the box's host cores:
ctapsim (installed unmodified into baseline/_ref) make_plan(threads = all host
threads) + evolve_real, i.e. the telescoped _advance with its pooled pointwise
multiplies and scipy.fft workers (propagator.py:84-107) -- or, where
baseline/_ref is absent, the bitwise-pinned port of it in oracle/.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "split-step steps/sec at 512³ complex128 (1/2/4/8 B200) and % of HBM roofline"
EXTENTS = (20e-6, 4e-6, 1000e-6)          # paper chip footprint (cfg/paper.cfg)
DT = 1e-6
BYTES_PER_POINT_STEP = 136                # 4 sweeps x 32 B + 8 B of V
NVLINK_GBS = 770.0                        # measured peer copy per direction (B200_PROFILING.md; nominal 900)
CONFIG_NAMES = {(64, 64, 64): "BASELINE config 1", (128, 128, 256): "BASELINE config 2",
                (256, 256, 256): "BASELINE config 3", (512, 512, 512): "BASELINE config 4",
                (1024, 1024, 512): "BASELINE config 5"}


def parse_grid(s: str) -> tuple:
    n = tuple(int(v) for v in s.lower().replace(",", "x").split("x"))
    if len(n) != 3:
        raise argparse.ArgumentTypeError("--grid takes NXxNYxNZ")
    return n


def _grid(n):
    from paper_1309_2451_b200 import qgrid

    dy = EXTENTS[1] / n[1]
    return qgrid.make_grid(*n, EXTENTS, origin=(-EXTENTS[0] / 2, dy / 2, 0.0))


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _config(n):
    """The workload both arms report (identical dicts: the arms differ only in
    the implementation; decomposition etc. go to `details`)."""
    name = CONFIG_NAMES.get(tuple(n), "synthetic grid")
    npts = int(n[0]) * int(n[1]) * int(n[2])
    return {"workload": f"{n[0]}x{n[1]}x{n[2]} CTAP split-step propagation, complex128, dt = 1 us, Li-6 ({name})",
            "grid": list(n), "extents_m": list(EXTENTS),
            "l2": (f"inputs larger than L2 (psi + V = {24 * npts / 2**20:.0f} MiB > 126 MB), no flush"
                   if 24 * npts > 126e6 else f"inputs {24 * npts / 2**20:.0f} MiB fit the 126 MB L2 (not flushed)")}


# ---------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
            time.sleep(0.25)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        return False

    def summary(self):
        sm, mx, reasons = [], None, set()
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for name, val in zip(self.NAMES, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------- our arm

def _gaussian_block(grid, x_slice, y_slice):
    """Normalized Gaussian in the left guide (qgrid.gaussian_packet's separable
    form), restricted to this rank's block; the normalisation uses the global
    separable norm so every rank agrees without communication."""
    c = (-7e-6, 1.43e-6, 200e-6)
    w = (0.25e-6, 0.12e-6, 15e-6)
    f = [np.exp(-((grid.axis(i) - c[i]) ** 2) / (2 * w[i] ** 2)) for i in range(3)]
    nrm = np.sqrt(float((f[0] ** 2).sum() * (f[1] ** 2).sum() * (f[2] ** 2).sum()) * grid.dvol)
    return f[0][x_slice] / nrm, f[1][y_slice], f[2]


class _Single:
    """N = 1: the plan's own advance (CUDA graphs of 16 steps)."""

    def __init__(self, grid, v, m):
        from paper_1309_2451_b200 import propagator

        self.plan = propagator.make_plan(grid, v, m, DT)
        self.native = self.plan.native
        self.transport = None

    def advance(self, psi, n):
        self.native.advance(psi.reshape(-1), n)


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1309_2451_b200 import _lib, chip, magfield, observables, pencil, propagator, qgrid, slab
    from paper_1309_2451_b200.constants import species_mass

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    dev_index = 0 if args.share_device else local
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    backend = "gloo" if args.share_device else "nccl"
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    m = species_mass("li6")
    n = args.grid
    grid = _grid(n)
    npts = grid.size

    # decomposition and this rank's block
    Pr = Pc = None
    if world == 1:
        x_sl, y_sl, decomp = slice(None), slice(None), None
        a2a_bytes = 0
    elif args.decomp == "pencil":
        Pc = args.pencil_c or (4 if world >= 8 else 2)
        Pr = world // Pc
        lay = pencil.PencilLayout(tuple(n), Pr, Pc, rank)
        x_sl, y_sl = lay.x_slice, lay.y_slice
        decomp = f"pencil {Pr}x{Pc} (NCCL row/column all-to-alls)"
        a2a_bytes = lay.a2a_bytes_per_step()
    else:
        lay = slab.SlabLayout(tuple(n), world, rank)
        x_sl, y_sl = lay.x_slice, slice(None)
        decomp = f"x-slab x{world} ({args.transport} transposes)"
        a2a_bytes = lay.a2a_bytes_per_step()
    if args.share_device and world > 1:
        decomp += "; share-device test mode: all ranks on cuda:0 over gloo (not a measurement)"
    nloc = npts // world

    # potential: this rank's block of the paper-chip CTAP potential (one-time)
    segs = chip.chip_segments("paper")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    v_local = magfield.potential_on_axes(segs, grid.axis(0)[x_sl], grid.axis(1)[y_sl], grid.axis(2))
    torch.cuda.synchronize()
    t_pot = time.perf_counter() - t0

    fx, fy, fz = _gaussian_block(grid, x_sl, y_sl)
    amp0 = (torch.from_numpy(fx)[:, None, None] * torch.from_numpy(fy)[None, :, None]
            * torch.from_numpy(fz)[None, None, :]).to(torch.complex128)
    psi = amp0.to(dev).contiguous()

    if world == 1:
        prop = _Single(grid, v_local, m)
    elif args.decomp == "pencil":
        rg, cg = pencil.make_groups(Pr, Pc)
        prop = pencil.PencilPropagator(grid, v_local, m, DT, Pr, Pc, rg, cg)
        prop.transport = "nccl"
    else:
        # the fused transport's own stream-ordered flag barrier (also with every
        # rank on one GPU: stream memory operations, no kernel waits on another)
        prop = slab.SlabPropagator(grid, v_local, m, DT, transport=args.transport, chunks=args.chunks,
                                   graphs=args.transport == "fused")
        if prop.transport == "fused":
            decomp += ", one CUDA graph per segment (passes + flag barriers)"
        if prop.chunks > 1:
            decomp += f", {prop.chunks} z chunks: chunk c's all-to-all overlaps chunk c+1's pass"
        if getattr(prop, "transport_fallback", None):
            decomp += f"; fused transport unavailable: {prop.transport_fallback}"

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # warm-up: W segments of the timed length (graph capture, NCCL setup)
    for _ in range(args.warmup):
        prop.advance(psi, args.steps)
    torch.cuda.synchronize()
    barrier()

    # timed region: K steps as one telescoped segment, CUDA events on the stream
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev_index) as clk:
        barrier()
        torch.cuda.synchronize()
        wall0 = time.perf_counter()
        ev0.record(stream)
        prop.advance(psi, args.steps)
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
        wall = time.perf_counter() - wall0
    ms_total = max_over_ranks(ev0.elapsed_time(ev1))
    ms_step = ms_total / args.steps
    steps_per_s = 1000.0 / ms_step
    sums = prop.observe(psi) if world > 1 else prop.native.observe(
        psi, torch.from_numpy(grid.axis(0)).to(dev), None, None, 2).tolist()
    norm = sums[0] * grid.dvol

    # per-pass device times (CUDA events, same stream) -> dominant kernel roofline
    per_pass = {}
    flat = psi.reshape(-1)
    if world == 1:
        bufs = {"psi": flat}
        passes = [("z_mid [z^-1 V z]", _lib.PASS_Z_MID, "psi", "psi", 40),
                  ("y_fwd", _lib.PASS_Y_FWD, "psi", "psi", 32),
                  ("x_kin [x K x^-1]", _lib.PASS_X_KIN, "psi", "psi", 32),
                  ("y_inv", _lib.PASS_Y_INV, "psi", "psi", 32)]
    elif args.decomp == "pencil":
        bufs = dict(prop.bufs, psi=flat)
        passes = [("z_mid [z^-1 V z]", _lib.PASS_PZ_MID, "zc", "zc", 40),
                  ("y_fwd", _lib.PASS_PY_FWD, "yb", "xp", 32),
                  ("x_kin [x K x^-1]", _lib.PASS_PX_KIN, "xr", "xr", 32),
                  ("y_inv", _lib.PASS_PY_INV, "xp", "yb", 32)]
    elif prop.transport == "fused":  # the fused passes need the peer buffers: z only
        bufs = {"psi": flat}
        passes = [("z_mid [z^-1 V z]", _lib.PASS_Z_MID, "psi", "psi", 40)]
    else:
        bufs = {"psi": flat, "send": prop.send, "recv": prop.recv}
        passes = [("z_mid [z^-1 V z]", _lib.PASS_Z_MID, "psi", "psi", 40),
                  ("y_fwd", _lib.PASS_Y_FWD_TO_PEER, "psi", "send", 32),
                  ("x_kin [x K x^-1]", _lib.PASS_X_KIN, "recv", "recv", 32),
                  ("y_inv", _lib.PASS_Y_INV_FROM_PEER, "send", "psi", 32)]
    reps = max(3, min(20, args.steps))
    for name, kind, src, dst, bpp in passes:
        for _ in range(2):
            prop.native.run_pass(kind, bufs[src], bufs[dst])
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(stream)
        for _ in range(reps):
            prop.native.run_pass(kind, bufs[src], bufs[dst])
        b.record(stream)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / reps
        per_pass[name] = {"ms": ms, "bytes_per_launch": bpp * nloc, "gbs": bpp * nloc / (ms * 1e-3) / 1e9}
    # cost of an observer event (PopulationRecorder sums) on top of a K-step
    # segment: fused into the segment-end pass vs the standalone reduction
    obs_cost = None
    if world == 1:
        part = observables.symmetric_partition(grid, 3.5e-6)
        xs_d = torch.from_numpy(grid.axis(0)).to(dev)
        xb = (torch.from_numpy(part.xb1).to(dev), torch.from_numpy(part.xb2).to(dev))

        # one-step segments, the three variants interleaved call by call
        # (A B C A B C ...; clock drift hits neighbours alike), each call
        # bracketed by its own CUDA events; medians of 25 calls per variant
        plain = lambda: prop.native.advance(flat, 1)
        fusedo = lambda: prop.native.advance_observe(flat, 1, xs_d, *xb, 2)
        separate = lambda: (prop.native.advance(flat, 1), prop.native.observe(flat, xs_d, *xb, 2))
        variants = (plain, fusedo, separate)
        for f in variants:
            f()
        evs = [[] for _ in variants]
        torch.cuda.synchronize()
        for _ in range(25):
            for i, f in enumerate(variants):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                f()
                b.record(stream)
                evs[i].append((a, b))
        torch.cuda.synchronize()
        t_p, t_f, t_s = (statistics.median(a.elapsed_time(b) for a, b in e) for e in evs)
        obs_cost = {"segment_steps": 1, "segment_ms": t_p,
                    "extra_ms_fused": t_f - t_p, "extra_ms_standalone_reduction": t_s - t_p,
                    "method": "CUDA events around each call, 1-step segments, the variants interleaved, "
                              "median of 25 per variant"}
    dom_name = max(per_pass, key=lambda k: per_pass[k]["ms"])
    dom = per_pass[dom_name]
    peak, peak_kind = _peaks()
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            tr = json.load(fh)
        traffic = tr.get(f"{world}:{dom_name.split()[0]}:tables0:{n[0]}x{n[1]}x{n[2]}")
    except Exception:
        pass

    # end to end through the public API: host-resident psi (pinned) -> the
    # propagation with a population observer -> psi back on the host
    e2e = None
    if not args.no_e2e:
        part = observables.symmetric_partition(grid, 3.5e-6)
        stride = max(1, args.steps // 4)
        host = torch.empty(tuple(amp0.shape), dtype=torch.complex128, pin_memory=True)
        host.copy_(amp0)
        if world == 1:
            plan = prop.plan
            # one untimed call of the same path first (pinned staging, graphs)
            wu = qgrid.Wavefunction(host.numpy().copy(), grid)
            wu, _ = propagator.evolve_real(wu, plan, args.steps, [observables.PopulationRecorder(part, stride=stride)])
            _ = wu.amplitudes
            del wu, _
            w = qgrid.Wavefunction(host.numpy(), grid)
            rec = observables.PopulationRecorder(part, stride=stride)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            w, _ = propagator.evolve_real(w, plan, args.steps, [rec])
            out = w.amplitudes
            t_e2e = time.perf_counter() - t0
            events = len(rec.trace)
            path = "propagator.evolve_real(host psi, make_plan, K, [PopulationRecorder]) + psi.amplitudes"
            del out, w
        else:
            host_out = torch.empty_like(host).pin_memory()
            events = propagator.event_schedule(args.steps, [observables.PopulationRecorder(part, stride=stride)])
            xb = (part.xb1, part.xb2)
            barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            d = host.to(dev, non_blocking=True)
            cur, rows = 0, []
            for ev in events:
                if ev > cur:
                    prop.advance(d, ev - cur)
                    cur = ev
                rows.append(prop.observe(d, *xb, 2))
            host_out.copy_(d)
            torch.cuda.synchronize()
            t_e2e = max_over_ranks(time.perf_counter() - t0)
            events = len(rows)
            path = f"{type(prop).__name__}.advance/observe on host-resident blocks (pinned), max over ranks"
            del host_out, d
        e2e = {"value": args.steps / t_e2e, "unit": "steps/s",
               "h2d_bytes_per_step": 16 * npts / args.steps,
               "d2h_bytes_per_step": (16 * npts + events * 5 * 8 * world) / args.steps,
               "path": path, "observer_events": events, "seconds": t_e2e}
        del host

    cpu = None
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline(grid, v_local.cpu().numpy(), amp0.numpy(), m, steps=args.cpu_steps)

    if rank == 0:
        hbm_floor_ms = BYTES_PER_POINT_STEP * nloc / (peak * 1e9) * 1e3
        nvl_floor_ms = a2a_bytes / (NVLINK_GBS * 1e9) * 1e3
        hbm_achieved = BYTES_PER_POINT_STEP * nloc / (ms_step * 1e-3) / 1e9
        l2_note = ("inputs (psi + V = 24 B/pt) exceed the 126 MB L2; no flush needed" if 24 * nloc > 126e6 else
                   "psi + V fit in the 126 MB L2 (L2-resident steps; HBM fraction is not a DRAM measurement)")
        line = {
            "metric": METRIC,
            "value": steps_per_s,
            "unit": "steps/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_step,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "complex128",
            "data": "synthetic: paper-chip CTAP potential (device Biot-Savart, 9605 segments) and a Gaussian packet",
            "config": _config(n),
            "details": {"decomposition": decomp or "single GPU",
                        "step_schedule": ("x-slab position blocks: %d planes on %d streams" % prop.native.step_schedule()
                                          if isinstance(prop, _Single) and prop.native.step_schedule()[0]
                                          else "plane order"),
                        "phase_factors": "both on the fly (exact recipe)",
                        "bytes_per_point_step": BYTES_PER_POINT_STEP, "l2": l2_note},
            "roofline": {"bound": "hbm", "kernel": dom_name, "achieved": dom["gbs"], "peak": peak,
                         "peak_source": peak_kind, "unit": "GB/s", "frac": dom["gbs"] / peak,
                         "bytes_per_launch": dom["bytes_per_launch"], "ms_per_launch": dom["ms"],
                         "traffic": traffic},
            "step_roofline": {"bytes_per_point": BYTES_PER_POINT_STEP, "achieved_gbs_per_gpu": hbm_achieved,
                              "hbm_fraction": hbm_achieved / peak, "hbm_floor_ms": hbm_floor_ms,
                              "nvlink_bytes_per_step_per_gpu": a2a_bytes,
                              "nvlink_gbs_per_gpu": a2a_bytes / (ms_step * 1e-3) / 1e9 if world > 1 else None,
                              "nvlink_peak_gbs": NVLINK_GBS if world > 1 else None,
                              "nvlink_fraction": (a2a_bytes / (ms_step * 1e-3) / 1e9) / NVLINK_GBS
                              if world > 1 else None,
                              "nvlink_floor_ms": nvl_floor_ms if world > 1 else None,
                              "combined": max(hbm_floor_ms, nvl_floor_ms) / ms_step},
            "per_pass_ms": {k: round(v["ms"], 4) for k, v in per_pass.items()},
            "observer_event": obs_cost,
            "clocks": clk.summary(),
            "gpu_launches": prop.native.launches(args.steps) if isinstance(prop, _Single) else 4 * args.steps + 1,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "setup": {"potential_seconds": t_pot, "norm_after": norm, "wall_seconds_timed": wall},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        if hasattr(prop, "close"):
            prop.close()
        dist.destroy_process_group()


# ----------------------------------------------------------- CPU oracle arm

def cpu_baseline(grid, v, amp0, mass, steps=3):
    """The reference's CPU path on the host cores, on the same workload (the
    same V and psi0): ctapsim's own make_plan + evolve_real when it is
    installed in baseline/_ref, else the bitwise-pinned port (oracle/, the
    reference's _advance with its pooled multiplies).  make_plan untimed,
    `steps` split steps timed."""
    cores = os.cpu_count()
    n = grid.n
    ref = _import_reference()
    if ref is not None:
        rprop, rq, _ = ref
        g = rq.make_grid(*n, tuple(grid.extents), origin=tuple(grid.origin))
        t0 = time.perf_counter()
        plan = rprop.make_plan(g, v, mass, DT, threads=cores)
        t_plan = time.perf_counter() - t0
        psi = rq.Wavefunction(np.array(amp0, dtype=np.complex128, copy=True), g)
        t0 = time.perf_counter()
        rprop.evolve_real(psi, plan, steps)
        dt = time.perf_counter() - t0
        kind, what = "reference", (f"ctapsim.propagator.evolve_real (the reference package, baseline/_ref), "
                                   f"make_plan(threads={cores})")
    else:
        from oracle import split_step as orc

        g = orc.as_grid(grid)
        t0 = time.perf_counter()
        f = orc.make_factors(g, v, mass, DT)
        t_plan = time.perf_counter() - t0
        amps = np.array(amp0, dtype=np.complex128, copy=True)
        t0 = time.perf_counter()
        amps = orc.advance(amps, f, steps)
        dt = time.perf_counter() - t0
        kind, what = "port", (f"oracle.split_step.advance = reference _advance: scipy.fft workers={cores}, "
                              f"multiplies chunked over a {cores}-thread pool")
    return {"value": steps / dt, "unit": "steps/s", "cores": cores, "kind": kind,
            "sample": f"{steps} telescoped split steps of the full {n[0]}x{n[1]}x{n[2]} grid ({what}); "
                      f"make_plan built untimed in {t_plan:.1f} s"}


def _import_reference():
    """The reference package itself (ctapsim), installed unmodified into
    baseline/_ref (`pip install --no-index --no-build-isolation --no-deps
    --target baseline/_ref <copy of /root/reference/pkg>`; git-ignored, travels
    to the GPU box with the snapshot).  None if it is not there."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(os.path.join(ref, "ctapsim")) and ref not in sys.path:
        sys.path.insert(0, ref)
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join("/tmp", "ctapsim_numba_cache"))
    try:
        from ctapsim import constants, propagator, qgrid  # noqa: F401

        return propagator, qgrid, constants
    except Exception:  # noqa: BLE001 - fall back to the pinned port
        return None


def _timed_steps(advance_k, budget: float, max_steps: int):
    """One untimed warm step, a 1-step estimate, then as many steps as fit the
    budget (bounded CPU sample) timed as one call: (steps, seconds)."""
    advance_k(1)
    t0 = time.perf_counter()
    advance_k(1)
    est = time.perf_counter() - t0
    k = max(1, min(max_steps, int(budget / max(est, 1e-3))))
    t0 = time.perf_counter()
    advance_k(k)
    return k, time.perf_counter() - t0


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n = args.grid
    cores = os.cpu_count()
    fx, fy, fz = _gaussian_block(_grid(n), slice(None), slice(None))
    amps = (fx[:, None, None] * fy[None, :, None] * fz[None, None, :]).astype(np.complex128)
    ref = _import_reference()
    if ref is not None:
        # the reference's own public API and stock code path: make_plan with
        # all host threads, evolve_real (telescoped _advance, pooled multiplies,
        # scipy.fft workers) -- what runner.run_bench times (runner.py:295-302)
        rprop, rq, rc = ref
        m = rc.species_mass("li6")
        dy = EXTENTS[1] / n[1]
        g = rq.make_grid(*n, EXTENTS, origin=(-EXTENTS[0] / 2, dy / 2, 0.0))
        x, y, z = g.meshgrid()
        c = [g.origin[i] + g.extents[i] / 2 for i in range(3)]
        om = 2 * np.pi * 5.0
        v = 0.5 * m * om ** 2 * ((x - c[0]) ** 2 + (y - c[1]) ** 2 + (z - c[2]) ** 2)  # runner.py:284-288
        del x, y, z
        plan = rprop.make_plan(g, v, m, DT, threads=cores)
        psi = rq.Wavefunction(amps, g)
        k, dt = _timed_steps(lambda s: rprop.evolve_real(psi, plan, s), 120.0, args.steps)
        kind = "reference"
        sample = (f"{k} steps of ctapsim.propagator.evolve_real (the reference package itself, installed "
                  f"unmodified in baseline/_ref) on the full {n[0]}x{n[1]}x{n[2]} grid, make_plan(threads={cores}):"
                  f" pooled multiplies + scipy.fft workers={cores}")
    else:
        from oracle import split_step as orc
        from paper_1309_2451_b200.constants import species_mass

        g = orc.as_grid(_grid(n))
        m = species_mass("li6")
        v = orc.bench_potential(g, m, 5.0)
        f = orc.make_factors(g, v, m, DT)
        state = {"a": amps}

        def adv(s):
            state["a"] = orc.advance(state["a"], f, s)

        k, dt = _timed_steps(adv, 120.0, args.steps)
        kind = "port"
        sample = (f"{k} telescoped split steps of the full {n[0]}x{n[1]}x{n[2]} grid on {cores} host threads "
                  f"(oracle.split_step.advance = reference _advance with its thread-pooled multiplies, "
                  f"scipy.fft workers={cores}); ctapsim is not installed in baseline/_ref here, so its "
                  f"bitwise-pinned port runs")
    val = k / dt
    line = {
        "metric": METRIC, "value": val, "unit": "steps/s", "n_gpus": args.gpus, "steps": k,
        "warmup": args.warmup, "ms_per_step": 1000.0 / val, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "complex128",
        "data": "synthetic: Gaussian packet; V = run_bench's harmonic trap of the same grid (the CPU step's "
                "cost does not depend on V's values; our arm uses the paper-chip V)",
        "config": _config(n),
        "details": {"decomposition": "host threads"},
        "impl": "reference",
        "cpu_baseline": {"value": val, "unit": "steps/s", "cores": cores, "kind": kind, "sample": sample},
        "e2e": {"value": val, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn(args):
    """`python bench.py --gpus N` without a launcher: re-run this script under
    torch.distributed.run, one process per GPU (rank 0 prints the line)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--grid", type=parse_grid, default=(512, 512, 512),
                    help="NXxNYxNZ (default 512x512x512, BASELINE config 4; 1024x1024x512 is config 5)")
    ap.add_argument("--decomp", choices=["slab", "pencil"], default="slab",
                    help="N > 1: x-slabs (default) or a Pr x Pc pencil grid")
    ap.add_argument("--pencil-c", type=int, default=0, help="pencil columns Pc (default 4 at N >= 8, else 2)")
    ap.add_argument("--transport", choices=["nccl", "fused"], default="nccl",
                    help="slab transposes: NCCL all-to-all (default) or fused CUDA-IPC peer stores")
    ap.add_argument("--chunks", type=int, default=4,
                    help="slab NCCL transport: z chunks whose all-to-alls overlap the next chunk's pass (1: serial)")
    ap.add_argument("--share-device", action="store_true",
                    help="all ranks on cuda:0 over gloo: a launch test of the N-rank path on one GPU")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-steps", type=int, default=3)
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
        return 0
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn(args)
    run_ours(args)
    return 0


if __name__ == "__main__":
    sys.exit(main())
