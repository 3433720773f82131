"""Benchmark of the B200 split-step propagator (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE config 4 / the metric's config): 512^3 complex128
split-step propagation of the 3D TDSE in the paper-chip CTAP potential
(V from the bit-exact device Biot-Savart kernel, tests/golden/segments_paper.npz),
dt = 1 us, Li-6.  A "step" is one Strang split step; K steps are timed as one
telescoped segment (what evolve_real runs between observer events).  N > 1
runs the x-slab decomposition (one process per GPU, NCCL all-to-all over
NVLink, strong scaling: the grid is fixed).  Rank 0 prints one JSON line.

--impl reference times the CPU oracle (numpy + scipy.fft, the reference
algorithm restated in oracle/) on the same workload with all host threads.
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

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "split-step steps/sec at 512³ complex128 (1/2/4/8 B200) and % of HBM roofline"
GRID_N = (512, 512, 512)
EXTENTS = (20e-6, 4e-6, 1000e-6)          # paper chip footprint (cfg/paper.cfg)
DT = 1e-6
BYTES_PER_POINT_STEP = 136                # 4 sweeps x 32 B + 8 B of V


def _grid():
    from paper_1309_2451_b200 import qgrid

    dy = EXTENTS[1] / GRID_N[1]
    return qgrid.make_grid(*GRID_N, EXTENTS, origin=(-EXTENTS[0] / 2, dy / 2, 0.0))


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


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

def _local_gaussian(grid, x_slice):
    """Normalized Gaussian in the left guide (qgrid.gaussian_packet's separable
    form), restricted to this rank's x-slab; the normalisation uses the global
    separable norm so every rank agrees without communication."""
    c = (-7e-6, 1.43e-6, 200e-6)
    w = (0.25e-6, 0.12e-6, 15e-6)
    f = [np.exp(-((grid.axis(i) - c[i]) ** 2) / (2 * w[i] ** 2)) for i in range(3)]
    nrm = np.sqrt(float((f[0] ** 2).sum() * (f[1] ** 2).sum() * (f[2] ** 2).sum()) * grid.dvol)
    fx = f[0][x_slice] / nrm
    return fx, f[1], f[2]


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1309_2451_b200 import _lib, magfield, observables, propagator, qgrid, slab
    from paper_1309_2451_b200.constants import species_mass

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    m = species_mass("li6")
    grid = _grid()
    lay = slab.SlabLayout(grid.n, world, rank)
    npts = grid.size

    # potential: this rank's x-slab of the paper-chip CTAP potential (one-time)
    chip = magfield.ChipSegments.from_arrays(np.load(os.path.join(ROOT, "tests", "golden", "segments_paper.npz")))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    v_local = magfield.potential_values(chip, grid, lay.x_slice)
    torch.cuda.synchronize()
    t_pot = time.perf_counter() - t0

    fx, fy, fz = _local_gaussian(grid, lay.x_slice)
    amp0 = (torch.from_numpy(fx)[:, None, None] * torch.from_numpy(fy)[None, :, None]
            * torch.from_numpy(fz)[None, None, :]).to(torch.complex128)
    psi = amp0.to(dev).contiguous()
    prop = slab.SlabPropagator(grid, v_local, m, DT, phase_tables=args.phase_tables,
                               transport=args.transport)
    tables = prop.phase_tables

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # warm-up
    for _ in range(args.warmup):
        prop.advance(psi, 1)
    torch.cuda.synchronize()
    barrier()

    # timed region: K steps as one telescoped segment, CUDA events on the stream
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
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
    norm_sums = prop.observe(psi)
    norm = norm_sums[0] * grid.dvol

    # per-pass device times (CUDA events, same stream) -> dominant kernel roofline
    nloc = lay.points
    if world > 1 and prop.transport == "fused":
        bufs = {"psi": psi.reshape(-1), "send": psi.reshape(-1), "recv": psi.reshape(-1)}
    else:
        bufs = {"psi": psi.reshape(-1), "send": prop.send, "recv": prop.recv}
    vtab = 16 if tables & propagator.PHASE_TABLE_V else 8
    ktab = 16 if tables & propagator.PHASE_TABLE_K else 0
    fused = world > 1 and prop.transport == "fused"
    passes = [("z_mid [z^-1 V z]", _lib.PASS_Z_MID, "psi", "psi", 32 + vtab),
              ("y_fwd", _lib.PASS_Y_FWD_TO_PEER if world > 1 else _lib.PASS_Y_FWD, "psi",
               "send" if world > 1 else "psi", 32),
              ("x_kin [x K x^-1]", _lib.PASS_X_KIN, "recv" if world > 1 else "psi",
               "recv" if world > 1 else "psi", 32 + ktab),
              ("y_inv", _lib.PASS_Y_INV_FROM_PEER if world > 1 else _lib.PASS_Y_INV,
               "send" if world > 1 else "psi", "psi", 32)]
    per_pass = {}
    reps = max(3, min(20, args.steps))
    if fused:  # the fused passes need the plan-owned exchange buffers
        passes = [("z_mid [z^-1 V z]", _lib.PASS_Z_MID, "psi", "psi", 32 + vtab)]
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
    dom_name = max(per_pass, key=lambda k: per_pass[k]["ms"])
    dom = per_pass[dom_name]
    peak, peak_kind = _peaks()
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            tr = json.load(fh)
        traffic = tr.get(f"{world}:{dom_name.split()[0]}:tables{tables}")
    except Exception:
        pass

    # end to end through the public API: host-resident psi in pinned memory ->
    # evolve_real with a population observer (single GPU) or the slab
    # propagator with the same event schedule (N GPUs) -> psi back on the host
    e2e = None
    if world > 1 and not args.no_e2e:
        host = torch.empty(lay.slab_shape, dtype=torch.complex128, pin_memory=True)
        host.copy_(amp0)
        host_out = torch.empty_like(host).pin_memory()
        part = observables.symmetric_partition(grid, 3.5e-6)
        stride = max(1, args.steps // 4)
        events = propagator.event_schedule(args.steps, [observables.PopulationRecorder(part, stride=stride)])
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        d = host.to(dev, non_blocking=True)
        cur, rows = 0, []
        for ev in events:
            if ev > cur:
                prop.advance(d, ev - cur)
                cur = ev
            rows.append(prop.observe(d, part.xb1, part.xb2, 2))
        host_out.copy_(d)
        torch.cuda.synchronize()
        t_e2e = max_over_ranks(time.perf_counter() - t0)
        e2e = {"value": args.steps / t_e2e, "unit": "steps/s",
               "h2d_bytes_per_step": 16 * npts / args.steps,
               "d2h_bytes_per_step": (16 * npts + len(rows) * 5 * 8 * world) / args.steps,
               "path": "slab.SlabPropagator.advance/observe on host-resident slabs (pinned), max over ranks",
               "observer_events": len(rows), "seconds": t_e2e}
        del host, host_out, d
    if world == 1 and not args.no_e2e:
        host = torch.empty(grid.n, dtype=torch.complex128, pin_memory=True)
        host.copy_(amp0)
        w = qgrid.Wavefunction(host.numpy(), grid)
        plan = propagator.make_plan(grid, v_local, m, DT, phase_tables=tables)
        part = observables.symmetric_partition(grid, 3.5e-6)
        stride = max(1, args.steps // 4)
        # one untimed warm-up call of the same path (pinned staging buffers,
        # graph capture) -- the timed call is the steady-state user call
        wu = qgrid.Wavefunction(host.numpy().copy(), grid)
        wu, _ = propagator.evolve_real(wu, plan, 2, [observables.PopulationRecorder(part, stride=1)])
        _ = wu.amplitudes
        del wu, _
        rec = observables.PopulationRecorder(part, stride=stride)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        w, _ = propagator.evolve_real(w, plan, args.steps, [rec])
        out = w.amplitudes
        t_e2e = time.perf_counter() - t0
        events = len(rec.trace)
        e2e = {"value": args.steps / t_e2e, "unit": "steps/s",
               "h2d_bytes_per_step": 16 * npts / args.steps,
               "d2h_bytes_per_step": (16 * npts + events * 5 * 8) / args.steps,
               "path": "propagator.evolve_real(host psi, make_plan, K, [PopulationRecorder]) + psi.amplitudes",
               "observer_events": events, "seconds": t_e2e}
        del out, host, w, plan

    cpu = None
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline(grid, v_local.cpu().numpy(), amp0.numpy(), m, steps=args.cpu_steps)

    if rank == 0:
        hbm_achieved = BYTES_PER_POINT_STEP * npts / world / (ms_step * 1e-3) / 1e9
        nvl_bytes = lay.a2a_bytes_per_step()
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
            "config": {"workload": "512^3 CTAP split-step propagation, complex128, dt = 1 us, Li-6 (BASELINE config 4)",
                       "grid": list(GRID_N), "extents_m": list(EXTENTS), "decomposition":
                       (f"x-slab x{world} ({prop.transport} transposes)"
                        + (f"; fused transport unavailable: {prop.transport_fallback}"
                           if getattr(prop, "transport_fallback", None) else "")) if world > 1 else "single GPU",
                       "phase_factors": {0: "both on the fly (exact recipe)", 1: "exp(-iV dt) table, K on the fly",
                                         2: "K table, V on the fly", 3: "both tables"}[tables],
                       "bytes_per_point_step_actual": 128 + vtab + ktab,
                       "l2": "inputs (psi 2 GiB + V 1 GiB) exceed the 126 MB L2; no flush needed"},
            "roofline": {"bound": "hbm", "kernel": dom_name, "achieved": dom["gbs"], "peak": peak,
                         "peak_source": peak_kind, "unit": "GB/s", "frac": dom["gbs"] / peak,
                         "bytes_per_launch": dom["bytes_per_launch"], "ms_per_launch": dom["ms"],
                         "traffic": traffic},
            "step_roofline": {"bytes_per_point": BYTES_PER_POINT_STEP, "achieved_gbs_per_gpu": hbm_achieved,
                              "frac": hbm_achieved / peak,
                              "nvlink_bytes_per_step_per_gpu": nvl_bytes,
                              "nvlink_frac_of_900": (nvl_bytes / (ms_step * 1e-3) / 1e9) / 900.0 if world > 1 else None},
            "per_pass_ms": {k: round(v["ms"], 4) for k, v in per_pass.items()},
            "clocks": clk.summary(),
            "gpu_launches": 4 * args.steps + 1,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "setup": {"potential_seconds": t_pot, "norm_after": norm, "wall_seconds_timed": wall},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ----------------------------------------------------------- CPU oracle arm

def cpu_baseline(grid, v, amp0, mass, steps=3):
    """The reference algorithm (oracle/, numpy + scipy.fft) on the host cores,
    on the same 512^3 workload: make_factors untimed, `steps` split steps timed."""
    from oracle import split_step as orc

    g = orc.as_grid(grid)
    t0 = time.perf_counter()
    f = orc.make_factors(g, v, mass, DT)
    t_plan = time.perf_counter() - t0
    amps = np.array(amp0, dtype=np.complex128, copy=True)
    t0 = time.perf_counter()
    amps = orc.advance(amps, f, steps)
    dt = time.perf_counter() - t0
    cores = os.cpu_count()
    return {"value": steps / dt, "unit": "steps/s", "cores": cores, "kind": "port",
            "sample": f"{steps} telescoped split steps of the full 512^3 grid (oracle.split_step.advance, "
                      f"scipy.fft workers={cores}); make_plan factors built untimed in {t_plan:.1f} s"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import split_step as orc
    from paper_1309_2451_b200.constants import species_mass

    grid = _grid()
    g = orc.as_grid(grid)
    m = species_mass("li6")
    # the CPU path's timing does not depend on the potential contents
    # (runner.py:275-278): the synthetic harmonic trap of run_bench stands in
    v = orc.bench_potential(g, m, 5.0)
    fx, fy, fz = _local_gaussian(grid, slice(None))
    amps = (fx[:, None, None] * fy[None, :, None] * fz[None, None, :]).astype(np.complex128)
    f = orc.make_factors(g, v, m, DT)
    for _ in range(max(0, min(args.warmup, 1))):
        amps = orc.advance(amps, f, 1)
    t0 = time.perf_counter()
    amps = orc.advance(amps, f, 1)
    est = time.perf_counter() - t0
    budget = 120.0
    k = max(1, min(args.steps, int(budget / max(est, 1e-3))))
    t0 = time.perf_counter()
    amps = orc.advance(amps, f, k)
    dt = time.perf_counter() - t0
    val = k / dt
    cores = os.cpu_count()
    line = {
        "metric": METRIC, "value": val, "unit": "steps/s", "n_gpus": args.gpus, "steps": k,
        "warmup": args.warmup, "ms_per_step": 1000.0 / val, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "complex128",
        "data": "synthetic: Gaussian packet; V = the run_bench harmonic field of the same shape (the split step's "
                "cost does not depend on V's values; the paper-chip V takes ~66 min of host numba at 512^3)",
        "config": {"workload": "512^3 CTAP split-step propagation, complex128, dt = 1 us, Li-6 (BASELINE config 4)",
                   "grid": list(GRID_N), "extents_m": list(EXTENTS), "decomposition": "host threads"},
        "impl": "reference",
        "cpu_baseline": {"value": val, "unit": "steps/s", "cores": cores, "kind": "port",
                         "sample": f"{k} telescoped split steps of the full 512^3 grid on {cores} host threads "
                                   f"(oracle.split_step.advance = reference _advance, scipy.fft workers={cores})"},
        "e2e": {"value": val, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--phase-tables", type=int, default=None,
                    help="mask: 1 = exp(-iV dt) table, 2 = exp(-ik^2dt/2) table (default: library default)")
    ap.add_argument("--transport", choices=["fused", "nccl"], default="fused",
                    help="slab transposes: fused NVLink peer stores (default) or NCCL all-to-all")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-steps", type=int, default=3)
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
