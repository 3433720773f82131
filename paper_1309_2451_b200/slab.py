"""x-slab domain decomposition of the split-step propagator over several GPUs
(one process per GPU, torch.distributed over NCCL / NVLink).

Rank r of P owns the x-planes [r*nx/P, (r+1)*nx/P) of psi and V (both
contiguous slabs).  The z and y transforms are local; the x transform needs
whole x-lines, so every step transposes twice:

    [z^-1 V z]  ->  y (output written peer-major)  -> all-to-all
    -> [x K x^-1] on the y-slab (x, y_local, z)     -> all-to-all
    -> y^-1 (input read peer-major)                 -> next step

The y passes write/read the all-to-all buffers directly in peer-major order
([peer][x_local][y_local][z]), so no pack/unpack sweep exists, and the
receive buffer of the first all-to-all is already the natural y-slab layout
the x pass runs on.  Observer sums are per-rank partials combined in rank
order on every rank (deterministic, no float atomics).

Two transports: "nccl" (the y/x passes write the all-to-all buffers, NCCL
all_to_all_single moves them) and "fused" (the y pass and the x pass store
their outputs directly into the other ranks' buffers through CUDA-IPC peer
mappings over NVLink, so the transpose rides inside the pass's own HBM write
and there is no separate all-to-all sweep; a stream-ordered barrier follows
each).  The schedules are independent of the compute backend, so the same
code drives the CUDA passes here, the virtual-rank GPU tests and the CPU
emulation in the gloo tests (tests/test_slab_gloo.py).
"""

from __future__ import annotations

import ctypes
import weakref
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import _device, _lib
from .propagator import REAL_TIME, NativePlan
from .qgrid import as_simgrid


@dataclass(frozen=True)
class SlabLayout:
    """Sizes of the x-slab / y-slab decomposition of an (nx, ny, nz) grid."""

    n: tuple
    P: int
    rank: int

    def __post_init__(self):
        nx, ny, _ = self.n
        if nx % self.P or ny % self.P:
            raise ValueError(f"nx={nx} and ny={ny} must be divisible by {self.P} ranks")
        if not 0 <= self.rank < self.P:
            raise ValueError(f"rank {self.rank} out of range for {self.P} ranks")

    @property
    def nx_local(self) -> int:
        return self.n[0] // self.P

    @property
    def ny_local(self) -> int:
        return self.n[1] // self.P

    @property
    def x_slice(self) -> slice:
        return slice(self.rank * self.nx_local, (self.rank + 1) * self.nx_local)

    @property
    def y_slice(self) -> slice:
        return slice(self.rank * self.ny_local, (self.rank + 1) * self.ny_local)

    @property
    def slab_shape(self) -> tuple:      # position-space x-slab
        return (self.nx_local, self.n[1], self.n[2])

    @property
    def yslab_shape(self) -> tuple:     # x-pass y-slab
        return (self.n[0], self.ny_local, self.n[2])

    @property
    def points(self) -> int:
        return self.nx_local * self.n[1] * self.n[2]

    def a2a_bytes_per_step(self, itemsize: int = 16) -> int:
        """Bytes this rank sends over NVLink per split step (2 transposes)."""
        return 2 * (self.P - 1) * self.points // self.P * itemsize


# pass sequence of one telescoped segment (propagator.py:98-107)
def segment_schedule(n_steps: int):
    """Yield the operations of n merged steps on one rank:
    ('pass', kind, src, dst) with buffer names 'psi' / 'send' / 'recv', and
    ('a2a', src, dst)."""
    if n_steps <= 0:
        return
    yield ("pass", _lib.PASS_Z_FIRST, "psi", "psi")
    for j in range(n_steps):
        yield ("pass", _lib.PASS_Y_FWD_TO_PEER, "psi", "send")
        yield ("a2a", "send", "recv")
        yield ("pass", _lib.PASS_X_KIN, "recv", "recv")
        yield ("a2a", "recv", "send")
        yield ("pass", _lib.PASS_Y_INV_FROM_PEER, "send", "psi")
        yield ("pass", _lib.PASS_Z_MID if j < n_steps - 1 else _lib.PASS_Z_LAST, "psi", "psi")


def segment_schedule_fused(n_steps: int):
    """The same n merged steps with the transposes fused into the passes:
    the y pass stores its output straight into every rank's y-slab buffer and
    the x pass into every rank's peer-major buffer (NVLink peer stores), each
    followed by a stream-ordered cross-rank barrier.  Ops: ('pass', kind, src,
    dst) and ('barrier',)."""
    if n_steps <= 0:
        return
    yield ("pass", _lib.PASS_Z_FIRST, "psi", "psi")
    for j in range(n_steps):
        yield ("pass", _lib.PASS_Y_FWD_TO_PEERS, "psi", "psi")
        yield ("barrier",)
        yield ("pass", _lib.PASS_X_KIN_TO_PEERS, "yslab", "yslab")
        yield ("barrier",)
        yield ("pass", _lib.PASS_Y_INV_FROM_PEER, "peer", "psi")
        yield ("pass", _lib.PASS_Z_MID if j < n_steps - 1 else _lib.PASS_Z_LAST, "psi", "psi")


def segment_schedule_chunked(n_steps: int, chunks: int):
    """The same n merged steps with the kinetic block split into `chunks` z
    chunks (chunk-major transpose buffers, ctap_pass_zchunk): ops
    ('pass', kind, src, dst), ('cpass', kind, src, dst, c) and
    ('a2a', src, dst, c).  Listed in issue order: all y passes, then the
    chunks' all-to-alls, ... so chunk c's transfer overlaps chunk c+1's pass
    when passes and transfers run on two streams."""
    if n_steps <= 0:
        return
    yield ("pass", _lib.PASS_Z_FIRST, "psi", "psi")
    C = range(chunks)
    for j in range(n_steps):
        for c in C:
            yield ("cpass", _lib.PASS_Y_FWD_TO_PEER, "psi", "send", c)
        for c in C:
            yield ("a2a", "send", "recv", c)
        for c in C:
            yield ("cpass", _lib.PASS_X_KIN, "recv", "recv", c)
        for c in C:
            yield ("a2a", "recv", "send", c)
        for c in C:
            yield ("cpass", _lib.PASS_Y_INV_FROM_PEER, "send", "psi", c)
        yield ("pass", _lib.PASS_Z_MID if j < n_steps - 1 else _lib.PASS_Z_LAST, "psi", "psi")


class DeviceBuffer:
    """cudaMalloc'd buffer owned by libctap (exportable through CUDA IPC)."""

    def __init__(self, nbytes: int):
        self.nbytes = int(nbytes)
        h = ctypes.c_void_p()
        _lib.call("ctap_device_alloc", self.nbytes, ctypes.byref(h))
        self.ptr = int(h.value)
        self._fin = weakref.finalize(self, _lib.load().ctap_device_free, ctypes.c_void_p(self.ptr))

    def ipc_handle(self) -> bytes:
        buf = ctypes.create_string_buffer(64)
        _lib.call("ctap_ipc_handle", ctypes.c_void_p(self.ptr), buf)
        return buf.raw


def open_ipc(handle: bytes) -> int:
    h = ctypes.c_void_p()
    _lib.call("ctap_ipc_open", ctypes.create_string_buffer(handle, 64), ctypes.byref(h))
    return int(h.value)


def _host_staged(group) -> bool:
    """Device tensors over a non-NCCL group (gloo: the CPU tests and the
    bench's --share-device mode, several ranks on one GPU) go through host
    memory."""
    return dist.get_backend(group) != "nccl"


def all_to_all_c(dst: torch.Tensor, src: torch.Tensor, group=None):
    """all_to_all_single of complex buffers (equal chunks, rank order)."""
    if src.is_cuda and _host_staged(group):
        h_dst = torch.empty(torch.view_as_real(dst).shape, dtype=torch.view_as_real(dst).dtype)
        dist.all_to_all_single(h_dst, torch.view_as_real(src).cpu(), group=group)
        torch.view_as_real(dst).copy_(h_dst)
    else:
        dist.all_to_all_single(torch.view_as_real(dst), torch.view_as_real(src), group=group)


def combine_in_rank_order(local: torch.Tensor, group=None) -> torch.Tensor:
    """Sum per-rank partial sums in rank order (bitwise identical on every rank)."""
    P = dist.get_world_size(group)
    dev = local.device
    if local.is_cuda and _host_staged(group):
        local = local.cpu()
    parts = [torch.empty_like(local) for _ in range(P)]
    dist.all_gather(parts, local, group=group)
    total = parts[0].clone()
    for p in parts[1:]:
        total += p
    return total.to(dev)


class SlabPropagator:
    """Real- or imaginary-time propagation of one rank's x-slab on its GPU."""

    def __init__(self, grid, v_local, mass: float, dt: float, group=None, mode: str = REAL_TIME,
                 v_shift: float = 0.0, phase_tables: int | None = None, precision: str = "complex128",
                 transport: str = "nccl", barrier=None, chunks: int = 1, graphs: bool = False):
        self.grid = as_simgrid(grid)
        self.group = group
        self.graphs = bool(graphs)  # fused transport: one CUDA graph per segment
        # fused transport's cross-rank barrier after each pass: "flags" (default:
        # stream-ordered peer flags, ctap_flag_barrier), "nccl" (a 1-float NCCL
        # all-reduce) or a callable (tests: host barriers)
        if not (barrier is None or callable(barrier) or barrier in ("flags", "nccl")):
            raise ValueError(f"unknown barrier {barrier!r}")
        self._barrier_fn = "flags" if barrier is None else barrier
        P = dist.get_world_size(group) if dist.is_initialized() else 1
        r = dist.get_rank(group) if dist.is_initialized() else 0
        self.layout = SlabLayout(tuple(self.grid.n), P, r)
        if tuple(v_local.shape) != self.layout.slab_shape:
            raise ValueError(f"local potential shape {tuple(v_local.shape)} != slab {self.layout.slab_shape}")
        self.v_local = _device.to_device_f64(v_local)
        from .propagator import DEFAULT_PHASE_TABLES

        if phase_tables is None:
            phase_tables = DEFAULT_PHASE_TABLES
        self.phase_tables = int(phase_tables)
        self.native = NativePlan(self.grid, self.v_local, mass, dt, mode, v_shift=v_shift,
                                 slab_p=P, slab_r=r, phase_tables=phase_tables, precision=precision)
        dev = self.v_local.device
        dt_ = self.native.torch_dtype
        if transport not in ("nccl", "fused"):
            raise ValueError(f"unknown transport {transport!r}")
        self.transport = transport if P > 1 else "nccl"
        # why the fused transport was not used (None when it was, or not asked for)
        self.transport_fallback = None
        if self.transport == "fused" and not self._setup_fused(dt_):
            self.transport = "nccl"
        if self.transport == "nccl":
            self.send = torch.empty(self.layout.points, dtype=dt_, device=dev)
            self.recv = torch.empty(self.layout.points, dtype=dt_, device=dev)
        # NCCL transport by z chunks: chunk c's all-to-all on a second stream
        # overlaps chunk c+1's pass (chunk-major buffers, ctap_pass_zchunk)
        nz = self.grid.n[2]
        self.chunks = int(chunks) if (self.transport == "nccl" and P > 1 and chunks > 1
                                      and nz % (8 * int(chunks)) == 0 and not (self.phase_tables & 2)) else 1
        self._comm = torch.cuda.Stream(device=dev) if self.chunks > 1 and dev.type == "cuda" else None

    def _setup_fused(self, dtype) -> bool:
        """Allocate this rank's y-slab and peer-major buffers, exchange CUDA IPC
        handles with every rank and register the peer-mapped addresses.

        Collective and all-or-nothing: every rank reaches the same collectives
        whatever fails locally, and if any rank cannot export or map a peer
        buffer (no P2P path, IPC blocked) ALL ranks return False and the plan
        uses the NCCL all-to-all transport instead (`transport_fallback` says
        why).  Either transport computes bitwise the same slabs."""
        itemsize = 8 if dtype == torch.complex64 else 16
        nbytes = self.layout.points * itemsize
        err = None
        mine = None
        try:
            self.yslab = DeviceBuffer(nbytes)
            self.peer = DeviceBuffer(nbytes)
            self.flags = DeviceBuffer(4 * self.layout.P)  # zeroed: the barrier's epoch slots
            mine = (self.yslab.ipc_handle(), self.peer.ipc_handle(), self.flags.ipc_handle())
        except Exception as e:  # noqa: BLE001 - reported to every rank below
            err = f"rank {self.layout.rank}: {e}"
        handles = [None] * self.layout.P
        dist.all_gather_object(handles, mine, group=self.group)
        self._opened = []
        tabs = ([], [])
        self._peer_flags = []
        if err is None and all(h is not None for h in handles):
            try:
                for q, (hy, hp, hf) in enumerate(handles):
                    if q == self.layout.rank:
                        tabs[0].append(self.yslab.ptr)
                        tabs[1].append(self.peer.ptr)
                        self._peer_flags.append(self.flags.ptr)
                    else:
                        py, pp, pf = open_ipc(hy), open_ipc(hp), open_ipc(hf)
                        self._opened += [py, pp, pf]
                        tabs[0].append(py)
                        tabs[1].append(pp)
                        self._peer_flags.append(pf)
                self.native.set_peer_buffers(0, tabs[0])
                self.native.set_peer_buffers(1, tabs[1])
            except Exception as e:  # noqa: BLE001
                err = f"rank {self.layout.rank}: {e}"
        elif err is None:
            err = "a peer rank could not export its buffers"
        on_dev = dist.get_backend(self.group) == "nccl"
        ok = torch.tensor([0.0 if err else 1.0], dtype=torch.float32,
                          device=self.v_local.device if on_dev else "cpu")
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=self.group)
        if ok.item() < 1.0:
            self.transport_fallback = err or "a peer rank could not map the peer buffers"
            # unregister before unmapping: no plan keeps a peer address of a
            # closed mapping (the fused passes then fail loudly instead)
            self.native.clear_peer_buffers()
            for ptr in self._opened:
                _lib.load().ctap_ipc_close(ctypes.c_void_p(ptr))
            self._opened = []
            self.yslab = self.peer = self.flags = None
            return False
        self._flag = torch.zeros(1, dtype=torch.float32, device=self.v_local.device)
        self._epoch = 0
        self._peer_flag_arr = (ctypes.c_void_p * self.layout.P)(*self._peer_flags)
        return True

    def close(self):
        """Release the fused transport's peer mappings (collective: every rank
        calls it).  A barrier first, so no rank unmaps a buffer another rank
        may still be storing into; then the plan's peer tables are cleared and
        the CUDA IPC mappings closed.  Idempotent; the NCCL transport has
        nothing to release."""
        if self.transport != "fused":
            return
        torch.cuda.synchronize(self.v_local.device)
        dist.barrier(group=self.group)
        self.native.clear_peer_buffers()
        for ptr in self._opened:
            _lib.load().ctap_ipc_close(ctypes.c_void_p(ptr))
        self._opened = []
        dist.barrier(group=self.group)  # every rank unmapped before the owners free
        self.yslab = self.peer = self.flags = None
        self.transport = "closed"

    def _barrier(self):
        # stream-ordered: every rank's preceding pass (and its system fence)
        # completes before any rank's next pass starts
        if self._barrier_fn == "flags":
            self._epoch += 1
            _lib.call("ctap_flag_barrier", self._peer_flag_arr, ctypes.c_void_p(self.flags.ptr), self.layout.P,
                      self.layout.rank, self._epoch, _device.stream_handle())
        elif self._barrier_fn == "nccl":
            dist.all_reduce(self._flag, group=self.group)
        else:
            self._barrier_fn()

    def _a2a(self, src: torch.Tensor, dst: torch.Tensor):
        if self.layout.P == 1:
            dst.copy_(src)
        else:
            all_to_all_c(dst, src, self.group)

    def advance(self, psi_local: torch.Tensor, n_steps: int):
        """n telescoped steps on this rank's slab (collective: all ranks call)."""
        if n_steps < 0:
            raise ValueError("n_steps must be >= 0")
        if self.layout.P == 1:
            self.native.advance(psi_local, n_steps)
            return
        if self.transport == "closed":
            raise RuntimeError("SlabPropagator was closed")
        if self.transport == "fused":
            if self.graphs and self._barrier_fn == "flags":
                self._advance_fused_graph(psi_local, n_steps)
                return
            self._fused_ops(psi_local, n_steps)
            return
        if self.chunks > 1:
            self._advance_chunked(psi_local, n_steps)
            return
        bufs = {"psi": psi_local.reshape(-1), "send": self.send, "recv": self.recv}
        for op in segment_schedule(n_steps):
            if op[0] == "pass":
                _, kind, src, dst = op
                self.native.run_pass(kind, bufs[src], bufs[dst])
            else:
                self._a2a(bufs[op[1]], bufs[op[2]])

    def _fused_ops(self, psi_local: torch.Tensor, n_steps: int):
        addr = {"psi": psi_local.data_ptr(), "yslab": self.yslab.ptr, "peer": self.peer.ptr}
        for op in segment_schedule_fused(n_steps):
            if op[0] == "pass":
                self.native.run_pass_ptr(op[1], addr[op[2]], addr[op[3]])
            else:
                self._barrier()

    def _advance_fused_graph(self, psi_local: torch.Tensor, n_steps: int):
        """The fused segment as ONE CUDA graph per rank: its passes and flag
        barriers (stream memory operations) captured once per (psi, n) and
        replayed.  A replay reuses the captured epochs 1..2n, so every rank
        clears its flag array and passes a host barrier first (one per
        segment, not per step)."""
        key = (psi_local.data_ptr(), int(n_steps))
        if getattr(self, "_graph_key", None) != key:
            g = torch.cuda.CUDAGraph()
            self._epoch = 0
            with torch.cuda.graph(g):
                self._fused_ops(psi_local, n_steps)
            self._graph, self._graph_key = g, key
        _lib.call("ctap_flag_barrier", None, ctypes.c_void_p(self.flags.ptr), self.layout.P, self.layout.rank, 0,
                  _device.stream_handle())
        torch.cuda.current_stream().synchronize()
        dist.barrier(group=self.group)
        self._graph.replay()

    def _advance_chunked(self, psi_local: torch.Tensor, n_steps: int):
        """segment_schedule_chunked on two streams: passes on the current
        stream, all-to-alls on the plan's comm stream, event-ordered per chunk."""
        K = self.chunks
        W = self.grid.n[2] // K
        csz = self.layout.points // K
        psi = psi_local.reshape(-1)
        bufs = {"send": self.send, "recv": self.recv}
        main = torch.cuda.current_stream()
        comm = self._comm
        ready = {}  # (buffer, chunk) -> event after which that chunk's data is complete
        for op in segment_schedule_chunked(n_steps, K):
            if op[0] == "pass":
                self.native.run_pass(op[1], psi, psi)
            elif op[0] == "cpass":
                _, kind, src, dst, c = op
                if (src, c) in ready:
                    main.wait_event(ready.pop((src, c)))
                s_ = psi if src == "psi" else bufs[src][c * csz:(c + 1) * csz]
                d_ = psi if dst == "psi" else bufs[dst][c * csz:(c + 1) * csz]
                self.native.run_pass_zchunk(kind, s_, d_, c * W, W)
                if dst != "psi":
                    ev = torch.cuda.Event()
                    ev.record(main)
                    ready[(dst, c)] = ev
            else:
                _, src, dst, c = op
                comm.wait_event(ready.pop((src, c)))
                with torch.cuda.stream(comm):
                    all_to_all_c(bufs[dst][c * csz:(c + 1) * csz], bufs[src][c * csz:(c + 1) * csz], self.group)
                    ev = torch.cuda.Event()
                    ev.record(comm)
                ready[(dst, c)] = ev
        main.wait_stream(comm)

    def observe(self, psi_local: torch.Tensor, xb1=None, xb2=None, margin: int = 2) -> list:
        """Global [sum rho, left, middle, right, edge] (raw sums, rank-ordered)."""
        xs = _device.to_device_f64(self.grid.x[self.layout.x_slice])
        b1 = None if xb1 is None else _device.to_device_f64(np.asarray(xb1))
        b2 = None if xb2 is None else _device.to_device_f64(np.asarray(xb2))
        local = self.native.observe(psi_local, xs, b1, b2, margin)
        if self.layout.P == 1:
            return local.tolist()
        return combine_in_rank_order(local, self.group).tolist()
