/*
 * ctap.h -- C ABI of libctap.so, the B200 (sm_100a) split-step Fourier
 * propagator for the 3D time-dependent Schrodinger equation on the CTAP
 * atom-chip grid.
 *
 * The reference (arXiv:1309.2451, package `ctapsim`) is pure Python and has
 * no FFI; each entry point below replaces one reference function and is what
 * its Python host layer (paper_1309_2451_b200/, or a ctypes stub inside
 * ctapsim itself) binds.  Reference paths are relative to
 * /root/reference/pkg/src/ctapsim/.
 *
 * Conventions
 *   - Plain pointers and sizes only.  Device pointers are CUDA global memory
 *     owned by the caller; `stream` is a cudaStream_t (NULL = legacy stream).
 *     All work is stream-ordered; nothing synchronises the host unless noted.
 *   - Wavefunctions are complex128 interleaved (re, im), C order (nx, ny, nz)
 *     with z fastest (qgrid.py:3-7).  Potentials are float64 in joules.
 *   - Every call returns a ctap_status; ctap_last_error() gives a thread-local
 *     message for the last failure on the calling thread.
 *   - A plan is not thread safe: one driver thread per plan (propagator.py:136-142).
 *   - Slab decomposition: with slab_p > 1 the plan describes rank slab_r of
 *     slab_p x-slabs (nx/slab_p x-planes each); the caller moves data between
 *     ranks (NCCL all-to-all) between the passes, see ctap_pass().
 */
#ifndef CTAP_H
#define CTAP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CTAP_API __attribute__((visibility("default")))

typedef enum ctap_status {
  CTAP_OK = 0,
  CTAP_EINVAL = 1,       /* invalid argument (reference raises ValueError) */
  CTAP_ECUDA = 2,        /* CUDA runtime error */
  CTAP_EUNSUPPORTED = 3, /* shape outside the compiled kernel set */
  CTAP_ENOMEM = 4
} ctap_status;

typedef enum ctap_dtype {
  CTAP_C128 = 0,  /* complex128 wavefunction (the reference's dtype) */
  CTAP_C64 = 1    /* optional complex64 mode: complex64 storage and transforms,
                     phases still evaluated exactly in FP64 (gate <= 1e-4) */
} ctap_dtype;

typedef enum ctap_mode {
  CTAP_REAL_TIME = 0,      /* propagator.REAL_TIME */
  CTAP_IMAGINARY_TIME = 1  /* propagator.IMAGINARY_TIME */
} ctap_mode;

/* Axis passes. */
typedef enum ctap_pass_kind {
  CTAP_PASS_Z_FWD = 0,
  CTAP_PASS_Z_INV = 1,
  CTAP_PASS_Z_FIRST = 2,  /* psi <- Fz (Vh psi)             segment start */
  CTAP_PASS_Z_MID = 3,    /* psi <- Fz V Fz^-1 psi          between steps */
  CTAP_PASS_Z_LAST = 4,   /* psi <- Vh Fz^-1 psi            segment end   */
  CTAP_PASS_Y_FWD = 5,
  CTAP_PASS_Y_INV = 6,
  CTAP_PASS_Y_FWD_TO_PEER = 7,   /* y FFT, output in peer-major send layout */
  CTAP_PASS_Y_INV_FROM_PEER = 8, /* input in peer-major receive layout, y^-1 */
  CTAP_PASS_X_KIN = 9,    /* psi <- Fx^-1 (K/N) Fx psi on the y-slab layout */
  CTAP_PASS_X_FWD = 10,
  CTAP_PASS_X_INV = 11,
  /* single-GPU step on the blocked k-space layout (out of place y passes):
   * B(x, y, z) = ((x >> lx) ny + y) 2^lx nz + (x & (2^lx - 1)) nz + z */
  CTAP_PASS_Y_FWD_BLK = 12,  /* y FFT, natural psi -> blocked buffer */
  CTAP_PASS_X_KIN_BLK = 13,  /* [x K x^-1] on the blocked buffer, in place */
  CTAP_PASS_Y_INV_BLK = 14,  /* y^-1, blocked buffer -> natural psi */
  /* slab decomposition with the transposes fused into the passes (no NCCL
   * all-to-all): the output goes straight into the other ranks' buffers
   * (peer memory over NVLink) registered with ctap_set_peer_buffers; the
   * caller inserts a stream-ordered cross-rank barrier after each. */
  CTAP_PASS_Y_FWD_TO_PEERS = 15, /* in: psi x-slab; out: every rank's y-slab buffer */
  CTAP_PASS_X_KIN_TO_PEERS = 16, /* in: this rank's y-slab buffer; out: every rank's
                                    peer-major buffer (then CTAP_PASS_Y_INV_FROM_PEER) */
  /* pencil decomposition (ctap_plan_desc.pencil_c > 1; Pr x Pc ranks, rank
   * r = a Pc + b owns x block a (nx/Pr), y block b (ny/Pc), all z).  Buffers:
   *   psi  natural (nx/Pr, ny/Pc, nz)                       position space
   *   Zc   [b'][x][y][z'] (z chunk b' of nz/Pc)            = send of the row all-to-all
   *   Yb   [b'][x][y'][z'] (y block b' of ny/Pc)           = receive of the row all-to-all
   *   Xp   [a'][x][y'][z'] (y block a' of ny/Pr)           = send of the column all-to-all
   *   Xr   [a'][x'][y][z'] = natural (nx, ny/Pr, nz/Pc)    = receive of the column all-to-all
   * One step: PZ_MID (Zc) -> row a2a -> PY_FWD (Yb -> Xp) -> column a2a ->
   * PX_KIN (Xr) -> column a2a -> PY_INV (Xp -> Yb) -> row a2a. */
  CTAP_PASS_PZ_FIRST = 17, /* Fz Vh: psi (natural) -> Zc, out of place */
  CTAP_PASS_PZ_MID = 18,   /* Fz V Fz^-1 on Zc, in place */
  CTAP_PASS_PZ_LAST = 19,  /* Vh Fz^-1: Zc -> psi (natural), out of place */
  CTAP_PASS_PY_FWD = 20,   /* Fy: Yb -> Xp */
  CTAP_PASS_PY_INV = 21,   /* Fy^-1: Xp -> Yb */
  CTAP_PASS_PX_KIN = 22    /* Fx^-1 (K/N) Fx on Xr, in place */
} ctap_pass_kind;

typedef struct ctap_plan ctap_plan;

/* Scalars of make_plan (propagator.py:55-81), computed by the host exactly as
 * the reference computes them:
 *   e0   = UnitSystem.energy  = hbar**2 / (mass * 1e-6**2)      (qgrid.py:41-43)
 *   dt_i = dt / UnitSystem.time, time = mass * 1e-6**2 / hbar   (qgrid.py:37-39)
 *   len2 = UnitSystem.length**2 (1e-12)
 *   v_shift = 0 in real time, potential.min() in imaginary time (propagator.py:75) */
typedef struct ctap_plan_desc {
  int64_t n[3];     /* global nx, ny, nz: powers of two in [8, 1024] */
  double e0;
  double dt_i;
  double len2;
  double v_shift;
  int32_t mode;     /* ctap_mode */
  int32_t slab_p;   /* number of x-slab ranks (1 = single GPU) */
  int32_t slab_r;   /* this rank */
  int32_t phase_tables; /* bit 0: keep exp(-i V dt) as a complex table in HBM
                           (+8 B/pt/step, no sincos in the z pass); bit 1: keep
                           exp(-i k^2 dt/2)/N as a table (+16 B/pt/step).  A
                           clear bit recomputes that factor per point every
                           step.  All variants use the identical phase
                           arithmetic (real time only; ignored otherwise). */
  int32_t dtype;    /* ctap_dtype of every wavefunction buffer passed to the plan */
  int32_t pencil_c; /* 0 or 1: x slabs over slab_p ranks; Pc > 1: the slab_p ranks form a
                       (slab_p / Pc) x Pc pencil grid over (x, y), slab_r = a Pc + b; the
                       potential (and psi) is then the (nx/Pr, ny/Pc, nz) block */
} ctap_plan_desc;

/* make_plan (propagator.py:55-81).  kx2/ky2/kz2 are HOST arrays of the squared
 * angular wavenumbers k_axis(i)**2 in m^-2 (qgrid.py:98-117), full global
 * length.  v_dev is the caller's device potential slab (nx/slab_p, ny, nz),
 * which must stay alive for the plan's lifetime; NULL makes a plan that only
 * serves FFTs and reductions (the potential passes then fail with EINVAL).  The phase factors are never
 * materialised: they are recomputed per point with the reference's exact
 * operation order inside the passes. */
CTAP_API int ctap_plan_create(const ctap_plan_desc* desc, const double* kx2, const double* ky2,
                              const double* kz2, const double* v_dev, ctap_plan** out);
CTAP_API int ctap_plan_destroy(ctap_plan* plan);

/* _advance (propagator.py:98-107): n telescoped Strang steps in place on the
 * device wavefunction (single-GPU plans only; slab plans use ctap_pass).
 * n_steps == 0 leaves psi untouched. */
CTAP_API int ctap_advance(ctap_plan* plan, void* psi_dev, int64_t n_steps, void* stream);

/* The step schedule ctap_advance uses for this plan (no reference
 * counterpart: introspection for benchmarks and tests).  *slab_planes = 0:
 * plane order, 4 launches per step; k > 0: x-slab position blocks of k
 * planes on *streams streams, the passes [y^-1] [z^-1 V z] [y] of each slab
 * run back to back between the x passes (1 + 3 nx/k launches per step). */
CTAP_API int ctap_step_schedule(const ctap_plan* plan, int64_t* slab_planes, int32_t* streams);

/* evolve_real's segment + observer event (propagator.py:160-168): n telescoped
 * steps, then the raw sums of ctap_observe ([sum rho, left, middle, right,
 * edge(margin)] into out_dev[5]) -- computed inside the segment-end pass
 * [z^-1 . Vh] from the registers it writes psi from (warp partials summed in
 * a fixed order; the middle guide as total - left - right), so the event
 * reads no extra byte of psi.  n == 0 (or an
 * imaginary-time plan) runs the standalone ctap_observe.  xs/xb1/xb2 as for
 * ctap_observe (device pointers; xb1 = xb2 = NULL: no partition). */
CTAP_API int ctap_advance_observe(ctap_plan* plan, void* psi_dev, int64_t n_steps, const double* xs,
                                  const double* xb1, const double* xb2, int32_t margin, double* out_dev,
                                  void* stream);

/* One axis pass (the building block of ctap_advance, exposed for the slab
 * decomposition and the plain 3D FFT of kinetic_expectation). z passes are in
 * place (in == out).  Y/X passes may be in place in the natural layout. */
CTAP_API int ctap_pass(ctap_plan* plan, int32_t pass_kind, const void* in_dev, void* out_dev,
                       void* stream);

/* Observer reductions (observables.py:74-110, qgrid.py:150-154) over the local
 * slab in one read of psi.  out_dev[5] (device) receives the raw sums
 *   [ sum |psi|^2, sum_{x<xb1(z)} |psi|^2, sum_middle, sum_{x>=xb2(z)}, sum_edge ]
 * where the edge set is every cell within `margin` cells of a global face.
 * xs_dev: local x axis values (m); xb1_dev/xb2_dev: partition boundaries per z
 * (may be NULL: populations are then reported as 0).  The caller scales by
 * dx*dy*dz exactly like the reference.  Deterministic (fixed-order tree). */
CTAP_API int ctap_observe(ctap_plan* plan, const void* psi_dev, const double* xs_dev,
                          const double* xb1_dev, const double* xb2_dev, int32_t margin,
                          double* out_dev, void* stream);

/* density_xz (observables.py:91-94) raw sums: out_dev[x][z] = sum_y |psi|^2
 * over the local slab (nx/slab_p, nz). */
CTAP_API int ctap_density_xz(ctap_plan* plan, const void* psi_dev, double* out_dev, void* stream);

/* Reductions of energy_expectation (propagator.py:176-195).
 * ctap_k2_sums: on a momentum-space array in the y-slab layout (x, y_local, z)
 *   out_dev[2] = [ sum k^2 |phi|^2 (m^-2), sum |phi|^2 ].
 * ctap_v_sums: on position space, out_dev[2] = [ sum V |psi|^2, sum |psi|^2 ]. */
CTAP_API int ctap_k2_sums(ctap_plan* plan, const void* phi_dev, double* out_dev, void* stream);
CTAP_API int ctap_v_sums(ctap_plan* plan, const void* psi_dev, double* out_dev, void* stream);
/* The same sums against a caller's potential V (device, the plan's block
 * shape): potential_expectation(psi, V) (propagator.py:188-190) on any plan
 * of the grid, e.g. a cached potential-free one, without building a plan
 * around V. */
CTAP_API int ctap_v_sums_with(ctap_plan* plan, const void* psi_dev, const double* v_dev, double* out_dev,
                              void* stream);

/* The slab kinetic block by z chunks (overlapped NCCL transport): kinds
 * CTAP_PASS_Y_FWD_TO_PEER (psi columns [z0, z0+zn) -> send chunk),
 * CTAP_PASS_X_KIN (recv chunk in place) and CTAP_PASS_Y_INV_FROM_PEER (send
 * chunk -> psi columns) with CHUNK-MAJOR transpose buffers: the chunk's
 * buffers are [peer][x_local][y_local][zn] and (nx, y_local, zn), so its
 * all-to-all moves contiguous per-peer blocks while the next chunk computes.
 * Bitwise equal to the unchunked passes.  zn a multiple of 8 dividing nz, z0
 * a multiple of zn; slab plans (slab_p > 1) only. */
CTAP_API int ctap_pass_zchunk(ctap_plan* plan, int32_t kind, const void* in, void* out, int64_t z0, int64_t zn,
                              void* stream);

/* Stream-ordered cross-rank barrier of the fused slab transport: write
 * `epoch` into slot `rank` of every peer's flag array (peer_flags[q]: rank q's
 * nranks x uint32 array as mapped in this process), then make `stream` wait
 * until every peer has written >= epoch into this rank's array (my_flags).
 * Stream memory operations (cuStreamWriteValue32 / cuStreamWaitValue32): no
 * kernel spins, no collective.  The flag arrays must start at 0 and epochs
 * increase by one per barrier; epoch 0 clears this rank's array instead
 * (stream-ordered), e.g. before replaying a captured segment that reuses
 * epochs 1, 2, ... (every rank must have cleared before any rank writes). */
CTAP_API int ctap_flag_barrier(void* const* peer_flags, const void* my_flags, int32_t nranks, int32_t rank,
                               uint32_t epoch, void* stream);

/* Register, for the fused slab passes, the device addresses (as seen by this
 * process: peer-mapped through ctap_ipc_open, or local) of every rank's
 * buffers: which = 0: the y-slab buffers (nx, ny/P, nz) the y pass writes;
 * which = 1: the peer-major buffers [P][nx/P][ny/P][nz] the x pass writes.
 * count must equal slab_p (<= 16).  count 0 (ptrs may be NULL) unregisters
 * both tables' entries of `which`: call it before closing the mappings, so a
 * fused pass fails with CTAP_EINVAL instead of storing through a stale one. */
CTAP_API int ctap_set_peer_buffers(ctap_plan* plan, int32_t which, void* const* ptrs, int32_t count);

/* CUDA IPC helpers for the peer mapping: export a device allocation made by
 * cudaMalloc (64-byte handle), open a peer's handle, close it. */
CTAP_API int ctap_ipc_handle(void* dev_ptr, void* handle64);
CTAP_API int ctap_ipc_open(const void* handle64, void** dev_ptr);
CTAP_API int ctap_ipc_close(void* dev_ptr);
/* cudaMalloc + zero fill (IPC-exportable; the flag arrays of ctap_flag_barrier rely on the zeros) */
CTAP_API int ctap_device_alloc(int64_t bytes, void** dev_ptr);
CTAP_API int ctap_device_free(void* dev_ptr);

/* StepPlan.exp_v_half / exp_v_full / exp_k (propagator.py:45-47, 65-68,
 * 76-78) materialised on the local slab for inspection (which = 0, 1, 2):
 * complex128 cos(phi) + i sin(phi) in real time, exp(phi) + 0i in imaginary
 * time.  The propagation never stores these fields. */
CTAP_API int ctap_phase_field(ctap_plan* plan, int32_t which, void* out_dev, void* stream);

/* Wavefunction.normalize (qgrid.py:159-162): psi /= divisor (IEEE division). */
CTAP_API int ctap_scale(ctap_plan* plan, void* psi_dev, double divisor, void* stream);

/* Single-GPU forward (direction -1) or inverse-unnormalised (+1) 3D FFT in
 * place, as scipy.fft.fftn in kinetic_expectation (propagator.py:181). */
CTAP_API int ctap_fft3d(ctap_plan* plan, void* data_dev, int32_t direction, void* stream);

/* _potential_kernel (magfield.py:107-144): V on the (local) grid, float64,
 * bit-identical to the reference's IEEE sequential evaluation (segments in
 * order, no FMA contraction).  All arrays are device pointers: xs (nx), ys
 * (ny), zs (nz) axis samples; seg_a/seg_b (n_seg x 3, row major) segment
 * end points; seg_cur (n_seg) currents.  V_out has shape (nx, ny, nz). */
CTAP_API int ctap_potential(const double* xs, int64_t nx, const double* ys, int64_t ny,
                            const double* zs, int64_t nz, const double* seg_a, const double* seg_b,
                            const double* seg_cur, int64_t n_seg, double b0x, double b0y, double b0z,
                            double mu_eff, double mass, double omega_z, double z_center,
                            double pref, double* V_out, void* stream);

/* Transverse minima of every z slice of V (the scan of _find_slice_minima,
 * magfield.py:188-208, run by assemble_potential :239-240 for each slice).
 * V_dev: (nx, ny, nz) float64.  count_dev[nz] (int64): number of interior
 * points with V < V[i-1,j], V <= V[i+1,j], V < V[i,j-1], V <= V[i,j+1];
 * best_dev[3 nz] (int64): row-major indices i*ny + j of the (up to) three
 * lowest of them by (V, index), -1 padded.  The parabolic refinement and the
 * x ordering of those points are host work (magfield.slice_minima). */
CTAP_API int ctap_slice_minima(const double* V_dev, int64_t nx, int64_t ny, int64_t nz, int64_t* count_dev,
                               int64_t* best_dev, void* stream);

CTAP_API const char* ctap_last_error(void);
CTAP_API const char* ctap_version(void);

#ifdef __cplusplus
}
#endif

#endif /* CTAP_H */
