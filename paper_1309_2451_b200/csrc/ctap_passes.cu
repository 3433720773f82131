// Axis passes of the split-step propagator: every kernel here reads the
// wavefunction once from HBM, performs a 1D FFT (and, where the step allows,
// its inverse) along one axis with the position- or momentum-space phase
// applied in registers, and writes the result once.
//
// Reference: propagator.py:98-107 (_advance).  One telescoped step is
//     psi <- Vh psi; n x [ psi <- F^-1 K F psi ; psi <- V psi ]   (last V = Vh)
// and the 3D F = Fx Fy Fz is split into axis passes so one step costs four
// sweeps:   [z^-1 . V . z]   y   [x . K . x^-1]   y^-1
// (segment ends use [Vh . z] and [z^-1 . Vh] instead of the middle z pass).
//
// All passes share one tile kernel.  A tile is 8 lines x L points; thread
// (t, col) owns points t + m*T (m < 8) of line col, so the 8 lanes of a
// quarter-warp hold the same point of 8 lines:
//   y/x passes: the 8 lines are 8 consecutive z columns -> every warp access
//               is 4 rows x 128 contiguous bytes;
//   z passes:   the 8 lines are 8 consecutive z-lines (stride L) -> 8 rows x
//               64 contiguous bytes.
// Either way twiddle gathers see at most 4 distinct addresses per warp and the
// exchange buffer [i][8] is bank-conflict free.
//
// Phase factors come either from the per-point exact recipes (on the fly,
// 8 B/pt of v_i = V/E0 per step) or from plan-owned complex tables of the
// same values (16 B/pt for the full V step and for K, no sincos per step);
// both give bit-identical phases.
#include "ctap_device.cuh"
#include "ctap_internal.h"

// resident threads per SM the register allocation is sized for
#ifndef CTAP_OCC
#define CTAP_OCC 1024
#endif

namespace ctap {

template <int L>
struct TileCfg {
  static constexpr int T = L / kElems;
  static constexpr int per_tile = T * 8;
  static constexpr int G = per_tile >= 128 ? 1 : 128 / per_tile;  // tiles per block
  static constexpr int threads = G * per_tile;
  static constexpr int line_stride = L + L / 8;  // padded line of the contiguous (z) layout
  static constexpr size_t smem = (size_t)G * 8 * line_stride * sizeof(double2);
  static constexpr int minb = CTAP_OCC / threads > 0 ? CTAP_OCC / threads : 1;
  // lanes of one warp along the line in the contiguous mapping
  static constexpr int TL = T < 8 ? T : 8;
};

// Element (o, i, col) of tile (o, chunk) lives at
//   lay(o, i) + chunk*8*cs + col*cs
//   natural:  lay = o*so + i*si
//   peer:     lay = o*so + (i >> lb)*sb + (i & (2^lb - 1))*si   (slab transpose buffers)
// cs = 1 for y/x passes (columns are z), cs = L for z passes (columns are lines).
struct Layout {
  uint32_t so, sb, si;
  int lb;
};

template <bool PEER>
__device__ __forceinline__ uint32_t lay(const Layout& l, uint32_t o, uint32_t i) {
  if constexpr (PEER) return o * l.so + (i >> l.lb) * l.sb + (i & ((1u << l.lb) - 1u)) * l.si;
  else return o * l.so + i * l.si;
}

struct TileArgs {
  const double2* in;
  double2* out;
  Layout lin, lout;
  uint32_t n_outer;     // number of outer indices
  uint32_t nchunk;      // 8-column chunks per outer index
  // potential phase (z passes)
  const double* vi;     // v_i = (V - shift)/E0 at the same element offsets as psi
  const double2* expv;  // exp(-i v_i dt_i) table (VTAB)
  // kinetic phase (x pass)
  const double* kx2;    // along the pass axis (length L)
  const double* ky2;    // along the outer axis (global)
  const double* kz2;    // along z
  const double2* expk;  // exp(-i k^2 dt/2)/N table in the x-pass layout (KTAB)
  uint32_t outer_off;   // global index of outer o = 0
  double len2, dt_i;
  double scale;         // folded inverse normalisation (power of two)
  int imag;
};

enum TileKind { T_FWD, T_INV, T_KIN, T_VFIRST, T_VMID, T_VLAST };

// v[m] *= exp(i coef v_i dt) (real time) or exp(coef v_i dt) (imaginary time)
__device__ __forceinline__ void mul_vphase(double2& v, double vi, double coef, const TileArgs& a) {
  const double phi = v_phase_i(vi, coef, a.dt_i);
  if (a.imag) {
    const double f = exp(phi);
    v = make_double2(v.x * f, v.y * f);
  } else {
    double s, c;
    fast_sincos(phi, &s, &c);
    v = cmul(v, make_double2(c, s));
  }
}

// Cache policy (measured on B200, 512^3): the z passes stream through L2
// only (an L1-allocated line would be hit again by the in-place store and
// cost L1 data bandwidth); the strided passes keep the default policy.
template <bool ZL>
__device__ __forceinline__ double2 ld_psi(const double2* p) {
  if constexpr (ZL) return __ldcg(p);
  else return *p;
}
template <bool ZL>
__device__ __forceinline__ void st_psi(double2* p, double2 v) {
  if constexpr (ZL) __stcg(p, v);
  else *p = v;
}

__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
__device__ __forceinline__ void prefetch_l2_bulk(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// Thread -> (line col, position t) of a tile.
//   strided (y/x): col = lane & 7 (8 consecutive z), t = rest  -> 4 rows x 128 B per access
//   contiguous (z): a warp covers TL consecutive t of 32/TL lines -> 4 rows x 128 B per access
template <int L, bool ZL>
struct TileMap {
  int col, t, g;
  __device__ __forceinline__ TileMap(int tid) {
    using C = TileCfg<L>;
    g = tid / C::per_tile;
    const int r = tid - g * C::per_tile;
    if constexpr (!ZL) {
      col = r & 7;
      t = r >> 3;
    } else {
      constexpr int TL = C::TL, CL = 32 / TL;           // lanes along the line / lines per warp
      constexpr int WPL = (C::T / TL);                   // warps along one line group
      const int lane = r & 31, w = r >> 5;
      t = (w % WPL) * TL + (lane % TL);
      col = (w / WPL) * CL + lane / TL;
    }
  }
};

template <int L, int KIND, bool PIN, bool POUT, bool ZL, bool TAB>
__global__ void __launch_bounds__(TileCfg<L>::threads, TileCfg<L>::minb) tile_kernel(TileArgs a,
                                                                               const double2* __restrict__ tw) {
  using C = TileCfg<L>;
  constexpr uint32_t cs = ZL ? L : 1;
  extern __shared__ double2 smem[];
  const TileMap<L, ZL> mp(threadIdx.x);
  const int t = mp.t;
  const uint32_t ntiles = a.n_outer * a.nchunk;
  const uint32_t ngroups = (ntiles + C::G - 1) / C::G;

  // persistent loop over tile groups; the next group is prefetched into L2
  // while this one is in flight
  for (uint32_t grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
    const uint32_t nxt = grp + gridDim.x;
    if (nxt < ngroups) {
      const uint32_t ntile = nxt * C::G + mp.g;
      if (ntile < ntiles) {
        const uint32_t no = ntile / a.nchunk;
        const uint32_t nco = (ntile - no * a.nchunk) * 8 * cs;
        if constexpr (ZL) {
          if ((threadIdx.x % C::per_tile) == 0) {
            prefetch_l2_bulk(a.in + lay<false>(a.lin, no, 0) + nco, 8u * L * sizeof(double2));
            if (KIND == T_VFIRST || KIND == T_VLAST || (KIND == T_VMID && !TAB))
              prefetch_l2_bulk(a.vi + lay<false>(a.lin, no, 0) + nco, 8u * L * sizeof(double));
            if (KIND == T_VMID && TAB)
              prefetch_l2_bulk(a.expv + lay<false>(a.lin, no, 0) + nco, 8u * L * sizeof(double2));
          }
        } else {
          const int row = threadIdx.x % C::per_tile;  // per_tile >= L rows of 128 B
          if (row < L) {
            prefetch_l2(a.in + lay<PIN>(a.lin, no, row) + nco);
            if (KIND == T_KIN && TAB) prefetch_l2(a.expk + lay<false>(a.lout, no, row) + nco);
          }
        }
      }
    }
    const uint32_t tile = grp * C::G + mp.g;
    const bool active = tile < ntiles;
    const uint32_t o = active ? tile / a.nchunk : 0;
    const uint32_t cofs = ((active ? (tile - o * a.nchunk) : 0) * 8 + mp.col) * cs;

    double2 v[kElems];
#pragma unroll
    for (int m = 0; m < kElems; ++m)
      v[m] = active ? ld_psi<ZL>(&a.in[lay<PIN>(a.lin, o, t + m * C::T) + cofs]) : make_double2(0.0, 0.0);

    auto body = [&](auto sm) {
      if constexpr (KIND == T_FWD) {
        line_fft<L, -1>(v, t, tw, sm, SyncBlock{});
      } else if constexpr (KIND == T_INV) {
        line_fft<L, +1>(v, t, tw, sm, SyncBlock{});
      } else if constexpr (KIND == T_VFIRST) {  // Vh, then forward
        if (active) {
#pragma unroll
          for (int m = 0; m < kElems; ++m)
            mul_vphase(v[m], __ldcg(&a.vi[lay<false>(a.lin, o, t + m * C::T) + cofs]), -0.5, a);
        }
        line_fft<L, -1>(v, t, tw, sm, SyncBlock{});
      } else if constexpr (KIND == T_VMID || KIND == T_VLAST) {  // inverse, V (or Vh) [, forward]
        line_fft<L, +1>(v, t, tw, sm, SyncBlock{});
        if (active) {
#pragma unroll
          for (int m = 0; m < kElems; ++m) {
            const uint32_t e = lay<false>(a.lin, o, t + m * C::T) + cofs;
            if (KIND == T_VMID && TAB) v[m] = cmul(v[m], __ldcg(&a.expv[e]));
            else mul_vphase(v[m], __ldcg(&a.vi[e]), KIND == T_VMID ? -1.0 : -0.5, a);
          }
        }
        if constexpr (KIND == T_VMID) line_fft<L, -1>(v, t, tw, sm, SyncBlock{});
      } else if constexpr (KIND == T_KIN) {  // forward, K/N, inverse
        line_fft<L, -1>(v, t, tw, sm, SyncBlock{});
        if (active) {
          if constexpr (TAB) {
#pragma unroll
            for (int m = 0; m < kElems; ++m)
              v[m] = cmul(v[m], __ldcg(&a.expk[lay<false>(a.lout, o, t + m * C::T) + cofs]));
          } else {
            const double ky2 = __ldg(&a.ky2[a.outer_off + o]);
            const double kz2 = __ldg(&a.kz2[cofs]);
#pragma unroll
            for (int m = 0; m < kElems; ++m) {
              const double phi = k_phase(__ldg(&a.kx2[t + m * C::T]), ky2, kz2, a.len2, a.dt_i);
              if (a.imag) {
                const double f = exp(phi) * a.scale;
                v[m] = make_double2(v[m].x * f, v[m].y * f);
              } else {
                double s, c;
                fast_sincos(phi, &s, &c);
                v[m] = cmul(v[m], make_double2(c * a.scale, s * a.scale));
              }
            }
          }
        }
        line_fft<L, +1>(v, t, tw, sm, SyncBlock{});
      }
    };
    if constexpr (ZL) body(SmemContig{smem + ((size_t)mp.g * 8 + mp.col) * C::line_stride});
    else body(SmemStrided{smem + (size_t)mp.g * L * 8 + mp.col});

    if (active) {
#pragma unroll
      for (int m = 0; m < kElems; ++m) st_psi<ZL>(&a.out[lay<POUT>(a.lout, o, t + m * C::T) + cofs], v[m]);
    }
    __syncthreads();  // the exchange buffer is reused by the next group
  }
}

// ---------------------------------------------------------------------------
// host-side dispatch
// ---------------------------------------------------------------------------

template <int L, int KIND, bool PIN, bool POUT, bool ZL, bool TAB>
static cudaError_t launch_tile(const TileArgs& a, const double2* tw, cudaStream_t st) {
  using C = TileCfg<L>;
  auto k = tile_kernel<L, KIND, PIN, POUT, ZL, TAB>;
  static cudaError_t init =
      C::smem > 48 * 1024 ? cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::smem)
                          : cudaSuccess;
  if (init != cudaSuccess) return init;
  static int max_blocks = [&] {
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, C::threads, C::smem);
    return sms * (per_sm > 0 ? per_sm : 1);
  }();
  const uint32_t ntiles = a.n_outer * a.nchunk;
  const uint32_t groups = (ntiles + C::G - 1) / C::G;
  const uint32_t blocks = groups < (uint32_t)max_blocks ? groups : (uint32_t)max_blocks;
  k<<<blocks, C::threads, C::smem, st>>>(a, tw);
  return cudaGetLastError();
}

template <int KIND, bool PIN, bool POUT, bool ZL, bool TAB>
static cudaError_t dispatch(int L, const TileArgs& a, const double2* tw, cudaStream_t st) {
  switch (L) {
    case 8: return launch_tile<8, KIND, PIN, POUT, ZL, TAB>(a, tw, st);
    case 16: return launch_tile<16, KIND, PIN, POUT, ZL, TAB>(a, tw, st);
    case 32: return launch_tile<32, KIND, PIN, POUT, ZL, TAB>(a, tw, st);
    case 64: return launch_tile<64, KIND, PIN, POUT, ZL, TAB>(a, tw, st);
    case 128: return launch_tile<128, KIND, PIN, POUT, ZL, TAB>(a, tw, st);
    case 256: return launch_tile<256, KIND, PIN, POUT, ZL, TAB>(a, tw, st);
    case 512: return launch_tile<512, KIND, PIN, POUT, ZL, TAB>(a, tw, st);
    case 1024: return launch_tile<1024, KIND, PIN, POUT, ZL, TAB>(a, tw, st);
  }
  return cudaErrorInvalidValue;
}

static int ilog2(int64_t v) {
  int l = 0;
  while ((int64_t(1) << l) < v) ++l;
  return l;
}

// materialised phase factors (StepPlan.exp_v_half / exp_v_full / exp_k,
// propagator.py:45-47) for inspection, and the plan's phase tables
__global__ void phase_field_kernel(double2* __restrict__ out, const double* __restrict__ vi,
                                   const double* __restrict__ kx2, const double* __restrict__ ky2,
                                   const double* __restrict__ kz2, uint32_t nx, uint32_t ny, uint32_t nz,
                                   uint32_t x_off, uint32_t y_off, int which, int imag, double dt_i,
                                   double len2, double scale) {
  const uint32_t n = nx * ny * nz;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double phi;
    if (which == 2) {
      const uint32_t x = i / (ny * nz), y = (i / nz) % ny, z = i % nz;
      phi = k_phase(kx2[x + x_off], ky2[y + y_off], kz2[z], len2, dt_i);
    } else {
      phi = v_phase_i(vi[i], which == 0 ? -0.5 : -1.0, dt_i);
    }
    if (imag) {
      out[i] = make_double2(exp(phi) * scale, 0.0);
    } else {
      double s, c;
      fast_sincos(phi, &s, &c);
      out[i] = make_double2(c * scale, s * scale);
    }
  }
}

__global__ void v_internal_kernel(const double* __restrict__ V, double* __restrict__ vi, uint32_t n,
                                  double shift, double e0) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    vi[i] = v_internal(V[i], shift, e0);
}

}  // namespace ctap

using namespace ctap;

cudaError_t ctap_run_v_internal(const ctap_plan* p, cudaStream_t st) {
  const uint32_t n = (uint32_t)(p->nx_local * p->n[1] * p->n[2]);
  v_internal_kernel<<<p->red_blocks, 256, 0, st>>>(p->v_dev, p->vi_dev, n, p->v_shift, p->e0);
  return cudaGetLastError();
}

// which: 0 exp_v_half, 1 exp_v_full, 2 exp_k (natural x-slab layout),
//        3 exp_k / N in the x-pass (y-slab) layout, for the tables
cudaError_t ctap_run_phase_field(const ctap_plan* p, int which, void* out, cudaStream_t st) {
  const int imag = p->mode == 1;
  if (which == 3) {
    const uint32_t nyl = (uint32_t)(p->n[1] / p->slab_p);
    phase_field_kernel<<<p->red_blocks, 256, 0, st>>>(
        (double2*)out, p->vi_dev, p->k2_dev[0], p->k2_dev[1], p->k2_dev[2], (uint32_t)p->n[0], nyl,
        (uint32_t)p->n[2], 0u, (uint32_t)p->slab_r * nyl, 2, imag, p->dt_i, p->len2, p->inv_scale);
  } else {
    phase_field_kernel<<<p->red_blocks, 256, 0, st>>>(
        (double2*)out, p->vi_dev, p->k2_dev[0], p->k2_dev[1], p->k2_dev[2], (uint32_t)p->nx_local,
        (uint32_t)p->n[1], (uint32_t)p->n[2], (uint32_t)(p->slab_r * p->nx_local), 0u, which, imag, p->dt_i,
        p->len2, 1.0);
  }
  return cudaGetLastError();
}

// Run one pass on the plan's local data.  `in`/`out` may alias (natural
// layouts, in place).  Returns a CUDA error code.
cudaError_t ctap_run_pass(const ctap_plan* p, int kind, const void* in, void* out, cudaStream_t st) {
  const int64_t nx = p->n[0], ny = p->n[1], nz = p->n[2];
  const int P = p->slab_p;
  const uint32_t nxl = (uint32_t)(nx / P), nyl = (uint32_t)(ny / P);
  TileArgs a;
  a.in = (const double2*)in;
  a.out = (double2*)out;
  a.vi = p->vi_dev;
  a.expv = p->expv_dev;
  a.kx2 = p->k2_dev[0];
  a.ky2 = p->k2_dev[1];
  a.kz2 = p->k2_dev[2];
  a.expk = p->expk_dev;
  a.len2 = p->len2;
  a.dt_i = p->dt_i;
  a.scale = p->inv_scale;
  a.imag = p->mode == 1;
  a.outer_off = 0;

  if (kind >= PASS_Z_FWD && kind <= PASS_Z_LAST) {
    if (in != out) return cudaErrorInvalidValue;
    // z-lines in groups of 8: element (o, i, col) at (8 o + col) L + i
    const Layout zl{8u * (uint32_t)nz, 0u, 1u, 0};
    a.lin = zl;
    a.lout = zl;
    a.n_outer = (uint32_t)(p->nx_local * ny / 8);
    a.nchunk = 1;
    const double2* tw = p->twiddles + (nz - 8);
    const int L = (int)nz;
    const bool vtab = p->expv_dev != nullptr;
    switch (kind) {
      case PASS_Z_FWD: return dispatch<T_FWD, false, false, true, false>(L, a, tw, st);
      case PASS_Z_INV: return dispatch<T_INV, false, false, true, false>(L, a, tw, st);
      case PASS_Z_FIRST: return dispatch<T_VFIRST, false, false, true, false>(L, a, tw, st);
      case PASS_Z_MID:
        return vtab ? dispatch<T_VMID, false, false, true, true>(L, a, tw, st)
                    : dispatch<T_VMID, false, false, true, false>(L, a, tw, st);
      case PASS_Z_LAST: return dispatch<T_VLAST, false, false, true, false>(L, a, tw, st);
    }
    return cudaErrorInvalidValue;
  }
  a.nchunk = (uint32_t)(nz / 8);
  // natural x-slab layout (x_local, y, z), lines along y
  const Layout y_nat{(uint32_t)(ny * nz), 0u, (uint32_t)nz, 0};
  // peer-major layout [peer][x_local][y_local][z] for the y <-> x transposes
  const Layout y_peer{nyl * (uint32_t)nz, nxl * nyl * (uint32_t)nz, (uint32_t)nz, ilog2(nyl)};
  const bool peer = P > 1;
  switch (kind) {
    case PASS_Y_FWD:
    case PASS_Y_INV:
    case PASS_Y_FWD_TO_PEER:
    case PASS_Y_INV_FROM_PEER: {
      a.n_outer = nxl;
      const double2* tw = p->twiddles + (ny - 8);
      const int L = (int)ny;
      if (kind == PASS_Y_FWD_TO_PEER && peer) {
        a.lin = y_nat;
        a.lout = y_peer;
        return dispatch<T_FWD, false, true, false, false>(L, a, tw, st);
      }
      if (kind == PASS_Y_INV_FROM_PEER && peer) {
        a.lin = y_peer;
        a.lout = y_nat;
        return dispatch<T_INV, true, false, false, false>(L, a, tw, st);
      }
      a.lin = y_nat;
      a.lout = y_nat;
      const bool fwd = (kind == PASS_Y_FWD || kind == PASS_Y_FWD_TO_PEER);
      return fwd ? dispatch<T_FWD, false, false, false, false>(L, a, tw, st)
                 : dispatch<T_INV, false, false, false, false>(L, a, tw, st);
    }
    case PASS_X_KIN:
    case PASS_X_FWD:
    case PASS_X_INV: {
      // y-slab layout (x, y_local, z): lines along x, outer index = local y
      const Layout x_nat{(uint32_t)nz, 0u, nyl * (uint32_t)nz, 0};
      a.lin = x_nat;
      a.lout = x_nat;
      a.n_outer = nyl;
      a.outer_off = (uint32_t)p->slab_r * nyl;
      const double2* tw = p->twiddles + (nx - 8);
      const int L = (int)nx;
      if (kind == PASS_X_KIN)
        return p->expk_dev ? dispatch<T_KIN, false, false, false, true>(L, a, tw, st)
                           : dispatch<T_KIN, false, false, false, false>(L, a, tw, st);
      if (kind == PASS_X_FWD) return dispatch<T_FWD, false, false, false, false>(L, a, tw, st);
      return dispatch<T_INV, false, false, false, false>(L, a, tw, st);
    }
  }
  return cudaErrorInvalidValue;
}
