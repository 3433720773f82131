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
#include <cstdio>

#include "ctap_device.cuh"
#include "ctap_internal.h"

namespace ctap {

// ---------------------------------------------------------------------------
// z passes: lines are contiguous (nz points, stride 1).  A block owns C lines.
// ---------------------------------------------------------------------------

template <int L>
struct ZCfg {
  static constexpr int T = L / kElems;
  static constexpr int C = (256 / T) > 0 ? (256 / T) : 1;  // lines per block
  static constexpr int threads = C * T;
  static constexpr int smem_line = L + L / 8;             // padded doubles2 per line
  static constexpr size_t smem = (size_t)C * smem_line * sizeof(double2);
};

struct ZArgs {
  double2* psi;
  const double* V;      // same layout as psi (local slab)
  int64_t nlines;       // nx_local * ny
  double e0, dt_i, vshift;
  int imag;             // 1: imaginary-time (real decay factors)
};

// multiply v[m] (points t + m*T of a line starting at flat index `off`) by the
// potential factor exp(i coef V dt) (real time) or exp(coef V dt) (imag time)
template <int L>
__device__ __forceinline__ void apply_v(double2* v, const double* __restrict__ V, int64_t off, int t,
                                        const ZArgs& a, double coef) {
  constexpr int T = L / kElems;
#pragma unroll
  for (int m = 0; m < kElems; ++m) {
    double vv = __ldg(&V[off + t + m * T]);
    double phi = v_phase(vv, a.vshift, a.e0, coef, a.dt_i);
    if (a.imag) {
      double f = exp(phi);
      v[m] = make_double2(v[m].x * f, v[m].y * f);
    } else {
      double s, c;
      sincos(phi, &s, &c);
      v[m] = cmul(v[m], make_double2(c, s));
    }
  }
}

template <int L, int KIND>
__global__ void __launch_bounds__(ZCfg<L>::threads) z_pass_kernel(ZArgs a, const double2* __restrict__ tw) {
  using C = ZCfg<L>;
  extern __shared__ double2 smem[];
  const int t = threadIdx.x % C::T;
  const int c = threadIdx.x / C::T;
  const int64_t line = (int64_t)blockIdx.x * C::C + c;
  const bool active = line < a.nlines;
  const int64_t off = line * L;
  SmemContig sm{smem + c * C::smem_line};
  double2 v[kElems];
#pragma unroll
  for (int m = 0; m < kElems; ++m) v[m] = active ? a.psi[off + t + m * C::T] : make_double2(0.0, 0.0);

  if constexpr (KIND == PASS_Z_FWD) {
    line_fft<L, -1>(v, t, tw, sm);
  } else if constexpr (KIND == PASS_Z_INV) {
    line_fft<L, +1>(v, t, tw, sm);
  } else if constexpr (KIND == PASS_Z_FIRST) {  // Vh then forward
    if (active) apply_v<L>(v, a.V, off, t, a, -0.5);
    line_fft<L, -1>(v, t, tw, sm);
  } else if constexpr (KIND == PASS_Z_MID) {  // inverse, V, forward
    line_fft<L, +1>(v, t, tw, sm);
    if (active) apply_v<L>(v, a.V, off, t, a, -1.0);
    __syncthreads();
    line_fft<L, -1>(v, t, tw, sm);
  } else if constexpr (KIND == PASS_Z_LAST) {  // inverse then Vh
    line_fft<L, +1>(v, t, tw, sm);
    if (active) apply_v<L>(v, a.V, off, t, a, -0.5);
  }
  if (active) {
#pragma unroll
    for (int m = 0; m < kElems; ++m) a.psi[off + t + m * C::T] = v[m];
  }
}

// ---------------------------------------------------------------------------
// strided passes (y and x): a tile is one outer index o, the whole line along
// the axis, and 8 consecutive z columns (128-byte coalesced rows).
// Element (o, i, c) of the tile lives at
//     o*so + (i / blk)*sb + (i % blk)*si + z0 + c
// which covers the natural layout (blk = L) and the peer-major layout of the
// slab decomposition (blk = points per rank along the axis).
// ---------------------------------------------------------------------------

template <int L>
struct SCfg {
  static constexpr int T = L / kElems;
  static constexpr int per_tile = T * 8;
  static constexpr int G = per_tile >= 128 ? 1 : 128 / per_tile;  // tiles per block
  static constexpr int threads = G * per_tile;
  static constexpr size_t smem = (size_t)G * L * 8 * sizeof(double2);
};

struct Layout {
  int64_t so, sb, si;
  int blk;
};

struct SArgs {
  const double2* in;
  double2* out;
  Layout lin, lout;
  int64_t n_outer;      // number of outer indices
  int nzc;              // number of 8-column chunks (nz / 8)
  // kinetic phase (x pass): global k^2 tables, offsets of this tile's outer index
  const double* kx2;    // along the pass axis (length L)
  const double* ky2;    // along the outer axis (global)
  const double* kz2;    // along z
  int64_t outer_off;    // global index of outer o = 0
  double len2, dt_i;
  double scale;         // folded inverse normalisation (power of two)
  int imag;
};

__device__ __forceinline__ int64_t lay(const Layout& l, int64_t o, int i) {
  return o * l.so + (int64_t)(i / l.blk) * l.sb + (int64_t)(i % l.blk) * l.si;
}

template <int L, int KIND>
__global__ void __launch_bounds__(SCfg<L>::threads) s_pass_kernel(SArgs a, const double2* __restrict__ tw) {
  using C = SCfg<L>;
  extern __shared__ double2 smem[];
  const int col = threadIdx.x & 7;
  const int t = (threadIdx.x >> 3) % C::T;
  const int g = threadIdx.x / C::per_tile;
  const int64_t tile = (int64_t)blockIdx.x * C::G + g;
  const int64_t ntiles = a.n_outer * a.nzc;
  const bool active = tile < ntiles;
  const int64_t o = active ? tile / a.nzc : 0;
  const int z = (int)(active ? (tile % a.nzc) : 0) * 8 + col;
  SmemStrided sm{smem + (size_t)g * L * 8 + col};

  double2 v[kElems];
#pragma unroll
  for (int m = 0; m < kElems; ++m)
    v[m] = active ? a.in[lay(a.lin, o, t + m * C::T) + z] : make_double2(0.0, 0.0);

  if constexpr (KIND == PASS_S_FWD) {
    line_fft<L, -1>(v, t, tw, sm);
  } else if constexpr (KIND == PASS_S_INV) {
    line_fft<L, +1>(v, t, tw, sm);
  } else if constexpr (KIND == PASS_S_KIN) {
    line_fft<L, -1>(v, t, tw, sm);
    if (active) {
      const double ky2 = __ldg(&a.ky2[a.outer_off + o]);
      const double kz2 = __ldg(&a.kz2[z]);
#pragma unroll
      for (int m = 0; m < kElems; ++m) {
        const double kx2 = __ldg(&a.kx2[t + m * C::T]);
        double phi = k_phase(kx2, ky2, kz2, a.len2, a.dt_i);
        if (a.imag) {
          double f = exp(phi) * a.scale;
          v[m] = make_double2(v[m].x * f, v[m].y * f);
        } else {
          double s, c;
          sincos(phi, &s, &c);
          v[m] = cmul(v[m], make_double2(c * a.scale, s * a.scale));
        }
      }
    }
    __syncthreads();
    line_fft<L, +1>(v, t, tw, sm);
  }
  if (active) {
#pragma unroll
    for (int m = 0; m < kElems; ++m) a.out[lay(a.lout, o, t + m * C::T) + z] = v[m];
  }
}

// ---------------------------------------------------------------------------
// host-side dispatch
// ---------------------------------------------------------------------------

template <int L, int KIND>
static cudaError_t launch_z(const ZArgs& a, const double2* tw, cudaStream_t st) {
  using C = ZCfg<L>;
  auto k = z_pass_kernel<L, KIND>;
  static bool init = false;
  if (!init) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::smem);
    if (e != cudaSuccess) return e;
    init = true;
  }
  int64_t blocks = (a.nlines + C::C - 1) / C::C;
  k<<<(unsigned)blocks, C::threads, C::smem, st>>>(a, tw);
  return cudaGetLastError();
}

template <int L, int KIND>
static cudaError_t launch_s(const SArgs& a, const double2* tw, cudaStream_t st) {
  using C = SCfg<L>;
  auto k = s_pass_kernel<L, KIND>;
  static bool init = false;
  if (!init) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::smem);
    if (e != cudaSuccess) return e;
    init = true;
  }
  int64_t ntiles = a.n_outer * a.nzc;
  int64_t blocks = (ntiles + C::G - 1) / C::G;
  k<<<(unsigned)blocks, C::threads, C::smem, st>>>(a, tw);
  return cudaGetLastError();
}

template <int KIND>
static cudaError_t dispatch_z(int L, const ZArgs& a, const double2* tw, cudaStream_t st) {
  switch (L) {
    case 8: return launch_z<8, KIND>(a, tw, st);
    case 16: return launch_z<16, KIND>(a, tw, st);
    case 32: return launch_z<32, KIND>(a, tw, st);
    case 64: return launch_z<64, KIND>(a, tw, st);
    case 128: return launch_z<128, KIND>(a, tw, st);
    case 256: return launch_z<256, KIND>(a, tw, st);
    case 512: return launch_z<512, KIND>(a, tw, st);
    case 1024: return launch_z<1024, KIND>(a, tw, st);
  }
  return cudaErrorInvalidValue;
}

template <int KIND>
static cudaError_t dispatch_s(int L, const SArgs& a, const double2* tw, cudaStream_t st) {
  switch (L) {
    case 8: return launch_s<8, KIND>(a, tw, st);
    case 16: return launch_s<16, KIND>(a, tw, st);
    case 32: return launch_s<32, KIND>(a, tw, st);
    case 64: return launch_s<64, KIND>(a, tw, st);
    case 128: return launch_s<128, KIND>(a, tw, st);
    case 256: return launch_s<256, KIND>(a, tw, st);
    case 512: return launch_s<512, KIND>(a, tw, st);
    case 1024: return launch_s<1024, KIND>(a, tw, st);
  }
  return cudaErrorInvalidValue;
}

// materialised phase factors (StepPlan.exp_v_half / exp_v_full / exp_k,
// propagator.py:45-47) for inspection; the propagation itself never stores them
__global__ void phase_field_kernel(double2* __restrict__ out, const double* __restrict__ V,
                                   const double* __restrict__ kx2, const double* __restrict__ ky2,
                                   const double* __restrict__ kz2, int64_t nxl, int64_t ny, int64_t nz,
                                   int64_t x_off, int which, int imag, double e0, double dt_i, double vshift,
                                   double len2) {
  const int64_t n = nxl * ny * nz;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    double phi;
    if (which == 2) {
      int64_t x = i / (ny * nz), y = (i / nz) % ny, z = i % nz;
      phi = k_phase(kx2[x + x_off], ky2[y], kz2[z], len2, dt_i);
    } else {
      phi = v_phase(V[i], vshift, e0, which == 0 ? -0.5 : -1.0, dt_i);
    }
    if (imag) {
      out[i] = make_double2(exp(phi), 0.0);
    } else {
      double s, c;
      sincos(phi, &s, &c);
      out[i] = make_double2(c, s);
    }
  }
}

}  // namespace ctap

using namespace ctap;

cudaError_t ctap_run_phase_field(const ctap_plan* p, int which, void* out, cudaStream_t st) {
  phase_field_kernel<<<p->red_blocks, 256, 0, st>>>((double2*)out, p->v_dev, p->k2_dev[0], p->k2_dev[1],
                                                    p->k2_dev[2], p->nx_local, p->n[1], p->n[2],
                                                    (int64_t)p->slab_r * p->nx_local, which, p->mode == 1, p->e0,
                                                    p->dt_i, p->v_shift, p->len2);
  return cudaGetLastError();
}

// Run one pass on the plan's local data.  `in`/`out` may alias (natural
// layouts, in place).  Returns a CUDA error code.
cudaError_t ctap_run_pass(const ctap_plan* p, int kind, const void* in, void* out, cudaStream_t st) {
  const double2* tw_z = p->twiddles + (p->n[2] - 8);
  if (kind >= PASS_Z_FWD && kind <= PASS_Z_LAST) {
    if (in != out) return cudaErrorInvalidValue;
    ZArgs a;
    a.psi = (double2*)out;
    a.V = p->v_dev;
    a.nlines = p->nx_local * p->n[1];
    a.e0 = p->e0;
    a.dt_i = p->dt_i;
    a.vshift = p->v_shift;
    a.imag = p->mode == 1;
    int L = (int)p->n[2];
    switch (kind) {
      case PASS_Z_FWD: return dispatch_z<PASS_Z_FWD>(L, a, tw_z, st);
      case PASS_Z_INV: return dispatch_z<PASS_Z_INV>(L, a, tw_z, st);
      case PASS_Z_FIRST: return dispatch_z<PASS_Z_FIRST>(L, a, tw_z, st);
      case PASS_Z_MID: return dispatch_z<PASS_Z_MID>(L, a, tw_z, st);
      case PASS_Z_LAST: return dispatch_z<PASS_Z_LAST>(L, a, tw_z, st);
    }
    return cudaErrorInvalidValue;
  }
  const int64_t nx = p->n[0], ny = p->n[1], nz = p->n[2];
  const int P = p->slab_p;
  const int64_t nxl = nx / P, nyl = ny / P;
  SArgs a;
  a.in = (const double2*)in;
  a.out = (double2*)out;
  a.nzc = (int)(nz / 8);
  a.kx2 = p->k2_dev[0];
  a.ky2 = p->k2_dev[1];
  a.kz2 = p->k2_dev[2];
  a.len2 = p->len2;
  a.dt_i = p->dt_i;
  a.scale = p->inv_scale;
  a.imag = p->mode == 1;
  a.outer_off = 0;
  // natural x-slab layout (x_local, y, z), lines along y
  Layout y_nat{ny * nz, 0, nz, (int)ny};
  // peer-major layout [peer][x_local][y_local][z] for the y <-> x transposes
  Layout y_peer{nyl * nz, nxl * nyl * nz, nz, (int)nyl};
  switch (kind) {
    case PASS_Y_FWD:
    case PASS_Y_INV:
    case PASS_Y_FWD_TO_PEER:
    case PASS_Y_INV_FROM_PEER: {
      a.n_outer = nxl;
      a.lin = (kind == PASS_Y_INV_FROM_PEER) ? y_peer : y_nat;
      a.lout = (kind == PASS_Y_FWD_TO_PEER) ? y_peer : y_nat;
      if (P == 1) { a.lin = y_nat; a.lout = y_nat; }
      const double2* tw = p->twiddles + (ny - 8);
      bool fwd = (kind == PASS_Y_FWD || kind == PASS_Y_FWD_TO_PEER);
      return fwd ? dispatch_s<PASS_S_FWD>((int)ny, a, tw, st) : dispatch_s<PASS_S_INV>((int)ny, a, tw, st);
    }
    case PASS_X_KIN:
    case PASS_X_FWD:
    case PASS_X_INV: {
      // y-slab layout (x, y_local, z): lines along x, outer index = local y
      Layout x_nat{nz, 0, nyl * nz, (int)nx};
      a.lin = x_nat;
      a.lout = x_nat;
      a.n_outer = nyl;
      a.outer_off = (int64_t)p->slab_r * nyl;
      const double2* tw = p->twiddles + (nx - 8);
      if (kind == PASS_X_KIN) return dispatch_s<PASS_S_KIN>((int)nx, a, tw, st);
      if (kind == PASS_X_FWD) return dispatch_s<PASS_S_FWD>((int)nx, a, tw, st);
      return dispatch_s<PASS_S_INV>((int)nx, a, tw, st);
    }
  }
  return cudaErrorInvalidValue;
}
