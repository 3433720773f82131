// Shared pieces of the axis-pass kernels: pass kinds, phase arguments and
// the exact phase multiplies, strided-tile layouts and the tile transform
// body (used by tile_kernel in ctap_passes.cu and tma_tile_kernel in
// ctap_tma.cu).
#pragma once

#include "ctap_device.cuh"

namespace ctap {

enum TileKind { T_FWD, T_INV, T_KIN, T_VFIRST, T_VMID, T_VLAST, T_COPY };

struct PhaseArgs {
  const double* vi;     // v_i = (V - shift)/E0 at the element offsets of psi (z passes)
  const void* expv;     // exp(-i v_i dt_i) table, complex of the plan's precision (VTAB)
  const double* kx2;    // k^2 along the pass axis (x pass)
  const double* ky2;    // k^2 along the outer axis, global
  const double* kz2;    // k^2 along z
  const void* expk;     // exp(-i k^2 dt/2)/N table in the x-pass layout (KTAB)
  uint32_t outer_off;   // global index of outer o = 0
  double len2, dt_i;
  double scale;         // folded inverse normalisation 1/N (power of two)
  int imag;             // imaginary time: real decay factors
  // k^2 regenerated in registers instead of loaded (kgen != 0): the plan
  // verified that (2 pi * (m * kval[a]))^2 reproduces every table entry
  const double2* sct;   // (cos, sin)(k pi/128) for fast_sincos
  const double2* sctk;  // the same times 1/N (the kinetic step's normalisation)
  int kgen;
  uint32_t z_off;  // global z of the pass's column 0 (z-chunked passes)
  uint32_t kn[3];
  double kval[3];
};

// arguments of the z passes (contiguous lines)
struct ZArgs {
  void* psi;
  uint32_t nlines;  // nx_local * ny
  PhaseArgs ph;
  // pencil z-chunked side (CH bit 0: input, bit 1: output): point z of line l
  // at (z >> lzc) cs + l 2^lzc + (z & (2^lzc - 1)), cs = nlines 2^lzc
  void* out;
  uint32_t lzc, cs;
  // fused observer sums of the segment-end pass [z^-1 . Vh] (single GPU):
  // per block [sum rho, left, middle, right, edge] into obs_partial[5 block]
  const double* xs;    // x axis (m)
  const double* xb1;   // guide boundaries per z (null: no partition)
  const double* xb2;
  double* obs_partial;
  // per (x, thread t of a line): bit m = xs[x] < xb1[t + m T], bit 8 + m =
  // xs[x] >= xb2[t + m T] (obs_mask_kernel; one load per thread and line
  // instead of two boundary loads per point)
  const uint16_t* obs_mask;
  uint32_t ny, nx;     // line = x ny + y
  uint32_t lny;        // log2(ny)
  int margin;
};

// squared angular wavenumber of FFT index i on an axis of n points with
// 1/(n d) = val, formed as numpy's 2*pi*fftfreq(n, d) then squared
// (qgrid.py k_axis / k_squared): ((2 pi) * (m * val))^2, m the signed index
__device__ __forceinline__ double k2_gen(uint32_t i, uint32_t n, double val) {
  const int m = i < (n >> 1) ? (int)i : (int)i - (int)n;
  const double k = __dmul_rn(6.283185307179586, __dmul_rn((double)m, val));
  return __dmul_rn(k, k);
}

// v *= (c + i s) and v *= f.  complex128: the butterflies' cmul.  complex64:
// the product is formed in FP64 and rounded once, so the factor itself is
// never rounded to float -- a rounded factor is the same at a grid point every
// step and its ~6e-8 modulus/argument error would grow linearly with the step
// count (1.3e-4 after 1000 steps at 256^3), whereas the rounding of the
// product changes from step to step and only random-walks.
__device__ __forceinline__ void rotate(double2& v, double c, double s) { v = cmul(v, make_double2(c, s)); }
__device__ __forceinline__ void rotate(float2& v, double c, double s) {
  const double x = v.x, y = v.y;
  v = make_float2((float)fma(x, c, -__dmul_rn(y, s)), (float)fma(x, s, __dmul_rn(y, c)));
}
__device__ __forceinline__ void dscale(double2& v, double f) { v = make_double2(v.x * f, v.y * f); }
__device__ __forceinline__ void dscale(float2& v, double f) {
  v = make_float2((float)__dmul_rn(v.x, f), (float)__dmul_rn(v.y, f));
}

// v *= exp(i coef v_i dt) (real time) or exp(coef v_i dt) (imaginary time)
// (the phase and its cos/sin are always evaluated in FP64)
template <typename CV>
__device__ __forceinline__ void mul_vphase(CV& v, double vi, double coef, const PhaseArgs& a) {
  const double phi = v_phase_i(vi, coef, a.dt_i);
  if (a.imag) {
    dscale(v, exp(phi));
  } else {
    double s, c;
    fast_sincos(phi, a.sct, &s, &c);
    rotate(v, c, s);
  }
}

// v *= exp(-i k^2 dt/2) / N at (kx2, ky2, kz2)
template <typename CV>
__device__ __forceinline__ void mul_kphase(CV& v, double kx2, double ky2, double kz2, const PhaseArgs& a) {
  const double phi = k_phase(kx2, ky2, kz2, a.len2, a.dt_i);
  if (a.imag) {
    dscale(v, exp(phi) * a.scale);
  } else {
    double s, c;
    fast_sincos(phi, a.sctk, &s, &c);  // 1/N folded into the table
    rotate(v, c, s);
  }
}

// Element (o, i, z) of a strided tile lives at outer(o) + inner(i) + z:
//   outer(o) = (o >> olb)*osb + (o & (2^olb - 1))*so      (olb = 31: o*so)
//   inner(i) = i*si                                       (plain)
//            = (i >> lb)*sb + (i & (2^lb - 1))*si          (blocked: the slab
//              transpose buffers and the blocked k-space layout)
struct Layout {
  uint32_t so, sb, si;
  int lb;
  uint32_t osb;
  int olb;
};

__device__ __forceinline__ uint32_t outer(const Layout& l, uint32_t o) {
  return (o >> l.olb) * l.osb + (o & ((1u << l.olb) - 1u)) * l.so;
}
template <bool BLK>
__device__ __forceinline__ uint32_t inner(const Layout& l, uint32_t i) {
  if constexpr (BLK) return (i >> l.lb) * l.sb + (i & ((1u << l.lb) - 1u)) * l.si;
  else return i * l.si;
}

constexpr int kMaxRanks = 16;

struct TileArgs {
  const void* in;
  void* out;
  Layout lin, lout;
  uint32_t n_outer;  // number of outer indices
  uint32_t nchunk;   // 8-column chunks per outer index (nz / 8)
  PhaseArgs ph;
  // fused slab transpose: destination of inner block b (= rank b) is peers[b]
  // (a peer GPU's buffer, mapped over NVLink, base offset included)
  void* peers[kMaxRanks];
};

template <int L, int E, int KIND, bool KTAB, bool KBLK, typename CV, int W, typename Sync = SyncBlock>
__device__ __forceinline__ void tile_body(const TileArgs& a, CV* v, int t, uint32_t o, uint32_t z,
                                          bool active, const TwOf<CV>* __restrict__ tw, SmemStrided<CV, W> sm,
                                          Sync sync = Sync{}) {
  constexpr int T = L / E;
  if constexpr (KIND == T_COPY) {  // diagnostics: the pass's memory traffic without the transform
  } else if constexpr (KIND == T_FWD) {
    line_fft<L, -1, E>(v, t, tw, sm, sync);
  } else if constexpr (KIND == T_INV) {
    line_fft<L, +1, E>(v, t, tw, sm, sync);
  } else {  // T_KIN: forward, K/N, inverse
    // per-column operands ahead of the forward transform; the per-point kx^2
    // after it (regenerated, or loaded), so no registers are held across it
    double ky2 = 0.0, kz2 = 0.0;
    CV f[KTAB ? E : 1];
    if constexpr (KTAB) {
      // expk spans the full nz: a z-chunked pass (a.out offset by z_off
      // columns) indexes it at the chunk's absolute column
      const CV* expk = (const CV*)a.ph.expk;
#pragma unroll
      for (int m = 0; m < E; ++m)
        f[m] = active ? __ldcg(&expk[outer(a.lout, o) + inner<KBLK>(a.lout, t + m * T) + a.ph.z_off + z])
                      : CT<CV>::mk(0, 0);
    } else if (a.ph.kgen) {
      ky2 = k2_gen(a.ph.outer_off + o, a.ph.kn[1], a.ph.kval[1]);
      kz2 = k2_gen(a.ph.z_off + z, a.ph.kn[2], a.ph.kval[2]);
    } else {
      ky2 = __ldg(&a.ph.ky2[a.ph.outer_off + o]);
      kz2 = __ldg(&a.ph.kz2[a.ph.z_off + z]);
    }
    line_fft<L, -1, E>(v, t, tw, sm, sync);
    if (active) {
      if constexpr (KTAB) {
#pragma unroll
        for (int m = 0; m < E; ++m) v[m] = cmul(v[m], f[m]);
      } else if (a.ph.kgen) {
#pragma unroll
        for (int m = 0; m < E; ++m)
          mul_kphase(v[m], k2_gen(t + m * T, a.ph.kn[0], a.ph.kval[0]), ky2, kz2, a.ph);
      } else {
#pragma unroll
        for (int m = 0; m < E; ++m) mul_kphase(v[m], __ldg(&a.ph.kx2[t + m * T]), ky2, kz2, a.ph);
      }
    }
    line_fft<L, +1, E>(v, t, tw, sm, sync);
  }
}


}  // namespace ctap
