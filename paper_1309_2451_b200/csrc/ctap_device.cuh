// Device-side building blocks of the split-step propagator (sm_100a).
//
// Complex128 values are `double2` (re, im), the interleaved layout numpy uses
// for complex128 (reference qgrid.py:3-7: C order (nx, ny, nz), z fastest).
//
// The per-line FFT is a register/shared-memory Stockham autosort transform:
// a line of L = 2^m points is owned by T = L/8 threads, thread t holding the
// eight points t + m*T.  Every radix stage reads those eight points, applies
// its twiddles and butterflies in registers, and scatters its outputs through
// shared memory to the natural position of the next stage; the last stage
// leaves thread t holding the natural-order outputs t + m*T in registers, so
// a pointwise multiply can be applied in registers and an inverse transform
// can start right away without another exchange (this is what lets one
// kernel apply  F^-1 . diag(phase) . F  along an axis in a single HBM sweep).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace ctap {

constexpr int kElems = 8;  // points per thread per line

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// a * conj(b)
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {
  return make_double2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
// multiply by -i (DIR=-1, forward) or +i (DIR=+1, inverse)
template <int DIR>
__device__ __forceinline__ double2 mul_i(double2 a) {
  return DIR < 0 ? make_double2(a.y, -a.x) : make_double2(-a.y, a.x);
}

// In-register DFT of size R with sign DIR (-1 forward, +1 inverse),
// natural order in and out: v[k] <- sum_j v[j] exp(DIR 2 pi i j k / R).
template <int R, int DIR>
struct Dft;

template <int DIR>
struct Dft<2, DIR> {
  __device__ __forceinline__ static void run(double2* v) {
    double2 a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
  }
};

template <int DIR>
struct Dft<4, DIR> {
  __device__ __forceinline__ static void run(double2* v) {
    double2 t0 = cadd(v[0], v[2]);
    double2 t1 = csub(v[0], v[2]);
    double2 t2 = cadd(v[1], v[3]);
    double2 t3 = mul_i<DIR>(csub(v[1], v[3]));
    v[0] = cadd(t0, t2);
    v[2] = csub(t0, t2);
    v[1] = cadd(t1, t3);
    v[3] = csub(t1, t3);
  }
};

template <int DIR>
struct Dft<8, DIR> {
  __device__ __forceinline__ static void run(double2* v) {
    constexpr double h = 0.70710678118654752440;  // sqrt(2)/2
    double2 e[4] = {v[0], v[2], v[4], v[6]};
    double2 o[4] = {v[1], v[3], v[5], v[7]};
    Dft<4, DIR>::run(e);
    Dft<4, DIR>::run(o);
    // o[k] *= exp(DIR i pi k / 4)
    double2 o1, o3;
    if (DIR < 0) {
      o1 = make_double2(h * (o[1].x + o[1].y), h * (o[1].y - o[1].x));
      o3 = make_double2(h * (o[3].y - o[3].x), -h * (o[3].x + o[3].y));
    } else {
      o1 = make_double2(h * (o[1].x - o[1].y), h * (o[1].x + o[1].y));
      o3 = make_double2(-h * (o[3].x + o[3].y), h * (o[3].x - o[3].y));
    }
    double2 o2 = mul_i<DIR>(o[2]);
    v[0] = cadd(e[0], o[0]);
    v[4] = csub(e[0], o[0]);
    v[1] = cadd(e[1], o1);
    v[5] = csub(e[1], o1);
    v[2] = cadd(e[2], o2);
    v[6] = csub(e[2], o2);
    v[3] = cadd(e[3], o3);
    v[7] = csub(e[3], o3);
  }
};

// Compile-time radix plan for a line of length L (8 <= L <= 1024): stages of
// radix 8 followed by at most one radix-2 or radix-4 stage.
template <int L>
struct Plan {
  static constexpr int T = L / kElems;  // threads per line
  static constexpr int log2L = (L >= 1024) ? 10 : (L >= 512) ? 9 : (L >= 256) ? 8 : (L >= 128) ? 7
                               : (L >= 64) ? 6 : (L >= 32) ? 5 : (L >= 16) ? 4 : 3;
  static constexpr int n8 = log2L / 3;
  static constexpr int rem = log2L % 3;          // 0, 1 or 2 -> trailing radix 1, 2, 4
  static constexpr int nstages = n8 + (rem ? 1 : 0);
  __host__ __device__ static constexpr int radix(int s) { return s < n8 ? 8 : (rem == 1 ? 2 : 4); }
  // Ns before stage s = product of the previous radices
  __host__ __device__ static constexpr int ns(int s) {
    int p = 1;
    for (int i = 0; i < s; ++i) p *= radix(i);
    return p;
  }
};

// Contiguous-line shared-memory position with one 16-byte pad every 8 points
// (keeps stride-8 scatters conflict free for 128-bit accesses).
__device__ __forceinline__ int pad8(int i) { return i + (i >> 3); }

// Accessor abstractions for the exchange buffer: element i of the thread's
// line, where `base` already selects the line (contiguous) or column (strided).
struct SmemContig {
  double2* base;
  __device__ __forceinline__ double2& at(int i) const { return base[pad8(i)]; }
};
struct SmemStrided {  // column-fastest tile: element i of column c at i*8 + c
  double2* base;      // points at column c
  __device__ __forceinline__ double2& at(int i) const { return base[i * 8]; }
};

// One Stockham stage on the eight registers of thread t.
//   radix R, stride Ns (product of earlier radices), line length L.
// Input: v[m] = x[t + m*T].  Output scattered to smem (unless last stage, in
// which case v[m] = X[t + m*T] stays in registers).
template <int L, int R, int NS, int DIR, bool LAST, typename Smem>
__device__ __forceinline__ void stockham_stage(double2* v, int t, const double2* __restrict__ tw, Smem sm) {
  constexpr int T = L / kElems;
  constexpr int NB = kElems / R;  // butterflies per thread
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    double2 u[R];
#pragma unroll
    for (int r = 0; r < R; ++r) u[r] = v[b + r * NB];
    const int j = t + b * T;
    const int k = j & (NS - 1);
    if (NS > 1) {
      // twiddle exp(DIR 2 pi i r k / (NS R)) = W_L^(r k L/(NS R))
      constexpr int step = L / (NS * R);
#pragma unroll
      for (int r = 1; r < R; ++r) {
        double2 w = __ldg(&tw[r * k * step]);
        u[r] = DIR < 0 ? cmul(u[r], w) : cmulc(u[r], w);
      }
    }
    Dft<R, DIR>::run(u);
    if (LAST) {
#pragma unroll
      for (int r = 0; r < R; ++r) v[b + r * NB] = u[r];
    } else {
      const int base = (j / NS) * NS * R + k;
#pragma unroll
      for (int r = 0; r < R; ++r) sm.at(base + r * NS) = u[r];
    }
  }
}

template <int L, int S, int DIR, typename Smem>
__device__ __forceinline__ void fft_stages(double2* v, int t, const double2* __restrict__ tw, Smem sm,
                                           void (*sync)()) {
  using P = Plan<L>;
  constexpr int T = P::T;
  if constexpr (S < P::nstages) {
    constexpr int R = P::radix(S);
    constexpr int NS = P::ns(S);
    constexpr bool LAST = (S == P::nstages - 1);
    stockham_stage<L, R, NS, DIR, LAST>(v, t, tw, sm);
    if constexpr (!LAST) {
      sync();
#pragma unroll
      for (int m = 0; m < kElems; ++m) v[m] = sm.at(t + m * T);
      sync();
      fft_stages<L, S + 1, DIR>(v, t, tw, sm, sync);
    }
  }
}

__device__ __forceinline__ void block_sync() { __syncthreads(); }

// Full in-register/shared 1D FFT of the thread's line.  On entry v[m] holds
// x[t + m*T], on exit X[t + m*T] (unnormalized, sign DIR).
template <int L, int DIR, typename Smem>
__device__ __forceinline__ void line_fft(double2* v, int t, const double2* __restrict__ tw, Smem sm) {
  fft_stages<L, 0, DIR>(v, t, tw, sm, block_sync);
}

// --- exact phase recipes (reference propagator.py:61-68, qgrid.py:98-117) ---
// These products must not be contracted into FMAs: a systematic one-ulp phase
// error fails the 1e-10 parity gate.

// potential phase: (coef * (V - shift)/E0) * dt_i with coef -0.5 (half) or -1.0 (full)
__device__ __forceinline__ double v_phase(double v, double shift, double e0, double coef, double dt_i) {
  double vi = __ddiv_rn(__dsub_rn(v, shift), e0);
  return __dmul_rn(__dmul_rn(coef, vi), dt_i);
}
__device__ __forceinline__ double v_phase_real(double v, double e0, double coef, double dt_i) {
  double vi = __ddiv_rn(v, e0);
  return __dmul_rn(__dmul_rn(coef, vi), dt_i);
}
// kinetic phase: (-0.5 * (((kx2 + ky2) + kz2) * L0^2)) * dt_i
__device__ __forceinline__ double k_phase(double kx2, double ky2, double kz2, double len2, double dt_i) {
  double k2 = __dadd_rn(__dadd_rn(kx2, ky2), kz2);
  return __dmul_rn(__dmul_rn(-0.5, __dmul_rn(k2, len2)), dt_i);
}

}  // namespace ctap
