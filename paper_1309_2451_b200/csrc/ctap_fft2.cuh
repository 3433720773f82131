// Two-stage line FFT for lines of L = 64 ... 1024 points (complex128).
//
// A line is owned by T = L/32 threads holding E = 32 points each (thread t
// holds points t + m*T, m = 0..31).  The transform is ONE Stockham step pair:
//
//   stage 1: a radix-32 DFT in registers over the thread's 32 points (no
//            twiddles), outputs scattered once through shared memory;
//   stage 2: 32/R2 radix-R2 DFTs per thread (R2 = L/32) on the gathered points
//            after the twiddles exp(DIR 2 pi i r k / L), outputs left in
//            registers in natural order X[t + m*T].
//
// So a transform costs ONE shared-memory exchange (a store and a load of every
// point) instead of the two of the radix-8 plan (ctap_device.cuh, three
// radix-8 stages at L = 512), and  F^-1 . diag . F  along a line costs two.
// On B200 the axis passes of the step are bound by the L1/shared data pipe
// (ncu, r02: l1tex__data_pipe_lsu_wavefronts 88 % of peak in [z^-1 V z], half
// of it shared-memory exchanges), which is what this halves.
//
// The in-register DFTs of 32 and 16 points are Cooley-Tukey composites of the
// radix-8/4/2 kernels of ctap_device.cuh with compile-time twiddles (the
// correctly rounded cos(2 pi m/32)); trivial factors (1, -1, +-i) are free.
#pragma once

#include "ctap_device.cuh"

namespace ctap {

// cos(2 pi m / 32), m = 0..8, correctly rounded
struct W32 {
  static constexpr double c8[9] = {1.0,
                                   0.9807852804032304,
                                   0.9238795325112867,
                                   0.8314696123025452,
                                   0.7071067811865476,
                                   0.5555702330196022,
                                   0.3826834323650898,
                                   0.19509032201612828,
                                   0.0};
  __host__ __device__ static constexpr double cosm(int e) {
    e &= 31;
    return e <= 8 ? c8[e] : e <= 16 ? -c8[16 - e] : e <= 24 ? -c8[e - 16] : c8[32 - e];
  }
  __host__ __device__ static constexpr double sinm(int e) { return cosm(8 - e); }
};

// a * exp(DIR 2 pi i E / N)  (N | 32, E compile-time)
template <int E, int N, int DIR>
__device__ __forceinline__ double2 twc(double2 a) {
  constexpr int e = ((E % N) + N) % N * (32 / N);  // the exponent in units of 2 pi / 32
  if constexpr (e == 0) {
    return a;
  } else if constexpr (e == 16) {
    return make_double2(-a.x, -a.y);
  } else if constexpr (e == 8) {
    return mul_i<DIR>(a);
  } else if constexpr (e == 24) {
    return mul_i<-DIR>(a);
  } else {
    constexpr double c = W32::cosm(e), s = DIR * W32::sinm(e);
    return make_double2(fma(a.x, c, -__dmul_rn(a.y, s)), fma(a.x, s, __dmul_rn(a.y, c)));
  }
}

// In-register DFT of N points with sign DIR, natural order in and out.
template <int N, int DIR>
struct Dft2;
template <int DIR>
struct Dft2<2, DIR> {
  __device__ __forceinline__ static void run(double2* v) { Dft<2, DIR>::run(v); }
};
template <int DIR>
struct Dft2<4, DIR> {
  __device__ __forceinline__ static void run(double2* v) { Dft<4, DIR>::run(v); }
};
template <int DIR>
struct Dft2<8, DIR> {
  __device__ __forceinline__ static void run(double2* v) { Dft<8, DIR>::run(v); }
};

// N = N1 * N2, j = j1 N2 + j2, k = k1 + N1 k2:
//   X[k1 + N1 k2] = sum_j2 w_N2^(j2 k2) w_N^(j2 k1) sum_j1 x[j1 N2 + j2] w_N1^(j1 k1)
template <int N1, int N2, int DIR>
struct DftComposite {
  template <int J2, int K1>
  __device__ __forceinline__ static void tw_row(double2* a) {
    if constexpr (K1 < N1) {
      a[K1] = twc<J2 * K1, N1 * N2, DIR>(a[K1]);
      tw_row<J2, K1 + 1>(a);
    }
  }
  template <int J2>
  __device__ __forceinline__ static void step_a(double2* v) {
    if constexpr (J2 < N2) {
      double2 a[N1];
#pragma unroll
      for (int j1 = 0; j1 < N1; ++j1) a[j1] = v[j1 * N2 + J2];
      Dft2<N1, DIR>::run(a);
      tw_row<J2, 1>(a);
#pragma unroll
      for (int k1 = 0; k1 < N1; ++k1) v[k1 * N2 + J2] = a[k1];
      step_a<J2 + 1>(v);
    }
  }
  __device__ __forceinline__ static void run(double2* v) {
    step_a<0>(v);
    double2 o[N1 * N2];
#pragma unroll
    for (int k1 = 0; k1 < N1; ++k1) {
      double2 b[N2];
#pragma unroll
      for (int j2 = 0; j2 < N2; ++j2) b[j2] = v[k1 * N2 + j2];
      Dft2<N2, DIR>::run(b);
#pragma unroll
      for (int k2 = 0; k2 < N2; ++k2) o[k1 + N1 * k2] = b[k2];
    }
#pragma unroll
    for (int i = 0; i < N1 * N2; ++i) v[i] = o[i];
  }
};
template <int DIR>
struct Dft2<16, DIR> : DftComposite<4, 4, DIR> {};
template <int DIR>
struct Dft2<32, DIR> : DftComposite<8, 4, DIR> {};

template <int L>
struct Plan2 {
  static_assert(L >= 64 && L <= 1024 && (L & (L - 1)) == 0, "two-stage plan: L = 64 ... 1024");
  static constexpr int E = 32;       // points per thread
  static constexpr int T = L / 32;   // threads per line
  static constexpr int R2 = L / 32;  // radix of stage 2
  static constexpr int NB = 32 / R2; // stage-2 butterflies per thread
  static constexpr int tw_size = (R2 - 1) * 32;  // stage-2 table [r-1][k] = exp(-2 pi i r k / L)
  static constexpr int smem_line = L + L / 32;   // padded (one 16-byte pad per 32 points)
};

// exchange position of element i: one pad every 32 elements keeps both the
// stage-1 scatter (thread stride 33) and the stage-2 gather conflict free
__device__ __forceinline__ int pad32(int i) { return i + (i >> 5); }

// One transform of the thread's 32 points v[m] = x[t + m T] (in) ->
// X[t + m T] (out).  `sm` is the line's exchange buffer (Plan2::smem_line
// double2), `tw` the stage-2 table of L, `sync` a barrier over the line's
// threads.
struct NoHook {
  __device__ __forceinline__ void operator()() const {}
};

// `mid` runs between the exchange and stage 2 (the exchange buffer is free
// from there until the next transform)
template <int L, int DIR, typename Sync, typename Mid = NoHook>
__device__ __forceinline__ void line_fft2(double2* v, int t, const double2* __restrict__ tw, double2* sm,
                                          Sync sync, Mid mid = Mid{}) {
  using P = Plan2<L>;
  Dft2<32, DIR>::run(v);
  // stage-1 output r of butterfly t goes to y[t * 32 + r]
#pragma unroll
  for (int r = 0; r < 32; ++r) sm[pad32(t * 32 + r)] = v[r];
  sync();
#pragma unroll
  for (int m = 0; m < 32; ++m) v[m] = sm[pad32(t + m * P::T)];
  sync();
  mid();
  // stage 2: butterfly j = t + b T reads y[j + 32 r] = v[b + NB r]
#pragma unroll
  for (int b = 0; b < P::NB; ++b) {
    const int j = t + b * P::T;
    double2 u[P::R2];
#pragma unroll
    for (int r = 0; r < P::R2; ++r) u[r] = v[b + P::NB * r];
#pragma unroll
    for (int r = 1; r < P::R2; ++r) u[r] = tw_mul<DIR>(u[r], __ldg(&tw[(r - 1) * 32 + j]));
    Dft2<P::R2, DIR>::run(u);
    // X[j + 32 r] = X[t + T (b + NB r)]
#pragma unroll
    for (int r = 0; r < P::R2; ++r) v[b + P::NB * r] = u[r];
  }
}

}  // namespace ctap
