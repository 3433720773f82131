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
//
// Index arithmetic is 32-bit throughout: a local slab never exceeds 2^30
// points (axes are <= 1024).
#pragma once

#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

namespace ctap {

constexpr int kElems = 8;  // points per thread per line

// Complex vector types: double2 (complex128, the reference's dtype) and
// float2 (the optional complex64 mode).  CT<C> maps a vector type to its
// scalar and builder.
template <typename C>
struct CT;
// TW is the twiddle-table entry: double2, or for complex64 a float-float
// pair (hi.x, hi.y, lo.x, lo.y) with hi + lo = the double twiddle to ~2^-48,
// so no rounded twiddle (or constant) is applied to the data: a rounded
// factor repeats every step at the same point and its ~3e-8 error would grow
// linearly with the step count (the rounding of products only random-walks).
template <>
struct CT<double2> {
  using R = double;
  using TW = double2;
  __device__ __forceinline__ static double2 mk(double a, double b) { return make_double2(a, b); }
};
template <>
struct CT<float2> {
  using R = float;
  using TW = float4;
  __device__ __forceinline__ static float2 mk(float a, float b) { return make_float2(a, b); }
};
template <typename C>
using TwOf = typename CT<C>::TW;

template <typename C>
__device__ __forceinline__ C cadd(C a, C b) { return CT<C>::mk(a.x + b.x, a.y + b.y); }
template <typename C>
__device__ __forceinline__ C csub(C a, C b) { return CT<C>::mk(a.x - b.x, a.y - b.y); }
// complex products with an explicit FMA pattern, so the rounding does not
// depend on how the compiler contracts the surrounding code (keeps e.g. the
// slab and single-GPU paths bitwise identical)
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -__dmul_rn(a.y, b.y)), fma(a.x, b.y, __dmul_rn(a.y, b.x)));
}
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -__fmul_rn(a.y, b.y)), fmaf(a.x, b.y, __fmul_rn(a.y, b.x)));
}
// a * conj(b)
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, __dmul_rn(a.y, b.y)), fma(a.y, b.x, -__dmul_rn(a.x, b.y)));
}
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, __fmul_rn(a.y, b.y)), fmaf(a.y, b.x, -__fmul_rn(a.x, b.y)));
}
// data x twiddle (DIR < 0) or x conj(twiddle) (DIR > 0)
template <int DIR>
__device__ __forceinline__ double2 tw_mul(double2 a, double2 w) { return DIR < 0 ? cmul(a, w) : cmulc(a, w); }
template <int DIR>
__device__ __forceinline__ float2 tw_mul(float2 a, float4 w) {
  const float wy = DIR < 0 ? w.y : -w.y, ly = DIR < 0 ? w.w : -w.w;
  // (a.x + i a.y)(hi + lo): the lo terms first, then the hi products on top
  const float cx = fmaf(a.x, w.z, -__fmul_rn(a.y, ly));
  const float cy = fmaf(a.x, ly, __fmul_rn(a.y, w.z));
  return make_float2(fmaf(a.x, w.x, fmaf(-a.y, wy, cx)), fmaf(a.x, wy, fmaf(a.y, w.x, cy)));
}
// sqrt(1/2) * a + b (the radix-8 constant).  complex128: one fused rounding.
// complex64: hi + lo = sqrt(1/2) to 2^-48 so no rounded constant is applied
// to the data; the product is rounded first (inside the fma the exact hi*a
// keeps the bits that carry lo*a through the rounding), then b is added --
// folding b into the inner fma instead would round lo*a away against b
// every time, i.e. apply hi alone (a systematic 1.2e-8 per use).
__device__ __forceinline__ double fma_h(double a, double b) { return fma(0.70710678118654752440, a, b); }
__device__ __forceinline__ float fma_h(float a, float b) {
  return fmaf(0x1.6a09e6p-1f, a, 0x1.9fcef4p-27f * a) + b;
}
// multiply by -i (DIR=-1, forward) or +i (DIR=+1, inverse)
template <int DIR, typename C>
__device__ __forceinline__ C mul_i(C a) {
  return DIR < 0 ? CT<C>::mk(a.y, -a.x) : CT<C>::mk(-a.y, a.x);
}

// In-register DFT of size R with sign DIR (-1 forward, +1 inverse),
// natural order in and out: v[k] <- sum_j v[j] exp(DIR 2 pi i j k / R).
template <int R, int DIR>
struct Dft;

template <int DIR>
struct Dft<2, DIR> {
  template <typename C>
  __device__ __forceinline__ static void run(C* v) {
    C a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
  }
};

template <int DIR>
struct Dft<4, DIR> {
  template <typename C>
  __device__ __forceinline__ static void run(C* v) {
    C t0 = cadd(v[0], v[2]);
    C t1 = csub(v[0], v[2]);
    C t2 = cadd(v[1], v[3]);
    C t3 = mul_i<DIR>(csub(v[1], v[3]));
    v[0] = cadd(t0, t2);
    v[2] = csub(t0, t2);
    v[1] = cadd(t1, t3);
    v[3] = csub(t1, t3);
  }
};

template <int DIR>
struct Dft<8, DIR> {
  template <typename C>
  __device__ __forceinline__ static void run(C* v) {
    C e[4] = {v[0], v[2], v[4], v[6]};
    C o[4] = {v[1], v[3], v[5], v[7]};
    Dft<4, DIR>::run(e);
    Dft<4, DIR>::run(o);
    // o[k] *= exp(DIR i pi k / 4); the sqrt(1/2) of k = 1, 3 is fused into
    // the final additions (h s + e with one rounding)
    using R = typename CT<C>::R;
    R s1, d1, s3, d3;  // o1 = h (s1, d1), o3 = h (s3, d3)
    if (DIR < 0) {
      s1 = o[1].x + o[1].y;
      d1 = o[1].y - o[1].x;
      s3 = o[3].y - o[3].x;
      d3 = -(o[3].x + o[3].y);
    } else {
      s1 = o[1].x - o[1].y;
      d1 = o[1].x + o[1].y;
      s3 = -(o[3].x + o[3].y);
      d3 = o[3].x - o[3].y;
    }
    C o2 = mul_i<DIR>(o[2]);
    v[0] = cadd(e[0], o[0]);
    v[4] = csub(e[0], o[0]);
    v[1] = CT<C>::mk(fma_h(s1, e[1].x), fma_h(d1, e[1].y));
    v[5] = CT<C>::mk(fma_h(-s1, e[1].x), fma_h(-d1, e[1].y));
    v[2] = cadd(e[2], o2);
    v[6] = csub(e[2], o2);
    v[3] = CT<C>::mk(fma_h(s3, e[3].x), fma_h(d3, e[3].y));
    v[7] = CT<C>::mk(fma_h(-s3, e[3].x), fma_h(-d3, e[3].y));
  }
};

// Compile-time radix plan for a line of length L (8 <= L <= 1024): stages of
// radix 8 followed by at most one radix-2 or radix-4 stage.
template <int L, int E = kElems>
struct Plan {
  static constexpr int T = L / E;  // threads per line
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
  // Stage-major twiddle table: stage s >= 1 holds (R_s - 1) x NS_s entries
  // T[r-1][k] = exp(-2 pi i r k / (NS_s R_s)); for a fixed r the k of a warp
  // are consecutive, so a twiddle gather touches as few 128-byte lines as the
  // data access does.
  __host__ __device__ static constexpr int tw_offset(int s) {
    int o = 0;
    for (int i = 1; i < s; ++i) o += (radix(i) - 1) * ns(i);
    return o;
  }
  static constexpr int tw_size = tw_offset(nstages);
};

// Contiguous-line shared-memory position with one 16-byte pad every 8 points
// (keeps stride-8 scatters conflict free for 128-bit accesses).
__device__ __forceinline__ int pad8(int i) { return i + (i >> 3); }

// Accessor abstractions for the exchange buffer: element i of the thread's
// line, where `base` already selects the line (contiguous) or column (strided).
template <typename C>
struct SmemContig {
  C* base;
  __device__ __forceinline__ C& at(int i) const { return base[pad8(i)]; }
};
template <typename C, int W = 8>
struct SmemStrided {  // column-fastest tile of W columns: element i of column c at i*W + c
  C* base;            // points at column c
  __device__ __forceinline__ C& at(int i) const { return base[i * W]; }
};

// Programmatic dependent launch (griddepcontrol): no-ops for grids launched
// without the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" :::); }

// Barrier among the threads that share one exchange buffer.
struct SyncBlock {
  __device__ __forceinline__ void operator()() const { __syncthreads(); }
};
struct SyncWarp {  // the whole line lives inside one warp
  __device__ __forceinline__ void operator()() const { __syncwarp(); }
};
struct SyncNamed {  // T threads (a multiple of 32) of one line: named barrier
  int id, count;
  __device__ __forceinline__ void operator()() const {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
  }
};

// Table loads: read-only global through the L1 (default), or plain loads of a
// CTA's shared-memory copy.  (Staging the 512-point twiddles and the kinetic
// sincos table in the ring x pass's shared memory measured slower: 1.14 ->
// 1.31-1.36 ms, the staged loads raise register pressure to spills; r02.)
struct LdgLoad {
  __device__ __forceinline__ static double2 ld(const double2* p) { return __ldg(p); }
};
struct SmemLoad {  // the pointer must derive from the kernel's shared array (LDS after inlining)
  __device__ __forceinline__ static double2 ld(const double2* p) { return *p; }
};

// Twiddles of a complex128 radix-8 butterfly: u[r] *= w^r (w = exp(-2 pi i
// k / (8 NS)), conjugated for DIR > 0).  Three table loads (w, w^2, w^4; the
// table's column k at stride NS) and the other four as their products: the
// axis passes are bound by the L1 data pipe (ncu r02), and a twiddle gather
// costs up to 4 wavefronts against 4 FP64 instructions for a product.  The
// products carry ~1 ulp more rounding than table values; FFT roundoff is not
// what the 1e-10 parity gate is sensitive to.  Every radix-8
// kernel uses this helper, so all of them stay bitwise interchangeable.
template <int DIR, typename LD = LdgLoad>
__device__ __forceinline__ void radix8_twiddles(double2* u, const double2* __restrict__ col, int NS) {
  const double2 w1 = LD::ld(col), w2 = LD::ld(col + NS), w4 = LD::ld(col + 3 * NS);
  const double2 w3 = cmul(w1, w2);
  u[1] = tw_mul<DIR>(u[1], w1);
  u[2] = tw_mul<DIR>(u[2], w2);
  u[3] = tw_mul<DIR>(u[3], w3);
  u[4] = tw_mul<DIR>(u[4], w4);
  u[5] = tw_mul<DIR>(u[5], cmul(w1, w4));
  u[6] = tw_mul<DIR>(u[6], cmul(w2, w4));
  u[7] = tw_mul<DIR>(u[7], cmul(w3, w4));
}

// One Stockham stage on the eight registers of thread t.
//   radix R, stride Ns (product of earlier radices), line length L.
// Input: v[m] = x[t + m*T].  Output scattered to smem (unless last stage, in
// which case v[m] = X[t + m*T] stays in registers).
template <int L, int E, int R, int NS, int TWO, int DIR, bool LAST, typename C, typename Smem>
__device__ __forceinline__ void stockham_stage(C* v, int t, const TwOf<C>* __restrict__ tw, Smem sm) {
  constexpr int T = L / E;
  constexpr int NB = E / R;  // butterflies per thread
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    C u[R];
#pragma unroll
    for (int r = 0; r < R; ++r) u[r] = v[b + r * NB];
    const int j = t + b * T;
    const int k = j & (NS - 1);
    if (NS > 1) {
      if constexpr (R == 8 && std::is_same<C, double2>::value) {
        radix8_twiddles<DIR>(u, tw + TWO + k, NS);
      } else {
        // twiddle exp(DIR 2 pi i r k / (NS R)) from the stage-major table
#pragma unroll
        for (int r = 1; r < R; ++r) {
          const TwOf<C> w = __ldg(&tw[TWO + (r - 1) * NS + k]);
          u[r] = tw_mul<DIR>(u[r], w);
        }
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

template <int L, int E, int S, int DIR, typename C, typename Smem, typename Sync>
__device__ __forceinline__ void fft_stages(C* v, int t, const TwOf<C>* __restrict__ tw, Smem sm,
                                           Sync sync) {
  using P = Plan<L, E>;
  constexpr int T = P::T;
  if constexpr (S < P::nstages) {
    constexpr int R = P::radix(S);
    constexpr int NS = P::ns(S);
    constexpr bool LAST = (S == P::nstages - 1);
    stockham_stage<L, E, R, NS, P::tw_offset(S), DIR, LAST>(v, t, tw, sm);
    if constexpr (!LAST) {
      sync();
#pragma unroll
      for (int m = 0; m < E; ++m) v[m] = sm.at(t + m * T);
      sync();
      fft_stages<L, E, S + 1, DIR>(v, t, tw, sm, sync);
    }
  }
}

// Full in-register/shared 1D FFT of the thread's line.  On entry v[m] holds
// x[t + m*T], on exit X[t + m*T] (unnormalized, sign DIR), T = L/E threads
// per line.  Every thread that shares the exchange buffer must call it
// (barriers inside).  The radix plan (and hence the twiddle table) depends
// only on L, not on E.
template <int L, int DIR, int E = kElems, typename C, typename Smem, typename Sync>
__device__ __forceinline__ void line_fft(C* v, int t, const TwOf<C>* __restrict__ tw, Smem sm, Sync sync) {
  fft_stages<L, E, 0, DIR>(v, t, tw, sm, sync);
}

// --- exact phase recipes (reference propagator.py:61-68, qgrid.py:98-117) ---
// These products must not be contracted into FMAs: a systematic one-ulp phase
// error fails the 1e-10 parity gate.

// v_i = (V - shift) / E0  (evaluated once per plan, propagator.py:65 / :75)
__device__ __forceinline__ double v_internal(double v, double shift, double e0) {
  return __ddiv_rn(__dsub_rn(v, shift), e0);
}
// potential phase (coef * v_i) * dt_i, coef -0.5 (half step) or -1.0 (full step)
__device__ __forceinline__ double v_phase_i(double vi, double coef, double dt_i) {
  return __dmul_rn(__dmul_rn(coef, vi), dt_i);
}
__device__ __forceinline__ double v_phase(double v, double shift, double e0, double coef, double dt_i) {
  return v_phase_i(v_internal(v, shift, e0), coef, dt_i);
}
// kinetic phase: (-0.5 * (((kx2 + ky2) + kz2) * L0^2)) * dt_i
__device__ __forceinline__ double k_phase(double kx2, double ky2, double kz2, double len2, double dt_i) {
  double k2 = __dadd_rn(__dadd_rn(kx2, ky2), kz2);
  return __dmul_rn(__dmul_rn(-0.5, __dmul_rn(k2, len2)), dt_i);
}


// sincos rotation table size: 2^kSCBits entries (cos, sin)(2 pi j / 2^kSCBits)
#ifndef CTAP_SC_BITS
#define CTAP_SC_BITS 8
#endif
constexpr int kSCBits = CTAP_SC_BITS;
constexpr int kSCN = 1 << kSCBits;
static_assert(kSCBits == 4 || kSCBits == 8, "sincos table: 16 or 256 entries");

// polynomial/reduction constants as constant-bank operands (no per-use
// register materialisation).  Step h = 2 pi / kSCN = C1 + C2 + C3 (27 + 27 +
// 53 bits: n C1 is exact for |n| < 2^26), the pi/128 split scaled by a power
// of two.
__constant__ double kSC[16] = {
    kSCN / 6.283185307179586476925286766559,  // 0: 1/h
    0x1.921fb54000000p-6 * (256 / kSCN),      // 1: C1
    0x1.10b4610000000p-36 * (256 / kSCN),     // 2: C2
    0x1.a62633145c06ep-64 * (256 / kSCN),     // 3: C3
    6755399441055744.0,                       // 4: 1.5 * 2^52
    -1.6666666666666666e-01,                  // 5: -1/3!
    8.3333333333333333e-03,                   // 6: 1/5!
    -1.9841269841269841e-04,                  // 7: -1/7!
    2.7557319223985893e-06,                   // 8: 1/9!
    -2.5052108385441720e-08,                  // 9: -1/11!
    -0.5,                                     // 10: -1/2!
    4.1666666666666664e-02,                   // 11: 1/4!
    -1.3888888888888889e-03,                  // 12: -1/6!
    2.4801587301587302e-05,                   // 13: 1/8!
    -2.7557319223985888e-07,                  // 14: -1/10!
    0.0,
};

// the out-of-range path of fast_sincos, kept out of line: inlined at every
// point of a kernel it would multiply the code size
__device__ __noinline__ inline void slow_sincos(double phi, double f, double* s, double* c) {
  double ss, cc;
  sincos(phi, &ss, &cc);
  *s = ss * f;
  *c = cc * f;
}

// sincos for the phase factors.  The phase itself is exact (computed with the
// recipes above); only cos/sin of it are evaluated here, to ~1.5 ulp:
//   n = rint(phi / h) via the 1.5*2^52 magic constant, r = phi - n h by a
//   three-term Cody-Waite split, Taylor polynomials on |r| <= h/2, and a
//   rotation by tab[n mod kSCN] = f (cos, sin)(n h) where f is a per-plan
//   factor (1, or the kinetic step's 1/N folded in -- a power of two, so the
//   folding is exact).
// With 256 entries (h = pi/128, the default) the polynomials stop at r^7 /
// r^6; the kinetic phases (k^2 varies fast along a line) scatter a warp's
// gather over ~30 128-byte lines.  With 16 entries (CTAP_SC_BITS=4: h = pi/8,
// polynomials to r^11 / r^10, truncation < 1e-17) a gather touches at most two
// lines, but the four extra FMAs cost more than the wavefronts they save:
// [x K x^-1] 1.177 -> 1.210 ms, [z^-1 V z] 1.067 -> 1.077 ms (B200, r02).
// |phi| >= 2^20 falls back to the library (never on CTAP grids, where
// |phi| < 1e6) and applies f = tab[0].x explicitly.  Errors of an ulp in the
// factor are harmless (only the phase must be bit-exact).
template <typename LD = LdgLoad>
__device__ __forceinline__ void fast_sincos(double phi, const double2* __restrict__ tab, double* s, double* c) {
  if (fabs(phi) < 1048576.0) {
    const double t = fma(phi, kSC[0], kSC[4]);
    const int n = __double2loint(t);
    const double nf = t - kSC[4];
    double r = fma(-nf, kSC[1], phi);
    r = fma(-nf, kSC[2], r);
    r = fma(-nf, kSC[3], r);
    const double r2 = r * r;
    double ps, pc;
    if constexpr (kSCBits == 4) {
      ps = fma(r2, kSC[9], kSC[8]);
      ps = fma(r2, ps, kSC[7]);
      ps = fma(r2, ps, kSC[6]);
      ps = fma(r2, ps, kSC[5]);
      pc = fma(r2, kSC[14], kSC[13]);
      pc = fma(r2, pc, kSC[12]);
      pc = fma(r2, pc, kSC[11]);
      pc = fma(r2, pc, kSC[10]);
    } else {
      ps = fma(r2, kSC[7], kSC[6]);
      ps = fma(r2, ps, kSC[5]);
      pc = fma(r2, kSC[12], kSC[11]);
      pc = fma(r2, pc, kSC[10]);
    }
    const double sr = fma(r * r2, ps, r);
    const double cr = fma(r2, pc, 1.0);
    const double2 tb = LD::ld(&tab[n & (kSCN - 1)]);
    *c = fma(tb.x, cr, -(tb.y * sr));
    *s = fma(tb.y, cr, tb.x * sr);
  } else {
    slow_sincos(phi, LD::ld(tab).x, s, c);
  }
}

}  // namespace ctap
