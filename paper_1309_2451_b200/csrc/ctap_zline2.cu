// z passes on the two-stage line FFT (ctap_fft2.cuh), complex128, L = 64..1024.
//
// Reference: propagator.py:98-107 (_advance).  The position-space pass of the
// telescoped step is  [z^-1 . V . z]:  inverse z transform, exp(-i V dt)
// with the reference's exact phase (propagator.py:65-67), forward z
// transform, in one HBM read and one write of psi (+ the 8-byte v_i read).
// Segment ends use [Vh . z] and [z^-1 . Vh].
//
// T = L/32 consecutive lanes own a line (32 points per lane, points t + m T),
// so every warp access is 32/T whole 16T-byte runs of contiguous memory and
// the exchange buffer of a line is warp-private (__syncwarp only).  Compared
// with the radix-8 kernel (zline_kernel, ctap_passes.cu) a transform makes one
// shared-memory round trip instead of two and gathers 15 twiddles per 16
// points instead of 14 per 8 (see ctap_fft2.cuh).
#include <cstdlib>

#include "ctap_fft2.cuh"
#include "ctap_internal.h"
#include "ctap_tile.cuh"

#ifndef CTAP_Z2_THREADS
#define CTAP_Z2_THREADS 128
#endif
#ifndef CTAP_Z2_MINB
#define CTAP_Z2_MINB 3
#endif
#ifndef CTAP_Z2_VASYNC
#define CTAP_Z2_VASYNC 1
#endif

namespace ctap {

template <int L>
struct Z2Cfg {
  using P = Plan2<L>;
  static constexpr int threads = CTAP_Z2_THREADS;
  static constexpr int lines = threads / P::T;  // lines per block
  static constexpr size_t smem = (size_t)lines * P::smem_line * sizeof(double2);
};

template <int L, int KIND, bool VTAB, int CH>
__global__ void __launch_bounds__(CTAP_Z2_THREADS, CTAP_Z2_MINB)
    zline2_kernel(ZArgs a, const double2* __restrict__ tw) {
  using P = Plan2<L>;
  using Cfg = Z2Cfg<L>;
  static_assert(P::T <= 32, "a line lives inside one warp");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int t = threadIdx.x % P::T;
  const int c = threadIdx.x / P::T;
  double2* sm = reinterpret_cast<double2*>(smem_raw) + c * P::smem_line;
  const uint32_t line = blockIdx.x * Cfg::lines + c;
  const bool active = line < a.nlines;
  const uint32_t off = line * L;
  const uint32_t zmask = (1u << a.lzc) - 1u, coff = line << a.lzc;
  auto at_in = [&](uint32_t zz) { return CH & 1 ? (zz >> a.lzc) * a.cs + coff + (zz & zmask) : off + zz; };
  auto at_out = [&](uint32_t zz) { return CH & 2 ? (zz >> a.lzc) * a.cs + coff + (zz & zmask) : off + zz; };
  const double2* in = (const double2*)a.psi;
  double2* out = (double2*)a.out;
  const auto sync = [] { __syncwarp(); };

  double2 v[32];
#pragma unroll
  for (int m = 0; m < 32; ++m) v[m] = active ? __ldcg(&in[at_in(t + m * P::T)]) : make_double2(0.0, 0.0);

  if constexpr (KIND == T_FWD) {
    line_fft2<L, -1>(v, t, tw, sm, sync);
  } else if constexpr (KIND == T_INV) {
    line_fft2<L, +1>(v, t, tw, sm, sync);
  } else if constexpr (KIND == T_VFIRST) {  // Vh, then forward
    if (active) {
#pragma unroll
      for (int m = 0; m < 32; ++m) mul_vphase(v[m], __ldcg(&a.ph.vi[off + t + m * P::T]), -0.5, a.ph);
    }
    line_fft2<L, -1>(v, t, tw, sm, sync);
  } else if constexpr (KIND == T_VMID && VTAB) {  // inverse, x exp(-iV dt) table, forward
    line_fft2<L, +1>(v, t, tw, sm, sync);
    if (active) {
      const double2* expv = (const double2*)a.ph.expv;
#pragma unroll
      for (int m = 0; m < 32; ++m) v[m] = cmul(v[m], __ldcg(&expv[off + t + m * P::T]));
    }
    line_fft2<L, -1>(v, t, tw, sm, sync);
  } else {  // T_VMID: inverse, V, forward; T_VLAST: inverse, Vh
#if CTAP_Z2_VASYNC
    // v_i of the line copied into the (then free) exchange buffer by cp.async
    // during stage 2 of the inverse transform, so its latency hides behind it
    double* vs = reinterpret_cast<double*>(sm);
    const auto fetch_v = [&] {
      if (active) {
#pragma unroll
        for (int m = 0; m < 32; ++m)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(vs + t + m * P::T)),
                       "l"(a.ph.vi + off + t + m * P::T)
                       : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    line_fft2<L, +1>(v, t, tw, sm, sync, fetch_v);
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncwarp();
    if (active) {
#pragma unroll
      for (int m = 0; m < 32; ++m) mul_vphase(v[m], vs[t + m * P::T], KIND == T_VMID ? -1.0 : -0.5, a.ph);
    }
    __syncwarp();
#else
    line_fft2<L, +1>(v, t, tw, sm, sync);
    if (active) {
#pragma unroll
      for (int m = 0; m < 32; ++m)
        mul_vphase(v[m], __ldcg(&a.ph.vi[off + t + m * P::T]), KIND == T_VMID ? -1.0 : -0.5, a.ph);
    }
#endif
    if constexpr (KIND == T_VMID) line_fft2<L, -1>(v, t, tw, sm, sync);
  }

  if (active) {
#pragma unroll
    for (int m = 0; m < 32; ++m) __stcg(&out[at_out(t + m * P::T)], v[m]);
  }
}

template <int L, int KIND, bool VTAB, int CH>
static cudaError_t launch_z2(const ZArgs& a, const double2* tw, cudaStream_t st) {
  using Cfg = Z2Cfg<L>;
  auto k = zline2_kernel<L, KIND, VTAB, CH>;
  static std::atomic<uint64_t> attr_done{0};
  if (cudaError_t e = ctap_smem_attr(k, Cfg::smem, attr_done)) return e;
  k<<<(a.nlines + Cfg::lines - 1) / Cfg::lines, Cfg::threads, Cfg::smem, st>>>(a, tw);
  return cudaGetLastError();
}

template <int KIND, bool VTAB, int CH>
static cudaError_t dispatch_z2(int L, const ZArgs& a, const double2* tw, cudaStream_t st) {
  switch (L) {
    case 64: return launch_z2<64, KIND, VTAB, CH>(a, tw, st);
    case 128: return launch_z2<128, KIND, VTAB, CH>(a, tw, st);
    case 256: return launch_z2<256, KIND, VTAB, CH>(a, tw, st);
    case 512: return launch_z2<512, KIND, VTAB, CH>(a, tw, st);
    case 1024: return launch_z2<1024, KIND, VTAB, CH>(a, tw, st);
  }
  return cudaErrorNotSupported;
}

}  // namespace ctap

using namespace ctap;

// host-side: the stage-2 twiddle tables of the two-stage plan for L = 64..1024,
// appended to the plan's twiddle vector (off2[i] = start, in double2, of L = 64 << i)
void ctap_append_twiddles2(std::vector<double>& t, int off2[5]) {
  for (int i = 0; i < 5; ++i) {
    const int L = 64 << i, R2 = L / 32;
    off2[i] = (int)(t.size() / 2);
    for (int r = 1; r < R2; ++r)
      for (int k = 0; k < 32; ++k) {
        const long double ang =
            2.0L * 3.14159265358979323846264338327950288L * (long double)(r * k) / (long double)L;
        t.push_back((double)cosl(ang));
        t.push_back((double)(-sinl(ang)));
      }
  }
}

// z pass kinds (natural and pencil z-chunked) on the two-stage kernel;
// cudaErrorNotSupported hands the pass back to zline_kernel.
// ch: bit 0 input z-chunked, bit 1 output z-chunked (pencil)
cudaError_t ctap_run_z2(const ctap_plan* p, int tkind, bool vtab, int ch, const ZArgs& a, cudaStream_t st) {
  const int L = (int)p->n[2];
  if (!p->z2 || p->dtype != CTAP_C128 || L < 64 || L > 1024) return cudaErrorNotSupported;
  const double2* tw = p->twiddles + p->tw2_off[ilog2i(L) - 6];
#define CTAP_Z2K(K, VT, C) return dispatch_z2<K, VT, C>(L, a, tw, st)
  switch (ch) {
    case 0:
      switch (tkind) {
        case T_FWD: CTAP_Z2K(T_FWD, false, 0);
        case T_INV: CTAP_Z2K(T_INV, false, 0);
        case T_VFIRST: CTAP_Z2K(T_VFIRST, false, 0);
        case T_VMID:
          if (vtab) CTAP_Z2K(T_VMID, true, 0);
          CTAP_Z2K(T_VMID, false, 0);
        case T_VLAST: CTAP_Z2K(T_VLAST, false, 0);
      }
      break;
    case 2:
      if (tkind == T_VFIRST) CTAP_Z2K(T_VFIRST, false, 2);
      break;
    case 3:
      if (tkind == T_VMID) CTAP_Z2K(T_VMID, false, 3);
      break;
    case 1:
      if (tkind == T_VLAST) CTAP_Z2K(T_VLAST, false, 1);
      break;
  }
#undef CTAP_Z2K
  return cudaErrorNotSupported;
}
