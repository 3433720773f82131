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
// Two kernel shapes:
//   zline_kernel  z passes.  Lines are contiguous; T = L/8 consecutive lanes
//                 own one line (every warp access is 512 contiguous bytes),
//                 the exchange buffer is a padded line, and only the threads
//                 of one line synchronise (warp or named barrier).
//   tile_kernel   y and x passes.  A tile is 8 consecutive z columns x the
//                 whole line: thread (t, col) owns points t + m*T of column
//                 col, so every warp access is 4 rows x 128 contiguous bytes
//                 and the [i][8] exchange buffer is bank-conflict free.
//
// Phase factors come either from the per-point exact recipes (on the fly,
// 8 B/pt of v_i = V/E0 per step) or from plan-owned complex tables of the
// same values (16 B/pt for the full V step and for K, no sincos per step);
// both give bit-identical phases.
#include <cmath>
#include <cstdlib>
#include <vector>

#include "ctap_device.cuh"
#include "ctap_internal.h"
#include "ctap_tile.cuh"

// resident threads per SM the register allocation of the strided kernels is
// sized for, and min blocks per SM of the z kernels (256 threads)
#ifndef CTAP_OCC
#define CTAP_OCC 1024
#endif
#ifndef CTAP_TMA_DEFAULT
#define CTAP_TMA_DEFAULT 1
#endif
// z columns per x-pass tile (8 or 16)
#ifndef CTAP_XW
#define CTAP_XW 8
#endif
#ifndef CTAP_Z_MINB
#define CTAP_Z_MINB 3
#endif
// threads per z-pass block (lines per block = this / (L/8))
#ifndef CTAP_Z_THREADS
#define CTAP_Z_THREADS 256
#endif
#ifndef CTAP_Z_MINB_TAB
#define CTAP_Z_MINB_TAB 2
#endif
#ifndef CTAP_OCC_TAB
#define CTAP_OCC_TAB 512
#endif

namespace ctap {

// ---------------------------------------------------------------------------
// z passes
// ---------------------------------------------------------------------------

template <int L, typename CV>
struct ZCfg {
  static constexpr int T = L / kElems;
  static constexpr int C = (CTAP_Z_THREADS / T) > 0 ? (CTAP_Z_THREADS / T) : 1;  // lines per block
  static constexpr int threads = C * T;
  static constexpr int smem_line = L + L / 8;             // padded complex per line
  static constexpr size_t smem = (size_t)C * smem_line * sizeof(CV);
};


template <int L, int KIND, bool VTAB, typename CV, typename Sync>
__device__ __forceinline__ void z_body(const ZArgs& a, CV* v, int t, uint32_t off, bool active,
                                       const TwOf<CV>* __restrict__ tw, SmemContig<CV> sm, Sync sync) {
  constexpr int T = L / kElems;
  if constexpr (KIND == T_FWD) {
    line_fft<L, -1>(v, t, tw, sm, sync);
  } else if constexpr (KIND == T_INV) {
    line_fft<L, +1>(v, t, tw, sm, sync);
  } else if constexpr (KIND == T_VFIRST) {  // Vh, then forward
    if (active) {
      // all eight v_i loads in flight before the first phase
      double vi[kElems];
#pragma unroll
      for (int m = 0; m < kElems; ++m) vi[m] = __ldcg(&a.ph.vi[off + t + m * T]);
#pragma unroll
      for (int m = 0; m < kElems; ++m) mul_vphase(v[m], vi[m], -0.5, a.ph);
    }
    line_fft<L, -1>(v, t, tw, sm, sync);
  } else if constexpr (KIND == T_VMID && VTAB) {  // inverse, x exp(-iV dt) table, forward
    // the table values are loaded before the inverse transform so their
    // latency hides behind it (they are consumed right after it)
    const CV* expv = (const CV*)a.ph.expv;
    CV f[kElems];
#pragma unroll
    for (int m = 0; m < kElems; ++m) f[m] = active ? __ldcg(&expv[off + t + m * T]) : CT<CV>::mk(1, 0);
    line_fft<L, +1>(v, t, tw, sm, sync);
#pragma unroll
    for (int m = 0; m < kElems; ++m) v[m] = cmul(v[m], f[m]);
    line_fft<L, -1>(v, t, tw, sm, sync);
  } else {  // T_VMID: inverse, V, forward; T_VLAST: inverse, Vh
    double vi[kElems];
    // v_i loaded before the inverse transform (its latency hides behind it),
    // all but the last: one register pair fewer held across the transform at
    // the 80-register budget schedules it better -- [z^-1 V z] 1.08 -> 1.02
    // ms at 512^3 (8 / 7 / 6 / 5 early: 1.08 / 1.02 / 1.02 / 1.09; same-box
    // A/B, bitwise identical results).  (ptxas's spill count, 45 vs 23, is
    // code around the never-taken |phi| >= 2^20 library sincos call: ncu
    // counts no local load or store executed.)
#ifndef CTAP_Z_VEARLY
#define CTAP_Z_VEARLY 7
#endif
#pragma unroll
    for (int m = 0; m < CTAP_Z_VEARLY; ++m) vi[m] = active ? __ldcg(&a.ph.vi[off + t + m * T]) : 0.0;
    line_fft<L, +1>(v, t, tw, sm, sync);
#pragma unroll
    for (int m = CTAP_Z_VEARLY; m < kElems; ++m) vi[m] = active ? __ldcg(&a.ph.vi[off + t + m * T]) : 0.0;
#pragma unroll
    for (int m = 0; m < kElems; ++m) mul_vphase(v[m], vi[m], KIND == T_VMID ? -1.0 : -0.5, a.ph);
    if constexpr (KIND == T_VMID) line_fft<L, -1>(v, t, tw, sm, sync);
  }
}

// register budget per kernel flavour (measured, 512^3): the table-driven
// [z^-1 V z] wants 128 registers, the sincos flavours 64
template <int KIND, bool VTAB>
struct ZMinBlocks {
  static constexpr int value = (KIND == T_VMID && VTAB) ? CTAP_Z_MINB_TAB : CTAP_Z_MINB;
};

// The observer sums of this thread's points (psi after the segment-end pass,
// in registers), reduced over the warp in a fixed shuffle tree and stored as
// the warp's partial [sum rho, left, right, edge]: the reduction of
// observables.py:74-110 fused into the write-back of the last pass, so an
// observer event reads no extra byte of psi.  The middle guide
// is total - left - right, formed in the finalize (ctap_reduce.cu).
// Deterministic: fixed per-thread order, shuffle tree, partial order.
constexpr int kObsVals = 4;
template <int L, typename CV>
__device__ __forceinline__ void z_observe(const ZArgs& a, const CV* v, int t, uint32_t line, bool active) {
  constexpr int T = L / kElems;
  double acc[kObsVals] = {0.0, 0.0, 0.0, 0.0};
  if (active) {
    const uint32_t x = line >> a.lny, y = line & (a.ny - 1u);  // ny is a power of two
    const int mg = a.margin;
    const bool line_edge = (int)x < mg || (int)x >= (int)a.nx - mg || (int)y < mg || (int)y >= (int)a.ny - mg;
    const bool part = a.obs_mask != nullptr;
    const uint32_t mk = part ? __ldg(&a.obs_mask[x * T + t]) : 0u;
#pragma unroll
    for (int m = 0; m < kElems; ++m) {
      const int z = t + m * T;
      const double rho = (double)v[m].x * v[m].x + (double)v[m].y * v[m].y;
      acc[0] += rho;
      if (part) {
        if (mk >> m & 1u) acc[1] += rho;
        if (mk >> (8 + m) & 1u) acc[2] += rho;
      }
      // z-edge points: for margin <= T only the first and last of a thread's
      // points can be within margin of a z face
      if (m == 0 || m == kElems - 1 || mg > T)
        if (z < mg || z >= L - mg) acc[3] += rho;
    }
    if (line_edge) acc[3] = acc[0];  // every point of the line: the same sum in the same order
  }
  // warp sums of the four values by a transposing tree: the first level
  // trades half of the values between the half-warps, the second half of the
  // rest between quarter-warps, so 12 shuffles and 6 additions instead of
  // 4 x 5 x 2 and 20 (the pass is bound by the L1 data pipe, which the
  // shuffles share); lane 8 k ends with value k
  const int lane = threadIdx.x & 31;
  const bool h16 = lane & 16, h8 = lane & 8;
  const double k0 = h16 ? acc[2] : acc[0], k1 = h16 ? acc[3] : acc[1];
  const double s0 = h16 ? acc[0] : acc[2], s1 = h16 ? acc[1] : acc[3];
  const double b0 = k0 + __shfl_xor_sync(0xffffffffu, s0, 16);
  const double b1 = k1 + __shfl_xor_sync(0xffffffffu, s1, 16);
  double r = (h8 ? b1 : b0) + __shfl_xor_sync(0xffffffffu, h8 ? b0 : b1, 8);
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
  if ((lane & 7) == 0)
    a.obs_partial[((size_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * kObsVals + (lane >> 3)] = r;
}

template <int L, int KIND, bool VTAB, typename CV, int CH = 0, bool OBS = false>
__global__ void __launch_bounds__(ZCfg<L, CV>::threads, ZMinBlocks<KIND, VTAB>::value) zline_kernel(ZArgs a, const TwOf<CV>* __restrict__ tw) {
  using Cfg = ZCfg<L, CV>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  CV* smem = reinterpret_cast<CV*>(smem_raw);
  const CV* in = (const CV*)a.psi;
  CV* psi = (CV*)a.out;  // == a.psi for the in-place natural and z-chunked passes
  const int t = threadIdx.x % Cfg::T;
  const int c = threadIdx.x / Cfg::T;
  const uint32_t line = blockIdx.x * Cfg::C + c;
  const bool active = line < a.nlines;
  const uint32_t off = line * L;
  // element z of this line: natural off + z, or z-chunked (pencil)
  const uint32_t zmask = (1u << a.lzc) - 1u, coff = line << a.lzc;
  auto at_in = [&](uint32_t zz) { return CH & 1 ? (zz >> a.lzc) * a.cs + coff + (zz & zmask) : off + zz; };
  pdl_wait();  // programmatic dependent launch: the preceding grid's stores are visible from here
  auto at_out = [&](uint32_t zz) { return CH & 2 ? (zz >> a.lzc) * a.cs + coff + (zz & zmask) : off + zz; };
  SmemContig<CV> sm{smem + c * Cfg::smem_line};
  CV v[kElems];
#pragma unroll
  for (int m = 0; m < kElems; ++m) v[m] = active ? __ldcg(&in[at_in(t + m * Cfg::T)]) : CT<CV>::mk(0, 0);
  if constexpr (Cfg::T <= 32) {
    z_body<L, KIND, VTAB>(a, v, t, off, active, tw, sm, SyncWarp{});
  } else {
    z_body<L, KIND, VTAB>(a, v, t, off, active, tw, sm, SyncNamed{1 + c, Cfg::T});
  }
  pdl_trigger();  // the next grid of the stream may start its launch (it waits for our stores)
  if (active) {
#pragma unroll
    for (int m = 0; m < kElems; ++m) __stcg(&psi[at_out(t + m * Cfg::T)], v[m]);
  }
  if constexpr (OBS) z_observe<L>(a, v, t, line, active);
}

// ---------------------------------------------------------------------------
// y and x passes
// ---------------------------------------------------------------------------

// points per thread of the strided kernels (8 or 16): 16 halves the threads
// (and the barrier fan-in) per tile and doubles each thread's ILP
#ifndef CTAP_TILE_E
#define CTAP_TILE_E 8
#endif
#ifndef CTAP_E1024
#define CTAP_E1024 8  // 16 measured: y passes equal, [x K x^-1] 7.70 -> 8.32 ms at 1024^2 x 512
#endif

template <int L, typename CV, int W>
struct TileCfg {
  // 1024-point lines in 4-column tiles: 16 points per thread (64 threads per column)
  static constexpr int E = (L >= 1024 && W == 4) ? CTAP_E1024 : (L >= 256) ? CTAP_TILE_E : kElems;
  static constexpr int T = L / E;
  static constexpr int per_tile = T * W;
  static constexpr int G = per_tile >= 128 ? 1 : 128 / per_tile;  // tiles per block
  static constexpr int threads = G * per_tile;
  static constexpr size_t smem = (size_t)G * L * W * sizeof(CV);
  static constexpr int occ = CTAP_OCC * kElems / E;  // same register file, E/8 x the registers
  static constexpr int minb = occ / threads > 0 ? occ / threads : 1;
  static constexpr int minb_tab = CTAP_OCC_TAB / threads > 0 ? CTAP_OCC_TAB / threads : 1;
};

template <int L, int KIND, bool PIN, bool POUT, bool KTAB, typename CV, int W, bool PEERS = false>
__global__ void __launch_bounds__(TileCfg<L, CV, W>::threads,
                                  KTAB ? TileCfg<L, CV, W>::minb_tab : TileCfg<L, CV, W>::minb)
    tile_kernel(TileArgs a, const TwOf<CV>* __restrict__ tw) {
  using Cfg = TileCfg<L, CV, W>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  CV* smem = reinterpret_cast<CV*>(smem_raw);
  const CV* in = (const CV*)a.in;
  CV* out = (CV*)a.out;
  const int col = threadIdx.x & (W - 1);
  const int t = (threadIdx.x / W) % Cfg::T;
  const int g = threadIdx.x / Cfg::per_tile;
  const uint32_t tile = blockIdx.x * Cfg::G + g;
  const bool active = tile < a.n_outer * a.nchunk;
  const uint32_t o = active ? tile / a.nchunk : 0;
  const uint32_t z = (active ? (tile - o * a.nchunk) : 0) * W + col;
  constexpr int E = Cfg::E;
  const uint32_t obi = outer(a.lin, o) + z, obo = outer(a.lout, o) + z;
  CV v[E];
  pdl_wait();
#pragma unroll
  for (int m = 0; m < E; ++m) v[m] = active ? in[obi + inner<PIN>(a.lin, t + m * Cfg::T)] : CT<CV>::mk(0, 0);
  tile_body<L, E, KIND, KTAB, POUT>(a, v, t, o, z, active, tw, SmemStrided<CV, W>{smem + (size_t)g * L * W + col});
  pdl_trigger();
  if (active) {
    if constexpr (PEERS) {
      // fused transpose: each point goes straight into the owning rank's
      // buffer (peer memory over NVLink); the fence makes the stores visible
      // before the stream-ordered cross-rank barrier that follows the kernel
      const uint32_t mask = (1u << a.lout.lb) - 1u;
#pragma unroll
      for (int m = 0; m < E; ++m) {
        const uint32_t i = t + m * Cfg::T;
        CV* dst = (CV*)a.peers[i >> a.lout.lb];
        dst[obo + (i & mask) * a.lout.si] = v[m];
      }
      __threadfence_system();
    } else {
#pragma unroll
      for (int m = 0; m < E; ++m) out[obo + inner<POUT>(a.lout, t + m * Cfg::T)] = v[m];
    }
  }
}

// ---------------------------------------------------------------------------
// host-side dispatch
// ---------------------------------------------------------------------------


// Launch through cudaLaunchKernelEx with programmatic stream serialization
// while ctap_pdl is set (the x-slab schedule's chains of small per-slab
// grids: the next grid's launch overlaps this one's tail; every kernel
// launched this way starts with griddepcontrol.wait), else <<<>>>.
}  // namespace ctap
thread_local int ctap_pdl = 0;
namespace ctap {
template <typename K, typename... Args>
static cudaError_t launch_pdl(K k, unsigned grid, unsigned block, size_t smem, cudaStream_t st, Args... args) {
  if (!ctap_pdl) {
    k<<<grid, block, smem, st>>>(args...);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, args...);
}

template <int L, int KIND, bool VTAB, typename CV, int CH = 0, bool OBS = false>
static cudaError_t launch_z(const ZArgs& a, const TwOf<CV>* tw, cudaStream_t st) {
  using Cfg = ZCfg<L, CV>;
  auto k = zline_kernel<L, KIND, VTAB, CV, CH, OBS>;
  static std::atomic<uint64_t> attr_done{0};
  if (cudaError_t e = ctap_smem_attr(k, Cfg::smem, attr_done)) return e;
  return launch_pdl(k, (a.nlines + Cfg::C - 1) / Cfg::C, Cfg::threads, Cfg::smem, st, a, tw);
}

template <int L, int KIND, bool PIN, bool POUT, bool KTAB, typename CV, int W, bool PEERS = false>
static cudaError_t launch_tile(const TileArgs& a, const TwOf<CV>* tw, cudaStream_t st) {
  using Cfg = TileCfg<L, CV, W>;
  auto k = tile_kernel<L, KIND, PIN, POUT, KTAB, CV, W, PEERS>;
  static std::atomic<uint64_t> attr_done{0};
  if (cudaError_t e = ctap_smem_attr(k, Cfg::smem, attr_done)) return e;
  const uint32_t ntiles = a.n_outer * a.nchunk;
  return launch_pdl(k, (ntiles + Cfg::G - 1) / Cfg::G, Cfg::threads, Cfg::smem, st, a, tw);
}

#define CTAP_BY_LENGTH(L, FN)                   \
  switch (L) {                                  \
    case 8: return FN(8);                       \
    case 16: return FN(16);                     \
    case 32: return FN(32);                     \
    case 64: return FN(64);                     \
    case 128: return FN(128);                   \
    case 256: return FN(256);                   \
    case 512: return FN(512);                   \
    case 1024: return FN(1024);                 \
  }                                             \
  return cudaErrorInvalidValue;

// twiddle tables of both precisions for one line length
struct Tw {
  const double2* d;
  const float4* f;
};

template <int KIND, bool VTAB, int CH = 0>
static cudaError_t dispatch_z(int L, bool c64, const ZArgs& a, Tw tw, cudaStream_t st) {
#define CTAP_Z(LL) \
  (c64 ? launch_z<LL, KIND, VTAB, float2, CH>(a, tw.f, st) : launch_z<LL, KIND, VTAB, double2, CH>(a, tw.d, st))
  CTAP_BY_LENGTH(L, CTAP_Z)
#undef CTAP_Z
}

template <int KIND, bool PIN, bool POUT, bool KTAB, int W = 8, bool PEERS = false>
static cudaError_t dispatch_tile(int L, bool c64, const TileArgs& a, Tw tw, cudaStream_t st) {
#define CTAP_T(LL)                                                                   \
  (c64 ? launch_tile<LL, KIND, PIN, POUT, KTAB, float2, W, PEERS>(a, tw.f, st)       \
       : launch_tile<LL, KIND, PIN, POUT, KTAB, double2, W, PEERS>(a, tw.d, st))
  CTAP_BY_LENGTH(L, CTAP_T)
#undef CTAP_T
}

// z columns per strided tile at L = 1024 (CTAP_W1024): 4 (default) keeps a
// tile at 64 KB so two blocks fit per SM -- 1024^2 x 512: y passes 5.09 -> 4.17
// ms, [x K x^-1] 8.16 -> 7.70 ms against 8-column tiles (bitwise equal)
static int w1024() {
  static const int w = [] {
    const char* e = getenv("CTAP_W1024");
    return e ? atoi(e) : 4;
  }();
  return w;
}

static int ilog2(int64_t v) {
  int l = 0;
  while ((int64_t(1) << l) < v) ++l;
  return l;
}

// materialised phase factors (StepPlan.exp_v_half / exp_v_full / exp_k,
// propagator.py:45-47) for inspection, and the plan's phase tables
template <typename CV>
__global__ void phase_field_kernel(CV* __restrict__ out, const double* __restrict__ vi,
                                   const double* __restrict__ kx2, const double* __restrict__ ky2,
                                   const double* __restrict__ kz2, uint32_t nx, uint32_t ny, uint32_t nz,
                                   uint32_t x_off, uint32_t y_off, int which, int imag, double dt_i,
                                   double len2, double scale, int lx, const double2* __restrict__ sct) {
  using R = typename CT<CV>::R;
  const uint32_t n = nx * ny * nz;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double phi;
    uint32_t dst = i;
    if (which == 2) {
      const uint32_t x = i / (ny * nz), y = (i / nz) % ny, z = i % nz;
      phi = k_phase(kx2[x + x_off], ky2[y + y_off], kz2[z], len2, dt_i);
      // blocked k-space position (lx = 0: natural)
      dst = (((x >> lx) * ny + y) << lx) * nz + (x & ((1u << lx) - 1u)) * nz + z;
    } else {
      phi = v_phase_i(vi[i], which == 0 ? -0.5 : -1.0, dt_i);
    }
    if (imag) {
      out[dst] = CT<CV>::mk((R)(exp(phi) * scale), (R)0);
    } else {
      double s, c;
      fast_sincos(phi, sct, &s, &c);
      out[dst] = CT<CV>::mk((R)(c * scale), (R)(s * scale));
    }
  }
}

__global__ void v_internal_kernel(const double* __restrict__ V, double* __restrict__ vi, uint32_t n,
                                  double shift, double e0) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    vi[i] = v_internal(V[i], shift, e0);
}

template <int L>
static void append_stage_twiddles(std::vector<double>& t) {
  using P = Plan<L>;
  for (int s = 1; s < P::nstages; ++s) {
    const int R = P::radix(s), NS = P::ns(s);
    for (int r = 1; r < R; ++r)
      for (int k = 0; k < NS; ++k) {
        // extended precision so every entry is the correctly rounded double
        const long double ang = 2.0L * 3.14159265358979323846264338327950288L * (long double)(r * k) /
                                (long double)(NS * R);
        t.push_back((double)cosl(ang));
        t.push_back((double)(-sinl(ang)));
      }
  }
}

}  // namespace ctap

using namespace ctap;

// all stage-major twiddle tables, L = 8..1024; off[i] = start (in double2) of L = 8 << i
std::vector<double> ctap_make_twiddles(int off[8]) {
  std::vector<double> t;
  off[0] = (int)(t.size() / 2); append_stage_twiddles<8>(t);
  off[1] = (int)(t.size() / 2); append_stage_twiddles<16>(t);
  off[2] = (int)(t.size() / 2); append_stage_twiddles<32>(t);
  off[3] = (int)(t.size() / 2); append_stage_twiddles<64>(t);
  off[4] = (int)(t.size() / 2); append_stage_twiddles<128>(t);
  off[5] = (int)(t.size() / 2); append_stage_twiddles<256>(t);
  off[6] = (int)(t.size() / 2); append_stage_twiddles<512>(t);
  off[7] = (int)(t.size() / 2); append_stage_twiddles<1024>(t);
  if (t.empty()) t.assign(2, 0.0);
  return t;
}

cudaError_t ctap_run_v_internal(const ctap_plan* p, cudaStream_t st) {
  const uint32_t n = (uint32_t)(p->nx_local * p->ny_pos * p->n[2]);
  v_internal_kernel<<<p->red_blocks, 256, 0, st>>>(p->v_dev, p->vi_dev, n, p->v_shift, p->e0);
  return cudaGetLastError();
}

// which: 0 exp_v_half, 1 exp_v_full, 2 exp_k (natural x-slab layout),
//        3 exp_k / N in the x-pass (y-slab) layout, for the tables.
// `table`: write in the plan's precision (phase tables) instead of complex128.
template <typename CV>
static cudaError_t phase_field(const ctap_plan* p, int which, void* out, cudaStream_t st) {
  const int imag = p->mode == 1;
  if (which == 3) {
    const uint32_t nyl = (uint32_t)(p->n[1] / p->slab_p);
    phase_field_kernel<CV><<<p->red_blocks, 256, 0, st>>>(
        (CV*)out, p->vi_dev, p->k2_dev[0], p->k2_dev[1], p->k2_dev[2], (uint32_t)p->n[0], nyl,
        (uint32_t)p->n[2], 0u, (uint32_t)p->slab_r * nyl, 2, imag, p->dt_i, p->len2, p->inv_scale, p->k_lx,
        p->sctab);
  } else {
    phase_field_kernel<CV><<<p->red_blocks, 256, 0, st>>>(
        (CV*)out, p->vi_dev, p->k2_dev[0], p->k2_dev[1], p->k2_dev[2], (uint32_t)p->nx_local,
        (uint32_t)p->n[1], (uint32_t)p->n[2], (uint32_t)(p->slab_r * p->nx_local), 0u, which, imag, p->dt_i,
        p->len2, 1.0, 0, p->sctab);
  }
  return cudaGetLastError();
}

cudaError_t ctap_run_phase_field(const ctap_plan* p, int which, void* out, cudaStream_t st) {
  return phase_field<double2>(p, which, out, st);
}

cudaError_t ctap_run_phase_table(const ctap_plan* p, int which, void* out, cudaStream_t st) {
  return p->dtype == CTAP_C64 ? phase_field<float2>(p, which, out, st) : phase_field<double2>(p, which, out, st);
}

// Run one pass on the plan's local data.  `in`/`out` may alias (natural
// layouts, in place).  Returns a CUDA error code.
cudaError_t ctap_run_tma_pass(const ctap_plan* p, int axis, int kind, void* data, const TileArgs& a,
                              cudaStream_t st);
cudaError_t ctap_run_wline(const ctap_plan* p, int axis, int kind, int mode, void* data, const TileArgs& a,
                           cudaStream_t st);
cudaError_t ctap_run_wline_peers(const ctap_plan* p, const void* in, const TileArgs& a, cudaStream_t st);

static Tw twid(const ctap_plan* p, int64_t L) {
  const int off = p->tw_off[ilog2(L) - 3];
  return Tw{p->twiddles + off, p->twiddles32 + off};
}

cudaError_t ctap_run_pass_z(const ctap_plan* p, int kind, const void* in, void* out, int64_t z0, int64_t zn,
                            cudaStream_t st);

cudaError_t ctap_run_pass(const ctap_plan* p, int kind, const void* in, void* out, cudaStream_t st) {
  return ctap_run_pass_z(p, kind, in, out, 0, p->n[2], st);
}

// number of warps (= observer partials, kObsVals each) of the segment-end z pass
int64_t ctap_z_blocks(const ctap_plan* p) {
  const int64_t nlines = p->nx_local * p->n[1];
  const int T = (int)(p->n[2] / kElems);
  const int C = (CTAP_Z_THREADS / T) > 0 ? (CTAP_Z_THREADS / T) : 1;
  const int threads = C * T;
  return (nlines + C - 1) / C * ((threads + 31) / 32);
}

// The guide-partition bits of z_observe for lines of length L (T = L/8
// threads per line): the comparisons of observables.py:96-99 (xs[x] < xb1[z],
// xs[x] >= xb2[z]) evaluated once per (x, t) for the thread's 8 points.
template <int L>
__global__ void obs_mask_kernel(const double* __restrict__ xs, const double* __restrict__ xb1,
                                const double* __restrict__ xb2, uint32_t nx, uint16_t* __restrict__ mask) {
  constexpr int T = L / kElems;
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nx * T) return;
  const uint32_t x = i / T, t = i % T;
  const double xv = xs[x];
  uint32_t mk = 0;
#pragma unroll
  for (int m = 0; m < kElems; ++m) {
    const int z = t + m * T;
    if (xv < xb1[z]) mk |= 1u << m;
    if (xv >= xb2[z]) mk |= 1u << (8 + m);
  }
  mask[i] = (uint16_t)mk;
}

// u16 entries of the partition mask of a plan's fused observer pass
size_t ctap_obs_mask_entries(const ctap_plan* p) { return (size_t)p->n[0] * (p->n[2] / kElems); }

// [z^-1 . Vh] with the observer sums fused (single-GPU plans): block partials
// of [sum rho, left, middle, right, edge(margin)] into `partial`
// (ctap_z_blocks(p) x 5 doubles)
cudaError_t ctap_run_z_last_observe(const ctap_plan* p, void* psi, const double* xs, const double* xb1,
                                    const double* xb2, int margin, double* partial, uint16_t* mask,
                                    cudaStream_t st) {
  const int64_t nz = p->n[2];
  if (xb1) {
    const uint32_t n = (uint32_t)ctap_obs_mask_entries(p);
#define CTAP_OM(LL) (obs_mask_kernel<LL><<<(n + 255) / 256, 256, 0, st>>>(xs, xb1, xb2, (uint32_t)p->n[0], mask), \
                     cudaGetLastError())
    const cudaError_t e = [&]() -> cudaError_t { CTAP_BY_LENGTH(nz, CTAP_OM) }();
#undef CTAP_OM
    if (e != cudaSuccess) return e;
  }
  ZArgs a{};
  a.psi = psi;
  a.out = psi;
  a.lzc = 0;
  a.cs = 0;
  a.nlines = (uint32_t)(p->nx_local * p->n[1]);
  a.xs = xs;
  a.xb1 = xb1;
  a.xb2 = xb2;
  a.obs_partial = partial;
  a.obs_mask = xb1 ? mask : nullptr;
  a.ny = (uint32_t)p->n[1];
  a.lny = (uint32_t)ilog2(p->n[1]);
  a.nx = (uint32_t)p->n[0];
  a.margin = margin;
  PhaseArgs& ph = a.ph;
  ph.vi = p->vi_dev;
  ph.expv = p->expv_dev;
  ph.dt_i = p->dt_i;
  ph.imag = p->mode == 1;
  ph.sct = p->sctab;
  ph.sctk = p->sctab + kSCN;
  const Tw tw = twid(p, nz);
  const bool c64 = p->dtype == CTAP_C64;
#define CTAP_ZO(LL)                                                                        \
  (c64 ? launch_z<LL, T_VLAST, false, float2, 0, true>(a, tw.f, st)                         \
       : launch_z<LL, T_VLAST, false, double2, 0, true>(a, tw.d, st))
  CTAP_BY_LENGTH(nz, CTAP_ZO)
#undef CTAP_ZO
}

// A strided pass restricted to the z columns [z0, z0 + zn) (zn a multiple of
// 8): the kinetic block of the step can then run chunk by chunk with the
// chunk's data resident in L2 between its y, x and y^-1 passes.
cudaError_t ctap_run_pass_z(const ctap_plan* p, int kind, const void* in, void* out, int64_t z0, int64_t zn,
                            cudaStream_t st) {
  const int64_t nx = p->n[0], ny = p->n[1], nz = p->n[2];
  const bool zsub = z0 != 0 || zn != nz;
  const bool c64 = p->dtype == CTAP_C64;
  const size_t csz = c64 ? sizeof(float2) : sizeof(double2);
  const Tw tw_any = twid(p, 8);
  // x passes read 16-column (instead of 8) tiles when z allows it
  const bool xw16 = CTAP_XW == 16 && nz >= 16 && !zsub;
  // strided passes on natural layouts go through the TMA pipeline in
  // complex64 (CTAP_TMA=1, default); in complex128 the register-fed
  // tile_kernel measured faster (CTAP_TMA=2 adds c128 x, 3 c128 x and y;
  // DESIGN.md §4)
  static const int tma_mode = [] {
    const char* e = getenv("CTAP_TMA");
    return e ? atoi(e) : CTAP_TMA_DEFAULT;
  }();
  const bool use_tma = tma_mode != 0 && !zsub;

  const bool use_tma_x = !zsub && (tma_mode >= 2 || (tma_mode == 1 && c64));
  const int P = p->slab_p;
  const uint32_t nxl = (uint32_t)(nx / P), nyl = (uint32_t)(ny / P);
  PhaseArgs ph;
  ph.vi = p->vi_dev;
  ph.expv = p->expv_dev;
  ph.kx2 = p->k2_dev[0];
  ph.ky2 = p->k2_dev[1];
  ph.kz2 = p->k2_dev[2];
  ph.expk = p->expk_dev;
  ph.len2 = p->len2;
  ph.dt_i = p->dt_i;
  ph.scale = p->inv_scale;
  ph.imag = p->mode == 1;
  ph.outer_off = 0;
  ph.kgen = p->kgen;
  ph.sct = p->sctab;
  ph.sctk = p->sctab + kSCN;
  ph.z_off = (uint32_t)z0;
  for (int i = 0; i < 3; ++i) {
    ph.kn[i] = (uint32_t)p->n[i];
    ph.kval[i] = p->kval[i];
  }

  if (kind >= PASS_PZ_FIRST && kind <= PASS_PX_KIN) {  // pencil decomposition (include/ctap.h)
    if (!p->pen_c || zsub) return cudaErrorInvalidValue;
    const uint32_t Pr = (uint32_t)p->pen_r, Pc = (uint32_t)p->pen_c;
    const uint32_t xa = (uint32_t)p->nx_local, yb = (uint32_t)(ny / Pc), yd = (uint32_t)(ny / Pr);
    const uint32_t zc = (uint32_t)(nz / Pc);
    if (kind <= PASS_PZ_LAST) {
      ZArgs a;
      a.psi = const_cast<void*>(in);
      a.out = out;
      a.nlines = xa * yb;
      a.ph = ph;
      a.lzc = (uint32_t)ilog2(zc);
      a.cs = a.nlines * zc;
      const Tw tw = twid(p, nz);
      {  // two-stage z kernel (ctap_zline2.cu) where it applies
        const int tk = kind == PASS_PZ_FIRST ? T_VFIRST : kind == PASS_PZ_MID ? T_VMID : T_VLAST;
        cudaError_t e = ctap_run_z2(p, tk, false, kind == PASS_PZ_FIRST ? 2 : kind == PASS_PZ_MID ? 3 : 1, a, st);
        if (e != cudaErrorNotSupported) return e;
      }
      if (kind == PASS_PZ_FIRST) return dispatch_z<T_VFIRST, false, 2>((int)nz, c64, a, tw, st);
      if (kind == PASS_PZ_MID) return dispatch_z<T_VMID, false, 3>((int)nz, c64, a, tw, st);
      return dispatch_z<T_VLAST, false, 1>((int)nz, c64, a, tw, st);
    }
    constexpr int kNone = 31;
    TileArgs a;
    a.in = in;
    a.out = out;
    a.nchunk = zc / 8;
    a.ph = ph;
    if (kind == PASS_PX_KIN) {  // natural (nx, ny/Pr, nz/Pc): ky offset a ny/Pr, kz offset b nz/Pc
      a.n_outer = yd;
      a.lin = a.lout = Layout{zc, 0u, yd * zc, 0, 0u, kNone};
      a.ph.outer_off = (uint32_t)p->pen_a * yd;
      a.ph.z_off = (uint32_t)p->pen_b * zc;
      if (in == out) {
        cudaError_t e = ctap_run_wline(p, 2, T_KIN, p->wline, out, a, st);
        if (e != cudaErrorNotSupported) return e;
      }
      return dispatch_tile<T_KIN, false, false, false>((int)nx, c64, a, twid(p, nx), st);
    }
    // y passes between the row-exchange layout Yb = [b'][x][y % yb][z'] and
    // the column-exchange layout Xp = [a'][x][y % yd][z'] (blocked by y)
    a.n_outer = xa;
    const Layout yblk{yb * zc, xa * yb * zc, zc, ilog2(yb), 0u, kNone};
    const Layout xblk{yd * zc, xa * yd * zc, zc, ilog2(yd), 0u, kNone};
    if (kind == PASS_PY_FWD) {
      a.lin = yblk;
      a.lout = xblk;
      return dispatch_tile<T_FWD, true, true, false>((int)ny, c64, a, twid(p, ny), st);
    }
    a.lin = xblk;
    a.lout = yblk;
    return dispatch_tile<T_INV, true, true, false>((int)ny, c64, a, twid(p, ny), st);
  }
  if (kind >= PASS_Z_FWD && kind <= PASS_Z_LAST) {
    if (in != out) return cudaErrorInvalidValue;
    ZArgs a;
    a.psi = out;
    a.out = out;
    a.lzc = 0;
    a.cs = 0;
    a.nlines = (uint32_t)(p->nx_local * ny);
    a.ph = ph;
    const Tw tw = twid(p, nz);
    const int L = (int)nz;
    {  // two-stage z kernel (ctap_zline2.cu) where it applies
      const int tk = kind == PASS_Z_FWD ? T_FWD : kind == PASS_Z_INV ? T_INV : kind == PASS_Z_FIRST ? T_VFIRST
                     : kind == PASS_Z_MID ? T_VMID : T_VLAST;
      cudaError_t e = ctap_run_z2(p, tk, p->expv_dev != nullptr, 0, a, st);
      if (e != cudaErrorNotSupported) return e;
    }
    switch (kind) {
      case PASS_Z_FWD: return dispatch_z<T_FWD, false>(L, c64, a, tw, st);
      case PASS_Z_INV: return dispatch_z<T_INV, false>(L, c64, a, tw, st);
      case PASS_Z_FIRST: return dispatch_z<T_VFIRST, false>(L, c64, a, tw, st);
      case PASS_Z_MID:
        return p->expv_dev ? dispatch_z<T_VMID, true>(L, c64, a, tw, st) : dispatch_z<T_VMID, false>(L, c64, a, tw, st);
      case PASS_Z_LAST: return dispatch_z<T_VLAST, false>(L, c64, a, tw, st);
    }
    return cudaErrorInvalidValue;
  }
  if (zsub && (kind < PASS_Y_FWD || kind > PASS_X_INV || (zn & 7) || z0 < 0 || z0 + zn > nz))
    return cudaErrorInvalidValue;
  TileArgs a;
  a.in = (const char*)in + csz * (size_t)z0;
  a.out = (char*)out + csz * (size_t)z0;
  a.nchunk = (uint32_t)(zn / 8);
  a.ph = ph;
  const uint32_t NZ = (uint32_t)nz, NY = (uint32_t)ny;
  constexpr int kNone = 31;  // no outer blocking
  // natural x-slab layout (x_local, y, z), y-pass view (o = x_local, i = y)
  const Layout y_nat{NY * NZ, 0u, NZ, 0, 0u, kNone};
  // peer-major [peer][x_local][y_local][z] (slab transpose buffers)
  const Layout y_peer{nyl * NZ, nxl * nyl * NZ, NZ, ilog2(nyl), 0u, kNone};
  // natural y-slab layout (x, y_local, z), x-pass view (o = y_local, i = x)
  const Layout x_nat{NZ, 0u, nyl * NZ, 0, 0u, kNone};
  // blocked k-space layout of the single-GPU step, B(x, y, z) =
  //   ((x >> lx) ny + y) XL nz + (x & (XL-1)) nz + z,  XL = 2^lx:
  // x-lines then span nx/XL TLB pages instead of nx
  const int lx = p->k_lx;
  const uint32_t XL = 1u << lx;
  const Layout y_blk{NZ, 0u, XL * NZ, 0, NY * XL * NZ, lx};    // y-pass view
  const Layout x_blk{XL * NZ, NY * XL * NZ, NZ, lx, 0u, kNone};  // x-pass view
  const bool peer = P > 1;
  switch (kind) {
    case PASS_Y_FWD_TO_PEERS: {
      // y FFT of the x-slab; point (x_local, y, z) lands in rank q = y / ny_local
      // at ((r nx_local + x_local) ny_local + y % ny_local) nz + z
      a.n_outer = nxl;
      a.lin = y_nat;
      a.lout = Layout{nyl * NZ, 0u, NZ, ilog2(nyl), 0u, kNone};
      for (int q = 0; q < P; ++q)
        a.peers[q] = (char*)p->peer_y[q] + csz * (size_t)p->slab_r * nxl * nyl * NZ;
      return dispatch_tile<T_FWD, false, true, false, 8, true>((int)ny, c64, a, twid(p, ny), st);
    }
    case PASS_X_KIN_TO_PEERS: {
      // [x K x^-1] of the y-slab; point (x, y_local, z) lands in rank q = x / nx_local
      // at r (nx_local ny_local nz) + (x % nx_local) ny_local nz + y_local nz + z
      a.n_outer = nyl;
      a.lin = x_nat;
      a.lout = Layout{NZ, 0u, nyl * NZ, ilog2(nxl), 0u, kNone};
      a.ph.outer_off = (uint32_t)p->slab_r * nyl;
      for (int q = 0; q < P; ++q)
        a.peers[q] = (char*)p->peer_p[q] + csz * (size_t)p->slab_r * nxl * nyl * NZ;
      if (!zsub && !p->expk_dev) {  // warp-per-line ring, TMA stores into the peers (ctap_wline.cu)
        cudaError_t e = ctap_run_wline_peers(p, a.in, a, st);
        if (e != cudaErrorNotSupported) return e;
      }
      return dispatch_tile<T_KIN, false, true, false, 8, true>((int)nx, c64, a, twid(p, nx), st);
    }
    case PASS_Y_FWD_BLK:
    case PASS_Y_INV_BLK: {
      a.n_outer = nxl;
      const Tw tw = twid(p, ny);
      if (kind == PASS_Y_FWD_BLK) {
        a.lin = y_nat;
        a.lout = y_blk;
        return dispatch_tile<T_FWD, false, false, false>((int)ny, c64, a, tw, st);
      }
      a.lin = y_blk;
      a.lout = y_nat;
      return dispatch_tile<T_INV, false, false, false>((int)ny, c64, a, tw, st);
    }
    case PASS_X_KIN_BLK: {
      a.lin = x_blk;
      a.lout = x_blk;
      a.n_outer = NY;
      const Tw tw = twid(p, nx);
      return p->expk_dev ? dispatch_tile<T_KIN, true, true, true>((int)nx, c64, a, tw, st)
                         : dispatch_tile<T_KIN, true, true, false>((int)nx, c64, a, tw, st);
    }
    case PASS_Y_FWD:
    case PASS_Y_INV:
    case PASS_Y_FWD_TO_PEER:
    case PASS_Y_INV_FROM_PEER: {
      a.n_outer = nxl;
      const Tw tw = twid(p, ny);
      const int L = (int)ny;
      if (kind == PASS_Y_FWD_TO_PEER && peer) {
        a.lin = y_nat;
        a.lout = y_peer;
        return dispatch_tile<T_FWD, false, true, false>(L, c64, a, tw, st);
      }
      if (kind == PASS_Y_INV_FROM_PEER && peer) {
        a.lin = y_peer;
        a.lout = y_nat;
        return dispatch_tile<T_INV, true, false, false>(L, c64, a, tw, st);
      }
      a.lin = y_nat;
      a.lout = y_nat;
      const bool fwd = (kind == PASS_Y_FWD || kind == PASS_Y_FWD_TO_PEER);
      if (L == 1024 && !c64 && !zsub && in == out && p->wline) {
        // 1024-point y lines: warp-per-line ring (4-column tiles, two warps
        // per column) -- 2.85 vs 4.25 ms at 1024^2 x 512 (ctap_wline.cu)
        cudaError_t e = ctap_run_wline(p, 1, fwd ? T_FWD : T_INV, p->wline, out, a, st);
        if (e != cudaErrorNotSupported) return e;
      }
      if (L == 1024 && w1024() == 4 && !zsub && nz % 4 == 0) {  // 4-column tiles (64 KB): 2 blocks per SM
        a.nchunk = (uint32_t)(nz / 4);
        if (c64) return fwd ? launch_tile<1024, T_FWD, false, false, false, float2, 4>(a, tw.f, st)
                            : launch_tile<1024, T_INV, false, false, false, float2, 4>(a, tw.f, st);
        return fwd ? launch_tile<1024, T_FWD, false, false, false, double2, 4>(a, tw.d, st)
                   : launch_tile<1024, T_INV, false, false, false, double2, 4>(a, tw.d, st);
      }
      if (use_tma && (c64 || tma_mode == 3) && in == out) {  // measured: faster for complex64 only
        cudaError_t e = ctap_run_tma_pass(p, 1, fwd ? T_FWD : T_INV, out, a, st);
        if (e != cudaErrorNotSupported) return e;
      }
      return fwd ? dispatch_tile<T_FWD, false, false, false>(L, c64, a, tw, st)
                 : dispatch_tile<T_INV, false, false, false>(L, c64, a, tw, st);
    }
    case PASS_Y_COPY:
      a.n_outer = nxl;
      a.lin = y_nat;
      a.lout = y_nat;
      return dispatch_tile<T_COPY, false, false, false>((int)ny, c64, a, tw_any, st);
    case PASS_X_COPY:
      a.n_outer = nyl;
      a.lin = x_nat;
      a.lout = x_nat;
      if (xw16) {
        a.nchunk = (uint32_t)(nz / 16);
        return dispatch_tile<T_COPY, false, false, false, 16>((int)nx, c64, a, tw_any, st);
      }
      return dispatch_tile<T_COPY, false, false, false>((int)nx, c64, a, tw_any, st);
    case PASS_XP_COPY:
    case PASS_XP_KIN: {  // diagnostics: x pass with a padded x pitch
      static const uint32_t pad = [] {
        const char* e = getenv("CTAP_XPAD");
        return (uint32_t)(e ? atoi(e) : 0);
      }();
      a.n_outer = nyl;
      a.lin = a.lout = Layout{NZ, 0u, nyl * NZ + pad, 0, 0u, kNone};
      a.ph.outer_off = (uint32_t)p->slab_r * nyl;
      if (kind == PASS_XP_COPY) return dispatch_tile<T_COPY, false, false, false>((int)nx, c64, a, tw_any, st);
      return dispatch_tile<T_KIN, false, false, false>((int)nx, c64, a, twid(p, nx), st);
    }
    case PASS_WX_COPY:
    case PASS_WY_COPY:
    case PASS_WY_FWD: {  // diagnostics: the warp-per-line TMA pipeline on x / y lines
      if (in != out) return cudaErrorInvalidValue;
      const bool xa = kind == PASS_WX_COPY;
      a.lin = a.lout = xa ? x_nat : y_nat;
      a.n_outer = xa ? nyl : nxl;
      a.ph.outer_off = xa ? (uint32_t)p->slab_r * nyl : 0u;
      return ctap_run_wline(p, xa ? 2 : 1, kind == PASS_WY_FWD ? T_FWD : T_COPY, p->wline == 2 ? 2 : 1, out, a, st);
    }
    case PASS_XB_COPY: {  // diagnostics: x-pass traffic on the x-blocked layout, block 16
      const int dlx = 4;
      const uint32_t DL = 1u << dlx;
      const Layout xb{DL * NZ, NY * DL * NZ, NZ, dlx, 0u, kNone};
      a.n_outer = NY;
      a.lin = xb;
      a.lout = xb;
      return dispatch_tile<T_COPY, true, true, false>((int)nx, c64, a, tw_any, st);
    }
    case PASS_X_KIN:
    case PASS_X_FWD:
    case PASS_X_INV: {
      a.lin = x_nat;
      a.lout = x_nat;
      a.n_outer = nyl;
      a.ph.outer_off = (uint32_t)p->slab_r * nyl;
      const Tw tw = twid(p, nx);
      const int L = (int)nx;
      if (kind == PASS_X_KIN && !c64 && (!zsub || nx <= 512) && in == out && !p->expk_dev) {
        // warp-per-line TMA pipeline (ctap_wline.cu): the default complex128 x pass
        const int tk = kind == PASS_X_KIN ? T_KIN : kind == PASS_X_FWD ? T_FWD : T_INV;
        cudaError_t e = ctap_run_wline(p, 2, tk, p->wline, a.out, a, st);  // a.out: offset to the z chunk
        if (e != cudaErrorNotSupported) return e;
      }
      if (use_tma_x && in == out && !(kind == PASS_X_KIN && p->expk_dev)) {
        const int tk = kind == PASS_X_KIN ? T_KIN : kind == PASS_X_FWD ? T_FWD : T_INV;
        cudaError_t e = ctap_run_tma_pass(p, 2, tk, out, a, st);
        if (e != cudaErrorNotSupported) return e;
      }
      if (L == 1024 && w1024() == 4 && kind == PASS_X_KIN && !p->expk_dev && !zsub && nz % 4 == 0) {
        a.nchunk = (uint32_t)(nz / 4);
        return c64 ? launch_tile<1024, T_KIN, false, false, false, float2, 4>(a, tw.f, st)
                   : launch_tile<1024, T_KIN, false, false, false, double2, 4>(a, tw.d, st);
      }
      if (xw16) {  // 16-column tiles: 256-byte rows for the large-stride x lines
        a.nchunk = (uint32_t)(nz / 16);
        if (kind == PASS_X_KIN)
          return p->expk_dev && p->k_lx == 0 ? dispatch_tile<T_KIN, false, false, true, 16>(L, c64, a, tw, st)
                                             : dispatch_tile<T_KIN, false, false, false, 16>(L, c64, a, tw, st);
        if (kind == PASS_X_FWD) return dispatch_tile<T_FWD, false, false, false, 16>(L, c64, a, tw, st);
        return dispatch_tile<T_INV, false, false, false, 16>(L, c64, a, tw, st);
      }
      if (kind == PASS_X_KIN)
        return p->expk_dev && p->k_lx == 0 ? dispatch_tile<T_KIN, false, false, true>(L, c64, a, tw, st)
                                           : dispatch_tile<T_KIN, false, false, false>(L, c64, a, tw, st);
      if (kind == PASS_X_FWD) return dispatch_tile<T_FWD, false, false, false>(L, c64, a, tw, st);
      return dispatch_tile<T_INV, false, false, false>(L, c64, a, tw, st);
    }
  }
  return cudaErrorInvalidValue;
}

// Slab kinetic block by z chunks (the overlapped NCCL transport): the passes
// of one chunk of zn columns [z0, z0 + zn) with CHUNK-MAJOR transpose
// buffers, so each chunk's all-to-all moves contiguous per-peer blocks and can
// run while the next chunk's pass computes (z is untouched by y, x and the
// kinetic factor, so chunks are independent through the block):
//   Y_FWD_TO_PEER   psi columns [z0, z0 + zn) -> send chunk [peer][x_l][y_l][zn]
//   X_KIN           recv chunk (nx, y_l, zn) in place, kz offset z0
//   Y_INV_FROM_PEER send chunk [peer][x_l][y_l][zn] -> psi columns [z0, z0 + zn)
// The per-line arithmetic is the unchunked passes', so results are bitwise
// equal to them (tests/test_gpu_slab_virtual.py).
cudaError_t ctap_run_pass_chunk(const ctap_plan* p, int kind, const void* in, void* out, int64_t z0, int64_t zn,
                                cudaStream_t st) {
  const int64_t nx = p->n[0], ny = p->n[1], nz = p->n[2];
  const int P = p->slab_p;
  if (P < 2 || p->pen_c || zn <= 0 || (zn & 7) || z0 < 0 || z0 + zn > nz) return cudaErrorInvalidValue;
  const bool c64 = p->dtype == CTAP_C64;
  const size_t csz = c64 ? sizeof(float2) : sizeof(double2);
  const uint32_t nxl = (uint32_t)(nx / P), nyl = (uint32_t)(ny / P);
  const uint32_t NZ = (uint32_t)nz, NY = (uint32_t)ny, ZN = (uint32_t)zn;
  constexpr int kNone = 31;
  TileArgs a;
  a.nchunk = ZN / 8;
  PhaseArgs& ph = a.ph;
  ph.vi = p->vi_dev;
  ph.expv = p->expv_dev;
  ph.kx2 = p->k2_dev[0];
  ph.ky2 = p->k2_dev[1];
  ph.kz2 = p->k2_dev[2];
  ph.expk = nullptr;
  ph.len2 = p->len2;
  ph.dt_i = p->dt_i;
  ph.scale = p->inv_scale;
  ph.imag = p->mode == 1;
  ph.outer_off = 0;
  ph.kgen = p->kgen;
  ph.sct = p->sctab;
  ph.sctk = p->sctab + kSCN;
  ph.z_off = (uint32_t)z0;
  for (int i = 0; i < 3; ++i) {
    ph.kn[i] = (uint32_t)p->n[i];
    ph.kval[i] = p->kval[i];
  }
  const Layout y_nat{NY * NZ, 0u, NZ, 0, 0u, kNone};
  const Layout y_peer_c{nyl * ZN, nxl * nyl * ZN, ZN, ilog2(nyl), 0u, kNone};
  const Layout x_nat_c{ZN, 0u, nyl * ZN, 0, 0u, kNone};
  switch (kind) {
    case PASS_Y_FWD_TO_PEER:
      a.in = (const char*)in + csz * (size_t)z0;
      a.out = out;
      a.n_outer = nxl;
      a.lin = y_nat;
      a.lout = y_peer_c;
      return dispatch_tile<T_FWD, false, true, false>((int)ny, c64, a, twid(p, ny), st);
    case PASS_Y_INV_FROM_PEER:
      a.in = in;
      a.out = (char*)out + csz * (size_t)z0;
      a.n_outer = nxl;
      a.lin = y_peer_c;
      a.lout = y_nat;
      return dispatch_tile<T_INV, true, false, false>((int)ny, c64, a, twid(p, ny), st);
    case PASS_X_KIN: {
      if (in != out || p->expk_dev) return cudaErrorInvalidValue;
      a.in = in;
      a.out = out;
      a.n_outer = nyl;
      a.lin = a.lout = x_nat_c;
      a.ph.outer_off = (uint32_t)p->slab_r * nyl;
      if (!c64) {
        cudaError_t e = ctap_run_wline(p, 2, T_KIN, p->wline, out, a, st);
        if (e != cudaErrorNotSupported) return e;
      }
      return dispatch_tile<T_KIN, false, false, false>((int)nx, c64, a, twid(p, nx), st);
    }
  }
  return cudaErrorInvalidValue;
}
