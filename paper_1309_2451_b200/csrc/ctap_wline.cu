// Warp-per-line strided passes (complex128): the [x K x^-1] sweep of the
// single-GPU step and the plain x (and, for diagnostics, y) FFT passes.
//
// Reference: propagator.py:98-107 (_advance) -- forward x FFT,
// exp(-i k^2 dt/2)/N, inverse x FFT of one telescoped step -- and the x FFTs
// of the 3D transform (ctap_fft3d).
//
// Why a second strided kernel: tile_kernel (ctap_passes.cu) spreads each
// 512-point column over 64 threads of a 512-thread block, so every radix
// exchange is a 16-warp __syncthreads; the x pass measured 1.43 ms at 512^3
// with the FP64 pipe ~40 % and DRAM ~34 % busy.  Here ONE WARP OWNS ONE
// COLUMN (E = L/32 points per lane, L = 256 or 512):
//   * every FFT exchange is warp-private, in place in the column's own slots
//     of the shared tile, synchronised by __syncwarp only;
//   * the tile is stored with a 128-byte XOR swizzle (element i of column c in
//     row i, 16-byte chunk c ^ (i & 7)) and the exchange index is further
//     permuted by sigma(e) = e ^ ((e >> 3) & 7), which makes the column reads
//     and every radix-8 scatter/gather bank-conflict free;
//   * the kinetic factor is symmetric in kx (k^2 of index i and L - i are
//     bitwise equal) and the mirror of lane t's point t + 32 m is held by lane
//     32 - t of the same warp: each lane evaluates the exact phase and its
//     sincos for half of its points and receives the other half by shuffle.
// Two tile movers (plan->wline, env CTAP_WLINE; DESIGN.md §4 has the measurements):
//   1 (ring)  persistent CTA per SM, 2 compute groups of 8 warps, a ring of 3
//             tile buffers filled and drained by TMA (cp.async.bulk.tensor,
//             hardware 128-byte swizzle); the last warp to finish a tile
//             stores it and refills the buffer;
//   2 (tile)  one tile per 256-thread CTA, 2 CTAs per SM, rows moved through
//             registers with coalesced 16-byte loads/stores (as tile_kernel).
// Arithmetic is identical to tile_kernel's (same radix plan and twiddles, same
// phase recipe and rotation), so the kernels are bitwise interchangeable
// (tests/test_gpu_parity.py::test_wline_bitwise_equals_tile_kernel).
#include <cuda.h>

#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "ctap_device.cuh"
#include "ctap_internal.h"
#include "ctap_tile.cuh"

namespace ctap {
namespace wl {

constexpr int kCols = 8;    // columns (lines) per tile, one warp each
#ifndef CTAP_WL_GROUPS
#define CTAP_WL_GROUPS 2
#endif
constexpr int kGroups = CTAP_WL_GROUPS;  // ring: tiles in computation at once
constexpr int kBufs = 3;    // ring: tile buffers
constexpr int kRingThreads = kGroups * kCols * 32;  // 2 groups: 16 warps, 4 per SM sub-partition, 128 registers each
constexpr int kTileThreads = kCols * 32;
// TMA box height (rows per cp.async.bulk.tensor request) and L2 promotion of
// the ring's tensor maps (A/B switches; 256 rows and 256-byte promotion by default)
#ifndef CTAP_WL_BOX
#define CTAP_WL_BOX 256
#endif
constexpr int kBoxRows = CTAP_WL_BOX;
#ifndef CTAP_WL_PROMO
#define CTAP_WL_PROMO 3
#endif
constexpr CUtensorMapL2promotion kL2Promo = (CUtensorMapL2promotion)CTAP_WL_PROMO;
// full/done mbarriers + fill counters of the ring, padded to 16 bytes
constexpr size_t kRingBarBytes = ((2 * kBufs * sizeof(uint64_t) + kBufs * sizeof(uint32_t)) + 15) / 16 * 16;
#ifndef CTAP_FFT512
#define CTAP_FFT512 1
#endif
constexpr bool kFft512 = CTAP_FFT512 != 0;  // specialised 512-point warp transform (fft512_warp)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void bar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void bar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WL_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WL_WAIT_%=;\n"
      "}\n" ::"r"(su32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
      "[%2];" ::"r"(su32(dst)),
      "l"(map), "r"(su32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tma_store(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(map),
               "r"(su32(src)), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Column c of a [row][W] complex128 tile with the TMA XOR swizzle of its row
// width (W = 8: 128-byte rows, CU_TENSOR_MAP_SWIZZLE_128B, 16-byte chunk
// c ^ (i & 7); W = 4: 64-byte rows, SWIZZLE_64B, chunk c ^ ((i >> 1) & 3)) on a
// 1 KB aligned buffer.  Either way the bank group of element i is a bijection
// of i & 7, so 8 consecutive rows never conflict, and at(e) -- the FFT
// exchange view permuted by sigma(e) = e ^ ((e >> 3) & 7) -- keeps every
// radix-8 scatter and gather conflict free.
template <int W = 8>
struct SwzColT {
  double2* buf;
  int c;
  __device__ __forceinline__ double2& nat(int i) const {
    return W == 8 ? buf[i * 8 + (c ^ (i & 7))] : buf[i * 4 + (c ^ ((i >> 1) & 3))];
  }
  __device__ __forceinline__ double2& at(int e) const { return nat(e ^ ((e >> 3) & 7)); }
};
using SwzCol = SwzColT<8>;

// exp(-i k^2 dt/2)/N (real time: (cos, sin); imaginary time: (decay, 0)),
// the recipe of mul_kphase (ctap_tile.cuh)
template <typename LD = LdgLoad>
__device__ __forceinline__ double2 kfactor(double kx2, double ky2, double kz2, const PhaseArgs& a,
                                           const double2* sctk) {
  const double phi = k_phase(kx2, ky2, kz2, a.len2, a.dt_i);
  if (a.imag) return make_double2(exp(phi) * a.scale, 0.0);
  double s, c;
  fast_sincos<LD>(phi, sctk, &s, &c);
  return make_double2(c, s);
}
__device__ __forceinline__ double2 kfactor(double kx2, double ky2, double kz2, const PhaseArgs& a) {
  return kfactor<LdgLoad>(kx2, ky2, kz2, a, a.sctk);
}
__device__ __forceinline__ void apply_k(double2& v, double2 f, int imag) {
  if (imag) dscale(v, f.x);
  else rotate(v, f.x, f.y);
}
__device__ __forceinline__ double kx2_of(uint32_t i, const PhaseArgs& a) {
  return a.kgen ? k2_gen(i, a.kn[0], a.kval[0]) : __ldg(&a.kx2[i]);
}
__device__ __forceinline__ double2 shfl2(double2 v, int src) {
  return make_double2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}

// The 512-point transform of one warp (16 points per lane) with the exchange
// addresses of the swizzled, sigma-permuted column precomputed per lane: the
// same stages, twiddles and butterflies as line_fft<512, DIR, 16> (bitwise
// equal), without the generic per-access index arithmetic.  In 16-byte units,
// with l7 = lane & 7 and u = r ^ l7, T(r) = 8 u + (c ^ u):
//   stage-0 scatter (NS = 1): 64 j + T(r),                  j = lane + 32 b
//   stage-1 scatter (NS = 8): 512 (j >> 3) + 64 r + T(r)
//   gathers of e = lane + 32 m: 256 m + R(m & 1), R(p) = 8 S + (c ^ (S & 7)),
//                               S = lane ^ ((lane >> 3) + 4 p)
template <int DIR, typename LD = LdgLoad>
__device__ __forceinline__ void fft512_warp(double2 (&v)[16], int lane, int c, const double2* __restrict__ tw,
                                            double2* buf) {
  using P = Plan<512, 16>;
  const int l7 = lane & 7;
  const int s0 = lane ^ (lane >> 3), s1 = lane ^ ((lane >> 3) + 4);
  const double2* rd0 = buf + 8 * s0 + (c ^ (s0 & 7));
  const double2* rd1 = buf + 8 * s1 + (c ^ (s1 & 7));
  // T(r) = 8 u + (c ^ u) with u = r ^ l7; the two terms occupy disjoint bits,
  // so T(r) = (9 r) ^ (9 l7 ^ c): one XOR with an immediate per scatter
  const int tk = (9 * l7) ^ c;
  auto toff = [&](int r) { return (9 * r) ^ tk; };
  auto gather = [&]() {
    __syncwarp();
#pragma unroll
    for (int m = 0; m < 16; ++m) v[m] = (m & 1 ? rd1 : rd0)[256 * m];
    __syncwarp();
  };
  // stage 0: radix 8, NS = 1 (no twiddles)
#pragma unroll
  for (int b = 0; b < 2; ++b) {
    double2 u[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) u[r] = v[b + 2 * r];
    Dft<8, DIR>::run(u);
    double2* wb = buf + 64 * lane + 2048 * b;
#pragma unroll
    for (int r = 0; r < 8; ++r) wb[toff(r)] = u[r];
  }
  gather();
  // stage 1: radix 8, NS = 8, k = j & 7 = l7
#pragma unroll
  for (int b = 0; b < 2; ++b) {
    double2 u[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) u[r] = v[b + 2 * r];
    radix8_twiddles<DIR, LD>(u, tw + P::tw_offset(1) + l7, 8);
    Dft<8, DIR>::run(u);
    double2* wb = buf + 512 * ((lane >> 3) + 4 * b);
#pragma unroll
    for (int r = 0; r < 8; ++r) wb[64 * r + toff(r)] = u[r];
  }
  gather();
  // stage 2 (last): radix 8, NS = 64, k = j = lane + 32 b; outputs stay in registers
#pragma unroll
  for (int b = 0; b < 2; ++b) {
    double2 u[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) u[r] = v[b + 2 * r];
    const int k = lane + 32 * b;
    radix8_twiddles<DIR, LD>(u, tw + P::tw_offset(2) + k, 64);
    Dft<8, DIR>::run(u);
#pragma unroll
    for (int r = 0; r < 8; ++r) v[b + 2 * r] = u[r];
  }
}

template <int L, int DIR, typename LD = LdgLoad>
__device__ __forceinline__ void warp_fft(double2 (&v)[L / 32], int lane, const double2* __restrict__ tw,
                                         const SwzCol& col) {
  if constexpr (L == 512 && kFft512) {
    fft512_warp<DIR, LD>(v, lane, col.c, tw, col.buf);
  } else {
    static_assert(std::is_same<LD, LdgLoad>::value, "shared-memory tables: 512-point warp transform only");
    line_fft<L, DIR, L / 32>(v, lane, tw, col, SyncWarp{});
  }
}

// The warp's column: read (natural order), transform, write back.  o = outer
// index (y of the x pass), z = the column's global z.
template <int L, int KIND, typename LD = LdgLoad>
__device__ __forceinline__ void column(const SwzCol& col, int lane, const double2* __restrict__ tw,
                                       const PhaseArgs& ph, uint32_t o, uint32_t z,
                                       const double2* sctk = nullptr) {
  if constexpr (std::is_same<LD, LdgLoad>::value) sctk = ph.sctk;
  constexpr int E = L / 32;
  // element lane + 32 m of the column: row lane + 32 m, chunk c ^ (lane & 7)
  double2* const nb = col.buf + 8 * lane + (col.c ^ (lane & 7));
  double2 v[E];
#pragma unroll
  for (int m = 0; m < E; ++m) v[m] = nb[256 * m];
  __syncwarp();
  if constexpr (KIND == T_COPY) {  // diagnostics: the tile mover alone
  } else if constexpr (KIND == T_FWD) {
    warp_fft<L, -1, LD>(v, lane, tw, col);
  } else if constexpr (KIND == T_INV) {
    warp_fft<L, +1, LD>(v, lane, tw, col);
  } else {  // T_KIN
    double ky2, kz2;
    if (ph.kgen) {
      ky2 = k2_gen(ph.outer_off + o, ph.kn[1], ph.kval[1]);
      kz2 = k2_gen(ph.z_off + z, ph.kn[2], ph.kval[2]);
    } else {
      ky2 = __ldg(&ph.ky2[ph.outer_off + o]);
      kz2 = __ldg(&ph.kz2[ph.z_off + z]);
    }
    warp_fft<L, -1, LD>(v, lane, tw, col);
    // Lane t evaluates the factor of its point t + 32 q (q < E/2, index <
    // L/2).  Its point m = E - q has index L - ((32 - t) + 32 (q - 1)), the
    // mirror of lane 32 - t's point of iteration q - 1, received by shuffle;
    // lane 0 (indices 32 m, self-mirrored at 0 and L/2) uses its own factor of
    // index 32 q for m = E - q and evaluates index L/2 at the end.
    const int mirror = (32 - lane) & 31;
    double2 shp = make_double2(0.0, 0.0);
#pragma unroll
    for (int q = 0; q < E / 2; ++q) {
      const double2 f = kfactor<LD>(kx2_of(lane + 32 * q, ph), ky2, kz2, ph, sctk);
      apply_k(v[q], f, ph.imag);
      if (q >= 1) apply_k(v[E - q], lane == 0 ? f : shp, ph.imag);
      shp = shfl2(f, mirror);
    }
    const double2 fn = kfactor<LD>(kx2_of(L / 2, ph), ky2, kz2, ph, sctk);
    apply_k(v[E / 2], lane == 0 ? fn : shp, ph.imag);
    warp_fft<L, +1, LD>(v, lane, tw, col);
  }
#pragma unroll
  for (int m = 0; m < E; ++m) nb[256 * m] = v[m];
}

// The same transform with TWO warps per column (64 threads, E = L/64 points
// each, named barrier per column): the ring then computes one tile with all
// 16 warps while two tiles load.  The kx-mirror factors cross the two warps,
// so they are exchanged through the column's own slots (indices < L/2,
// free between the transforms).
template <int L, int KIND, typename Col>
__device__ __forceinline__ void column2(const Col& col, int ct, const double2* __restrict__ tw,
                                        const PhaseArgs& ph, uint32_t o, uint32_t z, SyncNamed sync) {
  constexpr int E = L / 64;
  static_assert(E >= 8, "two warps per column need L >= 512 (radix-8 stages)");
  double2 v[E];
#pragma unroll
  for (int m = 0; m < E; ++m) v[m] = col.nat(ct + 64 * m);
  sync();
  if constexpr (KIND == T_COPY) {
  } else if constexpr (KIND == T_FWD) {
    line_fft<L, -1, E>(v, ct, tw, col, sync);
  } else if constexpr (KIND == T_INV) {
    line_fft<L, +1, E>(v, ct, tw, col, sync);
  } else {  // T_KIN
    double ky2, kz2;
    if (ph.kgen) {
      ky2 = k2_gen(ph.outer_off + o, ph.kn[1], ph.kval[1]);
      kz2 = k2_gen(ph.z_off + z, ph.kn[2], ph.kval[2]);
    } else {
      ky2 = __ldg(&ph.ky2[ph.outer_off + o]);
      kz2 = __ldg(&ph.kz2[ph.z_off + z]);
    }
    line_fft<L, -1, E>(v, ct, tw, col, sync);
    // factors of this thread's points below L/2, published in their slots
#pragma unroll
    for (int m = 0; m < E / 2; ++m) {
      const double2 f = kfactor(kx2_of(ct + 64 * m, ph), ky2, kz2, ph);
      col.nat(ct + 64 * m) = f;
      apply_k(v[m], f, ph.imag);
    }
    // index L/2 (thread 0's self-mirrored point m = E/2): warp 0 only
    double2 fn = make_double2(0.0, 0.0);
    if (ct < 32) fn = kfactor(kx2_of(L / 2, ph), ky2, kz2, ph);
    sync();
#pragma unroll
    for (int m = E / 2; m < E; ++m) {
      const int idx = L - (ct + 64 * m);  // the mirror point, < L/2 except ct = 0, m = E/2
      apply_k(v[m], idx == L / 2 ? fn : col.nat(idx), ph.imag);
    }
    sync();
    line_fft<L, +1, E>(v, ct, tw, col, sync);
  }
#pragma unroll
  for (int m = 0; m < E; ++m) col.nat(ct + 64 * m) = v[m];
}

// ---------------------------------------------------------------------------
// mover 1: persistent TMA ring
// ---------------------------------------------------------------------------
// Destinations of the fused slab transpose (AXIS 4): rows [q nxl, (q+1) nxl)
// of every x tile go to rank q's peer-major buffer, through one tensor map per
// rank over that (peer-mapped, NVLink) buffer.
struct PeerMaps {
  CUtensorMap m[kMaxRanks];
  int P;
};
struct NoPeers {};

// AXIS 1 / 2: y / x lines of the natural layout (in place); AXIS 4: x lines of
// the slab's y-slab, results stored by TMA straight into the other ranks'
// buffers (the transpose of the fused slab transport).
template <int L, int KIND, int AXIS, typename PM, int WPC = 1, int W = kCols>
__global__ void __launch_bounds__(kRingThreads, 1)
    ring_kernel(const __grid_constant__ CUtensorMap tmap, TileArgs a, const double2* __restrict__ tw,
                const __grid_constant__ PM pm) {
  constexpr int BOX = L < kBoxRows ? L : kBoxRows;
  constexpr uint32_t kTileBytes = (uint32_t)L * W * sizeof(double2);
  extern __shared__ unsigned char smem_raw[];
  unsigned char* base = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);  // swizzle atom: 1 KB
  double2* bufs = reinterpret_cast<double2*>(base);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + kBufs * kTileBytes);
  uint64_t* done = full + kBufs;
  uint32_t* cnt = reinterpret_cast<uint32_t*>(done + kBufs);  // columns finished per fill
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  const uint32_t ntiles = a.n_outer * a.nchunk;
  const uint32_t nloc = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  auto coords = [&](uint32_t j, int& c0, int& o) {
    const uint32_t tile = blockIdx.x + j * gridDim.x;
    const uint32_t oo = tile / a.nchunk;
    c0 = (int)((tile - oo * a.nchunk) * 2 * W);  // W complex = 2W scalars per column block
    o = (int)oo;
  };
  auto load = [&](uint32_t j) {
    const int b = j % kBufs;
    double2* buf = bufs + (size_t)b * L * W;
    int c0, o;
    coords(j, c0, o);
    fence_async_smem();
    bar_expect_tx(&full[b], kTileBytes);
#pragma unroll
    for (int q = 0; q < L / BOX; ++q)
      tma_load(buf + q * BOX * W, &tmap, &full[b], c0, AXIS != 1 ? o : q * BOX, AXIS != 1 ? q * BOX : o);
  };

  constexpr int kWarpsPerTile = W * WPC;  // (8, 1) or (4, 2): 2 groups; (8, 2): all 16 warps on one tile
  constexpr int kTileGroups = kGroups * kCols / kWarpsPerTile;
  if (threadIdx.x == 0) {
    for (int b = 0; b < kBufs; ++b) {
      bar_init(&full[b], 1);
      bar_init(&done[b], kWarpsPerTile);
      cnt[b] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (uint32_t j = 0; j < (uint32_t)kBufs && j < nloc; ++j) load(j);
  }
  __syncthreads();

  const int g = warp / kWarpsPerTile, c = (warp % kWarpsPerTile) / WPC;
  for (uint32_t j = g; j < nloc; j += kTileGroups) {
    const int b = j % kBufs;
    const uint32_t k = j / kBufs;
    // fill k - 1 of this buffer (the other group's tile) must be consumed
    // before waiting on fill k, or the full-barrier parity would alias
    if (k >= 1) bar_wait(&done[b], (k - 1) & 1);
    bar_wait(&full[b], k & 1);
    const uint32_t tile = blockIdx.x + j * gridDim.x;
    const uint32_t o = tile / a.nchunk;
    const uint32_t z = (tile - o * a.nchunk) * W + c;
    double2* buf = bufs + (size_t)b * L * W;
    if constexpr (WPC == 1) {
      column<L, KIND>(SwzCol{buf, c}, lane, tw, a.ph, o, z);
    } else {
      column2<L, KIND>(SwzColT<W>{buf, c}, (warp & 1) * 32 + lane, tw, a.ph, o, z, SyncNamed{1 + warp / 2, 64});
    }
    fence_async_smem();  // generic-proxy writes -> the TMA store
    __syncwarp();
    if (lane == 0) {
      // the last of the tile's 8 warps writes it back and refills the buffer
      // with tile j + kBufs (a dedicated producer warp would make 17 warps and
      // cap the registers at 96 per thread)
      __threadfence_block();
      const bool last = atomicAdd(&cnt[b], 1u) == kWarpsPerTile - 1;
      __threadfence_block();
      bar_arrive(&done[b]);
      if (last) {
        cnt[b] = 0;
        int c0, oo;
        coords(j, c0, oo);
        if constexpr (AXIS == 4) {
          const int nxl = L / pm.P, bx = nxl < BOX ? nxl : BOX;
          for (int q = 0; q < pm.P; ++q)
            for (int r0 = 0; r0 < nxl; r0 += bx) tma_store(&pm.m[q], buf + (q * nxl + r0) * W, c0, oo, r0);
        } else {
#pragma unroll
          for (int q = 0; q < L / BOX; ++q)
            tma_store(&tmap, buf + q * BOX * W, c0, AXIS == 2 ? oo : q * BOX, AXIS == 2 ? q * BOX : oo);
        }
        bulk_commit();
        bulk_wait_read0();  // the buffer may be refilled once the store has read it
        if (j + kBufs < nloc) load(j + kBufs);
      }
    }
  }
  if (lane == 0) {
    bulk_wait0();  // this thread's bulk stores are complete (no-op if it issued none)
    if constexpr (AXIS == 4) __threadfence_system();
  }
}

// ---------------------------------------------------------------------------
// mover 2: one tile per CTA, rows through registers
// ---------------------------------------------------------------------------
struct Strides {
  uint32_t rs, os;  // row (line-axis) and outer strides, in complex elements
};

template <int L, int KIND>
__global__ void __launch_bounds__(kTileThreads, 2)
    tile1_kernel(double2* __restrict__ psi, Strides s, TileArgs a, const double2* __restrict__ tw) {
  constexpr int kMoves = L / kCols / 4;  // 16-byte moves per lane (8 lanes per 128-byte row)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* buf = reinterpret_cast<double2*>(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t tile = blockIdx.x;
  const uint32_t o = tile / a.nchunk;
  const uint32_t zc = tile - o * a.nchunk;
  double2* g = psi + o * s.os + zc * 8 + (lane & 7);
  const int row0 = warp * (L / kCols) + (lane >> 3), ch = lane & 7;
  {
    double2 r[kMoves];
#pragma unroll
    for (int q = 0; q < kMoves; ++q) r[q] = __ldcg(g + (size_t)(row0 + 4 * q) * s.rs);
#pragma unroll
    for (int q = 0; q < kMoves; ++q) {
      const int row = row0 + 4 * q;
      buf[row * 8 + (ch ^ (row & 7))] = r[q];
    }
  }
  __syncthreads();
  column<L, KIND>(SwzCol{buf, warp}, lane, tw, a.ph, o, zc * 8 + warp);
  __syncthreads();
#pragma unroll
  for (int q = 0; q < kMoves; ++q) {
    const int row = row0 + 4 * q;
    __stcg(g + (size_t)row * s.rs, buf[row * 8 + (ch ^ (row & 7))]);
  }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return (EncodeTiledFn) nullptr;
    return (EncodeTiledFn)p;
  }();
  return fn;
}

// CTAs of the persistent ring: one per SM, or CTAP_RING_SMS (experiments:
// leave SMs to a concurrently running pass)
static int sm_count() {
  static const int cap = [] {
    const char* e = getenv("CTAP_RING_SMS");
    return e ? atoi(e) : 0;
  }();
  const int n = ctap_sm_count();
  return cap > 0 && cap < n ? cap : n;
}

// AXIS 2: x lines of an (L, n_outer, nz) array; AXIS 1: y lines of an
// (n_outer, L, nz) array (nz = 8 * a.nchunk)
template <int L, int KIND, int AXIS>
static cudaError_t launch_ring(const TileArgs& a, void* data, const double2* tw, cudaStream_t st, int wpc = 1) {
  constexpr int BOX = L < kBoxRows ? L : kBoxRows;
  // 1024-point lines: 4-column tiles (64 KB), two warps per column
  constexpr int W = L >= 1024 ? 4 : kCols;
  if (L >= 1024) wpc = 2;
  EncodeTiledFn enc = encode_fn();
  if (!enc) return cudaErrorNotSupported;
  const uint64_t nz2 = (uint64_t)a.nchunk * W * 2;  // scalars of the pass's z columns
  // z pitch of the array in scalars: the x pass of a z chunk (a.in offset
  // by z0) covers nz2 of them
  const uint64_t pitch2 = (uint64_t)(AXIS == 2 ? a.lin.so : a.lin.si) * 2;
  if (pitch2 < nz2) return cudaErrorInvalidValue;
  const uint64_t d1 = AXIS == 2 ? a.n_outer : L, d2 = AXIS == 2 ? L : a.n_outer;
  CUtensorMap map;
  std::memset(&map, 0, sizeof map);
  const cuuint64_t dims[3] = {nz2, d1, d2};
  const cuuint64_t strides[2] = {pitch2 * sizeof(double), pitch2 * sizeof(double) * d1};
  const cuuint32_t box[3] = {2 * W, AXIS == 2 ? 1u : (cuuint32_t)BOX, AXIS == 2 ? (cuuint32_t)BOX : 1u};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, data, dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, W == 8 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                   kL2Promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
  auto k = ring_kernel<L, KIND, AXIS, NoPeers, L >= 1024 ? 2 : 1, W>;
  if constexpr (L == 512 && KIND == T_KIN)
    if (wpc == 2) k = ring_kernel<L, KIND, AXIS, NoPeers, 2, W>;
  constexpr size_t smem = (size_t)kBufs * L * W * sizeof(double2) + kRingBarBytes + 1024;
  static std::atomic<uint64_t> attr_done[2];
  if (cudaError_t e = ctap_smem_attr(k, smem, attr_done[wpc == 2 ? 1 : 0])) return e;
  const uint32_t ntiles = a.n_outer * a.nchunk;
  const uint32_t grid = ntiles < (uint32_t)sm_count() ? ntiles : (uint32_t)sm_count();
  k<<<grid, kRingThreads, smem, st>>>(map, a, tw, NoPeers{});
  return cudaGetLastError();
}

// [x K x^-1] of the y-slab (L = nx, n_outer = ny/P, nz) with the fused
// transpose: tile rows of rank q's x range are TMA-stored into a.peers[q]
// (peer-major (nx/P, ny/P, nz) block of this rank inside rank q's buffer).
template <int L>
static cudaError_t launch_ring_peers(const TileArgs& a, const void* in, int P, const double2* tw, cudaStream_t st) {
  constexpr int BOX = L < kBoxRows ? L : kBoxRows;
  EncodeTiledFn enc = encode_fn();
  if (!enc || P < 2 || P > kMaxRanks || L % P) return cudaErrorNotSupported;
  const uint64_t nz2 = (uint64_t)a.nchunk * 8 * 2;
  const uint64_t nxl = L / P;
  const cuuint32_t estr[3] = {1, 1, 1};
  CUtensorMap map;
  std::memset(&map, 0, sizeof map);
  {
    const cuuint64_t dims[3] = {nz2, a.n_outer, (cuuint64_t)L};
    const cuuint64_t strides[2] = {nz2 * sizeof(double), nz2 * sizeof(double) * a.n_outer};
    const cuuint32_t box[3] = {16, 1, (cuuint32_t)BOX};
    if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(in), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, kL2Promo,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  PeerMaps pm;
  std::memset(&pm, 0, sizeof pm);
  pm.P = P;
  for (int q = 0; q < P; ++q) {
    const cuuint64_t dims[3] = {nz2, a.n_outer, nxl};
    const cuuint64_t strides[2] = {nz2 * sizeof(double), nz2 * sizeof(double) * a.n_outer};
    const cuuint32_t box[3] = {16, 1, (cuuint32_t)(nxl < (uint64_t)BOX ? nxl : BOX)};
    if (enc(&pm.m[q], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, a.peers[q], dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, kL2Promo,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  auto k = ring_kernel<L, T_KIN, 4, PeerMaps>;
  constexpr size_t smem = (size_t)kBufs * L * kCols * sizeof(double2) + kRingBarBytes + 1024;
  static std::atomic<uint64_t> attr_done{0};
  if (cudaError_t e = ctap_smem_attr(k, smem, attr_done)) return e;
  const uint32_t ntiles = a.n_outer * a.nchunk;
  const uint32_t grid = ntiles < (uint32_t)sm_count() ? ntiles : (uint32_t)sm_count();
  k<<<grid, kRingThreads, smem, st>>>(map, a, tw, pm);
  return cudaGetLastError();
}

template <int L, int KIND, int AXIS>
static cudaError_t launch_tile1(const TileArgs& a, void* data, const double2* tw, cudaStream_t st) {
  const uint32_t nz = a.nchunk * 8;
  Strides s;
  s.rs = AXIS == 2 ? a.n_outer * nz : nz;
  s.os = AXIS == 2 ? nz : (uint32_t)L * nz;
  auto k = tile1_kernel<L, KIND>;
  constexpr size_t smem = (size_t)L * kCols * sizeof(double2);
  static std::atomic<uint64_t> attr_done{0};
  if (cudaError_t e = ctap_smem_attr(k, smem, attr_done)) return e;
  k<<<a.n_outer * a.nchunk, kTileThreads, smem, st>>>((double2*)data, s, a, tw);
  return cudaGetLastError();
}

}  // namespace wl
}  // namespace ctap

using namespace ctap;

// In-place strided pass on lines of length L = 256, 512 or 1024 through the
// warp-per-line kernels: axis 2 = x lines of an (L, n_outer, nz) array
// (kinds T_FWD, T_INV, T_KIN, T_COPY), axis 1 = y lines of an (n_outer, L, nz)
// array (T_FWD, T_INV, T_COPY).  `mode` 1 ring, 2 tile, 3 ring with two warps
// per column for the 512-point kinetic pass (else as 1); returns
// cudaErrorNotSupported outside these shapes (the caller then uses tile_kernel).
cudaError_t ctap_run_wline(const ctap_plan* p, int axis, int kind, int mode, void* data, const TileArgs& a,
                           cudaStream_t st) {
  if (p->dtype != CTAP_C128 || mode < 1 || mode > 6) return cudaErrorNotSupported;
  const int64_t L = axis == 2 ? p->n[0] : p->n[1];
  if (L == 1024) {  // 4-column tiles, two warps per column, ring only (diagnostic kinds too)
    if (mode == 2 || mode == 5 || (axis == 1 && kind == T_KIN) || a.nchunk * 8 % 4) return cudaErrorNotSupported;
    TileArgs b = a;
    b.nchunk = a.nchunk * 2;  // the caller counts 8-column chunks
    const double2* tw = p->twiddles + p->tw_off[7];
    switch (kind) {
      // x lines at 1024 have an 8 MiB stride: 64-byte TMA rows move them at
      // ~2.3 TB/s (copy 7.4 ms at 1024^2 x 512), so [x K x^-1] stays on
      // tile_kernel's 16-byte loads unless forced (CTAP_WLINE >= 4)
      case T_KIN:
        return axis == 2 && mode >= 4 ? wl::launch_ring<1024, T_KIN, 2>(b, data, tw, st) : cudaErrorNotSupported;
      case T_FWD: return axis == 2 ? wl::launch_ring<1024, T_FWD, 2>(b, data, tw, st)
                                   : wl::launch_ring<1024, T_FWD, 1>(b, data, tw, st);
      case T_INV: return axis == 2 ? wl::launch_ring<1024, T_INV, 2>(b, data, tw, st)
                                   : wl::launch_ring<1024, T_INV, 1>(b, data, tw, st);
      case T_COPY: return axis == 2 ? wl::launch_ring<1024, T_COPY, 2>(b, data, tw, st)
                                    : wl::launch_ring<1024, T_COPY, 1>(b, data, tw, st);
    }
    return cudaErrorNotSupported;
  }
  if (L != 256 && L != 512) return cudaErrorNotSupported;
  // the 256-point kinetic pass stays on tile_kernel: with 8 points per lane
  // the ring measured slower there (0.158 vs 0.144 ms at 256^3); the
  // CTAP_WLINE >= 4 switch forces it (tests)
  if (axis == 2 && kind == T_KIN && L == 256 && mode < 4) return cudaErrorNotSupported;
  if (mode >= 4) mode -= 3;
  if (axis == 1 && kind == T_KIN) return cudaErrorNotSupported;
  const double2* tw = p->twiddles + p->tw_off[L == 256 ? 5 : 6];
#define CTAP_WL_K(LL, KK, AX)                                                                       \
  (mode != 2 ? wl::launch_ring<LL, KK, AX>(a, data, tw, st, mode == 3 ? 2 : 1)                      \
             : wl::launch_tile1<LL, KK, AX>(a, data, tw, st))
#define CTAP_WL(LL, AX)                          \
  switch (kind) {                                \
    case T_FWD: return CTAP_WL_K(LL, T_FWD, AX); \
    case T_INV: return CTAP_WL_K(LL, T_INV, AX); \
    case T_COPY: return CTAP_WL_K(LL, T_COPY, AX); \
  }                                              \
  return cudaErrorNotSupported;
  if (axis == 2) {
    if (kind == T_KIN) return L == 512 ? CTAP_WL_K(512, T_KIN, 2) : CTAP_WL_K(256, T_KIN, 2);
    if (L == 512) { CTAP_WL(512, 2) }
    CTAP_WL(256, 2)
  }
  if (L == 512) { CTAP_WL(512, 1) }
  CTAP_WL(256, 1)
#undef CTAP_WL
#undef CTAP_WL_K
}

// The fused slab transport's [x K x^-1] (PASS_X_KIN_TO_PEERS) through the ring
// with per-rank TMA stores; cudaErrorNotSupported outside complex128,
// nx = 256 / 512 (the caller then uses tile_kernel's peer stores).
cudaError_t ctap_run_wline_peers(const ctap_plan* p, const void* in, const TileArgs& a, cudaStream_t st) {
  if (p->dtype != CTAP_C128 || (p->wline != 1 && p->wline != 4)) return cudaErrorNotSupported;
  const int64_t L = p->n[0];
  const double2* tw = p->twiddles + p->tw_off[L == 256 ? 5 : 6];
  if (L == 512) return wl::launch_ring_peers<512>(a, in, p->slab_p, tw, st);
  if (L == 256 && p->wline >= 4) return wl::launch_ring_peers<256>(a, in, p->slab_p, tw, st);
  return cudaErrorNotSupported;
}
