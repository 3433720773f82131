// TMA-pipelined strided passes (y and x) for the single-GPU natural layout.
//
// Same tile and thread mapping as tile_kernel (ctap_passes.cu): a tile is
// 8 consecutive z columns x the whole line, thread (t, col) owns points
// t + m*T of column col.  The difference is how the tile reaches the SM: a
// persistent CTA per SM runs G independent compute groups (named barriers)
// over NB > G tile buffers, and each group, when it releases a buffer, streams
// a later tile into it with cp.async.bulk.tensor (TMA, completion on an
// mbarrier).  HBM reads of the next tiles therefore overlap the FP64 work of
// the current ones instead of waiting behind it.  The landed buffer is the
// [i][8] tile in natural order, which doubles as the FFT exchange buffer.
// Results go straight from registers to HBM (the stores do not stall).
#include <cuda.h>

#include <cstring>

#include "ctap_device.cuh"
#include "ctap_internal.h"
#include "ctap_tile.cuh"

namespace ctap {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
      "[%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// Shared-memory pipeline of one persistent CTA: G compute groups of L
// threads (8 columns x T = L/8 threads each) and NB > G tile buffers.  Local
// tile j (global tile blockIdx.x + j*gridDim.x) lands in buffer j % NB and is
// transformed by group j % G; when a group has finished a tile it streams tile
// j + NB into the buffer it just released, so while each group computes, the
// tiles of the next NB - G steps are already in flight.
template <int L, typename CV>
struct TmaCfg {
  static constexpr int G = 1024 / L < 4 ? 1024 / L : 4;  // compute groups
  static constexpr uint32_t kTileBytes = (uint32_t)L * 8 * sizeof(CV);
  static constexpr int kMaxBuf = (int)((200u * 1024u) / kTileBytes);
  static constexpr int NB = G + 2 <= kMaxBuf ? G + 2 : kMaxBuf;  // >= G + 1 required
  static constexpr bool ok = NB >= G + 1;
  static constexpr size_t smem = (size_t)NB * kTileBytes + 12 * NB;
};

// AXIS 1: y pass on (x, y, z) (o = x, line = y = tensor dim 1)
// AXIS 2: x pass on (x, y, z) (o = y, line = x = tensor dim 2)
template <int L, int KIND, typename CV, int AXIS>
__global__ void __launch_bounds__(L * TmaCfg<L, CV>::G, 1)
    tma_tile_kernel(const __grid_constant__ CUtensorMap tmap, TileArgs a, const TwOf<CV>* __restrict__ tw) {
  using Cfg = TmaCfg<L, CV>;
  constexpr int E = kElems;
  constexpr int T = L / E;  // threads per column; a group is 8 T = L threads
  constexpr int G = Cfg::G, NB = Cfg::NB;
  constexpr int BOX = L < 256 ? L : 256;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  CV* bufs = reinterpret_cast<CV*>(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + (size_t)NB * Cfg::kTileBytes);
  uint32_t* issued = reinterpret_cast<uint32_t*>(full + NB);  // fills issued per buffer - 1
  CV* out = (CV*)a.out;
  const int g = threadIdx.x / L;
  const int lt = threadIdx.x - g * L;
  const int col = lt & 7;
  const int t = lt >> 3;
  const SyncNamed gsync{1 + g, L};
  const uint32_t ntiles = a.n_outer * a.nchunk;
  const uint32_t nloc = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;

  auto issue = [&](uint32_t j) {
    const uint32_t tile = blockIdx.x + j * gridDim.x;
    CV* dst = bufs + (size_t)(j % NB) * L * 8;
    uint64_t* bar = &full[j % NB];
    const uint32_t o = tile / a.nchunk;
    const int c0 = (int)((tile - o * a.nchunk) * 8 * 2);  // in scalars (re, im)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(bar, Cfg::kTileBytes);
#pragma unroll
    for (int b = 0; b < L / BOX; ++b) {
      if constexpr (AXIS == 1) tma_load_3d(dst + b * BOX * 8, &tmap, bar, c0, b * BOX, (int)o);
      else tma_load_3d(dst + b * BOX * 8, &tmap, bar, c0, (int)o, b * BOX);
    }
  };

  if (threadIdx.x == 0) {
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      mbar_init(&full[b], 1);
      issued[b] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (uint32_t j = 0; j < (uint32_t)NB && j < nloc; ++j) issue(j);

  for (uint32_t j = g; j < nloc; j += G) {
    const int b = j % NB;
    const uint32_t use = j / NB;  // fill number of buffer b
    CV* cur = bufs + (size_t)b * L * 8;
    // a group may reach fill `use` of a buffer while fill `use - 1` (another
    // group's tile) is still in flight, where the mbarrier parity would alias:
    // first wait until that tile has been consumed and fill `use` issued
    if (use > 0)
      while (*(volatile uint32_t*)&issued[b] < use) {
      }
    mbar_wait(&full[b], use & 1);
    const uint32_t tile = blockIdx.x + j * gridDim.x;
    const uint32_t o = tile / a.nchunk;
    const uint32_t z = (tile - o * a.nchunk) * 8 + col;
    CV v[E];
#pragma unroll
    for (int m = 0; m < E; ++m) v[m] = cur[(t + m * T) * 8 + col];
    gsync();  // the group holds its points: the buffer becomes its exchange buffer
    tile_body<L, E, KIND, false, false>(a, v, t, o, z, true, tw, SmemStrided<CV, 8>{cur + col}, gsync);
    const uint32_t obo = outer(a.lout, o) + z;
#pragma unroll
    for (int m = 0; m < E; ++m) out[obo + inner<false>(a.lout, t + m * T)] = v[m];
    gsync();  // buffer released
    if (lt == 0 && j + NB < nloc) {
      issue(j + NB);
      __threadfence_block();
      *(volatile uint32_t*)&issued[b] = use + 1;
    }
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

template <int L, int KIND, typename CV, int AXIS>
static cudaError_t launch_tma(const TileArgs& a, void* data, uint64_t d1, uint64_t d2, const TwOf<CV>* tw,
                              cudaStream_t st) {
  constexpr int BOX = L < 256 ? L : 256;
  EncodeTiledFn enc = encode_fn();
  if (!enc) return cudaErrorNotSupported;
  const uint64_t nz2 = (uint64_t)a.nchunk * 8 * 2;  // scalars per z line
  CUtensorMap map;
  std::memset(&map, 0, sizeof map);
  const cuuint64_t dims[3] = {nz2, d1, d2};
  const cuuint64_t strides[2] = {nz2 * sizeof(CV) / 2, nz2 * sizeof(CV) / 2 * d1};
  const cuuint32_t box[3] = {16, AXIS == 1 ? (cuuint32_t)BOX : 1u, AXIS == 1 ? 1u : (cuuint32_t)BOX};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUtensorMapDataType dt =
      sizeof(CV) == 16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  CUresult r = enc(&map, dt, 3, data, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
  using Cfg = TmaCfg<L, CV>;
  if constexpr (!Cfg::ok) return cudaErrorNotSupported;
  auto k = tma_tile_kernel<L, KIND, CV, AXIS>;
  const size_t smem = Cfg::smem;
  static std::atomic<uint64_t> attr_done{0};
  if (cudaError_t e = ctap_smem_attr(k, smem, attr_done)) return e;
  const int sms = ctap_sm_count();
  const uint32_t ntiles = a.n_outer * a.nchunk;
  const uint32_t grid = ntiles < (uint32_t)sms ? ntiles : (uint32_t)sms;
  k<<<grid, L * Cfg::G, smem, st>>>(map, a, tw);
  return cudaGetLastError();
}

}  // namespace ctap

using namespace ctap;

// In-place strided pass through the TMA pipeline on the natural layout.
// axis 1: y lines of an (n0 = nx_local, ny, nz) array; axis 2: x lines of an
// (nx, n1 = ny_local, nz) array.  kind: T_FWD, T_INV or T_KIN.
// Returns cudaErrorNotSupported when the shape is outside the TMA kernels
// (the caller then uses tile_kernel).
cudaError_t ctap_run_tma_pass(const ctap_plan* p, int axis, int kind, void* data, const TileArgs& a,
                              cudaStream_t st) {
  const bool c64 = p->dtype == CTAP_C64;
  const int64_t L = axis == 1 ? p->n[1] : p->n[0];
  const uint64_t d1 = axis == 1 ? (uint64_t)p->n[1] : (uint64_t)(p->n[1] / p->slab_p);
  const uint64_t d2 = axis == 1 ? (uint64_t)p->nx_local : (uint64_t)p->n[0];
  const int off = p->tw_off[L == 128 ? 4 : L == 256 ? 5 : 6];
#define CTAP_TMA(LL, KK, AX)                                                                                  \
  (c64 ? launch_tma<LL, KK, float2, AX>(a, data, d1, d2, p->twiddles32 + off, st)                            \
       : launch_tma<LL, KK, double2, AX>(a, data, d1, d2, p->twiddles + off, st))
#define CTAP_TMA_L(KK, AX)               \
  switch (L) {                           \
    case 128: return CTAP_TMA(128, KK, AX); \
    case 256: return CTAP_TMA(256, KK, AX); \
    case 512: return CTAP_TMA(512, KK, AX); \
  }                                      \
  return cudaErrorNotSupported;
  if (axis == 1) {
    if (kind == T_FWD) { CTAP_TMA_L(T_FWD, 1) }
    if (kind == T_INV) { CTAP_TMA_L(T_INV, 1) }
  } else {
    if (kind == T_FWD) { CTAP_TMA_L(T_FWD, 2) }
    if (kind == T_INV) { CTAP_TMA_L(T_INV, 2) }
    if (kind == T_KIN) { CTAP_TMA_L(T_KIN, 2) }
  }
#undef CTAP_TMA_L
#undef CTAP_TMA
  return cudaErrorNotSupported;
}
