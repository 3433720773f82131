// TMA-pipelined strided passes (y and x) for the single-GPU natural layout.
//
// Same tile and thread mapping as tile_kernel (ctap_passes.cu): a tile is
// 8 consecutive z columns x the whole line, thread (t, col) owns points
// t + m*T of column col.  The difference is how the tile reaches the SM: a
// persistent CTA per SM keeps two tile buffers in shared memory and one
// elected thread streams the NEXT tile into the idle buffer with
// cp.async.bulk.tensor (TMA, completion on an mbarrier) while all threads
// transform the current one, so the HBM reads of tile k+1 overlap the
// FP64 work of tile k instead of waiting behind it.  The landed buffer is the
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

// AXIS 1: y pass on (x, y, z) (o = x, line = y = tensor dim 1)
// AXIS 2: x pass on (x, y, z) (o = y, line = x = tensor dim 2)
template <int L, int KIND, typename CV, int AXIS>
__global__ void __launch_bounds__(L, 1)
    tma_tile_kernel(const __grid_constant__ CUtensorMap tmap, TileArgs a, const CV* __restrict__ tw) {
  constexpr int E = kElems;
  constexpr int T = L / E;  // threads per column; blockDim = 8 T = L
  constexpr int BOX = L < 256 ? L : 256;
  constexpr uint32_t kTileBytes = (uint32_t)L * 8 * sizeof(CV);
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  CV* buf0 = reinterpret_cast<CV*>(smem_raw);
  CV* buf1 = buf0 + L * 8;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + 2 * kTileBytes);
  CV* out = (CV*)a.out;
  const int col = threadIdx.x & 7;
  const int t = threadIdx.x >> 3;
  const uint32_t ntiles = a.n_outer * a.nchunk;

  auto issue = [&](uint32_t tile, CV* dst, uint64_t* bar) {
    const uint32_t o = tile / a.nchunk;
    const int c0 = (int)((tile - o * a.nchunk) * 8 * 2);  // in scalars (re, im)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(bar, kTileBytes);
#pragma unroll
    for (int b = 0; b < L / BOX; ++b) {
      if constexpr (AXIS == 1) tma_load_3d(dst + b * BOX * 8, &tmap, bar, c0, b * BOX, (int)o);
      else tma_load_3d(dst + b * BOX * 8, &tmap, bar, c0, (int)o, b * BOX);
    }
  };

  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x < ntiles) issue(blockIdx.x, buf0, &bars[0]);

  uint32_t k = 0;
  for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++k) {
    const int s = k & 1;
    CV* cur = s ? buf1 : buf0;
    // stream the next tile into the other buffer (freed by the barrier that
    // ended the previous iteration) while this one is transformed
    if (threadIdx.x == 0 && tile + gridDim.x < ntiles) issue(tile + gridDim.x, s ? buf0 : buf1, &bars[s ^ 1]);
    mbar_wait(&bars[s], (k >> 1) & 1);
    const uint32_t o = tile / a.nchunk;
    const uint32_t z = (tile - o * a.nchunk) * 8 + col;
    CV v[E];
#pragma unroll
    for (int m = 0; m < E; ++m) v[m] = cur[(t + m * T) * 8 + col];
    __syncthreads();  // everyone holds its points: the buffer becomes the exchange buffer
    tile_body<L, E, KIND, false, false>(a, v, t, o, z, true, tw, SmemStrided<CV, 8>{cur + col});
    const uint32_t obo = outer(a.lout, o) + z;
#pragma unroll
    for (int m = 0; m < E; ++m) out[obo + inner<false>(a.lout, t + m * T)] = v[m];
    __syncthreads();  // buffer free for the TMA issued at the next iteration
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
static cudaError_t launch_tma(const TileArgs& a, void* data, uint64_t d1, uint64_t d2, const CV* tw,
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
  auto k = tma_tile_kernel<L, KIND, CV, AXIS>;
  const size_t smem = 2 * (size_t)L * 8 * sizeof(CV) + 16;
  static cudaError_t init = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (init != cudaSuccess) return init;
  static int sms = [] {
    int dev = 0, n = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  const uint32_t ntiles = a.n_outer * a.nchunk;
  const uint32_t grid = ntiles < (uint32_t)sms ? ntiles : (uint32_t)sms;
  k<<<grid, L, smem, st>>>(map, a, tw);
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
