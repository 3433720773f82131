// Internal plan object shared by the kernels and the C ABI (not exported).
#pragma once

#include <atomic>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/ctap.h"

namespace ctap {
enum PassKind {
  // z passes (contiguous lines, always in place)
  PASS_Z_FWD = CTAP_PASS_Z_FWD,
  PASS_Z_INV = CTAP_PASS_Z_INV,
  PASS_Z_FIRST = CTAP_PASS_Z_FIRST,  // Vh, then Fz
  PASS_Z_MID = CTAP_PASS_Z_MID,      // Fz^-1, V, Fz
  PASS_Z_LAST = CTAP_PASS_Z_LAST,    // Fz^-1, then Vh
  // y passes
  PASS_Y_FWD = CTAP_PASS_Y_FWD,
  PASS_Y_INV = CTAP_PASS_Y_INV,
  PASS_Y_FWD_TO_PEER = CTAP_PASS_Y_FWD_TO_PEER,
  PASS_Y_INV_FROM_PEER = CTAP_PASS_Y_INV_FROM_PEER,
  // x passes (y-slab layout)
  PASS_X_KIN = CTAP_PASS_X_KIN,  // Fx, K / N, Fx^-1
  PASS_X_FWD = CTAP_PASS_X_FWD,
  PASS_X_INV = CTAP_PASS_X_INV,
  // blocked k-space variants of the single-GPU step (internal)
  PASS_Y_FWD_BLK = CTAP_PASS_Y_FWD_BLK,  // y FFT, natural -> blocked k-space buffer
  PASS_X_KIN_BLK = CTAP_PASS_X_KIN_BLK,  // [x K x^-1] on the blocked buffer, in place
  PASS_Y_INV_BLK = CTAP_PASS_Y_INV_BLK,  // y^-1, blocked buffer -> natural
  PASS_Y_FWD_TO_PEERS = CTAP_PASS_Y_FWD_TO_PEERS,
  PASS_X_KIN_TO_PEERS = CTAP_PASS_X_KIN_TO_PEERS,
  PASS_PZ_FIRST = CTAP_PASS_PZ_FIRST,
  PASS_PZ_MID = CTAP_PASS_PZ_MID,
  PASS_PZ_LAST = CTAP_PASS_PZ_LAST,
  PASS_PY_FWD = CTAP_PASS_PY_FWD,
  PASS_PY_INV = CTAP_PASS_PY_INV,
  PASS_PX_KIN = CTAP_PASS_PX_KIN,
  // diagnostics: the strided passes' memory traffic without the transforms
  PASS_Y_COPY = 60,
  PASS_X_COPY = 61,
  PASS_XB_COPY = 62,
  PASS_XP_COPY = 63,  // x-pass traffic with the x pitch padded by CTAP_XPAD points (buffer must hold it)
  PASS_XP_KIN = 64,   // X_KIN on that padded pitch
  PASS_WX_COPY = 65,  // warp-per-line TMA pipeline (ctap_wline.cu) without the transform, x lines
  PASS_WY_COPY = 66,  // the same on y lines
  PASS_WY_FWD = 67,   // forward y FFT through that pipeline
  // strided kernel variants
  PASS_S_FWD = 100,
  PASS_S_INV = 101,
  PASS_S_KIN = 102,
};
}  // namespace ctap

struct ctap_plan {
  int64_t n[3];
  int64_t nx_local;        // x extent of this rank's position-space block
  int64_t ny_pos;          // y extent of it (ny for slabs, ny/Pc for pencils)
  int slab_p, slab_r;
  int pen_c, pen_r, pen_a, pen_b;  // pencil grid Pr x Pc and this rank's (a, b); pen_c = 0 for slabs
  int mode;  // 0 real, 1 imaginary
  double e0, dt_i, len2, v_shift;
  double inv_scale;        // 1 / (nx ny nz), exact power of two
  const double* v_dev;     // caller-owned potential slab (J)
  double* vi_dev;          // v_i = (V - v_shift) / e0, plan-owned (propagator.py:65, :75)
  void* expv_dev;          // optional table exp(-i v_i dt_i), plan precision (phase_tables, real time)
  void* expk_dev;          // optional table exp(-i k^2 dt/2) / N, x-pass layout
  double* k2_dev[3];       // squared wavenumbers per axis (global lengths)
  double2* sctab;          // [kSCN] (cos, sin)(2 pi j / kSCN), [kSCN] the same times 1/N (ctap_device.cuh)
  int kgen;                // k^2 regenerated on device from kval (tables verified)
  int wline;               // x-pass kernel: 1 warp-per-line ring, 2 warp-per-line tile, 0 tile_kernel
  int64_t zchunk;          // kinetic block in z chunks of this width (0: whole volume)
  double kval[3];          // 1/(n d) per axis (numpy fftfreq's val)
  int dtype;               // CTAP_C128 or CTAP_C64
  double2* twiddles;       // stage-major twiddle tables for L = 8..1024
  float4* twiddles32;      // the same as float-float pairs (complex64 mode)
  int tw_off[8];           // start of the table of L = 8 << i
  int tw2_off[5];          // start of the two-stage plan's stage-2 table of L = 64 << i (ctap_fft2.cuh)
  int z2;                  // z passes on the two-stage FFT (complex128, nz >= 64); CTAP_Z2=0 disables
  double2* kbuf;           // single-GPU k-space buffer (blocked layout, out of place y passes)
  int k_lx;                // log2 of the x block of the k-space layout (0: natural)
  void* peer_y[16];        // fused slab transposes: every rank's y-slab buffer
  void* peer_p[16];        // and peer-major buffer (peer-mapped device addresses)
  double* red_partial;     // reduction scratch
  double* obs_partial;     // per-block partials of the fused segment-end observer sums (lazy)
  uint16_t* obs_mask;      // guide-partition bits of the fused observer pass (lazy)
  int skip_last;           // ctap_advance_observe: ctap_advance stops before the segment-end pass
  // CUDA graph of M interior steps (launch-bound small grids), captured on a
  // private stream for one psi pointer and replayed on the caller's stream
  cudaStream_t cap_stream;
  cudaStream_t kin_stream[2];  // z-chunked kinetic block: two concurrent chunk pipelines
  cudaEvent_t kin_ev[3];
  cudaStream_t pb_stream[4];   // x-slab position blocks (ctap_advance)
  cudaEvent_t pb_ev[5];
  cudaGraphExec_t pb_exec[4];  // their pieces as graphs, by phase (0 step, 1 segment start, 2/3 ends) for pb_psi
  const void* pb_psi;
  cudaGraphExec_t g_exec;
  const void* g_psi;
  int g_steps;
  int red_blocks;
};

cudaError_t ctap_run_v_internal(const ctap_plan* p, cudaStream_t st);
cudaError_t ctap_run_phase_field(const ctap_plan* p, int which, void* out, cudaStream_t st);
cudaError_t ctap_run_phase_table(const ctap_plan* p, int which, void* out, cudaStream_t st);
#include <vector>
std::vector<double> ctap_make_twiddles(int off[8]);
void ctap_append_twiddles2(std::vector<double>& t, int off2[5]);
namespace ctap {
struct ZArgs;
}
int64_t ctap_z_blocks(const ctap_plan* p);
cudaError_t ctap_run_pass_chunk(const ctap_plan* p, int kind, const void* in, void* out, int64_t z0, int64_t zn,
                                cudaStream_t st);
extern thread_local int ctap_pdl;  // launch the z / y pass kernels with programmatic dependent launch
size_t ctap_obs_mask_entries(const ctap_plan* p);
cudaError_t ctap_run_z_last_observe(const ctap_plan* p, void* psi, const double* xs, const double* xb1,
                                    const double* xb2, int margin, double* partial, uint16_t* mask,
                                    cudaStream_t st);
cudaError_t ctap_run_finalize5(const ctap_plan* p, const double* partial, int64_t npartials, double* out,
                               int part, cudaStream_t st);
cudaError_t ctap_run_z2(const ctap_plan* p, int tkind, bool vtab, int ch, const ctap::ZArgs& a, cudaStream_t st);
static inline int ilog2i(int64_t v) {
  int l = 0;
  while ((int64_t(1) << l) < v) ++l;
  return l;
}
cudaError_t ctap_run_pass(const ctap_plan* p, int kind, const void* in, void* out, cudaStream_t st);
cudaError_t ctap_run_pass_z(const ctap_plan* p, int kind, const void* in, void* out, int64_t z0, int64_t zn,
                            cudaStream_t st);

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device):
// the attribute belongs to the function of the current device's context, so a
// process that also launches on a second device must set it there too.
// `done` is the call site's per-kernel bitmask of device ordinals.
template <typename K>
static inline cudaError_t ctap_smem_attr(K k, size_t bytes, std::atomic<uint64_t>& done) {
  if (bytes <= 48 * 1024) return cudaSuccess;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_relaxed) & bit) return cudaSuccess;
  e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) done.fetch_or(bit);
  return e;
}

// multiprocessor count of the current device, cached per device ordinal
static inline int ctap_sm_count() {
  static std::atomic<int> cache[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  int n = cache[dev].load(std::memory_order_relaxed);
  if (n == 0) {
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    cache[dev].store(n, std::memory_order_relaxed);
  }
  return n;
}
