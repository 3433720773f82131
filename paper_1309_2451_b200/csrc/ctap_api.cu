// C ABI of libctap.so (include/ctap.h): plan lifetime, error reporting and
// the per-segment driver loop that replaces propagator._advance.
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <cuda.h>
#include <nvtx3/nvToolsExt.h>

#include "ctap_device.cuh"
#include "ctap_internal.h"
#include "ctap_sincos_tab.h"

namespace {
// NVTX range over one ABI call (header-only NVTX 3: a no-op unless a tool such
// as nsys is attached), so device timelines show segments and passes by name
struct Range {
  explicit Range(const char* fmt, long long v = 0) {
    char buf[64];
    std::snprintf(buf, sizeof buf, fmt, v);
    nvtxRangePushA(buf);
  }
  ~Range() { nvtxRangePop(); }
};
}  // namespace

cudaError_t ctap_run_observe(const ctap_plan* p, const void* psi, const double* xs, const double* xb1,
                             const double* xb2, int margin, double* out, cudaStream_t st);
cudaError_t ctap_run_k2_sums(const ctap_plan* p, const void* phi, double* out, cudaStream_t st);
cudaError_t ctap_run_v_sums(const ctap_plan* p, const void* psi, const double* V, double* out, cudaStream_t st);
cudaError_t ctap_run_density_xz(const ctap_plan* p, const void* psi, double* out, cudaStream_t st);
cudaError_t ctap_run_scale(const ctap_plan* p, void* psi, double d, cudaStream_t st);
cudaError_t ctap_run_potential(const double* xs, int64_t nx, const double* ys, int64_t ny, const double* zs,
                               int64_t nz, const double* seg_a, const double* seg_b, const double* seg_cur,
                               int64_t n_seg, double b0x, double b0y, double b0z, double mu_eff, double mass,
                               double omega_z, double z_center, double pref, double* V_out, cudaStream_t st);
cudaError_t ctap_run_slice_minima(const double* V, int64_t nx, int64_t ny, int64_t nz, int64_t* count,
                                  int64_t* best, cudaStream_t st);

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  return fail(CTAP_ECUDA, "%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
}

bool pow2_in_range(int64_t n) { return n >= 8 && n <= 1024 && (n & (n - 1)) == 0; }

constexpr int kGraphSteps = 16;
bool graphs_enabled() {
  static const bool on = [] {
    const char* e = getenv("CTAP_GRAPHS");
    return e ? atoi(e) != 0 : true;
  }();
  return on;
}

}  // namespace

#define CUDA_TRY(expr, what)                       \
  do {                                             \
    cudaError_t e_ = (expr);                       \
    if (e_ != cudaSuccess) return cuda_fail(e_, what); \
  } while (0)

// Find val with fl(fl(2 pi * fl(m val))^2) == k2[i] for every index i
// (m = i for i < n/2, i - n otherwise), searching a few ulps around the
// estimate from k2[1].  Host arithmetic is plain IEEE double (no contraction
// in this translation unit's host code for these products).
static bool recover_kval(const double* k2, int64_t n, double* val) {
  if (n < 2 || !(k2[1] > 0.0)) return false;
  const double twopi = 6.283185307179586;
  volatile double est = std::sqrt(k2[1]) / twopi;
  double c = est;
  for (int step = 0; step < 8; ++step) c = std::nextafter(c, 0.0);
  for (int tries = 0; tries < 17; ++tries, c = std::nextafter(c, 1e300)) {
    bool ok = true;
    for (int64_t i = 0; i < n && ok; ++i) {
      const int64_t m = i < n / 2 ? i : i - n;
      volatile double mv = (double)m * c;
      volatile double k = twopi * mv;
      volatile double kk = k * k;
      ok = kk == k2[i];
    }
    if (ok) {
      *val = c;
      return true;
    }
  }
  return false;
}

extern "C" {

CTAP_API const char* ctap_last_error(void) { return g_err.c_str(); }
CTAP_API const char* ctap_version(void) { return "ctap 0.1.0 (sm_100a)"; }

CTAP_API int ctap_plan_create(const ctap_plan_desc* d, const double* kx2, const double* ky2, const double* kz2,
                              const double* v_dev, ctap_plan** out) {
  if (!d || !out || !kx2 || !ky2 || !kz2) return fail(CTAP_EINVAL, "null argument");
  *out = nullptr;
  for (int i = 0; i < 3; ++i)
    if (!pow2_in_range(d->n[i]))
      return fail(CTAP_EUNSUPPORTED, "grid counts must be powers of two in [8, 1024], got %lld",
                  (long long)d->n[i]);
  if (d->mode != CTAP_REAL_TIME && d->mode != CTAP_IMAGINARY_TIME)
    return fail(CTAP_EINVAL, "unknown mode %d", d->mode);
  if (d->dtype != CTAP_C128 && d->dtype != CTAP_C64) return fail(CTAP_EINVAL, "unknown dtype %d", d->dtype);
  int P = d->slab_p < 1 ? 1 : d->slab_p;
  const int Pc = d->pencil_c > 1 ? d->pencil_c : 0;
  if (Pc) {
    if (P % Pc) return fail(CTAP_EINVAL, "%d ranks do not form a pencil grid with %d columns", P, Pc);
    const int Pr = P / Pc;
    if (d->n[0] % Pr || d->n[1] % Pr || d->n[1] % Pc || d->n[2] % (8 * Pc))
      return fail(CTAP_EINVAL, "pencil grid %d x %d needs nx %% %d, ny %% %d, ny %% %d and nz %% %d == 0", Pr, Pc, Pr,
                  Pr, Pc, 8 * Pc);
  } else if (d->n[0] % P || d->n[1] % P) {
    return fail(CTAP_EINVAL, "nx and ny must be divisible by the %d slab ranks", P);
  }
  if (d->slab_r < 0 || d->slab_r >= P) return fail(CTAP_EINVAL, "slab rank %d out of range", d->slab_r);

  ctap_plan* p = new ctap_plan();
  std::memset(p, 0, sizeof *p);
  for (int i = 0; i < 3; ++i) p->n[i] = d->n[i];
  p->slab_p = P;
  p->slab_r = d->slab_r;
  p->nx_local = d->n[0] / P;
  p->ny_pos = d->n[1];
  if (Pc) {  // pencil: rank r = a Pc + b owns x block a, y block b
    p->pen_c = Pc;
    p->pen_r = P / Pc;
    p->pen_a = d->slab_r / Pc;
    p->pen_b = d->slab_r % Pc;
    p->nx_local = d->n[0] / p->pen_r;
    p->ny_pos = d->n[1] / Pc;
  }
  p->mode = d->mode;
  p->dtype = d->dtype;
  p->e0 = d->e0;
  p->dt_i = d->dt_i;
  p->len2 = d->len2;
  p->v_shift = d->v_shift;
  p->v_dev = v_dev;
  p->inv_scale = 1.0 / (double)(d->n[0] * d->n[1] * d->n[2]);  // exact: power of two
  const double* k2h[3] = {kx2, ky2, kz2};
  // plan creation is rare: order it against whatever stream produced V
  cudaError_t e = cudaDeviceSynchronize();
  for (int i = 0; i < 3 && e == cudaSuccess; ++i) {
    e = cudaMalloc((void**)&p->k2_dev[i], sizeof(double) * d->n[i]);
    if (e == cudaSuccess) e = cudaMemcpy(p->k2_dev[i], k2h[i], sizeof(double) * d->n[i], cudaMemcpyHostToDevice);
  }
  // the x pass regenerates k^2 in registers when the tables are numpy's
  // (2 pi * fftfreq(n, d))^2 for some val = 1/(n d), checked bit for bit
  p->kgen = 1;
  for (int i = 0; i < 3; ++i) p->kgen &= recover_kval(k2h[i], d->n[i], &p->kval[i]);
  if (const char* env = getenv("CTAP_KGEN")) p->kgen &= atoi(env) != 0;
  // x-pass kernel of the single-GPU step: 1 warp-per-line TMA ring (default;
  // nx = 512), 2 warp-per-line one tile per CTA, 3 ring with two warps per
  // column, 4-6 the same also for nx = 256, 0 tile_kernel (ctap_wline.cu)
  p->wline = 1;
  if (const char* env = getenv("CTAP_WLINE")) p->wline = atoi(env);
  p->zchunk = 0;
  if (const char* env = getenv("CTAP_ZCHUNK")) p->zchunk = atoll(env);
  if (p->zchunk % 8 || p->zchunk < 0 || (p->zchunk && d->n[2] % p->zchunk)) p->zchunk = 0;
  {  // sincos rotation tables: unscaled (V phases) and times 1/N (K phase)
    // kSCN entries (cos, sin)(2 pi j / kSCN) = entry j 256/kSCN of the 256 table
    std::vector<double> sc(4 * ctap::kSCN);
    for (int j = 0; j < ctap::kSCN; ++j) {
      const int k = j * (256 / ctap::kSCN);
      sc[2 * j] = kSinCos256[k][0];
      sc[2 * j + 1] = kSinCos256[k][1];
      sc[2 * ctap::kSCN + 2 * j] = kSinCos256[k][0] * p->inv_scale;  // exact: power of two
      sc[2 * ctap::kSCN + 2 * j + 1] = kSinCos256[k][1] * p->inv_scale;
    }
    if (e == cudaSuccess) e = cudaMalloc((void**)&p->sctab, sc.size() * sizeof(double));
    if (e == cudaSuccess) e = cudaMemcpy(p->sctab, sc.data(), sc.size() * sizeof(double), cudaMemcpyHostToDevice);
  }
  std::vector<double> tw = ctap_make_twiddles(p->tw_off);
  ctap_append_twiddles2(tw, p->tw2_off);
  p->z2 = 0;  // measured slower at 512^3: opt-in
  if (const char* env = getenv("CTAP_Z2")) p->z2 = atoi(env);
  if (e == cudaSuccess) e = cudaMalloc((void**)&p->twiddles, tw.size() * sizeof(double));
  if (e == cudaSuccess) e = cudaMemcpy(p->twiddles, tw.data(), tw.size() * sizeof(double), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) {  // complex64 copy of the (correctly rounded) double table
    // float-float split of every (re, im): hi = rn(d), lo = rn(d - hi)
    std::vector<float> tw32(2 * tw.size());
    for (size_t i = 0; i < tw.size() / 2; ++i) {
      const float hr = (float)tw[2 * i], hi = (float)tw[2 * i + 1];
      tw32[4 * i + 0] = hr;
      tw32[4 * i + 1] = hi;
      tw32[4 * i + 2] = (float)(tw[2 * i] - (double)hr);
      tw32[4 * i + 3] = (float)(tw[2 * i + 1] - (double)hi);
    }
    e = cudaMalloc((void**)&p->twiddles32, tw32.size() * sizeof(float));
    if (e == cudaSuccess) e = cudaMemcpy(p->twiddles32, tw32.data(), tw32.size() * sizeof(float), cudaMemcpyHostToDevice);
  }
  int dev = 0, sms = 148;
  if (e == cudaSuccess) e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  p->red_blocks = sms * 4;
  if (e == cudaSuccess) e = cudaMalloc((void**)&p->red_partial, sizeof(double) * 8 * p->red_blocks);
  const size_t nloc = (size_t)p->nx_local * p->ny_pos * d->n[2];
  const size_t csize = p->dtype == CTAP_C64 ? sizeof(float2) : sizeof(double2);
  // single GPU, opt-in (CTAP_KBLK_LX=lx > 0): out-of-place y passes into a
  // blocked k-space buffer so an x-line spans nx/2^lx address blocks instead of
  // nx.  Measured slower than the in-place natural layout on B200 at 512^3
  // (DESIGN.md §3), hence off by default.
  p->k_lx = 0;
  if (P == 1 && v_dev && d->n[0] >= 16) {
    int lx = 0;
    if (const char* env = getenv("CTAP_KBLK_LX")) lx = atoi(env);
    while (lx > 0 && (int64_t(1) << lx) > d->n[0]) --lx;
    p->k_lx = lx < 0 ? 0 : lx;
    if (p->k_lx > 0 && e == cudaSuccess) e = cudaMalloc((void**)&p->kbuf, csize * nloc);
  }
  if (v_dev) {  // a plan without a potential only serves FFTs and reductions
    if (e == cudaSuccess) e = cudaMalloc((void**)&p->vi_dev, sizeof(double) * nloc);
    if (e == cudaSuccess) e = ctap_run_v_internal(p, 0);
  }
  // pencil plans compute both phases on the fly (the tables' layouts are the
  // slab's; the phases are bitwise the same either way)
  const int tables = Pc ? 0 : d->phase_tables;
  if (e == cudaSuccess && v_dev && (tables & 1) && d->mode == CTAP_REAL_TIME) {
    e = cudaMalloc((void**)&p->expv_dev, csize * nloc);
    if (e == cudaSuccess) e = ctap_run_phase_table(p, 1, p->expv_dev, 0);
  }
  if (e == cudaSuccess && (tables & 2) && d->mode == CTAP_REAL_TIME) {
    e = cudaMalloc((void**)&p->expk_dev, csize * nloc);
    if (e == cudaSuccess) e = ctap_run_phase_table(p, 3, p->expk_dev, 0);
  }
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    ctap_plan_destroy(p);
    return cuda_fail(e, "ctap_plan_create");
  }
  *out = p;
  return CTAP_OK;
}

CTAP_API int ctap_plan_destroy(ctap_plan* p) {
  if (!p) return CTAP_OK;
  for (int i = 0; i < 3; ++i) cudaFree(p->k2_dev[i]);
  cudaFree(p->twiddles);
  cudaFree(p->twiddles32);
  cudaFree(p->sctab);
  cudaFree(p->obs_partial);
  cudaFree(p->obs_mask);
  cudaFree(p->red_partial);
  cudaFree(p->vi_dev);
  cudaFree(p->expv_dev);
  cudaFree(p->expk_dev);
  cudaFree(p->kbuf);
  if (p->g_exec) cudaGraphExecDestroy(p->g_exec);
  if (p->cap_stream) cudaStreamDestroy(p->cap_stream);
  for (int i = 0; i < 2; ++i)
    if (p->kin_stream[i]) cudaStreamDestroy(p->kin_stream[i]);
  for (int i = 0; i < 3; ++i)
    if (p->kin_ev[i]) cudaEventDestroy(p->kin_ev[i]);
  for (int i = 0; i < 4; ++i)
    if (p->pb_stream[i]) cudaStreamDestroy(p->pb_stream[i]);
  for (int i = 0; i < 5; ++i)
    if (p->pb_ev[i]) cudaEventDestroy(p->pb_ev[i]);
  for (auto g : p->pb_exec)
    if (g) cudaGraphExecDestroy(g);
  delete p;
  return CTAP_OK;
}

CTAP_API int ctap_pass(ctap_plan* p, int32_t kind, const void* in, void* out, void* stream) {
  Range nvtx("ctap_pass %lld", kind);
  if (!p || !in || !out) return fail(CTAP_EINVAL, "null argument");
  const bool diag = kind == ctap::PASS_Y_COPY || kind == ctap::PASS_X_COPY || kind == ctap::PASS_XB_COPY ||
                    kind == ctap::PASS_XP_COPY || kind == ctap::PASS_XP_KIN || (kind >= ctap::PASS_WX_COPY && kind <= ctap::PASS_WY_FWD);
  if (!diag && (kind < CTAP_PASS_Z_FWD || kind > CTAP_PASS_PX_KIN))
    return fail(CTAP_EINVAL, "unknown pass %d", kind);
  const bool blk = kind >= CTAP_PASS_Y_FWD_BLK && kind <= CTAP_PASS_Y_INV_BLK;
  if (blk && p->slab_p != 1) return fail(CTAP_EINVAL, "blocked k-space passes are single-GPU");
  if (blk && in == out && kind != CTAP_PASS_X_KIN_BLK) return fail(CTAP_EINVAL, "blocked y passes run out of place");
  const bool pen = kind >= CTAP_PASS_PZ_FIRST && kind <= CTAP_PASS_PX_KIN;
  if (pen != (p->pen_c > 0) && kind != CTAP_PASS_Z_FWD && kind != CTAP_PASS_Z_INV && !diag)
    return fail(CTAP_EINVAL, pen ? "pencil pass %d on a plan without a pencil grid" : "slab pass %d on a pencil plan",
                kind);
  if ((kind == CTAP_PASS_PZ_FIRST || kind == CTAP_PASS_PZ_LAST || kind == CTAP_PASS_PY_FWD ||
       kind == CTAP_PASS_PY_INV) && in == out)
    return fail(CTAP_EINVAL, "pencil pass %d runs out of place", kind);
  if ((kind == CTAP_PASS_PZ_MID || kind == CTAP_PASS_PX_KIN) && in != out)
    return fail(CTAP_EINVAL, "pencil pass %d runs in place", kind);
  if ((kind == CTAP_PASS_PZ_FIRST || kind == CTAP_PASS_PZ_MID || kind == CTAP_PASS_PZ_LAST) && !p->vi_dev)
    return fail(CTAP_EINVAL, "pass %d needs a plan with a potential", kind);
  if (kind == CTAP_PASS_Y_FWD_TO_PEERS || kind == CTAP_PASS_X_KIN_TO_PEERS) {
    void* const* tab = kind == CTAP_PASS_Y_FWD_TO_PEERS ? p->peer_y : p->peer_p;
    for (int q = 0; q < p->slab_p; ++q)
      if (!tab[q]) return fail(CTAP_EINVAL, "peer buffers not registered (ctap_set_peer_buffers)");
  }
  if (kind <= CTAP_PASS_Z_LAST && in != out) return fail(CTAP_EINVAL, "z passes run in place");
  if (p->pen_c && kind < CTAP_PASS_PZ_FIRST) return fail(CTAP_EINVAL, "pencil plans run the pencil passes only");
  if ((kind == CTAP_PASS_Z_FIRST || kind == CTAP_PASS_Z_MID || kind == CTAP_PASS_Z_LAST) && !p->vi_dev)
    return fail(CTAP_EINVAL, "plan has no potential");
  CUDA_TRY(ctap_run_pass(p, kind, in, out, (cudaStream_t)stream), "ctap_pass");
  return CTAP_OK;
}

CTAP_API int ctap_pass_zchunk(ctap_plan* p, int32_t kind, const void* in, void* out, int64_t z0, int64_t zn,
                              void* stream) {
  Range nvtx("ctap_pass_zchunk %lld", kind);
  if (!p || !in || !out) return fail(CTAP_EINVAL, "null argument");
  if (p->slab_p < 2 || p->pen_c) return fail(CTAP_EINVAL, "z-chunked passes serve slab plans (slab_p > 1)");
  if (kind != CTAP_PASS_Y_FWD_TO_PEER && kind != CTAP_PASS_X_KIN && kind != CTAP_PASS_Y_INV_FROM_PEER)
    return fail(CTAP_EINVAL, "pass %d has no z-chunked form", kind);
  if (zn <= 0 || zn % 8 || z0 < 0 || z0 + zn > p->n[2] || z0 % zn)
    return fail(CTAP_EINVAL, "z chunk [%lld, %lld) must be a multiple-of-8 slice of nz = %lld",
                (long long)z0, (long long)(z0 + zn), (long long)p->n[2]);
  if (kind == CTAP_PASS_X_KIN && (in != out || p->expk_dev))
    return fail(CTAP_EINVAL, "z-chunked kinetic pass runs in place without the exp(-ik^2dt/2) table");
  CUDA_TRY(ctap_run_pass_chunk(p, kind, in, out, z0, zn, (cudaStream_t)stream), "ctap_pass_zchunk");
  return CTAP_OK;
}

// y, [x K x^-1], y^-1 of one step.  With p->zchunk = W the three passes run
// per z chunk of W columns, so a chunk (nx ny W points) stays in L2 from the
// y pass to the y^-1 pass instead of making three HBM round trips.
static cudaError_t kin_block(ctap_plan* p, void* psi, cudaStream_t st) {
  const int64_t nz = p->n[2], W = p->zchunk;
  if (W <= 0 || W >= nz) {
    cudaError_t e = ctap_run_pass(p, CTAP_PASS_Y_FWD, psi, psi, st);
    if (e == cudaSuccess) e = ctap_run_pass(p, CTAP_PASS_X_KIN, psi, psi, st);
    if (e == cudaSuccess) e = ctap_run_pass(p, CTAP_PASS_Y_INV, psi, psi, st);
    return e;
  }
  // chunks alternate between two streams forked from (and joined back into)
  // st, so the FP64-bound x pass of one chunk co-runs with the HBM-bound y
  // passes of its neighbours (inside a graph capture this becomes two
  // parallel branches)
  cudaError_t e = cudaSuccess;
  for (int i = 0; i < 2 && e == cudaSuccess; ++i)
    if (!p->kin_stream[i]) e = cudaStreamCreateWithFlags(&p->kin_stream[i], cudaStreamNonBlocking);
  for (int i = 0; i < 3 && e == cudaSuccess; ++i)
    if (!p->kin_ev[i]) e = cudaEventCreateWithFlags(&p->kin_ev[i], cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventRecord(p->kin_ev[0], st);
  for (int i = 0; i < 2 && e == cudaSuccess; ++i) e = cudaStreamWaitEvent(p->kin_stream[i], p->kin_ev[0], 0);
  for (int64_t z0 = 0, c = 0; z0 < nz && e == cudaSuccess; z0 += W, ++c) {
    cudaStream_t s = p->kin_stream[c & 1];
    e = ctap_run_pass_z(p, CTAP_PASS_Y_FWD, psi, psi, z0, W, s);
    if (e == cudaSuccess) e = ctap_run_pass_z(p, CTAP_PASS_X_KIN, psi, psi, z0, W, s);
    if (e == cudaSuccess) e = ctap_run_pass_z(p, CTAP_PASS_Y_INV, psi, psi, z0, W, s);
  }
  for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
    e = cudaEventRecord(p->kin_ev[1 + i], p->kin_stream[i]);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, p->kin_ev[1 + i], 0);
  }
  return e;
}

// Position block by x-slabs: the passes between two x passes, [y^-1,
// z^-1 V z, y], are independent per x-plane, so each slab of x-planes runs
// its three passes back to back -- its psi and v_i stay in L2 between them --
// with consecutive slabs on kPBStreams streams (forked from and joined back
// into the caller's stream; graph branches under capture).  Slab size: three
// slabs' psi + v_i within ~80 MB of the 126 MB L2 (4 planes at 512^3); off
// when psi + v_i fit L2 anyway (launch-bound small grids).  CTAP_PBLOCK
// overrides (0 off, k planes).  Bitwise equal to the plane-order schedule:
// every pass computes each line and tile exactly as before.
constexpr int kPBStreams = 3;
static int64_t pblock_planes(const ctap_plan* p) {
  static const int64_t env = [] {
    const char* e = getenv("CTAP_PBLOCK");
    return e ? (int64_t)atoll(e) : (int64_t)-1;
  }();
  if (p->kbuf || p->zchunk || p->z2 || p->slab_p != 1) return 0;
  const size_t csz = p->dtype == CTAP_C64 ? 8 : 16;
  const double plane = (double)p->n[1] * p->n[2] * (csz + sizeof(double));
  int64_t v = env;
  if (v < 0) {
    // automatic for complex128 with y lines <= 512 points: the 1024-point y
    // ring and complex64's TMA y passes are persistent kernels that a
    // few-plane slab starves (1024^2 x 512: 18.3 -> 21.4 ms per step;
    // complex64 512^3: 2.82 -> 3.45 ms)
    if (p->dtype != CTAP_C128 || p->n[1] > 512 || plane * p->nx_local <= 126e6) return 0;
    v = 1;
    while (2 * v * plane * kPBStreams <= 80e6) v *= 2;
  }
  if (v <= 0 || v >= p->nx_local || p->nx_local % v) return 0;
  return v;
}
static int pblock_streams() {
  static const int v = [] {
    const char* e = getenv("CTAP_PBLOCK_STREAMS");
    return e ? atoi(e) : kPBStreams;
  }();
  return v < 1 ? 1 : v > 4 ? 4 : v;
}
// phase 1: slab's [z V_h] [y]; 0: [y^-1] [z^-1 V z] [y]; 2: [y^-1] [z^-1 V_h]
// (3: [y^-1] only, the observed segment end)
static cudaError_t pblock_triples(ctap_plan* p, void* psi, int phase, cudaStream_t st) {
  const int64_t planes = pblock_planes(p), ny = p->n[1], nz = p->n[2];
  const size_t csz = p->dtype == CTAP_C64 ? 8 : 16;
  const int ns = pblock_streams();
  cudaError_t e = cudaSuccess;
  if (ns > 1) {
    for (int i = 0; i < ns && e == cudaSuccess; ++i)
      if (!p->pb_stream[i]) e = cudaStreamCreateWithFlags(&p->pb_stream[i], cudaStreamNonBlocking);
    for (int i = 0; i <= ns && e == cudaSuccess; ++i)
      if (!p->pb_ev[i]) e = cudaEventCreateWithFlags(&p->pb_ev[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventRecord(p->pb_ev[0], st);
    for (int i = 0; i < ns && e == cudaSuccess; ++i) e = cudaStreamWaitEvent(p->pb_stream[i], p->pb_ev[0], 0);
  }
  static const int pdl = [] {
    const char* v = getenv("CTAP_PDL");
    return v ? atoi(v) : 1;
  }();
  for (int64_t x0 = 0, c = 0; x0 < p->nx_local && e == cudaSuccess; x0 += planes, ++c) {
    cudaStream_t s = ns > 1 ? p->pb_stream[c % ns] : st;
    // the first grid of each stream follows an event wait, not a grid
    ctap_pdl = pdl && c >= ns;
    ctap_plan t = *p;
    t.nx_local = planes;
    t.n[0] = planes;  // the y pass sizes its grid by n[0] / slab_p
    t.vi_dev = p->vi_dev + x0 * ny * nz;
    if (p->expv_dev) t.expv_dev = (char*)p->expv_dev + csz * (size_t)(x0 * ny * nz);
    void* ps = (char*)psi + csz * (size_t)(x0 * ny * nz);
    if (phase != 1) e = ctap_run_pass(&t, CTAP_PASS_Y_INV, ps, ps, s);
    if (phase != 3) {
      if (e == cudaSuccess)
        e = ctap_run_pass(&t, phase == 1 ? CTAP_PASS_Z_FIRST : phase == 0 ? CTAP_PASS_Z_MID : CTAP_PASS_Z_LAST, ps,
                          ps, s);
      if (e == cudaSuccess && phase != 2) e = ctap_run_pass(&t, CTAP_PASS_Y_FWD, ps, ps, s);
    }
  }
  ctap_pdl = 0;
  if (ns > 1)
    for (int i = 0; i < ns && e == cudaSuccess; ++i) {
      e = cudaEventRecord(p->pb_ev[1 + i], p->pb_stream[i]);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(st, p->pb_ev[1 + i], 0);
    }
  return e;
}

// One piece of the slab schedule: the segment start (phase 1: the slab
// triples alone) or an x pass followed by the triples of phase 0 / 2 / 3.
static cudaError_t pblock_piece(ctap_plan* p, void* psi, int phase, cudaStream_t s) {
  cudaError_t e = phase == 1 ? cudaSuccess : ctap_run_pass(p, CTAP_PASS_X_KIN, psi, psi, s);
  return e == cudaSuccess ? pblock_triples(p, psi, phase, s) : e;
}

// The same as a graph (hundreds of small launches), captured once per psi
// pointer and phase and replayed on st.
static cudaError_t pblock_graph(ctap_plan* p, void* psi, int phase, cudaStream_t st) {
  if (!graphs_enabled()) return pblock_piece(p, psi, phase, st);
  if (p->pb_psi != psi) {
    for (auto& g : p->pb_exec)
      if (g) {
        cudaGraphExecDestroy(g);
        g = nullptr;
      }
    p->pb_psi = psi;
  }
  cudaGraphExec_t& ex = p->pb_exec[phase];
  if (!ex) {
    cudaError_t e = cudaSuccess;
    if (!p->cap_stream) e = cudaStreamCreateWithFlags(&p->cap_stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamBeginCapture(p->cap_stream, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) return e;
    cudaGraph_t g = nullptr;
    cudaError_t ce = pblock_piece(p, psi, phase, p->cap_stream);
    cudaError_t ee = cudaStreamEndCapture(p->cap_stream, &g);
    if (ce == cudaSuccess) ce = ee;
    if (ce == cudaSuccess) ce = cudaGraphInstantiate(&ex, g, 0);
    if (g) cudaGraphDestroy(g);
    if (ce != cudaSuccess) {
      ex = nullptr;
      return ce;
    }
  }
  return cudaGraphLaunch(ex, st);
}

static int advance_pblock(ctap_plan* p, void* psi, int64_t n, cudaStream_t st) {
  CUDA_TRY(pblock_graph(p, psi, 1, st), "ctap_advance");
  int64_t j = 0;
  if (graphs_enabled() && n - 1 >= kGraphSteps) {
    if (p->g_exec == nullptr || p->g_psi != psi || p->g_steps != kGraphSteps) {
      if (p->g_exec) cudaGraphExecDestroy(p->g_exec);
      p->g_exec = nullptr;
      if (!p->cap_stream) CUDA_TRY(cudaStreamCreateWithFlags(&p->cap_stream, cudaStreamNonBlocking), "ctap_advance");
      cudaGraph_t g = nullptr;
      CUDA_TRY(cudaStreamBeginCapture(p->cap_stream, cudaStreamCaptureModeThreadLocal), "ctap_advance capture");
      cudaError_t ce = cudaSuccess;
      for (int m = 0; m < kGraphSteps && ce == cudaSuccess; ++m) {
        ce = ctap_run_pass(p, CTAP_PASS_X_KIN, psi, psi, p->cap_stream);
        if (ce == cudaSuccess) ce = pblock_triples(p, psi, 0, p->cap_stream);
      }
      cudaError_t ee = cudaStreamEndCapture(p->cap_stream, &g);
      if (ce == cudaSuccess) ce = ee;
      if (ce == cudaSuccess) ce = cudaGraphInstantiate(&p->g_exec, g, 0);
      if (g) cudaGraphDestroy(g);
      if (ce != cudaSuccess) {
        p->g_exec = nullptr;
        return cuda_fail(ce, "ctap_advance graph capture");
      }
      p->g_psi = psi;
      p->g_steps = kGraphSteps;
    }
    for (; j + kGraphSteps <= n - 1; j += kGraphSteps) CUDA_TRY(cudaGraphLaunch(p->g_exec, st), "ctap_advance");
  }
  for (; j < n; ++j) {
    CUDA_TRY(pblock_graph(p, psi, j < n - 1 ? 0 : p->skip_last ? 3 : 2, st), "ctap_advance");
  }
  return CTAP_OK;
}

CTAP_API int ctap_step_schedule(const ctap_plan* p, int64_t* slab_planes, int32_t* streams) {
  if (!p || !slab_planes || !streams) return fail(CTAP_EINVAL, "null argument");
  *slab_planes = pblock_planes(p);
  *streams = *slab_planes ? pblock_streams() : 1;
  return CTAP_OK;
}

CTAP_API int ctap_advance(ctap_plan* p, void* psi, int64_t n, void* stream) {
  Range nvtx("ctap_advance %lld steps", (long long)n);
  if (!p || !psi) return fail(CTAP_EINVAL, "null argument");
  if (n < 0) return fail(CTAP_EINVAL, "n_steps must be >= 0");
  if (p->slab_p != 1) return fail(CTAP_EINVAL, "ctap_advance drives single-GPU plans; use ctap_pass for slabs");
  if (!p->vi_dev) return fail(CTAP_EINVAL, "plan has no potential");
  if (n == 0) return CTAP_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (pblock_planes(p)) return advance_pblock(p, psi, n, st);
  CUDA_TRY(ctap_run_pass(p, CTAP_PASS_Z_FIRST, psi, psi, st), "ctap_advance");
  // interior steps in CUDA-graph chunks: one launch per kGraphSteps steps
  // instead of 4 (removes the per-kernel launch cost that dominates small grids)
  int64_t j = 0;
  if (graphs_enabled() && !p->kbuf && n - 1 >= kGraphSteps) {
    if (p->g_exec == nullptr || p->g_psi != psi || p->g_steps != kGraphSteps) {
      if (p->g_exec) cudaGraphExecDestroy(p->g_exec);
      p->g_exec = nullptr;
      if (!p->cap_stream) CUDA_TRY(cudaStreamCreateWithFlags(&p->cap_stream, cudaStreamNonBlocking), "ctap_advance");
      cudaGraph_t g = nullptr;
      CUDA_TRY(cudaStreamBeginCapture(p->cap_stream, cudaStreamCaptureModeThreadLocal), "ctap_advance capture");
      cudaError_t ce = cudaSuccess;
      for (int m = 0; m < kGraphSteps && ce == cudaSuccess; ++m) {
        ce = kin_block(p, psi, p->cap_stream);
        if (ce == cudaSuccess) ce = ctap_run_pass(p, CTAP_PASS_Z_MID, psi, psi, p->cap_stream);
      }
      cudaError_t ee = cudaStreamEndCapture(p->cap_stream, &g);
      if (ce == cudaSuccess) ce = ee;
      if (ce == cudaSuccess) ce = cudaGraphInstantiate(&p->g_exec, g, 0);
      if (g) cudaGraphDestroy(g);
      if (ce != cudaSuccess) {
        p->g_exec = nullptr;
        return cuda_fail(ce, "ctap_advance graph capture");
      }
      p->g_psi = psi;
      p->g_steps = kGraphSteps;
    }
    for (; j + kGraphSteps <= n - 1; j += kGraphSteps) CUDA_TRY(cudaGraphLaunch(p->g_exec, st), "ctap_advance");
  }
  for (; j < n; ++j) {
    if (p->kbuf) {
      CUDA_TRY(ctap_run_pass(p, ctap::PASS_Y_FWD_BLK, psi, p->kbuf, st), "ctap_advance");
      CUDA_TRY(ctap_run_pass(p, ctap::PASS_X_KIN_BLK, p->kbuf, p->kbuf, st), "ctap_advance");
      CUDA_TRY(ctap_run_pass(p, ctap::PASS_Y_INV_BLK, p->kbuf, psi, st), "ctap_advance");
    } else {
      CUDA_TRY(kin_block(p, psi, st), "ctap_advance");
    }
    if (j < n - 1 || !p->skip_last)
      CUDA_TRY(ctap_run_pass(p, j < n - 1 ? CTAP_PASS_Z_MID : CTAP_PASS_Z_LAST, psi, psi, st), "ctap_advance");
  }
  return CTAP_OK;
}

// ctap_advance followed by an observer event, the event's sums fused into the
// segment-end pass (evolve_real's advance + PopulationRecorder/EdgeMonitor,
// propagator.py:160-168, observables.py:74-110).
CTAP_API int ctap_advance_observe(ctap_plan* p, void* psi, int64_t n, const double* xs, const double* xb1,
                                  const double* xb2, int32_t margin, double* out, void* stream) {
  if (!p || !psi || !out || !xs) return fail(CTAP_EINVAL, "null argument");
  if ((xb1 == nullptr) != (xb2 == nullptr)) return fail(CTAP_EINVAL, "xb1 and xb2 must both be given");
  if (margin < 1) return fail(CTAP_EINVAL, "margin_cells must be >= 1");
  if (n < 0) return fail(CTAP_EINVAL, "n_steps must be >= 0");
  cudaStream_t st = (cudaStream_t)stream;
  if (n == 0 || p->slab_p != 1 || p->kbuf || p->mode != 0) {
    // nothing to fuse into (or a plan whose segment end is not the plain z
    // pass): the step(s), then the standalone reduction
    const int rc = ctap_advance(p, psi, n, stream);
    if (rc != CTAP_OK) return rc;
    CUDA_TRY(ctap_run_observe(p, psi, xs, xb1, xb2, margin, out, st), "ctap_advance_observe");
    return CTAP_OK;
  }
  if (!p->obs_partial)
    CUDA_TRY(cudaMalloc((void**)&p->obs_partial, sizeof(double) * 4 * ctap_z_blocks(p)), "ctap_advance_observe");
  // all but the last pass of the segment: ctap_advance of n steps minus its
  // final [z^-1 . Vh] (the same launches, graphs included)
  p->skip_last = 1;
  const int rc = ctap_advance(p, psi, n, stream);
  p->skip_last = 0;
  if (rc != CTAP_OK) return rc;
  if (xb1 && !p->obs_mask)
    CUDA_TRY(cudaMalloc((void**)&p->obs_mask, sizeof(uint16_t) * ctap_obs_mask_entries(p)), "ctap_advance_observe");
  CUDA_TRY(ctap_run_z_last_observe(p, psi, xs, xb1, xb2, margin, p->obs_partial, p->obs_mask, st),
           "ctap_advance_observe");
  CUDA_TRY(ctap_run_finalize5(p, p->obs_partial, ctap_z_blocks(p), out, xb1 != nullptr, st), "ctap_advance_observe");
  return CTAP_OK;
}

CTAP_API int ctap_fft3d(ctap_plan* p, void* data, int32_t direction, void* stream) {
  if (!p || !data) return fail(CTAP_EINVAL, "null argument");
  if (p->slab_p != 1) return fail(CTAP_EINVAL, "ctap_fft3d is single-GPU; slab plans compose ctap_pass");
  cudaStream_t st = (cudaStream_t)stream;
  if (direction < 0) {
    CUDA_TRY(ctap_run_pass(p, CTAP_PASS_Z_FWD, data, data, st), "ctap_fft3d");
    CUDA_TRY(ctap_run_pass(p, CTAP_PASS_Y_FWD, data, data, st), "ctap_fft3d");
    CUDA_TRY(ctap_run_pass(p, CTAP_PASS_X_FWD, data, data, st), "ctap_fft3d");
  } else {
    CUDA_TRY(ctap_run_pass(p, CTAP_PASS_X_INV, data, data, st), "ctap_fft3d");
    CUDA_TRY(ctap_run_pass(p, CTAP_PASS_Y_INV, data, data, st), "ctap_fft3d");
    CUDA_TRY(ctap_run_pass(p, CTAP_PASS_Z_INV, data, data, st), "ctap_fft3d");
  }
  return CTAP_OK;
}

CTAP_API int ctap_observe(ctap_plan* p, const void* psi, const double* xs, const double* xb1, const double* xb2,
                          int32_t margin, double* out, void* stream) {
  if (!p || !psi || !out || !xs) return fail(CTAP_EINVAL, "null argument");
  if ((xb1 == nullptr) != (xb2 == nullptr)) return fail(CTAP_EINVAL, "xb1 and xb2 must both be given");
  if (margin < 1) return fail(CTAP_EINVAL, "margin_cells must be >= 1");
  CUDA_TRY(ctap_run_observe(p, psi, xs, xb1, xb2, margin, out, (cudaStream_t)stream), "ctap_observe");
  return CTAP_OK;
}

CTAP_API int ctap_density_xz(ctap_plan* p, const void* psi, double* out, void* stream) {
  if (!p || !psi || !out) return fail(CTAP_EINVAL, "null argument");
  CUDA_TRY(ctap_run_density_xz(p, psi, out, (cudaStream_t)stream), "ctap_density_xz");
  return CTAP_OK;
}

CTAP_API int ctap_k2_sums(ctap_plan* p, const void* phi, double* out, void* stream) {
  if (!p || !phi || !out) return fail(CTAP_EINVAL, "null argument");
  if (p->pen_c) return fail(CTAP_EINVAL, "ctap_k2_sums takes slab (y-slab) layouts, not pencils");
  CUDA_TRY(ctap_run_k2_sums(p, phi, out, (cudaStream_t)stream), "ctap_k2_sums");
  return CTAP_OK;
}

CTAP_API int ctap_v_sums(ctap_plan* p, const void* psi, double* out, void* stream) {
  if (!p || !psi || !out) return fail(CTAP_EINVAL, "null argument");
  if (!p->v_dev) return fail(CTAP_EINVAL, "plan has no potential");
  CUDA_TRY(ctap_run_v_sums(p, psi, nullptr, out, (cudaStream_t)stream), "ctap_v_sums");
  return CTAP_OK;
}

CTAP_API int ctap_v_sums_with(ctap_plan* p, const void* psi, const double* v_dev, double* out, void* stream) {
  if (!p || !psi || !v_dev || !out) return fail(CTAP_EINVAL, "null argument");
  CUDA_TRY(ctap_run_v_sums(p, psi, v_dev, out, (cudaStream_t)stream), "ctap_v_sums_with");
  return CTAP_OK;
}

CTAP_API int ctap_set_peer_buffers(ctap_plan* p, int32_t which, void* const* ptrs, int32_t count) {
  if (!p) return fail(CTAP_EINVAL, "null argument");
  if (which != 0 && which != 1) return fail(CTAP_EINVAL, "which must be 0 (y-slab) or 1 (peer-major)");
  void** tab = which == 0 ? p->peer_y : p->peer_p;
  if (count == 0) {  // unregister (before the mappings are closed): the fused passes then fail with EINVAL
    for (int q = 0; q < 16; ++q) tab[q] = nullptr;
    return CTAP_OK;
  }
  if (!ptrs) return fail(CTAP_EINVAL, "null argument");
  if (count != p->slab_p || count > 16) return fail(CTAP_EINVAL, "expected %d peer buffers", p->slab_p);
  for (int q = 0; q < count; ++q) {
    if (!ptrs[q]) return fail(CTAP_EINVAL, "peer buffer %d is null", q);
    tab[q] = ptrs[q];
  }
  return CTAP_OK;
}

CTAP_API int ctap_ipc_handle(void* dev_ptr, void* handle64) {
  if (!dev_ptr || !handle64) return fail(CTAP_EINVAL, "null argument");
  cudaIpcMemHandle_t h;
  CUDA_TRY(cudaIpcGetMemHandle(&h, dev_ptr), "ctap_ipc_handle");
  std::memcpy(handle64, &h, sizeof h);
  return CTAP_OK;
}

CTAP_API int ctap_ipc_open(const void* handle64, void** dev_ptr) {
  if (!handle64 || !dev_ptr) return fail(CTAP_EINVAL, "null argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, sizeof h);
  CUDA_TRY(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess), "ctap_ipc_open");
  return CTAP_OK;
}

CTAP_API int ctap_ipc_close(void* dev_ptr) {
  if (!dev_ptr) return fail(CTAP_EINVAL, "null argument");
  CUDA_TRY(cudaIpcCloseMemHandle(dev_ptr), "ctap_ipc_close");
  return CTAP_OK;
}

// Stream-ordered flag barrier of the fused slab transport (stream memory
// operations on peer-mapped flags, no kernel spins and no collective):
// every rank writes `epoch` into its slot of every peer's flag array after
// its pass (the write carries a memory barrier, and the pass ends with a
// system-scope fence), then its stream waits until every peer has written
// `epoch` into its own array.  The waits are semaphore acquires in the
// stream front end, the mechanism cross-process event waits use.
typedef CUresult (*StreamWriteFn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*StreamWaitFn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

static void* driver_fn(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
    return nullptr;
  return p;
}

CTAP_API int ctap_flag_barrier(void* const* peer_flags, const void* my_flags, int32_t nranks, int32_t rank,
                               uint32_t epoch, void* stream) {
  if (!my_flags || nranks < 1 || rank < 0 || rank >= nranks) return fail(CTAP_EINVAL, "bad flag-barrier arguments");
  if (epoch == 0) {  // clear this rank's array (stream-ordered) before a new epoch sequence
    CUDA_TRY(cudaMemsetAsync(const_cast<void*>(my_flags), 0, 4 * (size_t)nranks, (cudaStream_t)stream),
             "ctap_flag_barrier");
    return CTAP_OK;
  }
  if (!peer_flags) return fail(CTAP_EINVAL, "bad flag-barrier arguments");
  static StreamWriteFn wr = (StreamWriteFn)driver_fn("cuStreamWriteValue32");
  static StreamWaitFn wt = (StreamWaitFn)driver_fn("cuStreamWaitValue32");
  if (!wr || !wt) return fail(CTAP_EUNSUPPORTED, "stream memory operations unavailable");
  CUstream st = (CUstream)stream;
  for (int q = 0; q < nranks; ++q) {
    if (q == rank) continue;
    if (!peer_flags[q]) return fail(CTAP_EINVAL, "peer flag array %d is null", q);
    const CUresult r = wr(st, (CUdeviceptr)((char*)peer_flags[q] + 4 * rank), epoch, CU_STREAM_WRITE_VALUE_DEFAULT);
    if (r != CUDA_SUCCESS) return fail(CTAP_ECUDA, "cuStreamWriteValue32 failed (%d)", (int)r);
  }
  // where the device supports it, the wait also flushes outstanding remote
  // writes, so peer stores ordered before the flag are visible to the next pass
  int dev = 0, can_flush = 0;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&can_flush, cudaDevAttrCanFlushRemoteWrites, dev);
  const unsigned wflags = CU_STREAM_WAIT_VALUE_GEQ | (can_flush ? CU_STREAM_WAIT_VALUE_FLUSH : 0u);
  for (int q = 0; q < nranks; ++q) {
    if (q == rank) continue;
    const CUresult r = wt(st, (CUdeviceptr)((const char*)my_flags + 4 * q), epoch, wflags);
    if (r != CUDA_SUCCESS) return fail(CTAP_ECUDA, "cuStreamWaitValue32 failed (%d)", (int)r);
  }
  return CTAP_OK;
}

CTAP_API int ctap_device_alloc(int64_t bytes, void** dev_ptr) {
  if (!dev_ptr || bytes <= 0) return fail(CTAP_EINVAL, "bad allocation request");
  CUDA_TRY(cudaMalloc(dev_ptr, (size_t)bytes), "ctap_device_alloc");
  CUDA_TRY(cudaMemset(*dev_ptr, 0, (size_t)bytes), "ctap_device_alloc");  // zeroed (flag arrays rely on it)
  return CTAP_OK;
}

CTAP_API int ctap_device_free(void* dev_ptr) {
  CUDA_TRY(cudaFree(dev_ptr), "ctap_device_free");
  return CTAP_OK;
}

CTAP_API int ctap_phase_field(ctap_plan* p, int32_t which, void* out, void* stream) {
  if (!p || !out) return fail(CTAP_EINVAL, "null argument");
  if (which < 0 || which > 2) return fail(CTAP_EINVAL, "which must be 0 (v_half), 1 (v_full) or 2 (k)");
  if (which < 2 && !p->vi_dev) return fail(CTAP_EINVAL, "plan has no potential");
  if (p->pen_c) return fail(CTAP_EINVAL, "ctap_phase_field takes slab plans");
  CUDA_TRY(ctap_run_phase_field(p, which, out, (cudaStream_t)stream), "ctap_phase_field");
  return CTAP_OK;
}

CTAP_API int ctap_scale(ctap_plan* p, void* psi, double divisor, void* stream) {
  if (!p || !psi) return fail(CTAP_EINVAL, "null argument");
  if (!(divisor > 0.0) || !std::isfinite(divisor)) return fail(CTAP_EINVAL, "divisor must be positive and finite");
  CUDA_TRY(ctap_run_scale(p, psi, divisor, (cudaStream_t)stream), "ctap_scale");
  return CTAP_OK;
}

CTAP_API int ctap_potential(const double* xs, int64_t nx, const double* ys, int64_t ny, const double* zs, int64_t nz,
                            const double* seg_a, const double* seg_b, const double* seg_cur, int64_t n_seg,
                            double b0x, double b0y, double b0z, double mu_eff, double mass, double omega_z,
                            double z_center, double pref, double* V_out, void* stream) {
  if (!xs || !ys || !zs || !V_out) return fail(CTAP_EINVAL, "null argument");
  if (n_seg < 0 || (n_seg > 0 && (!seg_a || !seg_b || !seg_cur))) return fail(CTAP_EINVAL, "bad segment arrays");
  if (nx <= 0 || ny <= 0 || nz <= 0) return fail(CTAP_EINVAL, "empty grid");
  CUDA_TRY(ctap_run_potential(xs, nx, ys, ny, zs, nz, seg_a, seg_b, seg_cur, n_seg, b0x, b0y, b0z, mu_eff, mass,
                              omega_z, z_center, pref, V_out, (cudaStream_t)stream),
           "ctap_potential");
  return CTAP_OK;
}

CTAP_API int ctap_slice_minima(const double* V_dev, int64_t nx, int64_t ny, int64_t nz, int64_t* count_dev,
                               int64_t* best_dev, void* stream) {
  if (!V_dev || !count_dev || !best_dev) return fail(CTAP_EINVAL, "null argument");
  if (nx <= 0 || ny <= 0 || nz <= 0) return fail(CTAP_EINVAL, "empty grid");
  if (nx * ny > (int64_t(1) << 31) || nz > (int64_t(1) << 30))
    return fail(CTAP_EUNSUPPORTED, "slice too large");
  CUDA_TRY(ctap_run_slice_minima(V_dev, nx, ny, nz, count_dev, best_dev, (cudaStream_t)stream),
           "ctap_slice_minima");
  return CTAP_OK;
}

}  // extern "C"
