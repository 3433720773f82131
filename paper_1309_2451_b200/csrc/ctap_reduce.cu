// Deterministic reductions over |psi|^2: observer sums (norm, guide
// populations, edge mass), energy sums, the y-integrated density map and the
// normalisation scale.  Reference: observables.py:74-110, qgrid.py:150-162,
// propagator.py:176-195.
//
// Every reduction is two fixed-shape stages (grid-stride partial sums per
// block in a fixed order, then one block summing the partials in a fixed
// tree), so results are bitwise reproducible run to run with no float atomics
// (reference determinism rule: test_propagator.py:147-154).
#include "ctap_device.cuh"
#include "ctap_internal.h"

namespace ctap {

constexpr int kRedThreads = 256;

template <int NV>
__device__ __forceinline__ void block_reduce_store(double (&acc)[NV], double* __restrict__ out) {
  __shared__ double sh[NV][kRedThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double v = acc[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) sh[k][warp] = v;
  }
  __syncthreads();
  if (threadIdx.x < NV) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kRedThreads / 32; ++w) s += sh[threadIdx.x][w];
    out[threadIdx.x] = s;
  }
}

template <int NV, typename F>
__global__ void __launch_bounds__(kRedThreads) reduce_kernel(F f, int64_t n, double* __restrict__ partial) {
  double acc[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) acc[k] = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) f(i, acc);
  block_reduce_store<NV>(acc, partial + (size_t)blockIdx.x * NV);
}

template <int NV>
__global__ void __launch_bounds__(kRedThreads) finalize_kernel(const double* __restrict__ partial, int nblocks,
                                                               double* __restrict__ out) {
  double acc[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) acc[k] = 0.0;
  for (int b = threadIdx.x; b < nblocks; b += blockDim.x) {
#pragma unroll
    for (int k = 0; k < NV; ++k) acc[k] += partial[(size_t)b * NV + k];
  }
  block_reduce_store<NV>(acc, out);
}

template <typename CV>
struct ObserveF {
  const CV* psi;
  const double* xs;
  const double* xb1;
  const double* xb2;
  int64_t nyz, ny, nz, nx_global, x_off, ny_global, y_off;
  int margin;
  int lyz, lz;  // log2(ny nz), log2(nz): every extent is a power of two (shifts, not divisions)
  __device__ __forceinline__ void operator()(int64_t i, double (&acc)[5]) const {
    const CV a = psi[i];
    const double rho = (double)a.x * a.x + (double)a.y * a.y;
    const int64_t x = i >> lyz;
    const int64_t y = (i >> lz) & (ny - 1);
    const int64_t z = i & (nz - 1);
    acc[0] += rho;
    if (xb1 != nullptr) {
      double xv = xs[x];
      bool in_l = xv < xb1[z];
      bool in_r = xv >= xb2[z];
      if (in_l) acc[1] += rho;
      if (in_r) acc[3] += rho;
      if (!(in_l || in_r)) acc[2] += rho;
    }
    int64_t gx = x + x_off;
    int64_t gy = y + y_off;
    bool edge = gx < margin || gx >= nx_global - margin || gy < margin || gy >= ny_global - margin ||
                z < margin || z >= nz - margin;
    if (edge) acc[4] += rho;
  }
};

template <typename CV>
struct K2F {
  const CV* phi;
  const double* kx2;
  const double* ky2;
  const double* kz2;
  int64_t nylz, nyl, nz, y_off;
  int lylz, lz;  // log2(nyl nz), log2(nz)
  __device__ __forceinline__ void operator()(int64_t i, double (&acc)[2]) const {
    const CV a = phi[i];
    const double rho = (double)a.x * a.x + (double)a.y * a.y;
    const int64_t x = i >> lylz;
    const int64_t y = (i >> lz) & (nyl - 1);
    const int64_t z = i & (nz - 1);
    double k2 = (kx2[x] + ky2[y + y_off]) + kz2[z];
    acc[0] += k2 * rho;
    acc[1] += rho;
  }
};

template <typename CV>
struct VF {
  const CV* psi;
  const double* V;
  __device__ __forceinline__ void operator()(int64_t i, double (&acc)[2]) const {
    const CV a = psi[i];
    const double rho = (double)a.x * a.x + (double)a.y * a.y;
    acc[0] += V[i] * rho;
    acc[1] += rho;
  }
};

template <int NV, typename F>
static cudaError_t run_reduce(const ctap_plan* p, F f, int64_t n, double* out, cudaStream_t st) {
  reduce_kernel<NV><<<p->red_blocks, kRedThreads, 0, st>>>(f, n, p->red_partial);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  finalize_kernel<NV><<<1, kRedThreads, 0, st>>>(p->red_partial, p->red_blocks, out);
  return cudaGetLastError();
}

template <typename CV>
__global__ void density_xz_kernel(const CV* __restrict__ psi, int64_t nxl, int64_t ny, int64_t nz,
                                  double* __restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nxl * nz) return;
  int64_t x = i / nz, z = i - (i / nz) * nz;
  const CV* base = psi + x * ny * nz + z;
  double s = 0.0;
  for (int64_t y = 0; y < ny; ++y) {
    const CV a = base[y * nz];
    s += (double)a.x * a.x + (double)a.y * a.y;
  }
  out[i] = s;
}

__global__ void scale_kernel(double2* __restrict__ psi, int64_t n, double d) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    double2 a = psi[i];
    psi[i] = make_double2(a.x / d, a.y / d);
  }
}
__global__ void scale_kernel(float2* __restrict__ psi, int64_t n, double d) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const float df = (float)d;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    float2 a = psi[i];
    psi[i] = make_float2(a.x / df, a.y / df);
  }
}

}  // namespace ctap

using namespace ctap;

template <typename CV>
static cudaError_t observe_t(const ctap_plan* p, const void* psi, const double* xs, const double* xb1,
                             const double* xb2, int margin, double* out, cudaStream_t st) {
  ObserveF<CV> f;
  f.psi = (const CV*)psi;
  f.xs = xs;
  f.xb1 = xb1;
  f.xb2 = xb2;
  f.nyz = p->ny_pos * p->n[2];
  f.ny = p->ny_pos;
  f.nz = p->n[2];
  f.nx_global = p->n[0];
  f.ny_global = p->n[1];
  // slab: x block slab_r; pencil: x block a, y block b
  f.x_off = (int64_t)(p->pen_c ? p->pen_a : p->slab_r) * p->nx_local;
  f.y_off = p->pen_c ? (int64_t)p->pen_b * p->ny_pos : 0;
  f.margin = margin;
  f.lyz = ilog2i(f.nyz);
  f.lz = ilog2i(f.nz);
  return run_reduce<5>(p, f, p->nx_local * f.nyz, out, st);
}

cudaError_t ctap_run_observe(const ctap_plan* p, const void* psi, const double* xs, const double* xb1,
                             const double* xb2, int margin, double* out, cudaStream_t st) {
  return p->dtype == CTAP_C64 ? observe_t<float2>(p, psi, xs, xb1, xb2, margin, out, st)
                              : observe_t<double2>(p, psi, xs, xb1, xb2, margin, out, st);
}

template <typename CV>
static cudaError_t k2_t(const ctap_plan* p, const void* phi, double* out, cudaStream_t st) {
  K2F<CV> f;
  f.phi = (const CV*)phi;
  f.kx2 = p->k2_dev[0];
  f.ky2 = p->k2_dev[1];
  f.kz2 = p->k2_dev[2];
  f.nyl = p->n[1] / p->slab_p;
  f.nz = p->n[2];
  f.nylz = f.nyl * f.nz;
  f.y_off = (int64_t)p->slab_r * f.nyl;
  f.lylz = ilog2i(f.nylz);
  f.lz = ilog2i(f.nz);
  return run_reduce<2>(p, f, p->n[0] * f.nylz, out, st);
}

struct PartialF {  // the fused z pass's warp partials [total, left, right, edge]
  const double* partial;
  __device__ __forceinline__ void operator()(int64_t i, double (&acc)[4]) const {
#pragma unroll
    for (int k = 0; k < 4; ++k) acc[k] += partial[i * 4 + k];
  }
};

// [total, left, right, edge] -> [total, left, total - left - right, right, edge]
// (no partition: the guide sums are 0, as ctap_observe reports them)
__global__ void obs_layout_kernel(const double* __restrict__ s4, double* __restrict__ out, int part) {
  if (threadIdx.x == 0) {
    const double t = s4[0], l = s4[1], r = s4[2], e = s4[3];
    out[0] = t;
    out[1] = l;
    out[2] = part ? (t - l) - r : 0.0;
    out[3] = r;
    out[4] = e;
  }
}

// fixed-order sum of the fused z pass's warp partials (ctap_advance_observe):
// the two-stage grid reduction of the observer sums (a single block walking
// the partials would be latency-bound: ~0.4 ms at 512^3), then the middle
// guide as total - left - right
cudaError_t ctap_run_finalize5(const ctap_plan* p, const double* partial, int64_t npartials, double* out,
                               int part, cudaStream_t st) {
  PartialF f{partial};
  double* s4 = p->red_partial + 8 * (int64_t)p->red_blocks - 8;  // past the grid partials (red_blocks x 4 used)
  cudaError_t e = run_reduce<4>(p, f, npartials, s4, st);
  if (e != cudaSuccess) return e;
  obs_layout_kernel<<<1, 32, 0, st>>>(s4, out, part);
  return cudaGetLastError();
}

cudaError_t ctap_run_k2_sums(const ctap_plan* p, const void* phi, double* out, cudaStream_t st) {
  return p->dtype == CTAP_C64 ? k2_t<float2>(p, phi, out, st) : k2_t<double2>(p, phi, out, st);
}

template <typename CV>
static cudaError_t v_t(const ctap_plan* p, const void* psi, const double* V, double* out, cudaStream_t st) {
  VF<CV> f;
  f.psi = (const CV*)psi;
  f.V = V;
  return run_reduce<2>(p, f, p->nx_local * p->ny_pos * p->n[2], out, st);
}

// V = nullptr: the plan's own potential
cudaError_t ctap_run_v_sums(const ctap_plan* p, const void* psi, const double* V, double* out, cudaStream_t st) {
  if (!V) V = p->v_dev;
  return p->dtype == CTAP_C64 ? v_t<float2>(p, psi, V, out, st) : v_t<double2>(p, psi, V, out, st);
}

cudaError_t ctap_run_density_xz(const ctap_plan* p, const void* psi, double* out, cudaStream_t st) {
  int64_t n = p->nx_local * p->n[2];
  int threads = 256;
  const unsigned blocks = (unsigned)((n + threads - 1) / threads);
  if (p->dtype == CTAP_C64)
    density_xz_kernel<<<blocks, threads, 0, st>>>((const float2*)psi, p->nx_local, p->ny_pos, p->n[2], out);
  else
    density_xz_kernel<<<blocks, threads, 0, st>>>((const double2*)psi, p->nx_local, p->ny_pos, p->n[2], out);
  return cudaGetLastError();
}

cudaError_t ctap_run_scale(const ctap_plan* p, void* psi, double d, cudaStream_t st) {
  int64_t n = p->nx_local * p->ny_pos * p->n[2];
  if (p->dtype == CTAP_C64)
    scale_kernel<<<p->red_blocks, kRedThreads, 0, st>>>((float2*)psi, n, d);
  else
    scale_kernel<<<p->red_blocks, kRedThreads, 0, st>>>((double2*)psi, n, d);
  return cudaGetLastError();
}
