// Trapping potential of the three-wire chip on the grid (one-time setup).
// Reference: magfield.py:107-144 (_potential_kernel, numba, parallel over z).
//
//   V(r) = mu_eff |b0 + sum_s w_s (u_s x d_s)| + 1/2 m w_z^2 (z - z_c)^2
//
// This file is compiled with -fmad=false: every product and sum is rounded
// separately, in the reference's operation order, with IEEE division and
// square root, and segments are accumulated sequentially in reference order.
// That makes V bit-identical to the reference's numba kernel (which LLVM
// does not contract), which the 1e-10 propagation parity depends on: the
// CTAP phase V*dt/hbar is >= 1312 rad per step.
#include "ctap_internal.h"

namespace ctap {

constexpr int kSegChunk = 128;
constexpr int kPotThreads = 256;

struct SegPre {  // per-segment quantities that do not depend on the point
  double ax, ay, az, ux, uy, uz, len, pc;
};

// per segment: e = b - a, len = |e|, u = e/len, pc = pref * current
__global__ void segment_prep_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                    const double* __restrict__ cur, int64_t n, double pref,
                                    SegPre* __restrict__ out) {
  int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  double ax = a[3 * s], ay = a[3 * s + 1], az = a[3 * s + 2];
  double ex = b[3 * s] - ax;
  double ey = b[3 * s + 1] - ay;
  double ez = b[3 * s + 2] - az;
  double len = sqrt(ex * ex + ey * ey + ez * ez);
  SegPre p;
  p.ax = ax;
  p.ay = ay;
  p.az = az;
  p.ux = ex / len;
  p.uy = ey / len;
  p.uz = ez / len;
  p.len = len;
  p.pc = pref * cur[s];
  out[s] = p;
}

__global__ void __launch_bounds__(kPotThreads)
    potential_kernel(const double* __restrict__ xs, const double* __restrict__ ys, const double* __restrict__ zs,
                     int64_t nx, int64_t ny, int64_t nz, const SegPre* __restrict__ segs, int64_t nseg,
                     double b0x, double b0y, double b0z, double mu_eff, double mass, double omega_z,
                     double z_center, double* __restrict__ out) {
  __shared__ SegPre sh[kSegChunk];
  const int64_t n = nx * ny * nz;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool active = i < n;
  const int64_t ii = active ? i : 0;
  const int64_t ix = ii / (ny * nz);
  const int64_t iy = (ii / nz) % ny;
  const int64_t iz = ii % nz;
  const double x = xs[ix], y = ys[iy], z = zs[iz];
  double bx = b0x, by = b0y, bz = b0z;
  for (int64_t s0 = 0; s0 < nseg; s0 += kSegChunk) {
    const int cnt = (int)((nseg - s0) < kSegChunk ? (nseg - s0) : kSegChunk);
    __syncthreads();
    if (threadIdx.x < cnt) sh[threadIdx.x] = segs[s0 + threadIdx.x];
    __syncthreads();
    for (int k = 0; k < cnt; ++k) {
      const SegPre& sg = sh[k];
      double r1x = x - sg.ax;
      double r1y = y - sg.ay;
      double r1z = z - sg.az;
      double t1 = r1x * sg.ux + r1y * sg.uy + r1z * sg.uz;
      double t2 = t1 - sg.len;
      double dx = r1x - t1 * sg.ux;
      double dy = r1y - t1 * sg.uy;
      double dz = r1z - t1 * sg.uz;
      double d2 = dx * dx + dy * dy + dz * dz;
      if (d2 > 0.0) {
        double n1 = sqrt(d2 + t1 * t1);
        double n2 = sqrt(d2 + t2 * t2);
        double w = sg.pc * (t1 / n1 - t2 / n2) / d2;
        bx += w * (sg.uy * dz - sg.uz * dy);
        by += w * (sg.uz * dx - sg.ux * dz);
        bz += w * (sg.ux * dy - sg.uy * dx);
      }
    }
  }
  if (active) {
    double vz = 0.5 * mass * omega_z * omega_z * (z - z_center) * (z - z_center);
    out[i] = mu_eff * sqrt(bx * bx + by * by + bz * bz) + vz;
  }
}

}  // namespace ctap

using namespace ctap;

cudaError_t ctap_run_potential(const double* xs, int64_t nx, const double* ys, int64_t ny, const double* zs,
                               int64_t nz, const double* seg_a, const double* seg_b, const double* seg_cur,
                               int64_t n_seg, double b0x, double b0y, double b0z, double mu_eff, double mass,
                               double omega_z, double z_center, double pref, double* V_out, cudaStream_t st) {
  SegPre* pre = nullptr;
  cudaError_t e = cudaSuccess;
  if (n_seg > 0) {
    e = cudaMallocAsync((void**)&pre, sizeof(SegPre) * (size_t)n_seg, st);
    if (e != cudaSuccess) return e;
    segment_prep_kernel<<<(unsigned)((n_seg + 255) / 256), 256, 0, st>>>(seg_a, seg_b, seg_cur, n_seg, pref, pre);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) {
    int64_t n = nx * ny * nz;
    potential_kernel<<<(unsigned)((n + kPotThreads - 1) / kPotThreads), kPotThreads, 0, st>>>(
        xs, ys, zs, nx, ny, nz, pre, n_seg, b0x, b0y, b0z, mu_eff, mass, omega_z, z_center, V_out);
    e = cudaGetLastError();
  }
  if (pre) {
    cudaError_t e2 = cudaFreeAsync(pre, st);
    if (e == cudaSuccess) e = e2;
  }
  return e;
}
