/* Plain-C restatement of the reference potential kernel -- TEST ORACLE ONLY.
 *
 * Restates magfield.py:107-144 (_potential_kernel, numba @njit(parallel=True))
 * of /root/reference/pkg/src/ctapsim: for every grid point, the wire field is
 * accumulated segment by segment, in segment order, with the closed-form
 * finite-segment Biot-Savart law, then V = mu_eff |B| + 1/2 m w_z^2 (z-zc)^2.
 * Compiled with -ffp-contract=off (no FMA), IEEE division and sqrt: this is
 * bit-identical to the numba kernel (pinned by tests/test_oracle_golden.py).
 * Points are independent, so splitting the z range over threads (as numba's
 * prange over iz, magfield.py:113) does not change any result bit.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>

static void potential_range(int64_t z_lo, int64_t z_hi, const double* xs, int64_t nx, const double* ys, int64_t ny, const double* zs, int64_t nz,
                      const double* seg_a, const double* seg_b, const double* seg_cur, int64_t ns, double b0x,
                      double b0y, double b0z, double mu_eff, double mass, double omega_z, double z_center,
                      double pref, double* out) {
  (void)nz;
  for (int64_t iz = z_lo; iz < z_hi; ++iz) {
    double z = zs[iz];
    double vz = 0.5 * mass * omega_z * omega_z * (z - z_center) * (z - z_center);
    for (int64_t ix = 0; ix < nx; ++ix) {
      double x = xs[ix];
      for (int64_t iy = 0; iy < ny; ++iy) {
        double y = ys[iy];
        double bx = b0x, by = b0y, bz = b0z;
        for (int64_t s = 0; s < ns; ++s) {
          double r1x = x - seg_a[3 * s + 0];
          double r1y = y - seg_a[3 * s + 1];
          double r1z = z - seg_a[3 * s + 2];
          double ex = seg_b[3 * s + 0] - seg_a[3 * s + 0];
          double ey = seg_b[3 * s + 1] - seg_a[3 * s + 1];
          double ez = seg_b[3 * s + 2] - seg_a[3 * s + 2];
          double length = sqrt(ex * ex + ey * ey + ez * ez);
          double ux = ex / length, uy = ey / length, uz = ez / length;
          double t1 = r1x * ux + r1y * uy + r1z * uz;
          double t2 = t1 - length;
          double dx = r1x - t1 * ux;
          double dy = r1y - t1 * uy;
          double dz = r1z - t1 * uz;
          double d2 = dx * dx + dy * dy + dz * dz;
          if (d2 > 0.0) {
            double n1 = sqrt(d2 + t1 * t1);
            double n2 = sqrt(d2 + t2 * t2);
            double w = pref * seg_cur[s] * (t1 / n1 - t2 / n2) / d2;
            bx += w * (uy * dz - uz * dy);
            by += w * (uz * dx - ux * dz);
            bz += w * (ux * dy - uy * dx);
          }
        }
        out[(ix * ny + iy) * nz + iz] = mu_eff * sqrt(bx * bx + by * by + bz * bz) + vz;
      }
    }
  }
}

typedef struct {
  int64_t z_lo, z_hi;
  const double *xs, *ys, *zs, *seg_a, *seg_b, *seg_cur;
  int64_t nx, ny, nz, ns;
  double b0x, b0y, b0z, mu_eff, mass, omega_z, z_center, pref;
  double* out;
} job_t;

static void* worker(void* arg) {
  job_t* j = (job_t*)arg;
  potential_range(j->z_lo, j->z_hi, j->xs, j->nx, j->ys, j->ny, j->zs, j->nz, j->seg_a, j->seg_b, j->seg_cur, j->ns,
                  j->b0x, j->b0y, j->b0z, j->mu_eff, j->mass, j->omega_z, j->z_center, j->pref, j->out);
  return 0;
}

void oracle_potential(const double* xs, int64_t nx, const double* ys, int64_t ny, const double* zs, int64_t nz,
                      const double* seg_a, const double* seg_b, const double* seg_cur, int64_t ns, double b0x,
                      double b0y, double b0z, double mu_eff, double mass, double omega_z, double z_center,
                      double pref, double* out, int threads) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  if (threads > nz) threads = (int)nz;
  pthread_t tid[256];
  job_t jobs[256];
  for (int t = 0; t < threads; ++t) {
    job_t j = {nz * t / threads, nz * (t + 1) / threads, xs, ys, zs, seg_a, seg_b, seg_cur, nx, ny, nz, ns,
               b0x, b0y, b0z, mu_eff, mass, omega_z, z_center, pref, out};
    jobs[t] = j;
    pthread_create(&tid[t], 0, worker, &jobs[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(tid[t], 0);
}
