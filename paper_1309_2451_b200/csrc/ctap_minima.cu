// Transverse minima of every z slice of V (reference magfield.py:188-208,
// _find_slice_minima), the per-slice scan of assemble_potential (:239-240)
// and build_partition (observables.py:35-60).
//
// A point (i, j) of slice z with 1 <= i < nx-1, 1 <= j < ny-1 is a minimum
// when   V < V[i-1,j],  V <= V[i+1,j],  V < V[i,j-1],  V <= V[i,j+1]
// (the reference's strict/non-strict pattern, NaN never qualifies).  The
// device returns, per slice, the number of minima and the three lowest by
// (V, row-major index i*ny + j) -- the reference keeps all minima when there
// are at most three and the three lowest by value otherwise; the parabolic
// refinement and the x ordering of those <= 3 points run on the host.
//
// Layout: V is (nx, ny, nz), z fastest.  Lane l of a warp owns slice
// z0 + l, so every load of a warp is one 256-byte row segment; a thread walks
// a row i along j keeping V[i, j-1..j+1] in registers and loads the rows
// i-1 and i+1, i.e. 3 loads per point.  Blocks split the rows of a 32-slice
// chunk; partial top-3 lists are merged in a fixed order (deterministic).
#include <cstdint>

#include "ctap_internal.h"

namespace ctap {

struct Cand {
  double v;
  int64_t lin;  // i * ny + j, or -1 (empty)
};

__device__ __forceinline__ bool before(const Cand& a, const Cand& b) {
  if (b.lin < 0) return a.lin >= 0;
  if (a.lin < 0) return false;
  return a.v < b.v || (a.v == b.v && a.lin < b.lin);
}

struct Top3 {
  Cand c[3];
  int64_t n;
  __device__ __forceinline__ void init() {
    n = 0;
#pragma unroll
    for (int k = 0; k < 3; ++k) c[k] = Cand{0.0, -1};
  }
  __device__ __forceinline__ void insert(const Cand& x) {
    if (!before(x, c[2])) return;
    if (before(x, c[1])) {
      c[2] = c[1];
      if (before(x, c[0])) {
        c[1] = c[0];
        c[0] = x;
      } else {
        c[1] = x;
      }
    } else {
      c[2] = x;
    }
  }
  __device__ __forceinline__ void merge(const Top3& o) {
    n += o.n;
#pragma unroll
    for (int k = 0; k < 3; ++k)
      if (o.c[k].lin >= 0) insert(o.c[k]);
  }
};

constexpr int kRowsPerBlock = 8;  // warps per block, each walks its own rows

__global__ void __launch_bounds__(32 * kRowsPerBlock)
    minima_scan_kernel(const double* __restrict__ V, int nx, int ny, int nz, int nsplit, Top3* partial) {
  __shared__ Top3 sh[kRowsPerBlock][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int zc = blockIdx.x / nsplit, s = blockIdx.x - zc * nsplit;
  const int z = zc * 32 + lane;
  // interior rows 1 .. nx-2 split evenly over the nsplit blocks of this chunk
  const int rows = nx - 2;
  const int r0 = 1 + (int)((int64_t)rows * s / nsplit), r1 = 1 + (int)((int64_t)rows * (s + 1) / nsplit);
  Top3 acc;
  acc.init();
  if (z < nz) {
    const int64_t sj = nz, si = (int64_t)ny * nz;
    for (int i = r0 + w; i < r1; i += kRowsPerBlock) {
      const double* row = V + i * si + z;
      double vl = __ldg(row), vc = __ldg(row + sj);
      for (int j = 1; j < ny - 1; ++j) {
        const double vr = __ldg(row + (j + 1) * sj);
        const double vu = __ldg(row - si + j * sj), vd = __ldg(row + si + j * sj);
        if (vc < vu && vc <= vd && vc < vl && vc <= vr) {
          ++acc.n;
          acc.insert(Cand{vc, (int64_t)i * ny + j});
        }
        vl = vc;
        vc = vr;
      }
    }
  }
  sh[w][lane] = acc;
  __syncthreads();
  if (w == 0) {
    for (int k = 1; k < kRowsPerBlock; ++k) acc.merge(sh[k][lane]);
    if (z < nz) partial[(int64_t)s * nz + z] = acc;
  }
}

__global__ void minima_merge_kernel(const Top3* __restrict__ partial, int nz, int nsplit, int64_t* count,
                                    int64_t* best) {
  const int z = blockIdx.x * blockDim.x + threadIdx.x;
  if (z >= nz) return;
  Top3 acc;
  acc.init();
  for (int s = 0; s < nsplit; ++s) acc.merge(partial[(int64_t)s * nz + z]);
  count[z] = acc.n;
#pragma unroll
  for (int k = 0; k < 3; ++k) best[3 * z + k] = acc.c[k].lin;
}

}  // namespace ctap

using namespace ctap;

// count[nz]: minima per slice; best[3 nz]: row-major indices i*ny + j of the
// (up to) three lowest minima by (V, index), -1 padded.  Device pointers.
cudaError_t ctap_run_slice_minima(const double* V, int64_t nx, int64_t ny, int64_t nz, int64_t* count,
                                  int64_t* best, cudaStream_t st) {
  if (nx < 3 || ny < 3) {
    cudaError_t e = cudaMemsetAsync(count, 0, sizeof(int64_t) * nz, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(best, 0xff, sizeof(int64_t) * 3 * nz, st);
    return e;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int nchunk = (int)((nz + 31) / 32);
  int nsplit = 2 * sms / nchunk;
  if (nsplit < 1) nsplit = 1;
  if (nsplit > nx - 2) nsplit = (int)(nx - 2);
  Top3* partial = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&partial, sizeof(Top3) * nsplit * nz, st);
  if (e != cudaSuccess) return e;
  minima_scan_kernel<<<nchunk * nsplit, 32 * kRowsPerBlock, 0, st>>>(V, (int)nx, (int)ny, (int)nz, nsplit,
                                                                      partial);
  e = cudaGetLastError();
  if (e == cudaSuccess) {
    minima_merge_kernel<<<(unsigned)((nz + 127) / 128), 128, 0, st>>>(partial, (int)nz, nsplit, count, best);
    e = cudaGetLastError();
  }
  cudaError_t f = cudaFreeAsync(partial, st);
  return e != cudaSuccess ? e : f;
}
