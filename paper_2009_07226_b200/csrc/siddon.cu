// K1/K2: Siddon ray tracing of the parallel-beam system matrix.
//
// Bit-exact restatement of geometry.trace_ray (src/geometry.py:117-164) on
// the device: every float64 operation is issued as an explicitly rounded
// __dadd_rn/__dmul_rn/__ddiv_rn so no FMA contraction can change a bit.
// The merged, sorted crossing list of the reference (np.sort of both
// axes' plane crossings) is produced by merging the two monotone crossing
// sequences on the fly, so a ray needs O(1) state instead of O(N) scratch.
//
// One thread per ray; rays r = k*n_det + c.  Count pass -> host/cub scan ->
// fill pass writes (int32 flat voxel iz*N+ix, float64 length) in traversal
// order, the canonical CSR row order of src/geometry.py:214-220.
#include "xct_common.h"

namespace {

constexpr double kSegEps = 1e-12;  // src/geometry.py:38

struct Axis {
  double o, d;     // origin and direction component
  bool active;     // |d| >= 1e-15 (src/geometry.py:139)
  int i, step, end;// iteration over plane indices in ascending-t order
};

__device__ __forceinline__ double crossing(const Axis& a, int i, double half, double vox) {
  // planes = -half + vox*arange(g+1); crossings = (planes - o) / d
  double plane = __dadd_rn(-half, __dmul_rn(vox, (double)i));
  return __ddiv_rn(__dadd_rn(plane, -a.o), a.d);
}

// Calls emit(flat_index, length) for every kept segment of ray (k, c), in
// traversal order.  Returns the number of kept segments.
template <typename Emit>
__device__ int64_t trace(double cs, double sn, int c, int n_det, int g, double vox,
                         Emit emit) {
  // (c - (N-1)/2.0) * pitch; both terms are exact small halves
  const double rho = __dmul_rn(__dadd_rn((double)c, -0.5 * (double)(n_det - 1)), vox);
  Axis ax[2];
  ax[0].o = __dmul_rn(rho, -sn);  // rho * normal, normal = (-sin, cos)
  ax[1].o = __dmul_rn(rho, cs);
  ax[0].d = cs;
  ax[1].d = sn;
  const double half = __dmul_rn((double)g, vox) / 2.0;  // exact halving
  double t_enter = -INFINITY, t_exit = INFINITY;
  for (int a = 0; a < 2; ++a) {
    Axis& A = ax[a];
    A.active = fabs(A.d) >= 1e-15;
    if (!A.active) {
      if (!(-half < A.o && A.o < half)) return 0;
      continue;
    }
    double t0 = __ddiv_rn(__dadd_rn(-half, -A.o), A.d);
    double t1 = __ddiv_rn(__dadd_rn(half, -A.o), A.d);
    // python max/min: max(a, b) keeps a unless b > a
    double lo = t1 < t0 ? t1 : t0;
    double hi = t1 > t0 ? t1 : t0;
    if (lo > t_enter) t_enter = lo;
    if (hi < t_exit) t_exit = hi;
    if (A.d > 0) { A.i = 0; A.step = 1; A.end = g + 1; }
    else { A.i = g; A.step = -1; A.end = -1; }
  }
  const double eps = __dmul_rn(kSegEps, vox);
  if (t_enter >= __dadd_rn(t_exit, -eps)) return 0;

  // next crossing strictly inside (t_enter, t_exit) on each axis
  double nxt[2];
  auto advance = [&](int a) {
    Axis& A = ax[a];
    while (A.i != A.end) {
      double t = crossing(A, A.i, half, vox);
      A.i += A.step;
      if (t > t_enter && t < t_exit) { nxt[a] = t; return; }
      if (t >= t_exit) break;   // ascending sequence: nothing further inside
    }
    nxt[a] = INFINITY;
    A.i = A.end;
  };
  for (int a = 0; a < 2; ++a) {
    if (ax[a].active) advance(a); else nxt[a] = INFINITY;
  }

  int64_t kept = 0;
  double prev = t_enter;
  bool done = false;
  while (!done) {
    double t;
    if (nxt[0] <= nxt[1] && nxt[0] != INFINITY) { t = nxt[0]; advance(0); }
    else if (nxt[1] != INFINITY) { t = nxt[1]; advance(1); }
    else { t = t_exit; done = true; }
    double seg = __dadd_rn(t, -prev);
    if (seg > eps) {
      double mid = __dadd_rn(prev, __dmul_rn(0.5, seg));
      double px = __dadd_rn(ax[0].o, __dmul_rn(mid, ax[0].d));
      double pz = __dadd_rn(ax[1].o, __dmul_rn(mid, ax[1].d));
      long long ix = (long long)floor(__ddiv_rn(__dadd_rn(px, half), vox));
      long long iz = (long long)floor(__ddiv_rn(__dadd_rn(pz, half), vox));
      ix = ix < 0 ? 0 : (ix > g - 1 ? g - 1 : ix);
      iz = iz < 0 ? 0 : (iz > g - 1 ? g - 1 : iz);
      emit(kept, (int32_t)(iz * g + ix), seg);
      ++kept;
    }
    prev = t;
  }
  return kept;
}

__global__ void siddon_count_kernel(const double* __restrict__ cos_t,
                                    const double* __restrict__ sin_t, int k0, int k1,
                                    int n_det, int g, double vox, int64_t* counts) {
  int64_t n_rays = (int64_t)(k1 - k0) * n_det;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_rays;
       r += (int64_t)gridDim.x * blockDim.x) {
    int k = k0 + (int)(r / n_det), c = (int)(r % n_det);
    counts[r] = trace(cos_t[k], sin_t[k], c, n_det, g, vox,
                      [](int64_t, int32_t, double) {});
  }
}

__global__ void siddon_fill_kernel(const double* __restrict__ cos_t,
                                   const double* __restrict__ sin_t, int k0, int k1,
                                   int n_det, int g, double vox,
                                   const int64_t* __restrict__ rowptr,
                                   int32_t* __restrict__ indices,
                                   double* __restrict__ values) {
  int64_t n_rays = (int64_t)(k1 - k0) * n_det;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_rays;
       r += (int64_t)gridDim.x * blockDim.x) {
    int k = k0 + (int)(r / n_det), c = (int)(r % n_det);
    int64_t base = rowptr[r];
    int32_t* ip = indices + base;
    double* vp = values + base;
    trace(cos_t[k], sin_t[k], c, n_det, g, vox,
          [&](int64_t j, int32_t flat, double len) {
            XCT_CHECK(j < rowptr[r + 1] - base && flat >= 0 && flat < g * g);
            ip[j] = flat;
            vp[j] = len;
          });
  }
}

int grid_for(int64_t n, int block) {
  int64_t b = (n + block - 1) / block;
  if (b > 148 * 64) b = 148 * 64;
  return (int)(b < 1 ? 1 : b);
}

int check_args(const double* cs, const double* sn, int k0, int k1, int n_det, int g,
               double vox) {
  if (!cs || !sn) return xct::fail(XCT_EINVAL, "siddon: null angle table");
  if (k0 < 0 || k1 < k0) return xct::fail(XCT_EINVAL, "siddon: bad angle range");
  if (n_det < 1 || g < 1) return xct::fail(XCT_EINVAL, "siddon: N must be >= 1");
  if ((int64_t)g * g > INT32_MAX) return xct::fail(XCT_EINVAL, "siddon: grid too large for int32 ids");
  if (!(vox > 0)) return xct::fail(XCT_EINVAL, "siddon: voxel_size must be positive");
  return XCT_OK;
}

}  // namespace

extern "C" int xct_siddon_count(const double* d_cos, const double* d_sin, int k0, int k1,
                                int n_det, int grid_n, double voxel_size,
                                int64_t* d_counts, void* stream) {
  int st = check_args(d_cos, d_sin, k0, k1, n_det, grid_n, voxel_size);
  if (st) return st;
  int64_t n = (int64_t)(k1 - k0) * n_det;
  if (n == 0) return XCT_OK;
  siddon_count_kernel<<<grid_for(n, 128), 128, 0, (cudaStream_t)stream>>>(
      d_cos, d_sin, k0, k1, n_det, grid_n, voxel_size, d_counts);
  XCT_CUDA_CHECK_LAUNCH("siddon_count");
  return XCT_OK;
}

extern "C" int xct_siddon_fill(const double* d_cos, const double* d_sin, int k0, int k1,
                               int n_det, int grid_n, double voxel_size,
                               const int64_t* d_rowptr, int32_t* d_indices,
                               double* d_values, void* stream) {
  int st = check_args(d_cos, d_sin, k0, k1, n_det, grid_n, voxel_size);
  if (st) return st;
  int64_t n = (int64_t)(k1 - k0) * n_det;
  if (n == 0) return XCT_OK;
  siddon_fill_kernel<<<grid_for(n, 128), 128, 0, (cudaStream_t)stream>>>(
      d_cos, d_sin, k0, k1, n_det, grid_n, voxel_size, d_rowptr, d_indices, d_values);
  XCT_CUDA_CHECK_LAUNCH("siddon_fill");
  return XCT_OK;
}

// ---------------------------------------------------------------------------
// Column-range restriction of a device CSR (streamed operator build: the
// back-projection format is built per band of voxels, src/matrixstore.py:
// 151-165 restricts rows the same way).  Count pass, then fill with columns
// rebased to col_lo; rows keep their order and their entries' CSR order.
namespace {
__global__ void csr_filter_count_kernel(const int64_t* __restrict__ indptr,
                                        const int32_t* __restrict__ indices, int64_t n_rows,
                                        int32_t lo, int32_t hi, int64_t* __restrict__ counts) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    int64_t c = 0;
    for (int64_t j = indptr[r]; j < indptr[r + 1]; ++j) c += (indices[j] >= lo && indices[j] < hi);
    counts[r] = c;
  }
}
__global__ void csr_filter_fill_kernel(const int64_t* __restrict__ indptr,
                                       const int32_t* __restrict__ indices,
                                       const double* __restrict__ values, int64_t n_rows,
                                       int32_t lo, int32_t hi, const int64_t* __restrict__ out_ptr,
                                       int32_t* __restrict__ out_idx, double* __restrict__ out_val) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    int64_t o = out_ptr[r];
    for (int64_t j = indptr[r]; j < indptr[r + 1]; ++j) {
      const int32_t c = indices[j];
      if (c >= lo && c < hi) {
        out_idx[o] = c - lo;
        out_val[o] = values[j];
        ++o;
      }
    }
  }
}
}  // namespace

extern "C" int xct_csr_filter_cols(const int64_t* d_indptr, const int32_t* d_indices,
                                   const double* d_values, int64_t n_rows, int32_t col_lo,
                                   int32_t col_hi, int64_t* d_counts, const int64_t* d_out_ptr,
                                   int32_t* d_out_idx, double* d_out_val, void* stream) {
  if (!d_indptr || n_rows < 0 || col_hi < col_lo)
    return xct::fail(XCT_EINVAL, "csr_filter_cols: bad argument");
  if (n_rows == 0) return XCT_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (d_counts) {
    csr_filter_count_kernel<<<grid_for(n_rows, 128), 128, 0, s>>>(d_indptr, d_indices, n_rows,
                                                                 col_lo, col_hi, d_counts);
  } else {
    if (!d_out_ptr || !d_out_idx || !d_out_val)
      return xct::fail(XCT_EINVAL, "csr_filter_cols: fill pass needs output arrays");
    csr_filter_fill_kernel<<<grid_for(n_rows, 128), 128, 0, s>>>(
        d_indptr, d_indices, d_values, n_rows, col_lo, col_hi, d_out_ptr, d_out_idx, d_out_val);
  }
  XCT_CUDA_CHECK_LAUNCH("csr_filter_cols");
  return XCT_OK;
}

// ---------------------------------------------------------------------------
// Row/column-mapped restriction of a device CSR (per-rank blocks of the
// data-partitioned operator, built streamed: src/matrixstore.py:130-165).
// Keeps entry j of row r when row_keep[r] (or row_keep == NULL) and
// col_map[col] >= 0; the kept column is rewritten to col_map[col].
namespace {
__global__ void csr_map_count_kernel(const int64_t* __restrict__ indptr,
                                     const int32_t* __restrict__ indices, int64_t n_rows,
                                     const uint8_t* __restrict__ row_keep,
                                     const int32_t* __restrict__ col_map,
                                     int64_t* __restrict__ counts) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    int64_t c = 0;
    if (!row_keep || row_keep[r])
      for (int64_t j = indptr[r]; j < indptr[r + 1]; ++j) c += col_map[indices[j]] >= 0;
    counts[r] = c;
  }
}
__global__ void csr_map_fill_kernel(const int64_t* __restrict__ indptr,
                                    const int32_t* __restrict__ indices,
                                    const double* __restrict__ values, int64_t n_rows,
                                    const uint8_t* __restrict__ row_keep,
                                    const int32_t* __restrict__ col_map,
                                    const int64_t* __restrict__ out_ptr,
                                    int32_t* __restrict__ out_idx, double* __restrict__ out_val) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    if (row_keep && !row_keep[r]) continue;
    int64_t o = out_ptr[r];
    for (int64_t j = indptr[r]; j < indptr[r + 1]; ++j) {
      const int32_t m = col_map[indices[j]];
      if (m >= 0) {
        out_idx[o] = m;
        out_val[o] = values[j];
        ++o;
      }
    }
  }
}
}  // namespace

extern "C" int xct_csr_filter_map(const int64_t* d_indptr, const int32_t* d_indices,
                                  const double* d_values, int64_t n_rows,
                                  const uint8_t* d_row_keep, const int32_t* d_col_map,
                                  int64_t* d_counts, const int64_t* d_out_ptr,
                                  int32_t* d_out_idx, double* d_out_val, void* stream) {
  if (!d_indptr || !d_col_map || n_rows < 0) return xct::fail(XCT_EINVAL, "csr_filter_map: bad argument");
  if (n_rows == 0) return XCT_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (d_counts) {
    csr_map_count_kernel<<<grid_for(n_rows, 128), 128, 0, s>>>(d_indptr, d_indices, n_rows,
                                                              d_row_keep, d_col_map, d_counts);
  } else {
    if (!d_out_ptr || !d_out_idx || !d_out_val)
      return xct::fail(XCT_EINVAL, "csr_filter_map: fill pass needs output arrays");
    csr_map_fill_kernel<<<grid_for(n_rows, 128), 128, 0, s>>>(
        d_indptr, d_indices, d_values, n_rows, d_row_keep, d_col_map, d_out_ptr, d_out_idx,
        d_out_val);
  }
  XCT_CUDA_CHECK_LAUNCH("csr_filter_map");
  return XCT_OK;
}

// ---------------------------------------------------------------------------
// K11: matrix-free FP32 projector pair over one chunk of 16 slices -- the
// same Siddon rays traced on the fly (no stored operator), lengths rounded
// to f32, accumulation in f32.  An independent implementation of the
// single-precision operator (cf. engine.project, src/engine.py:119-166, in
// "single" mode) used to check the staged K6 path at sizes whose FP32
// staged operator does not fit next to the FP16 one (bench.py in-run
// checks).  Back projection scatters with vector f32 atomics, so its sums
// are order-nondeterministic at the last bit.
namespace {
constexpr int kMfSlices = 16;

__global__ void siddon_project_f32_kernel(const double* __restrict__ cos_t,
                                          const double* __restrict__ sin_t, int k0, int k1,
                                          int n_det, int g, double vox,
                                          const float4* __restrict__ x, float4* __restrict__ y) {
  const int64_t n_rays = (int64_t)(k1 - k0) * n_det;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_rays;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int k = k0 + (int)(r / n_det), c = (int)(r % n_det);
    float4 acc[kMfSlices / 4];
#pragma unroll
    for (int q = 0; q < kMfSlices / 4; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    trace(cos_t[k], sin_t[k], c, n_det, g, vox, [&](int64_t, int32_t flat, double len) {
      const float l = (float)len;
      const float4* xp = x + (int64_t)flat * (kMfSlices / 4);
#pragma unroll
      for (int q = 0; q < kMfSlices / 4; ++q) {
        const float4 v = __ldg(xp + q);
        acc[q].x = fmaf(v.x, l, acc[q].x);
        acc[q].y = fmaf(v.y, l, acc[q].y);
        acc[q].z = fmaf(v.z, l, acc[q].z);
        acc[q].w = fmaf(v.w, l, acc[q].w);
      }
    });
#pragma unroll
    for (int q = 0; q < kMfSlices / 4; ++q) y[r * (kMfSlices / 4) + q] = acc[q];
  }
}

__global__ void siddon_backproject_f32_kernel(const double* __restrict__ cos_t,
                                              const double* __restrict__ sin_t, int k0, int k1,
                                              int n_det, int g, double vox,
                                              const float4* __restrict__ y, float4* __restrict__ x) {
  const int64_t n_rays = (int64_t)(k1 - k0) * n_det;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_rays;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int k = k0 + (int)(r / n_det), c = (int)(r % n_det);
    float4 yv[kMfSlices / 4];
#pragma unroll
    for (int q = 0; q < kMfSlices / 4; ++q) yv[q] = y[r * (kMfSlices / 4) + q];
    trace(cos_t[k], sin_t[k], c, n_det, g, vox, [&](int64_t, int32_t flat, double len) {
      const float l = (float)len;
      float4* xp = x + (int64_t)flat * (kMfSlices / 4);
#pragma unroll
      for (int q = 0; q < kMfSlices / 4; ++q)
        atomicAdd(xp + q, make_float4(yv[q].x * l, yv[q].y * l, yv[q].z * l, yv[q].w * l));
    });
  }
}
}  // namespace

extern "C" int xct_siddon_project_f32(const double* d_cos, const double* d_sin, int k0, int k1,
                                      int n_det, int grid_n, double voxel_size, int adjoint,
                                      const float* d_in, float* d_out, void* stream) {
  int st = check_args(d_cos, d_sin, k0, k1, n_det, grid_n, voxel_size);
  if (st) return st;
  if (!d_in || !d_out) return xct::fail(XCT_EINVAL, "siddon_project_f32: null vector");
  const int64_t n = (int64_t)(k1 - k0) * n_det;
  if (n == 0) return XCT_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (adjoint)
    siddon_backproject_f32_kernel<<<grid_for(n, 128), 128, 0, s>>>(
        d_cos, d_sin, k0, k1, n_det, grid_n, voxel_size, (const float4*)d_in, (float4*)d_out);
  else
    siddon_project_f32_kernel<<<grid_for(n, 128), 128, 0, s>>>(
        d_cos, d_sin, k0, k1, n_det, grid_n, voxel_size, (const float4*)d_in, (float4*)d_out);
  XCT_CUDA_CHECK_LAUNCH("siddon_project_f32");
  return XCT_OK;
}
