// K7 / K8 / K9: normalization, CGLS vector updates and float64 dots.
//
//   normalize        matrixstore.normalize      src/matrixstore.py:290-305
//   store / load     solver._VectorStore        src/solver.py:84-108
//   x/r/p updates    solver.cgls_solve          src/solver.py:172-186
//   dots             solver._dot                src/solver.py:111-112
//
// All reductions are deterministic: a fixed grid writes per-block f64
// partials that one block sums in a fixed order.  Max-abs reductions use
// atomicMax on the IEEE bits of |v| widened to f64 (order free, exact;
// NaN bits compare above +inf so non-finite data is detected).
// "load" of a stored vector: dtype 0 f64, 1 f32, 2 f16 payload * f32 factor
// rounded in f32 -- exactly payload.astype(f32) * np.float32(factor).
#include <cuda_fp16.h>

#include <algorithm>
#include <cstring>

#include "xct_common.h"

namespace {

constexpr int kThreads = 256;
constexpr int kRedBlocks = 148 * 8;   // fixed => deterministic partials

__device__ __forceinline__ double load_as_f64(const void* v, int dtype, float f, int64_t i) {
  if (dtype == 0) return ((const double*)v)[i];
  if (dtype == 1) return (double)((const float*)v)[i];
  return (double)__fmul_rn(__half2float(((const __half*)v)[i]), f);
}

__device__ __forceinline__ float load_f32(const void* v, int dtype, float f, int64_t i) {
  if (dtype == 1) return ((const float*)v)[i];
  return __fmul_rn(__half2float(((const __half*)v)[i]), f);
}

// 4 consecutive elements at i (multiple of 4) as f32: 16-byte load of f32,
// 8-byte load of f16 (x factor, rounded in f32 -- as load_f32)
__device__ __forceinline__ float4 load4_f32(const void* v, int dtype, float f, int64_t i) {
  if (dtype == 1) return *reinterpret_cast<const float4*>((const float*)v + i);
  const uint2 h = *reinterpret_cast<const uint2*>((const __half*)v + i);
  const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&h.x));
  const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&h.y));
  return make_float4(__fmul_rn(a.x, f), __fmul_rn(a.y, f), __fmul_rn(b.x, f), __fmul_rn(b.y, f));
}

__device__ __forceinline__ unsigned long long abs_bits(double x) {
  return (unsigned long long)__double_as_longlong(fabs(x));
}

__device__ double block_sum(double v) {
  __shared__ double red[32];
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
  __syncthreads();
  return t;
}

__device__ unsigned long long block_max(unsigned long long v) {
  __shared__ unsigned long long red[32];
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long u = __shfl_xor_sync(0xffffffffu, v, o);
    v = u > v ? u : v;
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  unsigned long long t = 0;
  if (threadIdx.x == 0)
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t = red[i] > t ? red[i] : t;
  __syncthreads();
  return t;
}

__global__ void final_sum_kernel(const double* partials, int n, double* out) {
  double v = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) v += partials[i];
  v = block_sum(v);
  if (threadIdx.x == 0) out[0] = v;
}

int blocks_for(int64_t n) {
  int64_t b = (n + kThreads - 1) / kThreads;
  if (b > kRedBlocks) b = kRedBlocks;
  return (int)(b < 1 ? 1 : b);
}

// ---- strided (element-major, slice-minor) inputs of pipeline._apply --------

__global__ void chunk_maxabs_strided(const void* v, int in_f64, int64_t n, int64_t n_slices,
                                     int64_t rs, int ff, unsigned long long* maxbits) {
  const int c = blockIdx.y;
  const int64_t j0 = (int64_t)c * ff;
  const int64_t w = (n_slices - j0) < ff ? (n_slices - j0) : ff;
  unsigned long long m = 0;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n * w;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = t / w, j = j0 + t % w;
    double x = in_f64 ? ((const double*)v)[i * rs + j] : (double)((const float*)v)[i * rs + j];
    unsigned long long b = abs_bits(x);
    m = b > m ? b : m;
  }
  m = block_max(m);
  if (threadIdx.x == 0 && m) atomicMax(&maxbits[c], m);
}

template <typename Out>
__device__ __forceinline__ Out cast_store(double v64, float v32, bool from64);

template <> __device__ __forceinline__ double cast_store<double>(double v64, float v32, bool f) {
  return f ? v64 : (double)v32;
}
template <> __device__ __forceinline__ float cast_store<float>(double v64, float v32, bool f) {
  return f ? (float)v64 : v32;   // f64 -> f32 round to nearest even
}
template <> __device__ __forceinline__ __half cast_store<__half>(double v64, float v32, bool f) {
  return f ? __double2half(v64) : __float2half_rn(v32);  // direct RNE casts
}

template <typename Out>
__global__ void normalize_strided(const void* v, int in_f64, int64_t n, int64_t n_slices,
                                  int64_t rs, int ff, int f_dev, const double* factors,
                                  Out* out) {
  const int c = blockIdx.y;
  const double fac = factors[c];
  const float fac32 = (float)fac;
  Out* oc = out + (int64_t)c * n * f_dev;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n * f_dev;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = t / f_dev;
    int jj = (int)(t % f_dev);
    int64_t j = (int64_t)c * ff + jj;
    Out o;
    if (jj < ff && j < n_slices) {
      if (in_f64) o = cast_store<Out>(__ddiv_rn(((const double*)v)[i * rs + j], fac), 0.f, true);
      else o = cast_store<Out>(0.0, __fdiv_rn(((const float*)v)[i * rs + j], fac32), false);
    } else {
      o = cast_store<Out>(0.0, 0.f, false);
    }
    oc[t] = o;
  }
}

// ---- chunked persistent vectors [n_chunks][n][f_dev] -----------------------

__global__ void chunk_maxabs_chunked_vec_k(const void* v, int dtype, float fv, int64_t per_chunk,
                                           unsigned long long* maxbits) {
  const int c = blockIdx.y;
  const int64_t base = (int64_t)c * per_chunk;
  unsigned long long m = 0;
  for (int64_t t = 4 * (blockIdx.x * (int64_t)blockDim.x + threadIdx.x); t < per_chunk;
       t += 4 * (int64_t)gridDim.x * blockDim.x) {
    const float4 x = load4_f32(v, dtype, fv, base + t);
    const float e[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const unsigned long long b = abs_bits((double)e[k]);
      m = b > m ? b : m;
    }
  }
  m = block_max(m);
  if (threadIdx.x == 0 && m) atomicMax(&maxbits[c], m);
}

__global__ void chunk_maxabs_chunked_k(const void* v, int dtype, float fv, int64_t per_chunk,
                                       unsigned long long* maxbits) {
  const int c = blockIdx.y;
  const int64_t base = (int64_t)c * per_chunk;
  unsigned long long m = 0;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < per_chunk;
       t += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long b = abs_bits(load_as_f64(v, dtype, fv, base + t));
    m = b > m ? b : m;
  }
  m = block_max(m);
  if (threadIdx.x == 0 && m) atomicMax(&maxbits[c], m);
}

// f32/f16 input, f32/f16 output, per_chunk % 4 == 0: four elements per step
template <typename Out>
__global__ void normalize_chunked_vec_k(const void* v, int dtype, float fv, int64_t per_chunk,
                                        const double* factors, Out* out) {
  const int c = blockIdx.y;
  const int64_t base = (int64_t)c * per_chunk;
  const float fac = (float)factors[c];
  for (int64_t t = 4 * (blockIdx.x * (int64_t)blockDim.x + threadIdx.x); t < per_chunk;
       t += 4 * (int64_t)gridDim.x * blockDim.x) {
    const float4 x = load4_f32(v, dtype, fv, base + t);
    const float e[4] = {__fdiv_rn(x.x, fac), __fdiv_rn(x.y, fac), __fdiv_rn(x.z, fac),
                        __fdiv_rn(x.w, fac)};
    if constexpr (sizeof(Out) == 4) {
      *reinterpret_cast<float4*>((float*)out + base + t) = make_float4(e[0], e[1], e[2], e[3]);
    } else {
      __half2 lo = __floats2half2_rn(e[0], e[1]), hi = __floats2half2_rn(e[2], e[3]);
      uint2 pk;
      pk.x = *reinterpret_cast<unsigned*>(&lo);
      pk.y = *reinterpret_cast<unsigned*>(&hi);
      *reinterpret_cast<uint2*>((__half*)out + base + t) = pk;
    }
  }
}

template <typename Out>
__global__ void normalize_chunked_k(const void* v, int dtype, float fv, int64_t per_chunk,
                                    const double* factors, Out* out) {
  const int c = blockIdx.y;
  const int64_t base = (int64_t)c * per_chunk;
  const double fac = factors[c];
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < per_chunk;
       t += (int64_t)gridDim.x * blockDim.x) {
    Out o;
    if (dtype == 0) o = cast_store<Out>(__ddiv_rn(((const double*)v)[base + t], fac), 0.f, true);
    else o = cast_store<Out>(0.0, __fdiv_rn(load_f32(v, dtype, fv, base + t), (float)fac), false);
    out[base + t] = o;
  }
}

__global__ void dot_partial_kernel(const void* a, const void* b, int dtype, int64_t n, float fa,
                                   float fb, double* partials) {
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    s += load_as_f64(a, dtype, fa, i) * load_as_f64(b, dtype, fb, i);
  s = block_sum(s);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

__global__ void maxabs_kernel(const void* v, int dtype, int64_t n, float fv,
                              unsigned long long* maxbits) {
  unsigned long long m = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long b = abs_bits(load_as_f64(v, dtype, fv, i));
    m = b > m ? b : m;
  }
  m = block_max(m);
  if (threadIdx.x == 0 && m) atomicMax(maxbits, m);
}

// out = load(a) + s * load(b); two roundings in the work dtype.
// mode 0: write out (f32/f64); mode 1: max|out| only; mode 2: write f16
// (out / factor) and sum load(stored)^2 into per-block partials.
__global__ void axpy_kernel(const void* a, int at, float fa, const void* b, int bt, float fb,
                            double s, int64_t n, void* out, int ot, float ofac, int mode,
                            unsigned long long* maxbits, double* partials) {
  const bool f64 = at == 0;
  const float s32 = (float)s;
  unsigned long long m = 0;
  double sq = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (f64) {
      double v = ((const double*)a)[i];
      if (b) v = __dadd_rn(v, __dmul_rn(s, ((const double*)b)[i]));
      ((double*)out)[i] = v;
      continue;
    }
    float v = load_f32(a, at, fa, i);
    if (b) v = __fadd_rn(v, __fmul_rn(s32, load_f32(b, bt, fb, i)));
    if (mode == 0) {
      ((float*)out)[i] = v;
    } else if (mode == 1) {
      unsigned long long bb = abs_bits((double)v);
      m = bb > m ? bb : m;
    } else {
      __half h = __float2half_rn(__fdiv_rn(v, ofac));
      ((__half*)out)[i] = h;
      double back = (double)__fmul_rn(__half2float(h), ofac);
      sq += back * back;
    }
  }
  if (mode == 1) {
    m = block_max(m);
    if (threadIdx.x == 0 && m) atomicMax(maxbits, m);
  } else if (mode == 2 && partials) {
    sq = block_sum(sq);
    if (threadIdx.x == 0) partials[blockIdx.x] = sq;
  }
}

// Vector form of axpy_kernel for f32/f16 operands (n % 4 == 0): the same
// per-element arithmetic, four consecutive elements per thread and step.
template <int MODE>
__global__ void axpy_vec_kernel(const void* a, int at, float fa, const void* b, int bt, float fb,
                                float s32, int64_t n, void* out, float ofac,
                                unsigned long long* maxbits, double* partials) {
  unsigned long long m = 0;
  double sq = 0.0;
  for (int64_t i = 4 * (blockIdx.x * (int64_t)blockDim.x + threadIdx.x); i < n;
       i += 4 * (int64_t)gridDim.x * blockDim.x) {
    float4 v = load4_f32(a, at, fa, i);
    if (b) {
      const float4 w = load4_f32(b, bt, fb, i);
      v.x = __fadd_rn(v.x, __fmul_rn(s32, w.x));
      v.y = __fadd_rn(v.y, __fmul_rn(s32, w.y));
      v.z = __fadd_rn(v.z, __fmul_rn(s32, w.z));
      v.w = __fadd_rn(v.w, __fmul_rn(s32, w.w));
    }
    if (MODE == 0) {
      *reinterpret_cast<float4*>((float*)out + i) = v;
    } else if (MODE == 1) {
      const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const unsigned long long bb = abs_bits((double)e[k]);
        m = bb > m ? bb : m;
      }
    } else {
      const __half h0 = __float2half_rn(__fdiv_rn(v.x, ofac));
      const __half h1 = __float2half_rn(__fdiv_rn(v.y, ofac));
      const __half h2 = __float2half_rn(__fdiv_rn(v.z, ofac));
      const __half h3 = __float2half_rn(__fdiv_rn(v.w, ofac));
      __half2 lo = __halves2half2(h0, h1), hi = __halves2half2(h2, h3);
      uint2 pk;
      pk.x = *reinterpret_cast<unsigned*>(&lo);
      pk.y = *reinterpret_cast<unsigned*>(&hi);
      *reinterpret_cast<uint2*>((__half*)out + i) = pk;
      const __half hh[4] = {h0, h1, h2, h3};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const double back = (double)__fmul_rn(__half2float(hh[k]), ofac);
        sq += back * back;
      }
    }
  }
  if (MODE == 1) {
    m = block_max(m);
    if (threadIdx.x == 0 && m) atomicMax(maxbits, m);
  } else if (MODE == 2 && partials) {
    sq = block_sum(sq);
    if (threadIdx.x == 0) partials[blockIdx.x] = sq;
  }
}

template <typename Out>
__global__ void chunk_from_f64_k(const double* in, int64_t n, int64_t n_slices, int ff,
                                 int f_dev, int64_t n_chunks, Out* out) {
  const int64_t total = n_chunks * n * f_dev;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t c = t / (n * f_dev), rem = t % (n * f_dev);
    int64_t i = rem / f_dev;
    int jj = (int)(rem % f_dev);
    int64_t j = c * ff + jj;
    double v = (jj < ff && j < n_slices) ? in[i * n_slices + j] : 0.0;
    out[t] = (Out)v;
  }
}

__global__ void unchunk_f64_k(const void* in, int dtype, float fin, int64_t n, int64_t n_slices,
                              int ff, int f_dev, double* out) {
  const int64_t total = n * n_slices;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = t / n_slices, j = t % n_slices;
    int64_t c = j / ff;
    int jj = (int)(j % ff);
    out[t] = load_as_f64(in, dtype, fin, (c * n + i) * f_dev + jj);
  }
}


// Row block [r0, r0+nr) of a row-major (n, n_slices) f64/f32 array (the
// caller's measurements, src/solver.py:137: Y = y.astype(f64)) -> the
// chunked work layout: out[(c*n + r0+i)*f_dev + jj] = wd(v) (f64, or f32 by
// round-to-nearest like ndarray.astype(float32)); also max|v| (f64 bits),
// max|wd(v)| and per-block f64 partial sums of v*v (deterministic order).
template <typename In, typename Out>
__global__ void rows_to_chunked_k(const In* __restrict__ in, int64_t r0, int64_t nr, int64_t n,
                                  int64_t n_slices, int ff, int f_dev, Out* __restrict__ out,
                                  unsigned long long* max_in, unsigned long long* max_out,
                                  double* partials) {
  const int64_t total = nr * n_slices;
  unsigned long long mi = 0, mo = 0;
  double sq = 0.0;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / n_slices, j = t % n_slices;
    const double v = (double)in[t];
    const Out w = (Out)in[t];
    out[((j / ff) * n + r0 + i) * f_dev + (j % ff)] = w;
    const unsigned long long bi = abs_bits(v), bo = abs_bits((double)w);
    mi = bi > mi ? bi : mi;
    mo = bo > mo ? bo : mo;
    sq += v * v;
  }
  mi = block_max(mi);
  mo = block_max(mo);
  sq = block_sum(sq);
  if (threadIdx.x == 0) {
    if (max_in && mi) atomicMax(max_in, mi);
    if (max_out && mo) atomicMax(max_out, mo);
    if (partials) partials[blockIdx.x] = sq;
  }
}

// rows [r0, r0+nr) of a chunked vector -> row-major (nr, n_slices) f64
__global__ void unchunk_rows_f64_k(const void* in, int dtype, float fin, int64_t n, int64_t r0,
                                   int64_t nr, int64_t n_slices, int ff, int f_dev, double* out) {
  const int64_t total = nr * n_slices;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / n_slices, j = t % n_slices;
    out[t] = load_as_f64(in, dtype, fin, ((j / ff) * n + r0 + i) * f_dev + (j % ff));
  }
}
}  // namespace

extern "C" int xct_chunk_maxabs(const void* d_v, int in_f64, int64_t n, int64_t n_slices,
                                int64_t row_stride, int32_t ffactor, int64_t n_chunks,
                                uint64_t* d_maxbits, void* stream) {
  if (!d_v || !d_maxbits || ffactor < 1) return xct::fail(XCT_EINVAL, "chunk_maxabs: bad argument");
  if (n == 0 || n_chunks == 0) return XCT_OK;
  int64_t per = n * ffactor;
  int gx = blocks_for(per);
  if (gx > 512) gx = 512;
  chunk_maxabs_strided<<<dim3(gx, (unsigned)n_chunks), kThreads, 0, (cudaStream_t)stream>>>(
      d_v, in_f64, n, n_slices, row_stride, ffactor, (unsigned long long*)d_maxbits);
  XCT_CUDA_CHECK_LAUNCH("chunk_maxabs");
  return XCT_OK;
}

extern "C" int xct_normalize(const void* d_v, int in_f64, int64_t n, int64_t n_slices,
                             int64_t row_stride, int32_t ffactor, int64_t n_chunks,
                             int32_t f_dev, const double* d_factors, int precision,
                             void* d_out, void* stream) {
  if (!d_v || !d_out || !d_factors || ffactor < 1 || f_dev < ffactor)
    return xct::fail(XCT_EINVAL, "normalize: bad argument");
  if (n == 0 || n_chunks == 0) return XCT_OK;
  int gx = blocks_for(n * f_dev);
  if (gx > 512) gx = 512;
  dim3 grid(gx, (unsigned)n_chunks);
  cudaStream_t s = (cudaStream_t)stream;
  if (precision == XCT_DOUBLE)
    normalize_strided<double><<<grid, kThreads, 0, s>>>(d_v, in_f64, n, n_slices, row_stride,
                                                        ffactor, f_dev, d_factors, (double*)d_out);
  else if (precision == XCT_SINGLE)
    normalize_strided<float><<<grid, kThreads, 0, s>>>(d_v, in_f64, n, n_slices, row_stride,
                                                       ffactor, f_dev, d_factors, (float*)d_out);
  else
    normalize_strided<__half><<<grid, kThreads, 0, s>>>(d_v, in_f64, n, n_slices, row_stride,
                                                        ffactor, f_dev, d_factors, (__half*)d_out);
  XCT_CUDA_CHECK_LAUNCH("normalize");
  return XCT_OK;
}

extern "C" int xct_dot(const void* d_a, const void* d_b, int dtype, int64_t n_elem, float fa,
                       float fb, double* d_scratch, double* d_result, void* stream) {
  if (!d_a || !d_b || !d_scratch || !d_result || dtype < 0 || dtype > 2)
    return xct::fail(XCT_EINVAL, "dot: bad argument");
  cudaStream_t s = (cudaStream_t)stream;
  int g = blocks_for(n_elem);
  dot_partial_kernel<<<g, kThreads, 0, s>>>(d_a, d_b, dtype, n_elem, fa, fb, d_scratch);
  final_sum_kernel<<<1, 1024, 0, s>>>(d_scratch, g, d_result);
  XCT_CUDA_CHECK_LAUNCH("dot");
  return XCT_OK;
}

extern "C" int xct_maxabs(const void* d_v, int dtype, int64_t n_elem, float fv,
                            uint64_t* d_maxbits, void* stream) {
  if (!d_v || !d_maxbits) return xct::fail(XCT_EINVAL, "maxabs: bad argument");
  if (n_elem == 0) return XCT_OK;
  maxabs_kernel<<<blocks_for(n_elem), kThreads, 0, (cudaStream_t)stream>>>(
      d_v, dtype, n_elem, fv, (unsigned long long*)d_maxbits);
  XCT_CUDA_CHECK_LAUNCH("maxabs");
  return XCT_OK;
}

extern "C" int xct_axpy(const void* d_a, int a_dtype, float fa, const void* d_b, int b_dtype,
                          float fb, double scale, int64_t n_elem, void* d_out, int out_dtype,
                          float out_factor, uint64_t* d_maxbits, double* d_scratch,
                          double* d_sumsq, void* stream) {
  if (!d_a) return xct::fail(XCT_EINVAL, "axpy: null input");
  if ((a_dtype == 0) != (out_dtype == 0) || (d_b && (b_dtype == 0) != (a_dtype == 0)))
    return xct::fail(XCT_EINVAL, "axpy: f64 operands must be all-f64");
  int mode;
  if (out_dtype != 2) mode = 0;
  else mode = d_out ? 2 : 1;
  if (mode == 0 && !d_out) return xct::fail(XCT_EINVAL, "axpy: null output");
  if (mode == 1 && !d_maxbits) return xct::fail(XCT_EINVAL, "axpy: max pass needs d_maxbits");
  if (n_elem == 0) return XCT_OK;
  cudaStream_t s = (cudaStream_t)stream;
  int g = blocks_for(n_elem);
  double* partials = (mode == 2 && d_sumsq) ? d_scratch : nullptr;
  const bool vec = a_dtype != 0 && n_elem % 4 == 0 && (mode != 0 || out_dtype == 1);
  if (vec) {
    const int gv = blocks_for(n_elem / 4);
    auto* mb = (unsigned long long*)d_maxbits;
    if (mode == 0)
      axpy_vec_kernel<0><<<gv, kThreads, 0, s>>>(d_a, a_dtype, fa, d_b, b_dtype, fb, (float)scale,
                                                 n_elem, d_out, out_factor, mb, partials);
    else if (mode == 1)
      axpy_vec_kernel<1><<<gv, kThreads, 0, s>>>(d_a, a_dtype, fa, d_b, b_dtype, fb, (float)scale,
                                                 n_elem, d_out, out_factor, mb, partials);
    else
      axpy_vec_kernel<2><<<gv, kThreads, 0, s>>>(d_a, a_dtype, fa, d_b, b_dtype, fb, (float)scale,
                                                 n_elem, d_out, out_factor, mb, partials);
    g = gv;
  } else {
    axpy_kernel<<<g, kThreads, 0, s>>>(d_a, a_dtype, fa, d_b, b_dtype, fb, scale, n_elem, d_out,
                                       out_dtype, out_factor, mode,
                                       (unsigned long long*)d_maxbits, partials);
  }
  if (partials) final_sum_kernel<<<1, 1024, 0, s>>>(partials, g, d_sumsq);
  XCT_CUDA_CHECK_LAUNCH("axpy");
  return XCT_OK;
}

extern "C" int xct_chunk_maxabs_chunked(const void* d_v, int dtype, float fv, int64_t n,
                                          int64_t n_chunks, int32_t f_dev, uint64_t* d_maxbits,
                                          void* stream) {
  if (!d_v || !d_maxbits) return xct::fail(XCT_EINVAL, "chunk_maxabs_chunked: bad argument");
  if (n == 0 || n_chunks == 0) return XCT_OK;
  int64_t per = n * f_dev;
  int gx = blocks_for(per);
  if (gx > 512) gx = 512;
  if (dtype != 0 && per % 4 == 0) {
    const int gv = std::max(1, std::min(512, blocks_for(per / 4)));
    chunk_maxabs_chunked_vec_k<<<dim3(gv, (unsigned)n_chunks), kThreads, 0, (cudaStream_t)stream>>>(
        d_v, dtype, fv, per, (unsigned long long*)d_maxbits);
  } else {
    chunk_maxabs_chunked_k<<<dim3(gx, (unsigned)n_chunks), kThreads, 0, (cudaStream_t)stream>>>(
        d_v, dtype, fv, per, (unsigned long long*)d_maxbits);
  }
  XCT_CUDA_CHECK_LAUNCH("chunk_maxabs_chunked");
  return XCT_OK;
}

extern "C" int xct_normalize_chunked(const void* d_v, int dtype, float fv, int64_t n,
                                     int64_t n_chunks, int32_t f_dev, const double* d_factors,
                                     int precision, void* d_out, void* stream) {
  if (!d_v || !d_out || !d_factors) return xct::fail(XCT_EINVAL, "normalize_chunked: bad argument");
  if (n == 0 || n_chunks == 0) return XCT_OK;
  int64_t per = n * f_dev;
  int gx = blocks_for(per);
  if (gx > 512) gx = 512;
  dim3 grid(gx, (unsigned)n_chunks);
  cudaStream_t s = (cudaStream_t)stream;
  if (precision == XCT_DOUBLE)
    normalize_chunked_k<double><<<grid, kThreads, 0, s>>>(d_v, dtype, fv, per, d_factors, (double*)d_out);
  else if (dtype != 0 && per % 4 == 0) {
    dim3 gv(std::max(1, std::min(512, blocks_for(per / 4))), (unsigned)n_chunks);
    if (precision == XCT_SINGLE)
      normalize_chunked_vec_k<float><<<gv, kThreads, 0, s>>>(d_v, dtype, fv, per, d_factors, (float*)d_out);
    else
      normalize_chunked_vec_k<__half><<<gv, kThreads, 0, s>>>(d_v, dtype, fv, per, d_factors, (__half*)d_out);
  } else if (precision == XCT_SINGLE)
    normalize_chunked_k<float><<<grid, kThreads, 0, s>>>(d_v, dtype, fv, per, d_factors, (float*)d_out);
  else
    normalize_chunked_k<__half><<<grid, kThreads, 0, s>>>(d_v, dtype, fv, per, d_factors, (__half*)d_out);
  XCT_CUDA_CHECK_LAUNCH("normalize_chunked");
  return XCT_OK;
}

extern "C" int xct_unchunk_f64(const void* d_in, int in_dtype, float fin, int64_t n,
                               int64_t n_slices, int32_t ffactor, int32_t f_dev, double* d_out,
                               void* stream) {
  if (!d_in || !d_out) return xct::fail(XCT_EINVAL, "unchunk: bad argument");
  if (n * n_slices == 0) return XCT_OK;
  unchunk_f64_k<<<blocks_for(n * n_slices), kThreads, 0, (cudaStream_t)stream>>>(
      d_in, in_dtype, fin, n, n_slices, ffactor, f_dev, d_out);
  XCT_CUDA_CHECK_LAUNCH("unchunk");
  return XCT_OK;
}

extern "C" int xct_chunk_from_f64(const double* d_in, int64_t n, int64_t n_slices,
                                  int32_t ffactor, int32_t f_dev, int out_dtype, void* d_out,
                                  void* stream) {
  if (!d_in || !d_out || (out_dtype != 0 && out_dtype != 1))
    return xct::fail(XCT_EINVAL, "chunk_from_f64: bad argument");
  int64_t n_chunks = (n_slices + ffactor - 1) / ffactor;
  int64_t total = n_chunks * n * f_dev;
  if (total == 0) return XCT_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (out_dtype == 0)
    chunk_from_f64_k<double><<<blocks_for(total), kThreads, 0, s>>>(d_in, n, n_slices, ffactor,
                                                                   f_dev, n_chunks, (double*)d_out);
  else
    chunk_from_f64_k<float><<<blocks_for(total), kThreads, 0, s>>>(d_in, n, n_slices, ffactor,
                                                                  f_dev, n_chunks, (float*)d_out);
  XCT_CUDA_CHECK_LAUNCH("chunk_from_f64");
  return XCT_OK;
}

extern "C" int xct_sum_f64(const double* d_v, int64_t n, double* d_result, void* stream) {
  if (!d_v || !d_result || n < 0 || n > INT32_MAX) return xct::fail(XCT_EINVAL, "sum_f64: bad argument");
  final_sum_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(d_v, (int)n, d_result);
  XCT_CUDA_CHECK_LAUNCH("sum_f64");
  return XCT_OK;
}

// ---------------------------------------------------------------------------
// K10: partial-result exchange helpers for the data-partitioned operator
// (comm.execute_plan / engine.reduce_partials, src/comm.py:420-472,
// src/engine.py:189-221).  Vectors are chunked [n_chunks][n][fd]; element
// rows are moved whole (fd values).  All ops are plain elementwise f32/f64,
// order fixed by the caller (owner first, then senders ascending).
namespace {
template <typename T>
__global__ void gather_rows_k(const T* src, int64_t n_src, const int32_t* idx, int64_t m,
                              int64_t n_chunks, int fd, T* dst) {
  const int64_t total = n_chunks * m * fd;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = t / (m * fd), rem = t % (m * fd);
    const int64_t i = rem / fd, f = rem % fd;
    XCT_CHECK(idx[i] >= 0 && idx[i] < n_src);
    dst[t] = src[(c * n_src + idx[i]) * fd + f];
  }
}
template <typename T>
__global__ void accumulate_rows_k(T* dst, int64_t n_dst, const T* src, const int32_t* pos,
                                  int64_t m, int64_t n_chunks, int fd) {
  const int64_t total = n_chunks * m * fd;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = t / (m * fd), rem = t % (m * fd);
    const int64_t i = rem / fd, f = rem % fd;
    XCT_CHECK(pos[i] >= 0 && pos[i] < n_dst);
    T* d = dst + (c * n_dst + pos[i]) * fd + f;
    *d = *d + src[t];
  }
}
template <typename T>
__global__ void scale_chunks_k(T* v, int64_t per_chunk, int64_t n_chunks, const double* factors,
                               double* partials) {
  double sq = 0.0;
  const int64_t total = n_chunks * per_chunk;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = t / per_chunk;
    T x = v[t] * (T)factors[c];     // denormalize: f32 * f32(factor) / f64 * factor
    v[t] = x;
    sq += (double)x * (double)x;
  }
  if (partials) {
    sq = block_sum(sq);
    if (threadIdx.x == 0) partials[blockIdx.x] = sq;
  }
}
// f32 rows of fd % 4 == 0 floats: one float4 per thread step, chunk =
// blockIdx.y, 32-bit row / piece arithmetic (fd/4 is a power of two)
__global__ void gather_rows_v4(const float4* src, int64_t n_src, const int32_t* idx, int m,
                               int lq, float4* dst) {
  const int c = blockIdx.y;
  const int total = m << lq;
  const float4* s = src + (int64_t)c * n_src * (1 << lq);
  float4* d = dst + (int64_t)c * total;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    const int i = t >> lq, q = t & ((1 << lq) - 1);
    XCT_CHECK(idx[i] >= 0 && idx[i] < n_src);
    d[t] = s[((int64_t)idx[i] << lq) + q];
  }
}

__global__ void accumulate_rows_v4(float4* dst, int64_t n_dst, const float4* src,
                                   const int32_t* pos, int m, int lq) {
  const int c = blockIdx.y;
  const int total = m << lq;
  const float4* s = src + (int64_t)c * total;
  float4* d = dst + (int64_t)c * n_dst * (1 << lq);
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    const int i = t >> lq, q = t & ((1 << lq) - 1);
    XCT_CHECK(pos[i] >= 0 && pos[i] < n_dst);
    float4* o = d + ((int64_t)pos[i] << lq) + q;
    float4 a = *o;
    const float4 b = s[t];
    a.x = a.x + b.x; a.y = a.y + b.y; a.z = a.z + b.z; a.w = a.w + b.w;
    *o = a;
  }
}

__global__ void scale_chunks_v4(float4* v, int64_t per4, const double* factors, double* partials) {
  const int c = blockIdx.y;
  const float f = (float)factors[c];
  float4* p = v + (int64_t)c * per4;
  double sq = 0.0;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < per4;
       t += (int64_t)gridDim.x * blockDim.x) {
    float4 x = p[t];
    x.x = x.x * f; x.y = x.y * f; x.z = x.z * f; x.w = x.w * f;
    p[t] = x;
    sq += (double)x.x * x.x + (double)x.y * x.y + (double)x.z * x.z + (double)x.w * x.w;
  }
  if (partials) {
    sq = block_sum(sq);
    if (threadIdx.x == 0) partials[(int64_t)blockIdx.y * gridDim.x + blockIdx.x] = sq;
  }
}

int log2_exact(int v) {
  int l = 0;
  while ((1 << l) < v) ++l;
  return (1 << l) == v ? l : -1;
}

}  // namespace

extern "C" int xct_gather_rows(const void* d_src, int64_t n_src, const int32_t* d_idx, int64_t m,
                               int64_t n_chunks, int32_t fd, int f64, void* d_dst, void* stream) {
  if (m == 0 || n_chunks == 0 || fd == 0) return XCT_OK;     // empty exchange list
  if (!d_src || !d_dst || !d_idx) return xct::fail(XCT_EINVAL, "gather_rows: bad argument");
  const int64_t total = n_chunks * m * fd;
  if (total == 0) return XCT_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int lq = fd % 4 == 0 ? log2_exact(fd / 4) : -1;
  if (!f64 && lq >= 0 && (m << lq) < (1LL << 31) && n_chunks <= 65535) {
    dim3 g(std::max(1, std::min(512, blocks_for(m << lq))), (unsigned)n_chunks);
    gather_rows_v4<<<g, kThreads, 0, s>>>((const float4*)d_src, n_src, d_idx, (int)m, lq,
                                          (float4*)d_dst);
  } else if (f64) gather_rows_k<double><<<blocks_for(total), kThreads, 0, s>>>((const double*)d_src, n_src, d_idx, m, n_chunks, fd, (double*)d_dst);
  else gather_rows_k<float><<<blocks_for(total), kThreads, 0, s>>>((const float*)d_src, n_src, d_idx, m, n_chunks, fd, (float*)d_dst);
  XCT_CUDA_CHECK_LAUNCH("gather_rows");
  return XCT_OK;
}

extern "C" int xct_accumulate_rows(void* d_dst, int64_t n_dst, const void* d_src,
                                   const int32_t* d_pos, int64_t m, int64_t n_chunks, int32_t fd,
                                   int f64, void* stream) {
  if (m == 0 || n_chunks == 0 || fd == 0) return XCT_OK;     // empty exchange list
  if (!d_src || !d_dst || !d_pos) return xct::fail(XCT_EINVAL, "accumulate_rows: bad argument");
  const int64_t total = n_chunks * m * fd;
  if (total == 0) return XCT_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int lq = fd % 4 == 0 ? log2_exact(fd / 4) : -1;
  if (!f64 && lq >= 0 && (m << lq) < (1LL << 31) && n_chunks <= 65535) {
    dim3 g(std::max(1, std::min(512, blocks_for(m << lq))), (unsigned)n_chunks);
    accumulate_rows_v4<<<g, kThreads, 0, s>>>((float4*)d_dst, n_dst, (const float4*)d_src, d_pos,
                                              (int)m, lq);
  } else if (f64) accumulate_rows_k<double><<<blocks_for(total), kThreads, 0, s>>>((double*)d_dst, n_dst, (const double*)d_src, d_pos, m, n_chunks, fd);
  else accumulate_rows_k<float><<<blocks_for(total), kThreads, 0, s>>>((float*)d_dst, n_dst, (const float*)d_src, d_pos, m, n_chunks, fd);
  XCT_CUDA_CHECK_LAUNCH("accumulate_rows");
  return XCT_OK;
}

extern "C" int xct_scale_chunks(void* d_v, int64_t per_chunk, int64_t n_chunks,
                                const double* d_factors, int f64, double* d_scratch,
                                double* d_sumsq, void* stream) {
  if ((!d_v && n_chunks * per_chunk) || !d_factors)
    return xct::fail(XCT_EINVAL, "scale_chunks: bad argument");
  const int64_t total = n_chunks * per_chunk;
  cudaStream_t s = (cudaStream_t)stream;
  if (total == 0) {
    if (d_sumsq) cudaMemsetAsync(d_sumsq, 0, sizeof(double), s);
    return XCT_OK;
  }
  double* partials = d_sumsq ? d_scratch : nullptr;
  if (!f64 && per_chunk % 4 == 0 && n_chunks <= 65535) {
    // partials: gx per chunk, gx * n_chunks <= kRedBlocks (the scratch size)
    const int gx = std::max(1, std::min(blocks_for(per_chunk / 4), (int)(kRedBlocks / n_chunks)));
    if (gx * n_chunks <= kRedBlocks) {
      scale_chunks_v4<<<dim3(gx, (unsigned)n_chunks), kThreads, 0, s>>>(
          (float4*)d_v, per_chunk / 4, d_factors, partials);
      if (partials) final_sum_kernel<<<1, 1024, 0, s>>>(partials, gx * (int)n_chunks, d_sumsq);
      XCT_CUDA_CHECK_LAUNCH("scale_chunks");
      return XCT_OK;
    }
  }
  const int g = blocks_for(total);
  if (f64) scale_chunks_k<double><<<g, kThreads, 0, s>>>((double*)d_v, per_chunk, n_chunks, d_factors, partials);
  else scale_chunks_k<float><<<g, kThreads, 0, s>>>((float*)d_v, per_chunk, n_chunks, d_factors, partials);
  if (partials) final_sum_kernel<<<1, 1024, 0, s>>>(partials, g, d_sumsq);
  XCT_CUDA_CHECK_LAUNCH("scale_chunks");
  return XCT_OK;
}

extern "C" int xct_rows_to_chunked(const void* d_rows, int in_dtype, int64_t r0, int64_t nr,
                                   int64_t n, int64_t n_slices, int32_t ffactor, int32_t f_dev,
                                   int out_dtype, void* d_out, uint64_t* d_max_in,
                                   uint64_t* d_max_out, double* d_scratch, double* d_sumsq,
                                   void* stream) {
  if (!d_rows || !d_out || (in_dtype != 0 && in_dtype != 1) || (out_dtype != 0 && out_dtype != 1) ||
      ffactor < 1 || f_dev < ffactor || r0 < 0 || nr < 0 || r0 + nr > n)
    return xct::fail(XCT_EINVAL, "rows_to_chunked: bad argument");
  const int64_t total = nr * n_slices;
  if (total == 0) return XCT_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int g = blocks_for(total);
  double* part = d_sumsq ? d_scratch : nullptr;
  if (d_sumsq && !d_scratch) return xct::fail(XCT_EINVAL, "rows_to_chunked: sumsq needs scratch");
  auto* mi = (unsigned long long*)d_max_in;
  auto* mo = (unsigned long long*)d_max_out;
  if (in_dtype == 0 && out_dtype == 0)
    rows_to_chunked_k<double, double><<<g, kThreads, 0, s>>>((const double*)d_rows, r0, nr, n,
        n_slices, ffactor, f_dev, (double*)d_out, mi, mo, part);
  else if (in_dtype == 0)
    rows_to_chunked_k<double, float><<<g, kThreads, 0, s>>>((const double*)d_rows, r0, nr, n,
        n_slices, ffactor, f_dev, (float*)d_out, mi, mo, part);
  else if (out_dtype == 0)
    rows_to_chunked_k<float, double><<<g, kThreads, 0, s>>>((const float*)d_rows, r0, nr, n,
        n_slices, ffactor, f_dev, (double*)d_out, mi, mo, part);
  else
    rows_to_chunked_k<float, float><<<g, kThreads, 0, s>>>((const float*)d_rows, r0, nr, n,
        n_slices, ffactor, f_dev, (float*)d_out, mi, mo, part);
  if (part) final_sum_kernel<<<1, 1024, 0, s>>>(part, g, d_sumsq);
  XCT_CUDA_CHECK_LAUNCH("rows_to_chunked");
  return XCT_OK;
}

extern "C" int xct_unchunk_rows_f64(const void* d_in, int in_dtype, float fin, int64_t n,
                                    int64_t r0, int64_t nr, int64_t n_slices, int32_t ffactor,
                                    int32_t f_dev, double* d_out, void* stream) {
  if (!d_in || !d_out || r0 < 0 || nr < 0 || r0 + nr > n || ffactor < 1)
    return xct::fail(XCT_EINVAL, "unchunk_rows_f64: bad argument");
  if (nr * n_slices == 0) return XCT_OK;
  unchunk_rows_f64_k<<<blocks_for(nr * n_slices), kThreads, 0, (cudaStream_t)stream>>>(
      d_in, in_dtype, fin, n, r0, nr, n_slices, ffactor, f_dev, d_out);
  XCT_CUDA_CHECK_LAUNCH("unchunk_rows_f64");
  return XCT_OK;
}

// ---------------------------------------------------------------------------
// K10 for the native domain partition (parallel.py): element-major exchange
// buffers [m][n_chunks][record], so each peer's rows are ONE contiguous
// NCCL message (footprints are ordered by owner) and no gather pass runs on
// the K6 output side.
namespace {
__global__ void gather_records_k(const uint4* __restrict__ src, int64_t n_src,
                                 const int32_t* __restrict__ idx, int64_t m, int64_t c0,
                                 int64_t nc, int rp, uint4* __restrict__ dst) {
  const int64_t total = m * nc * rp;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = t % rp, rc = t / rp;
    const int64_t c = rc % nc, i = rc / nc;
    XCT_CHECK(idx[i] >= 0 && idx[i] < n_src);
    dst[t] = src[((c0 + c) * n_src + idx[i]) * rp + q];
  }
}
template <typename T>
__global__ void accumulate_records_k(T* dst, int64_t n_dst, int64_t c0, const T* src,
                                     const int32_t* pos, int64_t m, int64_t nc, int fd) {
  const int64_t total = m * nc * fd;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t f = t % fd, rc = t / fd;
    const int64_t c = rc % nc, i = rc / nc;
    XCT_CHECK(pos[i] >= 0 && pos[i] < n_dst);
    T* d = dst + ((c0 + c) * n_dst + pos[i]) * fd + f;
    *d = *d + src[t];
  }
}
}  // namespace

extern "C" int xct_gather_records(const void* d_src, int64_t n_src, const int32_t* d_idx,
                                  int64_t m, int64_t c0, int64_t n_chunks, int32_t rec_bytes,
                                  void* d_dst, void* stream) {
  if ((m && (!d_src || !d_idx || !d_dst)) || rec_bytes < 16 || rec_bytes % 16 || n_chunks < 0)
    return xct::fail(XCT_EINVAL, "gather_records: bad argument");
  const int64_t total = m * n_chunks * (rec_bytes / 16);
  if (total == 0) return XCT_OK;
  gather_records_k<<<blocks_for(total), kThreads, 0, (cudaStream_t)stream>>>(
      (const uint4*)d_src, n_src, d_idx, m, c0, n_chunks, rec_bytes / 16, (uint4*)d_dst);
  XCT_CUDA_CHECK_LAUNCH("gather_records");
  return XCT_OK;
}

extern "C" int xct_accumulate_records(void* d_dst, int64_t n_dst, int64_t c0, const void* d_src,
                                      const int32_t* d_pos, int64_t m, int64_t n_chunks,
                                      int32_t fd, int f64, void* stream) {
  if ((m && (!d_dst || !d_src || !d_pos)) || fd < 1 || n_chunks < 0)
    return xct::fail(XCT_EINVAL, "accumulate_records: bad argument");
  const int64_t total = m * n_chunks * fd;
  if (total == 0) return XCT_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (f64)
    accumulate_records_k<double><<<blocks_for(total), kThreads, 0, s>>>(
        (double*)d_dst, n_dst, c0, (const double*)d_src, d_pos, m, n_chunks, fd);
  else
    accumulate_records_k<float><<<blocks_for(total), kThreads, 0, s>>>(
        (float*)d_dst, n_dst, c0, (const float*)d_src, d_pos, m, n_chunks, fd);
  XCT_CUDA_CHECK_LAUNCH("accumulate_records");
  return XCT_OK;
}

// ---------------------------------------------------------------------------
// CUDA IPC (fused exchange of the native domain partition, domain.py)
extern "C" int xct_ipc_alloc(int64_t bytes, void** d_ptr, void* h_handle) {
  if (!d_ptr || !h_handle || bytes < 1) return xct::fail(XCT_EINVAL, "ipc_alloc: bad argument");
  cudaError_t e = cudaMalloc(d_ptr, (size_t)bytes);
  if (e != cudaSuccess) return xct::fail(XCT_ENOMEM, std::string("ipc_alloc: ") + cudaGetErrorString(e));
  cudaIpcMemHandle_t h;
  e = cudaIpcGetMemHandle(&h, *d_ptr);
  if (e != cudaSuccess) {
    cudaFree(*d_ptr);
    *d_ptr = nullptr;
    return xct::fail(XCT_ECUDA, std::string("ipc_alloc: handle: ") + cudaGetErrorString(e));
  }
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  memcpy(h_handle, &h, sizeof(h));
  return XCT_OK;
}

extern "C" int xct_ipc_open(const void* h_handle, void** d_ptr) {
  if (!d_ptr || !h_handle) return xct::fail(XCT_EINVAL, "ipc_open: bad argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, h_handle, sizeof(h));
  cudaError_t e = cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return xct::fail(XCT_ECUDA, std::string("ipc_open: ") + cudaGetErrorString(e));
  return XCT_OK;
}

extern "C" int xct_ipc_close(void* d_ptr) {
  cudaError_t e = cudaIpcCloseMemHandle(d_ptr);
  if (e != cudaSuccess) return xct::fail(XCT_ECUDA, std::string("ipc_close: ") + cudaGetErrorString(e));
  return XCT_OK;
}

extern "C" int xct_ipc_free(void* d_ptr) {
  cudaError_t e = cudaFree(d_ptr);
  if (e != cudaSuccess) return xct::fail(XCT_ECUDA, std::string("ipc_free: ") + cudaGetErrorString(e));
  return XCT_OK;
}

// ---- binade histogram (matrixstore.half_rescale_exponent, src/matrixstore.py:264-275)
// d_hist[e] += count of positive f64 values with biased exponent e (2048
// bins); the median's binade without sorting 1e10 lengths.  Shared-memory
// bins per CTA, one global atomic per non-empty bin.
namespace {
__global__ void binade_hist_k(const double* __restrict__ v, int64_t n,
                              unsigned long long* __restrict__ hist) {
  __shared__ unsigned int h[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) h[i] = 0u;
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double x = v[i];
    if (x > 0.0) atomicAdd(&h[(unsigned)(__double_as_longlong(x) >> 52) & 2047u], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 2048; i += blockDim.x)
    if (h[i]) atomicAdd(&hist[i], (unsigned long long)h[i]);
}
}  // namespace

extern "C" int xct_binade_hist(const double* d_v, int64_t n, uint64_t* d_hist, void* stream) {
  if (n < 0 || (n > 0 && (!d_v || !d_hist))) return xct::fail(XCT_EINVAL, "binade_hist: bad argument");
  if (n == 0) return XCT_OK;
  // per-CTA counts stay < 2^32: at most 148*8 CTAs, n / CTAs values each
  const int64_t blocks = std::min<int64_t>(148 * 8, (n + 255) / 256);
  binade_hist_k<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
      d_v, n, (unsigned long long*)d_hist);
  XCT_CUDA_CHECK_LAUNCH("binade_hist");
  return XCT_OK;
}
