// K6: staged XCT SpMM for sm_100a -- forward projection (A.X) and back
// projection (A^T.Y) over F fused slices.
//
// Replaces engine.project/backproject/_apply_exec (src/engine.py:119-166)
// and fuses what the reference does after the kernel: output rescale and
// fp16 cast (src/engine.py:137-139), the partial upcast of the exchange
// (src/comm.py:432) and denormalize (src/matrixstore.py:308-316), plus an
// optional f64 sum of squares of the outputs for the CGLS dot products.
//
// Execution model (one CTA = one tile of rows, one F-chunk):
//   for each load group of the tile:
//     stage the group's input records x[elem][0:F] into shared memory with
//       cp.async (16 B per lane, LDGSTS), one record = L 16-byte pieces;
//     every lane of a warp owns 16 B (V slices) of one row's record and
//       walks the (group, warp) slab: 4 entries per 128-bit streaming load,
//       one 128-bit LDS per entry, V multiply-adds into registers;
//   epilogue writes the row's F outputs once.
// Accumulation per row is sequential in stored order, so results are
// deterministic and, with reference-stage keys, bit-identical to the
// reference: single/double multiply then add (two roundings), mixed uses
// FHFMA (fp16 x fp16 product is exact in fp32, one rounding), half uses
// HMUL2 then HADD2.
#include <cuda_fp16.h>

#include "xct_common.h"

namespace {

struct Params {
  const int32_t* cta_rows;
  const int32_t* cta_group_ptr;
  const int64_t* group_map_ptr;
  const int32_t* group_map;
  const int64_t* slab_off;
  const int32_t* slab_width;
  const uint16_t* slots;
  const void* values;
  const uint4* x;
  int64_t n_in;
  int32_t rows_per_cta, warps_per_cta, log2_lanes, n_cta;
  // epilogue
  void* out;
  int64_t row_stride, chunk_stride;
  int32_t valid_cols, ffactor, scale_exp;
  const double* factors;
  double* dot_partials;
};

__device__ __forceinline__ uint2 ld_stream_u2(const void* p) {
  uint2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];"
               : "=r"(v.x), "=r"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ uint4 ld_stream_u4(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

__device__ __forceinline__ float fhfma(unsigned short a, unsigned short b, float c) {
  float d;
  asm("fma.rn.f32.f16 %0, %1, %2, %3;" : "=f"(d) : "h"(a), "h"(b), "f"(c));
  return d;
}

// ---- per-precision arithmetic ---------------------------------------------

template <int PREC> struct Acc;

template <> struct Acc<XCT_MIXED> {          // fp16 storage, fp32 accumulate
  static constexpr int V = 8;                // slices per lane (16 B of halves)
  using Val4 = uint2;                        // 4 fp16 lengths
  float a[8];
  __device__ void zero() { for (int i = 0; i < 8; ++i) a[i] = 0.f; }
  __device__ static Val4 load4(const void* base, int64_t idx) {
    return ld_stream_u2((const uint16_t*)base + idx);
  }
  __device__ static unsigned short pick(const Val4& v, int e) {
    unsigned w = e < 2 ? v.x : v.y;
    return (unsigned short)((e & 1) ? (w >> 16) : (w & 0xffff));
  }
  __device__ void fma(const uint4& r, unsigned short len) {
    const unsigned w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      a[2 * i] = fhfma((unsigned short)(w[i] & 0xffff), len, a[2 * i]);
      a[2 * i + 1] = fhfma((unsigned short)(w[i] >> 16), len, a[2 * i + 1]);
    }
  }
  __device__ void result(float scale, float* out) const {
    for (int i = 0; i < 8; ++i) out[i] = __half2float(__float2half_rn(a[i] * scale));
  }
};

template <> struct Acc<XCT_HALF> {           // fp16 storage and accumulate
  static constexpr int V = 8;
  using Val4 = uint2;
  __half2 a[4];
  __device__ void zero() { for (int i = 0; i < 4; ++i) a[i] = __float2half2_rn(0.f); }
  __device__ static Val4 load4(const void* base, int64_t idx) {
    return ld_stream_u2((const uint16_t*)base + idx);
  }
  __device__ static unsigned short pick(const Val4& v, int e) {
    unsigned w = e < 2 ? v.x : v.y;
    return (unsigned short)((e & 1) ? (w >> 16) : (w & 0xffff));
  }
  __device__ void fma(const uint4& r, unsigned short len) {
    __half h = __ushort_as_half(len);
    __half2 l2 = __halves2half2(h, h);
    const unsigned w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __half2 x = *reinterpret_cast<const __half2*>(&w[i]);
      a[i] = __hadd2_rn(a[i], __hmul2_rn(x, l2));   // two roundings, as numpy f16
    }
  }
  __device__ void result(float scale, float* out) const {
    __half hs = __float2half_rn(scale);
    for (int i = 0; i < 4; ++i) {
      __half2 v = __hmul2_rn(a[i], __halves2half2(hs, hs));
      out[2 * i] = __low2float(v);
      out[2 * i + 1] = __high2float(v);
    }
  }
};

template <> struct Acc<XCT_SINGLE> {         // fp32 storage and accumulate
  static constexpr int V = 4;
  using Val4 = uint4;
  float a[4];
  __device__ void zero() { for (int i = 0; i < 4; ++i) a[i] = 0.f; }
  __device__ static Val4 load4(const void* base, int64_t idx) {
    return ld_stream_u4((const float*)base + idx);
  }
  __device__ static float pick(const Val4& v, int e) {
    unsigned w = e == 0 ? v.x : e == 1 ? v.y : e == 2 ? v.z : v.w;
    return __uint_as_float(w);
  }
  __device__ void fma(const uint4& r, float len) {
    const unsigned w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = __fadd_rn(a[i], __fmul_rn(__uint_as_float(w[i]), len));
  }
  __device__ void result(float scale, float* out) const {
    for (int i = 0; i < 4; ++i) out[i] = a[i] * scale;
  }
};

template <> struct Acc<XCT_DOUBLE> {         // fp64 storage and accumulate
  static constexpr int V = 2;
  struct Val4 { uint4 lo, hi; };
  double a[2];
  __device__ void zero() { a[0] = a[1] = 0.0; }
  __device__ static Val4 load4(const void* base, int64_t idx) {
    const double* p = (const double*)base + idx;
    return {ld_stream_u4(p), ld_stream_u4(p + 2)};
  }
  __device__ static double pick(const Val4& v, int e) {
    const uint4& q = e < 2 ? v.lo : v.hi;
    unsigned long long bits = (e & 1) ? ((unsigned long long)q.w << 32 | q.z)
                                      : ((unsigned long long)q.y << 32 | q.x);
    return __longlong_as_double((long long)bits);
  }
  __device__ void fma(const uint4& r, double len) {
    double x0 = __longlong_as_double((long long)((unsigned long long)r.y << 32 | r.x));
    double x1 = __longlong_as_double((long long)((unsigned long long)r.w << 32 | r.z));
    a[0] = __dadd_rn(a[0], __dmul_rn(x0, len));
    a[1] = __dadd_rn(a[1], __dmul_rn(x1, len));
  }
  __device__ void result(double scale, double* out) const {
    out[0] = a[0] * scale;
    out[1] = a[1] * scale;
  }
};

template <int PREC>
__global__ void __launch_bounds__(1024) spmm_staged_kernel(const Params p) {
  using A = Acc<PREC>;
  constexpr int V = A::V;
  extern __shared__ uint4 stage[];
  const int b = blockIdx.x;
  const int chunk = blockIdx.y;
  const int lg = p.log2_lanes;
  const int L = 1 << lg;
  const int rpw = 32 >> lg;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rin = lane >> lg, sub = lane & (L - 1);
  const int trow = warp * rpw + rin;
  const int row = p.cta_rows[(int64_t)b * p.rows_per_cta + trow];
  const uint4* xb = p.x + (int64_t)chunk * p.n_in * L;

  A acc;
  acc.zero();
  const int g0 = p.cta_group_ptr[b], g1 = p.cta_group_ptr[b + 1];
  for (int g = g0; g < g1; ++g) {
    const int64_t m0 = p.group_map_ptr[g];
    const int ns = (int)(p.group_map_ptr[g + 1] - m0);
    const int pieces = ns << lg;
    for (int i = threadIdx.x; i < pieces; i += blockDim.x) {
      const int32_t e = p.group_map[m0 + (i >> lg)];
      cp_async16(&stage[i], xb + (int64_t)e * L + (i & (L - 1)));
    }
    cp_async_wait_all();
    __syncthreads();

    const int64_t off = p.slab_off[(int64_t)g * p.warps_per_cta + warp];
    const int n4 = p.slab_width[(int64_t)g * p.warps_per_cta + warp] >> 2;
    const uint16_t* sl = p.slots + off;
    if (n4 > 0) {
      int64_t idx = (int64_t)rin * 4;
      uint2 s_next = ld_stream_u2(sl + idx);
      typename A::Val4 v_next = A::load4(p.values, off + idx);
      for (int k = 0; k < n4; ++k) {
        const uint2 s4 = s_next;
        const typename A::Val4 v4 = v_next;
        if (k + 1 < n4) {
          idx += (int64_t)rpw * 4;
          s_next = ld_stream_u2(sl + idx);
          v_next = A::load4(p.values, off + idx);
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const unsigned w = e < 2 ? s4.x : s4.y;
          const unsigned slot = (e & 1) ? (w >> 16) : (w & 0xffffu);
          const uint4 r = stage[(slot << lg) + sub];
          acc.fma(r, A::pick(v4, e));
        }
      }
    }
    __syncthreads();
  }

  // ---- epilogue -----------------------------------------------------------
  double sq = 0.0;
  if (row >= 0) {
    const int j0 = sub * V;
    if constexpr (PREC == XCT_DOUBLE) {
      double o[V];
      acc.result(ldexp(1.0, -p.scale_exp), o);
      const double f = p.factors ? p.factors[chunk] : 1.0;
      double* out = (double*)p.out + (int64_t)row * p.row_stride + (int64_t)chunk * p.chunk_stride;
      for (int i = 0; i < V; ++i) {
        int j = j0 + i;
        if (j < p.ffactor && chunk * p.ffactor + j < p.valid_cols) {
          double v = o[i] * f;
          out[j] = v;
          sq += v * v;
        }
      }
    } else {
      float o[V];
      acc.result(ldexpf(1.0f, -p.scale_exp), o);
      const float f = p.factors ? (float)p.factors[chunk] : 1.0f;
      float* out = (float*)p.out + (int64_t)row * p.row_stride + (int64_t)chunk * p.chunk_stride;
      for (int i = 0; i < V; ++i) {
        int j = j0 + i;
        if (j < p.ffactor && chunk * p.ffactor + j < p.valid_cols) {
          float v = o[i] * f;
          out[j] = v;
          sq += (double)v * (double)v;
        }
      }
    }
  }
  if (p.dot_partials) {
    for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
    __shared__ double red[32];
    if (lane == 0) red[warp] = sq;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
      p.dot_partials[(int64_t)chunk * p.n_cta + b] = t;
    }
  }
}

template <int PREC>
int launch(const Params& p, int64_t n_chunks, int threads, int64_t smem, cudaStream_t s) {
  static int configured = -1;
  if (configured != (int)smem) {
    cudaError_t e = cudaFuncSetAttribute(spmm_staged_kernel<PREC>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return xct::fail(XCT_ECUDA, std::string("spmm smem attribute: ") + cudaGetErrorString(e));
    configured = (int)smem;
  }
  dim3 grid((unsigned)p.n_cta, (unsigned)n_chunks);
  spmm_staged_kernel<PREC><<<grid, threads, smem, s>>>(p);
  XCT_CUDA_CHECK_LAUNCH("spmm_staged");
  return XCT_OK;
}

}  // namespace

extern "C" int xct_spmm(const xct_staged* a, int precision, const void* d_x, int64_t n_in,
                        int64_t n_chunks, int32_t f_dev, const xct_epilogue* ep,
                        int64_t smem_bytes, void* stream) {
  if (!a || !ep || !d_x || !ep->d_out) return xct::fail(XCT_EINVAL, "spmm: null argument");
  if (precision < 0 || precision > 3) return xct::fail(XCT_EINVAL, "spmm: bad precision");
  if (ep->accumulate) return xct::fail(XCT_EINVAL, "spmm: accumulate mode is reserved");
  const int vbytes = precision == XCT_DOUBLE ? 8 : precision == XCT_SINGLE ? 4 : 2;
  const int64_t rec = (int64_t)f_dev * vbytes;
  if (rec < 16 || rec > 512 || (rec & (rec - 1)))
    return xct::fail(XCT_EINVAL, "spmm: f_dev*elem_bytes must be a power of two in [16, 512]");
  int lg = 0;
  while ((16 << lg) < rec) ++lg;
  if (a->rows_per_warp != (32 >> lg))
    return xct::fail(XCT_EINVAL, "spmm: format rows_per_warp does not match f_dev/precision");
  if (a->n_cta == 0 || n_chunks == 0) return XCT_OK;
  if (n_chunks > 65535) return xct::fail(XCT_EINVAL, "spmm: too many chunks for one launch");
  const int threads = (int)(a->warps_per_cta * 32);
  if (threads < 32 || threads > 1024) return xct::fail(XCT_EINVAL, "spmm: CTA must have 1..32 warps");
  int64_t need = a->max_group_slots * rec;
  if (smem_bytes < need) smem_bytes = need;
  if (smem_bytes < 16) smem_bytes = 16;
  if (smem_bytes > 227 * 1024) return xct::fail(XCT_ESTAGE, "spmm: load group exceeds shared memory");

  Params p;
  p.cta_rows = a->d_cta_rows;
  p.cta_group_ptr = a->d_cta_group_ptr;
  p.group_map_ptr = a->d_group_map_ptr;
  p.group_map = a->d_group_map;
  p.slab_off = a->d_slab_off;
  p.slab_width = a->d_slab_width;
  p.slots = a->d_slots;
  p.values = a->d_values;
  p.x = (const uint4*)d_x;
  p.n_in = n_in;
  p.rows_per_cta = (int32_t)a->rows_per_cta;
  p.warps_per_cta = (int32_t)a->warps_per_cta;
  p.log2_lanes = lg;
  p.n_cta = (int32_t)a->n_cta;
  p.out = ep->d_out;
  p.row_stride = ep->row_stride;
  p.chunk_stride = ep->chunk_stride;
  p.valid_cols = ep->valid_cols;
  p.ffactor = ep->ffactor;
  p.scale_exp = ep->value_scale_exp;
  p.factors = ep->d_factors;
  p.dot_partials = ep->d_dot_partials;
  cudaStream_t s = (cudaStream_t)stream;
  switch (precision) {
    case XCT_DOUBLE: return launch<XCT_DOUBLE>(p, n_chunks, threads, smem_bytes, s);
    case XCT_SINGLE: return launch<XCT_SINGLE>(p, n_chunks, threads, smem_bytes, s);
    case XCT_HALF: return launch<XCT_HALF>(p, n_chunks, threads, smem_bytes, s);
    default: return launch<XCT_MIXED>(p, n_chunks, threads, smem_bytes, s);
  }
}

// ---------------------------------------------------------------------------
// Plain CSR float64 product for measurement synthesis
// (geometry.simulate_measurements, src/geometry.py:357-361): y[r, f] =
// sum_j v_j * x[idx_j, f], sequential per row in CSR order.
namespace {
__global__ void csr_spmm_f64_kernel(const int64_t* __restrict__ indptr,
                                    const int32_t* __restrict__ indices,
                                    const double* __restrict__ values, int64_t n_rows,
                                    const double* __restrict__ x, int64_t S,
                                    double* __restrict__ y) {
  const int64_t total = n_rows * S;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / S, f = t % S;
    double acc = 0.0;
    for (int64_t j = indptr[r]; j < indptr[r + 1]; ++j)
      acc = __dadd_rn(acc, __dmul_rn(values[j], x[(int64_t)indices[j] * S + f]));
    y[t] = acc;
  }
}
}  // namespace

extern "C" int xct_csr_spmm_f64(const int64_t* d_indptr, const int32_t* d_indices,
                                const double* d_values, int64_t n_rows, const double* d_x,
                                int64_t n_slices, double* d_y, void* stream) {
  if (!d_indptr || !d_x || !d_y || n_slices < 1) return xct::fail(XCT_EINVAL, "csr_spmm_f64: bad argument");
  int64_t total = n_rows * n_slices;
  if (total == 0) return XCT_OK;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  csr_spmm_f64_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
      d_indptr, d_indices, d_values, n_rows, d_x, n_slices, d_y);
  XCT_CUDA_CHECK_LAUNCH("csr_spmm_f64");
  return XCT_OK;
}
