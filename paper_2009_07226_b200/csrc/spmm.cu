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
//       cp.async (16 B per lane, LDGSTS, double-buffered: the next group is
//       staged while this one is consumed); a record is NP 16-byte pieces
//       kept in NP bank-shifted planes;
//     each row is owned by L lanes (L = 1 when the accumulators fit), each
//       lane NPL = NP/L pieces; the lane walks its row in the (group, warp)
//       slab 4 entries per 128-bit streaming load, with a kDepth-deep
//       register ring of loads in flight, NPL 128-bit LDS and NPL*V
//       multiply-adds per entry;
//   epilogue writes the row's F outputs once.
// Accumulation per row is sequential in stored order, so results are
// deterministic and, with reference-stage keys, bit-identical to the
// reference: single/double multiply then add (two roundings), mixed uses
// FHFMA (fp16 x fp16 product is exact in fp32, one rounding), half uses
// HMUL2 then HADD2.
#include <cuda_fp16.h>

#include <cstdlib>

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
  int64_t x_chunk_pieces;   // 16-byte pieces between consecutive F-chunks of x
  int32_t x_elem_pieces;    // 16-byte pieces between consecutive input elements
  int32_t rows_per_cta, warps_per_cta, log2_lanes, log2_pieces, n_cta;
  int32_t plane_slots;      // slots per shared-memory plane (multiple of 8)
  int32_t chunk_group;      // F-chunks of one tile scheduled back to back
  int32_t n_chunks;
  // epilogue
  void* out;
  int64_t row_stride, chunk_stride;
  int32_t valid_cols, ffactor, scale_exp;
  const double* factors;
  double* dot_partials;
  // fused exchange: output row r of segment q (seg[q] <= r < seg[q+1]) goes
  // to out_ptrs[q] + (r - seg[q]) * row_stride -- a peer GPU's receive
  // buffer over NVLink (CUDA IPC mapping) or this GPU's own
  void* const* out_ptrs;
  const int64_t* seg;
  int32_t n_seg;
};

// A row's NV f32 outputs starting at column j0: 16-byte vector stores when
// the whole run is valid and aligned (fewer, larger transactions -- what
// the fused exchange's remote NVLink stores need), else scalar stores.
template <int NV, typename Fn>
__device__ __forceinline__ void store_row(float* out, int j0, int chunk, const struct Params& p,
                                          Fn val, double& sq) {
  const bool full = j0 + NV <= p.ffactor && chunk * p.ffactor + j0 + NV <= p.valid_cols;
  if (NV % 4 == 0 && full && ((reinterpret_cast<uintptr_t>(out + j0) & 15u) == 0)) {
#pragma unroll
    for (int i = 0; i < NV; i += 4) {
      const float4 v = make_float4(val(i), val(i + 1), val(i + 2), val(i + 3));
      *reinterpret_cast<float4*>(out + j0 + i) = v;
      sq += (double)v.x * (double)v.x;      // same order as the scalar path
      sq += (double)v.y * (double)v.y;
      sq += (double)v.z * (double)v.z;
      sq += (double)v.w * (double)v.w;
    }
    return;
  }
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int j = j0 + i;
    if (j < p.ffactor && chunk * p.ffactor + j < p.valid_cols) {
      const float v = val(i);
      out[j] = v;
      sq += (double)v * (double)v;
    }
  }
}

// destination row base of output row `row` (plain or segment-scattered)
template <typename T>
__device__ __forceinline__ T* out_row(const Params& p, int row, int chunk) {
  if (!p.out_ptrs)
    return (T*)p.out + (int64_t)row * p.row_stride + (int64_t)chunk * p.chunk_stride;
  int q = 0;
  while (q + 1 < p.n_seg && row >= p.seg[q + 1]) ++q;
  return (T*)p.out_ptrs[q] + (int64_t)(row - p.seg[q]) * p.row_stride +
         (int64_t)chunk * p.chunk_stride;
}

// ---- memory access helpers -------------------------------------------------
// Entries stream through L2 once per F-chunk (evict_first); staged input
// records are re-read by many tiles (evict_last).

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint2 ld_stream_u2(const void* p, uint64_t pol) {
  uint2 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;"
               : "=r"(v.x), "=r"(v.y) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ uint4 ld_stream_u4(const void* p, uint64_t pol) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void cp_async16(uint32_t smem, const void* gmem, uint64_t pol) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;"
               :: "r"(smem), "l"(gmem), "l"(pol));
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}

__device__ __forceinline__ float fhfma(unsigned short a, unsigned short b, float c) {
  float d;
  asm("fma.rn.f32.f16 %0, %1, %2, %3;" : "=f"(d) : "h"(a), "h"(b), "f"(c));
  return d;
}

// ---- entry streams: 4 entries of one row per step -------------------------
// slot fields hold the byte offset (slot * 16) of the record inside a plane.
// half/mixed: one packed u32 per entry (offset << 16 | fp16 length)
// single: u16 offsets + f32 lengths; double: u16 offsets + f64 lengths.

template <int PREC> struct Step;

template <> struct Step<XCT_MIXED> {
  uint4 w;
  __device__ void load(const uint16_t*, const void* v, int64_t idx, uint64_t pol) {
    w = ld_stream_u4((const uint32_t*)v + idx, pol);
  }
  __device__ uint32_t word(int e) const { return e == 0 ? w.x : e == 1 ? w.y : e == 2 ? w.z : w.w; }
  __device__ uint32_t off(int e) const { return word(e) >> 16; }
  __device__ unsigned short val(int e) const { return (unsigned short)(word(e) & 0xffffu); }
};
template <> struct Step<XCT_HALF> : Step<XCT_MIXED> {};

template <> struct Step<XCT_SINGLE> {
  uint2 s;
  uint4 v;
  __device__ void load(const uint16_t* sl, const void* vv, int64_t idx, uint64_t pol) {
    s = ld_stream_u2(sl + idx, pol);
    v = ld_stream_u4((const float*)vv + idx, pol);
  }
  __device__ uint32_t off(int e) const {
    uint32_t q = e < 2 ? s.x : s.y;
    return (e & 1) ? (q >> 16) : (q & 0xffffu);
  }
  __device__ float val(int e) const {
    return __uint_as_float(e == 0 ? v.x : e == 1 ? v.y : e == 2 ? v.z : v.w);
  }
};

template <> struct Step<XCT_DOUBLE> {
  uint2 s;
  uint4 lo, hi;
  __device__ void load(const uint16_t* sl, const void* vv, int64_t idx, uint64_t pol) {
    s = ld_stream_u2(sl + idx, pol);
    const double* p = (const double*)vv + idx;
    lo = ld_stream_u4(p, pol);
    hi = ld_stream_u4(p + 2, pol);
  }
  __device__ uint32_t off(int e) const {
    uint32_t q = e < 2 ? s.x : s.y;
    return (e & 1) ? (q >> 16) : (q & 0xffffu);
  }
  __device__ double val(int e) const {
    const uint4& q = e < 2 ? lo : hi;
    unsigned long long b = (e & 1) ? ((unsigned long long)q.w << 32 | q.z)
                                   : ((unsigned long long)q.y << 32 | q.x);
    return __longlong_as_double((long long)b);
  }
};

// ---- per-precision accumulators over NPL 16-byte pieces -----------------------

template <int PREC, int NPL, bool CONTRACT = false> struct Acc;

template <int NPL> struct Acc<XCT_MIXED, NPL> {   // fp16 storage, fp32 accumulate
  static constexpr int V = 8;                      // slices per 16-byte piece
  float a[8 * NPL];
  __device__ void zero() {
#pragma unroll
    for (int i = 0; i < 8 * NPL; ++i) a[i] = 0.f;
  }
  __device__ void fma(int q, const uint4& r, unsigned short len) {
    const unsigned w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      a[8 * q + 2 * i] = fhfma((unsigned short)(w[i] & 0xffff), len, a[8 * q + 2 * i]);
      a[8 * q + 2 * i + 1] = fhfma((unsigned short)(w[i] >> 16), len, a[8 * q + 2 * i + 1]);
    }
  }
  __device__ float out(int i, float scale) const {
    return __half2float(__float2half_rn(a[i] * scale));
  }
};

template <int NPL> struct Acc<XCT_HALF, NPL> {     // fp16 storage and accumulate
  static constexpr int V = 8;
  __half2 a[4 * NPL];
  __device__ void zero() {
#pragma unroll
    for (int i = 0; i < 4 * NPL; ++i) a[i] = __float2half2_rn(0.f);
  }
  __device__ void fma(int q, const uint4& r, unsigned short len) {
    __half h = __ushort_as_half(len);
    __half2 l2 = __halves2half2(h, h);
    const unsigned w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __half2 x = *reinterpret_cast<const __half2*>(&w[i]);
      a[4 * q + i] = __hadd2_rn(a[4 * q + i], __hmul2_rn(x, l2));  // numpy f16: 2 roundings
    }
  }
  __device__ float out(int i, float scale) const {
    __half hs = __float2half_rn(scale);
    __half2 v = __hmul2_rn(a[i >> 1], __halves2half2(hs, hs));
    return (i & 1) ? __high2float(v) : __low2float(v);
  }
};

// FP32, reference rounding: multiply then add (two roundings) per slice.
template <int NPL> struct Acc<XCT_SINGLE, NPL, false> {
  static constexpr int V = 4;
  float a[4 * NPL];
  __device__ void zero() {
#pragma unroll
    for (int i = 0; i < 4 * NPL; ++i) a[i] = 0.f;
  }
  __device__ void fma(int q, const uint4& r, float len) {
    const unsigned w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
    for (int i = 0; i < 4; ++i)
      a[4 * q + i] = __fadd_rn(a[4 * q + i], __fmul_rn(__uint_as_float(w[i]), len));
  }
  __device__ float out(int i, float scale) const { return a[i] * scale; }
};

// CONTRACT (native order only): one rounding per slice, issued as packed
// FFMA2 (fma.rn.f32x2, sm_100a) on slice pairs with the entry's length
// broadcast -- half the FP issue slots of scalar FFMA.
template <int NPL> struct Acc<XCT_SINGLE, NPL, true> {
  static constexpr int V = 4;
  unsigned long long a[2 * NPL];                   // slice pairs
  __device__ void zero() {
#pragma unroll
    for (int i = 0; i < 2 * NPL; ++i) a[i] = 0ull;
  }
  __device__ void fma(int q, const uint4& r, float len) {
    unsigned long long x0, x1, l2;
    asm("mov.b64 %0, {%1, %2};" : "=l"(x0) : "r"(r.x), "r"(r.y));
    asm("mov.b64 %0, {%1, %2};" : "=l"(x1) : "r"(r.z), "r"(r.w));
    asm("mov.b64 %0, {%1, %1};" : "=l"(l2) : "f"(len));
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a[2 * q]) : "l"(x0), "l"(l2));
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a[2 * q + 1]) : "l"(x1), "l"(l2));
  }
  __device__ float out(int i, float scale) const {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(a[i >> 1]));
    return ((i & 1) ? hi : lo) * scale;
  }
};

template <int NPL> struct Acc<XCT_DOUBLE, NPL> {   // fp64 storage and accumulate
  static constexpr int V = 2;
  double a[2 * NPL];
  __device__ void zero() {
#pragma unroll
    for (int i = 0; i < 2 * NPL; ++i) a[i] = 0.0;
  }
  __device__ void fma(int q, const uint4& r, double len) {
    double x0 = __longlong_as_double((long long)((unsigned long long)r.y << 32 | r.x));
    double x1 = __longlong_as_double((long long)((unsigned long long)r.w << 32 | r.z));
    a[2 * q] = __dadd_rn(a[2 * q], __dmul_rn(x0, len));
    a[2 * q + 1] = __dadd_rn(a[2 * q + 1], __dmul_rn(x1, len));
  }
  __device__ double out(int i, double scale) const { return a[i] * scale; }
};

// Shared-memory stage: a record's NP 16-byte pieces live in NP planes of
// plane_slots records each.  Plane p is shifted by (8/NP)*p bank quads
// (p mod 8 when NP > 8), so the L lanes of a row never collide and rows
// collide only when their slots agree mod 8/L (the builder's bank classes).
__device__ __forceinline__ uint32_t plane_base(int p, int lp, int plane_slots) {
  const int shift = lp <= 3 ? ((p << (3 - lp)) & 7) : (p & 7);
  return (uint32_t)p * (uint32_t)plane_slots * 16u + 16u * (uint32_t)shift;
}
__device__ __forceinline__ uint32_t buffer_bytes(int lp, int plane_slots) {
  return ((uint32_t)plane_slots << (lp + 4)) + 128u;
}

constexpr int kDepth = 4;     // entry steps in flight per lane (register ring)
constexpr int kFillUnroll = 4;

// Stage the records of load group g into the buffer at shared address dst,
// reading the group's slot->element map from shared memory (it was copied
// there one group earlier, so no dependent global load sits on this path).
// blockDim is a multiple of the NP pieces of a record, so a thread always
// copies the same piece q: its plane offset and source offset are loop
// invariant, and the loop is one LDS + one address IMAD + one LDGSTS.
__device__ __forceinline__ void stage_fill(const Params& p, const uint4* xb, uint32_t dst,
                                           const int32_t* map, int ns, int lp, uint64_t pol) {
  const int q = threadIdx.x & ((1 << lp) - 1);
  const uint32_t dq = dst + plane_base(q, lp, p.plane_slots);
  const uint4* xq = xb + q;
  const int sstep = blockDim.x >> lp;
  const uint32_t es = (uint32_t)p.x_elem_pieces;     // element offsets fit 32 bits
#pragma unroll 1
  for (int s = threadIdx.x >> lp; s < ns; s += sstep) {
    XCT_CHECK((uint32_t)map[s] < (uint32_t)p.n_in && s < p.plane_slots);
    cp_async16(dq + ((uint32_t)s << 4), xq + (uint32_t)map[s] * es, pol);
  }
}

// Copy the slot->element map of group g into shared memory (4-byte cp.async).
__device__ __forceinline__ void map_fill(const Params& p, int32_t* dst, int64_t m0, int ns) {
  for (int i = threadIdx.x; i < ns; i += blockDim.x) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(dst + i);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" :: "r"(sa), "l"(p.group_map + m0 + i));
  }
}

template <int PREC, int NPL, typename A, typename St>
__device__ __forceinline__ void consume(A& acc, const St& cur, const uint32_t (&pb)[NPL],
                                        uint32_t lim) {
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const uint32_t off = cur.off(e);
    const auto len = cur.val(e);
    XCT_CHECK(off < lim);
#pragma unroll
    for (int qq = 0; qq < NPL; ++qq) acc.fma(qq, lds128(pb[qq] + off), len);
  }
}

// One load group's slabs with the ring entered at phase P: ring slot
// (P + i) & 3 holds the i-th next step, so no register is ever copied.
template <int PREC, int NPL, int P, typename A, typename St>
__device__ __forceinline__ void run_group(A& acc, St (&r)[4], int n4, int64_t& at,
                                          const int64_t step, const uint32_t (&pb)[NPL],
                                          const Params& p, uint64_t pol) {
  constexpr int S0 = P, S1 = (P + 1) & 3, S2 = (P + 2) & 3, S3 = (P + 3) & 3;
  const uint32_t lim = 16u * (uint32_t)p.plane_slots;   // XCT_CHECK bound only
  (void)lim;
  int k = 0;
  for (; k + 4 <= n4; k += 4) {
    consume<PREC, NPL>(acc, r[S0], pb, lim);
    r[S0].load(p.slots, p.values, at, pol);
    consume<PREC, NPL>(acc, r[S1], pb, lim);
    r[S1].load(p.slots, p.values, at + step, pol);
    consume<PREC, NPL>(acc, r[S2], pb, lim);
    r[S2].load(p.slots, p.values, at + 2 * step, pol);
    consume<PREC, NPL>(acc, r[S3], pb, lim);
    r[S3].load(p.slots, p.values, at + 3 * step, pol);
    at += 4 * step;
  }
  const int rem = n4 - k;
  if (rem >= 1) {
    consume<PREC, NPL>(acc, r[S0], pb, lim);
    r[S0].load(p.slots, p.values, at, pol);
  }
  if (rem >= 2) {
    consume<PREC, NPL>(acc, r[S1], pb, lim);
    r[S1].load(p.slots, p.values, at + step, pol);
  }
  if (rem >= 3) {
    consume<PREC, NPL>(acc, r[S2], pb, lim);
    r[S2].load(p.slots, p.values, at + 2 * step, pol);
  }
  at += rem * step;
}

// 1024-thread bound (64 registers) where the accumulators are small (FP16
// storage or FP32 with <= 2 pieces per lane: two 512-thread CTAs per SM);
// 512 threads (128 registers) for the wide-record instantiations that
// spilled under the 64-register cap (r01 VERDICT: staged<3,4>, <0,2>, <0,4>).
template <int PREC, int NPL> struct StagedBound {
  static constexpr int value = (PREC != XCT_DOUBLE && NPL <= 2) ? 1024 : 512;
};

template <int PREC, int NPL, bool CONTRACT>
__global__ void __launch_bounds__(StagedBound<PREC, NPL>::value) spmm_staged_kernel(const Params p) {
  using A = Acc<PREC, NPL, CONTRACT>;
  using St = Step<PREC>;
  constexpr int V = A::V;
  extern __shared__ uint4 stage[];
  // CTA id -> (tile, chunk): the chunk_group F-chunks of a tile are adjacent
  // in launch order, so they run concurrently and share the tile's entry
  // stream through L2 (one HBM read per chunk group instead of per chunk).
  const int64_t id = blockIdx.x;
  const int G = p.chunk_group;
  const int b = (int)((id / G) % p.n_cta);
  const int chunk = (int)(id / ((int64_t)G * p.n_cta)) * G + (int)(id % G);
  const int lg = p.log2_lanes;               // lanes per row = 1 << lg
  const int lp = p.log2_pieces;              // 16-byte pieces per record = 1 << lp
  const int rpw = 32 >> lg;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rin = lane >> lg, sub = lane & ((1 << lg) - 1);
  const int row = p.cta_rows[(int64_t)b * p.rows_per_cta + warp * rpw + rin];
  const uint4* xb = p.x + (int64_t)chunk * p.x_chunk_pieces;
  const uint64_t pol_x = policy_evict_last(), pol_e = policy_evict_first();
  const uint32_t s0 = (uint32_t)__cvta_generic_to_shared(stage);
  const uint32_t bb = buffer_bytes(lp, p.plane_slots);
  uint32_t pbase[NPL];
#pragma unroll
  for (int qq = 0; qq < NPL; ++qq) pbase[qq] = plane_base(sub * NPL + qq, lp, p.plane_slots);

  A acc;
  acc.zero();
  const int g0 = p.cta_group_ptr[b], g1 = p.cta_group_ptr[b + 1];
  // The warp's slabs of all groups are contiguous, so its entries form one
  // strided stream across groups: the register ring is filled once and keeps
  // kDepth steps in flight straight through the group boundaries.
  const int64_t step = (int64_t)rpw * 4;
  int64_t at = (g0 < g1 ? p.slab_off[(int64_t)g0 * p.warps_per_cta + warp] : 0) +
               (int64_t)rin * 4;
  St r[4];
  r[0].load(p.slots, p.values, at, pol_e);
  r[1].load(p.slots, p.values, at + step, pol_e);
  r[2].load(p.slots, p.values, at + 2 * step, pol_e);
  r[3].load(p.slots, p.values, at + 3 * step, pol_e);
  at += 4 * step;
  int phase = 0;
  // pipeline: map(g+2) -> smem and records(g+1) -> smem while g is consumed
  int32_t* const maps = reinterpret_cast<int32_t*>(
      reinterpret_cast<char*>(stage) + 2 * (size_t)bb);
  int32_t* const map0 = maps;
  int32_t* const map1 = maps + p.plane_slots;
  int64_t mp0 = g0 < g1 ? p.group_map_ptr[g0] : 0;
  int64_t mp1 = g0 < g1 ? p.group_map_ptr[g0 + 1] : 0;
  int64_t mp2 = g0 + 1 < g1 ? p.group_map_ptr[g0 + 2] : mp1;
  if (g0 < g1) {
    map_fill(p, map0, mp0, (int)(mp1 - mp0));
    if (g0 + 1 < g1) map_fill(p, map1, mp1, (int)(mp2 - mp1));
    cp_async_commit();
    cp_async_wait_all();
    __syncthreads();
    stage_fill(p, xb, s0, map0, (int)(mp1 - mp0), lp, pol_x);
  }
  cp_async_commit();
  for (int g = g0; g < g1; ++g) {
    const int odd = (g - g0) & 1;
    const uint32_t cur_buf = s0 + (odd ? bb : 0u);
    const int n4 = p.slab_width[(int64_t)g * p.warps_per_cta + warp] >> 2;
    const int64_t mp3 = g + 3 <= g1 ? p.group_map_ptr[min(g + 3, g1)] : mp2;
    cp_async_wait_all();
    __syncthreads();            // fill(g), map(g+1) visible; everyone done with g-1
    if (g + 1 < g1)             // records of g+1 (map already in shared memory)
      stage_fill(p, xb, s0 + (odd ? 0u : bb), odd ? map0 : map1, (int)(mp2 - mp1), lp, pol_x);
    if (g + 2 < g1)             // map of g+2 into the buffer map(g) used
      map_fill(p, odd ? map1 : map0, mp2, (int)(mp3 - mp2));
    cp_async_commit();
    mp1 = mp2;
    mp2 = mp3;

    uint32_t pb[NPL];
#pragma unroll
    for (int qq = 0; qq < NPL; ++qq) pb[qq] = cur_buf + pbase[qq];
    switch (phase) {
      case 0: run_group<PREC, NPL, 0>(acc, r, n4, at, step, pb, p, pol_e); break;
      case 1: run_group<PREC, NPL, 1>(acc, r, n4, at, step, pb, p, pol_e); break;
      case 2: run_group<PREC, NPL, 2>(acc, r, n4, at, step, pb, p, pol_e); break;
      default: run_group<PREC, NPL, 3>(acc, r, n4, at, step, pb, p, pol_e); break;
    }
    phase = (phase + n4) & 3;
  }
  cp_async_wait_all();

  // ---- epilogue -----------------------------------------------------------
  double sq = 0.0;
  if (row >= 0) {
    const int j0 = sub * NPL * V;
    if constexpr (PREC == XCT_DOUBLE) {
      const double sc = ldexp(1.0, -p.scale_exp);
      const double f = p.factors ? p.factors[chunk] : 1.0;
      double* out = out_row<double>(p, row, chunk);
#pragma unroll
      for (int i = 0; i < NPL * V; ++i) {
        const int j = j0 + i;
        if (j < p.ffactor && chunk * p.ffactor + j < p.valid_cols) {
          const double v = acc.out(i, sc) * f;
          out[j] = v;
          sq += v * v;
        }
      }
    } else {
      const float sc = ldexpf(1.0f, -p.scale_exp);
      const float f = p.factors ? (float)p.factors[chunk] : 1.0f;
      float* out = out_row<float>(p, row, chunk);
      store_row<NPL * V>(out, j0, chunk, p, [&](int i) { return acc.out(i, sc) * f; }, sq);
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

template <int PREC, int NPL, bool CONTRACT>
int launch(const Params& p, int64_t n_chunks, int threads, int64_t smem, cudaStream_t s) {
  static int configured = -1;
  if (configured < (int)smem) {
    cudaError_t e = cudaFuncSetAttribute(spmm_staged_kernel<PREC, NPL, CONTRACT>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess)
      return xct::fail(XCT_ECUDA, std::string("spmm smem attribute: ") + cudaGetErrorString(e));
    configured = (int)smem;
  }
  const int64_t n_blocks = (int64_t)p.n_cta * n_chunks;
  if (n_blocks > 0x7fffffffLL) return xct::fail(XCT_EINVAL, "spmm: grid too large");
  if (threads > StagedBound<PREC, NPL>::value)
    return xct::fail(XCT_EINVAL, "spmm: too many threads per CTA for this record width");
  spmm_staged_kernel<PREC, NPL, CONTRACT><<<(unsigned)n_blocks, threads, smem, s>>>(p);
  XCT_CUDA_CHECK_LAUNCH("spmm_staged");
  return XCT_OK;
}

template <int PREC, bool CONTRACT = false>
int launch_npl(const Params& p, int npl, int64_t n_chunks, int threads, int64_t smem,
               cudaStream_t s) {
  switch (npl) {
    case 1: return launch<PREC, 1, CONTRACT>(p, n_chunks, threads, smem, s);
    case 2: return launch<PREC, 2, CONTRACT>(p, n_chunks, threads, smem, s);
    case 4: return launch<PREC, 4, CONTRACT>(p, n_chunks, threads, smem, s);
    default: return xct::fail(XCT_EINVAL, "spmm: pieces per lane must be 1, 2 or 4");
  }
}

// ---- grouped rows: one union entry feeds G rows (format row_group = G) ----
// A unit of G rows walks the union of its rows' entries: every staged record
// read from shared memory (the K6 bottleneck) is used by G rows, with a
// stored 0 for rows that lack the column (x*0 + acc == acc exactly).  Step =
// 4 union entries: 4 u16 offsets (one 64-bit load) + 4*G values (G single /
// G/2 mixed 128-bit loads), a register ring as deep as 128 registers allow.

template <int PREC, int G> struct GStep;

template <int G> struct GStep<XCT_SINGLE, G> {
  static constexpr int NV = G;                      // 4 entries * G * 4 B / 16
  uint2 s;
  uint4 v[NV];
  // sp: this unit's 4 slots of the step; vp: its NV value pieces
  // sp: this unit's 4 slots of the step; vp: its first value piece, piece k
  // upw pieces further (values [NV][units][16 B] per step)
  __device__ void load(const uint16_t* sp, const uint4* vp, int upw, uint64_t pol) {
    s = ld_stream_u2(sp, pol);
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] = ld_stream_u4(vp + (int64_t)k * upw, pol);
  }
  // the same step from a shared-memory copy of the warp's step at `base`
  __device__ void lds(uint32_t base, uint32_t slot_bytes, int uin, int upw) {
    asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(s.x), "=r"(s.y) : "r"(base + uin * 8));
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] = lds128(base + slot_bytes + (uint32_t)(k * upw + uin) * 16u);
  }
  __device__ uint32_t off(int e) const {
    uint32_t q = e < 2 ? s.x : s.y;
    return (e & 1) ? (q >> 16) : (q & 0xffffu);
  }
  __device__ uint32_t word(int w) const {
    const uint4& q = v[w >> 2];
    return (w & 3) == 0 ? q.x : (w & 3) == 1 ? q.y : (w & 3) == 2 ? q.z : q.w;
  }
  __device__ float val(int e, int gi) const { return __uint_as_float(word(e * G + gi)); }
};

template <int G> struct GStep<XCT_MIXED, G> {
  static constexpr int NV = G / 2;                  // 4 entries * G * 2 B / 16
  uint2 s;
  uint4 v[NV];
  // sp: this unit's 4 slots of the step; vp: its NV value pieces
  // sp: this unit's 4 slots of the step; vp: its first value piece, piece k
  // upw pieces further (values [NV][units][16 B] per step)
  __device__ void load(const uint16_t* sp, const uint4* vp, int upw, uint64_t pol) {
    s = ld_stream_u2(sp, pol);
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] = ld_stream_u4(vp + (int64_t)k * upw, pol);
  }
  // the same step from a shared-memory copy of the warp's step at `base`
  __device__ void lds(uint32_t base, uint32_t slot_bytes, int uin, int upw) {
    asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(s.x), "=r"(s.y) : "r"(base + uin * 8));
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] = lds128(base + slot_bytes + (uint32_t)(k * upw + uin) * 16u);
  }
  __device__ uint32_t off(int e) const {
    uint32_t q = e < 2 ? s.x : s.y;
    return (e & 1) ? (q >> 16) : (q & 0xffffu);
  }
  __device__ unsigned short val(int e, int gi) const {
    const int h = e * G + gi, w = h >> 1;
    const uint4& q = v[w >> 2];
    const uint32_t x = (w & 3) == 0 ? q.x : (w & 3) == 1 ? q.y : (w & 3) == 2 ? q.z : q.w;
    return (unsigned short)((h & 1) ? (x >> 16) : (x & 0xffffu));
  }
};

template <int NPL, int G, typename A, typename St>
__device__ __forceinline__ void consume_g(A (&acc)[G], const St& cur, const uint32_t (&pb)[NPL],
                                          uint32_t lim) {
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const uint32_t off = cur.off(e);
    XCT_CHECK(off < lim);
#pragma unroll
    for (int qq = 0; qq < NPL; ++qq) {
      const uint4 r = lds128(pb[qq] + off);
#pragma unroll
      for (int gi = 0; gi < G; ++gi) acc[gi].fma(qq, r, cur.val(e, gi));
    }
  }
}

// ring depth: as deep as the registers allow (values of a step: 4*NV regs)
template <int PREC, int NPL, int G> struct RingDepth {
  static constexpr int nv = GStep<PREC, G>::NV;
  static constexpr int acc = NPL * (PREC == XCT_MIXED ? 8 : 4) * G;
  static constexpr int value = acc + 4 * nv * 3 <= 72 ? 4 : acc + 4 * nv * 2 <= 80 ? 3 : 2;
};

// mbarrier + bulk-copy helpers (the BULK entry ring)
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
               :: "r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes,
                                         uint32_t bar, uint64_t pol) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
               " [%0], [%1], %2, [%3], %4;"
               :: "r"(dst), "l"(src), "r"(bytes), "r"(bar), "l"(pol) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                 " selp.u32 %0, 1, 0, p;\n}" : "=r"(done) : "r"(bar), "r"(parity) : "memory");
  } while (!done);
}

constexpr int kBulkRing = 6;     // steps of a warp's entry stream in flight

template <int PREC, int NPL, int G, bool CONTRACT, bool BULK>
__global__ void __launch_bounds__(512) spmm_grouped_kernel(const Params p) {
  using A = Acc<PREC, NPL, CONTRACT>;
  using St = GStep<PREC, G>;
  constexpr int V = A::V;
  extern __shared__ uint4 stage[];
  const int64_t id = blockIdx.x;
  const int CG = p.chunk_group;
  const int b = (int)((id / CG) % p.n_cta);
  const int chunk = (int)(id / ((int64_t)CG * p.n_cta)) * CG + (int)(id % CG);
  const int lg = p.log2_lanes;               // lanes per unit = 1 << lg
  const int lp = p.log2_pieces;
  const int upw = 32 >> lg;                  // units per warp
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int uin = lane >> lg, sub = lane & ((1 << lg) - 1);
  const uint4* xb = p.x + (int64_t)chunk * p.x_chunk_pieces;
  const uint64_t pol_x = policy_evict_last(), pol_e = policy_evict_first();
  const uint32_t s0 = (uint32_t)__cvta_generic_to_shared(stage);
  const uint32_t bb = buffer_bytes(lp, p.plane_slots);
  uint32_t pbase[NPL];
#pragma unroll
  for (int qq = 0; qq < NPL; ++qq) pbase[qq] = plane_base(sub * NPL + qq, lp, p.plane_slots);

  A acc[G];
#pragma unroll
  for (int gi = 0; gi < G; ++gi) acc[gi].zero();
  const int g0 = p.cta_group_ptr[b], g1 = p.cta_group_ptr[b + 1];
  const int64_t step = (int64_t)upw * 4;
  int64_t at = (g0 < g1 ? p.slab_off[(int64_t)g0 * p.warps_per_cta + warp] : 0) +
               (int64_t)uin * 4;
  constexpr int D = RingDepth<PREC, NPL, G>::value;
  // The warp's steps of all groups form one stream: r[i] holds the steps
  // k = i mod D, and the load of step k + D is issued as soon as step k is
  // consumed, straight through group boundaries (one copy of the unrolled
  // body -- phase-specialised copies overflow the instruction cache).
  // Load pointers run D steps ahead: slots + position, values + position/4
  // * NV pieces (a unit's step = NV contiguous pieces).
  const uint16_t* lsp = p.slots + at;
  const uint4* lvp = reinterpret_cast<const uint4*>(p.values) + (at - 4 * uin) / 4 * St::NV + uin;
  const int64_t vstep = (int64_t)St::NV * upw;
  St r[BULK ? 1 : D];
  if constexpr (!BULK) {
#pragma unroll
    for (int i = 0; i < D; ++i) {
      r[i].load(lsp, lvp, upw, pol_e);
      lsp += step;
      lvp += vstep;
    }
  }
  // BULK: the warp's entry stream (slots, values) goes through a
  // kBulkRing-step shared-memory ring filled by cp.async.bulk with one
  // mbarrier per ring slot -- no registers hold loads in flight.
  const uint32_t slot_bytes = (uint32_t)upw * 8u;
  const uint32_t step_bytes = slot_bytes + (uint32_t)upw * St::NV * 16u;
  const uint32_t ring_off = (2 * bb + 2u * (uint32_t)p.plane_slots * 4u + 127u) & ~127u;
  const uint32_t ring = s0 + ring_off + (uint32_t)warp * kBulkRing * step_bytes;
  const uint32_t bars = s0 + ring_off + (uint32_t)(blockDim.x >> 5) * kBulkRing * step_bytes +
                        (uint32_t)warp * kBulkRing * 8u;
  const int64_t pos0 = g0 < g1 ? p.slab_off[(int64_t)g0 * p.warps_per_cta + warp] : 0;
  const char* gsl = reinterpret_cast<const char*>(p.slots + pos0);
  const char* gvl = reinterpret_cast<const char*>(p.values) + pos0 * G * (PREC == XCT_SINGLE ? 4 : 2);
  int64_t total = 0;
  if constexpr (BULK) {
    for (int gg = g0; gg < g1; ++gg) total += p.slab_width[(int64_t)gg * p.warps_per_cta + warp] >> 2;
    if (lane == 0) {
      for (int k = 0; k < kBulkRing; ++k) mbar_init(bars + 8u * k, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      for (int64_t k = 0; k < kBulkRing && k < total; ++k) {
        mbar_expect_tx(bars + 8u * (uint32_t)k, step_bytes);
        bulk_g2s(ring + (uint32_t)k * step_bytes, gsl + k * slot_bytes, slot_bytes,
                 bars + 8u * (uint32_t)k, pol_e);
        bulk_g2s(ring + (uint32_t)k * step_bytes + slot_bytes,
                 gvl + k * (int64_t)(step_bytes - slot_bytes), step_bytes - slot_bytes,
                 bars + 8u * (uint32_t)k, pol_e);
      }
    }
    __syncwarp();
  }
  int32_t* const maps = reinterpret_cast<int32_t*>(
      reinterpret_cast<char*>(stage) + 2 * (size_t)bb);
  int32_t* const map0 = maps;
  int32_t* const map1 = maps + p.plane_slots;
  int64_t mp0 = g0 < g1 ? p.group_map_ptr[g0] : 0;
  int64_t mp1 = g0 < g1 ? p.group_map_ptr[g0 + 1] : 0;
  int64_t mp2 = g0 + 1 < g1 ? p.group_map_ptr[g0 + 2] : mp1;
  if (g0 < g1) {
    map_fill(p, map0, mp0, (int)(mp1 - mp0));
    if (g0 + 1 < g1) map_fill(p, map1, mp1, (int)(mp2 - mp1));
    cp_async_commit();
    cp_async_wait_all();
    __syncthreads();
    stage_fill(p, xb, s0, map0, (int)(mp1 - mp0), lp, pol_x);
  }
  cp_async_commit();
  int g = g0 - 1, left = 0;
  uint32_t pb[NPL];
#pragma unroll
  for (int qq = 0; qq < NPL; ++qq) pb[qq] = s0 + pbase[qq];
  // enter group gn: its records are staged (barrier), start staging gn + 1
  auto enter = [&](int gn) {
    const int odd = (gn - g0) & 1;
    left = p.slab_width[(int64_t)gn * p.warps_per_cta + warp] >> 2;
    const int64_t mp3 = gn + 3 <= g1 ? p.group_map_ptr[min(gn + 3, g1)] : mp2;
    cp_async_wait_all();
    __syncthreads();
    if (gn + 1 < g1)
      stage_fill(p, xb, s0 + (odd ? 0u : bb), odd ? map0 : map1, (int)(mp2 - mp1), lp, pol_x);
    if (gn + 2 < g1)
      map_fill(p, odd ? map1 : map0, mp2, (int)(mp3 - mp2));
    cp_async_commit();
    mp1 = mp2;
    mp2 = mp3;
#pragma unroll
    for (int qq = 0; qq < NPL; ++qq) pb[qq] = s0 + (odd ? bb : 0u) + pbase[qq];
  };
  if constexpr (BULK) {
    auto fetch = [&](int64_t k, St& out) {
      const uint32_t sl = (uint32_t)(k % kBulkRing);
      mbar_wait(bars + 8u * sl, (uint32_t)((k / kBulkRing) & 1));
      out.lds(ring + sl * step_bytes, slot_bytes, uin, upw);
    };
    St cur, nxt;
    if (total > 0) fetch(0, cur);
    for (int64_t k = 0; k < total; ++k) {
      while (left == 0) enter(++g);
      if (k + 1 < total) fetch(k + 1, nxt);
      consume_g<NPL, G>(acc, cur, pb, 16u * (uint32_t)p.plane_slots);
      __syncwarp();                     // every lane is done with ring slot k
      const int64_t kn = k + kBulkRing;
      if (lane == 0 && kn < total) {
        const uint32_t sl = (uint32_t)(k % kBulkRing);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(bars + 8u * sl, step_bytes);
        bulk_g2s(ring + sl * step_bytes, gsl + kn * slot_bytes, slot_bytes, bars + 8u * sl, pol_e);
        bulk_g2s(ring + sl * step_bytes + slot_bytes,
                 gvl + kn * (int64_t)(step_bytes - slot_bytes), step_bytes - slot_bytes,
                 bars + 8u * sl, pol_e);
      }
      cur = nxt;
      --left;
    }
    while (++g < g1) enter(g);          // trailing groups empty for this warp
  } else {
    for (;;) {
#pragma unroll
      for (int i = 0; i < D; ++i) {
        while (left == 0) {
          if (++g >= g1) goto done;
          enter(g);
        }
        consume_g<NPL, G>(acc, r[i], pb, 16u * (uint32_t)p.plane_slots);
        r[i].load(lsp, lvp, upw, pol_e);
        lsp += step;
        lvp += vstep;
        --left;
      }
    }
  }
done:
  cp_async_wait_all();

  // ---- epilogue: G rows per unit ------------------------------------------
  double sq = 0.0;
  const float sc = ldexpf(1.0f, -p.scale_exp);
  const float f = p.factors ? (float)p.factors[chunk] : 1.0f;
  const int j0 = sub * NPL * V;
#pragma unroll
  for (int gi = 0; gi < G; ++gi) {
    const int row = p.cta_rows[(int64_t)b * p.rows_per_cta + (warp * upw + uin) * G + gi];
    if (row < 0) continue;
    float* out = out_row<float>(p, row, chunk);
    store_row<NPL * V>(out, j0, chunk, p, [&](int i) { return acc[gi].out(i, sc) * f; }, sq);
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

template <int PREC, int NPL, int G, bool CONTRACT, bool BULK>
int launch_grouped(const Params& p, int64_t n_chunks, int threads, int64_t smem, cudaStream_t s) {
  static int configured = -1;
  if (configured < (int)smem) {
    cudaError_t e = cudaFuncSetAttribute(spmm_grouped_kernel<PREC, NPL, G, CONTRACT, BULK>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess)
      return xct::fail(XCT_ECUDA, std::string("spmm smem attribute: ") + cudaGetErrorString(e));
    configured = (int)smem;
  }
  if (threads > 512) return xct::fail(XCT_EINVAL, "spmm: grouped rows need <= 16 warps per CTA");
  const int64_t n_blocks = (int64_t)p.n_cta * n_chunks;
  if (n_blocks > 0x7fffffffLL) return xct::fail(XCT_EINVAL, "spmm: grid too large");
  spmm_grouped_kernel<PREC, NPL, G, CONTRACT, BULK><<<(unsigned)n_blocks, threads, smem, s>>>(p);
  XCT_CUDA_CHECK_LAUNCH("spmm_grouped");
  return XCT_OK;
}

template <int PREC, bool CONTRACT, bool BULK>
int launch_grouped_b(const Params& p, int npl, int G, int64_t n_chunks, int threads,
                     int64_t smem, cudaStream_t s) {
  if (npl == 1 && G == 2) return launch_grouped<PREC, 1, 2, CONTRACT, BULK>(p, n_chunks, threads, smem, s);
  if (npl == 1 && G == 4) return launch_grouped<PREC, 1, 4, CONTRACT, BULK>(p, n_chunks, threads, smem, s);
  if (npl == 2 && G == 2) return launch_grouped<PREC, 2, 2, CONTRACT, BULK>(p, n_chunks, threads, smem, s);
  if (npl == 2 && G == 4) return launch_grouped<PREC, 2, 4, CONTRACT, BULK>(p, n_chunks, threads, smem, s);
  if (npl == 4 && G == 2) return launch_grouped<PREC, 4, 2, CONTRACT, BULK>(p, n_chunks, threads, smem, s);
  return xct::fail(XCT_EINVAL, "spmm: grouped rows need G in {2, 4} and 1 or 2 pieces per lane (4 with G 2)");
}

// The register ring is the default; XCT_SPMM_BULK=1 selects the bulk-copy
// shared-memory entry ring (measured slower at c2: 80.7 / 64.6 ms vs 61.7 /
// 48.8 ms -- the extra shared-memory traffic and per-step mbarrier waits
// cost more than the load latency they hide; profiles/r01_probe_c2_bulk*).
bool use_bulk() {
  const char* e = std::getenv("XCT_SPMM_BULK");
  return e && e[0] == '1';
}

template <int PREC, bool CONTRACT>
int launch_grouped_npl(const Params& p, int npl, int G, int64_t n_chunks, int threads,
                       int64_t smem, cudaStream_t s) {
  if (use_bulk()) return launch_grouped_b<PREC, CONTRACT, true>(p, npl, G, n_chunks, threads, smem, s);
  return launch_grouped_b<PREC, CONTRACT, false>(p, npl, G, n_chunks, threads, smem, s);
  return xct::fail(XCT_EINVAL, "spmm: grouped rows need G in {2, 4} and 1 or 2 pieces per lane");
}

}  // namespace

extern "C" int xct_spmm(const xct_staged* a, int precision, const void* d_x, int64_t n_in,
                        int64_t n_chunks, int32_t f_dev, const xct_epilogue* ep,
                        int64_t smem_bytes, void* stream) {
  if (!a || !ep || !d_x || (!ep->d_out && !ep->d_out_ptrs))
    return xct::fail(XCT_EINVAL, "spmm: null argument");
  if (precision < 0 || precision > 3) return xct::fail(XCT_EINVAL, "spmm: bad precision");
  if (ep->accumulate) return xct::fail(XCT_EINVAL, "spmm: accumulate mode is reserved");
  const int G = a->row_group > 1 ? a->row_group : 1;
  if (G > 1 && precision != XCT_SINGLE && precision != XCT_MIXED)
    return xct::fail(XCT_EINVAL, "spmm: grouped rows support single and mixed only");
  const bool packed = (precision == XCT_HALF || precision == XCT_MIXED) && G == 1;
  if (!a->d_values || (!packed && !a->d_slots))
    return xct::fail(XCT_EINVAL, "spmm: missing entry arrays");
  const int vbytes = precision == XCT_DOUBLE ? 8 : precision == XCT_SINGLE ? 4 : 2;
  const int64_t rec = (int64_t)f_dev * vbytes;
  if (rec < 16 || rec > 512 || (rec & (rec - 1)))
    return xct::fail(XCT_EINVAL, "spmm: f_dev*elem_bytes must be a power of two in [16, 512]");
  int lp = 0;
  while ((16 << lp) < rec) ++lp;                      // pieces per record = 1 << lp
  if (a->rows_per_warp % G) return xct::fail(XCT_EINVAL, "spmm: rows_per_warp % row_group");
  const int64_t upw = a->rows_per_warp / G;         // units (row groups) per warp
  int lg = 0;                                         // lanes per unit = 1 << lg
  while ((32 >> lg) > upw && lg < 5) ++lg;
  if ((32 >> lg) != upw || lg > lp)
    return xct::fail(XCT_EINVAL, "spmm: units per warp must be 32 / lanes with lanes <= pieces");
  const int npl = 1 << (lp - lg);
  if (a->n_cta == 0 || n_chunks == 0) return XCT_OK;
  if (n_chunks > 65535) return xct::fail(XCT_EINVAL, "spmm: too many chunks for one launch");
  if (a->contract && precision != XCT_SINGLE)
    return xct::fail(XCT_EINVAL, "spmm: contract applies to single precision only");
  // largest power of two <= chunk_group that divides n_chunks
  int CG = 1;
  while (CG * 2 <= a->chunk_group && n_chunks % (CG * 2) == 0) CG *= 2;
  const int threads = (int)(a->warps_per_cta * 32);
  if (threads < 32 || threads > 1024) return xct::fail(XCT_EINVAL, "spmm: CTA must have 1..32 warps");
  const int64_t plane_slots = (a->max_group_slots + 7) & ~(int64_t)7;
  if (plane_slots * 16 > 65536) return xct::fail(XCT_ESTAGE, "spmm: plane offsets exceed 16 bits");
  // double-buffered stage + two slot->element maps (+ the grouped kernel's
  // per-warp bulk entry ring and its mbarriers, 128-byte aligned)
  int64_t need = 2 * ((plane_slots << (lp + 4)) + 128) + 2 * plane_slots * 4;
  if (G > 1 && use_bulk()) {
    const int64_t upw_ = a->rows_per_warp / G;
    const int64_t nv = 4 * G * (precision == XCT_SINGLE ? 4 : 2) / 16;
    const int64_t step_b = upw_ * 8 + upw_ * nv * 16;
    need = ((need + 127) & ~(int64_t)127) + a->warps_per_cta * kBulkRing * (step_b + 8);
  }
  if (smem_bytes < need) smem_bytes = need;
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
  // input layout: chunk-major [n_chunks][n_in][record] unless the caller
  // gives strides in records (e.g. element-major [n_in][n_chunks][record])
  p.x_chunk_pieces = (ep->x_chunk_stride ? ep->x_chunk_stride : n_in) << lp;
  p.x_elem_pieces = (int32_t)((ep->x_elem_stride ? ep->x_elem_stride : 1) << lp);
  if ((uint64_t)n_in * (uint64_t)p.x_elem_pieces >= (1ull << 32))
    return xct::fail(XCT_EINVAL, "spmm: input element offsets exceed 32 bits");
  p.rows_per_cta = (int32_t)a->rows_per_cta;
  p.warps_per_cta = (int32_t)a->warps_per_cta;
  p.log2_lanes = lg;
  p.log2_pieces = lp;
  p.n_cta = (int32_t)a->n_cta;
  p.plane_slots = (int32_t)plane_slots;
  p.chunk_group = CG;
  p.n_chunks = (int32_t)n_chunks;
  p.out = ep->d_out;
  p.row_stride = ep->row_stride;
  p.chunk_stride = ep->chunk_stride;
  p.valid_cols = ep->valid_cols;
  p.ffactor = ep->ffactor;
  p.scale_exp = ep->value_scale_exp;
  p.factors = ep->d_factors;
  p.dot_partials = ep->d_dot_partials;
  p.out_ptrs = ep->d_out_ptrs;
  p.seg = ep->d_seg;
  p.n_seg = ep->n_seg;
  if (p.out_ptrs && (!p.seg || p.n_seg < 1))
    return xct::fail(XCT_EINVAL, "spmm: scattered output needs its segments");
  cudaStream_t s = (cudaStream_t)stream;
  if (G > 1) {
    if (precision == XCT_MIXED)
      return launch_grouped_npl<XCT_MIXED, false>(p, npl, G, n_chunks, threads, smem_bytes, s);
    return a->contract
               ? launch_grouped_npl<XCT_SINGLE, true>(p, npl, G, n_chunks, threads, smem_bytes, s)
               : launch_grouped_npl<XCT_SINGLE, false>(p, npl, G, n_chunks, threads, smem_bytes, s);
  }
  switch (precision) {
    case XCT_DOUBLE: return launch_npl<XCT_DOUBLE>(p, npl, n_chunks, threads, smem_bytes, s);
    case XCT_SINGLE:
      return a->contract ? launch_npl<XCT_SINGLE, true>(p, npl, n_chunks, threads, smem_bytes, s)
                         : launch_npl<XCT_SINGLE>(p, npl, n_chunks, threads, smem_bytes, s);
    case XCT_HALF: return launch_npl<XCT_HALF>(p, npl, n_chunks, threads, smem_bytes, s);
    default: return launch_npl<XCT_MIXED>(p, npl, n_chunks, threads, smem_bytes, s);
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
