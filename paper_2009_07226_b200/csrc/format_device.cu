// K5 on the device: the staged SpMM execution format built in HBM.
//
// Same format, same bytes as the host builder (format_build.cpp,
// xct_format_build with row_group 1) for the two staging-key families the
// B200 operator uses -- image bands for the projection A and view angles
// for the back projection A^T (matrixstore.forward_plan / adjoint_plan) --
// so the host builder is the device builder's test oracle at small sizes.
// Replaces matrixstore.build_staged / pack (src/matrixstore.py:250-262,
// :417-562) for those plans.
//
// A column's staging key and its coordinate inside the key follow from the
// column id (mode per CTA tile):
//   mode 0  key = col / B, coord = col % B   (z bands of A; views of A^T)
//   mode 1  key = col % B, coord = col / B   (x bands, ascending)
//   mode 2  key = B-1-col % B, coord = col / B (x bands, descending)
// so a tile's footprint sorted by (key, col) is, per key, the touched
// coordinates of [lo_key, hi_key] in ascending order.  Per tile:
//   ranges  lo/hi per key (shared-memory atomics over the tile's entries);
//   count   a bitmap of touched (key, coord) cells -> compact slot of every
//           cell, load groups of whole keys (<= capacity slots, the host's
//           greedy cut), slab widths per (group, warp);
//   fill    group maps, slab offsets, and the slabs: per (group, warp,
//           quarter-warp) the host's bank-conflict schedule (proper edge
//           colouring of rows x bank classes by alternating paths, then the
//           compressed overflow placement) run by one thread, entries
//           written as packed (slot << 20 | fp16) words or slot/value pairs.
// Rows must list their entries in non-decreasing key order (true for
// traversal-ordered rays with band keys and for ray-ordered A^T rows);
// violations, capacity and size limits raise flags and the caller falls
// back to the host builder.
#include <cuda_fp16.h>

#include <climits>

#include "xct_common.h"

namespace {

constexpr int kGMax = 256;        // load groups per tile
constexpr int kNcMax = 256;       // colours (steps) per quarter schedule
constexpr int kEMax = 2048;       // edges per quarter schedule
constexpr int kRqMax = 8;         // rows per quarter-warp
constexpr int kFillThreads = 256;  // latency-bound schedule: more threads in flight

enum { FLAG_UNSORTED = 1, FLAG_CAPACITY = 2, FLAG_GROUPS = 4, FLAG_SPAN = 8, FLAG_SCHED = 16 };

struct Part {
  const int64_t* indptr;
  const int32_t* indices;
  const double* values;
  int64_t n_rows;
  const int32_t* cta_rows;
  const int32_t* cta_mode;
  int64_t n_cta;
  int32_t rows_per_cta, rows_per_warp, warps;
  int32_t B, n_keys, capacity, rq, fast;
};

__device__ __forceinline__ void key_coord(int mode, int32_t col, int B, int& key, int& coord) {
  if (mode == 0) { key = col / B; coord = col % B; }
  else if (mode == 1) { key = col % B; coord = col / B; }
  else { key = B - 1 - col % B; coord = col / B; }
}
__device__ __forceinline__ int32_t col_of(int mode, int key, int coord, int B) {
  if (mode == 0) return key * B + coord;
  if (mode == 1) return coord * B + key;
  return coord * B + (B - 1 - key);
}

// ---- ranges -----------------------------------------------------------------
__global__ void fmtd_ranges_k(Part p, int32_t* g_lo, int32_t* g_hi, int64_t* g_span, int* flag) {
  extern __shared__ int32_t sm[];
  int32_t* lo = sm;
  int32_t* hi = sm + p.n_keys;
  const int64_t tile = blockIdx.x;
  const int mode = p.cta_mode[tile];
  for (int k = threadIdx.x; k < p.n_keys; k += blockDim.x) { lo[k] = INT_MAX; hi[k] = -1; }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  bool unsorted = false;
  for (int t = warp; t < p.rows_per_cta; t += nw) {
    const int32_t r = p.cta_rows[tile * p.rows_per_cta + t];
    if (r < 0) continue;
    const int64_t j0 = p.indptr[r], j1 = p.indptr[r + 1];
    for (int64_t j = j0 + lane; j < j1; j += 32) {
      int key, coord;
      key_coord(mode, p.indices[j], p.B, key, coord);
      atomicMin(&lo[key], coord);
      atomicMax(&hi[key], coord);
      if (j + 1 < j1) {
        int k2, c2;
        key_coord(mode, p.indices[j + 1], p.B, k2, c2);
        unsorted |= k2 < key;
      }
    }
  }
  if (unsorted) atomicOr(flag, FLAG_UNSORTED);
  __syncthreads();
  int64_t span = 0;
  for (int k = threadIdx.x; k < p.n_keys; k += blockDim.x) {
    g_lo[tile * p.n_keys + k] = lo[k];
    g_hi[tile * p.n_keys + k] = hi[k];
    if (hi[k] >= lo[k]) span += hi[k] - lo[k] + 1;
  }
  for (int o = 16; o > 0; o >>= 1) span += __shfl_xor_sync(0xffffffffu, span, o);
  __shared__ int64_t red[32];
  if (lane == 0) red[warp] = span;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t s = 0;
    for (int i = 0; i < nw; ++i) s += red[i];
    g_span[tile] = s;
  }
}

// ---- per-tile state shared by count and fill ----------------------------------
struct Tile {
  int32_t *lo, *hi, *kbase, *key_group, *gk, *gsb, *bm, *wpre, *width, *sc;
  int ng, n_slots, max_gs, mode;
};

// exclusive scan of n ints in shared memory by the whole block; returns total
__device__ int block_scan(int32_t* a, int n) {
  __shared__ int32_t part[1024 / 32 + 1];
  __shared__ int32_t tot;
  const int T = blockDim.x;
  const int per = (n + T - 1) / T;
  const int b0 = threadIdx.x * per, b1 = min(n, b0 + per);
  int s = 0;
  for (int i = b0; i < b1; ++i) s += a[i];
  // inclusive scan of thread sums
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int v = s;
  for (int o = 1; o < 32; o <<= 1) {
    int u = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += u;
  }
  if (lane == 31) part[w] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int i = 0; i < (T >> 5); ++i) { int x = part[i]; part[i] = run; run += x; }
    tot = run;
  }
  __syncthreads();
  int run = part[w] + v - s;
  for (int i = b0; i < b1; ++i) { int x = a[i]; a[i] = run; run += x; }
  __syncthreads();
  const int total = tot;
  __syncthreads();
  return total;
}

// number of touched cells before bit b of the tile's key-ordered bitmap
__device__ __forceinline__ int bit_rank(const Tile& T, int b) {
  const int w = b >> 5, s = b & 31;
  return s ? T.wpre[w] + __popc((unsigned)T.bm[w] & ((1u << s) - 1u)) : T.wpre[w];
}

// lo/hi -> key bit bases, bitmap of touched cells, word prefix counts, the
// greedy group cut.  Returns false (flag set) when the tile does not fit.
__device__ bool tile_setup(const Part& p, int64_t tile, const int32_t* g_lo, const int32_t* g_hi,
                           int bm_words, Tile& T, int* flag) {
  const int nk = p.n_keys;
  for (int k = threadIdx.x; k < nk; k += blockDim.x) {
    const int l = g_lo[tile * nk + k], h = g_hi[tile * nk + k];
    T.lo[k] = l;
    T.hi[k] = h;
    T.kbase[k] = h >= l ? h - l + 1 : 0;
  }
  if (threadIdx.x == 0) T.kbase[nk] = 0;
  __syncthreads();
  const int span = block_scan(T.kbase, nk + 1);       // kbase[nk] = span
  if (span > bm_words * 32) {
    if (threadIdx.x == 0) atomicOr(flag, FLAG_SPAN);
    return false;
  }
  const int nwords = (span + 31) >> 5;
  for (int i = threadIdx.x; i < nwords; i += blockDim.x) T.bm[i] = 0;
  __syncthreads();
  T.mode = p.cta_mode[tile];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int t = warp; t < p.rows_per_cta; t += nw) {
    const int32_t r = p.cta_rows[tile * p.rows_per_cta + t];
    if (r < 0) continue;
    for (int64_t j = p.indptr[r] + lane; j < p.indptr[r + 1]; j += 32) {
      int key, coord;
      key_coord(T.mode, p.indices[j], p.B, key, coord);
      const int b = T.kbase[key] + coord - T.lo[key];
      atomicOr((unsigned*)&T.bm[b >> 5], 1u << (b & 31));
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nwords; i += blockDim.x) T.wpre[i] = __popc((unsigned)T.bm[i]);
  if (threadIdx.x == 0) T.wpre[nwords] = 0;
  __syncthreads();
  block_scan(T.wpre, nwords + 1);
  // greedy cut of whole keys into groups (format_build.cpp phase A)
  if (threadIdx.x == 0) {
    int g = -1, cur = 0, maxgs = 0, bad = 0;
    int prev_rank = 0;
    for (int k = 0; k < nk; ++k) {
      const int rk = bit_rank(T, T.kbase[k + 1]);
      const int m = rk - prev_rank;
      prev_rank = rk;
      if (m == 0) { T.key_group[k] = g < 0 ? 0 : g; continue; }
      if (m > p.capacity) { bad |= FLAG_CAPACITY; T.key_group[k] = g < 0 ? 0 : g; continue; }
      if (g < 0 || cur + m > p.capacity) {
        if (g >= 0) maxgs = max(maxgs, cur);
        ++g;
        if (g >= kGMax) { bad |= FLAG_GROUPS; g = kGMax - 1; }
        T.gk[g] = k;
        T.gsb[g] = rk - m;
        cur = 0;
      }
      cur += m;
      T.key_group[k] = g;
    }
    if (g >= 0) maxgs = max(maxgs, cur);
    T.sc[0] = g + 1;                   // n_groups
    T.sc[1] = prev_rank;               // n_slots
    T.sc[2] = maxgs;
    T.sc[3] = bad;
    T.gk[g + 1] = nk;
    T.gsb[g + 1] = prev_rank;
    if (bad) atomicOr(flag, bad);
  }
  __syncthreads();
  T.ng = T.sc[0];
  T.n_slots = T.sc[1];
  T.max_gs = T.sc[2];
  const bool ok = T.sc[3] == 0;
  __syncthreads();
  return ok;
}

// shared-memory carve-up (ints): lo, hi, kbase[nk+1], key_group, gk[G+1],
// gsb[G+1], width[G*warps], bm[bmw], wpre[bmw+1], scalars
__device__ int tile_carve(const Part& p, int bm_words, int32_t* sm, Tile& T) {
  const int nk = p.n_keys;
  int o = 0;
  T.lo = sm + o; o += nk;
  T.hi = sm + o; o += nk;
  T.kbase = sm + o; o += nk + 1;
  T.key_group = sm + o; o += nk;
  T.gk = sm + o; o += kGMax + 1;
  T.gsb = sm + o; o += kGMax + 1;
  T.width = sm + o; o += kGMax * p.warps;
  T.bm = sm + o; o += bm_words;
  T.wpre = sm + o; o += bm_words + 1;
  T.sc = sm + o; o += 4;
  return o;
}

// ---- count ------------------------------------------------------------------
__global__ void fmtd_count_k(Part p, const int32_t* g_lo, const int32_t* g_hi, int bm_words,
                             int64_t* counts, int32_t* g_width, int* flag) {
  extern __shared__ int32_t sm[];
  __shared__ int s_ng, s_slots, s_maxgs;
  Tile T;
  int o = tile_carve(p, bm_words, sm, T);
  int32_t* cnt = sm + o;                         // [nw][kGMax] per CUDA warp
  const int64_t tile = blockIdx.x;
  if (!tile_setup(p, tile, g_lo, g_hi, bm_words, T, flag)) return;
  if (threadIdx.x == 0) { s_ng = T.ng; s_slots = T.n_slots; s_maxgs = T.max_gs; }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int i = threadIdx.x; i < kGMax * p.warps; i += blockDim.x) T.width[i] = 0;
  for (int i = threadIdx.x; i < nw * kGMax; i += blockDim.x) cnt[i] = 0;
  __syncthreads();
  const int mode = p.cta_mode[tile];
  int32_t* mine = cnt + warp * kGMax;
  for (int t = warp; t < p.rows_per_cta; t += nw) {
    const int32_t r = p.cta_rows[tile * p.rows_per_cta + t];
    if (r < 0) continue;
    const int64_t j0 = p.indptr[r], j1 = p.indptr[r + 1];
    if (j1 == j0) continue;
    for (int64_t j = j0 + lane; j < j1; j += 32) {
      int key, coord;
      key_coord(mode, p.indices[j], p.B, key, coord);
      atomicAdd(&mine[T.key_group[key]], 1);
    }
    __syncwarp();
    int kf, kl, c_;
    key_coord(mode, p.indices[j0], p.B, kf, c_);
    key_coord(mode, p.indices[j1 - 1], p.B, kl, c_);
    const int gf = T.key_group[kf], gl = T.key_group[kl];
    const int w = t / p.rows_per_warp;
    for (int g = gf + lane; g <= gl; g += 32) {
      const int c = mine[g];
      if (c) atomicMax(&T.width[g * p.warps + w], (c + 3) & ~3);
      mine[g] = 0;
    }
    __syncwarp();
  }
  __syncthreads();
  const int ng = s_ng;
  int64_t padded = 0;
  for (int i = threadIdx.x; i < ng * p.warps; i += blockDim.x) {
    g_width[tile * kGMax * p.warps + i] = T.width[i];
    padded += (int64_t)T.width[i] * p.rows_per_warp;
  }
  for (int o2 = 16; o2 > 0; o2 >>= 1) padded += __shfl_xor_sync(0xffffffffu, padded, o2);
  __shared__ int64_t red[32];
  if (lane == 0) red[warp] = padded;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t s = 0;
    for (int i = 0; i < nw; ++i) s += red[i];
    counts[tile * 4 + 0] = ng;
    counts[tile * 4 + 1] = s_slots;
    counts[tile * 4 + 2] = s_maxgs;
    counts[tile * 4 + 3] = s;
  }
}

// ---- the host's quarter-warp bank schedule (format_build.cpp Colorer /
// QuarterScheduler), one thread, scratch in global memory ------------------------
struct Sched {
  // colourer
  int nc, words, ne;
  int16_t* atL;     // [kRqMax * nc]
  int16_t* atR;     // [8 * nc]
  uint64_t* freeL;  // [kRqMax * 4]
  uint64_t* freeR;  // [8 * 4]
  uint8_t* er;      // [kEMax] row
  uint8_t* ec;      // [kEMax] class
  int16_t* col;     // [kEMax] colour = step
  int16_t* path;    // [kEMax]
  // scheduler
  int16_t* eslot;   // [kEMax]
  int16_t* eidx;    // [kEMax] entry index inside the row's group span
  uint8_t* busy;    // [kRqMax * kNcMax]
  int16_t* ccnt;    // [kNcMax * 8]
  int16_t* fslot;   // [kNcMax * 8]
  int16_t* sslot;   // [kNcMax]
  uint8_t* used;    // [kRqMax * kNcMax]

  __device__ void carve(char* base) {
    char* q = base;
    atL = (int16_t*)q; q += kRqMax * kNcMax * 2;
    atR = (int16_t*)q; q += 8 * kNcMax * 2;
    freeL = (uint64_t*)q; q += kRqMax * 4 * 8;
    freeR = (uint64_t*)q; q += 8 * 4 * 8;
    er = (uint8_t*)q; q += kEMax;
    ec = (uint8_t*)q; q += kEMax;
    col = (int16_t*)q; q += kEMax * 2;
    path = (int16_t*)q; q += kEMax * 2;
    eslot = (int16_t*)q; q += kEMax * 2;
    eidx = (int16_t*)q; q += kEMax * 2;
    busy = (uint8_t*)q; q += kRqMax * kNcMax;
    ccnt = (int16_t*)q; q += kNcMax * 8 * 2;
    fslot = (int16_t*)q; q += kNcMax * 8 * 2;
    sslot = (int16_t*)q; q += kNcMax * 2;
    used = (uint8_t*)q; q += kRqMax * kNcMax;
  }
  __host__ __device__ static constexpr int64_t bytes() {
    return kRqMax * kNcMax * 2 + 8 * kNcMax * 2 + kRqMax * 32 + 8 * 32 + 2 * kEMax +
           4 * kEMax * 2 + kRqMax * kNcMax + 2 * kNcMax * 8 * 2 + kNcMax * 2 + kRqMax * kNcMax;
  }
  __device__ void trim(uint64_t* f, int v) {
    const int rem = nc % 64;
    if (rem) f[v * 4 + words - 1] = (1ull << rem) - 1;
  }
  __device__ void reset(int nl, int ncol) {
    nc = ncol;
    words = (ncol + 63) / 64;
    ne = 0;
    for (int i = 0; i < nl * nc; ++i) atL[i] = -1;
    for (int i = 0; i < 8 * nc; ++i) atR[i] = -1;
    for (int v = 0; v < nl; ++v) {
      for (int w = 0; w < words; ++w) freeL[v * 4 + w] = ~0ull;
      trim(freeL, v);
    }
    for (int v = 0; v < 8; ++v) {
      for (int w = 0; w < words; ++w) freeR[v * 4 + w] = ~0ull;
      trim(freeR, v);
    }
  }
  __device__ int first_free(const uint64_t* f, int v) const {
    for (int w = 0; w < words; ++w) {
      const uint64_t m = f[v * 4 + w];
      if (m) return w * 64 + __ffsll((long long)m) - 1;
    }
    return -1;
  }
  __device__ void put(int e, int c) {
    col[e] = (int16_t)c;
    atL[er[e] * nc + c] = (int16_t)e;
    atR[ec[e] * nc + c] = (int16_t)e;
    freeL[er[e] * 4 + c / 64] &= ~(1ull << (c % 64));
    freeR[ec[e] * 4 + c / 64] &= ~(1ull << (c % 64));
  }
  __device__ void take(int e) {
    const int c = col[e];
    atL[er[e] * nc + c] = -1;
    atR[ec[e] * nc + c] = -1;
    freeL[er[e] * 4 + c / 64] |= 1ull << (c % 64);
    freeR[ec[e] * 4 + c / 64] |= 1ull << (c % 64);
  }
  // Colorer::add (max_path 0: alternating paths -- the host's algorithm;
  // max_path < 0: first fit, see below)
  static constexpr int16_t kOverflowCol = 0x7fff;
  __device__ bool add(int l, int r, int max_path = 0) {
    const int e = ne++;
    er[e] = (uint8_t)l;
    ec[e] = (uint8_t)r;
    col[e] = -1;
    const int a = first_free(freeL, l), b = first_free(freeR, r);
    if (a < 0 || b < 0) return false;
    if (atR[r * nc + a] >= 0) {
      // max_path < 0: no alternating path (first fit; the paired schedule
      // of A); a refused edge goes to the caller's overflow placement
      if (max_path < 0) { col[e] = kOverflowCol; return true; }
      int np = 0, v = r, want = a;
      bool right = true;
      for (;;) {
        const int e2 = right ? atR[v * nc + want] : atL[v * nc + want];
        if (e2 < 0) break;
        path[np++] = (int16_t)e2;
        v = right ? er[e2] : ec[e2];
        right = !right;
        want = want == a ? b : a;
      }
      for (int i = 0; i < np; ++i) take(path[i]);
      for (int i = 0; i < np; ++i) put(path[i], col[path[i]] == a ? b : a);
    }
    put(e, a);
    return true;
  }
};

struct FillArgs {
  Part p;
  const int32_t* g_lo;
  const int32_t* g_hi;
  int bm_words;
  const int32_t* g_width;
  const int64_t* tile_base;   // [n_cta][3]: group, slot, entry bases (part-relative)
  int precision, scale_exp;
  int32_t* group_map;
  int64_t* group_map_ptr;
  int64_t* slab_off;
  int32_t* slab_width;
  uint16_t* slots;            // unpacked (single/double), or null
  void* values;               // packed u32 (half/mixed) / f32 / f64
  char* scratch;
  int* flag;
  unsigned long long* qstats; // [0] max rel quant error bits, [1] underflow count
};

__device__ __forceinline__ void write_entry(const FillArgs& a, int64_t at, int slot, int64_t j,
                                            double scale, double& wmax, int64_t& nunder) {
  double v = 0.0, back = 0.0;
  XCT_CHECK(slot >= 0 && slot < a.p.capacity && at >= 0);
  XCT_CHECK(j < 0 || (j >= a.p.indptr[0] && j < a.p.indptr[a.p.n_rows]));
  if (j >= 0) v = a.p.values[j] * scale;
  if (a.precision == XCT_HALF || a.precision == XCT_MIXED) {
    uint32_t h = 0;
    if (j >= 0) {
      const __half hv = __double2half(v);
      h = __half_as_ushort(hv);
      back = (double)__half2float(hv);
    }
    ((uint32_t*)a.values)[at] = ((uint32_t)slot << 20) | h;
  } else {
    a.slots[at] = (uint16_t)(slot << 4);
    if (a.precision == XCT_SINGLE) {
      const float f = (float)v;
      ((float*)a.values)[at] = f;
      back = (double)f;
    } else {
      ((double*)a.values)[at] = v;
      back = v;
    }
  }
  if (j >= 0 && v != 0.0) {
    if (back == 0.0) ++nunder;
    const double rel = fabs(back - v) / fabs(v);
    if (rel > wmax) wmax = rel;
  }
}

// Fast bank schedule of one (group, warp, quarter-warp): first fit over
// step masks of NW 64-bit words (width <= 64 * NW) -- each entry takes the
// first step where its row is free and no other row of the quarter reads
// its bank class, else the first step where its row is free (one extra
// wavefront).  Same entries per row and slab as the host schedule, other
// steps: sums equal to rounding (native order).  Idle lanes re-read the
// slot the quarter's first busy row reads at that step (broadcast), as the
// host schedule does.
template <int NW>
__device__ void greedy_quarter(const FillArgs& a, const Tile& T, int64_t tile, int w, int q,
                               int rq, int rpw, int width, int k0, int k1, int gsb, int64_t so,
                               double scale, uint64_t* taken, double& wmax, int64_t& nunder) {
  const Part& p = a.p;
  const int cmask = rq - 1;
  uint64_t valid[NW];
#pragma unroll
  for (int k = 0; k < NW; ++k) {
    const int lo = k * 64;
    valid[k] = width >= lo + 64 ? ~0ull : (width > lo ? ((1ull << (width - lo)) - 1ull) : 0ull);
  }
  for (int i = 0; i < 8 * NW; ++i) taken[i] = 0ull;
  uint64_t used[kRqMax][NW];
#pragma unroll
  for (int rr = 0; rr < kRqMax; ++rr) {
#pragma unroll
    for (int k = 0; k < NW; ++k) used[rr][k] = 0ull;
    if (rr >= rq) continue;
    const int rin = q * rq + rr;
    const int32_t r = p.cta_rows[tile * p.rows_per_cta + w * rpw + rin];
    if (r < 0) continue;
    const int64_t hi_j = p.indptr[r + 1];
    int64_t L = p.indptr[r], H = hi_j;
    while (L < H) {
      const int64_t M = (L + H) >> 1;
      int key, coord;
      key_coord(T.mode, p.indices[M], p.B, key, coord);
      if (key < k0) L = M + 1; else H = M;
    }
    for (int64_t j = L; j < hi_j; ++j) {
      int key, coord;
      key_coord(T.mode, p.indices[j], p.B, key, coord);
      if (key >= k1) break;
      const int slot = bit_rank(T, T.kbase[key] + coord - T.lo[key]) - gsb;
      const int c = slot & cmask;
      int n = -1;
#pragma unroll
      for (int k = 0; k < NW; ++k) {
        const uint64_t m = ~used[rr][k] & ~taken[c * NW + k] & valid[k];
        if (n < 0 && m) n = k * 64 + __ffsll((long long)m) - 1;
      }
      if (n < 0) {
#pragma unroll
        for (int k = 0; k < NW; ++k) {
          const uint64_t m = ~used[rr][k] & valid[k];
          if (n < 0 && m) n = k * 64 + __ffsll((long long)m) - 1;
        }
      }
#pragma unroll
      for (int k = 0; k < NW; ++k)
        if ((n >> 6) == k) {
          used[rr][k] |= 1ull << (n & 63);
          taken[c * NW + k] |= 1ull << (n & 63);
        }
      write_entry(a, so + ((int64_t)(n >> 2) * rpw + rin) * 4 + (n & 3), slot, j, scale, wmax,
                  nunder);
    }
  }
  for (int n = 0; n < width; ++n) {
    int src = -1;
#pragma unroll
    for (int rr = kRqMax - 1; rr >= 0; --rr) {
      uint64_t bit = 0;
#pragma unroll
      for (int k = 0; k < NW; ++k)
        if ((n >> 6) == k) bit = used[rr][k] >> (n & 63) & 1ull;
      if (rr < rq && bit) src = rr;
    }
    if (src < 0) continue;
    const int64_t at0 = so + ((int64_t)(n >> 2) * rpw + q * rq + src) * 4 + (n & 3);
    const int slot = a.slots ? (a.slots[at0] >> 4) : (int)(((uint32_t*)a.values)[at0] >> 20);
    if (slot <= 0) continue;
#pragma unroll
    for (int rr = 0; rr < kRqMax; ++rr) {
      uint64_t bit = 1;
#pragma unroll
      for (int k = 0; k < NW; ++k)
        if ((n >> 6) == k) bit = used[rr][k] >> (n & 63) & 1ull;
      if (rr < rq && !bit)
        write_entry(a, so + ((int64_t)(n >> 2) * rpw + q * rq + rr) * 4 + (n & 3), slot, -1,
                    scale, wmax, nunder);
    }
  }
}

// greedy_quarter for slabs wider than 256 steps (tiles in the image corners
// see a few rays per view, so one load group spans many views): the same
// first fit with the step masks in the thread's global scratch, loops not
// unrolled (keeps the common path's registers).
constexpr int kWideWords = 16;
__device__ __noinline__ void greedy_quarter_wide(const FillArgs& a, const Tile& T, int64_t tile,
                                                 int w, int q, int rq, int rpw, int width, int k0,
                                                 int k1, int gsb, int64_t so, double scale,
                                                 uint64_t* used, uint64_t* taken, double& wmax,
                                                 int64_t& nunder) {
  const Part& p = a.p;
  const int cmask = rq - 1;
  const int nw = (width + 63) >> 6;
  auto valid = [&](int k) {
    const int lo = k * 64;
    return width >= lo + 64 ? ~0ull : (width > lo ? ((1ull << (width - lo)) - 1ull) : 0ull);
  };
  for (int i = 0; i < kRqMax * kWideWords; ++i) used[i] = 0ull;
  for (int i = 0; i < 8 * kWideWords; ++i) taken[i] = 0ull;
  for (int rr = 0; rr < rq; ++rr) {
    const int rin = q * rq + rr;
    const int32_t r = p.cta_rows[tile * p.rows_per_cta + w * rpw + rin];
    if (r < 0) continue;
    const int64_t hi_j = p.indptr[r + 1];
    int64_t L = p.indptr[r], H = hi_j;
    while (L < H) {
      const int64_t M = (L + H) >> 1;
      int key, coord;
      key_coord(T.mode, p.indices[M], p.B, key, coord);
      if (key < k0) L = M + 1; else H = M;
    }
    for (int64_t j = L; j < hi_j; ++j) {
      int key, coord;
      key_coord(T.mode, p.indices[j], p.B, key, coord);
      if (key >= k1) break;
      const int slot = bit_rank(T, T.kbase[key] + coord - T.lo[key]) - gsb;
      const int c = slot & cmask;
      int n = -1;
      for (int k = 0; k < nw && n < 0; ++k) {
        const uint64_t m = ~used[rr * kWideWords + k] & ~taken[c * kWideWords + k] & valid(k);
        if (m) n = k * 64 + __ffsll((long long)m) - 1;
      }
      for (int k = 0; k < nw && n < 0; ++k) {
        const uint64_t m = ~used[rr * kWideWords + k] & valid(k);
        if (m) n = k * 64 + __ffsll((long long)m) - 1;
      }
      used[rr * kWideWords + (n >> 6)] |= 1ull << (n & 63);
      taken[c * kWideWords + (n >> 6)] |= 1ull << (n & 63);
      write_entry(a, so + ((int64_t)(n >> 2) * rpw + rin) * 4 + (n & 3), slot, j, scale, wmax,
                  nunder);
    }
  }
  for (int n = 0; n < width; ++n) {
    int src = -1;
    for (int rr = 0; rr < rq && src < 0; ++rr)
      if (used[rr * kWideWords + (n >> 6)] >> (n & 63) & 1ull) src = rr;
    if (src < 0) continue;
    const int64_t at0 = so + ((int64_t)(n >> 2) * rpw + q * rq + src) * 4 + (n & 3);
    const int slot = a.slots ? (a.slots[at0] >> 4) : (int)(((uint32_t*)a.values)[at0] >> 20);
    if (slot <= 0) continue;
    for (int rr = 0; rr < rq; ++rr)
      if (!(used[rr * kWideWords + (n >> 6)] >> (n & 63) & 1ull))
        write_entry(a, so + ((int64_t)(n >> 2) * rpw + q * rq + rr) * 4 + (n & 3), slot, -1,
                    scale, wmax, nunder);
  }
}

// ---- paired half-warp schedule (sched modes 3 and 4) ------------------------
// A warp LDS.128 costs one shared-memory wavefront per half-warp (instead of
// two) when each quarter of the half reads at most 4 distinct 16-byte
// records and the half's records sit in distinct bank quads
// (tools/smem_share_bench.cu: "pairs" 2.07 cycles vs 4.04 for 32 distinct
// records).  With one lane per row, lanes (2k, 2k+1) of a half form pair k:
// at a "merged" step both lanes read the same record -- a voxel (ray) both
// rows touch, or one row's entry while its partner idles -- and the 8 pairs
// read records of 8 distinct bank classes.  Per (group, warp, half):
//   forced_k = max(0, n_a + n_b - shared_k - W) steps where pair k must read
//   two records; F = max_k forced_k, raised by a slack of (sched_fast bits
//   8-15) % for the tightest pairs.  Steps [F, W) are merged: the pairs'
//   tokens (shared entries and singles) are edge-coloured pairs x bank
//   classes.  Steps [0, F) are scheduled per quarter (lanes x bank classes)
//   and take, per pair, only the entries the merged steps cannot hold (mode
//   4; mode 3 fills them first).  A class overflowing the merged steps moves
//   to the per-quarter steps where its lanes have room and vice versa (a
//   free merged step of the pair whose class is free); what is left takes
//   the least-conflict free step.  Colourings: the quarter schedule's
//   alternating-path colourer (Sched), or first fit (sched_fast bit 16).
// Same entries per row and slab as every other schedule (only the steps
// differ), so sums agree to rounding (native order).  Device-only: the host
// builder has no such mode and stays the oracle for modes 0-2.
constexpr int kPairW = kNcMax;
struct PairScr {
  int16_t *slot, *jo, *stp;   // [16][kPairW] per lane entry: slot, index in group span, step
  int16_t *where;             // [4096] slot -> entry of lane b (-1 between uses)
  int16_t *at;                // [16][kPairW] step -> slot read by the lane
  int16_t *ta, *tb;           // [kEMax] merged-region token -> entry of lane a / b (-1: none)
  int16_t *tu;                // [kEMax] edge -> entry being coloured
  __device__ void carve(char* q) {
    slot = (int16_t*)q; q += 16 * kPairW * 2;
    jo = (int16_t*)q; q += 16 * kPairW * 2;
    stp = (int16_t*)q; q += 16 * kPairW * 2;
    where = (int16_t*)q; q += 4096 * 2;
    at = (int16_t*)q; q += 16 * kPairW * 2;
    ta = (int16_t*)q; q += kEMax * 2;
    tb = (int16_t*)q; q += kEMax * 2;
    tu = (int16_t*)q;
  }
  __host__ __device__ static constexpr int64_t bytes() {
    return 4 * 16 * kPairW * 2 + 4096 * 2 + 3 * kEMax * 2;
  }
};

__device__ __forceinline__ uint64_t step_bits(int k, int lo, int hi) {   // bits [lo,hi) of word k
  const int a = max(lo - 64 * k, 0), b = min(hi - 64 * k, 64);
  if (b <= a) return 0ull;
  const uint64_t top = b == 64 ? ~0ull : ((1ull << b) - 1ull);
  return top & ~((1ull << a) - 1ull);
}
__device__ __forceinline__ int first_bit(const uint64_t (&m)[4]) {
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (m[k]) return k * 64 + __ffsll((long long)m[k]) - 1;
  return -1;
}

constexpr int64_t kFillScratch = Sched::bytes() + PairScr::bytes();   // per fill thread

// Proper edge colouring of ne edges (row S.eidx[e] < nrows, bank class of
// slot[ent[e]]) by the quarter schedule's alternating-path colourer with
// max(ncol, class degree) colours; edges on colours >= ncol are the
// overflow.  Returns the colour count used, -1 when it does not fit.
__device__ int colour_core(Sched& S, int ne, int nrows, int ncol, const int16_t* ent,
                           const int16_t* slot, bool greedy) {
  if (ncol < 1) return -1;
  int cnt8[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int e = 0; e < ne; ++e) ++cnt8[slot[ent[e]] & 7];
  int maxdeg = ncol;
  for (int c = 0; c < 8; ++c) maxdeg = max(maxdeg, cnt8[c]);
  if (maxdeg > kNcMax) return -1;
  S.reset(nrows, maxdeg);
  for (int e = 0; e < ne; ++e)
    if (!S.add(S.eidx[e], slot[ent[e]] & 7, greedy ? -1 : 0)) return -1;
  return maxdeg;
}
// Overflow edges (colour >= ncol; colour -2 = moved elsewhere, skipped)
// onto the free step of their row where they conflict least.  Returns the
// number of conflicting placements, -1 when a row has no free step.
__device__ int place_overflow(Sched& S, int ne, int nrows, int ncol, const int16_t* ent,
                              const int16_t* slot) {
  bool any = false;
  for (int e = 0; e < ne && !any; ++e) any = S.col[e] >= ncol;
  if (!any) return 0;
  int conflicts = 0;
  for (int i = 0; i < nrows * ncol; ++i) S.busy[i] = 0;
  for (int i = 0; i < ncol * 8; ++i) { S.ccnt[i] = 0; S.fslot[i] = -1; }
  for (int e = 0; e < ne; ++e) {
    const int c = S.col[e], cl = slot[ent[e]] & 7;
    if (c < 0 || c >= ncol) continue;
    S.busy[S.er[e] * ncol + c] = 1;
    ++S.ccnt[c * 8 + cl];
    if (S.fslot[c * 8 + cl] < 0) S.fslot[c * 8 + cl] = slot[ent[e]];
  }
  for (int e = 0; e < ne; ++e) {
    if (S.col[e] < ncol) continue;
    const int r = S.er[e], sl = slot[ent[e]], c = sl & 7;
    int best = -1, best_cost = 1 << 30;
    for (int st = 0; st < ncol; ++st) {
      if (S.busy[r * ncol + st]) continue;
      const int fs = S.fslot[st * 8 + c];
      const int cost = fs < 0 || fs == sl ? 0 : S.ccnt[st * 8 + c];
      if (cost < best_cost) { best_cost = cost; best = st; if (!cost) break; }
    }
    if (best < 0) return -1;
    if (best_cost) ++conflicts;
    S.col[e] = (int16_t)best;
    S.busy[r * ncol + best] = 1;
    ++S.ccnt[best * 8 + c];
    if (S.fslot[best * 8 + c] < 0) S.fslot[best * 8 + c] = (int16_t)sl;
  }
  return conflicts;
}

// Returns false (nothing written) when the half does not fit the paired
// schedule's limits; the caller then schedules its two quarters as usual.
__device__ bool paired_half(const FillArgs& a, const Tile& T, int64_t tile, int w, int h,
                            int rpw, int W, int k0, int k1, int gsb, int64_t so, double scale,
                            Sched& S, PairScr& P, double& wmax, int64_t& nunder,
                            int64_t& merged, int64_t& uconf, int64_t& mconf) {
  const Part& p = a.p;
  if (W > kPairW || W < 1) return false;
  int n[16];
  int64_t ja[16];
  for (int i = 0; i < 16; ++i) {
    n[i] = 0;
    ja[i] = 0;
    const int32_t r = p.cta_rows[tile * p.rows_per_cta + w * rpw + h * 16 + i];
    if (r < 0) continue;
    const int64_t hi_j = p.indptr[r + 1];
    int64_t L = p.indptr[r], H = hi_j;
    while (L < H) {
      const int64_t M = (L + H) >> 1;
      int key, coord;
      key_coord(T.mode, p.indices[M], p.B, key, coord);
      if (key < k0) L = M + 1; else H = M;
    }
    ja[i] = L;
    int cnt = 0;                          // register count (n[] lives in local memory)
    int16_t* ps = P.slot + i * kPairW;
    int16_t* pj = P.jo + i * kPairW;
    int16_t* pt = P.stp + i * kPairW;
    for (int64_t j = L; j < hi_j; ++j) {
      int key, coord;
      key_coord(T.mode, p.indices[j], p.B, key, coord);
      if (key >= k1) break;
      if (cnt >= W) return false;
      ps[cnt] = (int16_t)(bit_rank(T, T.kbase[key] + coord - T.lo[key]) - gsb);
      pj[cnt] = (int16_t)(j - L);
      pt[cnt] = -1;
      ++cnt;
    }
    n[i] = cnt;
  }
  // forced double steps per pair
  int F = 0;
  for (int k = 0; k < 8; ++k) {
    const int A = 2 * k, B = A + 1;
    for (int e = 0; e < n[B]; ++e) P.where[P.slot[B * kPairW + e]] = (int16_t)e;
    int sh = 0;
    for (int e = 0; e < n[A]; ++e) sh += P.where[P.slot[A * kPairW + e]] >= 0;
    for (int e = 0; e < n[B]; ++e) P.where[P.slot[B * kPairW + e]] = -1;
    F = max(F, n[A] + n[B] - sh - W);
  }
  // extra per-quarter steps (slack for the tightest pair): pct of F, >= 1
  const int extra_pct = (p.fast >> 8) & 0xff;
  if (F > 0 && extra_pct) F = min(W, F + max(1, (F * extra_pct + 99) / 100));
  const int M = W - F;
  const bool minimal_u = (p.fast & 0xff) == 4;
  const bool greedy = (p.fast >> 16) & 1;  // first-fit colourings (faster fill)
  // per pair: which entries take the per-quarter steps [0, F) (marked -3),
  // the rest become merged-region tokens (ta: lane a entry, tb: lane b
  // entry, global indices lane * kPairW + e, -1: that lane idles)
  int nt = 0;
  int uc[16];                             // entries per lane on the per-quarter steps
  for (int k = 0; k < 8; ++k) {
    const int A = 2 * k, B = A + 1;
    int16_t* sa = P.slot + A * kPairW;
    int16_t* sb = P.slot + B * kPairW;
    int16_t* pa = P.stp + A * kPairW;
    int16_t* pb = P.stp + B * kPairW;
    for (int e = 0; e < n[B]; ++e) P.where[sb[e]] = (int16_t)e;
    int sh = 0;
    for (int e = 0; e < n[A]; ++e)
      if (P.where[sa[e]] >= 0) { ++sh; pb[P.where[sa[e]]] = -2; }   // B's copy of a shared entry
    const int ua = n[A] - sh, ub = n[B] - sh;
    // entries moved to the per-quarter steps: singles (alternating lanes),
    // then shared pairs, until the pair's merged-region tokens fit the M
    // merged steps (minimal; a slack of M/8 measured 0.7% slower at c5) or
    // until [0, F) is full (fill)
    const int tk0 = sh + ua + ub;
    int need = minimal_u ? max(0, tk0 - M) : tk0;
    int aU = 0, bU = 0, sU = 0;
    while (need > 0) {
      const bool ca_ok = aU < ua && aU + sU < F, cb_ok = bU < ub && bU + sU < F;
      if (ca_ok && (aU <= bU || !cb_ok)) ++aU;
      else if (cb_ok) ++bU;
      else if (sU < sh && aU + sU < F && bU + sU < F) ++sU;
      else break;
      --need;
    }
    if (sU > sh || aU + sU > F || bU + sU > F) {
      for (int e = 0; e < n[B]; ++e) P.where[sb[e]] = -1;
      return false;
    }
    uc[A] = aU + sU;
    uc[B] = bU + sU;
    const int tk = sh - sU + (ua - aU) + (ub - bU);
    if (tk > M || nt + tk > kEMax) {
      for (int e = 0; e < n[B]; ++e) P.where[sb[e]] = -1;
      return false;
    }
    int ca = 0, cb = 0, cs = 0;
    for (int e = 0; e < n[A]; ++e) {
      const int eb = P.where[sa[e]];
      if (eb < 0) {
        if (ca < aU) { pa[e] = -3; ++ca; }
        else { P.ta[nt] = (int16_t)(A * kPairW + e); P.tb[nt] = -1; ++nt; }
      } else if (cs < sU) {
        pa[e] = -3; pb[eb] = -3; ++cs;
      } else {
        P.ta[nt] = (int16_t)(A * kPairW + e); P.tb[nt] = (int16_t)(B * kPairW + eb);
        ++nt;
      }
    }
    for (int e = 0; e < n[B]; ++e) {
      if (pb[e] != -1) continue;          // shared (handled with A) or already placed
      if (cb < bU) { pb[e] = -3; ++cb; }
      else { P.ta[nt] = -1; P.tb[nt] = (int16_t)(B * kPairW + e); ++nt; }
    }
    for (int e = 0; e < n[B]; ++e) P.where[sb[e]] = -1;
  }
  // steps [F, W): pairs x bank classes edge-coloured with M colours; a
  // class's overflow moves to the per-quarter steps where its lanes have
  // room, else it takes the least-conflict free step of its pair
  int conflicts = 0;
  uint64_t mpair[8 * 4], mcls[8 * 4];     // merged steps taken per pair / per bank class
  for (int i = 0; i < 32; ++i) { mpair[i] = 0ull; mcls[i] = 0ull; }
  uint64_t mvalid[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) mvalid[k] = step_bits(k, 0, M);
  if (nt > 0) {
    for (int e = 0; e < nt; ++e) {
      P.tu[e] = P.ta[e] >= 0 ? P.ta[e] : P.tb[e];
      S.eidx[e] = (int16_t)((P.tu[e] / kPairW) >> 1);
    }
    if (colour_core(S, nt, 8, M, P.tu, P.slot, greedy) < 0) return false;
    for (int e = 0; e < nt; ++e) {
      if (S.col[e] < M) continue;
      const int ea = P.ta[e], eb = P.tb[e];
      const int la = ea >= 0 ? ea / kPairW : -1, lb = eb >= 0 ? eb / kPairW : -1;
      if ((la >= 0 && uc[la] >= F) || (lb >= 0 && uc[lb] >= F)) continue;
      if (la >= 0) { P.stp[ea] = -3; ++uc[la]; }
      if (lb >= 0) { P.stp[eb] = -3; ++uc[lb]; }
      S.col[e] = -2;
    }
    conflicts = place_overflow(S, nt, 8, M, P.tu, P.slot);
    if (conflicts < 0) return false;
    for (int e = 0; e < nt; ++e) {
      if (S.col[e] < 0) continue;
      const int st = F + S.col[e];
      if (P.ta[e] >= 0) P.stp[P.ta[e]] = (int16_t)st;
      if (P.tb[e] >= 0) P.stp[P.tb[e]] = (int16_t)st;
      const int k = S.er[e], c = P.slot[P.tu[e]] & 7;
      mpair[k * 4 + (S.col[e] >> 6)] |= 1ull << (S.col[e] & 63);
      mcls[c * 4 + (S.col[e] >> 6)] |= 1ull << (S.col[e] & 63);
    }
  }
  // steps [0, F): per quarter, lanes x bank classes edge-coloured with F
  // colours (the quarter schedule restricted to those steps)
  for (int qq = 0; qq < 2; ++qq) {
    int ne = 0;
    for (int i = 8 * qq; i < 8 * qq + 8; ++i)
      for (int e = 0; e < n[i]; ++e)
        if (P.stp[i * kPairW + e] == -3) {
          if (ne >= kEMax) return false;
          P.tu[ne] = (int16_t)(i * kPairW + e);
          S.eidx[ne] = (int16_t)(i & 7);
          ++ne;
        }
    if (!ne) continue;
    if (colour_core(S, ne, 8, F, P.tu, P.slot, greedy) < 0) return false;
    // a class's overflow takes a free merged step of its pair where its
    // class is free (the partner idles there), else conflicts on [0, F)
    for (int e = 0; e < ne; ++e) {
      if (S.col[e] < F) continue;
      const int k = (P.tu[e] / kPairW) >> 1, c = P.slot[P.tu[e]] & 7;
      uint64_t m[4];
#pragma unroll
      for (int w4 = 0; w4 < 4; ++w4) m[w4] = mvalid[w4] & ~mpair[k * 4 + w4] & ~mcls[c * 4 + w4];
      const int st = first_bit(m);
      if (st < 0) continue;
      mpair[k * 4 + (st >> 6)] |= 1ull << (st & 63);
      mcls[c * 4 + (st >> 6)] |= 1ull << (st & 63);
      P.stp[P.tu[e]] = (int16_t)(F + st);
      S.col[e] = -2;
    }
    const int uc_q = place_overflow(S, ne, 8, F, P.tu, P.slot);
    if (uc_q < 0) return false;
    uconf += uc_q;
    for (int e = 0; e < ne; ++e)
      if (S.col[e] >= 0) P.stp[P.tu[e]] = S.col[e];
  }
  // every entry on its own step of its lane (else nothing is written)
  int16_t* at = P.at;                     // [16][W] step -> slot (-1 idle)
  for (int i = 0; i < 16 * W; ++i) at[i] = -1;
  for (int i = 0; i < 16; ++i)
    for (int e = 0; e < n[i]; ++e) {
      const int st = P.stp[i * kPairW + e];
      if (st < 0 || st >= W || at[i * W + st] >= 0) return false;
      at[i * W + st] = P.slot[i * kPairW + e];
    }
  // write: entries, then idle lanes re-read a record already read at that step
  for (int i = 0; i < 16; ++i)
    for (int e = 0; e < n[i]; ++e) {
      const int st = P.stp[i * kPairW + e];
      write_entry(a, so + ((int64_t)(st >> 2) * rpw + h * 16 + i) * 4 + (st & 3),
                  P.slot[i * kPairW + e], ja[i] + P.jo[i * kPairW + e], scale, wmax, nunder);
    }
  for (int st = 0; st < W; ++st) {
    int16_t v[16];
    int first_q0 = -1, first_q1 = -1;     // first record read in each quarter
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      v[i] = at[i * W + st];
      if (v[i] >= 0) {
        if (i < 8) { if (first_q0 < 0) first_q0 = v[i]; }
        else if (first_q1 < 0) first_q1 = v[i];
      }
    }
    const int first_h = first_q0 >= 0 ? first_q0 : first_q1;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (v[i] >= 0) continue;
      // merged steps: the partner's record, else any record of the half;
      // per-quarter steps: the quarter's first busy lane (broadcast)
      const int src = st >= F ? (v[i ^ 1] >= 0 ? v[i ^ 1] : first_h)
                              : (i < 8 ? first_q0 : first_q1);
      if (src > 0)
        write_entry(a, so + ((int64_t)(st >> 2) * rpw + h * 16 + i) * 4 + (st & 3), src, -1,
                    scale, wmax, nunder);
    }
  }
  merged += M - conflicts;
  mconf += conflicts;
  return true;
}

__global__ void __launch_bounds__(kFillThreads) fmtd_fill_k(FillArgs a) {
  extern __shared__ int32_t sm[];
  __shared__ uint64_t s_taken[kFillThreads][8];      // greedy masks, slabs <= 64 steps
  const Part& p = a.p;
  Tile T;
  tile_carve(p, a.bm_words, sm, T);
  Sched S;
  PairScr P;
  {
    char* base = a.scratch + (int64_t)(blockIdx.x * blockDim.x + threadIdx.x) * kFillScratch;
    S.carve(base);
    P.carve(base + Sched::bytes());
    if ((p.fast & 0xff) >= 3)
      for (int i = 0; i < 4096; ++i) P.where[i] = -1;   // kept -1 between half jobs
  }
  int64_t merged = 0, half_steps = 0, uconf = 0, mconf = 0, fallbacks = 0;
  const double scale = ldexp(1.0, a.scale_exp);
  const bool sched = p.rq > 1;
  const int rq = sched ? p.rq : 1;
  double wmax = 0.0;
  int64_t nunder = 0;
  for (int64_t tile = blockIdx.x; tile < p.n_cta; tile += gridDim.x) {
    if (!tile_setup(p, tile, a.g_lo, a.g_hi, a.bm_words, T, a.flag)) return;
    const int ng = T.ng, W = p.warps, rpw = p.rows_per_warp;
    const int64_t gb = a.tile_base[tile * 3 + 0], sb = a.tile_base[tile * 3 + 1],
                  eb = a.tile_base[tile * 3 + 2];
    for (int i = threadIdx.x; i < ng * W; i += blockDim.x)
      T.width[i] = a.g_width[tile * kGMax * W + i];
    __syncthreads();
    // slab offsets: [tile][warp][group] order
    if (threadIdx.x == 0) {
      int64_t eo = eb;
      for (int w = 0; w < W; ++w)
        for (int g = 0; g < ng; ++g) {
          a.slab_off[(gb + g) * W + w] = eo;
          a.slab_width[(gb + g) * W + w] = T.width[g * W + w];
          eo += (int64_t)T.width[g * W + w] * rpw;
        }
      __threadfence_block();
    }
    for (int g = threadIdx.x; g < ng; g += blockDim.x) a.group_map_ptr[gb + g + 1] = sb + T.gsb[g + 1];
    // group maps: every touched cell, in (key, coord) order
    const int span = T.kbase[p.n_keys];
    for (int b = threadIdx.x; b < span; b += blockDim.x) {
      if (!((unsigned)T.bm[b >> 5] >> (b & 31) & 1u)) continue;
      int lo_k = 0, hi_k = p.n_keys - 1;            // key: last kbase <= b
      while (lo_k < hi_k) {
        const int mid = (lo_k + hi_k + 1) >> 1;
        if (T.kbase[mid] <= b) lo_k = mid; else hi_k = mid - 1;
      }
      const int coord = T.lo[lo_k] + b - T.kbase[lo_k];
      a.group_map[sb + bit_rank(T, b)] = col_of(T.mode, lo_k, coord, p.B);
    }
    __syncthreads();
    // paired half-warp schedule: one (group, warp, half) job per thread
    if ((p.fast & 0xff) >= 3 && rq == 8 && rpw % 16 == 0) {
      const int nh = rpw / 16;
      const int64_t hjobs = (int64_t)ng * W * nh;
      for (int64_t job = threadIdx.x; job < hjobs; job += blockDim.x) {
        const int h = (int)(job % nh);
        const int w = (int)((job / nh) % W);
        const int g = (int)(job / ((int64_t)nh * W));
        const int width = T.width[g * W + w];
        const int64_t so = a.slab_off[(gb + g) * W + w];
        if (paired_half(a, T, tile, w, h, rpw, width, T.gk[g], T.gk[g + 1], T.gsb[g], so, scale,
                        S, P, wmax, nunder, merged, uconf, mconf)) {
          half_steps += width;
          continue;
        }
        ++fallbacks;
        for (int q = 2 * h; q < 2 * h + 2; ++q) {
          bool ok = true;
          if (width <= 64)
            greedy_quarter<1>(a, T, tile, w, q, rq, rpw, width, T.gk[g], T.gk[g + 1], T.gsb[g],
                              so, scale, s_taken[threadIdx.x], wmax, nunder);
          else if (width <= 256)
            greedy_quarter<4>(a, T, tile, w, q, rq, rpw, width, T.gk[g], T.gk[g + 1], T.gsb[g],
                              so, scale, reinterpret_cast<uint64_t*>(S.atR), wmax, nunder);
          else if (width <= 64 * kWideWords) {
            uint64_t* scr = reinterpret_cast<uint64_t*>(S.atL);
            greedy_quarter_wide(a, T, tile, w, q, rq, rpw, width, T.gk[g], T.gk[g + 1],
                                T.gsb[g], so, scale, scr, scr + kRqMax * kWideWords, wmax,
                                nunder);
          } else {
            ok = false;
          }
          if (!ok) atomicOr(a.flag, FLAG_SCHED);
        }
        half_steps += width;
      }
      __syncthreads();
      continue;
    }
    // slabs: one (group, warp, quarter) job per thread at a time
    const int nq = rpw / rq;
    const int64_t jobs = (int64_t)ng * W * nq;
    for (int64_t job = threadIdx.x; job < jobs; job += blockDim.x) {
      const int q = (int)(job % nq);
      const int w = (int)((job / nq) % W);
      const int g = (int)(job / ((int64_t)nq * W));
      const int width = T.width[g * W + w];
      const int64_t so = a.slab_off[(gb + g) * W + w];
      const int k0 = T.gk[g], k1 = T.gk[g + 1];
      const int gsb = T.gsb[g];
      int ja_of[kRqMax];
      int ne = 0;
      bool over = false;
      // fast schedules: first fit over step masks (p.fast == 2 always; with
      // p.fast == 1 only where the exact schedule does not fit its limits)
      auto greedy = [&]() -> bool {
        if (width <= 64) {
          greedy_quarter<1>(a, T, tile, w, q, rq, rpw, width, k0, k1, gsb, so, scale,
                            s_taken[threadIdx.x], wmax, nunder);
        } else if (width <= 256) {
          greedy_quarter<4>(a, T, tile, w, q, rq, rpw, width, k0, k1, gsb, so, scale,
                            reinterpret_cast<uint64_t*>(S.atR), wmax, nunder);
        } else if (width <= 64 * kWideWords) {          // image-corner tiles, rare
          uint64_t* scr = reinterpret_cast<uint64_t*>(S.atL);     // this thread's scratch
          greedy_quarter_wide(a, T, tile, w, q, rq, rpw, width, k0, k1, gsb, so, scale, scr,
                              scr + kRqMax * kWideWords, wmax, nunder);
        } else {
          return false;
        }
        return true;
      };
      if (sched && (p.fast == 2 || (p.fast == 1 && width > kNcMax))) {
        if (!greedy()) atomicOr(a.flag, FLAG_SCHED);
        continue;
      }
      // edges: rows of the quarter in order, each row's group span in order
      for (int rr = 0; rr < rq; ++rr) {
        const int rin = q * rq + rr;
        const int32_t r = p.cta_rows[tile * p.rows_per_cta + w * rpw + rin];
        ja_of[rr] = 0;
        if (r < 0) continue;
        int64_t lo_j = p.indptr[r], hi_j = p.indptr[r + 1];
        // first entry with key >= k0, first with key >= k1 (keys sorted)
        auto first_ge = [&](int kk) {
          int64_t L = lo_j, H = hi_j;
          while (L < H) {
            const int64_t M = (L + H) >> 1;
            int key, coord;
            key_coord(T.mode, p.indices[M], p.B, key, coord);
            if (key < kk) L = M + 1; else H = M;
          }
          return L;
        };
        const int64_t ja = first_ge(k0), jb = first_ge(k1);
        ja_of[rr] = (int)(ja - p.indptr[r]);
        if (!sched) {
          for (int64_t j = ja; j < jb; ++j) {
            int key, coord;
            key_coord(T.mode, p.indices[j], p.B, key, coord);
            const int slot = bit_rank(T, T.kbase[key] + coord - T.lo[key]) - gsb;
            const int n = (int)(j - ja);
            write_entry(a, so + ((int64_t)(n >> 2) * rpw + rin) * 4 + (n & 3), slot, j, scale,
                        wmax, nunder);
          }
          continue;
        }
        for (int64_t j = ja; j < jb; ++j) {
          if (ne >= kEMax) { over = true; break; }
          int key, coord;
          key_coord(T.mode, p.indices[j], p.B, key, coord);
          S.er[ne] = (uint8_t)rr;
          S.eslot[ne] = (int16_t)(bit_rank(T, T.kbase[key] + coord - T.lo[key]) - gsb);
          S.eidx[ne] = (int16_t)(j - ja);
          ++ne;
        }
      }
      if (!sched) continue;
      // QuarterScheduler::run (compress on)
      int cnt8[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      const int cmask = rq - 1;
      for (int e = 0; e < ne; ++e) ++cnt8[S.eslot[e] & cmask];
      int maxdeg = width;
      for (int c = 0; c < 8; ++c) maxdeg = max(maxdeg, cnt8[c]);
      if (over || maxdeg > kNcMax || width > kNcMax) {
        if (!(p.fast && greedy())) atomicOr(a.flag, FLAG_SCHED);
        continue;
      }
      S.reset(rq, maxdeg);
      bool okc = true;
      for (int e = 0; e < ne && okc; ++e) {
        const int rr = S.er[e];
        okc = S.add(rr, S.eslot[e] & cmask);
      }
      if (!okc) {
        if (!(p.fast && greedy())) atomicOr(a.flag, FLAG_SCHED);
        continue;
      }
      if (maxdeg != width) {
        for (int i = 0; i < rq * width; ++i) S.busy[i] = 0;
        for (int i = 0; i < width * 8; ++i) { S.ccnt[i] = 0; S.fslot[i] = -1; }
        for (int e = 0; e < ne; ++e) {
          const int n = S.col[e];
          if (n >= width) continue;
          S.busy[S.er[e] * width + n] = 1;
          const int c = S.eslot[e] & cmask;
          ++S.ccnt[n * 8 + c];
          if (S.fslot[n * 8 + c] < 0) S.fslot[n * 8 + c] = S.eslot[e];
        }
        for (int e = 0; e < ne; ++e) {
          if (S.col[e] < width) continue;
          const int r = S.er[e], slot = S.eslot[e], c = slot & cmask;
          int best = -1, best_cost = 1 << 30;
          for (int n = 0; n < width; ++n) {
            if (S.busy[r * width + n]) continue;
            const int fs = S.fslot[n * 8 + c];
            const int cost = fs < 0 || fs == slot ? 0 : S.ccnt[n * 8 + c];
            if (cost < best_cost) { best_cost = cost; best = n; if (!cost) break; }
          }
          if (best < 0) { okc = false; break; }
          S.col[e] = (int16_t)best;
          S.busy[r * width + best] = 1;
          ++S.ccnt[best * 8 + c];
          if (S.fslot[best * 8 + c] < 0) S.fslot[best * 8 + c] = (int16_t)slot;
        }
        if (!okc) {
          if (!(p.fast && greedy())) atomicOr(a.flag, FLAG_SCHED);
          continue;
        }
      }
      for (int n = 0; n < width; ++n) S.sslot[n] = -1;
      for (int i = 0; i < rq * width; ++i) S.used[i] = 0;
      for (int e = 0; e < ne; ++e) {
        const int rr = S.er[e], n = S.col[e], rin = q * rq + rr;
        const int32_t r = p.cta_rows[tile * p.rows_per_cta + w * rpw + rin];
        const int64_t j = p.indptr[r] + ja_of[rr] + S.eidx[e];
        write_entry(a, so + ((int64_t)(n >> 2) * rpw + rin) * 4 + (n & 3), S.eslot[e], j, scale,
                    wmax, nunder);
        S.used[rr * width + n] = 1;
        if (S.sslot[n] < 0) S.sslot[n] = S.eslot[e];
      }
      // idle lanes re-read a slot another lane of the quarter reads (broadcast)
      for (int rr = 0; rr < rq; ++rr)
        for (int n = 0; n < width; ++n)
          if (!S.used[rr * width + n] && S.sslot[n] > 0)
            write_entry(a, so + ((int64_t)(n >> 2) * rpw + q * rq + rr) * 4 + (n & 3),
                        S.sslot[n], -1, scale, wmax, nunder);
    }
    __syncthreads();
  }
  if (wmax > 0.0) atomicMax(&a.qstats[0], (unsigned long long)__double_as_longlong(wmax));
  if (nunder) atomicAdd(&a.qstats[1], (unsigned long long)nunder);
  if (half_steps) {
    atomicAdd(&a.qstats[2], (unsigned long long)merged);
    atomicAdd(&a.qstats[3], (unsigned long long)half_steps);
    atomicAdd(&a.qstats[4], (unsigned long long)uconf);
    atomicAdd(&a.qstats[5], (unsigned long long)mconf);
    atomicAdd(&a.qstats[6], (unsigned long long)fallbacks);
  }
}

int smem_ints(const Part& p, int bm_words) {
  return 4 * p.n_keys + 1 + 2 * (kGMax + 1) + kGMax * p.warps + 2 * bm_words + 1 + 4;
}

int make_part(const xct_fmtd_part* in, Part& p) {
  if (!in || !in->d_indptr || !in->d_cta_rows || !in->d_cta_mode)
    return xct::fail(XCT_EINVAL, "fmtd: null argument");
  if (in->rows_per_cta < 1 || in->rows_per_warp < 1 || in->rows_per_cta % in->rows_per_warp ||
      in->base_b < 1 || in->n_keys < 1 || in->capacity < 1 || in->capacity > 4096)
    return xct::fail(XCT_EINVAL, "fmtd: bad shape arguments");
  if (in->sched_rq > 1 && (in->sched_rq > kRqMax || in->rows_per_warp % in->sched_rq))
    return xct::fail(XCT_EINVAL, "fmtd: bank model rows per quarter must divide rows_per_warp");
  p.indptr = in->d_indptr;
  p.indices = in->d_indices;
  p.values = in->d_values;
  p.n_rows = in->n_rows;
  p.cta_rows = in->d_cta_rows;
  p.cta_mode = in->d_cta_mode;
  p.n_cta = in->n_cta;
  p.rows_per_cta = (int32_t)in->rows_per_cta;
  p.rows_per_warp = (int32_t)in->rows_per_warp;
  p.warps = (int32_t)(in->rows_per_cta / in->rows_per_warp);
  p.B = in->base_b;
  p.n_keys = in->n_keys;
  p.capacity = in->capacity;
  p.rq = in->sched_rq;
  p.fast = in->sched_fast;
  return XCT_OK;
}

}  // namespace

extern "C" int64_t xct_fmtd_scratch_bytes(void) {
  return (int64_t)148 * 2 * kFillThreads * kFillScratch;
}

extern "C" int xct_fmtd_ranges(const xct_fmtd_part* in, int32_t* d_lo, int32_t* d_hi,
                               int64_t* d_span, int32_t* d_flag, void* stream) {
  Part p;
  int st = make_part(in, p);
  if (st) return st;
  if (p.n_cta == 0) return XCT_OK;
  const size_t smem = (size_t)2 * p.n_keys * 4;
  if (smem > 200 * 1024) return xct::fail(XCT_EINVAL, "fmtd_ranges: too many keys");
  cudaFuncSetAttribute(fmtd_ranges_k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  fmtd_ranges_k<<<(unsigned)p.n_cta, 512, smem, (cudaStream_t)stream>>>(p, d_lo, d_hi, d_span, d_flag);
  XCT_CUDA_CHECK_LAUNCH("fmtd_ranges");
  return XCT_OK;
}

extern "C" int xct_fmtd_count(const xct_fmtd_part* in, const int32_t* d_lo, const int32_t* d_hi,
                              int32_t bm_words, int64_t* d_counts, int32_t* d_widths,
                              int32_t* d_flag, void* stream) {
  Part p;
  int st = make_part(in, p);
  if (st) return st;
  if (p.n_cta == 0) return XCT_OK;
  const int threads = 512;
  const size_t smem = (size_t)(smem_ints(p, bm_words) + (threads / 32) * kGMax) * 4;
  if (smem > 227 * 1024) return xct::fail(XCT_ESTAGE, "fmtd_count: tile footprint exceeds shared memory");
  cudaFuncSetAttribute(fmtd_count_k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  fmtd_count_k<<<(unsigned)p.n_cta, threads, smem, (cudaStream_t)stream>>>(p, d_lo, d_hi, bm_words,
                                                                          d_counts, d_widths, d_flag);
  XCT_CUDA_CHECK_LAUNCH("fmtd_count");
  return XCT_OK;
}

extern "C" int xct_fmtd_fill(const xct_fmtd_part* in, const int32_t* d_lo, const int32_t* d_hi,
                             int32_t bm_words, const int32_t* d_widths, const int64_t* d_tile_base,
                             int precision, int value_scale_exp, int32_t* d_group_map,
                             int64_t* d_group_map_ptr, int64_t* d_slab_off, int32_t* d_slab_width,
                             uint16_t* d_slots, void* d_values, void* d_scratch,
                             int64_t scratch_bytes, int32_t* d_flag, uint64_t* d_qstats,
                             void* stream) {
  Part p;
  int st = make_part(in, p);
  if (st) return st;
  if (p.n_cta == 0) return XCT_OK;
  if (precision < 0 || precision > 3) return xct::fail(XCT_EINVAL, "fmtd_fill: bad precision");
  const bool packed = precision == XCT_HALF || precision == XCT_MIXED;
  if (!d_values || (!packed && !d_slots) || !d_scratch)
    return xct::fail(XCT_EINVAL, "fmtd_fill: missing output arrays");
  const int64_t grid = std::min<int64_t>(p.n_cta, 148 * 2);
  if (scratch_bytes < grid * kFillThreads * kFillScratch)
    return xct::fail(XCT_EINVAL, "fmtd_fill: scratch too small");
  const size_t smem = (size_t)smem_ints(p, bm_words) * 4;
  if (smem > 227 * 1024) return xct::fail(XCT_ESTAGE, "fmtd_fill: tile footprint exceeds shared memory");
  cudaFuncSetAttribute(fmtd_fill_k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  FillArgs a;
  a.p = p;
  a.g_lo = d_lo;
  a.g_hi = d_hi;
  a.bm_words = bm_words;
  a.g_width = d_widths;
  a.tile_base = d_tile_base;
  a.precision = precision;
  a.scale_exp = value_scale_exp;
  a.group_map = d_group_map;
  a.group_map_ptr = d_group_map_ptr;
  a.slab_off = d_slab_off;
  a.slab_width = d_slab_width;
  a.slots = d_slots;
  a.values = d_values;
  a.scratch = (char*)d_scratch;
  a.flag = d_flag;
  a.qstats = (unsigned long long*)d_qstats;
  fmtd_fill_k<<<(unsigned)grid, kFillThreads, smem, (cudaStream_t)stream>>>(a);
  XCT_CUDA_CHECK_LAUNCH("fmtd_fill");
  return XCT_OK;
}

// ---------------------------------------------------------------------------
// K4 on the device: the transposed operator A^T for a band of columns
// (voxels), rows ordered by ray id -- matrixstore.transpose
// (src/matrixstore.py:189-201, a stable argsort by column).  The rays are
// regenerated chunk by chunk (K2); each chunk's entries of the band are
// scattered to their voxel's row with an atomic cursor, then every voxel
// sorts the segment it received from the chunk by ray id, so each row is
// the concatenation of sorted per-chunk segments in ascending ray order.
namespace {
__global__ void csr_col_counts_k(const int64_t* __restrict__ indptr,
                                 const int32_t* __restrict__ indices, int64_t n_rows,
                                 int32_t lo, int32_t hi, int64_t* __restrict__ counts) {
  const int64_t n = indptr[n_rows] - indptr[0];
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int32_t c = indices[indptr[0] + j];
    if (c >= lo && c < hi) atomicAdd((unsigned long long*)&counts[c - lo], 1ull);
  }
}

__global__ void csr_scatter_cols_k(const int64_t* __restrict__ indptr,
                                   const int32_t* __restrict__ indices,
                                   const double* __restrict__ values, int64_t r0, int64_t r1,
                                   int64_t row_base, int32_t lo, int32_t hi,
                                   const int64_t* __restrict__ t_indptr, int32_t* cursor,
                                   int32_t* __restrict__ out_rows, double* __restrict__ out_vals) {
  for (int64_t r = r0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < r1;
       r += (int64_t)gridDim.x * blockDim.x) {
    for (int64_t j = indptr[r]; j < indptr[r + 1]; ++j) {
      const int32_t c = indices[j];
      if (c < lo || c >= hi) continue;
      const int32_t v = c - lo;
      const int64_t at = t_indptr[v] + atomicAdd(&cursor[v], 1);
      out_rows[at] = (int32_t)(row_base + r);
      out_vals[at] = values[j];
    }
  }
}

__global__ void csr_sort_segments_k(const int64_t* __restrict__ t_indptr, int32_t* prev,
                                    const int32_t* __restrict__ cursor, int64_t n,
                                    int32_t* __restrict__ rows, double* __restrict__ vals) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = t_indptr[v] + prev[v], e = t_indptr[v] + cursor[v];
    for (int64_t i = a + 1; i < e; ++i) {            // insertion sort by ray id
      const int32_t key = rows[i];
      const double val = vals[i];
      int64_t k = i - 1;
      while (k >= a && rows[k] > key) {
        rows[k + 1] = rows[k];
        vals[k + 1] = vals[k];
        --k;
      }
      rows[k + 1] = key;
      vals[k + 1] = val;
    }
    prev[v] = cursor[v];
  }
}

int grid_of(int64_t n, int block) {
  int64_t b = (n + block - 1) / block;
  if (b > 148 * 32) b = 148 * 32;
  return (int)(b < 1 ? 1 : b);
}
}  // namespace

extern "C" int xct_csr_col_counts(const int64_t* d_indptr, const int32_t* d_indices, int64_t n_rows,
                                  int32_t col_lo, int32_t col_hi, int64_t* d_counts, void* stream) {
  if (!d_indptr || !d_counts || col_hi < col_lo || n_rows < 0)
    return xct::fail(XCT_EINVAL, "csr_col_counts: bad argument");
  if (n_rows == 0) return XCT_OK;
  csr_col_counts_k<<<148 * 16, 256, 0, (cudaStream_t)stream>>>(d_indptr, d_indices, n_rows, col_lo,
                                                               col_hi, d_counts);
  XCT_CUDA_CHECK_LAUNCH("csr_col_counts");
  return XCT_OK;
}

extern "C" int xct_csr_transpose_band(const int64_t* d_indptr, const int32_t* d_indices,
                                      const double* d_values, int64_t n_rows, int64_t row_base,
                                      int64_t rows_per_pass, int32_t col_lo, int32_t col_hi,
                                      const int64_t* d_t_indptr, int32_t* d_cursor,
                                      int32_t* d_prev, int32_t* d_t_rows, double* d_t_vals,
                                      void* stream) {
  if (!d_indptr || !d_t_indptr || !d_cursor || !d_prev || !d_t_rows || !d_t_vals ||
      col_hi < col_lo || n_rows < 0 || rows_per_pass < 1)
    return xct::fail(XCT_EINVAL, "csr_transpose_band: bad argument");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t nb = col_hi - col_lo;
  for (int64_t r0 = 0; r0 < n_rows; r0 += rows_per_pass) {
    const int64_t r1 = std::min(n_rows, r0 + rows_per_pass);
    csr_scatter_cols_k<<<grid_of(r1 - r0, 128), 128, 0, s>>>(
        d_indptr, d_indices, d_values, r0, r1, row_base, col_lo, col_hi, d_t_indptr, d_cursor,
        d_t_rows, d_t_vals);
    csr_sort_segments_k<<<grid_of(nb, 256), 256, 0, s>>>(d_t_indptr, d_prev, d_cursor, nb,
                                                         d_t_rows, d_t_vals);
  }
  XCT_CUDA_CHECK_LAUNCH("csr_transpose_band");
  return XCT_OK;
}
