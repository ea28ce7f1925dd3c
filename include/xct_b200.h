/*
 * xct_b200 -- C ABI of the B200-native XCT hot path (libxct_b200.so).
 *
 * Drop-in boundary for the reference package's operator API
 * (/root/reference/pkg/src/xct).  The reference is pure Python and has no
 * FFI; each entry point below replaces one reference function on the hot
 * path (cited as src/<file>:<line>) and is bound from Python with ctypes
 * (paper_2009_07226_b200/_lib.py; INTEGRATION.md shows the binding).
 *
 * Conventions
 *   - every function returns an int status: XCT_OK (0) or an error code;
 *     xct_last_error() gives a message (thread-local);
 *   - "d_" pointers are device pointers owned by the caller; "h_" pointers
 *     are host pointers; nothing is allocated behind the caller's back
 *     except inside an xct_format handle (host memory);
 *   - all device work is stream-ordered on the given cudaStream_t (passed
 *     as void*; NULL = legacy default stream) and asynchronous;
 *   - precision codes follow src/matrixstore.py:41:
 *       0 double, 1 single, 2 half, 3 mixed (fp16 storage, fp32 compute).
 */
#ifndef XCT_B200_H
#define XCT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  XCT_OK = 0,
  XCT_EINVAL = 1,        /* ValueError in the reference                   */
  XCT_ECUDA = 2,         /* CUDA runtime failure                          */
  XCT_ESTAGE = 3,        /* StageSplitRequired (src/matrixstore.py:54-55) */
  XCT_ENOMEM = 4,
  XCT_ENONFINITE = 5     /* non-finite data (src/matrixstore.py:298-299)  */
};

enum { XCT_DOUBLE = 0, XCT_SINGLE = 1, XCT_HALF = 2, XCT_MIXED = 3 };

int xct_abi_version(void);
const char* xct_last_error(void);

/* ---------------------------------------------------------------------------
 * K1/K2  Siddon system-matrix construction
 * replaces geometry.trace_ray (src/geometry.py:117-164) and the row loop of
 * geometry.build_system_matrix (src/geometry.py:202-232).
 * Rays r = k*n_det + c for k in [k0, k1); d_cos/d_sin hold cos/sin of every
 * view angle (computed on the host exactly as make_geometry does,
 * src/geometry.py:84-85,112).  Results are bit-identical to the reference
 * in float64 (no FMA contraction).
 * ------------------------------------------------------------------------- */
int xct_siddon_count(const double* d_cos, const double* d_sin, int k0, int k1,
                     int n_det, int grid_n, double voxel_size,
                     int64_t* d_counts /* [(k1-k0)*n_det] */, void* stream);

int xct_siddon_fill(const double* d_cos, const double* d_sin, int k0, int k1,
                    int n_det, int grid_n, double voxel_size,
                    const int64_t* d_rowptr /* [(k1-k0)*n_det+1], relative */,
                    int32_t* d_indices, double* d_values, void* stream);

/* K11  matrix-free FP32 projector over one chunk of 16 slices: rays
 * [k0*n_det, k1*n_det) traced on the fly (same Siddon as K1/K2), lengths
 * rounded to f32, f32 accumulation.  adjoint == 0: d_out[r][16] =
 * sum_j len_j * d_in[vox_j][16] (rays relative to k0); adjoint != 0:
 * d_out[vox][16] += len * d_in[r][16] with f32 atomics (caller zeroes
 * d_out).  An independent single-precision operator (cf. engine.project in
 * "single" mode, src/engine.py:119-166) for checking the staged path. */
int xct_siddon_project_f32(const double* d_cos, const double* d_sin, int k0, int k1,
                           int n_det, int grid_n, double voxel_size, int adjoint,
                           const float* d_in, float* d_out, void* stream);

/* Column-range restriction of a device CSR for the streamed operator build
 * (the back-projection format is built one band of voxels at a time; cf.
 * matrixstore._restrict_rows, src/matrixstore.py:151-165).  Count pass when
 * d_counts != NULL (entries per row with col in [col_lo, col_hi)), else fill
 * pass into d_out_ptr/d_out_idx (col - col_lo)/d_out_val, order preserved. */
int xct_csr_filter_cols(const int64_t* d_indptr, const int32_t* d_indices,
                        const double* d_values, int64_t n_rows, int32_t col_lo,
                        int32_t col_hi, int64_t* d_counts, const int64_t* d_out_ptr,
                        int32_t* d_out_idx, double* d_out_val, void* stream);

/* Row/column-mapped restriction (per-rank blocks of the data-partitioned
 * operator, built streamed; cf. src/matrixstore.py:130-165): entry j of row
 * r is kept when d_row_keep[r] != 0 (or d_row_keep == NULL) and
 * d_col_map[col] >= 0, and its column becomes d_col_map[col].  Count pass
 * when d_counts != NULL, else fill pass; order preserved. */
int xct_csr_filter_map(const int64_t* d_indptr, const int32_t* d_indices,
                       const double* d_values, int64_t n_rows, const uint8_t* d_row_keep,
                       const int32_t* d_col_map, int64_t* d_counts, const int64_t* d_out_ptr,
                       int32_t* d_out_idx, double* d_out_val, void* stream);

/* ---------------------------------------------------------------------------
 * K5  staged execution format (host builder)
 * replaces matrixstore.build_staged / pack (src/matrixstore.py:250-262,
 * :417-562).  Rows of a CSR block are assigned to thread blocks ("CTA
 * tiles", rows_per_cta rows each, -1 = empty lane).  Each entry gets a key
 * key_tables[cta_table[cta]*n_cols + col]; a CTA's column footprint is
 * ordered by (key, col) and cut into load groups of whole keys holding at
 * most `capacity` elements (shared-memory slots).  A row's entries are
 * accumulated group by group, in (key, CSR position) order inside a group.
 * Per (group, warp) the entries of the warp's rows are stored as a
 * zero-padded slab [width/4][rows_per_warp][4] of (uint16 slot, value).
 * sched_log2_pieces >= 0 enables bank-conflict-free scheduling for a kernel
 * whose records are 2^sched_log2_pieces 16-byte pieces read by
 * 2^sched_log2_lanes lanes per row: within each (group, warp, quarter-warp)
 * the entries are placed on slab steps by a proper edge colouring of the
 * rows x shared-memory-bank-class multigraph, so no two rows of a quarter
 * read the same bank quads in one step (row order is then not traversal
 * order; sums agree to rounding).  -1 keeps (key, CSR position) order.
 * ------------------------------------------------------------------------- */
typedef struct xct_format xct_format;

typedef struct {
  int64_t n_cta, rows_per_cta, rows_per_warp, warps_per_cta;
  int64_t n_groups, n_slots, n_padded, nnz;
  int64_t max_group_slots;
  int32_t value_bytes;
  double max_rel_quant_error;     /* PackReport.max_rel_error            */
  int64_t underflow_count;        /* PackReport.underflow_count          */
  int32_t row_group;              /* values per slab position (G rows)   */
} xct_format_info;

int xct_format_build(int64_t n_rows, int64_t n_cols,
                     const int64_t* h_indptr, const int32_t* h_indices,
                     const double* h_values,
                     int64_t n_cta, int64_t rows_per_cta, int64_t rows_per_warp,
                     const int32_t* h_cta_rows,
                     const int32_t* h_key_tables, const int32_t* h_cta_table,
                     int64_t capacity, int precision, int value_scale_exp,
                     int sched_log2_pieces, int sched_log2_lanes,
                     int row_group, int n_threads, xct_format** out);
int xct_format_get_info(const xct_format* f, xct_format_info* info);
/* copies the format arrays into caller-provided host buffers sized from
 * xct_format_get_info; any pointer may be NULL to skip that array. */
int xct_format_export(const xct_format* f,
                      int32_t* h_cta_group_ptr /* [n_cta+1] */,
                      int64_t* h_group_map_ptr /* [n_groups+1] */,
                      int32_t* h_group_map /* [n_slots] */,
                      int64_t* h_slab_off /* [n_groups*warps_per_cta] */,
                      int32_t* h_slab_width /* [n_groups*warps_per_cta] */,
                      uint16_t* h_slots /* [n_padded] */,
                      void* h_values /* [n_padded*row_group] of value_bytes */);
void xct_format_free(xct_format* f);

/* K5 on the device (row_group 1; staging keys that are a function of the
 * column: image bands of A, view angles of A^T -- matrixstore.forward_plan
 * / adjoint_plan).  Produces the same arrays as xct_format_build +
 * upload (same footprints, groups, bank schedule and slab bytes), written
 * straight into device memory.  Three passes per part of the operator
 * (a chunk of views / a band of voxels):
 *   ranges: lo/hi coordinate per (tile, key) [n_cta * n_keys], footprint
 *           span per tile (bits of the tile's touched-cell bitmap);
 *   count:  per tile {n_groups, n_slots, max_group_slots, n_padded}
 *           [n_cta * 4] and slab widths [n_cta * 256 * warps];
 *   fill:   group maps, group_map_ptr[g+1], slab offsets/widths and the
 *           slabs (packed slot<<20|fp16 words for half/mixed, slot<<4 +
 *           f32/f64 values otherwise; slab arrays zeroed by the caller),
 *           from per-tile bases {group, slot, entry} [n_cta * 3].
 * d_flag (zeroed by the caller) collects reasons to fall back to the host
 * builder: 1 row not key-sorted, 2 key above capacity, 4 > 256 groups per
 * tile, 8 footprint above bm_words*32 bits, 16 schedule beyond its limits. */
typedef struct {
  const int64_t* d_indptr;     /* [n_rows+1], entry 0 of the part at 0     */
  const int32_t* d_indices;    /* global column ids                        */
  const double* d_values;
  int64_t n_rows;
  const int32_t* d_cta_rows;   /* [n_cta*rows_per_cta] part-local rows, -1 */
  const int32_t* d_cta_mode;   /* [n_cta] 0: key=col/B, coord=col%B;
                                  1: key=col%B, coord=col/B;
                                  2: key=B-1-col%B, coord=col/B            */
  int64_t n_cta, rows_per_cta, rows_per_warp;
  int32_t base_b, n_keys, capacity;
  int32_t sched_rq;            /* rows per quarter-warp of the bank model
                                  (8 >> log2 lanes per row); <= 1: no
                                  schedule, (key, CSR position) order      */
  int32_t sched_fast;          /* 0: the host's schedule exactly (edge
                                  colouring by alternating paths, one thread
                                  per quarter-warp); 1: that, and first fit
                                  over step masks where a slab exceeds its
                                  limits (> 256 steps); 2: first fit
                                  everywhere (same entries per row and slab,
                                  other step placement); 3: paired half-
                                  warp schedule where sched_rq == 8 (lanes
                                  2k, 2k+1 read one record at merged steps:
                                  one LDS wavefront per half-warp), first
                                  fit per quarter elsewhere (bits 8-15:
                                  slack steps in % of F; bit 16: first-
                                  fit colourings); d_qstats[2..3]
                                  = merged / scheduled half-warp steps,
                                  [4..5] = conflicting placements on the
                                  per-quarter / merged steps, [6] = half-
                                  warps that fell back to the quarter
                                  schedule                               */
} xct_fmtd_part;

int64_t xct_fmtd_scratch_bytes(void);
int xct_fmtd_ranges(const xct_fmtd_part* part, int32_t* d_lo, int32_t* d_hi, int64_t* d_span,
                    int32_t* d_flag, void* stream);
int xct_fmtd_count(const xct_fmtd_part* part, const int32_t* d_lo, const int32_t* d_hi,
                   int32_t bm_words, int64_t* d_counts, int32_t* d_widths, int32_t* d_flag,
                   void* stream);
int xct_fmtd_fill(const xct_fmtd_part* part, const int32_t* d_lo, const int32_t* d_hi,
                  int32_t bm_words, const int32_t* d_widths, const int64_t* d_tile_base,
                  int precision, int value_scale_exp, int32_t* d_group_map,
                  int64_t* d_group_map_ptr, int64_t* d_slab_off, int32_t* d_slab_width,
                  uint16_t* d_slots, void* d_values, void* d_scratch, int64_t scratch_bytes,
                  int32_t* d_flag, uint64_t* d_qstats, void* stream);

/* K4 on the device: entries per column in [col_lo, col_hi) of a device CSR
 * (atomic adds into d_counts, zeroed by the caller) and the band transpose:
 * rows [0, n_rows) of the CSR (global row id row_base + r), in passes of
 * rows_per_pass rows, scattered into the rows of A^T for columns
 * [col_lo, col_hi) at d_t_indptr[v] + cursor[v] and each pass's segment
 * of every row sorted by row id -- so calling it for consecutive CSR chunks
 * in ascending row order yields rows in ascending row id, exactly
 * xct_csr_transpose / src/matrixstore.py:189-201 (d_cursor, d_prev zeroed
 * per band by the caller). */
int xct_csr_col_counts(const int64_t* d_indptr, const int32_t* d_indices, int64_t n_rows,
                       int32_t col_lo, int32_t col_hi, int64_t* d_counts, void* stream);
int xct_csr_transpose_band(const int64_t* d_indptr, const int32_t* d_indices,
                           const double* d_values, int64_t n_rows, int64_t row_base,
                           int64_t rows_per_pass, int32_t col_lo, int32_t col_hi,
                           const int64_t* d_t_indptr, int32_t* d_cursor, int32_t* d_prev,
                           int32_t* d_t_rows, double* d_t_vals, void* stream);

/* stable counting transpose of a CSR block (src/matrixstore.py:189-201);
 * h_t_indptr [n_cols+1], h_t_indices/h_t_values [nnz]. */
int xct_csr_transpose(int64_t n_rows, int64_t n_cols, const int64_t* h_indptr,
                      const int32_t* h_indices, const double* h_values,
                      int64_t* h_t_indptr, int32_t* h_t_indices, double* h_t_values,
                      int n_threads);

/* ---------------------------------------------------------------------------
 * K6  staged SpMM (forward projection A.X and back projection A^T.Y)
 * replaces engine.project / backproject / _apply_exec
 * (src/engine.py:119-166) fused with the output scaling and cast
 * (src/engine.py:137-139), the partial-result upcast (src/comm.py:432) and
 * denormalize (src/matrixstore.py:308-316).
 * X is chunked slice-minor: [n_chunks][n_in][f_dev] at the storage dtype.
 * ------------------------------------------------------------------------- */
typedef struct {
  int64_t n_cta, rows_per_cta, warps_per_cta, rows_per_warp, n_groups;
  const int32_t* d_cta_rows;        /* [n_cta*rows_per_cta], -1 = empty  */
  const int32_t* d_cta_group_ptr;   /* [n_cta+1]                         */
  const int64_t* d_group_map_ptr;   /* [n_groups+1]                      */
  const int32_t* d_group_map;       /* [n_slots]: slot -> input element  */
  const int64_t* d_slab_off;        /* [n_groups*warps_per_cta]          */
  const int32_t* d_slab_width;      /* [n_groups*warps_per_cta]          */
  const uint16_t* d_slots;          /* [n_padded]                        */
  const void* d_values;             /* [n_padded] storage dtype          */
  int64_t max_group_slots;
  int32_t contract;    /* single only: FFMA (one rounding) instead of the
                          reference's multiply-then-add; native order only */
  int32_t chunk_group; /* F-chunks of a tile launched adjacently (their CTAs
                          share the tile's entry stream through L2); the
                          largest power of two <= this dividing n_chunks */
  int32_t row_group;   /* rows per unit of the format (xct_format_info)    */
} xct_staged;

typedef struct {
  void* d_out;            /* f32 (single/mixed/half) or f64 (double)      */
  int64_t row_stride;     /* elements between consecutive output rows    */
  int64_t chunk_stride;   /* elements between consecutive F-chunks       */
  int32_t valid_cols;     /* slices to write (drops the padded tail)     */
  int32_t ffactor;        /* slices per chunk as seen by the caller (F)  */
  int32_t value_scale_exp;/* outputs scaled by 2^-exp (src/engine.py:137) */
  int32_t accumulate;     /* 1: out += result (rank-ordered partial sums) */
  const double* d_factors;/* [n_chunks] denormalize factors, NULL = 1     */
  double* d_dot_partials; /* [n_chunks*n_cta] sum of out^2, NULL = skip   */
  int64_t x_chunk_stride; /* input records between F-chunks, 0 = n_in     */
  int64_t x_elem_stride;  /* input records between elements, 0 = 1        */
  /* fused exchange (native domain partition): when d_out_ptrs != NULL,
   * output row r with d_seg[q] <= r < d_seg[q+1] is written at
   * d_out_ptrs[q] + (r - d_seg[q]) * row_stride -- device pointers, peers'
   * receive buffers mapped over NVLink (xct_ipc_open) or local; d_out is
   * ignored.  d_out_ptrs [n_seg], d_seg [n_seg+1] in device memory. */
  void* const* d_out_ptrs;
  const int64_t* d_seg;
  int32_t n_seg;
} xct_epilogue;

int xct_spmm(const xct_staged* a, int precision, const void* d_x, int64_t n_in,
             int64_t n_chunks, int32_t f_dev, const xct_epilogue* ep,
             int64_t smem_bytes, void* stream);

/* float64 CSR product y = A x over n_slices columns (row-major x [n_cols][S],
 * y [n_rows][S]); measurement synthesis (src/geometry.py:347-367). */
int xct_csr_spmm_f64(const int64_t* d_indptr, const int32_t* d_indices,
                     const double* d_values, int64_t n_rows, const double* d_x,
                     int64_t n_slices, double* d_y, void* stream);

/* ---------------------------------------------------------------------------
 * K7  max-abs normalization per F-slice chunk
 * replaces matrixstore.normalize (src/matrixstore.py:290-305) for the chunk
 * loop of pipeline._apply (src/pipeline.py:160-168).
 * Input v is strided: element i, slice j at v[i*row_stride + j] (dtype
 * in_f64 ? f64 : f32), j < n_slices.  d_maxbits[n_chunks] receives the
 * max |v| of each chunk as raw IEEE bits (u64 of the f64 value).
 * xct_normalize writes chunk c of (v / factor_c) cast to the storage dtype
 * into d_out [n_chunks][n][f_dev], zero-padding slices >= n_slices.
 * ------------------------------------------------------------------------- */
int xct_chunk_maxabs(const void* d_v, int in_f64, int64_t n, int64_t n_slices,
                     int64_t row_stride, int32_t ffactor, int64_t n_chunks,
                     uint64_t* d_maxbits, void* stream);
int xct_normalize(const void* d_v, int in_f64, int64_t n, int64_t n_slices,
                  int64_t row_stride, int32_t ffactor, int64_t n_chunks,
                  int32_t f_dev, const double* d_factors, int precision,
                  void* d_out, void* stream);

/* ---------------------------------------------------------------------------
 * K8/K9  CGLS vector kernels (src/solver.py:84-192)
 * Persistent vectors live in the chunked layout [n_chunks][n][f_dev]:
 * double -> f64, single -> f32, half/mixed -> f16 payload + one scalar
 * factor (_VectorStore, src/solver.py:84-108).  "load" = payload*factor in
 * f32.  All reductions are deterministic (fixed-order block partials).
 * ------------------------------------------------------------------------- */
/* sum_i a_i*b_i in f64 over n_elem elements of dtype code (0 f64, 1 f32,
 * 2 f16 scaled by fa/fb as float32 loads) -> d_result[0] */
int xct_dot(const void* d_a, const void* d_b, int dtype, int64_t n_elem,
            float fa, float fb, double* d_scratch, double* d_result, void* stream);

/* fixed-order f64 sum of n partials (e.g. the SpMM epilogue's
 * d_dot_partials) -> d_result[0] */
int xct_sum_f64(const double* d_v, int64_t n, double* d_result, void* stream);

/* d_hist[e] += number of positive values of d_v[0..n) with biased f64
 * exponent e (2048 bins, caller zeroes): the binade histogram behind
 * matrixstore.half_rescale_exponent (src/matrixstore.py:264-275) for a
 * matrix streamed chunk by chunk */
int xct_binade_hist(const double* d_v, int64_t n, uint64_t* d_hist, void* stream);

/* max |load(v)| over n_elem -> d_maxbits[0] (IEEE bits of the f64 value,
 * atomicMax; caller zeroes it first) */
int xct_maxabs(const void* d_v, int dtype, int64_t n_elem, float fv,
               uint64_t* d_maxbits, void* stream);

/* out = load(a) + s*load(b)   (two roundings: multiply, then add; d_b may
 * be NULL for out = load(a)), s rounded to f32 unless all operands are f64.
 * out_dtype 0/1 writes f64/f32.  out_dtype 2 is the half store of
 * _VectorStore: pass 1 (d_out == NULL) reduces max|out| into d_maxbits;
 * pass 2 writes f16(out / out_factor) and, if d_sumsq, sum(load(stored)^2)
 * (deterministic, via d_scratch[148*8] partials). */
int xct_axpy(const void* d_a, int a_dtype, float fa, const void* d_b, int b_dtype,
             float fb, double scale, int64_t n_elem, void* d_out, int out_dtype,
             float out_factor, uint64_t* d_maxbits, double* d_scratch,
             double* d_sumsq, void* stream);

/* per-chunk normalize of a stored vector for the operator input:
 * max over chunk c of |load(v)| -> d_maxbits[c] (f64 bits, zeroed by caller) */
int xct_chunk_maxabs_chunked(const void* d_v, int dtype, float fv, int64_t n,
                             int64_t n_chunks, int32_t f_dev,
                             uint64_t* d_maxbits, void* stream);
/* out[c] = (load(v[c]) / factor_c) cast to the storage dtype of precision */
int xct_normalize_chunked(const void* d_v, int dtype, float fv, int64_t n,
                          int64_t n_chunks, int32_t f_dev, const double* d_factors,
                          int precision, void* d_out, void* stream);

/* layout conversion chunked [n_chunks][n][f_dev] (f64/f32) <-> strided
 * (n, n_slices) f64 */
int xct_unchunk_f64(const void* d_in, int in_dtype, float fin, int64_t n,
                    int64_t n_slices, int32_t ffactor, int32_t f_dev,
                    double* d_out, void* stream);
int xct_chunk_from_f64(const double* d_in, int64_t n, int64_t n_slices,
                       int32_t ffactor, int32_t f_dev, int out_dtype,
                       void* d_out, void* stream);

/* Measurements / results in the caller's row-major (n, n_slices) layout,
 * streamed one block of rows at a time (cgls_solve with host arrays,
 * src/solver.py:137 and :194-195):
 * rows_to_chunked: rows [r0, r0+nr) (d_rows = that block, f64 or f32) ->
 *   chunked work layout (f64 or f32, round to nearest); max|v| and
 *   max|wd(v)| as f64 bits (atomic max into zeroed slots) and, if d_sumsq,
 *   the f64 sum of v*v of the block (d_scratch[148*8]);
 * unchunk_rows_f64: rows [r0, r0+nr) of a chunked vector -> (nr, n_slices) f64. */
int xct_rows_to_chunked(const void* d_rows, int in_dtype, int64_t r0, int64_t nr, int64_t n,
                        int64_t n_slices, int32_t ffactor, int32_t f_dev, int out_dtype,
                        void* d_out, uint64_t* d_max_in, uint64_t* d_max_out,
                        double* d_scratch, double* d_sumsq, void* stream);
int xct_unchunk_rows_f64(const void* d_in, int in_dtype, float fin, int64_t n, int64_t r0,
                         int64_t nr, int64_t n_slices, int32_t ffactor, int32_t f_dev,
                         double* d_out, void* stream);

/* ---------------------------------------------------------------------------
 * K10  partial-result exchange of the data-partitioned operator
 * replaces comm.execute_plan / engine.reduce_partials (src/comm.py:420-472,
 * src/engine.py:189-221).  Chunked vectors [n_chunks][n][fd] (f32, or f64
 * when f64 != 0); whole element rows move.  The caller fixes the summation
 * order (owner's own partial first, then senders ascending = the
 * reference's direct plan); the bytes travel with NCCL over NVLink.
 * ------------------------------------------------------------------------- */
/* dst[c][i] = src[c][idx[i]] */
int xct_gather_rows(const void* d_src, int64_t n_src, const int32_t* d_idx, int64_t m,
                    int64_t n_chunks, int32_t fd, int f64, void* d_dst, void* stream);
/* dst[c][pos[i]] += src[c][i] */
int xct_accumulate_rows(void* d_dst, int64_t n_dst, const void* d_src, const int32_t* d_pos,
                        int64_t m, int64_t n_chunks, int32_t fd, int f64, void* stream);
/* v[c][*] *= factors[c] (denormalize, src/matrixstore.py:308-316) and, if
 * d_sumsq, the f64 sum of squares of the result (d_scratch[148*8]) */
int xct_scale_chunks(void* d_v, int64_t per_chunk, int64_t n_chunks, const double* d_factors,
                     int f64, double* d_scratch, double* d_sumsq, void* stream);

/* CUDA IPC for the fused exchange: device memory this process allocates
 * and exports (64-byte handle), and peers' exports mapped into this
 * process (peer pointers usable by kernels over NVLink / NVSwitch). */
int xct_ipc_alloc(int64_t bytes, void** d_ptr, void* h_handle /* [64] */);
int xct_ipc_open(const void* h_handle /* [64] */, void** d_ptr);
int xct_ipc_close(void* d_ptr);
int xct_ipc_free(void* d_ptr);

/* Element-major exchange buffers of the native domain partition
 * ([m][n_chunks][record]: each peer's rows are one contiguous message):
 * gather_records: dst[i][c] = src[c0 + c][idx[i]] (chunk-major source,
 *   records of rec_bytes, a multiple of 16);
 * accumulate_records: dst[c0 + c][pos[i]][f] += src[i][c][f] (f32/f64,
 *   the caller orders the calls: owner first, then senders ascending). */
int xct_gather_records(const void* d_src, int64_t n_src, const int32_t* d_idx, int64_t m,
                       int64_t c0, int64_t n_chunks, int32_t rec_bytes, void* d_dst,
                       void* stream);
int xct_accumulate_records(void* d_dst, int64_t n_dst, int64_t c0, const void* d_src,
                           const int32_t* d_pos, int64_t m, int64_t n_chunks, int32_t fd,
                           int f64, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* XCT_B200_H */
