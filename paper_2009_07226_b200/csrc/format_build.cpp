// K5: host builder of the staged SpMM execution format.
//
// B200 re-design of matrixstore.build_staged / pack
// (src/matrixstore.py:250-262, :417-562).  The reference cuts each of
// `block_partitions` row chunks' sorted column footprint into stages and
// stores warp-sliced ELL groups.  Here the unit of work is a CTA tile of
// rows (chosen by the caller: sinogram tiles for projection, voxel tiles for
// back projection) and the staging order is a caller-supplied key per
// column (image band / view angle / reference stage id).  A CTA's footprint
// sorted by (key, col) is cut into load groups of whole keys; each group is
// staged once into shared memory and every row accumulates its entries of
// that group in (key, CSR position) order.  This reproduces the reference's
// per-row accumulation order exactly when the keys are the reference's
// stage ids, and gives pure traversal order with band keys.
//
// Storage per (group, warp) is a zero-padded slab [width/4][rows_per_warp][4]
// of (uint16 slot, stored length): a lane fetches 4 entries with one vector
// load and the warp's loads are contiguous.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "xct_common.h"

namespace {

// float64 -> IEEE half, round to nearest even (numpy's direct f64->f16 cast).
uint16_t f64_to_f16(double x) {
  uint16_t sign = std::signbit(x) ? 0x8000 : 0;
  double a = std::fabs(x);
  if (std::isnan(a)) return sign | 0x7e00;
  if (std::isinf(a)) return sign | 0x7c00;
  if (a == 0.0) return sign;
  int q;
  std::frexp(a, &q);          // a = m * 2^q, m in [0.5, 1)
  int e = q - 1;              // a in [2^e, 2^(e+1))
  if (e < -14) {              // subnormal: quantum 2^-24
    double r = std::nearbyint(std::ldexp(a, 24));
    return sign | (uint16_t)r;  // r == 1024 encodes the smallest normal
  }
  double r = std::nearbyint(std::ldexp(a, 10 - e));  // in [1024, 2048]
  if (r == 2048.0) { r = 1024.0; ++e; }
  if (e > 15) return sign | 0x7c00;
  return sign | (uint16_t)(((e + 15) << 10) | ((int)r - 1024));
}

double f16_to_f64(uint16_t h) {
  int e = (h >> 10) & 0x1f, m = h & 0x3ff;
  double v;
  if (e == 0) v = std::ldexp((double)m, -24);
  else if (e == 31) v = m ? NAN : INFINITY;
  else v = std::ldexp((double)(m | 0x400), e - 25);
  return (h & 0x8000) ? -v : v;
}

struct KC { int32_t key, col; };
inline bool kc_less(const KC& a, const KC& b) {
  return a.key < b.key || (a.key == b.key && a.col < b.col);
}

struct CtaPlan {
  std::vector<KC> foot;              // footprint sorted by (key, col)
  std::vector<int64_t> gstart;       // group starts in foot (+ end)
  std::vector<int32_t> width;        // [n_groups_local * warps] padded widths
};

// Shared-memory bank class of a slot for the lanes of one row (mirrors the
// plane layout of spmm.cu: piece p of slot s sits at bank quad
// (s + p*8/NP) mod 8, the L lanes of a row read pieces L apart).  Two rows of
// a quarter-warp conflict iff their slots agree mod 8/L.
struct BankModel {
  int lp = -1, lg = 0, rq = 0;   // log2 pieces, log2 lanes per row, rows per quarter
  bool on() const { return lp >= 0 && rq > 1; }
  void init(int log2_pieces, int log2_lanes) {
    lp = log2_pieces;
    lg = log2_lanes;
    rq = lg <= 3 ? (8 >> lg) : 1;
  }
  int cls(int64_t slot) const { return (int)(slot & (rq - 1)); }
};

// Proper edge colouring of a bipartite multigraph rows x bank classes with
// `ncolor` >= max degree colours (Konig): colour = step of the slab, so no
// two rows of a quarter-warp read the same bank quads in one step.
struct Colorer {
  int ncolor = 0, words = 0;
  std::vector<int32_t> atL, atR;        // [vertex * ncolor + colour] -> edge or -1
  std::vector<uint64_t> freeL, freeR;   // free-colour bitmaps
  std::vector<int32_t> er, ec, col;
  std::vector<int32_t> path;

  void reset(int nl, int nr, int nc) {
    ncolor = nc;
    words = (nc + 63) / 64;
    atL.assign((size_t)nl * nc, -1);
    atR.assign((size_t)nr * nc, -1);
    freeL.assign((size_t)nl * words, ~0ull);
    freeR.assign((size_t)nr * words, ~0ull);
    for (int v = 0; v < nl; ++v) trim(freeL, v);
    for (int v = 0; v < nr; ++v) trim(freeR, v);
    er.clear(); ec.clear(); col.clear();
  }
  void trim(std::vector<uint64_t>& f, int v) {
    int rem = ncolor % 64;
    if (rem) f[(size_t)v * words + words - 1] = (1ull << rem) - 1;
  }
  int first_free(const std::vector<uint64_t>& f, int v) const {
    for (int w = 0; w < words; ++w) {
      uint64_t m = f[(size_t)v * words + w];
      if (m) return w * 64 + __builtin_ctzll(m);
    }
    return -1;
  }
  void put(int e, int c) {
    col[e] = c;
    atL[(size_t)er[e] * ncolor + c] = e;
    atR[(size_t)ec[e] * ncolor + c] = e;
    freeL[(size_t)er[e] * words + c / 64] &= ~(1ull << (c % 64));
    freeR[(size_t)ec[e] * words + c / 64] &= ~(1ull << (c % 64));
  }
  void take(int e) {
    int c = col[e];
    atL[(size_t)er[e] * ncolor + c] = -1;
    atR[(size_t)ec[e] * ncolor + c] = -1;
    freeL[(size_t)er[e] * words + c / 64] |= 1ull << (c % 64);
    freeR[(size_t)ec[e] * words + c / 64] |= 1ull << (c % 64);
  }
  bool add(int l, int r) {
    int e = (int)er.size();
    er.push_back(l); ec.push_back(r); col.push_back(-1);
    int a = first_free(freeL, l), b = first_free(freeR, r);
    if (a < 0 || b < 0) return false;
    if (atR[(size_t)r * ncolor + a] >= 0) {
      // flip the a/b alternating path that starts at r; it cannot reach l
      path.clear();
      int v = r, want = a;
      bool right = true;
      for (;;) {
        int e2 = right ? atR[(size_t)v * ncolor + want] : atL[(size_t)v * ncolor + want];
        if (e2 < 0) break;
        path.push_back(e2);
        v = right ? er[e2] : ec[e2];
        right = !right;
        want = want == a ? b : a;
      }
      for (int e2 : path) take(e2);
      for (int e2 : path) put(e2, col[e2] == a ? b : a);
    }
    put(e, a);
    return true;
  }
};

// Step schedule of one (group, warp, quarter-warp): each of the quarter's
// rows (lane sets) reads one staged slot per step, and two different slots
// of the same bank class in one step cost an extra shared-memory wavefront.
// A proper edge colouring of rows x bank classes needs max(row degree,
// class degree) steps; the slab width is only the row degree (rounded to 4,
// `width`).  Edges coloured beyond `width` are moved to the earlier step
// where their row is free and the fewest other slots of their class are
// read (a same-slot read is a broadcast, free) -- a few 2-way conflicts on
// one quarter instead of extra steps that every quarter of the warp pays
// for.  With compress == false the class degree sets the width (fully
// conflict-free, the round-1 v6 schedule).
struct QuarterScheduler {
  Colorer colorer;
  std::vector<int32_t> cls_cnt, first_slot, step_of;
  std::vector<char> busy;
  // edges: (row in quarter, slot); returns steps in step_of (same order)
  bool run(int rq, int width, const std::vector<std::pair<int32_t, int32_t>>& edges,
           const BankModel& bank, bool compress) {
    int maxdeg = width;
    if (compress) {
      int cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      for (auto& e : edges) ++cnt[bank.cls(e.second)];
      for (int c = 0; c < 8; ++c) maxdeg = std::max(maxdeg, cnt[c]);
    }
    colorer.reset(rq, 8, maxdeg);
    for (auto& e : edges)
      if (!colorer.add(e.first, bank.cls(e.second))) return false;
    step_of.assign(colorer.col.begin(), colorer.col.end());
    if (maxdeg == width) return true;
    busy.assign((size_t)rq * width, 0);
    cls_cnt.assign((size_t)width * 8, 0);
    first_slot.assign((size_t)width * 8, -1);
    for (size_t i = 0; i < edges.size(); ++i) {
      const int n = step_of[i];
      if (n >= width) continue;
      busy[(size_t)edges[i].first * width + n] = 1;
      const int c = bank.cls(edges[i].second);
      ++cls_cnt[(size_t)n * 8 + c];
      if (first_slot[(size_t)n * 8 + c] < 0) first_slot[(size_t)n * 8 + c] = edges[i].second;
    }
    for (size_t i = 0; i < edges.size(); ++i) {
      if (step_of[i] < width) continue;
      const int r = edges[i].first, slot = edges[i].second, c = bank.cls(slot);
      int best = -1, best_cost = 1 << 30;
      for (int n = 0; n < width; ++n) {
        if (busy[(size_t)r * width + n]) continue;
        const int fs = first_slot[(size_t)n * 8 + c];
        const int cost = fs < 0 || fs == slot ? 0 : cls_cnt[(size_t)n * 8 + c];
        if (cost < best_cost) { best_cost = cost; best = n; if (!cost) break; }
      }
      if (best < 0) return false;              // cannot happen: row degree <= width
      step_of[i] = best;
      busy[(size_t)r * width + best] = 1;
      ++cls_cnt[(size_t)best * 8 + c];
      if (first_slot[(size_t)best * 8 + c] < 0) first_slot[(size_t)best * 8 + c] = slot;
    }
    return true;
  }
};

// default on (measured 2.5-4% faster K6 at c2, FP32 and FP16);
// XCT_SCHED_COMPRESS=0 restores the fully conflict-free schedule
bool sched_compress() {
  const char* e = std::getenv("XCT_SCHED_COMPRESS");
  return !(e && e[0] == '0');
}

}  // namespace

struct xct_format {
  xct_format_info info{};
  std::vector<int32_t> cta_group_ptr;
  std::vector<int64_t> group_map_ptr;
  std::vector<int32_t> group_map;
  std::vector<int64_t> slab_off;
  std::vector<int32_t> slab_width;
  // slabs: uninitialised allocations, zeroed CTA by CTA in phase C
  std::unique_ptr<uint16_t[]> slots;
  std::unique_ptr<uint8_t[]> values;
  int64_t n_padded = 0;
  int vbytes = 0;
  int row_group = 1;     // values per slab position (rows sharing an entry)
};

namespace {

template <typename F>
void parallel_for(int64_t n, int n_threads, F fn) {
  if (n_threads < 1) n_threads = 1;
  std::atomic<int64_t> next{0};
  auto worker = [&]() {
    for (;;) {
      int64_t i = next.fetch_add(1);
      if (i >= n) break;
      fn(i);
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < n_threads; ++t) pool.emplace_back(worker);
  worker();
  for (auto& th : pool) th.join();
}

struct PhaseLog {
  bool on = std::getenv("XCT_VERBOSE") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void lap(const char* what) {
    if (!on) return;
    auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[xct] format_build %s %.3f s\n", what,
                 std::chrono::duration<double>(now - t).count());
    t = now;
  }
};

}  // namespace

namespace {

// ---- grouped rows (row_group G = 2 or 4) -----------------------------------
// G consecutive thread-rows of a CTA form a unit owned by one lane set; the
// unit walks the UNION of its rows' entries, so one staged-record read from
// shared memory serves G rows (the shared-memory crossbar, not HBM, bounds
// K6: SURVEY §7).  A union entry stores one slot and G values; a row absent
// from the entry stores 0, and x*0 + acc == acc exactly, so every row's sum
// is its own entries in stored order.  A column repeated inside one row gets
// one extra union entry per repeat.  Union entries of a load group are
// ordered by (key, column) -- ascending ray id per voxel for the back
// projection -- then placed on slab steps by the bank schedule.
// Slab layout per (group, warp): slots [width/4][units_per_warp][4] (as for
// G = 1) and values [width/4][NV][units_per_warp][16 B], NV = 4*G*vbytes/16:
// piece k of a unit holds its value words k*epp.., word = entry*G + row.
// A warp's step is then two contiguous runs (slots, values) that one bulk
// copy each moves into shared memory, and every 128-bit read of piece k by
// the warp's units is one conflict-free contiguous run.
struct UEnt {
  int32_t key, col, dup, slot;
  int64_t j[4];
};

int build_grouped(int64_t n_rows, int64_t n_cols, const int64_t* indptr, const int32_t* indices,
                  const double* values, int64_t n_cta, int64_t rows_per_cta,
                  int64_t rows_per_warp, const int32_t* cta_rows, const int32_t* key_tables,
                  const int32_t* cta_table, int64_t capacity, int precision, int value_scale_exp,
                  int sched_log2_pieces, int sched_log2_lanes, int G, int n_threads,
                  xct_format** out) {
  if (G != 2 && G != 4) return xct::fail(XCT_EINVAL, "format_build: row_group must be 1, 2 or 4");
  if (n_rows < 0 || n_cols < 0 || n_cta < 0 || rows_per_cta < 1 || rows_per_warp < 1 ||
      rows_per_cta % rows_per_warp || rows_per_warp % G)
    return xct::fail(XCT_EINVAL, "format_build: bad shape arguments");
  if (capacity < 1 || capacity > 65536)
    return xct::fail(XCT_ESTAGE, "format_build: capacity must be in [1, 65536] slots");
  if (precision != XCT_SINGLE && precision != XCT_MIXED)
    return xct::fail(XCT_EINVAL, "format_build: grouped rows support single and mixed only");
  if (!indptr || (!indices && indptr[n_rows] > 0) || !cta_rows || !key_tables || !cta_table)
    return xct::fail(XCT_EINVAL, "format_build: null input array");
  if (sched_log2_pieces < 0)
    return xct::fail(XCT_EINVAL, "format_build: grouped rows need the bank schedule");
  const int64_t warps = rows_per_cta / rows_per_warp;
  const int64_t upw = rows_per_warp / G;            // units per warp
  const int64_t upc = rows_per_cta / G;             // units per CTA
  const int vbytes = precision == XCT_SINGLE ? 4 : 2;
  if (sched_log2_lanes < 0 || sched_log2_lanes > sched_log2_pieces ||
      (32 >> sched_log2_lanes) != upw)
    return xct::fail(XCT_EINVAL, "format_build: schedule lanes do not match units per warp");
  BankModel bank;
  bank.init(sched_log2_pieces, sched_log2_lanes);
  const int64_t rq = bank.on() ? bank.rq : upw;
  const bool compress = sched_compress();
  PhaseLog plog;
  std::vector<CtaPlan> plans(n_cta);
  std::mutex err_mu;
  int err = XCT_OK;
  std::string err_msg;

  // ---- phase A: footprint, load groups, union widths per (group, warp) ----
  parallel_for(n_cta, n_threads, [&](int64_t b) {
    CtaPlan& P = plans[b];
    const int32_t* keys = key_tables + (int64_t)cta_table[b] * n_cols;
    static thread_local std::vector<int64_t> fstamp, ustamp, rstamp;
    static thread_local int64_t gen = 0;
    static thread_local std::vector<int32_t> group_of, cls_of;
    if ((int64_t)fstamp.size() < n_cols) {
      fstamp.assign(n_cols, -1); ustamp.assign(n_cols, -1); rstamp.assign(n_cols, -1);
      group_of.assign(n_cols, 0); cls_of.assign(n_cols, 0);
    }
    const int64_t fm = ++gen;
    std::vector<KC> all;
    for (int64_t t = 0; t < rows_per_cta; ++t) {
      int32_t r = cta_rows[b * rows_per_cta + t];
      if (r < 0) continue;
      for (int64_t j = indptr[r]; j < indptr[r + 1]; ++j) {
        const int32_t col = indices[j];
        if (fstamp[col] == fm) continue;
        fstamp[col] = fm;
        all.push_back({keys[col], col});
      }
    }
    std::sort(all.begin(), all.end(), kc_less);
    P.foot.swap(all);
    int64_t cur = 0, i = 0, n = (int64_t)P.foot.size();
    P.gstart.push_back(0);
    while (i < n) {
      int64_t j = i;
      while (j < n && P.foot[j].key == P.foot[i].key) ++j;
      int64_t m = j - i;
      if (m > capacity) {
        std::lock_guard<std::mutex> lk(err_mu);
        err = XCT_ESTAGE;
        err_msg = "format_build: one staging key needs " + std::to_string(m) +
                  " slots, capacity is " + std::to_string(capacity);
        return;
      }
      if (cur + m > capacity) { P.gstart.push_back(i); cur = 0; }
      cur += m;
      i = j;
    }
    if (n > 0) P.gstart.push_back(n);
    else P.gstart.clear();
    const int64_t ng = P.gstart.empty() ? 0 : (int64_t)P.gstart.size() - 1;
    P.width.assign(ng * warps, 0);
    for (int64_t g = 0; g < ng; ++g)
      for (int64_t p = P.gstart[g]; p < P.gstart[g + 1]; ++p) {
        group_of[P.foot[p].col] = (int32_t)g;
        cls_of[P.foot[p].col] = bank.on() ? bank.cls(p - P.gstart[g]) : 0;
      }
    std::vector<int32_t> cnt(ng), ccnt(ng * 8);
    for (int64_t u = 0; u < upc; ++u) {
      const int64_t w = u / upw;
      if (u % rq == 0) std::fill(ccnt.begin(), ccnt.end(), 0);
      std::fill(cnt.begin(), cnt.end(), 0);
      const int64_t um = ++gen;
      for (int gi = 0; gi < G; ++gi) {
        const int32_t r = cta_rows[b * rows_per_cta + u * G + gi];
        if (r < 0) continue;
        const int64_t rm = ++gen;
        for (int64_t j = indptr[r]; j < indptr[r + 1]; ++j) {
          const int32_t col = indices[j];
          bool fresh;
          if (rstamp[col] == rm) {
            fresh = true;                          // repeat inside the row
          } else {
            rstamp[col] = rm;
            fresh = ustamp[col] != um;
            ustamp[col] = um;
          }
          if (fresh) {
            ++cnt[group_of[col]];
            ++ccnt[group_of[col] * 8 + cls_of[col]];
          }
        }
      }
      for (int64_t g = 0; g < ng; ++g) {
        int32_t pw = (cnt[g] + 3) & ~3;
        if (pw > P.width[g * warps + w]) P.width[g * warps + w] = pw;
      }
      if (!compress && (u % rq == rq - 1 || u == upc - 1)) {
        for (int64_t g = 0; g < ng; ++g)
          for (int c = 0; c < 8; ++c) {
            int32_t pw = (ccnt[g * 8 + c] + 3) & ~3;
            if (pw > P.width[g * warps + w]) P.width[g * warps + w] = pw;
          }
      }
    }
  });
  if (err) return xct::fail(err, err_msg);
  plog.lap("A(grouped)");

  // ---- phase B: global offsets ---------------------------------------------
  xct_format* F = new (std::nothrow) xct_format();
  if (!F) return xct::fail(XCT_ENOMEM, "format_build: out of host memory");
  F->cta_group_ptr.assign(n_cta + 1, 0);
  int64_t n_groups = 0, n_slots = 0, n_padded = 0, max_gs = 0;
  for (int64_t b = 0; b < n_cta; ++b) {
    int64_t ng = plans[b].gstart.empty() ? 0 : (int64_t)plans[b].gstart.size() - 1;
    n_groups += ng;
    F->cta_group_ptr[b + 1] = (int32_t)n_groups;
    n_slots += (int64_t)plans[b].foot.size();
    for (int64_t g = 0; g < ng; ++g)
      max_gs = std::max(max_gs, plans[b].gstart[g + 1] - plans[b].gstart[g]);
    for (int32_t w : plans[b].width) n_padded += (int64_t)w * upw;
  }
  if (n_groups > INT32_MAX) { delete F; return xct::fail(XCT_EINVAL, "format_build: too many groups"); }
  try {
    F->group_map_ptr.assign(n_groups + 1, 0);
    F->group_map.assign(n_slots, 0);
    F->slab_off.assign(n_groups * warps, 0);
    F->slab_width.assign(n_groups * warps, 0);
    F->slots.reset(new uint16_t[std::max<int64_t>(n_padded, 1)]);
    F->values.reset(new uint8_t[std::max<int64_t>(n_padded, 1) * vbytes * G]);
    F->n_padded = n_padded;
    F->vbytes = vbytes;
    F->row_group = G;
  } catch (...) {
    delete F;
    return xct::fail(XCT_ENOMEM, "format_build: out of host memory");
  }
  std::vector<int64_t> cta_slot0(n_cta + 1, 0), cta_e0(n_cta + 1, 0);
  {
    int64_t gi = 0, so = 0, eo = 0;
    for (int64_t b = 0; b < n_cta; ++b) {
      cta_slot0[b] = so;
      cta_e0[b] = eo;
      const CtaPlan& P = plans[b];
      int64_t ng = P.gstart.empty() ? 0 : (int64_t)P.gstart.size() - 1;
      for (int64_t g = 0; g < ng; ++g) {
        so += P.gstart[g + 1] - P.gstart[g];
        F->group_map_ptr[gi + g + 1] = so;
      }
      for (int64_t w = 0; w < warps; ++w)
        for (int64_t g = 0; g < ng; ++g) {
          F->slab_off[(gi + g) * warps + w] = eo;
          F->slab_width[(gi + g) * warps + w] = P.width[g * warps + w];
          eo += (int64_t)P.width[g * warps + w] * upw;
        }
      gi += ng;
    }
    cta_e0[n_cta] = eo;
  }
  plog.lap("B(grouped)");

  // ---- phase C: fill maps and slabs ----------------------------------------
  const double scale = std::ldexp(1.0, value_scale_exp);
  std::vector<double> worst(n_cta, 0.0);
  std::vector<int64_t> under(n_cta, 0);
  parallel_for(n_cta, n_threads, [&](int64_t b) {
    if (err) return;
    const CtaPlan& P = plans[b];
    const int32_t* keys = key_tables + (int64_t)cta_table[b] * n_cols;
    const int64_t g0 = F->cta_group_ptr[b];
    std::memset(F->slots.get() + cta_e0[b], 0, (size_t)(cta_e0[b + 1] - cta_e0[b]) * 2);
    std::memset(F->values.get() + cta_e0[b] * vbytes * G, 0,
                (size_t)(cta_e0[b + 1] - cta_e0[b]) * vbytes * G);
    for (size_t i = 0; i < P.foot.size(); ++i) F->group_map[cta_slot0[b] + i] = P.foot[i].col;
    const int64_t ng = P.gstart.empty() ? 0 : (int64_t)P.gstart.size() - 1;
    static thread_local std::vector<int32_t> slot_of, group_of, uidx;
    static thread_local std::vector<int64_t> ustamp, rstamp;
    static thread_local int64_t gen = 0;
    if ((int64_t)slot_of.size() < n_cols) {
      slot_of.assign(n_cols, 0); group_of.assign(n_cols, 0); uidx.assign(n_cols, 0);
      ustamp.assign(n_cols, -1); rstamp.assign(n_cols, -1);
    }
    for (int64_t g = 0; g < ng; ++g)
      for (int64_t p = P.gstart[g]; p < P.gstart[g + 1]; ++p) {
        group_of[P.foot[p].col] = (int32_t)g;
        slot_of[P.foot[p].col] = (int32_t)(p - P.gstart[g]);
      }
    // union entries of every unit, sorted, with per-(unit, group) offsets
    std::vector<UEnt> flat;
    std::vector<int64_t> gofs((size_t)(ng + 1) * upc, 0);
    std::vector<UEnt> list;
    for (int64_t u = 0; u < upc; ++u) {
      list.clear();
      const int64_t um = ++gen;
      int32_t dupc = 0;
      for (int gi = 0; gi < G; ++gi) {
        const int32_t r = cta_rows[b * rows_per_cta + u * G + gi];
        if (r < 0) continue;
        const int64_t rm = ++gen;
        for (int64_t j = indptr[r]; j < indptr[r + 1]; ++j) {
          const int32_t col = indices[j];
          if (rstamp[col] != rm && ustamp[col] == um) {
            rstamp[col] = rm;
            list[uidx[col]].j[gi] = j;
            continue;
          }
          UEnt e{keys[col], col, 0, slot_of[col], {-1, -1, -1, -1}};
          e.j[gi] = j;
          if (rstamp[col] == rm) {
            e.dup = ++dupc;                         // repeat inside the row
          } else {
            rstamp[col] = rm;
            ustamp[col] = um;
            uidx[col] = (int32_t)list.size();
          }
          list.push_back(e);
        }
      }
      std::sort(list.begin(), list.end(), [](const UEnt& a, const UEnt& c) {
        if (a.key != c.key) return a.key < c.key;
        if (a.col != c.col) return a.col < c.col;
        return a.dup < c.dup;
      });
      const int64_t base = (int64_t)flat.size();
      int64_t at = 0;
      const int64_t m = (int64_t)list.size();
      for (int64_t g = 0; g <= ng; ++g) {
        while (g < ng && at < m && group_of[list[at].col] < g) ++at;
        gofs[(size_t)u * (ng + 1) + g] = base + (g < ng ? at : m);
      }
      flat.insert(flat.end(), list.begin(), list.end());
    }
    double wmax = 0.0;
    int64_t nunder = 0;
    auto write = [&](int64_t gg, int64_t w, int64_t uin, int64_t n, const UEnt* E, int32_t slot) {
      const int64_t at = F->slab_off[gg * warps + w] + ((n >> 2) * upw + uin) * 4 + (n & 3);
      F->slots[at] = (uint16_t)slot;
      if (!E) return;                          // padding: values stay 0
      const int64_t epp = 16 / vbytes;                        // values per piece
      const int64_t step0 = F->slab_off[gg * warps + w] + (n >> 2) * upw * 4;
      for (int gi = 0; gi < G; ++gi) {
        const int64_t j = E->j[gi];
        if (j < 0) continue;
        const double v = values[j] * scale;
        double back;
        const int64_t wd = (n & 3) * G + gi;                     // word of the unit's step
        const int64_t vi = step0 * G + ((wd / epp) * upw + uin) * epp + wd % epp;
        uint8_t* dst = F->values.get() + vi * vbytes;
        if (precision == XCT_SINGLE) {
          float f = (float)v;
          std::memcpy(dst, &f, 4);
          back = (double)f;
        } else {
          uint16_t h = f64_to_f16(v);
          std::memcpy(dst, &h, 2);
          back = f16_to_f64(h);
        }
        if (v != 0.0) {
          if (back == 0.0) ++nunder;
          double rel = std::fabs(back - v) / std::fabs(v);
          if (rel > wmax) wmax = rel;
        }
      }
    };
    QuarterScheduler qs;
    std::vector<std::pair<int32_t, int32_t>> qedges;
    std::vector<int32_t> step_slot;
    std::vector<std::pair<int64_t, const UEnt*>> owner;
    std::vector<char> used;
    for (int64_t g = 0; g < ng; ++g) {
      const int64_t gg = g0 + g;
      for (int64_t w = 0; w < warps; ++w) {
        const int64_t width = F->slab_width[gg * warps + w];
        for (int64_t q0 = 0; q0 < upw; q0 += rq) {
          step_slot.assign(width, -1);
          owner.clear();
          qedges.clear();
          for (int64_t rr = 0; rr < rq; ++rr) {
            const int64_t u = w * upw + q0 + rr;
            const int64_t a = gofs[(size_t)u * (ng + 1) + g], e = gofs[(size_t)u * (ng + 1) + g + 1];
            for (int64_t k = a; k < e; ++k) {
              qedges.push_back({(int32_t)rr, flat[k].slot});
              owner.push_back({q0 + rr, &flat[k]});
            }
          }
          if (!qs.run((int)rq, (int)width, qedges, bank, compress)) {
            std::lock_guard<std::mutex> lk(err_mu);
            err = XCT_EINVAL;
            err_msg = "format_build: bank schedule exceeded the slab width";
            return;
          }
          used.assign((size_t)rq * width, 0);
          for (size_t e = 0; e < owner.size(); ++e) {
            const int64_t uin = owner[e].first;
            const int64_t n = qs.step_of[e];
            write(gg, w, uin, n, owner[e].second, owner[e].second->slot);
            used[(size_t)(uin - q0) * width + n] = 1;
            if (step_slot[n] < 0) step_slot[n] = owner[e].second->slot;
          }
          for (int64_t rr = 0; rr < rq; ++rr)
            for (int64_t n = 0; n < width; ++n)
              if (!used[(size_t)rr * width + n] && step_slot[n] > 0)
                write(gg, w, q0 + rr, n, nullptr, step_slot[n]);
        }
      }
    }
    worst[b] = wmax;
    under[b] = nunder;
  });
  if (err) {
    delete F;
    return xct::fail(err, err_msg);
  }
  plog.lap("C(grouped)");
  F->info.n_cta = n_cta;
  F->info.rows_per_cta = rows_per_cta;
  F->info.rows_per_warp = rows_per_warp;
  F->info.warps_per_cta = warps;
  F->info.n_groups = n_groups;
  F->info.n_slots = n_slots;
  F->info.n_padded = n_padded;
  F->info.nnz = indptr[n_rows] - indptr[0];
  F->info.max_group_slots = max_gs;
  F->info.value_bytes = vbytes;
  F->info.row_group = G;
  double wm = 0.0;
  int64_t un = 0;
  for (int64_t b = 0; b < n_cta; ++b) { wm = std::max(wm, worst[b]); un += under[b]; }
  F->info.max_rel_quant_error = wm;
  F->info.underflow_count = un;
  *out = F;
  return XCT_OK;
}

}  // namespace


extern "C" int xct_format_build(int64_t n_rows, int64_t n_cols, const int64_t* indptr,
                                const int32_t* indices, const double* values,
                                int64_t n_cta, int64_t rows_per_cta, int64_t rows_per_warp,
                                const int32_t* cta_rows, const int32_t* key_tables,
                                const int32_t* cta_table, int64_t capacity, int precision,
                                int value_scale_exp, int sched_log2_pieces,
                                int sched_log2_lanes, int row_group, int n_threads,
                                xct_format** out) {
  if (!out) return xct::fail(XCT_EINVAL, "format_build: null output handle");
  if (row_group != 1)
    return build_grouped(n_rows, n_cols, indptr, indices, values, n_cta, rows_per_cta,
                         rows_per_warp, cta_rows, key_tables, cta_table, capacity, precision,
                         value_scale_exp, sched_log2_pieces, sched_log2_lanes, row_group,
                         n_threads, out);
  *out = nullptr;
  if (n_rows < 0 || n_cols < 0 || n_cta < 0 || rows_per_cta < 1 || rows_per_warp < 1 ||
      rows_per_cta % rows_per_warp)
    return xct::fail(XCT_EINVAL, "format_build: bad shape arguments");
  if (capacity < 1 || capacity > 65536)
    return xct::fail(XCT_ESTAGE, "format_build: capacity must be in [1, 65536] slots");
  if (precision < 0 || precision > 3) return xct::fail(XCT_EINVAL, "format_build: bad precision");
  if (!indptr || (!indices && indptr[n_rows] > 0) || !cta_rows || !key_tables || !cta_table)
    return xct::fail(XCT_EINVAL, "format_build: null input array");
  const int64_t warps = rows_per_cta / rows_per_warp;
  const int vbytes = precision == XCT_DOUBLE ? 8 : precision == XCT_SINGLE ? 4 : 2;

  BankModel bank;
  if (sched_log2_pieces >= 0) {
    if (sched_log2_lanes < 0 || sched_log2_lanes > sched_log2_pieces ||
        (32 >> sched_log2_lanes) != rows_per_warp)
      return xct::fail(XCT_EINVAL, "format_build: schedule lanes do not match rows_per_warp");
    bank.init(sched_log2_pieces, sched_log2_lanes);
  }
  const bool compress = sched_compress();
  PhaseLog plog;
  std::vector<CtaPlan> plans(n_cta);
  std::mutex err_mu;
  int err = XCT_OK;
  std::string err_msg;

  // ---- phase A: per-CTA footprint, load groups, slab widths ----------------
  parallel_for(n_cta, n_threads, [&](int64_t b) {
    CtaPlan& P = plans[b];
    const int32_t* keys = key_tables + (int64_t)cta_table[b] * n_cols;
    // distinct columns first (a per-thread stamp per column), then sort
    // only the footprint
    static thread_local std::vector<int64_t> stamp;
    static std::atomic<int64_t> stamp_gen{0};
    if ((int64_t)stamp.size() < n_cols) stamp.assign(n_cols, -1);
    const int64_t mark = stamp_gen.fetch_add(1);
    std::vector<KC> all;
    for (int64_t t = 0; t < rows_per_cta; ++t) {
      int32_t r = cta_rows[b * rows_per_cta + t];
      if (r < 0) continue;
      for (int64_t j = indptr[r]; j < indptr[r + 1]; ++j) {
        const int32_t col = indices[j];
        if (stamp[col] == mark) continue;
        stamp[col] = mark;
        all.push_back({keys[col], col});
      }
    }
    std::sort(all.begin(), all.end(), kc_less);
    P.foot.swap(all);
    // whole keys per group, at most `capacity` elements per group
    int64_t cur = 0, i = 0, n = (int64_t)P.foot.size();
    P.gstart.push_back(0);
    while (i < n) {
      int64_t j = i;
      while (j < n && P.foot[j].key == P.foot[i].key) ++j;
      int64_t m = j - i;
      if (m > capacity) {
        std::lock_guard<std::mutex> lk(err_mu);
        err = XCT_ESTAGE;
        err_msg = "format_build: one staging key needs " + std::to_string(m) +
                  " slots, capacity is " + std::to_string(capacity);
        return;
      }
      if (cur + m > capacity) { P.gstart.push_back(i); cur = 0; }
      cur += m;
      i = j;
    }
    if (n > 0) P.gstart.push_back(n);
    else P.gstart.clear();
    const int64_t ng = P.gstart.empty() ? 0 : (int64_t)P.gstart.size() - 1;
    P.width.assign(ng * warps, 0);
    // the key is a function of the column, so the column alone locates an
    // entry in the footprint: dense per-thread lookup tables
    static thread_local std::vector<int32_t> group_of, cls_of;
    if ((int64_t)group_of.size() < n_cols) { group_of.assign(n_cols, 0); cls_of.assign(n_cols, 0); }
    for (int64_t g = 0; g < ng; ++g)
      for (int64_t p = P.gstart[g]; p < P.gstart[g + 1]; ++p) {
        group_of[P.foot[p].col] = (int32_t)g;
        if (bank.on()) cls_of[P.foot[p].col] = bank.cls(p - P.gstart[g]);
      }
    std::vector<int32_t> cnt(ng);
    // per (group, quarter) bank-class loads of the current warp
    std::vector<int32_t> ccnt(bank.on() ? ng * 8 : 0);
    const int64_t rq = bank.on() ? bank.rq : rows_per_warp;
    for (int64_t t = 0; t < rows_per_cta; ++t) {
      int64_t w = t / rows_per_warp;
      if (bank.on() && t % rq == 0) std::fill(ccnt.begin(), ccnt.end(), 0);
      int32_t r = cta_rows[b * rows_per_cta + t];
      if (r >= 0) {
        std::fill(cnt.begin(), cnt.end(), 0);
        for (int64_t j = indptr[r]; j < indptr[r + 1]; ++j) {
          const int32_t col = indices[j];
          ++cnt[group_of[col]];
          if (bank.on()) ++ccnt[group_of[col] * 8 + cls_of[col]];
        }
        for (int64_t g = 0; g < ng; ++g) {
          int32_t pw = (cnt[g] + 3) & ~3;
          if (pw > P.width[g * warps + w]) P.width[g * warps + w] = pw;
        }
      }
      if (bank.on() && !compress && t % rq == rq - 1) {
        for (int64_t g = 0; g < ng; ++g)
          for (int c = 0; c < 8; ++c) {
            int32_t pw = (ccnt[g * 8 + c] + 3) & ~3;
            if (pw > P.width[g * warps + w]) P.width[g * warps + w] = pw;
          }
      }
    }
  });
  if (err) return xct::fail(err, err_msg);
  plog.lap("A");

  // ---- phase B: global offsets ---------------------------------------------
  xct_format* F = new (std::nothrow) xct_format();
  if (!F) return xct::fail(XCT_ENOMEM, "format_build: out of host memory");
  F->cta_group_ptr.assign(n_cta + 1, 0);
  int64_t n_groups = 0, n_slots = 0, n_padded = 0, max_gs = 0;
  for (int64_t b = 0; b < n_cta; ++b) {
    int64_t ng = plans[b].gstart.empty() ? 0 : (int64_t)plans[b].gstart.size() - 1;
    n_groups += ng;
    F->cta_group_ptr[b + 1] = (int32_t)n_groups;
    n_slots += (int64_t)plans[b].foot.size();
    for (int64_t g = 0; g < ng; ++g)
      max_gs = std::max(max_gs, plans[b].gstart[g + 1] - plans[b].gstart[g]);
    for (int32_t w : plans[b].width) n_padded += (int64_t)w * rows_per_warp;
  }
  if (n_groups > INT32_MAX) { delete F; return xct::fail(XCT_EINVAL, "format_build: too many groups"); }
  try {
    F->group_map_ptr.assign(n_groups + 1, 0);
    F->group_map.assign(n_slots, 0);
    F->slab_off.assign(n_groups * warps, 0);
    F->slab_width.assign(n_groups * warps, 0);
    F->slots.reset(new uint16_t[std::max<int64_t>(n_padded, 1)]);
    F->values.reset(new uint8_t[std::max<int64_t>(n_padded, 1) * vbytes]);
    F->n_padded = n_padded;
    F->vbytes = vbytes;
  } catch (...) {
    delete F;
    return xct::fail(XCT_ENOMEM, "format_build: out of host memory");
  }
  plog.lap("B-alloc");
  std::vector<int64_t> cta_slot0(n_cta + 1, 0), cta_e0(n_cta + 1, 0);
  {
    // a warp's slabs of all groups of its tile are contiguous ([tile][warp]
    // [group]): the kernel streams them as one strided sequence, prefetching
    // across group boundaries
    int64_t gi = 0, so = 0, eo = 0;
    for (int64_t b = 0; b < n_cta; ++b) {
      cta_slot0[b] = so;
      cta_e0[b] = eo;
      const CtaPlan& P = plans[b];
      int64_t ng = P.gstart.empty() ? 0 : (int64_t)P.gstart.size() - 1;
      for (int64_t g = 0; g < ng; ++g) {
        so += P.gstart[g + 1] - P.gstart[g];
        F->group_map_ptr[gi + g + 1] = so;
      }
      for (int64_t w = 0; w < warps; ++w)
        for (int64_t g = 0; g < ng; ++g) {
          F->slab_off[(gi + g) * warps + w] = eo;
          F->slab_width[(gi + g) * warps + w] = P.width[g * warps + w];
          eo += (int64_t)P.width[g * warps + w] * rows_per_warp;
        }
      gi += ng;
    }
    cta_e0[n_cta] = eo;
  }

  plog.lap("B");
  // ---- phase C: fill maps and slabs ----------------------------------------
  const double scale = std::ldexp(1.0, value_scale_exp);
  std::vector<double> worst(n_cta, 0.0);
  std::vector<int64_t> under(n_cta, 0);
  parallel_for(n_cta, n_threads, [&](int64_t b) {
    if (err) return;
    const CtaPlan& P = plans[b];
    const int32_t* keys = key_tables + (int64_t)cta_table[b] * n_cols;
    const int64_t g0 = F->cta_group_ptr[b];
    std::memset(F->slots.get() + cta_e0[b], 0, (size_t)(cta_e0[b + 1] - cta_e0[b]) * 2);
    std::memset(F->values.get() + cta_e0[b] * vbytes, 0,
                (size_t)(cta_e0[b + 1] - cta_e0[b]) * vbytes);
    for (size_t i = 0; i < P.foot.size(); ++i) F->group_map[cta_slot0[b] + i] = P.foot[i].col;
    const int64_t ng = P.gstart.empty() ? 0 : (int64_t)P.gstart.size() - 1;
    std::vector<std::pair<int32_t, int64_t>> ent;   // (key, csr position)
    static thread_local std::vector<int32_t> slot_of, group_of;
    if ((int64_t)slot_of.size() < n_cols) { slot_of.assign(n_cols, 0); group_of.assign(n_cols, 0); }
    for (int64_t g = 0; g < ng; ++g)
      for (int64_t p = P.gstart[g]; p < P.gstart[g + 1]; ++p) {
        group_of[P.foot[p].col] = (int32_t)g;
        slot_of[P.foot[p].col] = (int32_t)(p - P.gstart[g]);
      }
    double wmax = 0.0;
    int64_t nunder = 0;
    // entries of every (group, thread-row) in (key, CSR position) order, in
    // one flat buffer: a row's key-sorted entries visit the groups in order,
    // so (group, row) lists are contiguous spans
    struct Ent { int32_t slot; int64_t j; };
    struct Span { const Ent* p; int64_t n; size_t size() const { return (size_t)n; }
                  const Ent& operator[](size_t i) const { return p[i]; } };
    std::vector<Ent> flat;
    std::vector<int64_t> gofs((size_t)(ng + 1) * rows_per_cta, 0);
    flat.reserve(1024);
    for (int64_t t = 0; t < rows_per_cta; ++t) {
      int32_t r = cta_rows[b * rows_per_cta + t];
      const int64_t row0 = (int64_t)flat.size();
      if (r >= 0) {
        ent.clear();
        bool sorted = true;
        for (int64_t j = indptr[r]; j < indptr[r + 1]; ++j) {
          const int32_t k = keys[indices[j]];
          if (!ent.empty() && k < ent.back().first) sorted = false;
          ent.push_back({k, j});
        }
        if (!sorted)
          std::stable_sort(ent.begin(), ent.end(),
                           [](const std::pair<int32_t, int64_t>& a,
                              const std::pair<int32_t, int64_t>& c) { return a.first < c.first; });
        for (auto& e : ent) flat.push_back({slot_of[indices[e.second]], e.second});
      }
      // gofs[t*(ng+1)+g] = start of group g's span inside the flat buffer
      int64_t at = row0;
      const int64_t end = (int64_t)flat.size();
      for (int64_t g = 0; g <= ng; ++g) {
        while (g < ng && at < end && group_of[indices[flat[at].j]] < g) ++at;
        gofs[(size_t)t * (ng + 1) + g] = g < ng ? at : end;
      }
    }
    auto per_span = [&](int64_t g, int64_t t) {
      const int64_t a = gofs[(size_t)t * (ng + 1) + g], e = gofs[(size_t)t * (ng + 1) + g + 1];
      return Span{flat.data() + a, e - a};
    };
    auto write = [&](int64_t gg, int64_t w, int64_t rin, int64_t n, int32_t slot, int64_t j) {
      int64_t at = F->slab_off[gg * warps + w] + ((n >> 2) * rows_per_warp + rin) * 4 + (n & 3);
      F->slots[at] = (uint16_t)slot;
      if (j < 0) return;                       // padding: value stays 0
      double v = values[j] * scale;           // exact power-of-two rescale
      double back;
      uint8_t* dst = F->values.get() + at * vbytes;
      if (precision == XCT_DOUBLE) {
        std::memcpy(dst, &v, 8);
        back = v;
      } else if (precision == XCT_SINGLE) {
        float f = (float)v;
        std::memcpy(dst, &f, 4);
        back = (double)f;
      } else {
        uint16_t h = f64_to_f16(v);
        std::memcpy(dst, &h, 2);
        back = f16_to_f64(h);
      }
      if (v != 0.0) {
        if (back == 0.0) ++nunder;
        double rel = std::fabs(back - v) / std::fabs(v);
        if (rel > wmax) wmax = rel;
      }
    };
    QuarterScheduler qs;
    std::vector<std::pair<int32_t, int32_t>> qedges;
    std::vector<int32_t> step_slot;
    for (int64_t g = 0; g < ng; ++g) {
      const int64_t gg = g0 + g;
      for (int64_t w = 0; w < warps; ++w) {
        const int64_t width = F->slab_width[gg * warps + w];
        if (!bank.on()) {
          for (int64_t rin = 0; rin < rows_per_warp; ++rin) {
            const Span L = per_span(g, w * rows_per_warp + rin);
            for (size_t n = 0; n < L.size(); ++n) write(gg, w, rin, (int64_t)n, L[n].slot, L[n].j);
          }
          continue;
        }
        for (int64_t q0 = 0; q0 < rows_per_warp; q0 += bank.rq) {
          step_slot.assign(width, -1);
          std::vector<std::pair<int64_t, int32_t>> owner;   // edge -> (rin, list index)
          qedges.clear();
          for (int64_t rr = 0; rr < bank.rq; ++rr) {
            const Span L = per_span(g, w * rows_per_warp + q0 + rr);
            for (size_t n = 0; n < L.size(); ++n) {
              qedges.push_back({(int32_t)rr, L[n].slot});
              owner.push_back({q0 + rr, (int32_t)n});
            }
          }
          if (!qs.run((int)bank.rq, (int)width, qedges, bank, compress)) {
            std::lock_guard<std::mutex> lk(err_mu);
            err = XCT_EINVAL;
            err_msg = "format_build: bank schedule exceeded the slab width";
            return;
          }
          std::vector<char> used((size_t)bank.rq * width, 0);
          for (size_t e = 0; e < owner.size(); ++e) {
            const int64_t rin = owner[e].first;
            const Ent& E = per_span(g, w * rows_per_warp + rin)[owner[e].second];
            const int64_t n = qs.step_of[e];
            write(gg, w, rin, n, E.slot, E.j);
            used[(size_t)(rin - q0) * width + n] = 1;
            if (step_slot[n] < 0) step_slot[n] = E.slot;
          }
          // idle lanes re-read a slot another lane of the quarter reads in the
          // same step (broadcast, no extra bank traffic)
          for (int64_t rr = 0; rr < bank.rq; ++rr)
            for (int64_t n = 0; n < width; ++n)
              if (!used[(size_t)rr * width + n] && step_slot[n] > 0)
                write(gg, w, q0 + rr, n, step_slot[n], -1);
        }
      }
    }
    worst[b] = wmax;
    under[b] = nunder;
  });
  if (err) {
    delete F;
    return xct::fail(err, err_msg);
  }

  plog.lap("C");
  F->info.n_cta = n_cta;
  F->info.rows_per_cta = rows_per_cta;
  F->info.rows_per_warp = rows_per_warp;
  F->info.warps_per_cta = warps;
  F->info.n_groups = n_groups;
  F->info.n_slots = n_slots;
  F->info.n_padded = n_padded;
  F->info.nnz = indptr[n_rows] - indptr[0];
  F->info.max_group_slots = max_gs;
  F->info.value_bytes = vbytes;
  F->info.row_group = 1;
  double wm = 0.0;
  int64_t un = 0;
  for (int64_t b = 0; b < n_cta; ++b) { wm = std::max(wm, worst[b]); un += under[b]; }
  F->info.max_rel_quant_error = wm;
  F->info.underflow_count = un;
  *out = F;
  return XCT_OK;
}

extern "C" int xct_format_get_info(const xct_format* f, xct_format_info* info) {
  if (!f || !info) return xct::fail(XCT_EINVAL, "format_get_info: null argument");
  *info = f->info;
  return XCT_OK;
}

extern "C" int xct_format_export(const xct_format* f, int32_t* cta_group_ptr,
                                 int64_t* group_map_ptr, int32_t* group_map, int64_t* slab_off,
                                 int32_t* slab_width, uint16_t* slots, void* values) {
  if (!f) return xct::fail(XCT_EINVAL, "format_export: null handle");
  auto cp = [](void* dst, const void* src, size_t n) { if (dst && n) std::memcpy(dst, src, n); };
  cp(cta_group_ptr, f->cta_group_ptr.data(), f->cta_group_ptr.size() * 4);
  cp(group_map_ptr, f->group_map_ptr.data(), f->group_map_ptr.size() * 8);
  cp(group_map, f->group_map.data(), f->group_map.size() * 4);
  cp(slab_off, f->slab_off.data(), f->slab_off.size() * 8);
  cp(slab_width, f->slab_width.data(), f->slab_width.size() * 4);
  // the slabs are GBs: copy them in parallel blocks
  const int T = (int)std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
  auto pcp = [&](void* dst, const void* src, size_t n) {
    if (!dst || !n) return;
    const size_t blk = std::max<size_t>(1 << 22, (n + T - 1) / T);
    const int64_t nb = (int64_t)((n + blk - 1) / blk);
    parallel_for(nb, T, [&](int64_t i) {
      const size_t a = (size_t)i * blk, e = std::min(n, a + blk);
      std::memcpy((uint8_t*)dst + a, (const uint8_t*)src + a, e - a);
    });
  };
  pcp(slots, f->slots.get(), (size_t)f->n_padded * 2);
  pcp(values, f->values.get(), (size_t)f->n_padded * f->vbytes * f->row_group);
  return XCT_OK;
}

extern "C" void xct_format_free(xct_format* f) { delete f; }

extern "C" int xct_csr_transpose(int64_t n_rows, int64_t n_cols, const int64_t* indptr,
                                 const int32_t* indices, const double* values,
                                 int64_t* t_indptr, int32_t* t_indices, double* t_values,
                                 int n_threads) {
  if (!indptr || !t_indptr) return xct::fail(XCT_EINVAL, "csr_transpose: null argument");
  // Parallel stable counting transpose: rows are split into T contiguous
  // blocks; block t's entries of column c go after those of blocks < t, and
  // inside a block rows are visited in order, so every column lists its rows
  // ascending (and repeated (row, col) pairs in CSR order) -- exactly the
  // stable argsort of src/matrixstore.py:189-201.
  int T = n_threads < 1 ? 1 : n_threads;
  if ((int64_t)T * n_cols > (int64_t)1 << 31) T = std::max<int64_t>(1, ((int64_t)1 << 31) / std::max<int64_t>(n_cols, 1));
  if (T > n_rows) T = (int)std::max<int64_t>(1, n_rows);
  std::vector<int64_t> rb(T + 1);
  for (int t = 0; t <= T; ++t) rb[t] = n_rows * t / T;
  std::vector<int32_t> cnt((size_t)T * n_cols, 0);
  std::atomic<int> bad{0};
  parallel_for(T, T, [&](int64_t t) {
    int32_t* c = cnt.data() + (size_t)t * n_cols;
    for (int64_t j = indptr[rb[t]]; j < indptr[rb[t + 1]]; ++j) {
      const int32_t col = indices[j];
      if (col < 0 || col >= n_cols) { bad = 1; return; }
      ++c[col];
    }
  });
  if (bad) return xct::fail(XCT_EINVAL, "csr_transpose: column out of range");
  // column totals -> t_indptr; per-block starting offsets in place
  t_indptr[0] = 0;
  for (int64_t c = 0; c < n_cols; ++c) {
    int64_t run = t_indptr[c];
    for (int t = 0; t < T; ++t) {
      int32_t& x = cnt[(size_t)t * n_cols + c];
      const int64_t k = x;
      x = (int32_t)(run - t_indptr[c]);      // offset inside column c
      run += k;
    }
    t_indptr[c + 1] = run;
  }
  parallel_for(T, T, [&](int64_t t) {
    int32_t* c = cnt.data() + (size_t)t * n_cols;
    for (int64_t r = rb[t]; r < rb[t + 1]; ++r)
      for (int64_t j = indptr[r]; j < indptr[r + 1]; ++j) {
        const int32_t col = indices[j];
        const int64_t at = t_indptr[col] + c[col]++;
        t_indices[at] = (int32_t)r;
        t_values[at] = values[j];
      }
  });
  return XCT_OK;
}
