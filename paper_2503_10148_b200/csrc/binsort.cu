// a2 — sss_bin_sort: depth-ordered per-bin component lists.
//
// Definition (R8, R9; north_star "bins components into 16x16
// tiles with a depth-keyed sort"): the list of bin b holds every visible
// component whose tile rect overlaps b, ordered by (fp32 camera depth,
// component index).
//
// B200 design — two stages instead of one 64-bit key sort over all M
// instances:
//   1. a stable LSD radix sort (4 x 8-bit digits) of the N per-view depth keys
//      (keys of culled components are 0xFFFFFFFF and sort last, so the first
//      n_vis sorted entries are the visible components); each pass reorders
//      its 4096-key tile by digit in shared memory so the global stores leave
//      as per-digit runs (a depth mode reading the projection directly,
//      dropping culled keys and skipping constant digits, measured slower at
//      config 5: no digit is constant there and the extra operand logic cost
//      occupancy);
//   2. a stable counting scatter of the instances by bin, generated on the fly
//      from the depth-sorted components: per-chunk bin histograms (shared
//      memory), a column scan over chunks, a scan over bins, then a scatter in
//      which a warp flattens the bin rects of 32 components into instances
//      and writes 32 of them per step (balanced whatever the rect sizes); the
//      slot of (component, bin) is the warp's running count plus the number
//      of lower components covering the bin — a popcount of per-column and
//      per-row ballots — so bins receive their entries in depth order without
//      ever materialising 64-bit keys or serialising lanes.  A chunk's ids
//      are staged in shared memory and stored bin run by bin run.
// Every instance is written exactly once (4 B id, +8 B key if requested); the
// radix passes touch only N keys per view.  All views are processed by the
// same launches (grid.y = view).
//
// Truncated lists (max_per_bin > 0, see sss.h): a bin keeps only its first
// max_per_bin entries.  The chunk histograms give every (chunk, bin) its
// index range in the bin's full list, so a chunk's instance is kept iff its
// index is below the cap; a chunk with nothing to keep returns at once, and a
// component whose rect meets only bins already full before the chunk skips
// the walk (its instances could only land in full bins, so the slots of the
// open bins are unchanged).  The instance at index cap - 1 of a truncated
// bin records resume[b] = its sorted position + 1 for the raster.
#include <algorithm>

#include "radix.cuh"

namespace sss {
namespace {

#ifndef SSS_SCATTER_THREADS
#define SSS_SCATTER_THREADS 256
#endif
constexpr int kScatterThreads = SSS_SCATTER_THREADS;  // chunk_hist and scatter CTAs
#ifndef SSS_SCATTER_RUN_LANES
#define SSS_SCATTER_RUN_LANES 8
#endif
constexpr int kRunLanes = SSS_SCATTER_RUN_LANES;  // lanes storing one bin's staged run
constexpr int kScatterWarps = kScatterThreads / 32;

struct BinGeom {
  int tiles_x, tiles_y, shift, bins_x, bins_y, n_bins, bits;  // bits: ceil(log2(n_bins))
};

inline BinGeom bin_geom(const sss_camera& c, int shift) {
  BinGeom g;
  g.tiles_x = div_up(c.width, kTile);
  g.tiles_y = div_up(c.height, kTile);
  g.shift = shift;
  g.bins_x = div_up(g.tiles_x, 1 << shift);
  g.bins_y = div_up(g.tiles_y, 1 << shift);
  g.n_bins = g.bins_x * g.bins_y;
  g.bits = 1;
  while ((1 << g.bits) < g.n_bins) ++g.bits;
  return g;
}

#ifndef SSS_CHUNK
#define SSS_CHUNK 2048  // 256 components per warp (per-warp bin counts as u16); the per-bin fixed costs of a chunk CTA amortise over twice the components of 1024
#endif
constexpr int kChunk = SSS_CHUNK;  // depth-sorted components per histogram / scatter CTA
constexpr size_t kScatterSmemMax = 225 * 1024;  // dynamic shared memory of a scatter CTA
#ifndef SSS_SCATTER_STAGE_MAX
#define SSS_SCATTER_STAGE_MAX 16384
#endif
constexpr int64_t kScatterStageMax = SSS_SCATTER_STAGE_MAX;  // staged ids per chunk (64 KB)

struct WsLayout {
  size_t keys_a, keys_b, vals_a, vals_b, sorted, n_vis, radix_hist, chunk_hist, warp_hist, bin_total, bin_start,
      bin_cap, chunk_kept, total;
  int tiles_per_view, n_chunks, chunk;
};

inline size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

WsLayout ws_layout(int64_t n, int V, const BinGeom& g) {
  WsLayout L;
  L.tiles_per_view = div_up(n, kRadixTile);
  L.chunk = kChunk;
  L.n_chunks = div_up(n, L.chunk);
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += align_up(bytes); return o; };
  const size_t nv = (size_t)n * V;
  L.keys_a = take(nv * 4);
  L.keys_b = take(nv * 4);
  L.vals_a = take(nv * 4);
  L.vals_b = take(nv * 4);
  L.sorted = take(nv * 4);  // used when the caller passes no sorted array
  L.n_vis = take((size_t)V * 4);
  L.radix_hist = take(radix_ws_words(L.tiles_per_view, V) * 4);
  L.chunk_hist = take((size_t)V * L.n_chunks * (size_t)g.n_bins * 4);
  L.warp_hist = take((size_t)V * L.n_chunks * kScatterWarps * 2 * (size_t)g.n_bins);  // 8 x u16 per (chunk, bin)
  L.bin_total = take((size_t)V * g.n_bins * 4);
  L.bin_start = take((size_t)V * g.n_bins * 4);
  L.bin_cap = take((size_t)V * g.n_bins * 4);
  L.chunk_kept = take((size_t)V * L.n_chunks * ((g.n_bins + 31) / 32) * 4);
  L.total = off;
  return L;
}

// ------------------------------------------------------------- depth keys
__global__ void keys_init_kernel(const float* __restrict__ depth, const short4* __restrict__ rect,
                                 int64_t n, uint32_t* __restrict__ keys, int32_t* __restrict__ vals,
                                 int32_t* __restrict__ n_vis) {
  const int v = blockIdx.y;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool vis = false;
  if (i < n) {
    const short4 r = rect[(int64_t)v * n + i];
    vis = r.x <= r.z;
    keys[(int64_t)v * n + i] = vis ? __float_as_uint(depth[(int64_t)v * n + i]) : 0xFFFFFFFFu;
    vals[(int64_t)v * n + i] = (int32_t)i;
  }
  // one atomic per block (per-warp atomics on one address serialise)
  __shared__ int32_t wsum[8];
  const unsigned b = __ballot_sync(0xffffffffu, vis);
  if (lane_id() == 0) wsum[threadIdx.x >> 5] = __popc(b);
  __syncthreads();
  if (threadIdx.x == 0) {
    int32_t s = 0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) s += wsum[k];
    if (s) atomicAdd(&n_vis[v], s);
  }
}

// The same with four consecutive components per thread and 16-byte accesses
// (n % 4 == 0: every view's segment starts 16-byte aligned).
__global__ void keys_init4_kernel(const float4* __restrict__ depth, const int4* __restrict__ rect,
                                  int64_t n, uint4* __restrict__ keys, int4* __restrict__ vals,
                                  int32_t* __restrict__ n_vis) {
  const int v = blockIdx.y;
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // quad index in the view
  const int64_t nq = n >> 2;
  int cnt = 0;
  if (q < nq) {
    const int64_t o = (int64_t)v * nq + q;
    const int4 r01 = rect[2 * o], r23 = rect[2 * o + 1];  // two short4 per int4
    const float4 d = depth[o];
    // short4 {x0, y0, x1, y1}: visible iff x0 <= x1 (low halves of words 0 and 1)
    const bool v0 = (short)(r01.x & 0xffff) <= (short)(r01.y & 0xffff);
    const bool v1 = (short)(r01.z & 0xffff) <= (short)(r01.w & 0xffff);
    const bool v2 = (short)(r23.x & 0xffff) <= (short)(r23.y & 0xffff);
    const bool v3 = (short)(r23.z & 0xffff) <= (short)(r23.w & 0xffff);
    keys[o] = make_uint4(v0 ? __float_as_uint(d.x) : 0xFFFFFFFFu, v1 ? __float_as_uint(d.y) : 0xFFFFFFFFu,
                         v2 ? __float_as_uint(d.z) : 0xFFFFFFFFu, v3 ? __float_as_uint(d.w) : 0xFFFFFFFFu);
    const int32_t i0 = (int32_t)(4 * q);
    vals[o] = make_int4(i0, i0 + 1, i0 + 2, i0 + 3);
    cnt = (int)v0 + (int)v1 + (int)v2 + (int)v3;
  }
  __shared__ int32_t wsum[8];
  int c = cnt;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) c += __shfl_xor_sync(0xffffffffu, c, off);
  if (lane_id() == 0) wsum[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int32_t s = 0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) s += wsum[k];
    if (s) atomicAdd(&n_vis[v], s);
  }
}

// ------------------------------------------------------- bin histograms
__device__ __forceinline__ void bin_rect(short4 r, int shift, int& bx0, int& by0, int& bx1, int& by1) {
  bx0 = r.x >> shift; by0 = r.y >> shift; bx1 = r.z >> shift; by1 = r.w >> shift;
}

// Per (chunk, view): bin counts of the chunk's instances, per warp of the
// scatter's partition (warp w owns kChunk/8 consecutive depth-sorted
// components).  Writes the chunk totals (u32, for the scans) and the per-warp
// counts (u16: a warp's 256 components hit a bin at most 256 times; the 8
// warps' counts of a bin packed in one 16-byte word), so the scatter needs no
// counting pass of its own.  Each component adds its rect of bins as a 2-D
// difference (<= 4 shared atomics instead of one per instance: 9.2 per
// component at config 5), and the per-warp grids are prefix-summed by rows
// and columns before the write-out (bin_sort -0.6 ms per config-5 step).
__global__ void __launch_bounds__(kScatterThreads) chunk_hist_kernel(const int32_t* __restrict__ sorted_ids,
                                                         const int32_t* __restrict__ n_vis,
                                                         const short4* __restrict__ rect, int64_t n,
                                                         int chunk, int n_chunks, BinGeom g,
                                                         uint32_t* __restrict__ chunk_hist,
                                                         uint8_t* __restrict__ warp_hist) {
  extern __shared__ uint32_t hs[];  // [8][n_bins]
  const int v = blockIdx.y, c = blockIdx.x;
  const int nb = g.n_bins;
  for (int k = threadIdx.x; k < kScatterWarps * nb; k += blockDim.x) hs[k] = 0;
  __syncthreads();
  const int w = threadIdx.x >> 5;
  const int per_warp = chunk / kScatterWarps;
  const int64_t wlo = (int64_t)c * chunk + (int64_t)w * per_warp;
  const int64_t whi = min(wlo + per_warp, (int64_t)n_vis[v]);
  uint32_t* my = hs + (size_t)w * nb;
  for (int64_t j = wlo + lane_id(); j < whi; j += 32) {
    const int id = sorted_ids[(int64_t)v * n + j];
    int bx0, by0, bx1, by1;
    bin_rect(rect[(int64_t)v * n + id], g.shift, bx0, by0, bx1, by1);
    if (bx0 > bx1 || by0 > by1) continue;
    // the rect's bins as a 2-D difference (<= 4 corner updates, mod 2^32)
    const bool xe = bx1 + 1 < g.bins_x, ye = by1 + 1 < g.bins_y;
    atomicAdd(&my[by0 * g.bins_x + bx0], 1u);
    if (xe) atomicAdd(&my[by0 * g.bins_x + bx1 + 1], 0xFFFFFFFFu);
    if (ye) atomicAdd(&my[(by1 + 1) * g.bins_x + bx0], 0xFFFFFFFFu);
    if (xe && ye) atomicAdd(&my[(by1 + 1) * g.bins_x + bx1 + 1], 1u);
  }
  __syncthreads();
  // 2-D prefix sums of every warp's difference grid: rows, then columns
  for (int r = threadIdx.x; r < kScatterWarps * g.bins_y; r += blockDim.x) {
    uint32_t* row = hs + (size_t)(r / g.bins_y) * nb + (size_t)(r % g.bins_y) * g.bins_x;
    uint32_t acc = 0;
    for (int x = 0; x < g.bins_x; ++x) row[x] = acc += row[x];
  }
  __syncthreads();
  for (int cidx = threadIdx.x; cidx < kScatterWarps * g.bins_x; cidx += blockDim.x) {
    uint32_t* col = hs + (size_t)(cidx / g.bins_x) * nb + (cidx % g.bins_x);
    uint32_t acc = 0;
    for (int y = 0; y < g.bins_y; ++y) col[(size_t)y * g.bins_x] = acc += col[(size_t)y * g.bins_x];
  }
  __syncthreads();
  uint32_t* out = chunk_hist + ((size_t)v * n_chunks + c) * nb;
  uint4* wout = reinterpret_cast<uint4*>(warp_hist) + ((size_t)v * n_chunks + c) * nb;
  static_assert(kScatterWarps == 8, "8 per-warp u16 counts per 16-byte word");
  static_assert(kChunk / kScatterWarps <= 65535, "per-warp counts fit u16");
  for (int b = threadIdx.x; b < nb; b += blockDim.x) {
    uint32_t t = 0, pk[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t lo = hs[(size_t)(2 * q) * nb + b], hi = hs[(size_t)(2 * q + 1) * nb + b];
      pk[q] = lo | (hi << 16);
      t += lo + hi;
    }
    wout[b] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
    out[b] = t;
  }
}

// per (view, bin): exclusive scan over chunks in place; bin totals.  CTA =
// 32 bins (lane = bin, coalesced rows) x kColWarps warps, each warp a
// contiguous range of chunks: range sums, a prefix over warps, then the
// running write (32 warps: the short serial chains of loads per warp keep
// this latency-bound pass at 1.4% of bin_sort less than with 8).
#ifndef SSS_COLSCAN_WARPS
#define SSS_COLSCAN_WARPS 32
#endif
constexpr int kColWarps = SSS_COLSCAN_WARPS;  // warps splitting the chunk range of 32 bins
// Per-bin cap: the static max_per_bin (0xFFFFFFFF = none), or, with `used`
// (the previous sss_render_fwd's per-bin consumption), 1.25 used + 256 capped
// by it; used < 0 or >= 2^30 (unknown, or a tile with a pixel still live at
// the end of its list) keeps the static cap.
__device__ __forceinline__ uint32_t bin_cap_of(uint32_t static_cap, const int32_t* used, size_t k) {
  if (!used) return static_cap;
  const int32_t u = used[k];
  if (u < 0 || u >= (1 << 30)) return static_cap;
#ifndef SSS_CAP_NUM
#define SSS_CAP_NUM 5  // cap = used * SSS_CAP_NUM / 4 + SSS_CAP_ADD: 1.25 used + 256
#endif                 // (2 used + 1024 kept 1.6 M instances per config-5 view, this
#ifndef SSS_CAP_ADD    // 1.05 M: bin_sort -1.3 ms; no bin read the tail in 30 training
#define SSS_CAP_ADD 256u  // steps, tools/cap_drift.py)
#endif
  return min(static_cap, (uint32_t)(((uint64_t)u * SSS_CAP_NUM) >> 2) + SSS_CAP_ADD);
}

// The column scan also applies the caps: each (chunk, bin) keeps
// clamp(cap_b - start, 0, count) instances; the kept total of every chunk
// (warp sums over its 32 bins, one atomic per warp and chunk) lets the
// scatter skip chunks that keep nothing at once.  Writes bcap.
__global__ void __launch_bounds__(32 * kColWarps) column_scan_kernel(uint32_t* __restrict__ chunk_hist, int n_chunks,
                                                          int n_bins, uint32_t* __restrict__ bin_total,
                                                          uint32_t static_cap, const int32_t* __restrict__ used,
                                                          uint32_t* __restrict__ bcap,
                                                          uint32_t* __restrict__ chunk_kept) {
  __shared__ uint32_t wsum[kColWarps][32];
  const int v = blockIdx.y;
  const int w = threadIdx.x >> 5, lane = lane_id();
  const int b = blockIdx.x * 32 + lane;
  const bool ok = b < n_bins;
  const int per = (n_chunks + kColWarps - 1) / kColWarps;
  const int c0 = min(w * per, n_chunks), c1 = min(c0 + per, n_chunks);
  uint32_t* col = chunk_hist + (size_t)v * n_chunks * n_bins + (ok ? b : 0);
  const uint32_t cap = ok ? bin_cap_of(static_cap, used, (size_t)v * n_bins + b) : 0u;
  uint32_t s = 0;
  if (ok) {
    int c = c0;
    for (; c + 4 <= c1; c += 4)
      s += col[(size_t)c * n_bins] + col[(size_t)(c + 1) * n_bins] + col[(size_t)(c + 2) * n_bins] +
           col[(size_t)(c + 3) * n_bins];
    for (; c < c1; ++c) s += col[(size_t)c * n_bins];
  }
  wsum[w][lane] = s;
  __syncthreads();
  uint32_t run = 0, tot = 0;
#pragma unroll
  for (int k = 0; k < kColWarps; ++k) {
    run += k < w ? wsum[k][lane] : 0u;
    tot += wsum[k][lane];
  }
  // per (chunk, group of 32 bins): the kept count, summed by the scatter
  // (no atomics); nullptr when nothing is capped
  const int n_grp = gridDim.x;
  uint32_t* ck = chunk_kept ? chunk_kept + (size_t)v * n_chunks * n_grp + blockIdx.x : nullptr;
  int c = c0;
  for (; c + 4 <= c1; c += 4) {  // warp-uniform range; four loads in flight
    uint32_t x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) x[u] = ok ? col[(size_t)(c + u) * n_bins] : 0u;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (ok) col[(size_t)(c + u) * n_bins] = run;
      const uint32_t kept = run >= cap ? 0u : min(x[u], cap - run);
      run += x[u];
      if (ck) {
        const uint32_t ks = __reduce_add_sync(0xffffffffu, kept);
        if (lane == 0) ck[(size_t)(c + u) * n_grp] = ks;
      }
    }
  }
  for (; c < c1; ++c) {
    const uint32_t x = ok ? col[(size_t)c * n_bins] : 0u;
    if (ok) col[(size_t)c * n_bins] = run;
    const uint32_t kept = run >= cap ? 0u : min(x, cap - run);
    run += x;
    if (ck) {
      const uint32_t ks = __reduce_add_sync(0xffffffffu, kept);
      if (lane == 0) ck[(size_t)c * n_grp] = ks;
    }
  }
  if (w == 0 && ok) {
    bin_total[(size_t)v * n_bins + b] = tot;
    bcap[(size_t)v * n_bins + b] = cap;
  }
}

// per view: exclusive scan over bins of the materialised counts
// min(total_b, cap) -> bin_start, ranges, totals, overflow; resume = n_vis
// for complete lists (the scatter writes it for truncated ones)
// (bcap from the column scan; `used` is reset to 0 for the forward that follows)
__global__ void __launch_bounds__(1024) bin_scan_kernel(const uint32_t* __restrict__ bin_total, int n_bins,
                                                        int64_t capacity, int32_t* __restrict__ used,
                                                        const uint32_t* __restrict__ bcap,
                                                        uint32_t* __restrict__ bin_start,
                                                        int32_t* __restrict__ ranges,
                                                        int64_t* __restrict__ totals,
                                                        int32_t* __restrict__ overflow,
                                                        const int32_t* __restrict__ n_vis,
                                                        int32_t* __restrict__ resume) {
  __shared__ unsigned long long part[1024];
  __shared__ int over;
  const int v = blockIdx.x, t = threadIdx.x;
  const uint32_t* bt = bin_total + (size_t)v * n_bins;
  const int per = (n_bins + 1023) / 1024;
  const int lo = t * per, hi = min(lo + per, n_bins);
  unsigned long long s = 0;
  for (int k = lo; k < hi; ++k) {
    s += min(bt[k], bcap[(size_t)v * n_bins + k]);
    if (used) used[(size_t)v * n_bins + k] = 0;
  }
  part[t] = s;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {
    unsigned long long x = t >= off ? part[t - off] : 0ull;
    __syncthreads();
    part[t] += x;
    __syncthreads();
  }
  const unsigned long long total = part[1023];
  if (t == 0) {
    totals[v] = (int64_t)total;
    over = total > (unsigned long long)capacity;
    if (over) atomicExch(overflow, 1);
  }
  __syncthreads();
  unsigned long long run = part[t] - s;
  for (int k = lo; k < hi; ++k) {
    const uint32_t full = bt[k];
    const uint32_t cap = bcap[(size_t)v * n_bins + k];
    const uint32_t x = min(full, cap);
    if (resume && full <= cap) resume[(size_t)v * n_bins + k] = n_vis[v];
    bin_start[(size_t)v * n_bins + k] = (uint32_t)run;
    ranges[((size_t)v * n_bins + k) * 2 + 0] = over ? 0 : (int32_t)run;
    ranges[((size_t)v * n_bins + k) * 2 + 1] = over ? 0 : (int32_t)(run + x);
    run += x;
  }
}

// Per-warp scratch of the scatter walk (shared memory).
struct alignas(16) WalkRec {  // one of the step's (compacted) components
  int32_t excl;               // first instance index of the component in the step
  int32_t id;
  uint32_t packed;            // bx0 | by0 << 10 | (width - 1) << 20 (bins)
  uint32_t magic;             // ceil(2^31 / width): floor(k / w) = umulhi(2k, magic) for k, w < 2^15
};
struct alignas(16) WalkScratch {
  WalkRec rec[32];
  int4 stage[32];     // {bx0 | by0 << 16, bx1 | by1 << 16, id, depth bits}
  uint32_t dbits[32];
  int32_t spos[32];   // position of the rank's component in the depth-sorted order
};

// Truncation state of one scatter CTA (chunk): see the file header.
struct TruncCtx {
  const uint32_t* cap;                // [n_bins] per-bin caps (UINT32_MAX: none)
  const uint64_t* openrow;            // smem [bins_y]: bit bx of row by = bin (bx, by) keeps something here
  const uint32_t* ch;                 // the chunk's index of each bin in its full list (global)
  const uint32_t* bs;                 // materialised start of each bin (global)
  const uint32_t* btot;               // full list length of each bin (global)
  int32_t* resume;                    // [n_bins] of this view, or nullptr
};

// Clips a bin rect to the bounding box of its bins still open in this chunk
// (per bin row, a 64-bit mask of the open bins); false if none is open.  An
// open bin of the rect stays inside the clipped rect, so the slots of open
// bins (counts of lower components covering them) are unchanged; instances
// in full bins are dropped anyway.  Views more than 64 bins wide: no clip.
__device__ __forceinline__ bool rect_clip_open(const TruncCtx& tc, const BinGeom& g, int& bx0, int& by0, int& bx1,
                                               int& by1) {
  if (g.bins_x > 64) return true;
  const uint64_t xm = (~0ull >> (63 - (bx1 - bx0))) << bx0;
  uint64_t hit = 0;
  int y0 = 1 << 20, y1 = -1;
  for (int by = by0; by <= by1; ++by) {
    const uint64_t m = tc.openrow[by] & xm;
    if (m) {
      y0 = min(y0, by);
      y1 = by;
      hit |= m;
    }
  }
  if (!hit) return false;
  by0 = y0;
  by1 = y1;
  bx0 = __ffsll((long long)hit) - 1;
  bx1 = 63 - __clzll((long long)hit);
  return true;
}

template <bool STAGED, bool TRUNC>
__device__ __forceinline__ void warp_walk(const int32_t* __restrict__ sid, const short4* __restrict__ rv,
                                          const float* __restrict__ dv, int64_t wlo, int64_t whi,
                                          const BinGeom& g, uint32_t* wbase, uint32_t* colmask,
                                          uint32_t* rowmask, WalkScratch& S, int32_t* __restrict__ dst,
                                          uint64_t* __restrict__ kv, const uint32_t* soff,
                                          const TruncCtx& tc) {
  const int lane = lane_id();
  const unsigned full = 0xffffffffu;
  const unsigned lt = (1u << lane) - 1u;
  // the warp's components in groups of 4 x 32: every id, then every rect,
  // loaded up front (two dependent round trips per group instead of two per
  // step: the walk of a chunk that keeps little is latency-bound)
  constexpr int kWalkSteps = kChunk / kScatterWarps / 32;
  constexpr int kGroup = 4;
  static_assert(kWalkSteps % kGroup == 0, "whole preload groups");
  for (int g0 = 0; g0 < kWalkSteps; g0 += kGroup) {
  if (wlo + g0 * 32 >= whi) break;
  int idp[kGroup];
  short4 rp[kGroup];
#pragma unroll
  for (int st = 0; st < kGroup; ++st) {
    const int64_t j = wlo + (g0 + st) * 32 + lane;
    idp[st] = j < whi ? sid[j] : -1;
  }
#pragma unroll
  for (int st = 0; st < kGroup; ++st) rp[st] = idp[st] >= 0 ? rv[idp[st]] : make_short4(1, 1, 0, 0);
#pragma unroll
  for (int st = 0; st < kGroup; ++st) {
    const int64_t j0 = wlo + (g0 + st) * 32;
    if (j0 >= whi) break;
    const int id0 = idp[st];
    const short4 r0 = rp[st];
    const bool valid = j0 + lane < whi;
    {
      int bx0 = r0.x >> g.shift, by0 = r0.y >> g.shift;
      int bx1 = r0.z >> g.shift, by1 = r0.w >> g.shift;
      bool ne = valid && bx0 <= bx1 && by0 <= by1;
      if (TRUNC && ne) ne = rect_clip_open(tc, g, bx0, by0, bx1, by1);
      const unsigned NE = __ballot_sync(full, ne);
      if (ne) {
        S.stage[__popc(NE & lt)] = make_int4(bx0 | (by0 << 16), bx1 | (by1 << 16), id0,
                                             kv ? (int)__float_as_uint(dv[id0]) : 0);
        if (TRUNC) S.spos[__popc(NE & lt)] = (int32_t)(j0 + lane);
      }
      __syncwarp();
      const bool act = lane < __popc(NE);
      int cbx0 = 1, cby0 = 1, cbx1 = 0, cby1 = 0, n_i = 0;
      if (act) {
        const int4 st = S.stage[lane];
        cbx0 = st.x & 0xffff; cby0 = st.x >> 16; cbx1 = st.y & 0xffff; cby1 = st.y >> 16;
        const int wd = cbx1 - cbx0 + 1;
        n_i = wd * (cby1 - cby0 + 1);
        WalkRec rr;
        rr.id = st.z;
        rr.packed = (uint32_t)cbx0 | ((uint32_t)cby0 << 10) | ((uint32_t)(wd - 1) << 20);
        rr.magic = (uint32_t)((0x80000000ull + (uint64_t)wd - 1) / (uint64_t)wd);
        S.rec[lane] = rr;  // excl below
        if (kv) S.dbits[lane] = (uint32_t)st.w;
      }
      int incl = n_i;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(full, incl, o);
        if (lane >= o) incl += t;
      }
      const int T = __shfl_sync(full, incl, 31);
      const int excl = incl - n_i;
      if (act) S.rec[lane].excl = excl;
      // window bit of this rank's first instance: shl.b32 clamps shift
      // counts >= 32 to a zero result, so one shift covers "outside the
      // window" (below it the unsigned difference wraps); inactive ranks
      // start far beyond any window
      const uint32_t start_t = act ? (uint32_t)excl : 0x40000000u;
      // covering ranks per bin column / row, over the step's union rect
      const int ux0 = (int)__reduce_min_sync(full, act ? (unsigned)cbx0 : 0xffffu);
      const int ux1 = (int)__reduce_max_sync(full, act ? (unsigned)cbx1 : 0u);
      const int uy0 = (int)__reduce_min_sync(full, act ? (unsigned)cby0 : 0xffffu);
      const int uy1 = (int)__reduce_max_sync(full, act ? (unsigned)cby1 : 0u);
      for (int x = ux0; x <= ux1; ++x) {
        const unsigned m = __ballot_sync(full, cbx0 <= x && x <= cbx1);
        if (lane == 0) colmask[x] = m;
      }
      for (int y = uy0; y <= uy1; ++y) {
        const unsigned m = __ballot_sync(full, cby0 <= y && y <= cby1);
        if (lane == 0) rowmask[y] = m;
      }
      __syncwarp();
      int base = 0;  // ranks starting before the window
      for (int t0 = 0; t0 < T; t0 += 32) {
        unsigned bit;
        asm("shl.b32 %0, 1, %1;" : "=r"(bit) : "r"(start_t - (uint32_t)t0));
        const unsigned B = __reduce_or_sync(full, bit);
        const int own = base + __popc(B & ((2u << lane) - 1u)) - 1;
        base += __popc(B);
        const int t = t0 + lane;
        int upd_b = -1;
        uint32_t upd_v = 0;
        if (t < T) {
          const WalkRec R = S.rec[own];
          const int k = t - R.excl;
          const int q = (int)__umulhi(2u * (uint32_t)k, R.magic);
          const int wd = (int)(R.packed >> 20) + 1;
          const int bx = (int)(R.packed & 1023u) + (k - q * wd);
          const int by = (int)((R.packed >> 10) & 1023u) + q;
          const int b = by * g.bins_x + bx;
          const unsigned m = colmask[bx] & rowmask[by];
          const uint32_t w0 = wbase[b];
          const uint32_t pos = w0 + __popc(m & ((1u << own) - 1u));
          if (!TRUNC) {
            dst[pos] = R.id;
            if (!STAGED && kv) kv[pos] = ((uint64_t)b << 32) | S.dbits[own];
          } else {
            // kept iff the instance's index in the bin's full list is < cap:
            // staged, the bin's kept run ends at soff[b + 1]; direct, soff[b]
            // holds the bin's global limit bs[b] + cap
            const uint32_t lim = STAGED ? soff[b + 1] : soff[b];
            if (pos < lim) {
              dst[pos] = R.id;
              if (!STAGED && kv) kv[pos] = ((uint64_t)b << 32) | S.dbits[own];
              if (pos + 1 == lim && tc.resume) {  // last kept of this chunk: is it the cap-th entry?
                const uint32_t idx = STAGED ? tc.ch[b] + (pos - soff[b]) : pos - tc.bs[b];
                const uint32_t cb = tc.cap[b];
                if (idx + 1 == cb && tc.btot[b] > cb) tc.resume[b] = S.spos[own] + 1;
              }
            }
          }
          if (((m >> own) >> 1) == 0u) {  // highest covering rank: advance the bin
            upd_b = b;
            upd_v = w0 + __popc(m);
          }
        }
        __syncwarp();
        if (upd_b >= 0) wbase[upd_b] = upd_v;
        __syncwarp();
      }
    }
  }
  }
}

// stable scatter: CTA per (chunk of kChunk depth-sorted components, view);
// warp w owns kChunk/8 consecutive components.  The per-(warp, bin) counts of
// chunk_hist_kernel, prefix-summed over warps, give each warp's first slot in
// the chunk's run of every bin.  The chunk's runs are laid out back to back
// in shared memory (an exclusive scan of the chunk's bin counts), the warps
// write their ids there, and the CTA then stores each run to its global
// segment bs[b] + ch[b] with consecutive lanes on consecutive slots (a
// 4-byte store per instance scattered over the bins' segments leaves
// partial sectors that L2 has to merge or read-modify-write).
__global__ void __launch_bounds__(kScatterThreads) scatter_kernel(
    const int32_t* __restrict__ sorted_ids, const int32_t* __restrict__ n_vis,
    const short4* __restrict__ rect, const float* __restrict__ depth, int64_t n, int n_chunks, BinGeom g,
    const uint32_t* __restrict__ chunk_hist, const uint4* __restrict__ warp_hist,
    const uint32_t* __restrict__ chunk_kept,
    const uint32_t* __restrict__ bin_start, const uint32_t* __restrict__ bin_total,
    const int64_t* __restrict__ totals, int64_t capacity, const uint32_t* __restrict__ bin_cap, int stage_cap,
    int32_t* __restrict__ ids, uint64_t* __restrict__ keys, int32_t* __restrict__ resume) {
  extern __shared__ uint4 sm4[];
  __shared__ uint32_t red[kScatterWarps];
  const int v = blockIdx.y, c = blockIdx.x;
  if (totals[v] > capacity) return;
  const int64_t lo = (int64_t)c * kChunk;
  const int64_t nvis = n_vis[v];
  if (lo >= nvis) return;
  if (chunk_kept) {  // nothing to keep (the column scan's per-group counts)
    const int n_grp = (g.n_bins + 31) / 32;
    const uint32_t* ck = chunk_kept + ((size_t)v * n_chunks + c) * n_grp;
    uint32_t k = 0;
    for (int q = lane_id(); q < n_grp; q += 32) k += ck[q];
    if (__syncthreads_or(k != 0) == 0) return;
  }
  const bool trunc = resume != nullptr;
  const uint32_t* bcv = bin_cap + (size_t)v * g.n_bins;
  const int nb = g.n_bins;
  WalkScratch* scratch = reinterpret_cast<WalkScratch*>(sm4);             // [8]
  uint32_t* wbase = reinterpret_cast<uint32_t*>(scratch + kScatterWarps);  // [8][n_bins] next slot per bin
  uint32_t* masks = wbase + (size_t)kScatterWarps * nb;                    // [8][bins_x + bins_y] rank masks
  uint32_t* soff = masks + kScatterWarps * (g.bins_x + g.bins_y);          // [n_bins + 1] run starts (stage) / limits
  uint32_t* gst = soff + nb + 1;                                           // [n_bins] run starts (global)
  uint64_t* openrow = reinterpret_cast<uint64_t*>(gst + nb + 1);  // [bins_y] open-bin row masks (8-B aligned: 10 nb + 8 (bx + by) + 2 words in)
  int32_t* sids = reinterpret_cast<int32_t*>(openrow + g.bins_y);          // [stage_cap] staged ids
  const uint32_t* ch = chunk_hist + ((size_t)v * n_chunks + c) * nb;
  const uint4* wh = warp_hist + ((size_t)v * n_chunks + c) * nb;  // 8 per-warp u16 counts per bin
  const uint32_t* bs = bin_start + (size_t)v * nb;
  const int w = threadIdx.x >> 5, lane = lane_id();
  for (int k = threadIdx.x; k < g.bins_y; k += kScatterThreads) openrow[k] = 0ull;
  // the chunk's kept bin counts (all of them without a cap), scanned over
  // bins: thread t owns bins [b0, b1)
  const int per = (nb + kScatterThreads - 1) / kScatterThreads;
  const int b0 = min((int)threadIdx.x * per, nb), b1 = min(b0 + per, nb);
  uint32_t mine = 0;
  for (int b = b0; b < b1; ++b) {
    const uint4 w8 = wh[b];
    const uint32_t cb = __dp2a_lo(w8.x, 0x0101u, __dp2a_lo(w8.y, 0x0101u,
                          __dp2a_lo(w8.z, 0x0101u, __dp2a_lo(w8.w, 0x0101u, 0u))));  // (u16 lo + u16 hi) per word
    const uint32_t cs = ch[b], cap = bcv[b];
    mine += cs >= cap ? 0u : min(cb, cap - cs);
  }
  uint32_t incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) red[w] = incl;
  __syncthreads();
  uint32_t wpre = 0, total = 0;
#pragma unroll
  for (int ww = 0; ww < kScatterWarps; ++ww) {
    wpre += ww < w ? red[ww] : 0u;
    total += red[ww];
  }
  if (total == 0) return;  // every instance of the chunk lands in a full bin (CTA-uniform)
  const bool staged = keys == nullptr && total <= (uint32_t)stage_cap;  // CTA-uniform
  uint32_t run = wpre + incl - mine;
  for (int b = b0; b < b1; ++b) {
    const uint4 w8 = wh[b];
    const uint32_t cb = __dp2a_lo(w8.x, 0x0101u, __dp2a_lo(w8.y, 0x0101u,
                          __dp2a_lo(w8.z, 0x0101u, __dp2a_lo(w8.w, 0x0101u, 0u))));  // (u16 lo + u16 hi) per word
    const uint32_t cs = ch[b], cap = bcv[b];
    const uint32_t kept = cs >= cap ? 0u : min(cb, cap - cs);
    const uint32_t gb = bs[b] + cs;
    gst[b] = gb;
    // staged: the stage offset of the bin's kept run; direct: the bin's
    // global limit (its materialised start + cap)
    soff[b] = staged ? run : (cap != 0xFFFFFFFFu ? bs[b] + cap : 0xFFFFFFFFu);
    uint32_t acc = staged ? run : gb;  // + exclusive prefix of the per-warp counts
#pragma unroll
    for (int ww = 0; ww < kScatterWarps; ++ww) {
      wbase[(size_t)ww * nb + b] = acc;
      const uint32_t word = ww < 2 ? w8.x : ww < 4 ? w8.y : ww < 6 ? w8.z : w8.w;
      acc += (word >> (16 * (ww & 1))) & 0xffffu;
    }
    if (kept && g.bins_x <= 64) {
      const int by = b / g.bins_x;
      atomicOr(reinterpret_cast<unsigned long long*>(&openrow[by]), 1ull << (b - by * g.bins_x));
    }
    run += kept;
  }
  if (threadIdx.x == 0) soff[nb] = total;
  __syncthreads();
  constexpr int per_warp = kChunk / kScatterWarps;
  const int64_t wlo = lo + (int64_t)w * per_warp;
  const int64_t whi = min(wlo + per_warp, nvis);
  uint32_t* colmask = masks + w * (g.bins_x + g.bins_y);
  uint32_t* rowmask = colmask + g.bins_x;
  const int32_t* sid = sorted_ids + (int64_t)v * n;
  const short4* rv = rect + (int64_t)v * n;
  const float* dv = depth + (int64_t)v * n;
  int32_t* idv = ids + (int64_t)v * capacity;
  uint64_t* kv = keys ? keys + (int64_t)v * capacity : nullptr;
  const TruncCtx tc{bcv, openrow, ch, bs, bin_total + (size_t)v * nb, resume ? resume + (size_t)v * nb : nullptr};
  uint32_t* wb = wbase + (size_t)w * nb;
  if (!staged) {
    if (trunc) warp_walk<false, true>(sid, rv, dv, wlo, whi, g, wb, colmask, rowmask, scratch[w], idv, kv, soff, tc);
    else warp_walk<false, false>(sid, rv, dv, wlo, whi, g, wb, colmask, rowmask, scratch[w], idv, kv, soff, tc);
    return;
  }
  if (trunc) warp_walk<true, true>(sid, rv, dv, wlo, whi, g, wb, colmask, rowmask, scratch[w], sids, nullptr, soff, tc);
  else warp_walk<true, false>(sid, rv, dv, wlo, whi, g, wb, colmask, rowmask, scratch[w], sids, nullptr, soff, tc);
  __syncthreads();
  // copy-out: each group of kRunLanes lanes stores one bin's run (runs
  // average ~30 ids at bin_shift 2) with consecutive lanes on consecutive slots
  constexpr int kGroups = 32 / kRunLanes;
  const int gl = lane % kRunLanes;
  for (int b = kGroups * w + lane / kRunLanes; b < nb; b += kGroups * kScatterWarps) {
    const uint32_t s0 = soff[b], cnt = soff[b + 1] - s0;
    int32_t* out = idv + gst[b];
    for (uint32_t i = gl; i < cnt; i += kRunLanes) out[i] = sids[s0 + i];
  }
}


// Tile mask of a bin-list entry (sss_bins.tmask): bit ly * 2^shift + lx
// for each tile (bx + lx, by + ly) of the bin whose 16x16 block of pixel
// centres the ellipse h(dx, dy) = A dx^2 + B2 dx dy + C dy^2 <= hmax may
// reach.  The rect is not read: it is a conservative bound of the same
// ellipse, so a bit outside it marks a tile where no pixel passes anyway and
// the raster's results cannot change.  Row by row: the ellipse's x-extent
// over the row's band of pixel-centre y, then the tile columns that interval
// meets.  Conservative by construction (fp32 throughout, every rounding
// covered by a margin):
//  * the raster's fp32 h carries a rounding error of a few ulp of
//    M = A|dx|^2 + |B2||dx||dy| + C|dy|^2 (M over the bin box), so the
//    ellipse is taken at hm = hmax + 1e-5 M;
//  * det = A C - (B2/2)^2 by Kahan's 2x2 determinant (fma residuals), a
//    few ulp relative even for thin ellipses;
//  * for a band [d0, d1] (relative to my) the leftmost point is
//    x = (-hB dy - sqrt(A hm - det dy^2)) / A, convex in dy with its minimum
//    at dyL = hB xe / C (xe = sqrt(C hm / det), the ellipse's half-width):
//    -xe whenever dyL lies in the band (with a tolerance), else the value at
//    the band end nearest dyL; the right end mirrors it;
//  * the discriminant's absolute error (~1e-7 A hm) moves x by <= 5e-4 xe:
//    the interval is widened by 1e-3 xe + 1e-5 of its terms + 1e-3 px, the
//    half-extents by 1e-5 + 1e-3 px and the bands by 1e-3 px.
// A degenerate record (det <= 0, A or C <= 0, NaN, overflow) keeps every bit.
// MUFU approximations (relative error <= 2^-22), covered by the margins below.
__device__ __forceinline__ float sqrt_apx(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_apx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t entry_tile_mask(float mx, float my, float A, float B2, float C, float hmax,
                                                    int bx, int by, int sft) {
  const int S = 1 << sft;
  const uint32_t rowbits = (1u << S) - 1u;
  const float X0 = (float)(bx * kTile) + 0.5f, X1 = (float)((bx + S) * kTile) - 0.5f;
  const float Y0 = (float)(by * kTile) + 0.5f, Y1 = (float)((by + S) * kTile) - 0.5f;
  const float mdx = fmaxf(fabsf(X0 - mx), fabsf(X1 - mx)), mdy = fmaxf(fabsf(Y0 - my), fabsf(Y1 - my));
  const float M = fmaf(A * mdx, mdx, fmaf(fabsf(B2) * mdx, mdy, C * mdy * mdy));
  const float hm = fmaf(1e-5f, M, hmax);
  const float hB = 0.5f * B2;
  const float p1 = A * C, p2 = hB * hB;
  const float det = (p1 - p2) + (fmaf(A, C, -p1) - fmaf(hB, hB, -p2));
  if (!(det > 1e-30f) || !(A > 0.f) || !(C > 0.f) || !(hm >= 0.f) || !(M < 1e30f)) {
    uint32_t m = 0u;
    for (int ly = 0; ly < S; ++ly) m |= rowbits << (ly << sft);
    return m;
  }
  const float idet = rcp_apx(det);
  const float Ah = A * hm;
  const float ym = sqrt_apx(Ah * idet);  // the ellipse's dy half-extent
  const float ymw = fmaf(ym, 1e-5f, ym) + 1e-3f;
  const float xe = sqrt_apx(C * hm * idet);  // its dx half-extent
  const float xew = fmaf(xe, 1e-5f, xe) + 1e-3f;
  const float dyL = hB * xe * rcp_apx(C);  // the leftmost point's dy (the rightmost's is -dyL)
  const float tol = fmaf(1e-4f, fabsf(dyL), 1e-3f);
  const float iA = rcp_apx(A);
  const float marg = fmaf(1e-3f, xe, 1e-3f);
  uint32_t m = 0u;
  for (int ly = 0; ly < S; ++ly) {
    const float b0 = (float)((by + ly) * kTile) + 0.5f - my - 1e-3f;
    const float b1 = (float)((by + ly) * kTile) + (kTile - 0.5f) - my + 1e-3f;
    if (b0 > ymw || b1 < -ymw) continue;
    float d0 = fmaxf(b0, -ym), d1 = fminf(b1, ym);
    if (d0 > d1) d0 = d1 = (b0 > 0.f ? ym : -ym);  // the band only grazes a tip
    float L, R;
    if (dyL >= d0 - tol && dyL <= d1 + tol) {
      L = -xew;
    } else {
      const float dl = fminf(fmaxf(dyL, d0), d1);
      const float sl = sqrt_apx(fmaxf(fmaf(-det * dl, dl, Ah), 0.f));
      const float t = -hB * dl;
      L = (t - sl) * iA - fmaf(1e-5f, (fabsf(t) + sl) * iA, marg);
    }
    if (-dyL >= d0 - tol && -dyL <= d1 + tol) {
      R = xew;
    } else {
      const float dr = fminf(fmaxf(-dyL, d0), d1);
      const float sr = sqrt_apx(fmaxf(fmaf(-det * dr, dr, Ah), 0.f));
      const float t = -hB * dr;
      R = (t + sr) * iA + fmaf(1e-5f, (fabsf(t) + sr) * iA, marg);
    }
    // tile column bx + lx (pixel centres [16 (bx+lx) + 0.5, + 15.5]) meets [mx + L, mx + R]
    const float lo_f = ceilf((mx + L - (kTile - 0.5f)) * (1.f / kTile)) - (float)bx;
    const float hi_f = floorf((mx + R - 0.5f) * (1.f / kTile)) - (float)bx;
    const int lo = lo_f > 0.f ? (int)lo_f : 0;
    const int hi = hi_f < (float)(S - 1) ? (int)hi_f : S - 1;
    if (lo <= hi) m |= ((2u << hi) - (1u << lo)) << (ly << sft);
  }
  return m;
}

#ifndef SSS_MASK_PER
#define SSS_MASK_PER 4
#endif
constexpr int kMaskPer = SSS_MASK_PER;  // entries per lane per step, all gathers in flight together
// sss_bins.tmask for every materialised entry: grid (G, V); CTA c owns a
// contiguous slice of its view's entries [0, totals[v]) (the bins'
// materialised ranges are contiguous from 0), its warps take 32 kMaskPer entries
// at a time.  The bin of an entry
// is found once per warp by binary search over the range starts, then by
// walking forward.
#ifdef SSS_MASK_MINB
#define SSS_MASK_LB __launch_bounds__(256, SSS_MASK_MINB)
#else
#define SSS_MASK_LB __launch_bounds__(256)
#endif
__global__ void SSS_MASK_LB tile_mask_kernel(const int32_t* __restrict__ ids,
                                                        const int32_t* __restrict__ ranges,
                                                        const int64_t* __restrict__ totals, int64_t capacity,
                                                        const float4* __restrict__ rec, int64_t n, BinGeom g,
                                                        uint16_t* __restrict__ tmask) {
  const int v = blockIdx.y;
  const int64_t tot = totals[v];
  if (tot > capacity) return;  // overflowed: nothing scattered
  const int64_t per = ((tot + gridDim.x - 1) / gridDim.x + 32 * kMaskPer - 1) & ~(int64_t)(32 * kMaskPer - 1);
  const int64_t c0 = (int64_t)blockIdx.x * per, c1 = min(tot, c0 + per);
  const int w = threadIdx.x >> 5, lane = lane_id();
  int64_t base = c0 + (int64_t)w * 32 * kMaskPer;
  if (base >= c1) return;
  const int2* rg = reinterpret_cast<const int2*>(ranges) + (size_t)v * g.n_bins;
  const int32_t* idv = ids + (int64_t)v * capacity;
  uint16_t* tmv = tmask + (int64_t)v * capacity;
  const float4* recv = rec + (int64_t)v * n * 2;  // 32-byte geometry records: one sector each
  int bw = 0;  // last bin whose start <= base (empty bins share their successor's start)
  {
    int hi = g.n_bins - 1;
    while (bw < hi) {
      const int mid = (bw + hi + 1) >> 1;
      if (__ldg(&rg[mid].x) <= base) bw = mid; else hi = mid - 1;
    }
  }
  for (; base < c1; base += kMaskPer * 32 * (int64_t)(blockDim.x >> 5)) {
    while (base >= __ldg(&rg[bw].y)) ++bw;  // warp-uniform
    int id[kMaskPer];
#pragma unroll
    for (int q = 0; q < kMaskPer; ++q) id[q] = base + q * 32 + lane < c1 ? __ldg(idv + base + q * 32 + lane) : 0;
    float4 a[kMaskPer];
    float2 e[kMaskPer];
#pragma unroll
    for (int q = 0; q < kMaskPer; ++q) {
      a[q] = __ldg(recv + (int64_t)id[q] * 2);
      e[q] = __ldg(reinterpret_cast<const float2*>(recv + (int64_t)id[q] * 2 + 1));
    }
    int b = bw;
#pragma unroll
    for (int q = 0; q < kMaskPer; ++q) {
      const int64_t p = base + q * 32 + lane;
      while (p >= __ldg(&rg[b].y) && b < g.n_bins - 1) ++b;
      if (p < c1)
        tmv[p] = (uint16_t)entry_tile_mask(a[q].x, a[q].y, a[q].z, a[q].w, e[q].x, e[q].y, (b % g.bins_x) << g.shift,
                                           (b / g.bins_x) << g.shift, g.shift);
    }
  }
}

}  // namespace
}  // namespace sss

using namespace sss;

extern "C" size_t sss_bin_sort_workspace(int64_t n, int32_t n_views, const sss_camera* cams,
                                         int32_t bin_shift) {
  if (n < 0 || n_views <= 0 || !cams || bin_shift < 0 || bin_shift > 6) return 0;
  if (cams[0].width <= 0 || cams[0].height <= 0) return 0;
  const BinGeom g = bin_geom(cams[0], bin_shift);
  return ws_layout(n > 0 ? n : 1, n_views, g).total;
}

extern "C" sss_status sss_bin_sort(const sss_projected* pr, const sss_camera* cams, int32_t n_views,
                                   void* ws, size_t ws_bytes, sss_bins* out, void* stream) {
  sss_status st;
  if (!pr || !out) { set_error("sss_bin_sort: null argument"); return SSS_ERR_ARG; }
  if ((st = validate_cams(cams, n_views, "sss_bin_sort")) != SSS_OK) return st;
  if (pr->n_views != n_views || out->n_views != n_views) {
    set_error("sss_bin_sort: n_views mismatch");
    return SSS_ERR_ARG;
  }
  if (out->bin_shift < 0 || out->bin_shift > 6) { set_error("sss_bin_sort: bin_shift outside [0,6]"); return SSS_ERR_ARG; }
  const BinGeom g = bin_geom(cams[0], out->bin_shift);
  if (g.n_bins > SSS_MAX_BINS || g.bins_x > 1024 || g.bins_y > 1024) {
    set_error("sss_bin_sort: %d x %d bins: need <= SSS_MAX_BINS (%d) and <= 1024 per axis; raise bin_shift",
              g.bins_x, g.bins_y, SSS_MAX_BINS);
    return SSS_ERR_SHAPE;
  }
  const int64_t n = pr->n;
  if (!out->ranges || !out->totals || !out->overflow || (!out->ids && out->capacity > 0) || out->capacity < 0) {
    set_error("sss_bin_sort: null output buffer");
    return SSS_ERR_ARG;
  }
  if (out->max_per_bin < 0 ||
      ((out->max_per_bin > 0 || out->used) && (!out->sorted || !out->n_vis || !out->resume))) {
    set_error("sss_bin_sort: truncated lists (max_per_bin > 0 or used) need sorted, n_vis and resume");
    return SSS_ERR_ARG;
  }
  if (out->tmask && out->bin_shift > 2) {
    set_error("sss_bin_sort: tile masks (tmask) need bin_shift <= 2 (16 tiles per bin)");
    return SSS_ERR_ARG;
  }
  if (out->tmask && !pr->rec) { set_error("sss_bin_sort: tile masks need the projected records"); return SSS_ERR_ARG; }
  if (n > 0x7fffffffLL - out->capacity) {  // virtual list positions (start + n) must fit int32
    set_error("sss_bin_sort: n + capacity must be < 2^31");
    return SSS_ERR_SHAPE;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const WsLayout L = ws_layout(n > 0 ? n : 1, n_views, g);
  if (!ws || ws_bytes < L.total) {
    set_error("sss_bin_sort: workspace %zu < %zu bytes", ws_bytes, L.total);
    return SSS_ERR_ARG;
  }
  char* w = (char*)ws;
  uint32_t* keys_a = (uint32_t*)(w + L.keys_a);
  uint32_t* keys_b = (uint32_t*)(w + L.keys_b);
  int32_t* vals_a = (int32_t*)(w + L.vals_a);
  int32_t* vals_b = (int32_t*)(w + L.vals_b);
  int32_t* sorted = out->sorted ? out->sorted : (int32_t*)(w + L.sorted);
  int32_t* n_vis = out->n_vis ? out->n_vis : (int32_t*)(w + L.n_vis);
  uint32_t* rhist = (uint32_t*)(w + L.radix_hist);
  uint32_t* chist = (uint32_t*)(w + L.chunk_hist);
  uint8_t* whist = (uint8_t*)(w + L.warp_hist);
  uint32_t* ckept = (uint32_t*)(w + L.chunk_kept);
  uint32_t* btot = (uint32_t*)(w + L.bin_total);
  uint32_t* bstart = (uint32_t*)(w + L.bin_start);
  const short4* rect = (const short4*)pr->rect;
  const bool trunc = out->max_per_bin > 0 || out->used;
  const uint32_t static_cap = out->max_per_bin > 0 ? (uint32_t)out->max_per_bin : 0xFFFFFFFFu;
  int32_t* resume = trunc ? out->resume : nullptr;
  uint32_t* bcap = (uint32_t*)(w + L.bin_cap);

  static thread_local bool attr_set = false;
  if (!attr_set) {  // large dynamic shared memory for the per-warp bin counters
    cudaFuncSetAttribute(scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kScatterSmemMax);
    cudaFuncSetAttribute(chunk_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr_set = true;
  }
  // out->overflow is sticky: set here on overflow, never cleared (the caller
  // resets it after checking), so a check after many calls sees every one
  cudaMemsetAsync(n_vis, 0, sizeof(int32_t) * n_views, s);
  if (n > 0) {
    // 16-byte key initialisation when every view's segment is 16-byte aligned
    const bool vec = n % 4 == 0 && ((reinterpret_cast<uintptr_t>(pr->depth) | reinterpret_cast<uintptr_t>(rect) |
                                     reinterpret_cast<uintptr_t>(keys_a) | reinterpret_cast<uintptr_t>(vals_a)) &
                                    15u) == 0;
    if (vec) {
      const dim3 gi(div_up(n / 4, 256), n_views);
      keys_init4_kernel<<<gi, 256, 0, s>>>((const float4*)pr->depth, (const int4*)rect, n, (uint4*)keys_a,
                                           (int4*)vals_a, n_vis);
    } else {
      const dim3 gi(div_up(n, 256), n_views);
      keys_init_kernel<<<gi, 256, 0, s>>>(pr->depth, rect, n, keys_a, vals_a, n_vis);
    }
    count_launch();
    // culled keys (0xFFFFFFFF) sort last: sorted[:n_vis] are the visible ones
    radix_sort_pairs(keys_a, vals_a, keys_b, vals_b, n, n_views, L.tiles_per_view, rhist, s, sorted);
    const dim3 gc(L.n_chunks, n_views);
    const size_t hsm = (size_t)kScatterWarps * g.n_bins * 4;
    chunk_hist_kernel<<<gc, kScatterThreads, hsm, s>>>(sorted, n_vis, rect, n, L.chunk, L.n_chunks, g, chist, whist);
    column_scan_kernel<<<dim3(div_up(g.n_bins, 32), n_views), 32 * kColWarps, 0, s>>>(
        chist, L.n_chunks, g.n_bins, btot, static_cap, out->used, bcap, trunc ? ckept : nullptr);
    count_launch(2);
  } else {
    cudaMemsetAsync(btot, 0, sizeof(uint32_t) * n_views * g.n_bins, s);
    cudaMemsetAsync(bcap, 0xFF, sizeof(uint32_t) * n_views * g.n_bins, s);
  }
  bin_scan_kernel<<<n_views, 1024, 0, s>>>(btot, g.n_bins, out->capacity, out->used, bcap, bstart,
                                            out->ranges, out->totals, out->overflow, n_vis, resume);
  count_launch();
  if (n > 0) {
    // stage: the chunk's mean share of the capacity (the caller sizes the
    // capacity with headroom over the measured instance count), within the
    // shared memory left; larger chunks take the direct path
    const size_t fixed = sizeof(WalkScratch) * kScatterWarps +
                         ((size_t)kScatterWarps * g.n_bins + kScatterWarps * (g.bins_x + g.bins_y) +
                          2 * (size_t)g.n_bins + 2 + 2 * (size_t)g.bins_y) * 4;
    int64_t want = (out->capacity + L.n_chunks - 1) / L.n_chunks;
    want = std::min<int64_t>(std::max<int64_t>(want, 256), kScatterStageMax);
    // truncated lists: most chunks keep little, and the walk is latency-bound,
    // so a small stage (more CTAs per SM) wins; the few front chunks that keep
    // more than it take the direct path
#ifndef SSS_SCATTER_TRUNC_STAGE
#define SSS_SCATTER_TRUNC_STAGE 4096
#endif
    if (trunc) want = std::min<int64_t>(want, SSS_SCATTER_TRUNC_STAGE);
    const int64_t room = ((int64_t)kScatterSmemMax - (int64_t)fixed) / 4;
    const int stage_cap = (int)std::max<int64_t>(0, std::min<int64_t>((want + 31) & ~31, room));
    const size_t ssm = fixed + (size_t)stage_cap * 4;
    scatter_kernel<<<dim3(L.n_chunks, n_views), kScatterThreads, ssm, s>>>(
        sorted, n_vis, rect, pr->depth, n, L.n_chunks, g, chist, (const uint4*)whist, trunc ? ckept : nullptr,
        bstart, btot,
        out->totals,
        out->capacity, bcap, stage_cap, out->ids, out->keys, resume);
    count_launch();
    if (out->tmask) {
#ifndef SSS_MASK_GX
#define SSS_MASK_GX 148
#endif
      // 148 CTAs per view, launched view-major: ~8 views in flight, so a
      // record line fetched for one bin is often still in L2 for the
      // component's other bins (config 5: -0.26 ms vs all 64 views at once
      // with 18 CTAs each; 296 / 592 / 1184 per view: -0.22 / -0.13 / 0)
      const int gx = SSS_MASK_GX;
      tile_mask_kernel<<<dim3(gx, n_views), 256, 0, s>>>(out->ids, out->ranges, out->totals, out->capacity,
                                                               (const float4*)pr->rec, n, g, out->tmask);
      count_launch();
    }
  }
  return check_launch("sss_bin_sort");
}

extern "C" sss_status sss_check_overflow(const sss_bins* bins, void* stream) {
  if (!bins || !bins->overflow) { set_error("sss_check_overflow: null"); return SSS_ERR_ARG; }
  int32_t h = 0;
  if (cudaMemcpyAsync(&h, bins->overflow, sizeof(int32_t), cudaMemcpyDeviceToHost, (cudaStream_t)stream) !=
          cudaSuccess ||
      cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess)
    return check_launch("sss_check_overflow");
  return h ? SSS_ERR_CAPACITY : SSS_OK;
}
