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
//      (keys of culled components are 0xFFFFFFFF and sort last);
//   2. a stable counting scatter of the instances by bin, generated on the fly
//      from the depth-sorted components: per-chunk bin histograms (shared
//      memory), a column scan over chunks, a scan over bins, then a scatter in
//      which each warp walks its components in order, so bins receive their
//      entries in depth order without ever materialising 64-bit keys.
// Every instance is written exactly once (4 B id, +8 B key if requested); the
// radix passes touch only N keys per view.  All views are processed by the
// same launches (grid.y = view).
#include "common.cuh"

namespace sss {
namespace {

#ifndef SSS_RADIX_MATCH
#define SSS_RADIX_MATCH 0  // warp peers of a digit: 0 = 8 ballots, 1 = match.any
#endif
constexpr int kRadixThreads = 256;
constexpr int kRadixItems = 16;
constexpr int kRadixTile = kRadixThreads * kRadixItems;  // 4096 keys per CTA
constexpr int kScatterThreads = 256;
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

inline int chunk_size(int64_t n, int V) {
  // components per scatter chunk: enough CTAs to fill 148 SMs a few times,
  // but few enough chunks that the [chunk][bin] histograms stay small.
  int64_t c = (n * (int64_t)V) / (148 * 4);
  int cs = 1024;
  while (cs < c && cs < 8192) cs *= 2;
  return cs;
}

struct WsLayout {
  size_t keys_a, keys_b, vals_a, vals_b, n_vis, radix_hist, chunk_hist, bin_total, bin_start, total;
  int tiles_per_view, n_chunks, chunk;
};

inline size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

WsLayout ws_layout(int64_t n, int V, const BinGeom& g) {
  WsLayout L;
  L.tiles_per_view = div_up(n, kRadixTile);
  L.chunk = chunk_size(n, V);
  L.n_chunks = div_up(n, L.chunk);
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += align_up(bytes); return o; };
  const size_t nv = (size_t)n * V;
  L.keys_a = take(nv * 4);
  L.keys_b = take(nv * 4);
  L.vals_a = take(nv * 4);
  L.vals_b = take(nv * 4);
  L.n_vis = take((size_t)V * 4);
  L.radix_hist = take((size_t)V * 256 * (size_t)L.tiles_per_view * 4);
  L.chunk_hist = take((size_t)V * L.n_chunks * (size_t)g.n_bins * 4);
  L.bin_total = take((size_t)V * g.n_bins * 4);
  L.bin_start = take((size_t)V * g.n_bins * 4);
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

// Positive fp32 depths (> z_near > 0) order like their bit patterns.
__device__ __forceinline__ unsigned peers_of(unsigned d) {
#if SSS_RADIX_MATCH
  return __match_any_sync(0xffffffffu, d);
#endif
  unsigned m = 0xffffffffu;
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    const unsigned bal = __ballot_sync(0xffffffffu, (d >> b) & 1u);
    m &= ((d >> b) & 1u) ? bal : ~bal;
  }
  return m;
}

__global__ void __launch_bounds__(kRadixThreads) radix_upsweep_kernel(const uint32_t* __restrict__ keys,
                                                                      int64_t n, int shift, int tiles,
                                                                      uint32_t* __restrict__ hist) {
  __shared__ uint32_t h[256];
  const int v = blockIdx.y, tile = blockIdx.x;
  h[threadIdx.x] = 0;
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = lane_id();
  const int64_t base = (int64_t)tile * kRadixTile + w * (32 * kRadixItems);
  for (int c = 0; c < kRadixItems; ++c) {
    const int64_t i = base + c * 32 + lane;
    const bool ok = i < n;
    const unsigned d = ok ? (keys[(int64_t)v * n + i] >> shift) & 255u : 256u;
    const unsigned valid = __ballot_sync(0xffffffffu, ok);
    const unsigned pm = peers_of(d & 255u) & valid;
    if (ok && (pm & ((1u << lane) - 1u)) == 0) atomicAdd(&h[d], __popc(pm));
  }
  __syncthreads();
  hist[((size_t)v * 256 + threadIdx.x) * tiles + tile] = h[threadIdx.x];
}

// exclusive scan of one view's digit-major histogram (256 * tiles entries)
__global__ void __launch_bounds__(1024) scan_u32_kernel(uint32_t* __restrict__ data, int64_t len_per_seg) {
  __shared__ uint32_t part[1024];
  uint32_t* d = data + (size_t)blockIdx.x * len_per_seg;
  const int t = threadIdx.x;
  const int64_t per = (len_per_seg + 1023) / 1024;
  const int64_t lo = t * per, hi = lo + per < len_per_seg ? lo + per : len_per_seg;
  uint32_t s = 0;
  for (int64_t k = lo; k < hi; ++k) s += d[k];
  part[t] = s;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {
    uint32_t x = t >= off ? part[t - off] : 0;
    __syncthreads();
    part[t] += x;
    __syncthreads();
  }
  uint32_t run = part[t] - s;
  for (int64_t k = lo; k < hi; ++k) {
    const uint32_t x = d[k];
    d[k] = run;
    run += x;
  }
}

__global__ void __launch_bounds__(kRadixThreads) radix_downsweep_kernel(
    const uint32_t* __restrict__ keys_in, const int32_t* __restrict__ vals_in, int64_t n, int shift,
    int tiles, const uint32_t* __restrict__ hist, uint32_t* __restrict__ keys_out,
    int32_t* __restrict__ vals_out) {
  __shared__ uint32_t run[kScatterWarps][256];
  __shared__ uint32_t tile_off[256];
  const int v = blockIdx.y, tile = blockIdx.x;
  const int w = threadIdx.x >> 5, lane = lane_id();
  for (int k = threadIdx.x; k < kScatterWarps * 256; k += kRadixThreads) (&run[0][0])[k] = 0;
  tile_off[threadIdx.x] = hist[((size_t)v * 256 + threadIdx.x) * tiles + tile];
  __syncthreads();
  const int64_t base = (int64_t)tile * kRadixTile + w * (32 * kRadixItems);
  uint32_t key[kRadixItems];
  int32_t val[kRadixItems];
  uint32_t loc[kRadixItems];
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int c = 0; c < kRadixItems; ++c) {
    const int64_t i = base + c * 32 + lane;
    const bool ok = i < n;
    key[c] = ok ? keys_in[(int64_t)v * n + i] : 0u;
    val[c] = ok ? vals_in[(int64_t)v * n + i] : 0;
    const unsigned d = (key[c] >> shift) & 255u;
    const unsigned valid = __ballot_sync(0xffffffffu, ok);
    const unsigned pm = peers_of(d) & valid;
    const uint32_t before = ok ? run[w][d] : 0u;
    loc[c] = before + __popc(pm & lt);
    __syncwarp();
    if (ok && (pm & lt) == 0) run[w][d] = before + __popc(pm);
    __syncwarp();
  }
  __syncthreads();
  // exclusive prefix over warps per digit -> warp base
  {
    const int d = threadIdx.x;
    uint32_t acc = tile_off[d];
    for (int ww = 0; ww < kScatterWarps; ++ww) {
      const uint32_t x = run[ww][d];
      run[ww][d] = acc;
      acc += x;
    }
  }
  __syncthreads();
#pragma unroll
  for (int c = 0; c < kRadixItems; ++c) {
    const int64_t i = base + c * 32 + lane;
    if (i < n) {
      const unsigned d = (key[c] >> shift) & 255u;
      const uint32_t pos = run[w][d] + loc[c];
      keys_out[(int64_t)v * n + pos] = key[c];
      vals_out[(int64_t)v * n + pos] = val[c];
    }
  }
}

// ------------------------------------------------------- bin histograms
__device__ __forceinline__ void bin_rect(short4 r, int shift, int& bx0, int& by0, int& bx1, int& by1) {
  bx0 = r.x >> shift; by0 = r.y >> shift; bx1 = r.z >> shift; by1 = r.w >> shift;
}

__global__ void __launch_bounds__(256) chunk_hist_kernel(const int32_t* __restrict__ sorted_ids,
                                                         const int32_t* __restrict__ n_vis,
                                                         const short4* __restrict__ rect, int64_t n,
                                                         int chunk, int n_chunks, BinGeom g,
                                                         uint32_t* __restrict__ chunk_hist) {
  extern __shared__ uint32_t hs[];
  const int v = blockIdx.y, c = blockIdx.x;
  for (int b = threadIdx.x; b < g.n_bins; b += blockDim.x) hs[b] = 0;
  __syncthreads();
  const int64_t lo = (int64_t)c * chunk;
  const int64_t hi = min((int64_t)(c + 1) * chunk, (int64_t)n_vis[v]);
  for (int64_t j = lo + threadIdx.x; j < hi; j += blockDim.x) {
    const int id = sorted_ids[(int64_t)v * n + j];
    int bx0, by0, bx1, by1;
    bin_rect(rect[(int64_t)v * n + id], g.shift, bx0, by0, bx1, by1);
    for (int by = by0; by <= by1; ++by)
      for (int bx = bx0; bx <= bx1; ++bx) atomicAdd(&hs[by * g.bins_x + bx], 1u);
  }
  __syncthreads();
  uint32_t* out = chunk_hist + ((size_t)v * n_chunks + c) * g.n_bins;
  for (int b = threadIdx.x; b < g.n_bins; b += blockDim.x) out[b] = hs[b];
}

// per (view, bin): exclusive scan over chunks in place; bin totals
__global__ void column_scan_kernel(uint32_t* __restrict__ chunk_hist, int n_chunks, int n_bins,
                                   uint32_t* __restrict__ bin_total) {
  const int v = blockIdx.y;
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= n_bins) return;
  uint32_t* col = chunk_hist + (size_t)v * n_chunks * n_bins + b;
  uint32_t run = 0;
  int c = 0;
  for (; c + 4 <= n_chunks; c += 4) {
    const uint32_t x0 = col[(size_t)(c + 0) * n_bins], x1 = col[(size_t)(c + 1) * n_bins];
    const uint32_t x2 = col[(size_t)(c + 2) * n_bins], x3 = col[(size_t)(c + 3) * n_bins];
    col[(size_t)(c + 0) * n_bins] = run; run += x0;
    col[(size_t)(c + 1) * n_bins] = run; run += x1;
    col[(size_t)(c + 2) * n_bins] = run; run += x2;
    col[(size_t)(c + 3) * n_bins] = run; run += x3;
  }
  for (; c < n_chunks; ++c) {
    const uint32_t x = col[(size_t)c * n_bins];
    col[(size_t)c * n_bins] = run;
    run += x;
  }
  bin_total[(size_t)v * n_bins + b] = run;
}

// per view: exclusive scan over bins -> bin_start, ranges, totals, overflow
__global__ void __launch_bounds__(1024) bin_scan_kernel(const uint32_t* __restrict__ bin_total, int n_bins,
                                                        int64_t capacity, uint32_t* __restrict__ bin_start,
                                                        int32_t* __restrict__ ranges,
                                                        int64_t* __restrict__ totals,
                                                        int32_t* __restrict__ overflow) {
  __shared__ unsigned long long part[1024];
  __shared__ int over;
  const int v = blockIdx.x, t = threadIdx.x;
  const uint32_t* bt = bin_total + (size_t)v * n_bins;
  const int per = (n_bins + 1023) / 1024;
  const int lo = t * per, hi = min(lo + per, n_bins);
  unsigned long long s = 0;
  for (int k = lo; k < hi; ++k) s += bt[k];
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
    const uint32_t x = bt[k];
    bin_start[(size_t)v * n_bins + k] = (uint32_t)run;
    ranges[((size_t)v * n_bins + k) * 2 + 0] = over ? 0 : (int32_t)run;
    ranges[((size_t)v * n_bins + k) * 2 + 1] = over ? 0 : (int32_t)(run + x);
    run += x;
  }
}

// Walks the instances (component, bin) of the warp's components
// [wlo, whi) in order — component-major, bin row-major — 32 instances per
// step: the instance counts of 32 consecutive components are prefix-summed
// across the warp, each lane finds the component owning its flat index by a
// 5-step binary search over the lanes, and lanes hitting the same bin in the
// same step are ranked by lane order (match.any), which preserves the
// (depth, index) order within every bin.  COUNT: per-warp bin counts;
// otherwise write ids (and keys) at base[b] + the warp's running offset.
template <bool COUNT>
__device__ __forceinline__ void warp_instances(const int32_t* __restrict__ sid, const short4* __restrict__ rv,
                                               const float* __restrict__ dv, int64_t wlo, int64_t whi,
                                               const BinGeom& g, uint16_t* my, const uint32_t* base,
                                               int32_t* __restrict__ idv, uint64_t* __restrict__ kv) {
  const int lane = lane_id();
  const unsigned lt = (1u << lane) - 1u;
  // software pipeline: the next group's (id, rect) gathers are in flight
  // while the current group's instances are placed
  int id_n = 0;
  short4 r_n = make_short4(1, 1, 0, 0);
  if (wlo + lane < whi) {
    id_n = sid[wlo + lane];
    r_n = rv[id_n];
  }
  for (int64_t j0 = wlo; j0 < whi; j0 += 32) {
    const int64_t j = j0 + lane;
    const int id = id_n;
    const short4 r = r_n;
    if (j + 32 < whi) {
      id_n = sid[j + 32];
      r_n = rv[id_n];
    }
    int bx0 = 0, by0 = 0, bw = 1, nb = 0;
    uint32_t dbits = 0;
    if (j < whi) {
      bx0 = r.x >> g.shift;
      by0 = r.y >> g.shift;
      bw = (r.z >> g.shift) - bx0 + 1;
      nb = bw * ((r.w >> g.shift) - by0 + 1);
      if (!COUNT && kv) dbits = __float_as_uint(dv[id]);
    }
    int incl = nb;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const int excl = incl - nb;
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    for (int f0 = 0; f0 < total; f0 += 32) {
      const int f = f0 + lane;
      const bool act = f < total;
      int k = 0;  // owner lane: the largest k with excl_k <= f
#pragma unroll
      for (int step = 16; step > 0; step >>= 1) {
        const int e = __shfl_sync(0xffffffffu, excl, k + step);
        if (e <= f) k += step;
      }
      const int t = f - __shfl_sync(0xffffffffu, excl, k);
      const int kbw = __shfl_sync(0xffffffffu, bw, k);
      const int kbx0 = __shfl_sync(0xffffffffu, bx0, k);
      const int kby0 = __shfl_sync(0xffffffffu, by0, k);
      const int row = t / kbw;
      const int b = (kby0 + row) * g.bins_x + kbx0 + (t - row * kbw);
      // lanes of this step with the same bin (ballots on its bits; cheaper
      // than match.any on sm_100)
      unsigned peers = __ballot_sync(0xffffffffu, act);
      for (int i = 0; i < g.bits; ++i) {
        const bool bit = (b >> i) & 1;
        const unsigned bal = __ballot_sync(0xffffffffu, bit);
        peers &= bit ? bal : ~bal;
      }
      const int rank = __popc(peers & lt);
      if (!COUNT) {
        const int kid = __shfl_sync(0xffffffffu, id, k);
        const uint32_t kd = __shfl_sync(0xffffffffu, dbits, k);
        if (act) {
          const uint32_t pos = base[b] + my[b] + rank;
          idv[pos] = kid;
          if (kv) kv[pos] = ((uint64_t)b << 32) | kd;
        }
      }
      __syncwarp();
      if (act && rank == 0) my[b] += (uint16_t)__popc(peers);
      __syncwarp();
    }
  }
}

// stable scatter: CTA per (chunk, view); warp w owns components
// [chunk*c + w*chunk/8, ...) and walks their instances in order.
__global__ void __launch_bounds__(kScatterThreads) scatter_kernel(
    const int32_t* __restrict__ sorted_ids, const int32_t* __restrict__ n_vis,
    const short4* __restrict__ rect, const float* __restrict__ depth, int64_t n, int chunk,
    int n_chunks, BinGeom g, const uint32_t* __restrict__ chunk_hist,
    const uint32_t* __restrict__ bin_start, const int64_t* __restrict__ totals, int64_t capacity,
    int32_t* __restrict__ ids, uint64_t* __restrict__ keys) {
  extern __shared__ uint32_t sm[];
  const int v = blockIdx.y, c = blockIdx.x;
  if (totals[v] > capacity) return;
  const int64_t lo = (int64_t)c * chunk;
  const int64_t nvis = n_vis[v];
  if (lo >= nvis) return;
  uint32_t* base = sm;                                    // [n_bins]
  uint16_t* woff = (uint16_t*)(sm + g.n_bins);            // [8][n_bins]
  const uint32_t* ch = chunk_hist + ((size_t)v * n_chunks + c) * g.n_bins;
  const uint32_t* bs = bin_start + (size_t)v * g.n_bins;
  for (int b = threadIdx.x; b < g.n_bins; b += blockDim.x) base[b] = bs[b] + ch[b];
  for (int k = threadIdx.x; k < kScatterWarps * g.n_bins; k += blockDim.x) woff[k] = 0;
  __syncthreads();
  const int w = threadIdx.x >> 5;
  const int per_warp = chunk / kScatterWarps;
  const int64_t wlo = lo + (int64_t)w * per_warp;
  const int64_t whi = min(wlo + per_warp, nvis);
  uint16_t* my = woff + (size_t)w * g.n_bins;
  const int32_t* sid = sorted_ids + (int64_t)v * n;
  const short4* rv = rect + (int64_t)v * n;
  const float* dv = depth + (int64_t)v * n;
  int32_t* idv = ids + (int64_t)v * capacity;
  uint64_t* kv = keys ? keys + (int64_t)v * capacity : nullptr;
  warp_instances<true>(sid, rv, dv, wlo, whi, g, my, base, idv, kv);  // phase 1: counts
  __syncthreads();
  for (int b = threadIdx.x; b < g.n_bins; b += blockDim.x) {
    uint32_t acc = 0;
    for (int ww = 0; ww < kScatterWarps; ++ww) {
      const uint32_t x = woff[(size_t)ww * g.n_bins + b];
      woff[(size_t)ww * g.n_bins + b] = (uint16_t)acc;
      acc += x;
    }
  }
  __syncthreads();
  warp_instances<false>(sid, rv, dv, wlo, whi, g, my, base, idv, kv);  // phase 2: scatter
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
  if (g.n_bins > SSS_MAX_BINS) {
    set_error("sss_bin_sort: %d bins > SSS_MAX_BINS (%d); raise bin_shift", g.n_bins, SSS_MAX_BINS);
    return SSS_ERR_SHAPE;
  }
  const int64_t n = pr->n;
  if (!out->ranges || !out->totals || !out->overflow || (!out->ids && out->capacity > 0) || out->capacity < 0) {
    set_error("sss_bin_sort: null output buffer");
    return SSS_ERR_ARG;
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
  int32_t* n_vis = (int32_t*)(w + L.n_vis);
  uint32_t* rhist = (uint32_t*)(w + L.radix_hist);
  uint32_t* chist = (uint32_t*)(w + L.chunk_hist);
  uint32_t* btot = (uint32_t*)(w + L.bin_total);
  uint32_t* bstart = (uint32_t*)(w + L.bin_start);
  const short4* rect = (const short4*)pr->rect;

  cudaMemsetAsync(out->overflow, 0, sizeof(int32_t), s);
  cudaMemsetAsync(n_vis, 0, sizeof(int32_t) * n_views, s);
  if (n > 0) {
    dim3 gi(div_up(n, 256), n_views);
    keys_init_kernel<<<gi, 256, 0, s>>>(pr->depth, rect, n, keys_a, vals_a, n_vis);
    count_launch();
    const dim3 gr(L.tiles_per_view, n_views);
    uint32_t *kin = keys_a, *kout = keys_b;
    int32_t *vin = vals_a, *vout = vals_b;
    for (int pass = 0; pass < 4; ++pass) {
      radix_upsweep_kernel<<<gr, kRadixThreads, 0, s>>>(kin, n, pass * 8, L.tiles_per_view, rhist);
      scan_u32_kernel<<<n_views, 1024, 0, s>>>(rhist, (int64_t)256 * L.tiles_per_view);
      radix_downsweep_kernel<<<gr, kRadixThreads, 0, s>>>(kin, vin, n, pass * 8, L.tiles_per_view, rhist,
                                                          kout, vout);
      count_launch(3);
      uint32_t* tk = kin; kin = kout; kout = tk;
      int32_t* tv = vin; vin = vout; vout = tv;
    }
    // after 4 passes the sorted ids are in vals_a
    const dim3 gc(L.n_chunks, n_views);
    const size_t hsm = (size_t)g.n_bins * 4;
    chunk_hist_kernel<<<gc, 256, hsm, s>>>(vin, n_vis, rect, n, L.chunk, L.n_chunks, g, chist);
    column_scan_kernel<<<dim3(div_up(g.n_bins, 128), n_views), 128, 0, s>>>(chist, L.n_chunks, g.n_bins, btot);
    count_launch(2);
  } else {
    cudaMemsetAsync(btot, 0, sizeof(uint32_t) * n_views * g.n_bins, s);
  }
  bin_scan_kernel<<<n_views, 1024, 0, s>>>(btot, g.n_bins, out->capacity, bstart, out->ranges, out->totals,
                                            out->overflow);
  count_launch();
  if (n > 0) {
    static thread_local bool attr_set = false;
    if (!attr_set) {
      cudaFuncSetAttribute(scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      cudaFuncSetAttribute(chunk_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      attr_set = true;
    }
    const size_t ssm = (size_t)g.n_bins * 4 + (size_t)kScatterWarps * g.n_bins * 2;
    scatter_kernel<<<dim3(L.n_chunks, n_views), kScatterThreads, ssm, s>>>(
        vals_a, n_vis, rect, pr->depth, n, L.chunk, L.n_chunks, g, chist, bstart, out->totals,
        out->capacity, out->ids, out->keys);
    count_launch();
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
