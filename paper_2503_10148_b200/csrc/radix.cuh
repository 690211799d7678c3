// Stable LSD radix sort of (uint32 key, int32 value) pairs, 4 x 8-bit digit
// passes, for independent segments of equal length (grid.y = segment).  Used
// by a2 (per-view depth keys) and NEXT-2 (relocation targets).
//
// Onesweep structure (single-pass prefix per digit with decoupled
// look-back): one kernel reads every key once and builds the four global
// digit histograms of each segment; then each pass is ONE kernel.  A CTA
// takes the next 4096-key tile of its segment in launch order (atomic
// ticket), ranks its keys with per-warp digit counters (8 ballots per 32
// keys, in key order), publishes its per-digit counts, looks back over its
// predecessors' published counts/prefixes (thread d handles digit d) to get
// its exclusive per-digit offset, publishes its inclusive prefix, and writes
// its keys reordered by digit in shared memory so the global stores leave
// as per-digit runs.  Status words pack a 2-bit flag and a 30-bit count.
//
// Depth mode (a2's per-view depth sort): the keys are read straight from the
// projection (key = float bits of the depth of a visible component; culled
// components are dropped, so the sort also compacts), the values are the
// component indices (implicit), and a digit pass runs only if its digit
// takes more than one value over the view's visible keys (the histogram
// kernel builds all four digit histograms first; config 5's depths lie in
// [2, 8), so the top byte is constant and three passes remain).  A per-view
// schedule picks each active pass's source / destination buffers; the last
// active pass writes only the values, into the caller's sorted-id array.
#pragma once
#include "common.cuh"

namespace sss {
namespace {

constexpr int kRadixThreads = 256;
constexpr int kRadixWarps = kRadixThreads / 32;
#ifndef SSS_RADIX_ITEMS
#define SSS_RADIX_ITEMS 16
#endif
constexpr int kRadixItems = SSS_RADIX_ITEMS;
constexpr int kRadixTile = kRadixThreads * kRadixItems;  // 4096 keys per CTA
constexpr uint32_t kStAgg = 1u << 30, kStInc = 2u << 30, kStCount = (1u << 30) - 1u;

// 32-bit words of scratch radix_sort_pairs needs (status words of the four
// passes, global histograms and their offsets, tile tickets).
inline size_t radix_ws_words(int tiles, int n_segs) {
  return (size_t)n_segs * (4 * 256 * (size_t)tiles + 2 * 4 * 256 + 4);
}

// lanes of the warp holding the same 8-bit digit (ballots on its bits)
__device__ __forceinline__ unsigned peers_of(unsigned d) {
  unsigned m = 0xffffffffu;
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    const unsigned bal = __ballot_sync(0xffffffffu, (d >> b) & 1u);
    m &= ((d >> b) & 1u) ? bal : ~bal;
  }
  return m;
}

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t x) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, x, o);
    if ((int)lane_id() >= o) x += t;
  }
  return x;
}

__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// the four digit histograms of every segment, one read of the keys
__global__ void __launch_bounds__(kRadixThreads) radix_hist_kernel(const uint32_t* __restrict__ keys, int64_t n,
                                                                   uint32_t* __restrict__ ghist) {
  __shared__ uint32_t h[4][256];
  const int v = blockIdx.y;
  for (int k = threadIdx.x; k < 4 * 256; k += kRadixThreads) (&h[0][0])[k] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kRadixTile;
  const uint32_t* kin = keys + (int64_t)v * n;
  uint32_t k[kRadixItems];
#pragma unroll
  for (int c = 0; c < kRadixItems; ++c) {
    const int64_t i = base + c * kRadixThreads + threadIdx.x;
    k[c] = i < n ? kin[i] : 0u;
  }
  const int m = (int)min((int64_t)kRadixItems, (n - base - threadIdx.x + kRadixThreads - 1) / kRadixThreads);
  // run-length pre-aggregation per thread: the high digits of depth keys take
  // a handful of values, which would serialise shared atomics on one address
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    uint32_t ld = 0, cnt = 0;
#pragma unroll
    for (int c = 0; c < kRadixItems; ++c) {
      if (c >= m) break;
      const uint32_t d = (k[c] >> (8 * p)) & 255u;
      if (cnt && d != ld) {
        atomicAdd(&h[p][ld], cnt);
        cnt = 0;
      }
      ld = d;
      ++cnt;
    }
    if (cnt) atomicAdd(&h[p][ld], cnt);
  }
  __syncthreads();
  uint32_t* g = ghist + (size_t)v * 4 * 256;
  for (int k = threadIdx.x; k < 4 * 256; k += kRadixThreads) {
    const uint32_t x = (&h[0][0])[k];
    if (x) atomicAdd(&g[k], x);
  }
}

// per (segment, pass): exclusive scan of the 256 digit counts
__global__ void __launch_bounds__(256) radix_digit_offsets_kernel(const uint32_t* __restrict__ ghist,
                                                                  uint32_t* __restrict__ goff) {
  __shared__ uint32_t ws[8];
  const int sp = blockIdx.x;  // segment * 4 + pass
  const uint32_t x = ghist[(size_t)sp * 256 + threadIdx.x];
  const uint32_t inc = warp_incl_scan(x);
  const int w = threadIdx.x >> 5;
  if (lane_id() == 31) ws[w] = inc;
  __syncthreads();
  uint32_t wo = 0;
  for (int k = 0; k < w; ++k) wo += ws[k];
  goff[(size_t)sp * 256 + threadIdx.x] = wo + inc - x;
}

// Depth mode: the four digit histograms of the visible depth keys of every
// view, and the visible count n_vis[v] (one atomic per CTA).
__device__ __forceinline__ bool rect_visible(short4 r) { return r.x <= r.z; }

__global__ void __launch_bounds__(kRadixThreads) depth_hist_kernel(const float* __restrict__ depth,
                                                                   const short4* __restrict__ rect, int64_t n,
                                                                   uint32_t* __restrict__ ghist,
                                                                   int32_t* __restrict__ n_vis) {
  __shared__ uint32_t h[4][256];
  __shared__ int32_t cnt;
  const int v = blockIdx.y;
  for (int k = threadIdx.x; k < 4 * 256; k += kRadixThreads) (&h[0][0])[k] = 0;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kRadixTile;
  const float* dv = depth + (int64_t)v * n;
  const short4* rv = rect + (int64_t)v * n;
  uint32_t k[kRadixItems];
  bool ok[kRadixItems];
  int mine = 0;
#pragma unroll
  for (int c = 0; c < kRadixItems; ++c) {
    const int64_t i = base + c * kRadixThreads + threadIdx.x;
    ok[c] = i < n && rect_visible(rv[i]);
    k[c] = ok[c] ? __float_as_uint(dv[i]) : 0u;
    mine += ok[c] ? 1 : 0;
  }
  // run-length pre-aggregation per thread (the high digits of depth keys take
  // a handful of values, which would serialise shared atomics on one address)
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    uint32_t ld = 0, cn = 0;
#pragma unroll
    for (int c = 0; c < kRadixItems; ++c) {
      if (!ok[c]) continue;
      const uint32_t d = (k[c] >> (8 * p)) & 255u;
      if (cn && d != ld) {
        atomicAdd(&h[p][ld], cn);
        cn = 0;
      }
      ld = d;
      ++cn;
    }
    if (cn) atomicAdd(&h[p][ld], cn);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
  if (lane_id() == 0 && mine) atomicAdd(&cnt, mine);
  __syncthreads();
  uint32_t* g = ghist + (size_t)v * 4 * 256;
  for (int q = threadIdx.x; q < 4 * 256; q += kRadixThreads) {
    const uint32_t x = (&h[0][0])[q];
    if (x) atomicAdd(&g[q], x);
  }
  if (threadIdx.x == 0 && cnt) atomicAdd(&n_vis[v], cnt);
}

// Per view (one warp): which digit passes run and where each reads / writes.
// src 0 = the projection (depth, rect), 1 = buffer A, 2 = buffer B; dst 1 =
// A, 2 = B; last = the values go to the final sorted array (keys dropped).
// Pass 0 always runs (it compacts the visible components).
struct RadixSched {
  int32_t active, src, dst, last;
};

__global__ void depth_sched_kernel(const uint32_t* __restrict__ ghist, RadixSched* __restrict__ sched) {
  const int v = blockIdx.x, lane = lane_id();
  int act[4];
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const uint32_t* hp = ghist + ((size_t)v * 4 + p) * 256;
    int nz = 0;
    for (int d = lane; d < 256; d += 32) nz += hp[d] != 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nz += __shfl_xor_sync(0xffffffffu, nz, o);
    act[p] = p == 0 || nz > 1;
  }
  if (lane != 0) return;
  int lastp = 0;
  for (int p = 0; p < 4; ++p) if (act[p]) lastp = p;
  int cur = 0;  // where the data are: 0 = projection, 1 = A, 2 = B
  for (int p = 0; p < 4; ++p) {
    RadixSched s;
    s.active = act[p];
    s.src = cur;
    s.dst = cur == 1 ? 2 : 1;
    s.last = p == lastp;
    if (act[p]) cur = s.dst;
    sched[v * 4 + p] = s;
  }
}

// One onesweep pass: stable scatter of one 4096-key tile by the digit at
// 8 * pass (see the header).  DEPTH: depth mode (schedule, compaction,
// implicit values, final array); otherwise plain (keys_in, vals_in) ->
// (keys_out, vals_out) over n keys per segment.
#ifndef SSS_RADIX_MINB
#define SSS_RADIX_MINB 4  // 64 registers (the depth mode spills at 48); the per-tile ranking is latency-bound
#endif
struct DepthSrc {  // depth-mode operands (unused in plain mode)
  const float* depth;
  const short4* rect;
  const int32_t* n_vis;
  const RadixSched* sched;
  uint32_t *ka, *kb;
  int32_t *va, *vb, *vf;  // vf: final sorted values [segment][n]
};

template <bool DEPTH>
__global__ void __launch_bounds__(kRadixThreads, SSS_RADIX_MINB) radix_onesweep_kernel(
    const uint32_t* __restrict__ keys_in, const int32_t* __restrict__ vals_in, int64_t n, int pass,
    int tiles, uint32_t* __restrict__ status, const uint32_t* __restrict__ goff,
    uint32_t* __restrict__ tickets, uint32_t* __restrict__ keys_out, int32_t* __restrict__ vals_out,
    DepthSrc ds) {
  __shared__ uint32_t run[kRadixWarps][256];
  __shared__ uint32_t tile_off[256];
  __shared__ uint32_t lstart[256];
  __shared__ uint32_t wsum[kRadixWarps];
  __shared__ uint32_t skey[kRadixTile];
  __shared__ int32_t sval[kRadixTile];
  __shared__ int s_tile;
  const int v = blockIdx.y;
  const int shift = 8 * pass;
  const int w = threadIdx.x >> 5, lane = lane_id();
  // this pass's operands
  bool from_proj = false, last = false;
  int64_t count = n;
  const uint32_t* kin;
  const int32_t* vin;
  uint32_t* kout;
  int32_t* vout;
  if (DEPTH) {
    const RadixSched sc = ds.sched[v * 4 + pass];
    if (!sc.active) return;
    from_proj = sc.src == 0;
    last = sc.last;
    count = from_proj ? n : (int64_t)ds.n_vis[v];
    kin = sc.src == 1 ? ds.ka : ds.kb;
    vin = sc.src == 1 ? ds.va : ds.vb;
    kout = sc.dst == 1 ? ds.ka : ds.kb;
    vout = last ? ds.vf : (sc.dst == 1 ? ds.va : ds.vb);
  } else {
    kin = keys_in; vin = vals_in; kout = keys_out; vout = vals_out;
  }
  if (threadIdx.x == 0) s_tile = (int)atomicAdd(&tickets[v * 4 + pass], 1u);  // launch order
  for (int k = threadIdx.x; k < kRadixWarps * 256; k += kRadixThreads) (&run[0][0])[k] = 0;
  __syncthreads();
  const int tile = s_tile;
  const int64_t tbase = (int64_t)tile * kRadixTile;
  if (tbase >= count) return;  // past the (compacted) segment: no later tile depends on it
  const int64_t base = tbase + w * (32 * kRadixItems);
  kin += (int64_t)v * n;
  vin += (int64_t)v * n;
  const float* dpv = DEPTH ? ds.depth + (int64_t)v * n : nullptr;
  const short4* rpv = DEPTH ? ds.rect + (int64_t)v * n : nullptr;
  uint32_t key[kRadixItems];
  uint32_t loc[kRadixItems];
  uint32_t okm = 0;  // bit c: item c is a valid (in range / visible) key
  const unsigned lt = (1u << lane) - 1u;
  // every tile but a segment's last: no bounds checks (never in the
  // filtering first depth pass)
  const bool full = !from_proj && tbase + kRadixTile <= count;
  if (full) {
#pragma unroll
    for (int c = 0; c < kRadixItems; ++c) key[c] = kin[base + c * 32 + lane];
    okm = (1u << kRadixItems) - 1u;
#pragma unroll
    for (int c = 0; c < kRadixItems; ++c) {
      const unsigned d = (key[c] >> shift) & 255u;
      const unsigned pm = peers_of(d);
      const uint32_t before = run[w][d];
      loc[c] = before + __popc(pm & lt);
      __syncwarp();
      if ((pm & lt) == 0) run[w][d] = before + __popc(pm);
      __syncwarp();
    }
  } else {
#pragma unroll
    for (int c = 0; c < kRadixItems; ++c) {
      const int64_t i = base + c * 32 + lane;
      bool ok;
      if (DEPTH && from_proj) {
        ok = i < n && rect_visible(rpv[i]);
        key[c] = ok ? __float_as_uint(dpv[i]) : 0u;
      } else {
        ok = i < count;
        key[c] = ok ? kin[i] : 0xFFFFFFFFu;
      }
      okm |= ok ? (1u << c) : 0u;
    }
#pragma unroll
    for (int c = 0; c < kRadixItems; ++c) {
      const bool ok = (okm >> c) & 1u;
      const unsigned d = (key[c] >> shift) & 255u;
      const unsigned valid = __ballot_sync(0xffffffffu, ok);
      const unsigned pm = peers_of(d) & valid;
      const uint32_t before = ok ? run[w][d] : 0u;
      loc[c] = before + __popc(pm & lt);
      __syncwarp();
      if (ok && (pm & lt) == 0) run[w][d] = before + __popc(pm);
      __syncwarp();
    }
  }
  __syncthreads();
  // per digit d (thread d): prefix over warps, tile count, tile-local start,
  // then the decoupled look-back for the tile's global offset
  int cnt;
  {
    const int d = threadIdx.x;
    uint32_t acc = 0;
    for (int ww = 0; ww < kRadixWarps; ++ww) {
      const uint32_t x = run[ww][d];
      run[ww][d] = acc;
      acc += x;
    }
    uint32_t* st = status + ((size_t)(v * 4 + pass) * tiles) * 256;
    st_relaxed(&st[(size_t)tile * 256 + d], (tile == 0 ? kStInc : kStAgg) | acc);
    uint32_t prefix = 0;
    for (int k = tile - 1; k >= 0; --k) {
      uint32_t s;
      do {
        s = ld_relaxed(&st[(size_t)k * 256 + d]);
      } while ((s & ~kStCount) == 0u);
      prefix += s & kStCount;
      if ((s & ~kStCount) == kStInc) break;
    }
    if (tile > 0) st_relaxed(&st[(size_t)tile * 256 + d], kStInc | (prefix + acc));
    tile_off[d] = goff[(size_t)(v * 4 + pass) * 256 + d] + prefix;
    const uint32_t inc = warp_incl_scan(acc);
    if (lane == 31) wsum[w] = inc;
    __syncthreads();
    uint32_t wo = 0, tot = 0;
    for (int ww = 0; ww < kRadixWarps; ++ww) {
      wo += ww < w ? wsum[ww] : 0u;
      tot += wsum[ww];
    }
    cnt = (int)tot;  // keys of this tile (after filtering)
    const uint32_t stt = wo + inc - acc;
    lstart[d] = stt;
    for (int ww = 0; ww < kRadixWarps; ++ww) run[ww][d] += stt;
  }
  __syncthreads();
#pragma unroll
  for (int c = 0; c < kRadixItems; ++c) {
    const int64_t i = base + c * 32 + lane;
    if ((okm >> c) & 1u) {
      const unsigned d = (key[c] >> shift) & 255u;
      const uint32_t lp = run[w][d] + loc[c];
      skey[lp] = key[c];
      sval[lp] = (DEPTH && from_proj) ? (int32_t)i : vin[i];
    }
  }
  __syncthreads();
  uint32_t* ko = kout + (int64_t)v * n;
  int32_t* vo = vout + (int64_t)v * n;
  for (int i = threadIdx.x; i < cnt; i += kRadixThreads) {
    const uint32_t k = skey[i];
    const unsigned d = (k >> shift) & 255u;
    const uint32_t pos = tile_off[d] + (uint32_t)i - lstart[d];
    if (!last) ko[pos] = k;
    vo[pos] = sval[i];
  }
}

// Sorts `n` pairs per segment (n_segs segments laid out back to back) by
// key, stably; the result is in (keys_a, vals_a), (keys_b, vals_b) is
// scratch.  ws: radix_ws_words(tiles, n_segs) uint32, tiles = ceil(n / 4096).
void radix_sort_pairs(uint32_t* keys_a, int32_t* vals_a, uint32_t* keys_b, int32_t* vals_b, int64_t n,
                      int n_segs, int tiles, uint32_t* ws, cudaStream_t s) {
  uint32_t* status = ws;
  uint32_t* ghist = status + (size_t)n_segs * 4 * 256 * tiles;
  uint32_t* goff = ghist + (size_t)n_segs * 4 * 256;
  uint32_t* tickets = goff + (size_t)n_segs * 4 * 256;
  cudaMemsetAsync(ws, 0, radix_ws_words(tiles, n_segs) * sizeof(uint32_t), s);
  const dim3 gr(tiles, n_segs);
  radix_hist_kernel<<<gr, kRadixThreads, 0, s>>>(keys_a, n, ghist);
  radix_digit_offsets_kernel<<<n_segs * 4, 256, 0, s>>>(ghist, goff);
  count_launch(2);
  uint32_t *kin = keys_a, *kout = keys_b;
  int32_t *vin = vals_a, *vout = vals_b;
  for (int pass = 0; pass < 4; ++pass) {
    radix_onesweep_kernel<false><<<gr, kRadixThreads, 0, s>>>(kin, vin, n, pass, tiles, status, goff, tickets,
                                                              kout, vout, DepthSrc{});
    count_launch();
    uint32_t* tk = kin; kin = kout; kout = tk;
    int32_t* tv = vin; vin = vout; vout = tv;
  }
}

// Depth mode (a2): per view, the visible components of the projection in
// (fp32 depth, index) order into sorted[v][0 .. n_vis[v]) and the visible
// count into n_vis[v] (zeroed here).  ka/kb/va/vb: [n_segs][n] scratch;
// ws: radix_ws_words(tiles, n_segs) words + n_segs * 4 RadixSched.
void depth_sort(const float* depth, const short4* rect, int64_t n, int n_segs, int tiles, uint32_t* ka,
                uint32_t* kb, int32_t* va, int32_t* vb, int32_t* sorted, int32_t* n_vis, uint32_t* ws,
                cudaStream_t s) {
  uint32_t* status = ws;
  uint32_t* ghist = status + (size_t)n_segs * 4 * 256 * tiles;
  uint32_t* goff = ghist + (size_t)n_segs * 4 * 256;
  uint32_t* tickets = goff + (size_t)n_segs * 4 * 256;
  RadixSched* sched = reinterpret_cast<RadixSched*>(ws + radix_ws_words(tiles, n_segs));
  cudaMemsetAsync(ws, 0, radix_ws_words(tiles, n_segs) * sizeof(uint32_t), s);
  cudaMemsetAsync(n_vis, 0, sizeof(int32_t) * n_segs, s);
  const dim3 gr(tiles, n_segs);
  depth_hist_kernel<<<gr, kRadixThreads, 0, s>>>(depth, rect, n, ghist, n_vis);
  radix_digit_offsets_kernel<<<n_segs * 4, 256, 0, s>>>(ghist, goff);
  depth_sched_kernel<<<n_segs, 32, 0, s>>>(ghist, sched);
  count_launch(3);
  const DepthSrc ds{depth, rect, n_vis, sched, ka, kb, va, vb, sorted};
  for (int pass = 0; pass < 4; ++pass) {
    radix_onesweep_kernel<true><<<gr, kRadixThreads, 0, s>>>(nullptr, nullptr, n, pass, tiles, status, goff,
                                                             tickets, nullptr, nullptr, ds);
    count_launch();
  }
}

inline size_t depth_sort_ws_words(int tiles, int n_segs) {
  return radix_ws_words(tiles, n_segs) + (size_t)n_segs * 4 * (sizeof(RadixSched) / 4);
}

}  // namespace
}  // namespace sss
