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

// One onesweep pass: stable scatter of one 4096-key tile by the digit at
// 8 * pass (see the header).
#ifndef SSS_RADIX_MINB
#define SSS_RADIX_MINB 4  // 64 registers, no spills: with interleaved views -0.05 ms vs 5 (48 registers + 40 B of stack), +0.45 ms at 6
#endif
__global__ void __launch_bounds__(kRadixThreads, SSS_RADIX_MINB) radix_onesweep_kernel(
    const uint32_t* __restrict__ keys_in, const int32_t* __restrict__ vals_in, int64_t n, int pass,
    int tiles, uint32_t* __restrict__ status, const uint32_t* __restrict__ goff,
    uint32_t* __restrict__ tickets, uint32_t* __restrict__ keys_out, int32_t* __restrict__ vals_out) {
  __shared__ uint32_t run[kRadixWarps][256];
  __shared__ uint32_t tile_off[256];
  __shared__ uint32_t lstart[256];
  __shared__ uint32_t wsum[kRadixWarps];
  __shared__ uint32_t skey[kRadixTile];
  __shared__ int32_t sval[kRadixTile];
  __shared__ int s_tile;
  // segments interleaved in launch order (block b: segment b % n_segs): a
  // tile's predecessor in its segment started n_segs blocks earlier, so its
  // published counts are usually there when the look-back reads them
  const int n_segs = (int)(gridDim.x / (unsigned)tiles);
  const int v = (int)(blockIdx.x % (unsigned)n_segs);
  const int shift = 8 * pass;
  const int w = threadIdx.x >> 5, lane = lane_id();
  if (threadIdx.x == 0) s_tile = (int)atomicAdd(&tickets[v * 4 + pass], 1u);  // launch order
  for (int k = threadIdx.x; k < kRadixWarps * 256; k += kRadixThreads) (&run[0][0])[k] = 0;
  __syncthreads();
  const int tile = s_tile;
  const int64_t tbase = (int64_t)tile * kRadixTile;
  const int64_t base = tbase + w * (32 * kRadixItems);
  const uint32_t* kin = keys_in + (int64_t)v * n;
  const int32_t* vin = vals_in + (int64_t)v * n;
  uint32_t key[kRadixItems];
  uint32_t loc[kRadixItems];
  const unsigned lt = (1u << lane) - 1u;
  const bool full = tbase + kRadixTile <= n;  // every tile but a segment's last: no bounds checks
  if (full) {
#pragma unroll
    for (int c = 0; c < kRadixItems; ++c) key[c] = kin[base + c * 32 + lane];
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
      key[c] = i < n ? kin[i] : 0xFFFFFFFFu;
    }
#pragma unroll
    for (int c = 0; c < kRadixItems; ++c) {
      const int64_t i = base + c * 32 + lane;
      const bool ok = i < n;
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
    uint32_t wo = 0;
    for (int ww = 0; ww < w; ++ww) wo += wsum[ww];
    const uint32_t stt = wo + inc - acc;
    lstart[d] = stt;
    for (int ww = 0; ww < kRadixWarps; ++ww) run[ww][d] += stt;
  }
  __syncthreads();
#pragma unroll
  for (int c = 0; c < kRadixItems; ++c) {
    const int64_t i = base + c * 32 + lane;
    if (full || i < n) {
      const unsigned d = (key[c] >> shift) & 255u;
      const uint32_t lp = run[w][d] + loc[c];
      skey[lp] = key[c];
      sval[lp] = vin[i];
    }
  }
  __syncthreads();
  const int cnt = (int)min((int64_t)kRadixTile, n - tbase);
  uint32_t* kout = keys_out + (int64_t)v * n;
  int32_t* vout = vals_out + (int64_t)v * n;
  for (int i = threadIdx.x; i < cnt; i += kRadixThreads) {
    const uint32_t k = skey[i];
    const unsigned d = (k >> shift) & 255u;
    const uint32_t pos = tile_off[d] + (uint32_t)i - lstart[d];
    kout[pos] = k;
    vout[pos] = sval[i];
  }
}

// Sorts `n` pairs per segment (n_segs segments laid out back to back) by
// key, stably; the result is in (keys_a, vals_a), (keys_b, vals_b) is
// scratch -- or, with vals_final, the sorted values go there (keys_a then
// holds the keys after the third pass only).  ws: radix_ws_words(tiles,
// n_segs) uint32, tiles = ceil(n / 4096).
void radix_sort_pairs(uint32_t* keys_a, int32_t* vals_a, uint32_t* keys_b, int32_t* vals_b, int64_t n,
                      int n_segs, int tiles, uint32_t* ws, cudaStream_t s, int32_t* vals_final = nullptr) {
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
    if (pass == 3 && vals_final) vout = vals_final;
    radix_onesweep_kernel<<<dim3(tiles * n_segs), kRadixThreads, 0, s>>>(kin, vin, n, pass, tiles, status, goff,
                                                                       tickets, kout, vout);
    count_launch();
    uint32_t* tk = kin; kin = kout; kout = tk;
    int32_t* tv = vin; vin = vout; vout = tv;
  }
}

}  // namespace
}  // namespace sss
