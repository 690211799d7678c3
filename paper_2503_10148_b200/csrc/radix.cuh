// Stable LSD radix sort of (uint32 key, int32 value) pairs, 4 x 8-bit digit
// passes, for independent segments of equal length (grid.y = segment).  Used
// by a2 (per-view depth keys) and NEXT-2 (relocation targets).  Each pass:
// per-tile digit histograms (upsweep), one exclusive scan per segment over
// the digit-major [256][tiles] table, then a stable downsweep that ranks
// keys with per-warp digit counters and reorders the 4096-key tile by digit
// in shared memory so that global stores leave as per-digit runs.
#pragma once
#include "common.cuh"

namespace sss {
namespace {

constexpr int kRadixThreads = 256;
constexpr int kRadixWarps = kRadixThreads / 32;
constexpr int kRadixItems = 16;
constexpr int kRadixTile = kRadixThreads * kRadixItems;  // 4096 keys per CTA

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

// exclusive scan of one view's digit-major histogram (256 * tiles entries):
// one CTA per view walks the array in coalesced 4096-entry chunks (4 per
// thread, warp-shuffle scans) carrying the running total.
__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t x) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, x, o);
    if ((int)lane_id() >= o) x += t;
  }
  return x;
}

__global__ void __launch_bounds__(1024) scan_u32_kernel(uint32_t* __restrict__ data, int64_t len_per_seg) {
  __shared__ uint32_t wsum[32];
  __shared__ uint32_t carry_s;
  uint32_t* d = data + (size_t)blockIdx.x * len_per_seg;
  const int t = threadIdx.x, w = t >> 5, lane = lane_id();
  uint32_t carry = 0;
  for (int64_t c0 = 0; c0 < len_per_seg; c0 += 4096) {
    uint32_t x[4];
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {  // thread t owns 4 consecutive entries
      const int64_t i = c0 + 4 * t + k;
      x[k] = i < len_per_seg ? d[i] : 0u;
      s += x[k];
    }
    const uint32_t inc = warp_incl_scan(s);
    if (lane == 31) wsum[w] = inc;
    __syncthreads();
    if (w == 0) {
      const uint32_t ws = wsum[lane];
      const uint32_t wi = warp_incl_scan(ws);
      wsum[lane] = wi - ws;
      if (lane == 31) carry_s = wi;
    }
    __syncthreads();
    uint32_t run = carry + wsum[w] + inc - s;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t i = c0 + 4 * t + k;
      if (i < len_per_seg) d[i] = run;
      run += x[k];
    }
    carry += carry_s;
    __syncthreads();
  }
}

// Stable scatter of one 4096-key tile by the digit at `shift`: ranks by
// per-warp digit counters (8 ballots per 32 keys, in key order), then the
// tile is reordered by digit in shared memory so that global stores go out
// as per-digit runs (~16 consecutive keys) instead of 32 random addresses
// per warp store.
__global__ void __launch_bounds__(kRadixThreads, 3) radix_downsweep_kernel(
    const uint32_t* __restrict__ keys_in, const int32_t* __restrict__ vals_in, int64_t n, int shift,
    int tiles, const uint32_t* __restrict__ hist, uint32_t* __restrict__ keys_out,
    int32_t* __restrict__ vals_out) {
  __shared__ uint32_t run[kRadixWarps][256];
  __shared__ uint32_t tile_off[256];
  __shared__ uint32_t lstart[256];
  __shared__ uint32_t wsum[kRadixWarps];
  __shared__ uint32_t skey[kRadixTile];
  __shared__ int32_t sval[kRadixTile];
  const int v = blockIdx.y, tile = blockIdx.x;
  const int w = threadIdx.x >> 5, lane = lane_id();
  for (int k = threadIdx.x; k < kRadixWarps * 256; k += kRadixThreads) (&run[0][0])[k] = 0;
  tile_off[threadIdx.x] = hist[((size_t)v * 256 + threadIdx.x) * tiles + tile];
  __syncthreads();
  const int64_t tbase = (int64_t)tile * kRadixTile;
  const int64_t base = tbase + w * (32 * kRadixItems);
  const uint32_t* kin = keys_in + (int64_t)v * n;
  const int32_t* vin = vals_in + (int64_t)v * n;
  uint32_t key[kRadixItems];
  uint32_t loc[kRadixItems];
#pragma unroll
  for (int c = 0; c < kRadixItems; ++c) {
    const int64_t i = base + c * 32 + lane;
    key[c] = i < n ? kin[i] : 0xFFFFFFFFu;
  }
  const unsigned lt = (1u << lane) - 1u;
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
  __syncthreads();
  // per digit: exclusive prefix over warps, tile count; then tile-local digit starts
  {
    const int d = threadIdx.x;
    uint32_t acc = 0;
    for (int ww = 0; ww < kRadixWarps; ++ww) {
      const uint32_t x = run[ww][d];
      run[ww][d] = acc;
      acc += x;
    }
    const uint32_t inc = warp_incl_scan(acc);
    if (lane == 31) wsum[w] = inc;
    __syncthreads();
    uint32_t wo = 0;
    for (int ww = 0; ww < w; ++ww) wo += wsum[ww];
    const uint32_t st = wo + inc - acc;
    lstart[d] = st;
    for (int ww = 0; ww < kRadixWarps; ++ww) run[ww][d] += st;
  }
  __syncthreads();
#pragma unroll
  for (int c = 0; c < kRadixItems; ++c) {
    const int64_t i = base + c * 32 + lane;
    if (i < n) {
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
// scratch.  hist: 256 * tiles * n_segs uint32, tiles = ceil(n / 4096).
void radix_sort_pairs(uint32_t* keys_a, int32_t* vals_a, uint32_t* keys_b, int32_t* vals_b, int64_t n,
                             int n_segs, int tiles, uint32_t* hist, cudaStream_t s) {
  const dim3 gr(tiles, n_segs);
  uint32_t *kin = keys_a, *kout = keys_b;
  int32_t *vin = vals_a, *vout = vals_b;
  for (int pass = 0; pass < 4; ++pass) {
    radix_upsweep_kernel<<<gr, kRadixThreads, 0, s>>>(kin, n, pass * 8, tiles, hist);
    scan_u32_kernel<<<n_segs, 1024, 0, s>>>(hist, (int64_t)256 * tiles);
    radix_downsweep_kernel<<<gr, kRadixThreads, 0, s>>>(kin, vin, n, pass * 8, tiles, hist, kout, vout);
    count_launch(3);
    uint32_t* tk = kin; kin = kout; kout = tk;
    int32_t* tv = vin; vin = vout; vout = tv;
  }
}

}  // namespace
}  // namespace sss
