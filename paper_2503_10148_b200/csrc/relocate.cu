// NEXT-2 — sss_relocate: one component-recycling pass (PAPER.md:168-183,
// Eqs. 11-12; SM "Component Recycling" PAPER.md:1317-1460; implementation
// PAPER.md:1081 "recycle components with low opacity to high opacity
// components every n iterations by creating a Multinomial distribution of
// opacity values").  Readings R29-R31:
//   dead      |o| < threshold, o = fp32(tanh(raw_o)) (fp64 tanh, rounded once);
//   selected  the first floor(cap_frac n) dead in index order (5% cap);
//   targets   multinomial over the live components, P(i) ~ |o_i|, with exact
//             integer weights w_i = floor(|o_i| 2^32): draw j maps 64 Philox
//             bits r_j (counter (j, 0x52454C4F, step), key seed) to
//             u = floor(r_j total / 2^64) and takes the first i whose
//             inclusive prefix sum of w exceeds u;
//   groups    a target keeps at most n_max - 1 dead, in draw order;
//   Eq. 12    N = group size incl. the target, nu_new = nu_old:
//             (1 - o_new)^N = 1 - o_old,
//             Sigma_new = o_old^2 (beta(1/2, (nu+2)/2) / K)^2 Sigma_old,
//             K = sum_{i=1}^N sum_{k<i} C(i-1,k) (-1)^k o_new^{k+1}
//                 beta(1/2, ((k+1)(nu+3)-1)/2)          (fp64, ln Gamma);
//             every member takes the target's mean, rotation, nu and SH,
//             raw_o = atanh(o_new), log_scale += ln(Sigma scale)/2; momentum
//             and Adam moments of the members are reset.
// Every integer decision (dead set, targets, groups) is exact and matches
// the oracle bit for bit.
//
// B200 design: elementwise weight pass, a decoupled multi-block inclusive
// scan of the 64-bit weights and of the dead flags, compaction of the
// selected dead, one thread per draw (binary search over the prefix sums),
// the shared stable radix sort (radix.cuh) of (target, draw) pairs, and one
// thread per group head for the fp64 Eq. 12 arithmetic and the copies.  The
// pass runs every n iterations, so it is latency-, not bandwidth-, critical.
#include <curand_philox4x32_x.h>

#include "radix.cuh"

namespace sss {
namespace {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;  // 1024 values per block

struct RelocWs {
  size_t w, dead, bsum_w, bsum_d, list, keys_a, vals_a, keys_b, vals_b, hist, scal, total;
  int64_t cap;
  int n_blocks, tiles;
};

inline size_t a256(size_t x) { return (x + 255) & ~(size_t)255; }

RelocWs reloc_ws(int64_t n) {
  RelocWs L;
  L.cap = n;  // worst case (cap_frac <= 1)
  L.n_blocks = div_up(n > 0 ? n : 1, kScanTile);
  L.tiles = div_up(L.cap > 0 ? L.cap : 1, kRadixTile);
  size_t off = 0;
  auto take = [&](size_t b) { size_t o = off; off += a256(b); return o; };
  L.w = take((size_t)n * 8);          // weights -> inclusive prefix sums
  L.dead = take((size_t)n * 8);       // dead flags -> inclusive prefix counts
  L.bsum_w = take((size_t)L.n_blocks * 8);
  L.bsum_d = take((size_t)L.n_blocks * 8);
  L.list = take((size_t)L.cap * 4);   // selected dead, index order
  L.keys_a = take((size_t)L.cap * 4);
  L.vals_a = take((size_t)L.cap * 4);
  L.keys_b = take((size_t)L.cap * 4);
  L.vals_b = take((size_t)L.cap * 4);
  L.hist = take(radix_ws_words(L.tiles, 1) * 4);
  L.scal = take(64);                  // n_sel (int64), total (uint64)
  L.total = off;
  return L;
}

// weights and dead flags
__device__ __forceinline__ double opacity_d(double raw, bool positive) {
  return positive ? 1.0 / (1.0 + exp(-raw)) : tanh(raw);
}

__global__ void reloc_weights_kernel(const float* __restrict__ raw_o, int64_t n, float thr, bool positive,
                                     uint64_t* __restrict__ w, uint64_t* __restrict__ dead) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float a = fabsf((float)opacity_d((double)raw_o[i], positive));
  const bool d = a < thr;
  dead[i] = d ? 1ull : 0ull;
  w[i] = d ? 0ull : (uint64_t)floor((double)a * 4294967296.0);
}

__device__ __forceinline__ uint64_t warp_incl_scan64(uint64_t x) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t t = __shfl_up_sync(0xffffffffu, x, o);
    if ((int)lane_id() >= o) x += t;
  }
  return x;
}

// block-local inclusive scan of 1024 values (4 consecutive per thread); the
// block total goes to bsum
__device__ void block_scan_tile(uint64_t* data, int64_t n, uint64_t* bsum, uint64_t carry_in, bool add_carry) {
  __shared__ uint64_t ws[kScanThreads / 32];
  const int64_t base = (int64_t)blockIdx.x * kScanTile + threadIdx.x * kScanItems;
  uint64_t x[kScanItems];
  uint64_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    x[k] = base + k < n ? data[base + k] : 0ull;
    s += x[k];
  }
  const uint64_t inc = warp_incl_scan64(s);
  const int w = threadIdx.x >> 5;
  if (lane_id() == 31) ws[w] = inc;
  __syncthreads();
  uint64_t wo = 0;
  for (int k = 0; k < w; ++k) wo += ws[k];
  uint64_t run = wo + inc - s + (add_carry ? carry_in : 0ull);
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    run += x[k];
    if (base + k < n) data[base + k] = run;
  }
  if (bsum && threadIdx.x == kScanThreads - 1) bsum[blockIdx.x] = wo + inc;
}

__global__ void __launch_bounds__(kScanThreads) scan_tiles_kernel(uint64_t* data, int64_t n, uint64_t* bsum) {
  block_scan_tile(data, n, bsum, 0ull, false);
}

// exclusive scan of the block totals (one block, sequential chunks)
__global__ void __launch_bounds__(1024) scan_bsum_kernel(uint64_t* bsum, int nb) {
  __shared__ uint64_t ws[32];
  __shared__ uint64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int c0 = 0; c0 < nb; c0 += 1024) {
    const int i = c0 + threadIdx.x;
    const uint64_t x = i < nb ? bsum[i] : 0ull;
    const uint64_t inc = warp_incl_scan64(x);
    const int w = threadIdx.x >> 5;
    if (lane_id() == 31) ws[w] = inc;
    __syncthreads();
    uint64_t wo = 0;
    for (int k = 0; k < w; ++k) wo += ws[k];
    const uint64_t c = carry;
    if (i < nb) bsum[i] = c + wo + inc - x;
    __syncthreads();
    if (threadIdx.x == 1023) carry = c + wo + inc;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kScanThreads) add_carry_kernel(uint64_t* data, int64_t n, const uint64_t* bsum) {
  const int64_t base = (int64_t)blockIdx.x * kScanTile;
  const uint64_t c = bsum[blockIdx.x];
  for (int k = threadIdx.x; k < kScanTile; k += kScanThreads)
    if (base + k < n) data[base + k] += c;
}

// n_sel = min(n_dead, cap); total weight
__global__ void reloc_counts_kernel(const uint64_t* cum_w, const uint64_t* cum_d, int64_t n, int64_t cap,
                                    int64_t* n_sel, uint64_t* total) {
  const int64_t nd = (int64_t)cum_d[n - 1];
  *n_sel = nd < cap ? nd : cap;
  *total = cum_w[n - 1];
}

__global__ void reloc_compact_kernel(const uint64_t* __restrict__ cum_d, int64_t n, const int64_t* n_sel,
                                     int32_t* __restrict__ list) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t c = cum_d[i];
  const bool d = c != (i > 0 ? cum_d[i - 1] : 0ull);
  if (d && (int64_t)c - 1 < *n_sel) list[c - 1] = (int32_t)i;
}

__global__ void reloc_draw_kernel(const uint64_t* __restrict__ cum_w, int64_t n, const int64_t* n_sel,
                                  const uint64_t* total_p, int64_t cap, uint32_t key0, uint32_t key1,
                                  uint32_t s_lo, uint32_t s_hi, uint32_t* __restrict__ tkey,
                                  int32_t* __restrict__ tval) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= cap) return;
  const int64_t ns = *n_sel;
  const uint64_t total = *total_p;
  if (j >= ns || total == 0) {  // padding sorts last and is never a group
    tkey[j] = 0xFFFFFFFFu;
    tval[j] = (int32_t)j;
    return;
  }
  const uint4 x = curand_Philox4x32_10(make_uint4((uint32_t)j, 0x52454C4Fu, s_lo, s_hi), make_uint2(key0, key1));
  const uint64_t r64 = (uint64_t)x.x | ((uint64_t)x.y << 32);
  const uint64_t u = __umul64hi(r64, total);
  int64_t lo = 0, hi = n - 1;  // first i with cum_w[i] > u
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (cum_w[mid] > u) hi = mid; else lo = mid + 1;
  }
  tkey[j] = (uint32_t)lo;
  tval[j] = (int32_t)j;
}

__device__ double beta_lg(double x, double y) { return exp(lgamma(x) + lgamma(y) - lgamma(x + y)); }

// one thread per sorted position; group heads do the work
__global__ void reloc_apply_kernel(const uint32_t* __restrict__ tkey, const int32_t* __restrict__ tval,
                                   const int32_t* __restrict__ list, const int64_t* n_sel, int n_max,
                                   sss_params P, sss_params Mo, sss_params Vo, float* __restrict__ r,
                                   int32_t* __restrict__ target_of, int64_t* __restrict__ n_moved) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t ns = *n_sel;
  if (s >= ns) return;
  const uint32_t t = tkey[s];
  if (t == 0xFFFFFFFFu || (s > 0 && tkey[s - 1] == t)) return;  // not a group head
  int acc = 0;
  while (acc < n_max - 1 && s + acc < ns && tkey[s + acc] == t) ++acc;
  const int N = 1 + acc;
  const int64_t n = P.n;
  const int Pn = 12 + 3 * (P.sh_degree + 1) * (P.sh_degree + 1);
  // Eq. 12 in fp64 from the target's fp32 state
  const bool positive = P.variant & SSS_VARIANT_POSITIVE;
  const double o_old = opacity_d((double)P.raw_opacity[t], positive);
  const double raw_nu = (double)P.raw_nu[t];
  const double sp = raw_nu > 30.0 ? raw_nu : log1p(exp(raw_nu));
  const double nu = fmin(1.0 + sp, 1e4);
  const double o_new = 1.0 - pow(1.0 - o_old, 1.0 / N);
  double K = 0.0;
  for (int k = 0; k < N; ++k) {  // sum_{i=k+1}^{N} C(i-1, k) = C(N, k+1) terms of the double sum
    double binom_sum = 0.0, binom = 1.0;  // C(i-1, k) for i = k+1 .. N
    for (int i = k + 1; i <= N; ++i) {
      binom_sum += binom;
      binom = binom * (double)i / (double)(i - k);
    }
    K += binom_sum * ((k & 1) ? -1.0 : 1.0) * pow(o_new, k + 1) * beta_lg(0.5, ((k + 1) * (nu + 3.0) - 1.0) / 2.0);
  }
  const double b = beta_lg(0.5, (nu + 2.0) / 2.0);
  const double scale = o_old * o_old * (b / K) * (b / K);
  const float raw_o_new = (float)(positive ? log(o_new / (1.0 - o_new)) : atanh(o_new));
  const double dls = 0.5 * log(scale);
  // the target's new state, then copied to every member
  P.raw_opacity[t] = raw_o_new;
  for (int j = 0; j < 3; ++j) P.log_scale[j * n + t] = (float)((double)P.log_scale[j * n + t] + dls);
  auto reset = [&](int64_t d) {
    for (int p = 0; p < Pn; ++p) {
      Mo.mean[(int64_t)p * n + d] = 0.f;  // planes are consecutive from mean (flat buffer)
      Vo.mean[(int64_t)p * n + d] = 0.f;
    }
    for (int a = 0; a < 3; ++a) r[(int64_t)a * n + d] = 0.f;
  };
  reset(t);
  for (int q = 0; q < acc; ++q) {
    const int64_t d = list[tval[s + q]];
    for (int p = 0; p < Pn; ++p) P.mean[(int64_t)p * n + d] = P.mean[(int64_t)p * n + t];
    reset(d);
    if (target_of) target_of[d] = (int32_t)t;
  }
  atomicAdd((unsigned long long*)n_moved, (unsigned long long)acc);
}

}  // namespace
}  // namespace sss

using namespace sss;

extern "C" size_t sss_relocate_workspace(int64_t n) {
  if (n < 0) return 0;
  return reloc_ws(n).total;
}

static bool flat_planes(const sss_params* p) {
  const int64_t n = p->n;
  const int K = (p->sh_degree + 1) * (p->sh_degree + 1);
  return p->log_scale == p->mean + 3 * n && p->rot == p->mean + 6 * n && p->raw_nu == p->mean + 10 * n &&
         p->raw_opacity == p->mean + 11 * n && p->sh == p->mean + 12 * n && K >= 1;
}

extern "C" sss_status sss_relocate(sss_params* p, sss_params* adam_m, sss_params* adam_v, float* momentum,
                                   const sss_relocate_params* rp, int32_t* target_of, int64_t* n_moved,
                                   void* ws, size_t ws_bytes, void* stream) {
  sss_status st;
  if ((st = validate_params(p, "sss_relocate")) != SSS_OK) return st;
  if ((st = validate_params(adam_m, "sss_relocate(m)")) != SSS_OK) return st;
  if ((st = validate_params(adam_v, "sss_relocate(v)")) != SSS_OK) return st;
  if (!rp || !n_moved || (p->n > 0 && !momentum)) { set_error("sss_relocate: null argument"); return SSS_ERR_ARG; }
  if (adam_m->n != p->n || adam_v->n != p->n || adam_m->sh_degree != p->sh_degree || adam_v->sh_degree != p->sh_degree) {
    set_error("sss_relocate: n / sh_degree mismatch");
    return SSS_ERR_ARG;
  }
  if (p->n > 0 && (!flat_planes(p) || !flat_planes(adam_m) || !flat_planes(adam_v))) {
    set_error("sss_relocate: parameter planes must be one flat [P][n] buffer");
    return SSS_ERR_ARG;
  }
  if (!(rp->threshold > 0.f && rp->threshold < 1.f) || !(rp->cap_frac >= 0.f && rp->cap_frac <= 1.f) ||
      rp->n_max < 2 || rp->n_max > 64) {
    set_error("sss_relocate: threshold in (0,1), cap_frac in [0,1], n_max in [2,64]");
    return SSS_ERR_ARG;
  }
  if (p->n > (int64_t)0x7FFFFFFF) { set_error("sss_relocate: n >= 2^31"); return SSS_ERR_ARG; }
  cudaStream_t s = (cudaStream_t)stream;
  cudaMemsetAsync(n_moved, 0, sizeof(int64_t), s);
  const int64_t n = p->n;
  if (target_of && n > 0) cudaMemsetAsync(target_of, 0xFF, sizeof(int32_t) * n, s);
  const int64_t cap = (int64_t)floor((double)rp->cap_frac * (double)n);
  if (n == 0 || cap == 0) return check_launch("sss_relocate");
  const RelocWs L = reloc_ws(n);
  if (!ws || ws_bytes < L.total) { set_error("sss_relocate: workspace %zu < %zu bytes", ws_bytes, L.total); return SSS_ERR_ARG; }
  char* w = (char*)ws;
  uint64_t* cw = (uint64_t*)(w + L.w);
  uint64_t* cd = (uint64_t*)(w + L.dead);
  uint64_t* bw = (uint64_t*)(w + L.bsum_w);
  uint64_t* bd = (uint64_t*)(w + L.bsum_d);
  int32_t* list = (int32_t*)(w + L.list);
  uint32_t* ka = (uint32_t*)(w + L.keys_a);
  int32_t* va = (int32_t*)(w + L.vals_a);
  uint32_t* kb = (uint32_t*)(w + L.keys_b);
  int32_t* vb = (int32_t*)(w + L.vals_b);
  uint32_t* hist = (uint32_t*)(w + L.hist);
  int64_t* n_sel = (int64_t*)(w + L.scal);
  uint64_t* total = (uint64_t*)(w + L.scal + 8);
  const int eb = div_up(n, 256);
  reloc_weights_kernel<<<eb, 256, 0, s>>>(p->raw_opacity, n, rp->threshold, (p->variant & SSS_VARIANT_POSITIVE) != 0,
                                          cw, cd);
  for (int q = 0; q < 2; ++q) {
    uint64_t* data = q ? cd : cw;
    uint64_t* bs = q ? bd : bw;
    scan_tiles_kernel<<<L.n_blocks, kScanThreads, 0, s>>>(data, n, bs);
    scan_bsum_kernel<<<1, 1024, 0, s>>>(bs, L.n_blocks);
    add_carry_kernel<<<L.n_blocks, kScanThreads, 0, s>>>(data, n, bs);
  }
  reloc_counts_kernel<<<1, 1, 0, s>>>(cw, cd, n, cap, n_sel, total);
  reloc_compact_kernel<<<eb, 256, 0, s>>>(cd, n, n_sel, list);
  reloc_draw_kernel<<<div_up(cap, 256), 256, 0, s>>>(cw, n, n_sel, total, cap, (uint32_t)rp->seed,
                                                      (uint32_t)(rp->seed >> 32), (uint32_t)rp->step,
                                                      (uint32_t)((uint64_t)rp->step >> 32), ka, va);
  count_launch(10);
  const int tiles = div_up(cap, kRadixTile);
  radix_sort_pairs(ka, va, kb, vb, cap, 1, tiles, hist, s);
  reloc_apply_kernel<<<div_up(cap, 256), 256, 0, s>>>(ka, va, list, n_sel, rp->n_max, *p, *adam_m, *adam_v,
                                                       momentum, target_of, n_moved);
  count_launch();
  return check_launch("sss_relocate");
}
