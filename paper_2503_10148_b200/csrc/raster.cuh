// Shared pieces of the forward and backward compositors (a3, a4).
#pragma once
#include "common.cuh"

namespace sss {

// A CTA renders one 16x16 tile of one view; each thread owns kPX horizontally
// adjacent pixels (a warp a 16 x 32/(16/kPX) strip).  With kPX = 4 the
// per-entry shared-memory loads, the warp inclusion test and (backward) the
// warp reduction are amortised over 128 pixels instead of 32.
#ifndef SSS_RASTER_PX
#define SSS_RASTER_PX 4
#endif
constexpr int kPX = SSS_RASTER_PX;
static_assert(kPX == 4, "4 pixels per thread (processed as pairs): one warp per 16x8 strip");
constexpr int kPairs = kPX / 2;
constexpr int kRasterThreads = 256 / kPX;
constexpr int kRasterWarps = kRasterThreads / 32;
constexpr int kBatch = kRasterThreads < 128 ? kRasterThreads : 128;  // entries per smem batch
constexpr int kWarpW = 16;                        // warp strip: 16x4 or 16x8 pixels
constexpr int kWarpH = 32 * kPX / kWarpW;
constexpr int kLanesPerRow = kWarpW / kPX;
// resident CTAs per SM the register allocation must allow (occupancy hides
// the fixed-latency FP32/MUFU dependency chains of the hot loops)
#ifndef SSS_FWD_MINB
#define SSS_FWD_MINB 20  // 48 registers: 40 warps per SM (measured: -7% vs 56 registers)
#endif
#ifndef SSS_BWD_MINB
// bwd: <= 93 registers (80 + 8 B of stack): 11 CTAs/SM, -0.6% vs 10 CTAs at
// 90 registers (with the lane constants opaque the loop needs fewer live
// values); deferring the warp reduction by one entry to overlap it with the
// next entry measured +9%
#define SSS_BWD_MINB 11
#endif
constexpr int kFwdMinBlocks = SSS_FWD_MINB;
constexpr int kBwdMinBlocks = SSS_BWD_MINB;
constexpr int kWarpsPerRow = 16 / kWarpW;
static_assert(kRasterWarps == SSS_TILE_LISTS, "one composited-entry list per warp strip");

// Per-warp staging of the bin-list entries: batches of 32 entries, double
// buffered, the 48-byte records (32-byte geometry + 16-byte colour) gathered
// with cp.async (LDGSTS) one batch
// ahead of the compute.
constexpr int kWB = 32;
#ifndef SSS_BWD_AOS
#define SSS_BWD_AOS 1
#endif
#if SSS_BWD_AOS
// one 64-byte slot per staged entry (the replay loop addresses its fields
// from one base with immediate offsets)
struct alignas(16) StageSlot {
  float4 r[3];
  int32_t pos, id, pad0, pad1;  // id: the caller's tag of the entry
};
struct WarpStage {
  StageSlot s[2][kWB];  // [buffer][slot]
  __device__ __forceinline__ float4& rec(int buf, int k, int j) { return s[buf][j].r[k]; }
  __device__ __forceinline__ int32_t& pos(int buf, int j) { return s[buf][j].pos; }
  __device__ __forceinline__ int32_t& id(int buf, int j) { return s[buf][j].id; }
};
#else
struct WarpStage {
  float4 r_[2][3][kWB];  // [buffer][record float4][slot]
  int32_t pos_[2][kWB], id_[2][kWB];  // id: the caller's tag of the entry
  __device__ __forceinline__ float4& rec(int buf, int k, int j) { return r_[buf][k][j]; }
  __device__ __forceinline__ int32_t& pos(int buf, int j) { return pos_[buf][j]; }
  __device__ __forceinline__ int32_t& id(int buf, int j) { return id_[buf][j]; }
};
#endif

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// Stages one batch: the lanes with `ok` are compacted in lane order (ballot)
// into slots of buffer `buf` (position and tag), their geometry and colour records
// gathered by cp.async;
// commits one async group (also when empty) and returns the entry count.
__device__ __forceinline__ int stage_batch(WarpStage& S, int buf, bool ok, int32_t pos, int32_t id,
                                           const float4* __restrict__ rv, const float4* __restrict__ cv,
                                           unsigned lt, int32_t tag) {
  const unsigned bal = __ballot_sync(0xffffffffu, ok);
  if (ok) {
    const int slot = __popc(bal & lt);
    const float4* src = rv + (int64_t)id * 2;
    cp_async16(&S.rec(buf, 0, slot), src);
    cp_async16(&S.rec(buf, 1, slot), src + 1);
    cp_async16(&S.rec(buf, 2, slot), cv + id);
    S.pos(buf, slot) = pos;
    S.id(buf, slot) = tag;
  }
  cp_async_commit();
  return __popc(bal);
}



// Development counters (variant builds with -DSSS_COUNTERS only).
#ifdef SSS_COUNTERS
static __device__ unsigned long long g_cnt[16];  // one set per translation unit
#define SSS_COUNT(i, x) atomicAdd(&g_cnt[(i)], (unsigned long long)(x))
#define SSS_COUNTER_ACCESSOR(NAME)                                                                  \
  extern "C" __attribute__((visibility("default"))) int NAME(unsigned long long* h, int reset) {   \
    if (cudaMemcpyFromSymbol(h, sss::g_cnt, sizeof(unsigned long long) * 16) != cudaSuccess) return 1; \
    if (reset) {                                                                                    \
      unsigned long long z[16] = {0};                                                               \
      if (cudaMemcpyToSymbol(sss::g_cnt, z, sizeof(z)) != cudaSuccess) return 1;                    \
    }                                                                                               \
    return 0;                                                                                       \
  }
#else
#define SSS_COUNTER_ACCESSOR(NAME)
#define SSS_COUNT(i, x) ((void)0)
#endif

struct RasterGeom {
  int width, height, tiles_x, tiles_y, shift, bins_x, n_bins;
  int64_t n, capacity;
  // truncated bin lists (sss_bins.max_per_bin > 0): the tile's list is the
  // bin's materialised entries [start, mend) followed by the virtual tail
  // sorted[resume .. n_vis) (positions mend, mend + 1, ...), rect-filtered;
  // nullptr = complete lists
  const int32_t* sorted;
  const int32_t* n_vis;
  const int32_t* resume;
  int32_t* used;  // adaptive truncation: per-bin consumption written by the forward (nullable)
  const uint16_t* tmask;  // per-entry tile masks of the bin lists (nullable, sss.h)
};

// Does bin-list entry `pos` (component id) belong to tile (tx, ty)?  The
// entry's tile mask bit when the bins carry masks (listed entries only),
// else its tile rect (a truncated list's tail is always rect-tested).
__device__ __forceinline__ bool entry_in_tile(const RasterGeom& G, const uint16_t* __restrict__ tmv, int32_t pos,
                                              int32_t mend, int id, const short4* __restrict__ rcv, int tx,
                                              int ty) {
  if (G.tmask && pos < mend) {
    const int m = G.shift;
    const int bit = ((ty & ((1 << m) - 1)) << m) | (tx & ((1 << m) - 1));
    return (__ldg(tmv + pos) >> bit) & 1;
  }
  const short4 r = rcv[id];
  return tx >= r.x && tx <= r.z && ty >= r.y && ty <= r.w;
}

// The list of the tile's bin as the raster walks it: positions [start, end)
// with end = mend + tail length; position p maps to a component through
// ids (p < mend) or the depth-sorted tail (p >= mend, always rect-filtered).
struct BinList {
  int32_t start, mend, end, tail0;  // tail0: sorted index of position mend
  const int32_t* ids;               // the view's ids
  const int32_t* tail;              // the view's sorted ids (or nullptr)
  __device__ __forceinline__ int32_t id(int32_t p) const {
    return p < mend ? __ldg(ids + p) : __ldg(tail + tail0 + (p - mend));
  }
};

__device__ __forceinline__ BinList bin_list(const RasterGeom& G, const int32_t* __restrict__ ids,
                                            const int32_t* __restrict__ ranges, int v, int bin) {
  BinList L;
  L.start = ranges[((int64_t)v * G.n_bins + bin) * 2 + 0];
  L.mend = ranges[((int64_t)v * G.n_bins + bin) * 2 + 1];
  L.end = L.mend;
  L.ids = ids + (int64_t)v * G.capacity;
  L.tail = nullptr;
  L.tail0 = 0;
  if (G.sorted) {
    L.tail0 = G.resume[(int64_t)v * G.n_bins + bin];
    L.end = L.mend + (G.n_vis[v] - L.tail0);
    L.tail = G.sorted + (int64_t)v * G.n;
  }
  return L;
}

bool raster_geom(const sss_projected* pr, const sss_bins* bins, const sss_camera* cams, int n_views,
                 RasterGeom& G);

// First pixel of this thread (the others follow at lx + 1, ...) and the
// origin of its warp's strip, within the tile.
__device__ __forceinline__ void pixels_of(int tid, int& lx, int& ly, int& sx, int& sy) {
  const int w = tid >> 5, l = tid & 31;
  sx = (w % kWarpsPerRow) * kWarpW;
  sy = (w / kWarpsPerRow) * kWarpH;
  lx = sx + (l % kLanesPerRow) * kPX;
  ly = sy + l / kLanesPerRow;
}

// The fp32 inclusion quadratic h = A dx^2 + B2 dx dy + C dy^2 in the exact
// order of DESIGN.md §2 (intrinsics: never contracted / reassociated), so the
// inclusion decision h <= hmax is bit-identical to the fp64 reference's fp32
// test.  bdy = B2*dy and cdy2 = (C*dy)*dy depend only on the row.
__device__ __forceinline__ float h_f32_row(float px, float mx, float A, float bdy, float cdy2) {
  const float dx = __fsub_rn(px, mx);
  return __fmaf_rn(dx, __fmaf_rn(A, dx, bdy), cdy2);
}

// Packed FP32x2 arithmetic (FADD2 / FMUL2 / FFMA2, sm_100): a thread's pixels
// are processed as horizontally adjacent pairs, so one issue slot does the
// work of two scalar instructions.  Each lane of a packed op is the IEEE
// round-to-nearest result of the scalar op, never contracted.
__device__ __forceinline__ float2 bc2(float s) { return make_float2(s, s); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 sub2(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }

// h_f32_row for a pixel pair (same three rounded operations per lane), also
// returning dx.
__device__ __forceinline__ float2 h_f32_pair(float2 px, float mx, float A, float bdy, float cdy2, float2& dx) {
  dx = __fadd2_rn(px, bc2(-mx));
  return __ffma2_rn(dx, __ffma2_rn(bc2(A), dx, bc2(bdy)), bc2(cdy2));
}

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float lg2_approx(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// log2(1 + t) for t >= 0.  Small nu (<= 32): MUFU lg2 (abs error ~2^-22,
// times |e| <= 17 in the exponent).  Large nu: the exponent e = -(nu+2)/2
// magnifies the error, so use the accurate log1p (warp-uniform branch: all
// lanes evaluate the same component).
__device__ __forceinline__ float log2_1p(float t, bool precise) {
  return precise ? log1pf(t) * 1.4426950408889634f : lg2_approx(1.0f + t);
}

}  // namespace sss
