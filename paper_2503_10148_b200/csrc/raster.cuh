// Shared pieces of the forward and backward compositors (a3, a4).
#pragma once
#include "common.cuh"

namespace sss {

constexpr int kRasterThreads = 256;  // one thread per pixel of a 16x16 tile
constexpr int kBatch = 256;          // bin entries staged per shared-memory batch

struct RasterGeom {
  int width, height, tiles_x, tiles_y, shift, bins_x, n_bins;
  int64_t n, capacity;
};

bool raster_geom(const sss_projected* pr, const sss_bins* bins, const sss_camera* cams, int n_views,
                 RasterGeom& G);

// Pixel of this thread: warp w covers an 8x4 block so the lanes of a warp
// are spatially compact (coherent inclusion decisions per warp).
__device__ __forceinline__ void pixel_of(int tid, int& lx, int& ly) {
  const int w = tid >> 5, l = tid & 31;
  lx = ((w & 1) << 3) + (l & 7);
  ly = ((w >> 1) << 2) + (l >> 3);
}

// The fp32 inclusion quadratic h = A dx^2 + B2 dx dy + C dy^2 in the exact
// order of DESIGN.md §2 (intrinsics: never contracted / reassociated), so the
// inclusion decision h <= hmax is bit-identical to the oracle's.
__device__ __forceinline__ float h_f32(float px, float py, float4 a, float C) {
  const float dx = __fsub_rn(px, a.x);
  const float dy = __fsub_rn(py, a.y);
  const float bdy = __fmul_rn(a.w, dy);
  const float cdy = __fmul_rn(C, dy);
  const float cdy2 = __fmul_rn(cdy, dy);
  return __fmaf_rn(dx, __fmaf_rn(a.z, dx, bdy), cdy2);
}

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
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
