// Shared device helpers of the SSS CUDA path (sm_100a).  Nothing here is
// shared with oracle/ (the oracle is an independent fp64 CPU program).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "sss.h"

namespace sss {

constexpr int kTile = SSS_TILE;
constexpr int kMaxViewsPerLaunch = 128;
constexpr float kAlphaMax = 0.99f;   // R10
constexpr float kWStop = 1e-4f;      // R11
constexpr double kNuMax = 1e4;
constexpr float kLowpass = 0.3f;     // setting 1's low-pass
constexpr float kGaussExp2 = -0.72134752044448170f;  // -log2(e)/2: exp(-h/2) = 2^(kGaussExp2 h)

struct DevCamera {  // a camera as the kernels see it
  float R[9];
  float t[3];
  float fx, fy, cx, cy;
  float center[3];  // -R^T t
  float z_near;
};

struct CamPack {  // passed by value (kernel parameter space)
  int n;
  int width, height, tiles_x, tiles_y;
  DevCamera cam[kMaxViewsPerLaunch];
};

inline int div_up(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

// thread-local error plumbing (abi.cu)
void set_error(const char* fmt, ...);
sss_status check_launch(const char* what);
void count_launch(int64_t k = 1);
bool fill_campack(const sss_camera* cams, int first, int count, CamPack& cp);
sss_status validate_params(const sss_params* p, const char* what, bool allow_block = false);

// The plane pointers and plane stride of component i's storage: plain [P][n]
// (stride n), or its block of a component-blocked set (sss.h sss_params.block;
// pointers offset so that plane_ptr[k * stride + i] addresses component i).
__device__ __forceinline__ sss_params block_view(const sss_params& G, int64_t i, int64_t& stride) {
  if (G.block <= 0) {
    stride = G.n;
    return G;
  }
  const int64_t B = G.block, b = i / B;
  stride = B;
  float* base = G.mean + b * (int64_t)G.block_planes * B - b * B;
  sss_params V = G;
  V.mean = base;
  V.log_scale = base + 3 * B;
  V.rot = base + 6 * B;
  V.raw_nu = base + 10 * B;
  V.raw_opacity = base + 11 * B;
  V.sh = base + 12 * B;
  return V;
}
sss_status validate_cams(const sss_camera* cams, int n_views, const char* what);

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31; }


}  // namespace sss
