// C-ABI plumbing shared by the entry points: validation, status strings,
// thread-local error message and launch counter.
#include <cmath>
#include <cstdarg>
#include <cstdio>

#include "common.cuh"

namespace sss {

static thread_local char g_err[512] = "";
static thread_local int64_t g_launches = 0;

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

sss_status check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return SSS_ERR_CUDA;
  }
  return SSS_OK;
}

void count_launch(int64_t k) { g_launches += k; }

sss_status validate_params(const sss_params* p, const char* what, bool allow_block) {
  if (!p) { set_error("%s: null params", what); return SSS_ERR_ARG; }
  if (p->n < 0) { set_error("%s: n < 0", what); return SSS_ERR_ARG; }
  if (p->block != 0) {
    if (!allow_block || p->block < 0 || p->block_planes < 12 + 3 * (p->sh_degree + 1) * (p->sh_degree + 1)) {
      set_error("%s: component-blocked layout not accepted here (or block_planes too small)", what);
      return SSS_ERR_ARG;
    }
    if (p->n > 0 && !p->mean) { set_error("%s: null buffer", what); return SSS_ERR_ARG; }
    if (p->n > (int64_t)INT32_MAX) { set_error("%s: n too large", what); return SSS_ERR_ARG; }
    return SSS_OK;
  }
  if (p->sh_degree < 0 || p->sh_degree > 3) {
    set_error("%s: sh_degree %d outside [0,3]", what, p->sh_degree);
    return SSS_ERR_ARG;
  }
  if (p->variant < 0 || p->variant > 7) { set_error("%s: variant %d outside [0,7]", what, p->variant); return SSS_ERR_ARG; }
  if (p->n > 0 && (!p->mean || !p->log_scale || !p->rot || !p->raw_nu || !p->raw_opacity || !p->sh)) {
    set_error("%s: null plane pointer", what);
    return SSS_ERR_ARG;
  }
  if (p->n > (int64_t)INT32_MAX) { set_error("%s: n too large", what); return SSS_ERR_ARG; }
  return SSS_OK;
}

sss_status validate_cams(const sss_camera* cams, int n_views, const char* what) {
  if (!cams || n_views <= 0) { set_error("%s: no cameras", what); return SSS_ERR_ARG; }
  for (int v = 0; v < n_views; ++v) {
    const sss_camera& c = cams[v];
    if (!(c.fx > 0.f) || !(c.fy > 0.f) || !(c.z_near > 0.f) || !std::isfinite(c.cx) ||
        !std::isfinite(c.cy)) {
      set_error("%s: camera %d has non-positive focal length or z_near", what, v);
      return SSS_ERR_ARG;
    }
    if (c.width <= 0 || c.height <= 0) {
      set_error("%s: camera %d has a zero-size image", what, v);
      return SSS_ERR_SHAPE;
    }
    if (c.width != cams[0].width || c.height != cams[0].height) {
      set_error("%s: all views must share one image size", what);
      return SSS_ERR_SHAPE;
    }
    if (c.width > 32767 * kTile || c.height > 32767 * kTile) {
      set_error("%s: image too large", what);
      return SSS_ERR_SHAPE;
    }
  }
  return SSS_OK;
}

bool fill_campack(const sss_camera* cams, int first, int count, CamPack& cp) {
  if (count > kMaxViewsPerLaunch) return false;
  cp.width = cams[0].width;
  cp.height = cams[0].height;
  cp.tiles_x = div_up(cp.width, kTile);
  cp.tiles_y = div_up(cp.height, kTile);
  for (int k = 0; k < count; ++k) {
    const sss_camera& c = cams[first + k];
    DevCamera& d = cp.cam[k];
    for (int i = 0; i < 9; ++i) d.R[i] = c.rot[i];
    for (int i = 0; i < 3; ++i) d.t[i] = c.trans[i];
    d.fx = c.fx; d.fy = c.fy; d.cx = c.cx; d.cy = c.cy; d.z_near = c.z_near;
    for (int i = 0; i < 3; ++i) {
      double s = (double)c.rot[0 * 3 + i] * c.trans[0] + (double)c.rot[1 * 3 + i] * c.trans[1] +
                 (double)c.rot[2 * 3 + i] * c.trans[2];
      d.center[i] = (float)(-s);
    }
  }
  return true;
}

}  // namespace sss

extern "C" const char* sss_status_string(sss_status s) {
  switch (s) {
    case SSS_OK: return "SSS_OK";
    case SSS_ERR_ARG: return "SSS_ERR_ARG: invalid argument";
    case SSS_ERR_SHAPE: return "SSS_ERR_SHAPE: invalid image / view shape";
    case SSS_ERR_CAPACITY: return "SSS_ERR_CAPACITY: bin capacity exceeded";
    case SSS_ERR_CUDA: return "SSS_ERR_CUDA: CUDA error";
  }
  return "SSS_ERR_UNKNOWN";
}

extern "C" const char* sss_last_error(void) { return sss::g_err; }

extern "C" int64_t sss_launch_count(int32_t reset) {
  int64_t v = sss::g_launches;
  if (reset) sss::g_launches = 0;
  return v;
}

