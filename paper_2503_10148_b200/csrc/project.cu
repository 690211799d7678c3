// a1 — sss_project: EWA projection of every component into V views.
//
// PAPER.md:85-92 (Eq. 4: mu2D = (W mu + t)_{1:2} / (W mu + t)_3,
// Sigma2D = (J W Sigma W^T J^T)_{1:2,1:2}), 1116-1215 (affine closure and
// marginalisation -> 2D t with exponent -(nu+2)/2), 1077-1079 (nu in
// [1, 1e4], opacity-aware truncation, no low-pass filter).
//
// Design (B200): one thread per component, looping over up to 128 views of
// the launch, so the 60 parameter floats (240 B at SH degree 3) are read from
// HBM once per launch instead of once per view.  Loads are coalesced SoA
// plane reads; the per-view outputs (32 B geometry record + 16 B colour record
// + 4 B depth + 8 B rect) are written contiguously.  HBM-bound: 240 B + 60 B/view per component.
//
// Precision: every quantity that feeds a discrete decision (depth key, tile
// rect, the fp32 inclusion test of the compositor) is computed in fp64 in the
// canonical evaluation order of DESIGN.md §2 and rounded to fp32 once.  This
// file is compiled with -fmad=false so no multiply-add is contracted (the
// canonical order is left-to-right sums of products).  The SH colour is not
// discrete-feeding and is computed in fp32.
#include <math.h>

#include "common.cuh"

namespace sss {
namespace {

struct ViewIndep {  // view-independent fp64 quantities of one component
  double nu, o, hmax;
  double Sig[9];
};

__device__ __forceinline__ void sh_eval(int deg, float x, float y, float z, const float* sh,
                                        float out[3]) {
  // Real SH basis, degree <= 3 (3DGS-lineage sign convention, R7).
  float Y[16];
  Y[0] = 0.28209479177387814f;
  int K = 1;
  if (deg >= 1) {
    Y[1] = -0.4886025119029199f * y;
    Y[2] = 0.4886025119029199f * z;
    Y[3] = -0.4886025119029199f * x;
    K = 4;
  }
  if (deg >= 2) {
    const float xx = x * x, yy = y * y, zz = z * z;
    Y[4] = 1.0925484305920792f * x * y;
    Y[5] = -1.0925484305920792f * y * z;
    Y[6] = 0.31539156525252005f * (2.f * zz - xx - yy);
    Y[7] = -1.0925484305920792f * x * z;
    Y[8] = 0.5462742152960396f * (xx - yy);
    K = 9;
  }
  if (deg >= 3) {
    const float xx = x * x, yy = y * y, zz = z * z;
    Y[9] = -0.5900435899266435f * y * (3.f * xx - yy);
    Y[10] = 2.890611442640554f * x * y * z;
    Y[11] = -0.4570457994644658f * y * (4.f * zz - xx - yy);
    Y[12] = 0.3731763325901154f * z * (2.f * zz - 3.f * xx - 3.f * yy);
    Y[13] = -0.4570457994644658f * x * (4.f * zz - xx - yy);
    Y[14] = 1.445305721320277f * z * (xx - yy);
    Y[15] = -0.5900435899266435f * x * (xx - 3.f * yy);
    K = 16;
  }
  // colour is not discrete-feeding: fused multiply-adds (explicit, this file
  // is compiled with -fmad=false for the fp64 geometry)
  for (int c = 0; c < 3; ++c) {
    float acc = 0.f;
    for (int m = 0; m < K; ++m) acc = __fmaf_rn(sh[m * 3 + c], Y[m], acc);
    out[c] = fmaxf(acc + 0.5f, 0.f);
  }
}

// The cameras as the fp64 geometry uses them: converted to double once on the
// host (exact), so the per-view loop does no float->double conversions
// (F2F.F64.F32 runs on the XU pipe with the fp64 divisions and square roots).
struct DevCameraD {
  double R[9];
  double t[3];
  double fx, fy, cx, cy, z_near;
  float center[3];  // fp32 (the SH view direction is fp32)
  float pad;
};
struct CamPackD {
  int n, width, height, tiles_x, tiles_y;
  DevCameraD cam[kMaxViewsPerLaunch];
};
static_assert(sizeof(CamPackD) < 32000, "kernel parameter space");

void fill_campack_d(const CamPack& f, int nv, CamPackD& d) {
  d.n = nv; d.width = f.width; d.height = f.height; d.tiles_x = f.tiles_x; d.tiles_y = f.tiles_y;
  for (int k = 0; k < nv; ++k) {
    const DevCamera& c = f.cam[k];
    DevCameraD& o = d.cam[k];
    for (int i = 0; i < 9; ++i) o.R[i] = (double)c.R[i];
    for (int i = 0; i < 3; ++i) o.t[i] = (double)c.t[i];
    o.fx = c.fx; o.fy = c.fy; o.cx = c.cx; o.cy = c.cy; o.z_near = c.z_near;
    for (int i = 0; i < 3; ++i) o.center[i] = c.center[i];
    o.pad = 0.f;
  }
}

template <int DEG>
#ifndef SSS_PROJ_MINB
#define SSS_PROJ_MINB 4  // 128 registers, 16 warps/SM (measured -20% vs 160 registers)
#endif
__global__ void __launch_bounds__(128, SSS_PROJ_MINB) project_kernel(sss_params P, const __grid_constant__ CamPackD cp,
                                                       int nv, int v0, float4* __restrict__ rec,
                                                       float4* __restrict__ col,
                                                       float* __restrict__ depth,
                                                       short4* __restrict__ rect) {
  constexpr int K = (DEG + 1) * (DEG + 1);
  const int64_t n = P.n;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int tiles_x = cp.tiles_x, tiles_y = cp.tiles_y;
  // ---- parameters (coalesced plane loads)
  double mu[3], q[4], s[3];
  for (int k = 0; k < 3; ++k) mu[k] = P.mean[k * n + i];
  for (int k = 0; k < 3; ++k) s[k] = P.log_scale[k * n + i];
  for (int k = 0; k < 4; ++k) q[k] = P.rot[k * n + i];
  const double raw_nu = P.raw_nu[i];
  const double raw_o = P.raw_opacity[i];
  float sh[3 * K];
#pragma unroll
  for (int k = 0; k < 3 * K; ++k) sh[k] = P.sh[k * n + i];
  const float muf[3] = {(float)mu[0], (float)mu[1], (float)mu[2]};

  // ---- view-independent part (fp64, canonical order)
  ViewIndep vi;
  {
    const double sp = raw_nu > 30.0 ? raw_nu : log1p(exp(raw_nu));
    vi.nu = fmin(1.0 + sp, kNuMax);
    vi.o = (P.variant & SSS_VARIANT_POSITIVE) ? 1.0 / (1.0 + exp(-raw_o)) : tanh(raw_o);
    const double qn = sqrt(((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3]);
    const double w = q[0] / qn, x = q[1] / qn, y = q[2] / qn, z = q[3] / qn;
    double R[9];
    R[0] = 1.0 - 2.0 * (y * y + z * z);
    R[1] = 2.0 * (x * y - w * z);
    R[2] = 2.0 * (x * z + w * y);
    R[3] = 2.0 * (x * y + w * z);
    R[4] = 1.0 - 2.0 * (x * x + z * z);
    R[5] = 2.0 * (y * z - w * x);
    R[6] = 2.0 * (x * z - w * y);
    R[7] = 2.0 * (y * z + w * x);
    R[8] = 1.0 - 2.0 * (x * x + y * y);
    const double S[3] = {exp(s[0]), exp(s[1]), exp(s[2])};
    double M[9];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) M[a * 3 + b] = R[a * 3 + b] * S[b];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b)
        vi.Sig[a * 3 + b] = (M[a * 3 + 0] * M[b * 3 + 0] + M[a * 3 + 1] * M[b * 3 + 1]) + M[a * 3 + 2] * M[b * 3 + 2];
    vi.hmax = vi.nu * expm1((2.0 / (vi.nu + 2.0)) * log(255.0 * fabs(vi.o)));
    if (P.variant & SSS_VARIANT_GAUSSIAN) vi.hmax = 2.0 * log(255.0 * fabs(vi.o));  // |o| e^{-h/2} = 1/255
  }
  const bool opaque_enough = 255.0 * fabs(vi.o) > 1.0;  // R25
  const float hmax_f = (float)vi.hmax;
  const float o_f = (float)vi.o;
  // Gaussian variant: inv_nu = 0 marks the kernel exp(-h/2) in the record
  const bool gauss = P.variant & SSS_VARIANT_GAUSSIAN;
  const float inv_nu_f = gauss ? 0.f : (float)(1.0 / vi.nu);
  const float e_f = gauss ? -0.5f : (float)(-(vi.nu + 2.0) / 2.0);
  const bool lowpass = P.variant & SSS_VARIANT_LOWPASS;

  for (int vv = 0; vv < nv; ++vv) {
    const DevCameraD& cam = cp.cam[vv];
    const int64_t o_idx = (int64_t)(v0 + vv) * n + i;
    double p[3];
    for (int a = 0; a < 3; ++a)
      p[a] = ((cam.R[a * 3 + 0] * mu[0] + cam.R[a * 3 + 1] * mu[1]) +
              cam.R[a * 3 + 2] * mu[2]) + cam.t[a];
    depth[o_idx] = (float)p[2];
    short4 rr = make_short4(1, 1, 0, 0);  // culled
    float4 r0 = make_float4(0.f, 0.f, 0.f, 0.f), r1 = r0, r2 = r0;
    bool vis = opaque_enough && (p[2] > cam.z_near);
    if (vis) {
      const double px = p[0], py = p[1], pz = p[2];
      const double fx = cam.fx, fy = cam.fy;
      // one fp64 reciprocal per view instead of six divisions (canonical
      // order of DESIGN.md §2, mirrored by the oracle)
      const double iz = 1.0 / pz;
      double J[6];
      J[0] = fx * iz; J[1] = 0.0; J[2] = -(fx * px) * (iz * iz);
      J[3] = 0.0; J[4] = fy * iz; J[5] = -(fy * py) * (iz * iz);
      double T1[9], Sc[9];
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b)
          T1[a * 3 + b] = (cam.R[a * 3 + 0] * vi.Sig[0 * 3 + b] + cam.R[a * 3 + 1] * vi.Sig[1 * 3 + b]) +
                          cam.R[a * 3 + 2] * vi.Sig[2 * 3 + b];
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b)
          Sc[a * 3 + b] = (T1[a * 3 + 0] * cam.R[b * 3 + 0] + T1[a * 3 + 1] * cam.R[b * 3 + 1]) +
                          T1[a * 3 + 2] * cam.R[b * 3 + 2];
      // K = J Sc and Sigma2D = K J^T in the canonical left-to-right order with
      // the structural zeros of J (J01 = J10 = 0) dropped: a (finite) zero
      // product added to a sum leaves it unchanged, so the values equal the
      // full sums the oracle evaluates
      double K2[6];
      for (int b = 0; b < 3; ++b) {
        K2[0 * 3 + b] = J[0] * Sc[0 * 3 + b] + J[2] * Sc[2 * 3 + b];
        K2[1 * 3 + b] = J[4] * Sc[1 * 3 + b] + J[5] * Sc[2 * 3 + b];
      }
      double cxx = K2[0] * J[0] + K2[2] * J[2];
      const double cxy = K2[1] * J[4] + K2[2] * J[5];
      double cyy = K2[4] * J[4] + K2[5] * J[5];
      if (lowpass) {
        cxx = cxx + 0.3;
        cyy = cyy + 0.3;
      }
      const double det = cxx * cyy - cxy * cxy;
      const double idet = 1.0 / det;
      const double A = cyy * idet, B = -cxy * idet, C = cxx * idet;
      const double mx = (fx * px) * iz + cam.cx;
      const double my = (fy * py) * iz + cam.cy;
      const float mx_f = (float)mx, my_f = (float)my;
      const float A_f = (float)A, B2_f = (float)(2.0 * B), C_f = (float)C;
      vis = ((float)det > 0.0f) && isfinite(mx_f) && isfinite(my_f) && isfinite(A_f) &&
            isfinite(B2_f) && isfinite(C_f) && isfinite(hmax_f);
      if (vis) {
        const double ex = sqrt((double)hmax_f * cxx) + 1.0;
        const double ey = sqrt((double)hmax_f * cyy) + 1.0;
        double fx0 = floor(((double)mx_f - ex) / kTile), fx1 = floor(((double)mx_f + ex) / kTile);
        double fy0 = floor(((double)my_f - ey) / kTile), fy1 = floor(((double)my_f + ey) / kTile);
        fx0 = fmax(fx0, 0.0); fy0 = fmax(fy0, 0.0);
        fx1 = fmin(fx1, (double)(tiles_x - 1)); fy1 = fmin(fy1, (double)(tiles_y - 1));
        vis = (fx0 <= fx1) && (fy0 <= fy1);
        if (vis) {
          rr = make_short4((short)fx0, (short)fy0, (short)fx1, (short)fy1);
          // SH colour from the view direction (fp32, not discrete-feeding)
          float d[3] = {muf[0] - cam.center[0], muf[1] - cam.center[1], muf[2] - cam.center[2]};
          const float inv = rsqrtf(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
          float col[3];
          sh_eval(DEG, d[0] * inv, d[1] * inv, d[2] * inv, sh, col);
          r0 = make_float4(mx_f, my_f, A_f, B2_f);
          r1 = make_float4(C_f, hmax_f, o_f, inv_nu_f);
          r2 = make_float4(e_f, col[0], col[1], col[2]);
        }
      }
    }
    rec[o_idx * 2 + 0] = r0;
    rec[o_idx * 2 + 1] = r1;
    col[o_idx] = r2;
    rect[o_idx] = rr;
  }
}

}  // namespace
}  // namespace sss

using namespace sss;

extern "C" sss_status sss_project(const sss_params* p, const sss_camera* cams, int32_t n_views,
                                  sss_projected* out, void* stream) {
  sss_status st = validate_params(p, "sss_project");
  if (st != SSS_OK) return st;
  if ((st = validate_cams(cams, n_views, "sss_project")) != SSS_OK) return st;
  if (!out || !out->rec || !out->depth || !out->rect || !out->col) {
    if (p->n > 0) { set_error("sss_project: null output"); return SSS_ERR_ARG; }
  }
  if (out->n != p->n || out->n_views != n_views) {
    set_error("sss_project: output sized for n=%lld V=%d, got n=%lld V=%d", (long long)out->n,
              out->n_views, (long long)p->n, n_views);
    return SSS_ERR_ARG;
  }
  if (p->n == 0) return SSS_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int threads = 128;
  const int blocks = div_up(p->n, threads);
  // Cameras travel as a __grid_constant__ kernel parameter (<= 128 views per
  // launch), so the call allocates nothing and is CUDA-graph capturable.
  for (int v0 = 0; v0 < n_views; v0 += kMaxViewsPerLaunch) {
    const int nv = n_views - v0 < kMaxViewsPerLaunch ? n_views - v0 : kMaxViewsPerLaunch;
    CamPack cpf;
    fill_campack(cams, v0, nv, cpf);
    static thread_local CamPackD cp;  // ~19 KB: kept off the stack
    fill_campack_d(cpf, nv, cp);
    float4* rec = (float4*)out->rec;
    float4* col = (float4*)out->col;
    short4* rect = (short4*)out->rect;
    switch (p->sh_degree) {
      case 0: project_kernel<0><<<blocks, threads, 0, s>>>(*p, cp, nv, v0, rec, col, out->depth, rect); break;
      case 1: project_kernel<1><<<blocks, threads, 0, s>>>(*p, cp, nv, v0, rec, col, out->depth, rect); break;
      case 2: project_kernel<2><<<blocks, threads, 0, s>>>(*p, cp, nv, v0, rec, col, out->depth, rect); break;
      default: project_kernel<3><<<blocks, threads, 0, s>>>(*p, cp, nv, v0, rec, col, out->depth, rect); break;
    }
    count_launch();
    if ((st = check_launch("sss_project")) != SSS_OK) return st;
  }
  return SSS_OK;
}
