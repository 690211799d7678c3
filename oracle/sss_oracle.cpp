// ============================================================================
// SSS ORACLE — TEST INFRASTRUCTURE ONLY.
//
// Plain, slow, fp64 CPU reference for the hot path of Student Splatting and
// Scooping (arXiv 2503.10148).  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs may load this library.  It
// shares no code, header, table or constant with the CUDA path
// (paper_2503_10148_b200/csrc, include/sss.h); the two meet only through the
// seeded inputs of sss_synth/.
//
// Every function cites the PAPER.md passage it follows (line numbers refer to
// /root/reference/PAPER.md; section names in brackets).  Where the paper is
// silent the DESIGN.md reading "Rnn" is named.  Parity status per function is
// listed in DESIGN.md §3 ("oracle pins").
//
// Build: g++ -O2 -std=c++17 -fopenmp -ffp-contract=off -fPIC -shared
// (-ffp-contract=off: the fp32 inclusion test must be evaluated exactly as
// written, see orc_h_f32).
// ============================================================================
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

extern "C" {

typedef struct {
  double R[9];   // world->camera rotation W (row-major); PAPER.md:88-92 (Eq. 4)
  double t[3];   // translation t (Eq. 4)
  double fx, fy, cx, cy;
  int32_t width, height;
  double z_near;  // R24
} orc_cam;

typedef struct {
  int64_t n;
  int32_t sh_degree;
  int32_t variant;  // NEXT-3 ablation variants (bit flags, see kVar*); 0 = SSS
  const double* planes;  // [P][n], P = 12 + 3K; mean 0..2, log_scale 3..5,
                         // rot 6..9 (w,x,y,z), raw_nu 10, raw_opacity 11,
                         // sh 12 + 3k + c
} orc_params;

typedef struct {
  float *mx, *my, *A, *B2, *C, *hmax, *depth;  // [n] fp32-rounded (R9, §8(c) step 4)
  int32_t* rect;                               // [n][4] inclusive tile rect
  int32_t *n_tiles, *cull;                     // [n]
  double* p;                                   // [n][3] camera-space mean
  double* mean2d;                              // [n][2]
  double* cov2d;                               // [n][3] xx, xy, yy
  double* conic;                               // [n][3] A, B, C of (Sigma2D)^-1
  double *nu, *o;                              // [n]
  double* color;                               // [n][3] clamped SH colour
} orc_proj_out;

typedef struct {
  double lr, friction, noise, gate_k, gate_t;
  int32_t burn_in, g_adam;
  double lr_scale, lr_rot, lr_nu, lr_opacity, lr_sh;
  double beta1, beta2, adam_eps, grad_scale;
  int64_t step;
  uint64_t seed;
  double eps_o, eps_sigma;  // regularizer weights of Eq. 8
  int32_t mu_mode;   // NEXT-3: 0 SGHMC (Eq. 10), 1 SGLD (F disabled), 2 Adam on mu (setting 1)
  int32_t variant;   // parameter-set variant (opacity map of the gate / regularizer)
} orc_sghmc_hp;

}  // extern "C"

namespace {

constexpr int kTile = 16;
constexpr double kNuMax = 1e4;        // PAPER.md:1077 "limit the range of nu from 1 to 10000"
constexpr double kAlphaClamp = 0.99;  // R10
constexpr double kWStop = 1e-4;       // R11

inline int sh_K(int deg) { return (deg + 1) * (deg + 1); }

// NEXT-3: the paper's ablation variants (R32), as flags
// of the parameter set: positive opacity o = sigmoid(raw) (settings 1-2,
// "positive t-dis"), the Gaussian kernel of 3DGS ("SGHMC with Gaussian
// distributions"), and the +0.3 low-pass on the projected covariance
// (setting 1).
constexpr int kVarPositive = 1, kVarGaussian = 2, kVarLowpass = 4;
constexpr double kLowpass = 0.3;
inline int n_planes(int deg) { return 12 + 3 * sh_K(deg); }

// ---------------------------------------------------------------- SH basis
// Real spherical harmonics, degree <= 3, in the 3DGS-lineage sign convention
// the paper builds on ("represented by spherical harmonics and
// view-dependent").  Constants are written from their closed
// forms; pinned against scipy.special.sph_harm_y in tests (R7).
void sh_basis(int deg, double x, double y, double z, double* Y) {
  const double pi = M_PI;
  const double c0 = 0.5 * std::sqrt(1.0 / pi);
  Y[0] = c0;
  if (deg < 1) return;
  const double c1 = std::sqrt(3.0 / (4.0 * pi));
  Y[1] = -c1 * y;
  Y[2] = c1 * z;
  Y[3] = -c1 * x;
  if (deg < 2) return;
  const double c20 = 0.5 * std::sqrt(15.0 / pi);
  const double c22 = 0.25 * std::sqrt(5.0 / pi);
  const double c24 = 0.25 * std::sqrt(15.0 / pi);
  Y[4] = c20 * x * y;
  Y[5] = -c20 * y * z;
  Y[6] = c22 * (2.0 * z * z - x * x - y * y);
  Y[7] = -c20 * x * z;
  Y[8] = c24 * (x * x - y * y);
  if (deg < 3) return;
  const double c30 = 0.25 * std::sqrt(35.0 / (2.0 * pi));
  const double c31 = 0.5 * std::sqrt(105.0 / pi);
  const double c32 = 0.25 * std::sqrt(21.0 / (2.0 * pi));
  const double c33 = 0.25 * std::sqrt(7.0 / pi);
  const double c35 = 0.25 * std::sqrt(105.0 / pi);
  Y[9] = -c30 * y * (3.0 * x * x - y * y);
  Y[10] = c31 * x * y * z;
  Y[11] = -c32 * y * (4.0 * z * z - x * x - y * y);
  Y[12] = c33 * z * (2.0 * z * z - 3.0 * x * x - 3.0 * y * y);
  Y[13] = -c32 * x * (4.0 * z * z - x * x - y * y);
  Y[14] = c35 * z * (x * x - y * y);
  Y[15] = -c30 * x * (x * x - 3.0 * y * y);
}

// d Y_m / d(x, y, z), treating the direction components as free variables.
void sh_basis_grad(int deg, double x, double y, double z, double* G /*[16][3]*/) {
  const double pi = M_PI;
  for (int i = 0; i < 48; ++i) G[i] = 0.0;
  if (deg < 1) return;
  const double c1 = std::sqrt(3.0 / (4.0 * pi));
  G[1 * 3 + 1] = -c1;
  G[2 * 3 + 2] = c1;
  G[3 * 3 + 0] = -c1;
  if (deg < 2) return;
  const double c20 = 0.5 * std::sqrt(15.0 / pi);
  const double c22 = 0.25 * std::sqrt(5.0 / pi);
  const double c24 = 0.25 * std::sqrt(15.0 / pi);
  G[4 * 3 + 0] = c20 * y;   G[4 * 3 + 1] = c20 * x;
  G[5 * 3 + 1] = -c20 * z;  G[5 * 3 + 2] = -c20 * y;
  G[6 * 3 + 0] = -2.0 * c22 * x; G[6 * 3 + 1] = -2.0 * c22 * y; G[6 * 3 + 2] = 4.0 * c22 * z;
  G[7 * 3 + 0] = -c20 * z;  G[7 * 3 + 2] = -c20 * x;
  G[8 * 3 + 0] = 2.0 * c24 * x; G[8 * 3 + 1] = -2.0 * c24 * y;
  if (deg < 3) return;
  const double c30 = 0.25 * std::sqrt(35.0 / (2.0 * pi));
  const double c31 = 0.5 * std::sqrt(105.0 / pi);
  const double c32 = 0.25 * std::sqrt(21.0 / (2.0 * pi));
  const double c33 = 0.25 * std::sqrt(7.0 / pi);
  const double c35 = 0.25 * std::sqrt(105.0 / pi);
  G[9 * 3 + 0] = -6.0 * c30 * x * y;
  G[9 * 3 + 1] = -c30 * (3.0 * x * x - 3.0 * y * y);
  G[10 * 3 + 0] = c31 * y * z; G[10 * 3 + 1] = c31 * x * z; G[10 * 3 + 2] = c31 * x * y;
  G[11 * 3 + 0] = 2.0 * c32 * x * y;
  G[11 * 3 + 1] = -c32 * (4.0 * z * z - x * x - 3.0 * y * y);
  G[11 * 3 + 2] = -8.0 * c32 * y * z;
  G[12 * 3 + 0] = -6.0 * c33 * x * z;
  G[12 * 3 + 1] = -6.0 * c33 * y * z;
  G[12 * 3 + 2] = c33 * (6.0 * z * z - 3.0 * x * x - 3.0 * y * y);
  G[13 * 3 + 0] = -c32 * (4.0 * z * z - 3.0 * x * x - y * y);
  G[13 * 3 + 1] = 2.0 * c32 * x * y;
  G[13 * 3 + 2] = -8.0 * c32 * x * z;
  G[14 * 3 + 0] = 2.0 * c35 * x * z;
  G[14 * 3 + 1] = -2.0 * c35 * y * z;
  G[14 * 3 + 2] = c35 * (x * x - y * y);
  G[15 * 3 + 0] = -c30 * (3.0 * x * x - 3.0 * y * y);
  G[15 * 3 + 1] = 6.0 * c30 * x * y;
}

// ------------------------------------------------------ parameter maps
// R1: nu = min(1 + softplus(raw), 1e4)
double nu_of(double raw) {
  const double sp = raw > 30.0 ? raw : std::log1p(std::exp(raw));
  return std::min(1.0 + sp, kNuMax);
}
double dnu_draw(double raw) {
  if (nu_of(raw) >= kNuMax) return 0.0;
  return 1.0 / (1.0 + std::exp(-raw));
}
// R2: o = tanh(raw)  ("we constrain the opacity by a tanh function");
// positive variant (R32): o = sigmoid(raw), the 3DGS opacity.
double opacity_of(double raw, int variant = 0) {
  if (variant & kVarPositive) return 1.0 / (1.0 + std::exp(-raw));
  return std::tanh(raw);
}
double dopacity_draw(double o, int variant) {
  return (variant & kVarPositive) ? o * (1.0 - o) : 1.0 - o * o;
}

// Rotation from a (w,x,y,z) unit quaternion ("Sigma = R S S^T R^T").
void quat_to_R(const double q[4], double R[9]) {
  const double w = q[0], x = q[1], y = q[2], z = q[3];
  R[0] = 1.0 - 2.0 * (y * y + z * z);
  R[1] = 2.0 * (x * y - w * z);
  R[2] = 2.0 * (x * z + w * y);
  R[3] = 2.0 * (x * y + w * z);
  R[4] = 1.0 - 2.0 * (x * x + z * z);
  R[5] = 2.0 * (y * z - w * x);
  R[6] = 2.0 * (x * z - w * y);
  R[7] = 2.0 * (y * z + w * x);
  R[8] = 1.0 - 2.0 * (x * x + y * y);
}

struct Comp {  // one component's parameters, promoted to fp64
  double mu[3], s[3], q[4], raw_nu, raw_o;
  double sh[48];
};

void load_comp(const orc_params* P, int64_t i, Comp& c) {
  const int64_t n = P->n;
  const double* a = P->planes;
  for (int k = 0; k < 3; ++k) c.mu[k] = a[(0 + k) * n + i];
  for (int k = 0; k < 3; ++k) c.s[k] = a[(3 + k) * n + i];
  for (int k = 0; k < 4; ++k) c.q[k] = a[(6 + k) * n + i];
  c.raw_nu = a[10 * n + i];
  c.raw_o = a[11 * n + i];
  const int K = sh_K(P->sh_degree);
  for (int k = 0; k < 3 * K; ++k) c.sh[k] = a[(12 + k) * n + i];
}

// All intermediate quantities of the projection of one component into one
// view.  Evaluation order of every quantity that feeds a discrete decision
// follows DESIGN.md §2 "canonical order" (left-to-right sums, no fusion).
struct Proj {
  int variant;
  // Eq. 3 / R1-R3
  double nu, o, qn, qh[4], Rq[9], S[3], M[9], Sig[9];
  // Eq. 4
  double p[3], J[6], Sc[9], cov[3], det, conic[3], mean2d[2];
  double hmax;
  // colour
  double dir[3], dist, Y[16], pre[3], color[3];
  // fp32 record + culling
  float mx_f, my_f, A_f, B2_f, C_f, hmax_f, depth_f;
  int rect[4];
  int n_tiles;
  int cull;
};

void project(const Comp& c, int deg, const orc_cam& cam, Proj& r, int variant = 0) {
  r.variant = variant;
  r.nu = nu_of(c.raw_nu);
  r.o = opacity_of(c.raw_o, variant);
  // q normalisation
  r.qn = std::sqrt(((c.q[0] * c.q[0] + c.q[1] * c.q[1]) + c.q[2] * c.q[2]) + c.q[3] * c.q[3]);
  for (int k = 0; k < 4; ++k) r.qh[k] = c.q[k] / r.qn;
  quat_to_R(r.qh, r.Rq);
  for (int k = 0; k < 3; ++k) r.S[k] = std::exp(c.s[k]);
  // M = R S ; Sigma = M M^T = R S S^T R^T
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r.M[i * 3 + j] = r.Rq[i * 3 + j] * r.S[j];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      r.Sig[i * 3 + j] = (r.M[i * 3 + 0] * r.M[j * 3 + 0] + r.M[i * 3 + 1] * r.M[j * 3 + 1]) +
                         r.M[i * 3 + 2] * r.M[j * 3 + 2];
  // camera-space mean  p = W mu + t   (Eq. 4)
  for (int i = 0; i < 3; ++i)
    r.p[i] = ((cam.R[i * 3 + 0] * c.mu[0] + cam.R[i * 3 + 1] * c.mu[1]) + cam.R[i * 3 + 2] * c.mu[2]) +
             cam.t[i];
  r.cull = 0;
  r.n_tiles = 0;
  r.rect[0] = r.rect[1] = 0;
  r.rect[2] = r.rect[3] = -1;
  // view direction for SH colour (R7): from the camera centre to mu
  {
    double cc[3];
    for (int i = 0; i < 3; ++i)
      cc[i] = -((cam.R[0 * 3 + i] * cam.t[0] + cam.R[1 * 3 + i] * cam.t[1]) + cam.R[2 * 3 + i] * cam.t[2]);
    double v[3] = {c.mu[0] - cc[0], c.mu[1] - cc[1], c.mu[2] - cc[2]};
    r.dist = std::sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
    for (int i = 0; i < 3; ++i) r.dir[i] = v[i] / r.dist;
    for (int m = 0; m < 16; ++m) r.Y[m] = 0.0;
    sh_basis(deg, r.dir[0], r.dir[1], r.dir[2], r.Y);
    const int K = sh_K(deg);
    for (int ch = 0; ch < 3; ++ch) {
      double acc = 0.0;
      for (int m = 0; m < K; ++m) acc += c.sh[m * 3 + ch] * r.Y[m];
      r.pre[ch] = acc + 0.5;
      r.color[ch] = std::max(0.0, r.pre[ch]);
    }
  }
  const double px = r.p[0], py = r.p[1], pz = r.p[2];
  r.depth_f = (float)pz;
  // R24: near-plane cull
  if (!(pz > cam.z_near)) { r.cull = 1; return; }
  // Jacobian of the pinhole map at p (EWA affine approximation; Eq. 4, R4),
  // through the one reciprocal iz = 1/pz (canonical order)
  const double iz = 1.0 / pz;
  r.J[0] = cam.fx * iz; r.J[1] = 0.0; r.J[2] = -(cam.fx * px) * (iz * iz);
  r.J[3] = 0.0; r.J[4] = cam.fy * iz; r.J[5] = -(cam.fy * py) * (iz * iz);
  // Sigma_c = W Sigma W^T
  double T1[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      T1[i * 3 + j] = (cam.R[i * 3 + 0] * r.Sig[0 * 3 + j] + cam.R[i * 3 + 1] * r.Sig[1 * 3 + j]) +
                      cam.R[i * 3 + 2] * r.Sig[2 * 3 + j];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      r.Sc[i * 3 + j] = (T1[i * 3 + 0] * cam.R[j * 3 + 0] + T1[i * 3 + 1] * cam.R[j * 3 + 1]) +
                        T1[i * 3 + 2] * cam.R[j * 3 + 2];
  // Sigma2D = (J W Sigma W^T J^T)   (Eq. 4)
  double K2[6];
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 3; ++j)
      K2[i * 3 + j] = (r.J[i * 3 + 0] * r.Sc[0 * 3 + j] + r.J[i * 3 + 1] * r.Sc[1 * 3 + j]) +
                      r.J[i * 3 + 2] * r.Sc[2 * 3 + j];
  r.cov[0] = (K2[0] * r.J[0] + K2[1] * r.J[1]) + K2[2] * r.J[2];
  r.cov[1] = (K2[0] * r.J[3] + K2[1] * r.J[4]) + K2[2] * r.J[5];
  r.cov[2] = (K2[3] * r.J[3] + K2[4] * r.J[4]) + K2[5] * r.J[5];
  if (variant & kVarLowpass) {  // setting 1's "small value (0.3)"
    r.cov[0] = r.cov[0] + kLowpass;
    r.cov[2] = r.cov[2] + kLowpass;
  }
  r.det = r.cov[0] * r.cov[2] - r.cov[1] * r.cov[1];
  const double idet = 1.0 / r.det;  // conic = (Sigma2D)^-1 through one reciprocal
  r.conic[0] = r.cov[2] * idet;
  r.conic[1] = -r.cov[1] * idet;
  r.conic[2] = r.cov[0] * idet;
  r.mean2d[0] = (cam.fx * px) * iz + cam.cx;
  r.mean2d[1] = (cam.fy * py) * iz + cam.cy;
  // L9 cutoff: pair included iff |o| T >= 1/255  <=>  h <= hmax  (R9)
  r.hmax = r.nu * std::expm1((2.0 / (r.nu + 2.0)) * std::log(255.0 * std::fabs(r.o)));
  if (variant & kVarGaussian) r.hmax = 2.0 * std::log(255.0 * std::fabs(r.o));  // |o| e^{-h/2} = 1/255
  r.mx_f = (float)r.mean2d[0];
  r.my_f = (float)r.mean2d[1];
  r.A_f = (float)r.conic[0];
  r.B2_f = (float)(2.0 * r.conic[1]);
  r.C_f = (float)r.conic[2];
  r.hmax_f = (float)r.hmax;
  if (!(255.0 * std::fabs(r.o) > 1.0)) { r.cull = 2; return; }  // R25
  if (!((float)r.det > 0.0f)) { r.cull = 3; return; }
  if (!(std::isfinite(r.mx_f) && std::isfinite(r.my_f) && std::isfinite(r.A_f) &&
        std::isfinite(r.B2_f) && std::isfinite(r.C_f) && std::isfinite(r.hmax_f))) {
    r.cull = 3;
    return;
  }
  // Tile AABB of the h <= hmax ellipse, +1 px margin, from fp32 values.
  const double ex = std::sqrt((double)r.hmax_f * r.cov[0]) + 1.0;
  const double ey = std::sqrt((double)r.hmax_f * r.cov[2]) + 1.0;
  const int tw = (cam.width + kTile - 1) / kTile, th = (cam.height + kTile - 1) / kTile;
  double fx0 = std::floor(((double)r.mx_f - ex) / kTile), fx1 = std::floor(((double)r.mx_f + ex) / kTile);
  double fy0 = std::floor(((double)r.my_f - ey) / kTile), fy1 = std::floor(((double)r.my_f + ey) / kTile);
  fx0 = std::max(fx0, 0.0); fy0 = std::max(fy0, 0.0);
  fx1 = std::min(fx1, (double)(tw - 1)); fy1 = std::min(fy1, (double)(th - 1));
  if (!(fx0 <= fx1 && fy0 <= fy1)) { r.cull = 4; return; }
  r.rect[0] = (int)fx0; r.rect[1] = (int)fy0; r.rect[2] = (int)fx1; r.rect[3] = (int)fy1;
  r.n_tiles = (r.rect[2] - r.rect[0] + 1) * (r.rect[3] - r.rect[1] + 1);
}

// The fp32 inclusion quadratic h (§8(c) step 7).  Must be evaluated exactly
// in this order with explicit fmaf and no contraction (-ffp-contract=off).
inline float h_f32(float px, float py, const Proj& r) {
  const float dx = px - r.mx_f;
  const float dy = py - r.my_f;
  const float bdy = r.B2_f * dy;
  const float cdy = r.C_f * dy;
  const float cdy2 = cdy * dy;
  return std::fma(dx, std::fma(r.A_f, dx, bdy), cdy2);
}

// 2D t kernel (Eq. 4): T2D = [1 + h/nu]^-(nu+2)/2
inline double t2d(double h, double nu) { return std::pow(1.0 + h / nu, -(nu + 2.0) / 2.0); }
// dT/dh
inline double dT_dh(double h, double nu) {
  return -(nu + 2.0) / (2.0 * nu) * std::pow(1.0 + h / nu, -(nu + 4.0) / 2.0);
}
// dT/dnu: full derivative (R13); `paper` selects the printed form of
// PAPER.md:1301-1314 which omits the -1/2 ln(1+h/nu) T term.
inline double dT_dnu(double h, double nu, bool paper) {
  const double g = 1.0 + h / nu;
  if (paper) return (nu + 2.0) / 2.0 * h / (nu * nu) * std::pow(g, -(nu + 4.0) / 2.0);
  const double T = std::pow(g, -(nu + 2.0) / 2.0);
  return T * (-0.5 * std::log(g) + (nu + 2.0) * h / (2.0 * nu * nu * g));
}

// The component's kernel at h: the 2D t of Eq. 4, or the Gaussian e^{-h/2}
// of 3DGS (Eq. 1) for the Gaussian variant (dT/dnu = 0).
inline double kernel_T(const Proj& r, double h) {
  return (r.variant & kVarGaussian) ? std::exp(-0.5 * h) : t2d(h, r.nu);
}
inline double kernel_dT_dh(const Proj& r, double h) {
  return (r.variant & kVarGaussian) ? -0.5 * std::exp(-0.5 * h) : dT_dh(h, r.nu);
}
inline double kernel_dT_dnu(const Proj& r, double h, bool paper) {
  return (r.variant & kVarGaussian) ? 0.0 : dT_dnu(h, r.nu, paper);
}

struct View {
  int W, H, tw, th;
  std::vector<Proj> pr;
  std::vector<int> order;               // visible components sorted by (depth_f, index), R8
  std::vector<std::vector<int>> tiles;  // per-tile lists in depth order
};

void build_view(const orc_params* P, const orc_cam& cam, View& v, bool bin) {
  const int64_t n = P->n;
  v.W = cam.width; v.H = cam.height;
  v.tw = (cam.width + kTile - 1) / kTile; v.th = (cam.height + kTile - 1) / kTile;
  v.pr.resize(n);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    Comp c;
    load_comp(P, i, c);
    project(c, P->sh_degree, cam, v.pr[i], P->variant);
  }
  v.order.clear();
  for (int64_t i = 0; i < n; ++i)
    // every component the inclusion test may accept: visible ones (cull 0)
    // and those whose tile AABB misses the image (cull 4, no tiles) -- the
    // brute force tests them too, so a non-conservative rect would show
    if (v.pr[i].cull == 0 || v.pr[i].cull == 4) v.order.push_back((int)i);
  // R8: global per-view order by fp32 camera depth, ties by component index
  std::stable_sort(v.order.begin(), v.order.end(), [&](int a, int b) {
    if (v.pr[a].depth_f != v.pr[b].depth_f) return v.pr[a].depth_f < v.pr[b].depth_f;
    return a < b;
  });
  if (!bin) return;
  v.tiles.assign((size_t)v.tw * v.th, std::vector<int>());
  for (int i : v.order) {
    const Proj& r = v.pr[i];
    for (int ty = r.rect[1]; ty <= r.rect[3]; ++ty)
      for (int tx = r.rect[0]; tx <= r.rect[2]; ++tx) v.tiles[(size_t)ty * v.tw + tx].push_back(i);
  }
}

struct Entry {
  int id;
  double h, dx, dy, T, alpha, W;  // W = transmittance before this component
  bool clamped;
};

// The included sequence of one pixel (Eq. 7 with R9-R11).
//   mode 0 (brute force): every visible component in (depth, index) order
//     (R8), included iff its fp32 h at the pixel centre is <= hmax (R9) --
//     no tile rect, no tile list: the plain per-pixel definition;
//   mode 1 (tiled): the pixel's tile list (components whose tile rect covers
//     the tile, same order), the same h test -- the acceleration the GPU
//     mirrors; mode 0 == mode 1 bit for bit is the pin that the rect is
//     conservative (tests/test_oracle_pins.py);
//   mode 2: a frozen list (every listed component included, no stop test).
// Stop rule (R11): the component that drives W below 1e-4
// is composited, then the pixel stops; nothing after it is considered, even
// a negative component that would re-grow W.
void pixel_list(const View& v, int x, int y, int mode, const int32_t* frozen, int cap,
                std::vector<Entry>& out, double* tie) {
  out.clear();
  const float pxf = (float)x + 0.5f, pyf = (float)y + 0.5f;
  const double pxd = x + 0.5, pyd = y + 0.5;
  const int tx = x / kTile, ty = y / kTile;
  double W = 1.0;
  double tmin = std::numeric_limits<double>::infinity();
  auto consider = [&](int i, int gate) -> bool {  // gate: 0 none, 1 h test, 2 rect + h test; true = stop
    const Proj& r = v.pr[i];
    if (gate == 2 && !(tx >= r.rect[0] && tx <= r.rect[2] && ty >= r.rect[1] && ty <= r.rect[3])) return false;
    if (gate >= 1) {
      const float h32 = h_f32(pxf, pyf, r);
      if (!(h32 <= r.hmax_f)) return false;
    }
    Entry e;
    e.id = i;
    e.dx = pxd - r.mean2d[0];
    e.dy = pyd - r.mean2d[1];
    e.h = r.conic[0] * e.dx * e.dx + 2.0 * r.conic[1] * e.dx * e.dy + r.conic[2] * e.dy * e.dy;
    e.T = kernel_T(r, e.h);
    const double a = r.o * e.T;
    e.clamped = (a > kAlphaClamp) || (a < -kAlphaClamp);
    e.alpha = std::min(std::max(a, -kAlphaClamp), kAlphaClamp);
    e.W = W;
    out.push_back(e);
    W = W * (1.0 - e.alpha);
    tmin = std::min(tmin, std::fabs(W - kWStop) / kWStop);
    return gate >= 1 && W < kWStop;
  };
  if (mode == 2) {
    const int32_t* L = frozen + ((size_t)y * v.W + x) * cap;
    for (int k = 0; k < cap && L[k] >= 0; ++k) consider(L[k], 0);
  } else if (mode == 1) {
    for (int i : v.tiles[(size_t)ty * v.tw + tx])
      if (consider(i, 2)) break;
  } else {
    for (int i : v.order)
      if (consider(i, 1)) break;
  }
  if (tie) *tie = tmin;
}

}  // namespace

extern "C" {

int orc_num_planes(int sh_degree) { return n_planes(sh_degree); }

// ---- primitives exposed for the pins ------------------------------------
double orc_nu_of(double raw) { return nu_of(raw); }
double orc_opacity_of(double raw) { return opacity_of(raw); }
double orc_opacity_of_v(double raw, int32_t variant) { return opacity_of(raw, variant); }
double orc_t2d(double h, double nu) { return t2d(h, nu); }
double orc_t3d(double h, double nu) { return std::pow(1.0 + h / nu, -(nu + 3.0) / 2.0); }  // Eq. 3
double orc_dT_dh(double h, double nu) { return dT_dh(h, nu); }
double orc_dT_dnu(double h, double nu, int paper) { return dT_dnu(h, nu, paper != 0); }
void orc_sh_basis(int deg, const double* d, double* Y) {
  for (int m = 0; m < 16; ++m) Y[m] = 0.0;
  sh_basis(deg, d[0], d[1], d[2], Y);
}
void orc_cov3d(const double* log_scale, const double* q, double* out) {
  Comp c{};
  for (int k = 0; k < 3; ++k) c.s[k] = log_scale[k];
  for (int k = 0; k < 4; ++k) c.q[k] = q[k];
  c.raw_nu = 0.0; c.raw_o = 0.5;
  orc_cam cam{};
  cam.R[0] = cam.R[4] = cam.R[8] = 1.0; cam.t[2] = 5.0;
  cam.fx = cam.fy = 1.0; cam.width = cam.height = 16; cam.z_near = 0.2;
  Proj r;
  project(c, 0, cam, r);
  for (int k = 0; k < 9; ++k) out[k] = r.Sig[k];
}

// ---- a1: projection of every component into one view --------------------
// PAPER.md:85-92 (Eq. 4), 1116-1215 (SM forward), 1077-1079 (nu range,
// truncation, no low-pass filter).
int orc_project(const orc_params* P, const orc_cam* cam, orc_proj_out* out) {
  const int64_t n = P->n;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    Comp c;
    load_comp(P, i, c);
    Proj r;
    project(c, P->sh_degree, *cam, r, P->variant);
    out->mx[i] = r.mx_f; out->my[i] = r.my_f; out->A[i] = r.A_f; out->B2[i] = r.B2_f;
    out->C[i] = r.C_f; out->hmax[i] = r.hmax_f; out->depth[i] = r.depth_f;
    for (int k = 0; k < 4; ++k) out->rect[i * 4 + k] = r.rect[k];
    out->n_tiles[i] = r.n_tiles;
    out->cull[i] = r.cull;
    for (int k = 0; k < 3; ++k) out->p[i * 3 + k] = r.p[k];
    out->mean2d[i * 2 + 0] = r.mean2d[0]; out->mean2d[i * 2 + 1] = r.mean2d[1];
    for (int k = 0; k < 3; ++k) out->cov2d[i * 3 + k] = r.cov[k];
    for (int k = 0; k < 3; ++k) out->conic[i * 3 + k] = r.conic[k];
    out->nu[i] = r.nu; out->o[i] = r.o;
    for (int k = 0; k < 3; ++k) out->color[i * 3 + k] = r.color[k];
  }
  return 0;
}

// ---- a2: binning -------------------------------------------------------
// Instances (tile, depth, index) of every visible component, sorted
// lexicographically (R8).  Writes per-tile counts; if ids/keys are non-null
// writes the sorted instance list (key = tile << 32 | float bits of depth).
// Returns the total instance count M.
int64_t orc_bin(const orc_params* P, const orc_cam* cam, int32_t* tile_counts, int32_t* ids,
                uint64_t* keys) {
  View v;
  build_view(P, *cam, v, true);
  int64_t M = 0;
  for (size_t t = 0; t < v.tiles.size(); ++t) {
    if (tile_counts) tile_counts[t] = (int32_t)v.tiles[t].size();
    for (int i : v.tiles[t]) {
      if (ids) ids[M] = i;
      if (keys) {
        uint32_t bits;
        std::memcpy(&bits, &v.pr[i].depth_f, 4);
        keys[M] = ((uint64_t)t << 32) | (uint64_t)bits;
      }
      ++M;
    }
  }
  return M;
}

// Per-tile list of selected tiles only (for full-size sampled parity).
int64_t orc_tile_lists(const orc_params* P, const orc_cam* cam, int32_t n_sel, const int32_t* sel,
                       int32_t* counts, int32_t* ids, int64_t cap) {
  View v;
  build_view(P, *cam, v, false);
  int64_t M = 0;
  for (int s = 0; s < n_sel; ++s) {
    const int t = sel[s];
    const int tx = t % v.tw, ty = t / v.tw;
    int cnt = 0;
    for (int i : v.order) {
      const Proj& r = v.pr[i];
      if (tx >= r.rect[0] && tx <= r.rect[2] && ty >= r.rect[1] && ty <= r.rect[3]) {
        if (ids && M < cap) ids[M] = i;
        ++M; ++cnt;
      }
    }
    counts[s] = cnt;
  }
  return M;
}

// ---- a3: forward compositing (Eq. 7) --------
// C(u) = sum_i c_i a_i prod_{j<i} (1 - a_j) + bg W_final with signed
// a = clamp(o T2D, +-0.99) (R10), stop after W < 1e-4 (R11), background R12.
// mode 0 brute force, 1 tiled, 2 frozen lists (lists_in [H][W][cap], -1 end).
// lists_out (nullable) records the included ids per pixel.
// If pix_sel != NULL only the n_sel listed pixels (y*W+x) are evaluated and
// the outputs are written compactly (index s instead of y*W+x).
int orc_render(const orc_params* P, const orc_cam* cam, const double* bg, int32_t mode,
               double* rgb, double* final_T, int32_t* n_contrib, double* tie,
               const int32_t* lists_in, int32_t* lists_out, int32_t cap, int32_t n_sel,
               const int32_t* pix_sel) {
  View v;
  build_view(P, *cam, v, mode == 1);
  const int64_t npx = pix_sel ? (int64_t)n_sel : (int64_t)v.W * v.H;
  const int64_t plane = npx;
#pragma omp parallel
  {
    std::vector<Entry> L;
#pragma omp for schedule(dynamic, 64)
    for (int64_t s = 0; s < npx; ++s) {
      const int64_t pix = pix_sel ? (int64_t)pix_sel[s] : s;
      const int x = (int)(pix % v.W), y = (int)(pix / v.W);
      double tmin;
      pixel_list(v, x, y, mode, lists_in, cap, L, &tmin);
      double C[3] = {0.0, 0.0, 0.0};
      double W = 1.0;
      for (const Entry& e : L) {
        const Proj& r = v.pr[e.id];
        for (int k = 0; k < 3; ++k) C[k] += r.color[k] * e.alpha * e.W;
        W = e.W * (1.0 - e.alpha);
      }
      for (int k = 0; k < 3; ++k) rgb[k * plane + s] = C[k] + bg[k] * W;
      final_T[s] = W;
      n_contrib[s] = (int32_t)L.size();
      if (tie) tie[s] = tmin;
      if (lists_out) {
        int32_t* o = lists_out + s * cap;
        int k = 0;
        for (; k < (int)L.size() && k < cap; ++k) o[k] = L[k].id;
        for (; k < cap; ++k) o[k] = -1;
      }
    }
  }
  return 0;
}

// ---- a4 + a5: backward ------------------------------
// Reverse mode of orc_render (gating frozen: inclusion and termination are
// constants, SPEC.md:316 / R22) followed by the chain to the six parameter
// groups ("dL/dmu, dL/dS, dL/dR, dL/dc, dL/do, dL/dnu").
// grad_planes [P][n] is accumulated (+=); g2d [n][10] (+=, nullable) holds
// dL/d{mean2d x,y, conic A,B,C, colour r,g,b, o, nu} per component.
// If pix_sel != NULL only the n_sel listed pixels (y*W+x) contribute and
// d_rgb is compact ([3][n_sel]).
int orc_backward(const orc_params* P, const orc_cam* cam, const double* bg, const double* d_rgb,
                 int32_t mode, int32_t nu_grad_paper, double* grad_planes, double* g2d_out,
                 const int32_t* lists_in, int32_t cap, int32_t n_sel, const int32_t* pix_sel) {
  View v;
  build_view(P, *cam, v, mode == 1);
  const int64_t n = P->n;
  const int64_t npx = pix_sel ? (int64_t)n_sel : (int64_t)v.W * v.H;
  std::vector<double> g2d((size_t)n * 10, 0.0);
#pragma omp parallel
  {
    std::vector<Entry> L;
#pragma omp for schedule(dynamic, 64)
    for (int64_t s = 0; s < npx; ++s) {
      const int64_t pix = pix_sel ? (int64_t)pix_sel[s] : s;
      const int x = (int)(pix % v.W), y = (int)(pix / v.W);
      pixel_list(v, x, y, mode, lists_in, cap, L, nullptr);
      if (L.empty()) continue;
      const double g[3] = {d_rgb[0 * npx + s], d_rgb[1 * npx + s], d_rgb[2 * npx + s]};
      // suffix S_i: colour behind i normalised by W_{i+1}; S_n = bg
      double S[3] = {bg[0], bg[1], bg[2]};
      for (int k = (int)L.size() - 1; k >= 0; --k) {
        const Entry& e = L[k];
        const Proj& r = v.pr[e.id];
        double dc[3], da = 0.0;
        for (int ch = 0; ch < 3; ++ch) {
          dc[ch] = g[ch] * e.alpha * e.W;                  // dC/dc_i = a_i W_i
          da += g[ch] * (r.color[ch] - S[ch]);             // dC/da_i = W_i (c_i - S_i)
        }
        da *= e.W;
        for (int ch = 0; ch < 3; ++ch) S[ch] = r.color[ch] * e.alpha + (1.0 - e.alpha) * S[ch];
        if (e.clamped) da = 0.0;  // R10: zero gradient through an active clamp
        const double d_o = da * e.T;      // a = o T
        const double d_T = da * r.o;
        const double d_h = d_T * kernel_dT_dh(r, e.h);
        const double d_nu = d_T * kernel_dT_dnu(r, e.h, nu_grad_paper != 0);
        // h = A dx^2 + 2 B dx dy + C dy^2, d = u - mean2d
        const double A = r.conic[0], B = r.conic[1], Cc = r.conic[2];
        const double dmx = d_h * -2.0 * (A * e.dx + B * e.dy);
        const double dmy = d_h * -2.0 * (B * e.dx + Cc * e.dy);
        const double dA = d_h * e.dx * e.dx;
        const double dB = d_h * 2.0 * e.dx * e.dy;
        const double dC = d_h * e.dy * e.dy;
        double* G = &g2d[(size_t)e.id * 10];
        const double vals[10] = {dmx, dmy, dA, dB, dC, dc[0], dc[1], dc[2], d_o, d_nu};
        for (int q = 0; q < 10; ++q) {
#pragma omp atomic
          G[q] += vals[q];
        }
      }
    }
  }
  // chain rule per component: g2d -> parameters
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    const double* G = &g2d[(size_t)i * 10];
    bool any = false;
    for (int q = 0; q < 10; ++q) any = any || (G[q] != 0.0);
    if (g2d_out)
      for (int q = 0; q < 10; ++q) g2d_out[i * 10 + q] += G[q];
    if (!any) continue;
    Comp c;
    load_comp(P, i, c);
    Proj r;
    project(c, P->sh_degree, *cam, r, P->variant);
    const double px = r.p[0], py = r.p[1], pz = r.p[2];
    // conic gradient as a symmetric matrix, then Sigma2D: G_S = -Q G_Q Q
    const double Q[4] = {r.conic[0], r.conic[1], r.conic[1], r.conic[2]};
    const double GQ[4] = {G[2], 0.5 * G[3], 0.5 * G[3], G[4]};
    double QG[4], GS[4];
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 2; ++b) QG[a * 2 + b] = Q[a * 2 + 0] * GQ[0 * 2 + b] + Q[a * 2 + 1] * GQ[1 * 2 + b];
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 2; ++b) GS[a * 2 + b] = -(QG[a * 2 + 0] * Q[0 * 2 + b] + QG[a * 2 + 1] * Q[1 * 2 + b]);
    // Sigma2D = J Sc J^T (Eq. 4): dL/dSc = J^T GS J ; dL/dJ = 2 GS J Sc
    double GSc[9], GJ[6];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) {
        double s = 0.0;
        for (int k = 0; k < 2; ++k)
          for (int l = 0; l < 2; ++l) s += r.J[k * 3 + a] * GS[k * 2 + l] * r.J[l * 3 + b];
        GSc[a * 3 + b] = s;
      }
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 3; ++b) {
        double s = 0.0;
        for (int k = 0; k < 2; ++k)
          for (int l = 0; l < 3; ++l) s += GS[a * 2 + k] * r.J[k * 3 + l] * r.Sc[l * 3 + b];
        GJ[a * 3 + b] = 2.0 * s;
      }
    // Sc = W Sigma W^T: dL/dSigma = W^T GSc W
    double GSig[9];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) {
        double s = 0.0;
        for (int k = 0; k < 3; ++k)
          for (int l = 0; l < 3; ++l) s += cam->R[k * 3 + a] * GSc[k * 3 + l] * cam->R[l * 3 + b];
        GSig[a * 3 + b] = s;
      }
    // Sigma = M M^T, M = R S: dL/dM = 2 GSig M; dL/dR = dL/dM S; dL/dS_j = sum_i dL/dM_ij R_ij
    double GM[9], GR[9];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) {
        double s = 0.0;
        for (int k = 0; k < 3; ++k) s += GSig[a * 3 + k] * r.M[k * 3 + b];
        GM[a * 3 + b] = 2.0 * s;
      }
    double dls[3];
    for (int j = 0; j < 3; ++j) {
      double s = 0.0;
      for (int a = 0; a < 3; ++a) s += GM[a * 3 + j] * r.Rq[a * 3 + j];
      dls[j] = s * r.S[j];  // d/dlog_scale = d/dS * S
    }
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) GR[a * 3 + b] = GM[a * 3 + b] * r.S[b];
    // R(q) polynomial -> unit quaternion -> raw quaternion (normalisation)
    const double w = r.qh[0], x = r.qh[1], y = r.qh[2], z = r.qh[3];
    double gq[4];
    gq[0] = 2.0 * (-z * GR[1] + y * GR[2] + z * GR[3] - x * GR[5] - y * GR[6] + x * GR[7]);
    gq[1] = 2.0 * (y * GR[1] + z * GR[2] + y * GR[3] - 2.0 * x * GR[4] - w * GR[5] + z * GR[6] +
                   w * GR[7] - 2.0 * x * GR[8]);
    gq[2] = 2.0 * (-2.0 * y * GR[0] + x * GR[1] + w * GR[2] + x * GR[3] + z * GR[5] - w * GR[6] +
                   z * GR[7] - 2.0 * y * GR[8]);
    gq[3] = 2.0 * (-2.0 * z * GR[0] - w * GR[1] + x * GR[2] + w * GR[3] - 2.0 * z * GR[4] + y * GR[5] +
                   x * GR[6] + y * GR[7]);
    const double dotq = gq[0] * w + gq[1] * x + gq[2] * y + gq[3] * z;
    double drot[4];
    for (int k = 0; k < 4; ++k) drot[k] = (gq[k] - r.qh[k] * dotq) / r.qn;
    // camera-space mean: through mean2d and through J(p)
    double dp[3] = {0.0, 0.0, 0.0};
    dp[0] += cam->fx / pz * G[0];
    dp[1] += cam->fy / pz * G[1];
    dp[2] += -cam->fx * px / (pz * pz) * G[0] - cam->fy * py / (pz * pz) * G[1];
    dp[2] += GJ[0] * (-cam->fx / (pz * pz)) + GJ[4] * (-cam->fy / (pz * pz)) +
             GJ[2] * (2.0 * cam->fx * px / (pz * pz * pz)) + GJ[5] * (2.0 * cam->fy * py / (pz * pz * pz));
    dp[0] += GJ[2] * (-cam->fx / (pz * pz));
    dp[1] += GJ[5] * (-cam->fy / (pz * pz));
    double dmu[3];
    for (int a = 0; a < 3; ++a) dmu[a] = cam->R[0 * 3 + a] * dp[0] + cam->R[1 * 3 + a] * dp[1] + cam->R[2 * 3 + a] * dp[2];
    // SH colour: c = max(0, sum sh Y(d) + 1/2)
    const int deg = P->sh_degree, K = sh_K(deg);
    double gdc[3];
    for (int ch = 0; ch < 3; ++ch) gdc[ch] = (r.pre[ch] > 0.0) ? G[5 + ch] : 0.0;
    double dsh[48];
    for (int m = 0; m < K; ++m)
      for (int ch = 0; ch < 3; ++ch) dsh[m * 3 + ch] = gdc[ch] * r.Y[m];
    double GY[48];
    sh_basis_grad(deg, r.dir[0], r.dir[1], r.dir[2], GY);
    double gdir[3] = {0.0, 0.0, 0.0};
    for (int m = 0; m < K; ++m)
      for (int ch = 0; ch < 3; ++ch)
        for (int a = 0; a < 3; ++a) gdir[a] += gdc[ch] * c.sh[m * 3 + ch] * GY[m * 3 + a];
    const double dd = gdir[0] * r.dir[0] + gdir[1] * r.dir[1] + gdir[2] * r.dir[2];
    for (int a = 0; a < 3; ++a) dmu[a] += (gdir[a] - r.dir[a] * dd) / r.dist;
    // reparameterisations (R1, R2)
    const double draw_o = G[8] * dopacity_draw(r.o, P->variant);
    const double draw_nu = G[9] * dnu_draw(c.raw_nu);
    double* gp = grad_planes;
    for (int a = 0; a < 3; ++a) gp[(0 + a) * n + i] += dmu[a];
    for (int a = 0; a < 3; ++a) gp[(3 + a) * n + i] += dls[a];
    for (int a = 0; a < 4; ++a) gp[(6 + a) * n + i] += drot[a];
    gp[10 * n + i] += draw_nu;
    gp[11 * n + i] += draw_o;
    for (int k = 0; k < 3 * K; ++k) gp[(12 + k) * n + i] += dsh[k];
  }
  return 0;
}

// ---- Philox4x32-10 (Salmon et al., SC'11), written independently ---------
void orc_philox4x32_10(const uint32_t* ctr_in, const uint32_t* key_in, uint32_t* out) {
  uint32_t c[4] = {ctr_in[0], ctr_in[1], ctr_in[2], ctr_in[3]};
  uint32_t k0 = key_in[0], k1 = key_in[1];
  for (int round = 0; round < 10; ++round) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    const uint32_t n0 = hi1 ^ c[1] ^ k0;
    const uint32_t n1 = lo1;
    const uint32_t n2 = hi0 ^ c[3] ^ k1;
    const uint32_t n3 = lo0;
    c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  for (int k = 0; k < 4; ++k) out[k] = c[k];
}

// Three standard normals for (component, step): Philox counter
// (i lo, i hi, step lo, step hi), key (seed lo, seed hi); uniforms
// u = ((x >> 8) + 1/2) 2^-24; Box-Muller (R14).
void orc_normals3(uint64_t seed, int64_t i, int64_t step, double* z) {
  const uint32_t ctr[4] = {(uint32_t)i, (uint32_t)((uint64_t)i >> 32), (uint32_t)step,
                           (uint32_t)((uint64_t)step >> 32)};
  const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t x[4];
  orc_philox4x32_10(ctr, key, x);
  double u[4];
  for (int k = 0; k < 4; ++k) u[k] = ((double)(x[k] >> 8) + 0.5) * (1.0 / 16777216.0);
  const double r0 = std::sqrt(-2.0 * std::log(u[0]));
  const double r1 = std::sqrt(-2.0 * std::log(u[2]));
  z[0] = r0 * std::cos(2.0 * M_PI * u[1]);
  z[1] = r0 * std::sin(2.0 * M_PI * u[1]);
  z[2] = r1 * std::cos(2.0 * M_PI * u[3]);
}

// ---- a7: gated SGHMC on mu + Adam on the rest ----------------------------
// PAPER.md:151-163 (Eq. 10), 1492-1523 (SM one-step form, sigmoid switch,
// burn-in), 1083/1514 (Adam on all other parameters).  Readings R14-R19:
//   r'  = (1 - eps C) r - eps g + (eta/eps) xi
//   mu' = mu - eps^2 g + gate (F + N),  F = eps (1 - eps C) r,  N = eta xi
//   gate = sigmoid(-k (|o| - t));  burn-in: F = 0, N = eta Sigma xi.
int orc_sghmc_step(int64_t n, int32_t sh_degree, double* planes, const double* grad, double* m,
                   double* v, double* r, const orc_sghmc_hp* hp) {
  const int P = n_planes(sh_degree);
  const double b1t = 1.0 - std::pow(hp->beta1, (double)hp->step);
  const double b2t = 1.0 - std::pow(hp->beta2, (double)hp->step);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    // opacity and covariance of the current (pre-update) state
    Comp c;
    orc_params pp{n, sh_degree, 0, planes};
    load_comp(&pp, i, c);
    const double o = opacity_of(c.raw_o, hp->variant);
    const double gate = 1.0 / (1.0 + std::exp(hp->gate_k * (std::fabs(o) - hp->gate_t)));
    double Sig[9];
    if (hp->burn_in) {
      double qn = std::sqrt(c.q[0] * c.q[0] + c.q[1] * c.q[1] + c.q[2] * c.q[2] + c.q[3] * c.q[3]);
      double qh[4] = {c.q[0] / qn, c.q[1] / qn, c.q[2] / qn, c.q[3] / qn};
      double R[9];
      quat_to_R(qh, R);
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) {
          double s = 0.0;
          for (int k = 0; k < 3; ++k) s += R[a * 3 + k] * std::exp(2.0 * c.s[k]) * R[b * 3 + k];
          Sig[a * 3 + b] = s;
        }
    }
    double xi[3];
    orc_normals3(hp->seed, i, hp->step, xi);
    // Adam moments on every non-mean plane; on the mean planes only when
    // g_adam is set (R17: "we employ the Adam gradient in SGHMC").
    double adir[64];
    // Eq. 8 regularizers (R27): eps_o sum |o| and
    // eps_Sigma sum_j sqrt(lambda_j); the eigenvalues of Sigma = R S S^T R^T
    // are exp(2 s_j), so sqrt(lambda_j) = exp(s_j) and
    //   d/ds_j = eps_Sigma exp(s_j),  d/draw_o = eps_o sign(o) (1 - o^2).
    double reg[64] = {0.0};
    for (int j = 0; j < 3; ++j) reg[3 + j] = hp->eps_sigma * std::exp(c.s[j]);
    reg[11] = hp->eps_o * (o > 0.0 ? 1.0 : (o < 0.0 ? -1.0 : 0.0)) * dopacity_draw(o, hp->variant);
    for (int p = 0; p < P; ++p) {
      if (p < 3 && !hp->g_adam && hp->mu_mode != 2) { adir[p] = 0.0; continue; }
      const double g = grad[(int64_t)p * n + i] * hp->grad_scale + reg[p];
      double& mm = m[(int64_t)p * n + i];
      double& vv = v[(int64_t)p * n + i];
      mm = hp->beta1 * mm + (1.0 - hp->beta1) * g;
      vv = hp->beta2 * vv + (1.0 - hp->beta2) * g * g;
      adir[p] = (mm / b1t) / (std::sqrt(vv / b2t) + hp->adam_eps);
    }
    const double eps = hp->lr, C = hp->friction, eta = hp->noise;
    double noise[3];
    if (hp->burn_in) {
      for (int a = 0; a < 3; ++a) noise[a] = eta * (Sig[a * 3 + 0] * xi[0] + Sig[a * 3 + 1] * xi[1] + Sig[a * 3 + 2] * xi[2]);
    } else {
      for (int a = 0; a < 3; ++a) noise[a] = eta * xi[a];
    }
    for (int a = 0; a < 3; ++a) {
      if (hp->mu_mode == 2) {  // setting 1: Adam on the means, no sampler state
        planes[(int64_t)a * n + i] = c.mu[a] - eps * adir[a];
        continue;
      }
      const double g = hp->g_adam ? adir[a] : grad[(int64_t)a * n + i] * hp->grad_scale;
      const double ra = r[(int64_t)a * n + i];
      const double F = (hp->burn_in || hp->mu_mode == 1) ? 0.0 : eps * (1.0 - eps * C) * ra;
      planes[(int64_t)a * n + i] = c.mu[a] - eps * eps * g + gate * (F + noise[a]);
      r[(int64_t)a * n + i] = (1.0 - eps * C) * ra - eps * g + (eta / eps) * xi[a];
    }
    for (int p = 3; p < P; ++p) {
      double lr;
      if (p < 6) lr = hp->lr_scale;
      else if (p < 10) lr = hp->lr_rot;
      else if (p == 10) lr = hp->lr_nu;
      else if (p == 11) lr = hp->lr_opacity;
      else lr = hp->lr_sh;
      planes[(int64_t)p * n + i] -= lr * adir[p];
    }
  }
  return 0;
}

// ---- NEXT-1: the image part of Eq. 8 ------------------
// L_img = (1 - eps_D) L1 + eps_D (1 - SSIM), per view and channel-averaged:
//   L1   = mean over the 3HW values of |C - target|;
//   SSIM = mean over channels and valid window positions p (R28: 11x11
//          window fully inside the image, no padding) of
//          SSIM_p = (2 mx my + C1)(2 sxy + C2) / ((mx^2 + my^2 + C1)(sx2 + sy2 + C2)),
//          with Gaussian-weighted local statistics (w = g g^T,
//          g_k = exp(-(k-5)^2 / (2 1.5^2)) / sum, K1 = 0.01, K2 = 0.03, range 1):
//          mx = sum w x, sx2 = sum w x^2 - mx^2, sxy = sum w x y - mx my.
// dL/dC by the chain rule through mx, sx2, sxy (fp64, plain loops):
//   dSSIM_p/dx_q = w_{q-p} (dS/dmx + dS/dsx2 (2 x_q - 2 mx) + dS/dsxy (y_q - my)).
// rgb, target, d_rgb: [3][H][W]; returns L_img (d_rgb overwritten).
double orc_image_loss(const double* rgb, const double* target, int32_t H, int32_t W, double eps_d,
                      double* d_rgb) {
  const int64_t P = (int64_t)H * W;
  double l1 = 0.0;
  for (int64_t k = 0; k < 3 * P; ++k) {
    const double d = rgb[k] - target[k];
    l1 += std::fabs(d);
    d_rgb[k] = (1.0 - eps_d) * (d > 0.0 ? 1.0 : (d < 0.0 ? -1.0 : 0.0)) / (3.0 * P);
  }
  l1 /= (double)(3 * P);
  if (eps_d == 0.0) return l1;
  if (H < 11 || W < 11) return std::numeric_limits<double>::quiet_NaN();
  double g[11], gs = 0.0;
  for (int k = 0; k < 11; ++k) { g[k] = std::exp(-(k - 5) * (k - 5) / (2.0 * 1.5 * 1.5)); gs += g[k]; }
  for (int k = 0; k < 11; ++k) g[k] /= gs;
  const double C1 = 0.01 * 0.01, C2 = 0.03 * 0.03;
  const int Hv = H - 10, Wv = W - 10;
  const double npos = 3.0 * Hv * Wv;
  double ssum = 0.0;
  for (int c = 0; c < 3; ++c) {
    const double* x = rgb + c * P;
    const double* y = target + c * P;
    double* dx = d_rgb + c * P;
    for (int py = 0; py < Hv; ++py)
      for (int px = 0; px < Wv; ++px) {
        double mx = 0, my = 0, xx = 0, yy = 0, xy = 0;
        for (int i = 0; i < 11; ++i)
          for (int j = 0; j < 11; ++j) {
            const double w = g[i] * g[j];
            const double a = x[(int64_t)(py + i) * W + px + j], b = y[(int64_t)(py + i) * W + px + j];
            mx += w * a; my += w * b; xx += w * a * a; yy += w * b * b; xy += w * a * b;
          }
        const double sx2 = xx - mx * mx, sy2 = yy - my * my, sxy = xy - mx * my;
        const double n1 = 2 * mx * my + C1, n2 = 2 * sxy + C2;
        const double d1 = mx * mx + my * my + C1, d2 = sx2 + sy2 + C2;
        const double S = (n1 * n2) / (d1 * d2);
        ssum += S;
        // partials of S
        const double dS_dmx = (2 * my * n2) / (d1 * d2) - S * (2 * mx) / d1;
        const double dS_dsx2 = -S / d2;
        const double dS_dsxy = (2 * n1) / (d1 * d2);
        const double k = -eps_d / npos;  // d(eps_D (1 - mean SSIM)) / dSSIM_p
        for (int i = 0; i < 11; ++i)
          for (int j = 0; j < 11; ++j) {
            const double w = g[i] * g[j];
            const int64_t q = (int64_t)(py + i) * W + px + j;
            dx[q] += k * w * (dS_dmx + dS_dsx2 * (2 * x[q] - 2 * mx) + dS_dsxy * (y[q] - my));
          }
      }
  }
  return (1.0 - eps_d) * l1 + eps_d * (1.0 - ssum / npos);
}

// Eq. 8 regularizer values: out[0] = sum_i |o_i|, out[1] = sum_i sum_j sqrt(lambda_ij)
// with lambda the eigenvalues of Sigma_i (= exp(2 s_ij), R27).
void orc_regularizers(int64_t n, int32_t sh_degree, const double* planes, double* out, int32_t variant) {
  orc_params pp{n, sh_degree, variant, planes};
  double so = 0.0, ss = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    Comp c;
    load_comp(&pp, i, c);
    so += std::fabs(opacity_of(c.raw_o, variant));
    for (int j = 0; j < 3; ++j) ss += std::exp(c.s[j]);
  }
  out[0] = so;
  out[1] = ss;
}

// ---- NEXT-2: component recycling (Eqs. 11-12, SM
// "Component Recycling" PAPER.md:1317-1460, implementation PAPER.md:1081) --

// beta(x, y) through ln Gamma, as the paper evaluates it.
double orc_beta(double x, double y) { return std::exp(std::lgamma(x) + std::lgamma(y) - std::lgamma(x + y)); }

// (1 - o_new)^N = 1 - o_old (Eq. 12), signed o as printed (R29: the sign of
// o_new follows o_old).
double orc_reloc_opacity(double o_old, int32_t N) { return 1.0 - std::pow(1.0 - o_old, 1.0 / N); }

// K of Eq. 12, the paper's double sum in its order:
//   K = sum_{i=1}^{N} sum_{k=0}^{i-1} C(i-1, k) (-1)^k o_new^{k+1} Z_k,
//   Z_k = beta(1/2, ((k+1)(nu_new + 3) - 1) / 2).
double orc_reloc_K(int32_t N, double o_new, double nu_new) {
  double K = 0.0;
  for (int i = 1; i <= N; ++i) {
    double binom = 1.0;  // C(i-1, 0)
    for (int k = 0; k <= i - 1; ++k) {
      const double Z = orc_beta(0.5, ((k + 1) * (nu_new + 3.0) - 1.0) / 2.0);
      K += binom * ((k % 2) ? -1.0 : 1.0) * std::pow(o_new, k + 1) * Z;
      binom = binom * (double)(i - 1 - k) / (double)(k + 1);
    }
  }
  return K;
}

// Sigma_new / Sigma_old of Eq. 12:
//   (o_old)^2 (nu_old / nu_new) (beta(1/2, (nu_old + 2)/2) / K)^2.
double orc_reloc_scale(double o_old, double nu_old, double nu_new, int32_t N) {
  const double o_new = orc_reloc_opacity(o_old, N);
  const double K = orc_reloc_K(N, o_new, nu_new);
  const double b = orc_beta(0.5, (nu_old + 2.0) / 2.0);
  return o_old * o_old * (nu_old / nu_new) * (b / K) * (b / K);
}

// One recycling pass (readings R29-R31):
//  1. dead = components with |o| < threshold, o = fp32(tanh(raw_o)) (the
//     decision is taken in fp32, as on the GPU), in index order;
//  2. at most floor(cap_frac * n) of them (the first ones) are relocated;
//  3. targets: multinomial over the live components with probability
//     proportional to |o| ("Multinomial distribution of opacity values"),
//     as integer weights w_i = floor(|o_i| 2^32); draw j takes
//     u = floor(r_j * total / 2^64), r_j = 64 Philox bits (counter
//     (j, 0x52454C4F, step lo, step hi), key seed), target = first i with
//     w_0 + ... + w_i > u;
//  4. a target keeps at most n_max - 1 dead (in j order); the others stay
//     dead for the next pass;
//  5. per target t with N - 1 accepted dead (N members after relocation):
//     o_new, Sigma_new of Eq. 12 with nu_new = nu_old (R30); every member
//     takes t's mean, rotation, nu and SH, raw_o = atanh(o_new) and
//     log_scale_t + ln(scale)/2; momentum and Adam moments of all members
//     are reset to 0 (R31).
// target_of[n] (out): t for every relocated dead component, -1 otherwise.
// Returns the number of relocated components.
int64_t orc_relocate(int64_t n, int32_t sh_degree, double* planes, double* m, double* v, double* r,
                     double threshold, double cap_frac, int32_t n_max, uint64_t seed, int64_t step,
                     int32_t* target_of, int32_t variant) {
  const int P = n_planes(sh_degree);
  std::vector<int64_t> dead;
  std::vector<uint64_t> cum(n);
  uint64_t total = 0;
  const float thr = (float)threshold;
  for (int64_t i = 0; i < n; ++i) {
    target_of[i] = -1;
    const float o32 = (float)opacity_of(planes[11 * n + i], variant);
    const float a = std::fabs(o32);
    if (a < thr) {
      dead.push_back(i);
    } else {
      total += (uint64_t)std::floor((double)a * 4294967296.0);
    }
    cum[i] = total;
  }
  const int64_t cap = (int64_t)std::floor(cap_frac * (double)n);
  const int64_t n_sel = std::min<int64_t>((int64_t)dead.size(), cap);
  if (n_sel == 0 || total == 0) return 0;
  // 3. draws
  std::vector<int64_t> tgt(n_sel);
  const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  for (int64_t j = 0; j < n_sel; ++j) {
    const uint32_t ctr[4] = {(uint32_t)j, 0x52454C4Fu, (uint32_t)step, (uint32_t)((uint64_t)step >> 32)};
    uint32_t x[4];
    orc_philox4x32_10(ctr, key, x);
    const uint64_t r64 = (uint64_t)x[0] | ((uint64_t)x[1] << 32);
    const uint64_t u = (uint64_t)(((unsigned __int128)r64 * total) >> 64);
    int64_t lo = 0, hi = n - 1;  // first i with cum[i] > u
    while (lo < hi) {
      const int64_t mid = (lo + hi) / 2;
      if (cum[mid] > u) hi = mid; else lo = mid + 1;
    }
    tgt[j] = lo;
  }
  // 4. groups in j order, at most n_max - 1 dead per target
  std::vector<std::vector<int64_t>> members(n);
  for (int64_t j = 0; j < n_sel; ++j)
    if ((int32_t)members[tgt[j]].size() < n_max - 1) members[tgt[j]].push_back(dead[j]);
  // 5. Eq. 12 per group
  int64_t moved = 0;
  for (int64_t t = 0; t < n; ++t) {
    if (members[t].empty()) continue;
    const int N = 1 + (int)members[t].size();
    const double o_old = opacity_of(planes[11 * n + t], variant);
    const double nu = nu_of(planes[10 * n + t]);
    const double o_new = orc_reloc_opacity(o_old, N);
    const double scale = orc_reloc_scale(o_old, nu, nu, N);
    planes[11 * n + t] = (variant & kVarPositive) ? std::log(o_new / (1.0 - o_new)) : std::atanh(o_new);
    for (int j = 0; j < 3; ++j) planes[(3 + j) * n + t] += 0.5 * std::log(scale);
    std::vector<int64_t> all = members[t];
    all.push_back(t);
    for (int64_t d : all) {
      for (int p = 0; p < P; ++p) {
        planes[(int64_t)p * n + d] = planes[(int64_t)p * n + t];
        m[(int64_t)p * n + d] = 0.0;
        v[(int64_t)p * n + d] = 0.0;
      }
      for (int a = 0; a < 3; ++a) r[(int64_t)a * n + d] = 0.0;
      if (d != t) target_of[d] = (int32_t)t;
    }
    moved += (int64_t)members[t].size();
  }
  return moved;
}

}  // extern "C"
