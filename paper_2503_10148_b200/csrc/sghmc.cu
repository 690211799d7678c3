// a7 — sss_sghmc_step: gated SGHMC on the means + Adam on every other group,
// one fused elementwise pass over the parameter, gradient, moment and
// momentum planes (Eq. 10; SM one-step form and sigmoid
// switch PAPER.md:1502-1521; burn-in PAPER.md:163, 1523; Adam PAPER.md:152,
// 1083, 1514).  Readings R14-R19:
//   g     = grad * grad_scale
//   r'    = (1 - eps C) r - eps g + (eta / eps) xi
//   mu'   = mu - eps^2 g + gate (F + N),  F = eps (1 - eps C) r,  N = eta xi
//   gate  = sigmoid(-k (|o| - t))
//   burn-in: F = 0, N = eta Sigma xi (Sigma of the pre-update component)
//   plane range [p0, p1): only those planes are written (ZeRO-1 shard).
//   NEXT-3 mu_mode: 1 = SGLD (F = 0), 2 = Adam on the means;
//   the opacity map follows the parameter variant (sigmoid for POSITIVE).
//   Eq. 8 regularizers (R27): g(log_scale_j) += eps_Sigma exp(s_j),
//         g(raw_o) += eps_o sign(o)(1 - o^2)  (sqrt(lambda_j(Sigma)) = exp(s_j))
//   Adam: m' = b1 m + (1-b1) g, v' = b2 v + (1-b2) g^2,
//         theta -= lr (m'/(1-b1^t)) / (sqrt(v'/(1-b2^t)) + eps_hat)
// xi: three standard normals from Philox4x32-10 (cuRAND's device function),
// key = seed, counter = (i, step); uniforms ((x >> 8) + 1/2) 2^-24 and
// Box-Muller in fp64 (R14).  Identical on every rank, so data-parallel
// replicas stay bit-identical without a broadcast.
// HBM-bound: 4 x 240 B read + 3 x 240 B written + 24 B momentum per
// component at SH degree 3 (~1.7 KB).
#include <curand_philox4x32_x.h>

#include "common.cuh"

namespace sss {
namespace {

#ifndef SSS_SGHMC_SH_BATCH
#define SSS_SGHMC_SH_BATCH 8
#endif
constexpr int kShBatch = SSS_SGHMC_SH_BATCH;  // SH planes whose loads are in flight together

struct HP {
  float lr, friction, noise, gate_k, gate_t;
  int burn_in, g_adam;
  float lr_group[5];  // log_scale, rot, nu, opacity, sh
  float beta1, beta2, adam_eps, grad_scale;
  float eps_o, eps_sigma;  // Eq. 8 regularizer weights
  int mu_mode;             // 0 SGHMC, 1 SGLD (F = 0), 2 Adam on the means
  int p0, p1;              // planes updated by this call
  float inv_b1t, inv_b2t;  // 1 / (1 - beta^t)
  uint32_t ctr2, ctr3;     // step (lo, hi)
  uint32_t key0, key1;     // seed (lo, hi)
  const int32_t* skip_if;  // device flag: nonzero = write nothing
  const sss_step_state* st;  // device step state (graph capture): overrides inv_b*t and ctr*
};

// Graph-capturable step: the step's constants from the device counter, with
// the host formula (fp64 pow, rounded once), then the counter advances.
__global__ void step_prep_kernel(sss_step_state* st, float beta1, float beta2) {
  const int64_t t = st->step;
  st->inv_b1t = (float)(1.0 / (1.0 - pow((double)beta1, (double)t)));
  st->inv_b2t = (float)(1.0 / (1.0 - pow((double)beta2, (double)t)));
  st->ctr2 = (uint32_t)t;
  st->ctr3 = (uint32_t)((uint64_t)t >> 32);
  st->step = t + 1;
}

__device__ __forceinline__ float adam_dir(float g, float* m, float* v, int64_t idx, const HP& hp) {
  const float mm = hp.beta1 * m[idx] + (1.f - hp.beta1) * g;
  const float vv = hp.beta2 * v[idx] + (1.f - hp.beta2) * g * g;
  m[idx] = mm;
  v[idx] = vv;
  return (mm * hp.inv_b1t) / (sqrtf(vv * hp.inv_b2t) + hp.adam_eps);
}

__device__ __forceinline__ void adam_plane(float* theta, const float* grad, float* m, float* v, int64_t i,
                                           float lr, const HP& hp, float reg = 0.f) {
  const float g = fmaf(grad[i], hp.grad_scale, reg);
  theta[i] -= lr * adam_dir(g, m, v, i, hp);
}

// Adam on planes [k0, k1) (k1 - k0 <= U) of one group: every load is issued
// before the first store (the planes of a parameter struct may alias as far
// as the compiler knows, which would otherwise serialise each plane's loads
// behind the previous plane's stores).  `first` is the group's first plane
// index in the [P] numbering (the ZeRO plane range).
template <int U, bool EXPREG = false>
__device__ __forceinline__ void adam_planes(float* theta, const float* grad, float* m, float* v, int64_t i,
                                            int64_t n, int k0, int k1, int first, float lr, const HP& hp,
                                            int64_t gn) {  // gn: the gradient's plane stride
  float t[U], g[U], mo[U], vo[U];
  bool on[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int k = k0 + u;
    on[u] = k < k1 && first + k >= hp.p0 && first + k < hp.p1;
    if (on[u]) {
      const int64_t idx = (int64_t)k * n + i;
      t[u] = theta[idx];
      g[u] = grad[(int64_t)k * gn + i];
      mo[u] = m[idx];
      vo[u] = v[idx];
    }
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    if (!on[u]) continue;
    const int64_t idx = (int64_t)(k0 + u) * n + i;
    // EXPREG: Eq. 8's eps_Sigma exp(s) on the log-scales (R27)
    const float reg = EXPREG && hp.eps_sigma != 0.f ? hp.eps_sigma * expf(t[u]) : 0.f;
    const float gg = fmaf(g[u], hp.grad_scale, reg);
    const float mm = hp.beta1 * mo[u] + (1.f - hp.beta1) * gg;
    const float vv = hp.beta2 * vo[u] + (1.f - hp.beta2) * gg * gg;
    m[idx] = mm;
    v[idx] = vv;
    theta[idx] = t[u] - lr * ((mm * hp.inv_b1t) / (sqrtf(vv * hp.inv_b2t) + hp.adam_eps));
  }
}

template <bool BLOCKED>  // gradient in the component-blocked layout (sss.h sss_params.block)
#ifndef SSS_SGHMC_MINB
#define SSS_SGHMC_MINB 4  // 62 registers, 32 warps/SM: 5.9 TB/s vs 5.6 at 80 registers (tools/sghmc_time.py)
#endif
#define SSS_SGHMC_LB __launch_bounds__(256, SSS_SGHMC_MINB)
__global__ void SSS_SGHMC_LB sghmc_kernel(sss_params P, sss_params Gr, sss_params Mo,
                                                    sss_params Vo, float* __restrict__ r, HP hp) {
  const int64_t n = P.n;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (hp.skip_if && *hp.skip_if) return;  // e.g. the iteration's binning overflowed
  if (hp.st) {  // graph-captured step: this step's constants from the device
    hp.inv_b1t = hp.st->inv_b1t;
    hp.inv_b2t = hp.st->inv_b2t;
    hp.ctr2 = hp.st->ctr2;
    hp.ctr3 = hp.st->ctr3;
  }
  int64_t gn = n;  // plane stride of the gradient (plain or component-blocked, sss.h)
  if (BLOCKED) Gr = block_view(Gr, i, gn);
  const int K = (P.sh_degree + 1) * (P.sh_degree + 1);
  // gate and (burn-in) covariance from the pre-update state
  const bool positive = P.variant & SSS_VARIANT_POSITIVE;
  const float o = positive ? 1.f / (1.f + expf(-P.raw_opacity[i])) : tanhf(P.raw_opacity[i]);
  const float gate = 1.f / (1.f + expf(hp.gate_k * (fabsf(o) - hp.gate_t)));
  float Sig[9];
  if (hp.burn_in) {
    float q[4], s[3];
    for (int k = 0; k < 4; ++k) q[k] = P.rot[k * n + i];
    for (int k = 0; k < 3; ++k) s[k] = P.log_scale[k * n + i];
    const float qn = sqrtf(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    const float w = q[0] / qn, x = q[1] / qn, y = q[2] / qn, z = q[3] / qn;
    const float R[9] = {1.f - 2.f * (y * y + z * z), 2.f * (x * y - w * z), 2.f * (x * z + w * y),
                        2.f * (x * y + w * z), 1.f - 2.f * (x * x + z * z), 2.f * (y * z - w * x),
                        2.f * (x * z - w * y), 2.f * (y * z + w * x), 1.f - 2.f * (x * x + y * y)};
    const float e2[3] = {expf(2.f * s[0]), expf(2.f * s[1]), expf(2.f * s[2])};
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b)
        Sig[a * 3 + b] = R[a * 3 + 0] * e2[0] * R[b * 3 + 0] + R[a * 3 + 1] * e2[1] * R[b * 3 + 1] +
                         R[a * 3 + 2] * e2[2] * R[b * 3 + 2];
  }
  // noise xi ~ N(0, I3)
  const uint4 x = curand_Philox4x32_10(make_uint4((uint32_t)i, (uint32_t)((uint64_t)i >> 32), hp.ctr2, hp.ctr3),
                                       make_uint2(hp.key0, hp.key1));
  const double u0 = ((double)(x.x >> 8) + 0.5) * (1.0 / 16777216.0);
  const double u1 = ((double)(x.y >> 8) + 0.5) * (1.0 / 16777216.0);
  const double u2 = ((double)(x.z >> 8) + 0.5) * (1.0 / 16777216.0);
  const double u3 = ((double)(x.w >> 8) + 0.5) * (1.0 / 16777216.0);
  const double r0 = sqrt(-2.0 * log(u0)), r1 = sqrt(-2.0 * log(u2));
  double s1, c1, s3, c3;
  sincospi(2.0 * u1, &s1, &c1);
  sincospi(2.0 * u3, &s3, &c3);
  const float xi[3] = {(float)(r0 * c1), (float)(r0 * s1), (float)(r1 * c3)};
  // ---- mean: gated SGHMC
  auto mine = [&](int p) { return p >= hp.p0 && p < hp.p1; };
  const float eps = hp.lr, Cf = hp.friction, eta = hp.noise;
  float noise[3];
  if (hp.burn_in) {
    for (int a = 0; a < 3; ++a) noise[a] = eta * (Sig[a * 3 + 0] * xi[0] + Sig[a * 3 + 1] * xi[1] + Sig[a * 3 + 2] * xi[2]);
  } else {
    for (int a = 0; a < 3; ++a) noise[a] = eta * xi[a];
  }
  // every load of the three mean planes before the first store (see adam_planes)
  const bool need_mv = hp.g_adam || hp.mu_mode == 2;
  float pm[3], gm[3], mo[3], vo[3], rm[3];
  bool onm[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    onm[a] = mine(a);
    if (!onm[a]) continue;
    const int64_t idx = a * n + i;
    pm[a] = P.mean[idx];
    gm[a] = Gr.mean[a * gn + i];
    if (need_mv) {
      mo[a] = Mo.mean[idx];
      vo[a] = Vo.mean[idx];
    }
    if (hp.mu_mode != 2) rm[a] = r[idx];
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if (!onm[a]) continue;
    const int64_t idx = a * n + i;
    const float graw = gm[a] * hp.grad_scale;
    float dir = 0.f;
    if (need_mv) {  // Adam direction, as adam_dir
      const float mm = hp.beta1 * mo[a] + (1.f - hp.beta1) * graw;
      const float vv = hp.beta2 * vo[a] + (1.f - hp.beta2) * graw * graw;
      Mo.mean[idx] = mm;
      Vo.mean[idx] = vv;
      dir = (mm * hp.inv_b1t) / (sqrtf(vv * hp.inv_b2t) + hp.adam_eps);
    }
    if (hp.mu_mode == 2) {  // setting 1: Adam on the means, no sampler state
      P.mean[idx] = pm[a] - eps * dir;
      continue;
    }
    const float g = hp.g_adam ? dir : graw;
    const float ra = rm[a];
    const float F = (hp.burn_in || hp.mu_mode == 1) ? 0.f : eps * (1.f - eps * Cf) * ra;
    P.mean[idx] = pm[a] - eps * eps * g + gate * (F + noise[a]);
    r[idx] = (1.f - eps * Cf) * ra - eps * g + (eta / eps) * xi[a];
  }
  // ---- Adam on the other groups
  adam_planes<3, true>(P.log_scale, Gr.log_scale, Mo.log_scale, Vo.log_scale, i, n, 0, 3, 3, hp.lr_group[0], hp, gn);
  adam_planes<4>(P.rot, Gr.rot, Mo.rot, Vo.rot, i, n, 0, 4, 6, hp.lr_group[1], hp, gn);
  {  // raw nu and raw opacity: both planes' loads before the stores
    const bool on_nu = mine(10), on_o = mine(11);
    float t2[2] = {0.f, 0.f}, g2[2] = {0.f, 0.f}, m2[2] = {0.f, 0.f}, v2[2] = {0.f, 0.f};
    if (on_nu) { t2[0] = P.raw_nu[i]; g2[0] = Gr.raw_nu[i]; m2[0] = Mo.raw_nu[i]; v2[0] = Vo.raw_nu[i]; }
    if (on_o) { t2[1] = P.raw_opacity[i]; g2[1] = Gr.raw_opacity[i]; m2[1] = Mo.raw_opacity[i]; v2[1] = Vo.raw_opacity[i]; }
    const float reg_o = hp.eps_o * (o > 0.f ? 1.f : (o < 0.f ? -1.f : 0.f)) * (positive ? o * (1.f - o) : 1.f - o * o);
    auto step = [&](int k, float reg, float lr, float* theta, float* m, float* v) {  // as adam_plane
      const float g = fmaf(g2[k], hp.grad_scale, reg);
      const float mm = hp.beta1 * m2[k] + (1.f - hp.beta1) * g;
      const float vv = hp.beta2 * v2[k] + (1.f - hp.beta2) * g * g;
      m[i] = mm;
      v[i] = vv;
      theta[i] = t2[k] - lr * ((mm * hp.inv_b1t) / (sqrtf(vv * hp.inv_b2t) + hp.adam_eps));
    };
    if (on_nu) step(0, 0.f, hp.lr_group[2], P.raw_nu, Mo.raw_nu, Vo.raw_nu);
    if (on_o) step(1, reg_o, hp.lr_group[3], P.raw_opacity, Mo.raw_opacity, Vo.raw_opacity);
  }
  for (int k = 0; k < 3 * K; k += kShBatch)
    adam_planes<kShBatch>(P.sh, Gr.sh, Mo.sh, Vo.sh, i, n, k, min(k + kShBatch, 3 * K), 12, hp.lr_group[4], hp, gn);
}

}  // namespace
}  // namespace sss

using namespace sss;

extern "C" sss_status sss_sghmc_step(sss_params* p, const sss_params* grad, sss_params* adam_m,
                                     sss_params* adam_v, float* momentum, const sss_sghmc_hparams* h,
                                     void* stream) {
  sss_status st;
  if ((st = validate_params(p, "sss_sghmc_step")) != SSS_OK) return st;
  if ((st = validate_params(grad, "sss_sghmc_step(grad)", true)) != SSS_OK) return st;
  if ((st = validate_params(adam_m, "sss_sghmc_step(m)")) != SSS_OK) return st;
  if ((st = validate_params(adam_v, "sss_sghmc_step(v)")) != SSS_OK) return st;
  if (!h || (!momentum && p->n > 0)) { set_error("sss_sghmc_step: null hparams / momentum"); return SSS_ERR_ARG; }
  if (grad->n != p->n || adam_m->n != p->n || adam_v->n != p->n || grad->sh_degree != p->sh_degree ||
      adam_m->sh_degree != p->sh_degree || adam_v->sh_degree != p->sh_degree) {
    set_error("sss_sghmc_step: n / sh_degree mismatch");
    return SSS_ERR_ARG;
  }
  if ((!h->step_state && h->step < 1) || !(h->lr > 0.f)) { set_error("sss_sghmc_step: step must be >= 1 and lr > 0"); return SSS_ERR_ARG; }
  if (p->n == 0) return SSS_OK;
  HP hp;
  hp.lr = h->lr; hp.friction = h->friction; hp.noise = h->noise; hp.gate_k = h->gate_k; hp.gate_t = h->gate_t;
  hp.burn_in = h->burn_in; hp.g_adam = h->g_adam;
  hp.lr_group[0] = h->lr_scale; hp.lr_group[1] = h->lr_rot; hp.lr_group[2] = h->lr_nu;
  hp.lr_group[3] = h->lr_opacity; hp.lr_group[4] = h->lr_sh;
  hp.beta1 = h->beta1; hp.beta2 = h->beta2; hp.adam_eps = h->adam_eps; hp.grad_scale = h->grad_scale;
  hp.eps_o = h->eps_o; hp.eps_sigma = h->eps_sigma;
  hp.mu_mode = h->mu_mode;
  hp.skip_if = h->skip_if;
  const int Pn = 12 + 3 * (p->sh_degree + 1) * (p->sh_degree + 1);
  hp.p0 = h->plane_begin;
  hp.p1 = (h->plane_begin == 0 && h->plane_end == 0) ? Pn : h->plane_end;
  if (hp.p0 < 0 || hp.p1 > Pn || hp.p0 > hp.p1) { set_error("sss_sghmc_step: bad plane range"); return SSS_ERR_ARG; }
  if (hp.p0 == hp.p1) return SSS_OK;
  if (hp.mu_mode < 0 || hp.mu_mode > 2) { set_error("sss_sghmc_step: mu_mode outside [0,2]"); return SSS_ERR_ARG; }
  hp.inv_b1t = (float)(1.0 / (1.0 - pow((double)h->beta1, (double)h->step)));
  hp.inv_b2t = (float)(1.0 / (1.0 - pow((double)h->beta2, (double)h->step)));
  hp.ctr2 = (uint32_t)h->step; hp.ctr3 = (uint32_t)((uint64_t)h->step >> 32);
  hp.key0 = (uint32_t)h->seed; hp.key1 = (uint32_t)(h->seed >> 32);
  cudaStream_t s = (cudaStream_t)stream;
  hp.st = h->step_state;
  if (h->step_state) {
    step_prep_kernel<<<1, 1, 0, s>>>(h->step_state, h->beta1, h->beta2);
    count_launch();
  }
  if (grad->block > 0)
    sghmc_kernel<true><<<div_up(p->n, 256), 256, 0, s>>>(*p, *grad, *adam_m, *adam_v, momentum, hp);
  else
    sghmc_kernel<false><<<div_up(p->n, 256), 256, 0, s>>>(*p, *grad, *adam_m, *adam_v, momentum, hp);
  count_launch();
  return check_launch("sss_sghmc_step");
}
