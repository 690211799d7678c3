// NEXT-1 — sss_image_loss: the image part of Eq. 8,
//   L_v = (1 - eps) mean|C - T| + eps (1 - SSIM(C, T)),
// and its gradient dL_v/dC, ready for sss_render_bwd's d_rgb.
//
// SSIM (R28): per channel, mean over the valid 11x11 window positions p
// (window inside the image) of
//   S_p = (2 mx my + C1)(2 sxy + C2) / ((mx^2 + my^2 + C1)(sx2 + sy2 + C2)),
// with Gaussian-weighted moments (w = g g^T, sigma 1.5, K1 = 0.01, K2 = 0.03).
// By the chain rule through mx, sx2 = E[x^2] - mx^2 and sxy = E[xy] - mx my,
//   dS_p/dx_q = w_{q-p} (A_p + B_p x_q + C_p y_q),
//   A = dS/dmx - 2 mx dS/dsx2 - my dS/dsxy,  B = 2 dS/dsx2,  C = dS/dsxy,
// so the gradient is three window correlations of the A, B, C maps:
//   dL/dx_q = k ((w * A)_q + x_q (w * B)_q + y_q (w * C)_q),  k = -eps / (3 Hv Wv).
//
// B200 design: two separable-filter passes over 32x32 tiles staged in shared
// memory, register-blocked (a thread sums 4 neighbouring outputs from one
// 14-value window of loads).  HBM traffic: the image pair is read twice, the
// three maps written once and read once, the gradient written once — 132 B
// per pixel.
//   ssim_maps_kernel:  image tiles + 10-pixel halo -> 5 moments (horizontal
//                      then vertical 11-tap sums) -> S (block-summed into the
//                      loss), k A, k B, k C at the tile's valid positions;
//   image_grad_kernel: k A, k B, k C tiles + halo -> 3 correlations -> the
//                      gradient, plus the L1 term (1 - eps) sign(x - y)/(3HW).
#include <cmath>

#include "common.cuh"

namespace sss {
namespace {

constexpr int kWin = 11;            // window edge
constexpr int kLT = 32;             // output tile edge
constexpr int kLS = kLT + kWin - 1;  // staged edge (tile + halo)
constexpr float kC1 = 0.01f * 0.01f, kC2 = 0.03f * 0.03f;

struct LossGeom {
  int H, W, Hv, Wv;  // image and valid-position extents
  float eps, k_ssim, k_l1;  // eps_dssim, -eps / (3 Hv Wv), (1 - eps) / (3 H W)
  float g[kWin];  // normalised 1D Gaussian (sigma 1.5)
};

__device__ __forceinline__ float block_sum256(float v, float* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5;
  if (lane_id() == 0) red[w] = v;
  __syncthreads();
  float s = 0.f;
  if (threadIdx.x == 0)
    for (int k = 0; k < 8; ++k) s += red[k];
  return s;  // valid in thread 0
}

// grid (tiles_x, tiles_y, V * 3), 256 threads
__global__ void __launch_bounds__(256) ssim_maps_kernel(const float* __restrict__ rgb,
                                                        const float* __restrict__ target, LossGeom G,
                                                        float* __restrict__ maps, float* __restrict__ loss) {
  __shared__ float xs[kLS][kLS + 1], ys[kLS][kLS + 1];
  __shared__ float hm[5][kLS][kLT + 1];
  __shared__ float red[8];
  const int plane = blockIdx.z;  // v * 3 + c
  const int px0 = blockIdx.x * kLT, py0 = blockIdx.y * kLT;
  const int64_t HW = (int64_t)G.H * G.W;
  const float* x = rgb + plane * HW;
  const float* y = target + plane * HW;
  for (int k = threadIdx.x; k < kLS * kLS; k += 256) {
    const int r = k / kLS, c = k % kLS;
    const int gy = py0 + r, gx = px0 + c;
    const bool in = gy < G.H && gx < G.W;
    xs[r][c] = in ? x[(int64_t)gy * G.W + gx] : 0.f;
    ys[r][c] = in ? y[(int64_t)gy * G.W + gx] : 0.f;
  }
  __syncthreads();
  // horizontal 11-tap sums, 4 consecutive columns per work item (register
  // blocked: 14 loads of x and y serve 4 outputs)
  for (int k = threadIdx.x; k < kLS * (kLT / 4); k += 256) {
    const int r = k / (kLT / 4), c0 = (k % (kLT / 4)) * 4;
    float xa[kWin + 3], ya[kWin + 3];
#pragma unroll
    for (int t = 0; t < kWin + 3; ++t) { xa[t] = xs[r][c0 + t]; ya[t] = ys[r][c0 + t]; }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f, s4 = 0.f;
#pragma unroll
      for (int t = 0; t < kWin; ++t) {
        const float a = xa[q + t], b = ya[q + t], w = G.g[t];
        s0 = fmaf(w, a, s0);
        s1 = fmaf(w, b, s1);
        s2 = fmaf(w * a, a, s2);
        s3 = fmaf(w * b, b, s3);
        s4 = fmaf(w * a, b, s4);
      }
      hm[0][r][c0 + q] = s0; hm[1][r][c0 + q] = s1; hm[2][r][c0 + q] = s2;
      hm[3][r][c0 + q] = s3; hm[4][r][c0 + q] = s4;
    }
  }
  __syncthreads();
  const int64_t HvWv = (int64_t)G.Hv * G.Wv;
  float* mA = maps + (int64_t)plane * 3 * HvWv;
  float* mB = mA + HvWv;
  float* mC = mB + HvWv;
  float ssum = 0.f;
  // vertical sums -> S, A, B, C; 4 consecutive rows per work item
  for (int k = threadIdx.x; k < (kLT / 4) * kLT; k += 256) {
    const int c = k % kLT, r0 = (k / kLT) * 4;
    float mom[5][4];
#pragma unroll
    for (int m = 0; m < 5; ++m) {
      float col[kWin + 3];
#pragma unroll
      for (int t = 0; t < kWin + 3; ++t) col[t] = hm[m][r0 + t][c];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float acc = 0.f;
#pragma unroll
        for (int t = 0; t < kWin; ++t) acc = fmaf(G.g[t], col[q + t], acc);
        mom[m][q] = acc;
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int py = py0 + r0 + q, px = px0 + c;
      if (py >= G.Hv || px >= G.Wv) continue;
      const float mx = mom[0][q], my = mom[1][q], xx = mom[2][q], yy = mom[3][q], xy = mom[4][q];
      const float sx2 = xx - mx * mx, sy2 = yy - my * my, sxy = xy - mx * my;
      const float n1 = 2.f * mx * my + kC1, n2 = 2.f * sxy + kC2;
      const float d1 = mx * mx + my * my + kC1, d2 = sx2 + sy2 + kC2;
      const float inv = 1.f / (d1 * d2);
      const float S = n1 * n2 * inv;
      ssum += S;
      const float dS_dmx = 2.f * my * n2 * inv - S * 2.f * mx / d1;
      const float dS_dsx2 = -S / d2;
      const float dS_dsxy = 2.f * n1 * inv;
      const int64_t o = (int64_t)py * G.Wv + px;
      mA[o] = G.k_ssim * (dS_dmx - 2.f * mx * dS_dsx2 - my * dS_dsxy);
      mB[o] = G.k_ssim * (2.f * dS_dsx2);
      mC[o] = G.k_ssim * dS_dsxy;
    }
  }
  const float bs = block_sum256(ssum, red);
  if (threadIdx.x == 0 && loss) {
    // eps (1 - mean S): the constant eps once per view, -eps S / npos per tile
    float add = G.k_ssim * bs;
    if (blockIdx.x == 0 && blockIdx.y == 0 && plane % 3 == 0) add += G.eps;
    atomicAdd(loss, add);
  }
}

// grid (ceil(W/32), ceil(H/32), V * 3), 256 threads
__global__ void __launch_bounds__(256) image_grad_kernel(const float* __restrict__ rgb,
                                                         const float* __restrict__ target, LossGeom G,
                                                         const float* __restrict__ maps, int with_ssim,
                                                         float* __restrict__ d_rgb, float* __restrict__ loss) {
  __shared__ float ms[3][kLS][kLS + 1];
  __shared__ float hm[3][kLS][kLT + 1];
  __shared__ float red[8];
  const int plane = blockIdx.z;
  const int qx0 = blockIdx.x * kLT, qy0 = blockIdx.y * kLT;
  const int64_t HW = (int64_t)G.H * G.W;
  const float* x = rgb + plane * HW;
  const float* y = target + plane * HW;
  float* d = d_rgb + plane * HW;
  if (with_ssim) {
    const int64_t HvWv = (int64_t)G.Hv * G.Wv;
    const float* mA = maps + (int64_t)plane * 3 * HvWv;
    // positions p = q - (0..10): stage p in [q0 - 10, q0 + 31] (zero outside the valid range)
    for (int k = threadIdx.x; k < kLS * kLS; k += 256) {
      const int r = k / kLS, c = k % kLS;
      const int py = qy0 - (kWin - 1) + r, px = qx0 - (kWin - 1) + c;
      const bool in = py >= 0 && px >= 0 && py < G.Hv && px < G.Wv;
      const int64_t o = in ? (int64_t)py * G.Wv + px : 0;
#pragma unroll
      for (int m = 0; m < 3; ++m) ms[m][r][c] = in ? mA[m * HvWv + o] : 0.f;
    }
    __syncthreads();
    // horizontal: sum_dx g[dx] M[r][c + 10 - dx], 4 columns per work item
    for (int k = threadIdx.x; k < kLS * (kLT / 4); k += 256) {
      const int r = k / (kLT / 4), c0 = (k % (kLT / 4)) * 4;
#pragma unroll
      for (int m = 0; m < 3; ++m) {
        float row[kWin + 3];
#pragma unroll
        for (int t = 0; t < kWin + 3; ++t) row[t] = ms[m][r][c0 + t];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float acc = 0.f;
#pragma unroll
          for (int t = 0; t < kWin; ++t) acc = fmaf(G.g[t], row[q + kWin - 1 - t], acc);
          hm[m][r][c0 + q] = acc;
        }
      }
    }
    __syncthreads();
  }
  float lsum = 0.f;
  // 4 consecutive rows per work item: vertical correlations + gradient
  for (int k = threadIdx.x; k < (kLT / 4) * kLT; k += 256) {
    const int c = k % kLT, r0 = (k / kLT) * 4;
    float f[3][4];
    if (with_ssim) {
#pragma unroll
      for (int m = 0; m < 3; ++m) {
        float col[kWin + 3];
#pragma unroll
        for (int t = 0; t < kWin + 3; ++t) col[t] = hm[m][r0 + t][c];
#pragma unroll
        for (int q = 0; q < 4; ++q) {  // sum_dy g[dy] H[r + 10 - dy][c]
          float acc = 0.f;
#pragma unroll
          for (int t = 0; t < kWin; ++t) acc = fmaf(G.g[t], col[q + kWin - 1 - t], acc);
          f[m][q] = acc;
        }
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int qy = qy0 + r0 + q, qx = qx0 + c;
      if (qy >= G.H || qx >= G.W) continue;
      const int64_t o = (int64_t)qy * G.W + qx;
      const float a = x[o], b = y[o];
      const float df = a - b;
      lsum += fabsf(df);
      float gq = G.k_l1 * (df > 0.f ? 1.f : (df < 0.f ? -1.f : 0.f));
      if (with_ssim) gq += f[0][q] + a * f[1][q] + b * f[2][q];
      d[o] = gq;
    }
  }
  const float bs = block_sum256(lsum, red);
  if (threadIdx.x == 0 && loss) atomicAdd(loss, G.k_l1 * bs);
}

}  // namespace
}  // namespace sss

using namespace sss;

extern "C" size_t sss_image_loss_workspace(int32_t n_views, int32_t height, int32_t width) {
  if (n_views <= 0 || height <= 0 || width <= 0) return 0;
  if (height < kWin || width < kWin) return 4;  // no SSIM maps possible (eps must be 0)
  return (size_t)n_views * 3 * 3 * (height - kWin + 1) * (width - kWin + 1) * sizeof(float);
}

extern "C" sss_status sss_image_loss(const float* rgb, const float* target, int32_t n_views, int32_t height,
                                     int32_t width, float eps_dssim, float* d_rgb, float* loss, void* ws,
                                     size_t ws_bytes, void* stream) {
  if (!rgb || !target || !d_rgb) { set_error("sss_image_loss: null buffer"); return SSS_ERR_ARG; }
  if (n_views <= 0 || height <= 0 || width <= 0) { set_error("sss_image_loss: empty batch or image"); return SSS_ERR_SHAPE; }
  if (!(eps_dssim >= 0.f && eps_dssim <= 1.f)) { set_error("sss_image_loss: eps_dssim outside [0, 1]"); return SSS_ERR_ARG; }
  const bool ssim = eps_dssim > 0.f;
  if (ssim && (height < kWin || width < kWin)) {
    set_error("sss_image_loss: D-SSIM needs images of at least %d x %d", kWin, kWin);
    return SSS_ERR_SHAPE;
  }
  if (ssim && (!ws || ws_bytes < sss_image_loss_workspace(n_views, height, width))) {
    set_error("sss_image_loss: workspace too small");
    return SSS_ERR_ARG;
  }
  LossGeom G;
  G.H = height; G.W = width;
  G.Hv = height - kWin + 1; G.Wv = width - kWin + 1;
  G.eps = eps_dssim;
  G.k_ssim = ssim ? (float)(-(double)eps_dssim / (3.0 * G.Hv * G.Wv)) : 0.f;
  G.k_l1 = (float)((1.0 - (double)eps_dssim) / (3.0 * (double)height * width));
  double gs = 0.0, gd[kWin];
  for (int k = 0; k < kWin; ++k) { gd[k] = std::exp(-(k - 5) * (k - 5) / (2.0 * 1.5 * 1.5)); gs += gd[k]; }
  for (int k = 0; k < kWin; ++k) G.g[k] = (float)(gd[k] / gs);
  cudaStream_t s = (cudaStream_t)stream;
  float* maps = (float*)ws;
  if (ssim) {
    const dim3 grid(div_up(G.Wv, kLT), div_up(G.Hv, kLT), n_views * 3);
    ssim_maps_kernel<<<grid, 256, 0, s>>>(rgb, target, G, maps, loss);
    count_launch();
  }
  const dim3 grid(div_up(width, kLT), div_up(height, kLT), n_views * 3);
  image_grad_kernel<<<grid, 256, 0, s>>>(rgb, target, G, maps, ssim ? 1 : 0, d_rgb, loss);
  count_launch();
  return check_launch("sss_image_loss");
}
