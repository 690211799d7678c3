// a4 + a5 (+ a6) — sss_render_bwd: closed-form backward of Eq. 7 (SM
// "Backward Pass") to the six parameter groups
// (PAPER.md:165).
//
// a4 raster backward.  One CTA per tile and view, 64 threads with four
// pixels each; each warp (a 16x8 strip) replays, back to front, the list of
// entries its strip composited (the forward's per-strip list; or, if that
// overflowed, the bin range below the strip's last composited entry) on its
// own: no CTA barrier, records staged per warp by cp.async one 32-entry batch
// ahead.  Per pair (PAPER.md:1230-1268 chain, R10, R13):
//   W_i = W_{i+1} / (1 - a_i),  dL/dc = g a_i W_i,
//   dL/da = W_i sum_k g_k (c_k - S_k),  S <- c a + (1 - a) S,
//   dL/do = dL/da T,  dL/dT = dL/da o,
//   dT/dh = -(nu+2)/(2 nu) T / (1 + h/nu)
//   dT/dnu = T [-1/2 ln(1 + h/nu) + (nu+2) h / (2 nu^2 (1 + h/nu))]  (R13)
//   dh/dmu2D = -2 Q d,  dh/d(A, B, C) = (dx^2, 2 dx dy, dy^2).
// The replay keeps only W and the scalar g.S per pixel; a thread sums its
// four pixels' contributions (the five geometry gradients from three row
// sums), the warp reduces the 10 values with a butterfly reduce-scatter (12
// shuffles instead of 50) and issues one RED (10 lanes, one 40-byte record)
// into the screen-space gradient record g2d[v][i] in the workspace.
//
// a6: with target != NULL the L1 image gradient sign(C - target)/(3HW) is
// formed in the same kernel (no image-gradient buffer) and the loss summed.
//
// a5 projection backward.  One thread per component loops over the views
// of the launch: it reads g2d[v][i] (and clears it), recomputes the view's
// projection in fp32 and applies the chain of Eq. 4 (Sigma2D = J W Sigma W^T
// J^T, mu2D = pinhole(W mu + t)), the SH view direction and colour clamp,
// and finally the chain Sigma -> (R(q), S) -> (q, log_scale) and the
// reparameterisations o = tanh(raw), nu = 1 + softplus(raw) once for all
// views.  grad += result (one read-modify-write of the 240 B per component).
#include <cstdlib>

#include "raster.cuh"

namespace sss {
namespace {

// 10-value butterfly reduce-scatter (12 shuffles): returns, in lane L, the
// warp sum of value index reduce10_index(L) (< 0: L holds nothing).  Both
// lanes of an even/odd pair hold the same sum.
__device__ __forceinline__ float warp_reduce10(const float* v, int lane) {
  const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4, b1 = lane & 2;
  float a[5];
#pragma unroll
  for (int k = 0; k < 5; ++k) {  // xor 16: keep index k + 5 b4
    const float send = b4 ? v[k] : v[k + 5];
    const float keep = b4 ? v[k + 5] : v[k];
    a[k] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
  // xor 8: b3 = 0 keeps (0, 1, 2), b3 = 1 keeps (3, 4)
  const float c0 = (b3 ? a[3] : a[0]) + __shfl_xor_sync(0xffffffffu, b3 ? a[0] : a[3], 8);
  const float c1 = (b3 ? a[4] : a[1]) + __shfl_xor_sync(0xffffffffu, b3 ? a[1] : a[4], 8);
  const float c2 = (b3 ? 0.f : a[2]) + __shfl_xor_sync(0xffffffffu, b3 ? a[2] : 0.f, 8);
  // xor 4: b2 = 0 keeps (c0, c1), b2 = 1 keeps (c2)
  const float d0 = (b2 ? c2 : c0) + __shfl_xor_sync(0xffffffffu, b2 ? c0 : c2, 4);
  const float d1 = (b2 ? 0.f : c1) + __shfl_xor_sync(0xffffffffu, b2 ? c1 : 0.f, 4);
  // xor 2, xor 1
  const float e = (b1 ? d1 : d0) + __shfl_xor_sync(0xffffffffu, b1 ? d0 : d1, 2);
  return e + __shfl_xor_sync(0xffffffffu, e, 1);
}

__device__ __forceinline__ int reduce10_index(int lane) {
  const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4, b1 = lane & 2;
  const int sub = b3 ? (b2 ? -1 : 3 + (b1 ? 1 : 0)) : (b2 ? (b1 ? -1 : 2) : (b1 ? 1 : 0));
  return sub < 0 ? -1 : 5 * (b4 ? 1 : 0) + sub;
}

// Backward state of a horizontally adjacent pixel pair (packed FP32x2).
// Only the scalar gS = g . S of the suffix colour S is needed:
// dL/da_i = W_i (g.c_i - g.S_i) and g.S_{i-1} = a_i g.c_i + (1 - a_i) g.S_i.
struct PixB2 {
  float2 W, gS, g0, g1, g2;
};

// Per-thread sums over its pixels for one entry (lane-wise over the pairs;
// the two lanes are added once per entry).  The thread's pixels share a row
// (one dy), so the five geometry moments S1..S5 = sum dh (dx, dy, dx^2,
// dx dy, dy^2) follow from sum dh, sum dh dx and sum dh dx^2; the record
// stores them and the projection backward maps them once per record:
//   d mu2D = -2 Q (S1, S2),  d(A, B, C) = (S3, 2 S4, S5).
struct EntrySums2 {
  float2 sdh, sdhdx, sdhdx2, dc0, dc1, dc2, dO, dnu;
};

__device__ __forceinline__ float& lane_of(float2& v, int k) { return (k & 1) ? v.y : v.x; }

// Adds one composited pair's contribution (for both pixels of a pixel pair)
// to the thread's entry sums and steps the replay state (W_i = W_{i+1} /
// (1 - a_i), g.S).  Predicated per pixel on `inc`: with a = 0 the replay
// state is bit-unchanged (W / (1 - 0) = W, gS + (gc - gS) 0 = gS) and every
// contribution is zero, so a warp runs its pixels' chains branch-free.
// T / (1 + h/nu) comes from one ex2 of (e - 1) log2(1 + h/nu) (T = that
// times 1 + h/nu), so a pair costs lg2, ex2 and rcp(1 - a) on the MUFU pipe.
// GENERAL handles the rare warp-uniform cases (as the forward): nu > 32
// (accurate log1p), the Gaussian kernel of the ablation variant (inv_nu = 0:
// T = exp(-h/2), dT/dh = -T/2, dT/dnu = 0) and |o| > 0.989, where the +-0.99
// clamp (R10) can bind and then cuts the gradient.
// FIRST: the entry's sums start at this pair (assigned, not added to zeros)
template <bool NU_PAPER, bool GENERAL, bool FIRST>
__device__ __forceinline__ void pair_grad2(PixB2& p, float2 dx, float2 h, float4 b, float4 c, float einu,
                                           EntrySums2& e, bool inc0, bool inc1) {
  const float2 t = mul2(h, bc2(b.w));
  // 1 + h/nu, kept finite: an excluded pixel far from a very thin splat can
  // have h = inf, and T = Topt (1 + h/nu) must give 0 there, not 0 * inf
  const float2 opt1 = add2(t, bc2(1.f));  // the forward's rounding (never contracted)
  const float2 opt = make_float2(fminf(opt1.x, 3.0e38f), fminf(opt1.y, 3.0e38f));
  float2 lg, exm;
  if (GENERAL && b.w == 0.f) {  // Gaussian variant: T = exp(-h/2), t = 0, lg = 0
    lg = bc2(0.f);
    exm = mul2(h, bc2(kGaussExp2));
  } else {
    if (GENERAL && b.w < (1.f / 32.f)) {
      lg = make_float2(log2_1p(t.x, true), log2_1p(t.y, true));
    } else {
      lg = make_float2(lg2_approx(opt.x), lg2_approx(opt.y));
    }
    exm = mul2(lg, bc2(c.x - 1.f));
  }
  if (!GENERAL) {  // an excluded pixel gets T = 0: every contribution and the replay step vanish
    exm.x = inc0 ? exm.x : -INFINITY;
    exm.y = inc1 ? exm.y : -INFINITY;
  }
  const float2 Topt = make_float2(ex2_approx(exm.x), ex2_approx(exm.y));  // T / (1 + h/nu)
  const float2 T = mul2(Topt, opt);
  const float2 araw = mul2(T, bc2(b.z));
  float2 alpha;
  if (GENERAL) {
    alpha.x = inc0 ? fminf(fmaxf(araw.x, -kAlphaMax), kAlphaMax) : 0.f;
    alpha.y = inc1 ? fminf(fmaxf(araw.y, -kAlphaMax), kAlphaMax) : 0.f;
  } else {
    alpha = araw;  // 0 for excluded pixels (T = 0)
  }
  const float2 oma = sub2(bc2(1.f), alpha);  // 1 - a >= 0.01 (R10): no range fix-up
  const float2 Wi = mul2(p.W, make_float2(rcp_approx(oma.x), rcp_approx(oma.y)));
  const float2 aw = mul2(alpha, Wi);
  e.dc0 = FIRST ? mul2(p.g0, aw) : fma2(p.g0, aw, e.dc0);
  e.dc1 = FIRST ? mul2(p.g1, aw) : fma2(p.g1, aw, e.dc1);
  e.dc2 = FIRST ? mul2(p.g2, aw) : fma2(p.g2, aw, e.dc2);
  const float2 gc = fma2(p.g0, bc2(c.y), fma2(p.g1, bc2(c.z), mul2(p.g2, bc2(c.w))));
  const float2 diff = sub2(gc, p.gS);
  float2 da = mul2(diff, Wi);
  p.gS = fma2(diff, alpha, p.gS);
  p.W = Wi;
  if (GENERAL) {  // R10: no gradient through the clamp
    da.x = (inc0 && fabsf(araw.x) <= kAlphaMax) ? da.x : 0.f;
    da.y = (inc1 && fabsf(araw.y) <= kAlphaMax) ? da.y : 0.f;
  }  // (fast path: an excluded pixel's da multiplies T = 0 and Topt = 0 below)
  e.dO = FIRST ? mul2(da, T) : fma2(da, T, e.dO);
  const float2 dT = mul2(da, bc2(b.z));
  const float2 dh = mul2(mul2(dT, bc2(einu)), Topt);
  const float2 met = mul2(t, bc2(-einu));
  const float2 dTdnu = NU_PAPER ? mul2(met, Topt)
                                : fma2(met, Topt, mul2(T, mul2(lg, bc2(-0.34657359027997264f))));
  e.dnu = FIRST ? mul2(dT, dTdnu) : fma2(dT, dTdnu, e.dnu);
  const float2 dhdx = mul2(dh, dx);
  e.sdh = FIRST ? dh : add2(e.sdh, dh);
  e.sdhdx = FIRST ? dhdx : add2(e.sdhdx, dhdx);
  e.sdhdx2 = FIRST ? mul2(dhdx, dx) : fma2(dhdx, dx, e.sdhdx2);
}

#ifndef SSS_BWD_SMEM_PTRS
#define SSS_BWD_SMEM_PTRS 1
#endif
template <bool FILTER, bool L1, bool NUP>
__global__ void __launch_bounds__(kRasterThreads, kBwdMinBlocks) render_bwd_kernel(
    const float4* __restrict__ rec, const float4* __restrict__ col, const short4* __restrict__ rect,
    const int32_t* __restrict__ ids,
    const int32_t* __restrict__ ranges, RasterGeom G, float bg0, float bg1, float bg2,
    const float* __restrict__ rgb, const float* __restrict__ final_T, const int32_t* __restrict__ last,
    const float* __restrict__ d_rgb, const void* __restrict__ target, float* __restrict__ loss_out,
    float* __restrict__ g2d, const int32_t* __restrict__ tile_list, const int32_t* __restrict__ tile_count,
    int32_t tile_cap, int v0, bool tu8) {
  __shared__ WarpStage stage[kRasterWarps];
  // views v0 + blockIdx.y; g2d points at view v0's records and the entry
  // tags are 32-bit record offsets from it (the host sizes the view groups
  // so that they fit), so the RED address is one 32-bit add + one wide IMAD
  const int v = v0 + (int)blockIdx.y;
  const uint32_t vtag = (uint32_t)blockIdx.y * (uint32_t)G.n * (uint32_t)SSS_G2D_FLOATS;
  const int tile = blockIdx.x;
  const int tx = tile % G.tiles_x, ty = tile / G.tiles_x;
  const int bin = (ty >> G.shift) * G.bins_x + (tx >> G.shift);
  const BinList BL = bin_list(G, ids, ranges, v, bin);
  const int32_t start = BL.start;
  int lx, ly, sx, sy;
  pixels_of(threadIdx.x, lx, ly, sx, sy);
  const int x0 = tx * kTile + lx, y = ty * kTile + ly;
  const float py = (float)y + 0.5f;
  const int w = threadIdx.x >> 5, lane = lane_id();
  const unsigned lt = (1u << lane) - 1u;
  const int64_t HW = (int64_t)G.width * G.height;
  const float inv3P = 1.0f / (3.0f * (float)HW);

  PixB2 q[kPairs];
  float2 px[kPairs];
  int32_t qlast[kPX];
  float lsum = 0.f;
  int32_t m = start;
#pragma unroll
  for (int k = 0; k < kPX; ++k) {
    PixB2& qq = q[k >> 1];
    float &W = lane_of(qq.W, k), &gS = lane_of(qq.gS, k);
    float &g0 = lane_of(qq.g0, k), &g1 = lane_of(qq.g1, k), &g2 = lane_of(qq.g2, k);
    W = 1.f;
    gS = g0 = g1 = g2 = 0.f;
    qlast[k] = start;
    lane_of(px[k >> 1], k) = (float)(x0 + k) + 0.5f;
    if (!(x0 + k < G.width && y < G.height)) continue;
    const int64_t pix = (int64_t)y * G.width + x0 + k;
    qlast[k] = last[(int64_t)v * HW + pix];
    W = final_T[(int64_t)v * HW + pix];
    m = max(m, qlast[k]);
    if (L1) {
      const float* cimg = rgb + (int64_t)v * 3 * HW + pix;
      float t0, t1, t2;
      if (tu8) {  // 8-bit targets: u / 255, correctly rounded (SSS_BWD_TARGET_U8)
        const uint8_t* t8 = static_cast<const uint8_t*>(target) + (int64_t)v * 3 * HW + pix;
        t0 = __fdiv_rn((float)t8[0], 255.f);
        t1 = __fdiv_rn((float)t8[HW], 255.f);
        t2 = __fdiv_rn((float)t8[2 * HW], 255.f);
      } else {
        const float* timg = static_cast<const float*>(target) + (int64_t)v * 3 * HW + pix;
        t0 = timg[0];
        t1 = timg[HW];
        t2 = timg[2 * HW];
      }
      const float d0 = cimg[0] - t0, d1 = cimg[HW] - t1, d2 = cimg[2 * HW] - t2;
      g0 = d0 > 0.f ? inv3P : (d0 < 0.f ? -inv3P : 0.f);
      g1 = d1 > 0.f ? inv3P : (d1 < 0.f ? -inv3P : 0.f);
      g2 = d2 > 0.f ? inv3P : (d2 < 0.f ? -inv3P : 0.f);
      lsum += fabsf(d0) + fabsf(d1) + fabsf(d2);
    } else {
      const float* gimg = d_rgb + (int64_t)v * 3 * HW + pix;
      g0 = gimg[0];
      g1 = gimg[HW];
      g2 = gimg[2 * HW];
    }
    gS = fmaf(g0, bg0, fmaf(g1, bg1, g2 * bg2));  // S_n = bg (R12)
  }
  // the warp's replay start = max over its pixels of `last`; loss partial sums
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (L1) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
    if (loss_out && lane == 0) atomicAdd(loss_out, lsum * inv3P);
  }
  const int32_t wlast = m;
  if (lane == 0) SSS_COUNT(7, wlast - start);

  const float4* rv = rec + (int64_t)v * G.n * 2;  // geometry records (2 x float4)
  const float4* cv = col + (int64_t)v * G.n;      // colour records
  const short4* rcv = rect + (int64_t)v * G.n;
  const uint16_t* tmv = G.tmask ? G.tmask + (int64_t)v * G.capacity : nullptr;
  WarpStage& S = stage[w];
  const int ridx = reduce10_index(lane);
  // opaque copies of the lane and of the lane's slot in the 10-float record
  // (-1: not a writer): otherwise the compiler re-derives them from %tid in
  // every entry (an S2R and ~15 integer ops)
  int lane_o, roff;
  lane_o = __shfl_sync(0xffffffffu, lane, lane);  // opaque to ptxas too (an asm mov is not: -0.3 ms)
  asm volatile("mov.b32 %0, %1;" : "=r"(roff) : "r"(!(lane & 1) && ridx >= 0 ? ridx : -1));

  // The forward's list of the entries this warp's strip composited: replay
  // only those; else (no lists, or this list overflowed) the whole
  // [start, wlast) range.  Each warp walks its entries on its own (no CTA
  // barrier): batches of 32 list indices from the top; lanes keep the
  // entries before the warp's replay start (and, unlisted with bins, those
  // whose rect covers the tile), compact them by ballot and gather their
  // records into the next stage buffer.  Pipeline: positions two batches
  // ahead, ids one batch ahead (registers), records one batch ahead
  // (cp.async).
  const int64_t lslot = ((int64_t)v * G.tiles_x * G.tiles_y + tile) * kRasterWarps + w;
  const int32_t tcount = tile_list ? tile_count[lslot] : 0;
  const bool use_list = tile_list != nullptr && tcount <= tile_cap;
  const int32_t* tl = use_list ? tile_list + lslot * tile_cap : nullptr;
  const int32_t lbeg = use_list ? 0 : start;
  const int32_t lend = use_list ? tcount : wlast;
#if SSS_BWD_SMEM_PTRS
  // the warp's per-batch bases live in shared memory (the compiler would
  // otherwise rebuild the 64-bit addresses from the block indices at every
  // batch: the registers are all taken by the pixel state)
  __shared__ const void* s_bp[kRasterWarps][5];
  if (lane == 0) {
    s_bp[w][0] = tl;
    s_bp[w][1] = BL.ids;
    s_bp[w][2] = BL.tail ? BL.tail + BL.tail0 - BL.mend : nullptr;  // index by the list position
    s_bp[w][3] = rv;
    s_bp[w][4] = cv;
  }
  __syncwarp();
  auto pos_at = [&](int32_t h) -> int32_t {  // lane's entry of the batch [max(lbeg, h - 32), h)
    const int32_t li = h - kWB + lane;
    if (h <= lbeg || li < lbeg) return INT32_MAX;
    return use_list ? __ldg(static_cast<const int32_t*>(s_bp[w][0]) + li) : li;
  };
  auto id_at = [&](int32_t p) -> int32_t {
    return p >= wlast ? -1 : p < BL.mend ? __ldg(static_cast<const int32_t*>(s_bp[w][1]) + p)
                                         : __ldg(static_cast<const int32_t*>(s_bp[w][2]) + p);
  };
#else
  auto pos_at = [&](int32_t h) -> int32_t {  // lane's entry of the batch [max(lbeg, h - 32), h)
    const int32_t li = h - kWB + lane;
    if (h <= lbeg || li < lbeg) return INT32_MAX;
    return use_list ? __ldg(tl + li) : li;
  };
  auto id_at = [&](int32_t p) -> int32_t { return p < wlast ? BL.id(p) : -1; };
#endif
  auto issue = [&](int buf, int32_t p, int32_t id) -> int {
    bool ok = id >= 0;
    // unlisted replay: filter by the tile rect with bins, and always in the
    // truncated list's tail (the depth-sorted visible set)
    if (!use_list && ok && (FILTER || p >= BL.mend)) ok = entry_in_tile(G, tmv, p, BL.mend, id, rcv, tx, ty);
    // tag: the entry's g2d record offset from view v0's (uint32, see above)
#if SSS_BWD_SMEM_PTRS
    return stage_batch(S, buf, ok, p, id, static_cast<const float4*>(s_bp[w][3]),
                       static_cast<const float4*>(s_bp[w][4]), lt, (int32_t)(vtag + (uint32_t)id * SSS_G2D_FLOATS));
#else
    return stage_batch(S, buf, ok, p, id, rv, cv, lt, (int32_t)(vtag + (uint32_t)id * SSS_G2D_FLOATS));
#endif
  };

  int32_t hi = lend;
  int nb = 0;
  int32_t p2, i2, p3;
  {
    const int32_t p1 = pos_at(hi);
    nb = issue(0, p1, id_at(p1));
    p2 = pos_at(hi - kWB);
    i2 = id_at(p2);
    p3 = pos_at(hi - 2 * kWB);
  }
  int buf = 0;
  for (; hi > lbeg; hi -= kWB) {
    const int nb_next = hi - kWB > lbeg ? issue(buf ^ 1, p2, i2) : (cp_async_commit(), 0);
    i2 = id_at(p3);
    p2 = p3;
    p3 = pos_at(hi - 3 * kWB);
    cp_async_wait1();  // this batch's records have landed
    __syncwarp();
    if (lane == 0) { SSS_COUNT(0, 1); SSS_COUNT(6, nb); }
    for (int j = nb - 1; j >= 0; --j) {
      if (lane == 0) SSS_COUNT(1, 1);
      const int32_t pj = S.pos(buf, j);
      const float4 a = S.rec(buf, 0, j);
      const float4 b = S.rec(buf, 1, j);  // {C, hmax, o, inv_nu}
      const float dy = __fsub_rn(py, a.y);
      const float bdy = __fmul_rn(a.w, dy);
      const float cdy2 = __fmul_rn(__fmul_rn(b.x, dy), dy);
      float2 h[kPairs], dx[kPairs];
      bool inc[kPX];
      bool any = false;
#pragma unroll
      for (int k = 0; k < kPairs; ++k) {
        h[k] = h_f32_pair(px[k], a.x, a.z, bdy, cdy2, dx[k]);  // dx kept for the gradient
        inc[2 * k] = pj < qlast[2 * k] && h[k].x <= b.y;
        inc[2 * k + 1] = pj < qlast[2 * k + 1] && h[k].y <= b.y;
        any = any || inc[2 * k] || inc[2 * k + 1];
      }
#ifdef SSS_COUNTERS
      {
        const unsigned ba = __ballot_sync(0xffffffffu, any);
        int ninc = 0, nlive = 0;
        for (int k = 0; k < kPX; ++k) {
          ninc += __popc(__ballot_sync(0xffffffffu, inc[k]));
          nlive += __popc(__ballot_sync(0xffffffffu, pj < qlast[k]));
        }
        if (lane == 0) { SSS_COUNT(3, ba != 0); SSS_COUNT(4, ninc); SSS_COUNT(5, nlive); }
      }
#endif
      if (!__any_sync(0xffffffffu, any)) continue;
      const float4 c = S.rec(buf, 2, j);  // {e, r, g, b}
      // e / nu = -(nu+2)/(2 nu): dT/dh = einu T/(1 + h/nu); -1/2 for the Gaussian variant
      const float einu = b.w == 0.f ? -0.5f : c.x * b.w;
      static_assert(kPairs == 2, "two pixel pairs per thread");
      EntrySums2 e2;
      if (fabsf(b.z) > 0.989f || b.w < (1.f / 32.f)) {  // warp-uniform, rare
        pair_grad2<NUP, true, true>(q[0], dx[0], h[0], b, c, einu, e2, inc[0], inc[1]);
        pair_grad2<NUP, true, false>(q[1], dx[1], h[1], b, c, einu, e2, inc[2], inc[3]);
      } else {
        pair_grad2<NUP, false, true>(q[0], dx[0], h[0], b, c, einu, e2, inc[0], inc[1]);
        pair_grad2<NUP, false, false>(q[1], dx[1], h[1], b, c, einu, e2, inc[2], inc[3]);
      }
      // geometry: the five moments sum dh (dx, dy, dx^2, dx dy, dy^2); the
      // linear map to d mu2D (through the conic) is applied once per record
      // by the projection backward
      const float sdh = e2.sdh.x + e2.sdh.y, sdhdx = e2.sdhdx.x + e2.sdhdx.y;
      const float dysdh = dy * sdh;
      float vals[10];
      vals[0] = sdhdx;                                  // S1 = sum dh dx
      vals[1] = dysdh;                                  // S2 = sum dh dy
      vals[2] = e2.sdhdx2.x + e2.sdhdx2.y;              // S3 = sum dh dx^2 = d A
      vals[3] = dy * sdhdx;                             // S4 = sum dh dx dy = d B / 2
      vals[4] = dy * dysdh;                             // S5 = sum dh dy^2 = d C
      vals[5] = e2.dc0.x + e2.dc0.y;
      vals[6] = e2.dc1.x + e2.dc1.y;
      vals[7] = e2.dc2.x + e2.dc2.y;
      vals[8] = e2.dO.x + e2.dO.y;
      vals[9] = e2.dnu.x + e2.dnu.y;
      const float r = warp_reduce10(vals, lane_o);
      // one RED per warp and entry: lanes 0, 2, .. hold the 10 sums of the
      // 40-byte screen-space gradient record g2d[v][id]
      if (roff >= 0 && r != 0.f) atomicAdd(g2d + ((uint32_t)S.id(buf, j) + (uint32_t)roff), r);
    }
    __syncwarp();  // this buffer is refilled two batches on
    nb = nb_next;
    buf ^= 1;
  }
}

// ------------------------------------------------------------ a5
__device__ __forceinline__ void sh_basis_f(int deg, float x, float y, float z, float* Y) {
  Y[0] = 0.28209479177387814f;
  if (deg >= 1) {
    Y[1] = -0.4886025119029199f * y;
    Y[2] = 0.4886025119029199f * z;
    Y[3] = -0.4886025119029199f * x;
  }
  if (deg >= 2) {
    const float xx = x * x, yy = y * y, zz = z * z;
    Y[4] = 1.0925484305920792f * x * y;
    Y[5] = -1.0925484305920792f * y * z;
    Y[6] = 0.31539156525252005f * (2.f * zz - xx - yy);
    Y[7] = -1.0925484305920792f * x * z;
    Y[8] = 0.5462742152960396f * (xx - yy);
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
  }
}

// sum_m coef_m * dY_m/d(x,y,z), coef_m = sum_c gdc_c sh_{m,c}
__device__ __forceinline__ void sh_dir_grad(int deg, float x, float y, float z, const float* coef, float g[3]) {
  g[0] = g[1] = g[2] = 0.f;
  if (deg < 1) return;
  const float c1 = 0.4886025119029199f;
  g[1] += -c1 * coef[1];
  g[2] += c1 * coef[2];
  g[0] += -c1 * coef[3];
  if (deg < 2) return;
  const float c20 = 1.0925484305920792f, c22 = 0.31539156525252005f, c24 = 0.5462742152960396f;
  g[0] += c20 * y * coef[4];  g[1] += c20 * x * coef[4];
  g[1] += -c20 * z * coef[5]; g[2] += -c20 * y * coef[5];
  g[0] += -2.f * c22 * x * coef[6]; g[1] += -2.f * c22 * y * coef[6]; g[2] += 4.f * c22 * z * coef[6];
  g[0] += -c20 * z * coef[7]; g[2] += -c20 * x * coef[7];
  g[0] += 2.f * c24 * x * coef[8]; g[1] += -2.f * c24 * y * coef[8];
  if (deg < 3) return;
  const float c30 = 0.5900435899266435f, c31 = 2.890611442640554f, c32 = 0.4570457994644658f;
  const float c33 = 0.3731763325901154f, c35 = 1.445305721320277f;
  const float xx = x * x, yy = y * y, zz = z * z;
  g[0] += -6.f * c30 * x * y * coef[9];
  g[1] += -c30 * (3.f * xx - 3.f * yy) * coef[9];
  g[0] += c31 * y * z * coef[10]; g[1] += c31 * x * z * coef[10]; g[2] += c31 * x * y * coef[10];
  g[0] += 2.f * c32 * x * y * coef[11];
  g[1] += -c32 * (4.f * zz - xx - 3.f * yy) * coef[11];
  g[2] += -8.f * c32 * y * z * coef[11];
  g[0] += -6.f * c33 * x * z * coef[12];
  g[1] += -6.f * c33 * y * z * coef[12];
  g[2] += c33 * (6.f * zz - 3.f * xx - 3.f * yy) * coef[12];
  g[0] += -c32 * (4.f * zz - 3.f * xx - yy) * coef[13];
  g[1] += 2.f * c32 * x * y * coef[13];
  g[2] += -8.f * c32 * x * z * coef[13];
  g[0] += 2.f * c35 * x * z * coef[14];
  g[1] += -2.f * c35 * y * z * coef[14];
  g[2] += c35 * (xx - yy) * coef[14];
  g[0] += -c30 * (3.f * xx - 3.f * yy) * coef[15];
  g[1] += 6.f * c30 * x * y * coef[15];
}

template <int DEG>
#ifndef SSS_PROJB_L2_AHEAD
#define SSS_PROJB_L2_AHEAD 1  // L2 prefetch of the record two views on (-3.5% project_bwd)
#endif
#ifndef SSS_PROJB_MINB
#define SSS_PROJB_MINB 3  // 168 registers (80 B spilled at degree 3, 432 B at 4 CTAs/SM): -0.7 ms per 64 views
#endif
__global__ void __launch_bounds__(128, SSS_PROJB_MINB) project_bwd_kernel(sss_params P, const __grid_constant__ CamPack cp,
                                                           int nv, int v0, float2* __restrict__ g2d,
                                                           sss_params Gd, int64_t i0, int64_t i1, bool assign) {
  constexpr int K = (DEG + 1) * (DEG + 1);
  const int64_t n = P.n;
  const int64_t i = i0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= i1) return;
  float mu[3], s[3], q[4];
  for (int k = 0; k < 3; ++k) mu[k] = P.mean[k * n + i];
  for (int k = 0; k < 3; ++k) s[k] = P.log_scale[k * n + i];
  for (int k = 0; k < 4; ++k) q[k] = P.rot[k * n + i];
  const float raw_nu = P.raw_nu[i], raw_o = P.raw_opacity[i];
  float sh[3 * K];
#pragma unroll
  for (int k = 0; k < 3 * K; ++k) sh[k] = P.sh[k * n + i];
  // view-independent
  const float qn = sqrtf(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
  const float qw = q[0] / qn, qx = q[1] / qn, qy = q[2] / qn, qz = q[3] / qn;
  float R[9];
  R[0] = 1.f - 2.f * (qy * qy + qz * qz);
  R[1] = 2.f * (qx * qy - qw * qz);
  R[2] = 2.f * (qx * qz + qw * qy);
  R[3] = 2.f * (qx * qy + qw * qz);
  R[4] = 1.f - 2.f * (qx * qx + qz * qz);
  R[5] = 2.f * (qy * qz - qw * qx);
  R[6] = 2.f * (qx * qz - qw * qy);
  R[7] = 2.f * (qy * qz + qw * qx);
  R[8] = 1.f - 2.f * (qx * qx + qy * qy);
  const float S[3] = {expf(s[0]), expf(s[1]), expf(s[2])};
  float M[9], Sig[9];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) M[a * 3 + b] = R[a * 3 + b] * S[b];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b)
      Sig[a * 3 + b] = M[a * 3 + 0] * M[b * 3 + 0] + M[a * 3 + 1] * M[b * 3 + 1] + M[a * 3 + 2] * M[b * 3 + 2];

  float gSig[9] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  float gmu[3] = {0.f, 0.f, 0.f};
  float gsh[3 * K];
#pragma unroll
  for (int k = 0; k < 3 * K; ++k) gsh[k] = 0.f;
  float g_o = 0.f, g_nu = 0.f;
  bool any = false;

  // software pipeline: the next view's 40-byte record is in flight while this
  // view's chain runs (streaming loads: each record is read once)
  float2 N[5];
#pragma unroll
  for (int k = 0; k < 5; ++k) N[k] = make_float2(0.f, 0.f);
  if (nv > 0) {
    const float2* gp0 = g2d + ((int64_t)v0 * n + i) * 5;
#pragma unroll
    for (int k = 0; k < 5; ++k) N[k] = __ldcs(gp0 + k);
  }
  for (int vv = 0; vv < nv; ++vv) {
    float2* gp = g2d + ((int64_t)(v0 + vv) * n + i) * 5;
    const float4 G0 = make_float4(N[0].x, N[0].y, N[1].x, N[1].y);
    const float4 G1 = make_float4(N[2].x, N[2].y, N[3].x, N[3].y);
    const float2 G2 = N[4];
    if (vv + 1 < nv) {
      const float2* gq = gp + (int64_t)n * 5;
#pragma unroll
      for (int k = 0; k < 5; ++k) N[k] = __ldcs(gq + k);
#if SSS_PROJB_L2_AHEAD
      if (vv + 1 + SSS_PROJB_L2_AHEAD < nv)  // the record SSS_PROJB_L2_AHEAD views further on, into L2
        asm volatile("prefetch.global.L2 [%0];" ::"l"(gq + (int64_t)n * 5 * SSS_PROJB_L2_AHEAD));
#endif
    }
    const bool nz = (G0.x != 0.f) | (G0.y != 0.f) | (G0.z != 0.f) | (G0.w != 0.f) | (G1.x != 0.f) |
                    (G1.y != 0.f) | (G1.z != 0.f) | (G1.w != 0.f) | (G2.x != 0.f) | (G2.y != 0.f);
    if (!nz) continue;
    any = true;
    const float2 z2 = make_float2(0.f, 0.f);
#pragma unroll
    for (int k = 0; k < 5; ++k) __stcs(gp + k, z2);  // consume-and-clear (workspace stays zero)
    const DevCamera& cam = cp.cam[vv];
    float p[3];
    for (int a = 0; a < 3; ++a) p[a] = cam.R[a * 3 + 0] * mu[0] + cam.R[a * 3 + 1] * mu[1] + cam.R[a * 3 + 2] * mu[2] + cam.t[a];
    const float px = p[0], py = p[1], pz = p[2];
    const float iz = 1.f / pz;
    const float J00 = cam.fx * iz, J02 = -cam.fx * px * iz * iz, J11 = cam.fy * iz, J12 = -cam.fy * py * iz * iz;
    // Sc = Rc Sig Rc^T
    float T1[9], Sc[9];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b)
        T1[a * 3 + b] = cam.R[a * 3 + 0] * Sig[0 * 3 + b] + cam.R[a * 3 + 1] * Sig[1 * 3 + b] + cam.R[a * 3 + 2] * Sig[2 * 3 + b];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b)
        Sc[a * 3 + b] = T1[a * 3 + 0] * cam.R[b * 3 + 0] + T1[a * 3 + 1] * cam.R[b * 3 + 1] + T1[a * 3 + 2] * cam.R[b * 3 + 2];
    // J (2x3) with J01 = J10 = 0
    const float J[6] = {J00, 0.f, J02, 0.f, J11, J12};
    float K2[6];
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 3; ++b) K2[a * 3 + b] = J[a * 3 + 0] * Sc[0 * 3 + b] + J[a * 3 + 1] * Sc[1 * 3 + b] + J[a * 3 + 2] * Sc[2 * 3 + b];
    float cxx = K2[0] * J[0] + K2[2] * J[2];
    const float cxy = K2[1] * J[4] + K2[2] * J[5];
    float cyy = K2[4] * J[4] + K2[5] * J[5];
    if (P.variant & SSS_VARIANT_LOWPASS) {  // conic of Sigma2D + 0.3 I; d(Sigma2D + 0.3 I) = d Sigma2D
      cxx += kLowpass;
      cyy += kLowpass;
    }
    const float idet = 1.f / (cxx * cyy - cxy * cxy);
    const float QA = cyy * idet, QB = -cxy * idet, QC = cxx * idet;
    // the raster's moments S1..S5 (G0.xyzw, G1.x): dA = S3, dB/2 = S4,
    // dC = S5, d mu2D = -2 Q (S1, S2) (h = d^T Q d, dh/dmu2D = -2 Q d)
    // G_S = -Q G_Q Q with G_Q = [[dA, dB/2], [dB/2, dC]]
    const float gA = G0.z, gB = G0.w, gC = G1.x;
    const float QG00 = QA * gA + QB * gB, QG01 = QA * gB + QB * gC;
    const float QG10 = QB * gA + QC * gB, QG11 = QB * gB + QC * gC;
    const float GS00 = -(QG00 * QA + QG01 * QB);
    const float GS01 = -(QG00 * QB + QG01 * QC);
    const float GS11 = -(QG10 * QB + QG11 * QC);
    const float GS[4] = {GS00, GS01, GS01, GS11};
    // dL/dSc = J^T GS J ; dL/dJ = 2 GS J Sc
    float GSc[9];
    {
      float U[6];  // GS J (2x3), then GSc = J^T (GS J)
      for (int k = 0; k < 2; ++k)
        for (int b = 0; b < 3; ++b) U[k * 3 + b] = GS[k * 2 + 0] * J[0 * 3 + b] + GS[k * 2 + 1] * J[1 * 3 + b];
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) GSc[a * 3 + b] = J[0 * 3 + a] * U[0 * 3 + b] + J[1 * 3 + a] * U[1 * 3 + b];
    }
    float JS[6];
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 3; ++b) JS[a * 3 + b] = J[a * 3 + 0] * Sc[0 * 3 + b] + J[a * 3 + 1] * Sc[1 * 3 + b] + J[a * 3 + 2] * Sc[2 * 3 + b];
    float GJ[6];
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 3; ++b) GJ[a * 3 + b] = 2.f * (GS[a * 2 + 0] * JS[0 * 3 + b] + GS[a * 2 + 1] * JS[1 * 3 + b]);
    // dL/dSigma += Rc^T (GSc Rc): two 3x3 products (54 FMAs instead of 81 triple terms)
    {
      float T2[9];
      for (int k = 0; k < 3; ++k)
        for (int b = 0; b < 3; ++b)
          T2[k * 3 + b] = GSc[k * 3 + 0] * cam.R[0 * 3 + b] + GSc[k * 3 + 1] * cam.R[1 * 3 + b] + GSc[k * 3 + 2] * cam.R[2 * 3 + b];
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b)
          gSig[a * 3 + b] += cam.R[0 * 3 + a] * T2[0 * 3 + b] + cam.R[1 * 3 + a] * T2[1 * 3 + b] + cam.R[2 * 3 + a] * T2[2 * 3 + b];
    }
    // camera-space mean through mean2d and J(p)
    const float dmx = -2.f * (QA * G0.x + QB * G0.y), dmy = -2.f * (QB * G0.x + QC * G0.y);
    const float iz2 = iz * iz, iz3 = iz2 * iz;
    float dp0 = cam.fx * iz * dmx + GJ[2] * (-cam.fx * iz2);
    float dp1 = cam.fy * iz * dmy + GJ[5] * (-cam.fy * iz2);
    float dp2 = -cam.fx * px * iz2 * dmx - cam.fy * py * iz2 * dmy + GJ[0] * (-cam.fx * iz2) +
                GJ[4] * (-cam.fy * iz2) + GJ[2] * (2.f * cam.fx * px * iz3) + GJ[5] * (2.f * cam.fy * py * iz3);
    for (int a = 0; a < 3; ++a) gmu[a] += cam.R[0 * 3 + a] * dp0 + cam.R[1 * 3 + a] * dp1 + cam.R[2 * 3 + a] * dp2;
    // SH colour (clamp mask) and view direction
    float dvec[3] = {mu[0] - cam.center[0], mu[1] - cam.center[1], mu[2] - cam.center[2]};
    const float dist = sqrtf(dvec[0] * dvec[0] + dvec[1] * dvec[1] + dvec[2] * dvec[2]);
    const float idist = 1.f / dist;
    const float dx = dvec[0] * idist, dy = dvec[1] * idist, dz = dvec[2] * idist;
    float Y[16];
    sh_basis_f(DEG, dx, dy, dz, Y);
    float gdc[3] = {G1.y, G1.z, G1.w};
    for (int c = 0; c < 3; ++c) {
      float pre = 0.5f;
      for (int mm = 0; mm < K; ++mm) pre += sh[mm * 3 + c] * Y[mm];
      if (!(pre > 0.f)) gdc[c] = 0.f;
    }
#pragma unroll
    for (int mm = 0; mm < K; ++mm)
      for (int c = 0; c < 3; ++c) gsh[mm * 3 + c] += gdc[c] * Y[mm];
    if (DEG > 0) {
      float coef[16];
      for (int mm = 0; mm < K; ++mm) coef[mm] = gdc[0] * sh[mm * 3 + 0] + gdc[1] * sh[mm * 3 + 1] + gdc[2] * sh[mm * 3 + 2];
      float gd[3];
      sh_dir_grad(DEG, dx, dy, dz, coef, gd);
      const float dd = gd[0] * dx + gd[1] * dy + gd[2] * dz;
      gmu[0] += (gd[0] - dx * dd) * idist;
      gmu[1] += (gd[1] - dy * dd) * idist;
      gmu[2] += (gd[2] - dz * dd) * idist;
    }
    g_o += G2.x;
    g_nu += G2.y;
  }
  if (!any) {
    if (assign) {  // grad = 0 for a component no view touched
      int64_t gz;
      const sss_params Gz = block_view(Gd, i, gz);
      for (int a = 0; a < 3; ++a) Gz.mean[a * gz + i] = 0.f;
      for (int a = 0; a < 3; ++a) Gz.log_scale[a * gz + i] = 0.f;
      for (int a = 0; a < 4; ++a) Gz.rot[a * gz + i] = 0.f;
      Gz.raw_nu[i] = 0.f;
      Gz.raw_opacity[i] = 0.f;
#pragma unroll
      for (int k = 0; k < 3 * K; ++k) Gz.sh[k * gz + i] = 0.f;
    }
    return;
  }
  // Sigma = M M^T, M = R S
  float GM[9];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) GM[a * 3 + b] = 2.f * (gSig[a * 3 + 0] * M[0 * 3 + b] + gSig[a * 3 + 1] * M[1 * 3 + b] + gSig[a * 3 + 2] * M[2 * 3 + b]);
  float gls[3];
  for (int b = 0; b < 3; ++b) gls[b] = (GM[0 * 3 + b] * R[0 * 3 + b] + GM[1 * 3 + b] * R[1 * 3 + b] + GM[2 * 3 + b] * R[2 * 3 + b]) * S[b];
  float GR[9];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) GR[a * 3 + b] = GM[a * 3 + b] * S[b];
  float gq[4];
  gq[0] = 2.f * (-qz * GR[1] + qy * GR[2] + qz * GR[3] - qx * GR[5] - qy * GR[6] + qx * GR[7]);
  gq[1] = 2.f * (qy * GR[1] + qz * GR[2] + qy * GR[3] - 2.f * qx * GR[4] - qw * GR[5] + qz * GR[6] + qw * GR[7] - 2.f * qx * GR[8]);
  gq[2] = 2.f * (-2.f * qy * GR[0] + qx * GR[1] + qw * GR[2] + qx * GR[3] + qz * GR[5] - qw * GR[6] + qz * GR[7] - 2.f * qy * GR[8]);
  gq[3] = 2.f * (-2.f * qz * GR[0] - qw * GR[1] + qx * GR[2] + qw * GR[3] - 2.f * qz * GR[4] + qy * GR[5] + qx * GR[6] + qy * GR[7]);
  const float dotq = gq[0] * qw + gq[1] * qx + gq[2] * qy + gq[3] * qz;
  const float qh[4] = {qw, qx, qy, qz};
  // reparameterisations
  const bool positive = P.variant & SSS_VARIANT_POSITIVE;
  const float o = positive ? 1.f / (1.f + expf(-raw_o)) : tanhf(raw_o);
  const float sp = raw_nu > 30.f ? raw_nu : log1pf(expf(raw_nu));
  const float dnu = (1.f + sp >= (float)kNuMax) ? 0.f : 1.f / (1.f + expf(-raw_nu));
  // grad += result: every plane's load is issued before the first store (the
  // planes may alias as far as the compiler knows, which would otherwise
  // serialise each read-modify-write behind the previous store)
  float grot[4];
#pragma unroll
  for (int a = 0; a < 4; ++a) grot[a] = (gq[a] - qh[a] * dotq) / qn;
  const float gnu = g_nu * dnu, gro = g_o * (positive ? o * (1.f - o) : 1.f - o * o);
  int64_t gn;  // plane stride of the gradient (plain or component-blocked, sss.h)
  Gd = block_view(Gd, i, gn);
  {
    float cur[12];
    if (assign) {
#pragma unroll
      for (int a = 0; a < 12; ++a) cur[a] = 0.f;
    } else {
#pragma unroll
      for (int a = 0; a < 3; ++a) cur[a] = Gd.mean[a * gn + i];
#pragma unroll
      for (int a = 0; a < 3; ++a) cur[3 + a] = Gd.log_scale[a * gn + i];
#pragma unroll
      for (int a = 0; a < 4; ++a) cur[6 + a] = Gd.rot[a * gn + i];
      cur[10] = Gd.raw_nu[i];
      cur[11] = Gd.raw_opacity[i];
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) Gd.mean[a * gn + i] = cur[a] + gmu[a];
#pragma unroll
    for (int a = 0; a < 3; ++a) Gd.log_scale[a * gn + i] = cur[3 + a] + gls[a];
#pragma unroll
    for (int a = 0; a < 4; ++a) Gd.rot[a * gn + i] = cur[6 + a] + grot[a];
    Gd.raw_nu[i] = cur[10] + gnu;
    Gd.raw_opacity[i] = cur[11] + gro;
  }
#pragma unroll
  for (int k0 = 0; k0 < 3 * K; k0 += 8) {
    float cur[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (k0 + u < 3 * K) cur[u] = assign ? 0.f : Gd.sh[(k0 + u) * gn + i];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (k0 + u < 3 * K) Gd.sh[(k0 + u) * gn + i] = cur[u] + gsh[k0 + u];
  }
}

}  // namespace
}  // namespace sss

using namespace sss;

SSS_COUNTER_ACCESSOR(sss_dev_counters_bwd)

namespace sss {
// the a5 kernel over components [i0, i1), views in launches of <= 128
static sss_status project_bwd_launch(const sss_params& p, const sss_camera* cams, int n_views, float* g2d,
                                     const sss_params& grad, int64_t i0, int64_t i1, cudaStream_t s,
                                     bool assign = false) {
  if (i1 <= i0) return SSS_OK;
  const int threads = 128;
  const int blocks = div_up(i1 - i0, threads);
  sss_status st;
  for (int v0 = 0; v0 < n_views; v0 += kMaxViewsPerLaunch) {
    const int nv = n_views - v0 < kMaxViewsPerLaunch ? n_views - v0 : kMaxViewsPerLaunch;
    CamPack cp;
    fill_campack(cams, v0, nv, cp);
    switch (p.sh_degree) {
      case 0: project_bwd_kernel<0><<<blocks, threads, 0, s>>>(p, cp, nv, v0, (float2*)g2d, grad, i0, i1,
                                                                 assign && v0 == 0); break;
      case 1: project_bwd_kernel<1><<<blocks, threads, 0, s>>>(p, cp, nv, v0, (float2*)g2d, grad, i0, i1,
                                                                 assign && v0 == 0); break;
      case 2: project_bwd_kernel<2><<<blocks, threads, 0, s>>>(p, cp, nv, v0, (float2*)g2d, grad, i0, i1,
                                                                 assign && v0 == 0); break;
      default: project_bwd_kernel<3><<<blocks, threads, 0, s>>>(p, cp, nv, v0, (float2*)g2d, grad, i0, i1,
                                                                 assign && v0 == 0); break;
    }
    count_launch();
    if ((st = check_launch("sss_render_bwd(projection)")) != SSS_OK) return st;
  }
  return SSS_OK;
}
}  // namespace sss

extern "C" sss_status sss_project_bwd_range(const sss_params* p, const sss_camera* cams, int32_t n_views,
                                            void* ws, size_t ws_bytes, sss_params* grad, int64_t i0, int64_t i1,
                                            void* stream) {
  sss_status st;
  if ((st = validate_params(p, "sss_project_bwd_range")) != SSS_OK) return st;
  if ((st = validate_params(grad, "sss_project_bwd_range(grad)", true)) != SSS_OK) return st;
  if ((st = validate_cams(cams, n_views, "sss_project_bwd_range")) != SSS_OK) return st;
  if (grad->n != p->n || grad->sh_degree != p->sh_degree) {
    set_error("sss_project_bwd_range: n / sh_degree mismatch");
    return SSS_ERR_ARG;
  }
  if (i0 < 0 || i1 > p->n || i0 > i1) { set_error("sss_project_bwd_range: bad range"); return SSS_ERR_ARG; }
  const size_t need = (size_t)p->n * n_views * SSS_G2D_FLOATS * sizeof(float);
  if (ws_bytes < need || (need > 0 && !ws)) {
    set_error("sss_project_bwd_range: workspace %zu < %zu bytes", ws_bytes, need);
    return SSS_ERR_ARG;
  }
  return project_bwd_launch(*p, cams, n_views, (float*)ws, *grad, i0, i1, (cudaStream_t)stream);
}

extern "C" size_t sss_render_bwd_workspace(int64_t n, int32_t n_views) {
  if (n < 0 || n_views <= 0) return 0;
  return (size_t)n * n_views * SSS_G2D_FLOATS * sizeof(float);
}

extern "C" sss_status sss_render_bwd(const sss_params* p, const sss_projected* pr, const sss_bins* bins,
                                     const sss_camera* cams, int32_t n_views, const float* bg,
                                     const sss_frame* fwd, const float* d_rgb, const void* target,
                                     float* loss_out, sss_params* grad, void* ws, size_t ws_bytes,
                                     int32_t flags, void* stream) {
  sss_status st;
  if ((st = validate_params(p, "sss_render_bwd")) != SSS_OK) return st;
  if ((st = validate_params(grad, "sss_render_bwd(grad)", true)) != SSS_OK) return st;
  if ((st = validate_cams(cams, n_views, "sss_render_bwd")) != SSS_OK) return st;
  if (!pr || !bins || !fwd || !bg) { set_error("sss_render_bwd: null argument"); return SSS_ERR_ARG; }
  if (grad->n != p->n || grad->sh_degree != p->sh_degree || pr->n != p->n) {
    set_error("sss_render_bwd: n / sh_degree mismatch");
    return SSS_ERR_ARG;
  }
  if (!(flags & SSS_BWD_PROJECTION_ONLY) && !d_rgb && !target) {
    set_error("sss_render_bwd: need d_rgb or target");
    return SSS_ERR_ARG;
  }
  RasterGeom G;
  if (!raster_geom(pr, bins, cams, n_views, G)) { set_error("sss_render_bwd: geometry mismatch"); return SSS_ERR_SHAPE; }
  if (p->n > (int64_t)(0xffffffffu / SSS_G2D_FLOATS)) {  // 32-bit record offsets in the raster
    set_error("sss_render_bwd: n = %lld > %u components", (long long)p->n, 0xffffffffu / SSS_G2D_FLOATS);
    return SSS_ERR_SHAPE;
  }
  const size_t need = sss_render_bwd_workspace(p->n, n_views);
  if (ws_bytes < need || (need > 0 && !ws)) {
    set_error("sss_render_bwd: workspace %zu < %zu bytes", ws_bytes, need);
    return SSS_ERR_ARG;
  }
  if (!fwd->rgb || !fwd->final_T || !fwd->last) { set_error("sss_render_bwd: null frame buffer"); return SSS_ERR_ARG; }
  if (!(flags & SSS_BWD_PROJECTION_ONLY) && p->n > 0 && (!pr->rec || !pr->col || !pr->rect)) {
    set_error("sss_render_bwd: null projection buffer");
    return SSS_ERR_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  float* g2d = (float*)ws;
  // view groups whose g2d records (n * 10 floats each) span < 2^32 floats:
  // the raster's 32-bit record tags (one group at config 5: 64 x 3M x 10)
  int vg = (int)std::max<int64_t>(1, std::min<int64_t>(n_views, (int64_t)0xffffffffu /
                                                                    std::max<int64_t>(1, p->n * SSS_G2D_FLOATS)));
  if (const char* e = getenv("SSS_BWD_VIEW_GROUP")) vg = std::max(1, std::min(vg, atoi(e)));  // tests: force groups
  const float4* rec = (const float4*)pr->rec;
  const float4* col = (const float4*)pr->col;
  const short4* rect = (const short4*)pr->rect;
#define SSS_BWD_LAUNCH(F, L, N)                                                                           \
  for (int gv0 = 0; gv0 < n_views; gv0 += vg)                                                              \
  render_bwd_kernel<F, L, N><<<dim3(G.tiles_x * G.tiles_y, std::min(vg, n_views - gv0)), kRasterThreads, 0, s>>>( \
      rec, col, rect, bins->ids, bins->ranges, G, bg[0], bg[1], bg[2], fwd->rgb, fwd->final_T, fwd->last,  \
      d_rgb, target, loss_out, g2d + (int64_t)gv0 * p->n * SSS_G2D_FLOATS, fwd->tile_list, fwd->tile_count, \
      fwd->tile_cap, gv0, (flags & SSS_BWD_TARGET_U8) != 0)
#define SSS_BWD_LAUNCH_N(F, L)              \
  do {                                      \
    if (nup) SSS_BWD_LAUNCH(F, L, true);    \
    else SSS_BWD_LAUNCH(F, L, false);       \
  } while (0)
  const bool l1 = d_rgb == nullptr;
  const bool nup = flags & SSS_BWD_NU_GRAD_PAPER;
  if (!(flags & SSS_BWD_PROJECTION_ONLY)) {
    if (G.shift > 0) {
      if (l1) SSS_BWD_LAUNCH_N(true, true); else SSS_BWD_LAUNCH_N(true, false);
    } else {
      if (l1) SSS_BWD_LAUNCH_N(false, true); else SSS_BWD_LAUNCH_N(false, false);
    }
    count_launch((n_views + vg - 1) / vg);
    if ((st = check_launch("sss_render_bwd(raster)")) != SSS_OK) return st;
  }
#undef SSS_BWD_LAUNCH_N
#undef SSS_BWD_LAUNCH
  if (p->n == 0 || (flags & SSS_BWD_RASTER_ONLY)) return SSS_OK;
  return project_bwd_launch(*p, cams, n_views, g2d, *grad, 0, p->n, s, (flags & SSS_BWD_GRAD_ASSIGN) != 0);
  return SSS_OK;
}
