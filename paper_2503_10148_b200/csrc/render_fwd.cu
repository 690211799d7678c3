// a3 — sss_render_fwd: signed front-to-back compositing (Eq. 7,
// PAPER.md:131-135, 1224-1228) of the 2D t kernels of Eq. 4
// (T2D = [1 + h/nu]^-(nu+2)/2).
//
// B200 design: one CTA per 16x16 tile and view (grid = tiles x V), 64
// threads with kPX = 4 horizontally adjacent pixels each (a warp owns a
// 16x8 strip), so per-entry shared-memory loads and loop overhead are shared
// by four pixels.  The tile's bin list is streamed through shared memory in
// batches of 64 entries; for bins coarser than a tile (bin_shift > 0) the
// batch is filtered by the component's tile rect and compacted in order
// (warp ballots) before the 48-byte records are staged.  Each warp walks the
// batch with broadcast shared-memory reads; when any of its pixels is hit the
// four pixel chains run predicated (branch-free).  A pixel stops after the
// component that drives W below 1e-4 (R11); a warp leaves the batch when all
// its pixels stopped, the CTA when no pixel is live.  The hot loop is
// FP32-issue bound (~8 ops per h test, ~17 more + 2 MUFU per composited
// pair).  Each warp records the entries its 16x8 strip composited (bit masks
// per batch, appended in order) for the backward's replay.  (Measured and
// rejected: per-warp bounding-box or exact ellipse-strip culling — the warps
// of a tile then drift apart at the batch barrier — register prefetching of
// the next batch, and per-warp batches staged by cp.async without the CTA
// barrier, +5%: each warp then gathers every record itself; round 2: a
// conservative ellipse-vs-strip box test at staging with per-strip staging
// arrays, so each warp walks only entries that can reach its strip: +5% at
// config 5 -- the duplicated staging and the 64 registers it needs cost more
// than the culled entries save.)
#include "raster.cuh"

namespace sss {
namespace {

struct PixF2 {  // forward colour state of a horizontally adjacent pixel pair
  float2 W, C0, C1, C2;
};

// One pair of Eq. 7 for both pixels of a pair, predicated per pixel on `inc`
// (a = 0 leaves C and W bit-unchanged: C + c*0 = C, W - 0*W = W), so a warp
// runs its pixels' chains branch-free.  GENERAL handles the two rare
// warp-uniform cases: nu > 32 (accurate log1p, see log2_1p), the Gaussian
// kernel of the ablation variant (inv_nu = 0 in the record) and |o| > 0.989,
// where the +-0.99 clamp (R10) can bind (T <= 1 for h >= 0, so |o| <= 0.989
// leaves |o T| < 0.99 even for an h rounded slightly below 0).
template <bool GENERAL>
__device__ __forceinline__ void composite2(PixF2& p, float2 h, float4 b, float4 c, bool inc0, bool inc1) {
  const float2 t = mul2(h, bc2(b.w));
  float2 lg;
  float2 e;
  if (GENERAL && b.w == 0.f) {  // Gaussian variant: T = exp(-h/2) = 2^(kGaussExp2 h)
    e = mul2(h, bc2(kGaussExp2));
  } else {
    if (GENERAL && b.w < (1.f / 32.f)) {
      lg = make_float2(log2_1p(t.x, true), log2_1p(t.y, true));
    } else {
      const float2 opt = add2(t, bc2(1.f));
      lg = make_float2(lg2_approx(opt.x), lg2_approx(opt.y));
    }
    e = mul2(lg, bc2(c.x));
  }
  float2 araw = mul2(make_float2(ex2_approx(e.x), ex2_approx(e.y)), bc2(b.z));
  if (GENERAL) {
    araw.x = fminf(fmaxf(araw.x, -kAlphaMax), kAlphaMax);
    araw.y = fminf(fmaxf(araw.y, -kAlphaMax), kAlphaMax);
  }
  float2 alpha;
  alpha.x = inc0 ? araw.x : 0.f;
  alpha.y = inc1 ? araw.y : 0.f;
  const float2 aw = mul2(alpha, p.W);
  p.C0 = fma2(bc2(c.y), aw, p.C0);
  p.C1 = fma2(bc2(c.z), aw, p.C1);
  p.C2 = fma2(bc2(c.w), aw, p.C2);
  p.W = fma2(make_float2(-alpha.x, -alpha.y), p.W, p.W);
}

__device__ __forceinline__ float& lane_of(float2& v, int k) { return (k & 1) ? v.y : v.x; }

template <bool FILTER, bool COUNT, bool REC>
__global__ void __launch_bounds__(kRasterThreads, kFwdMinBlocks) render_fwd_kernel(
    const float4* __restrict__ rec, const float4* __restrict__ col, const short4* __restrict__ rect,
    const int32_t* __restrict__ ids,
    const int32_t* __restrict__ ranges, RasterGeom G, float bg0, float bg1, float bg2,
    float* __restrict__ rgb, float* __restrict__ final_T, int32_t* __restrict__ n_contrib,
    int32_t* __restrict__ last, int32_t* __restrict__ tile_list, int32_t* __restrict__ tile_count,
    int32_t tile_cap) {
  static_assert(kBatch == kRasterThreads, "one staged entry per thread");
#ifndef SSS_FWD_SMEM_PTRS
#define SSS_FWD_SMEM_PTRS 1
#endif
#ifndef SSS_FWD_AOS
#define SSS_FWD_AOS 1
#endif
#if SSS_FWD_AOS
  // one 64-byte slot per staged entry: the composite loop addresses all four
  // fields from one base (immediate offsets) instead of four array bases
  struct alignas(16) StageSlot { float4 a, b, c; int32_t pos, pad0, pad1, pad2; };
  __shared__ StageSlot stg[kBatch];
#define SA(j) stg[j].a
#define SB(j) stg[j].b
#define SC(j) stg[j].c
#define SPOS(j) stg[j].pos
#else
  __shared__ float4 sa[kBatch], sb[kBatch], sc[kBatch];
  __shared__ int32_t spos[kBatch];
#define SA(j) sa[j]
#define SB(j) sb[j]
#define SC(j) sc[j]
#define SPOS(j) spos[j]
#endif
  __shared__ int32_t wcnt[kRasterWarps];
  const int v = blockIdx.y;
  const int tile = blockIdx.x;
  const int tx = tile % G.tiles_x, ty = tile / G.tiles_x;
  const int bin = (ty >> G.shift) * G.bins_x + (tx >> G.shift);
  const BinList BL = bin_list(G, ids, ranges, v, bin);
  const int32_t start = BL.start, end = BL.end;
  int lx, ly, sx, sy;
  pixels_of(threadIdx.x, lx, ly, sx, sy);
  const int x0 = tx * kTile + lx, y = ty * kTile + ly;
  const float py = (float)y + 0.5f;
  const int w = threadIdx.x >> 5, lane = lane_id();
  const unsigned lt = (1u << lane) - 1u;

  const float4* rv = rec + (int64_t)v * G.n * 2;  // geometry records (2 x float4)
  const float4* cv = col + (int64_t)v * G.n;      // colour records
  const short4* rcv = rect + (int64_t)v * G.n;
  const uint16_t* tmv = G.tmask ? G.tmask + (int64_t)v * G.capacity : nullptr;

  if (threadIdx.x == 0) SSS_COUNT(7, end - start);
  PixF2 p[kPairs];
  float2 px[kPairs];
  int32_t cnt[kPX], lastc[kPX];
#pragma unroll
  for (int k = 0; k < kPX; ++k) {
    const bool inside = x0 + k < G.width && y < G.height;
    // a pixel is live while W >= 1e-4 (R11); pixels outside the image start
    // with W = 0 and so are never composited (their outputs are unused)
    PixF2& pp = p[k >> 1];
    lane_of(pp.W, k) = inside ? 1.f : 0.f;
    lane_of(pp.C0, k) = lane_of(pp.C1, k) = lane_of(pp.C2, k) = 0.f;
    // a stopped (or outside) pixel's coordinate is NaN: its h is NaN and
    // fails h <= hmax, so the inclusion test needs no liveness term
    lane_of(px[k >> 1], k) = inside ? (float)(x0 + k) + 0.5f : __int_as_float(0x7fffffff);
    cnt[k] = 0;
    lastc[k] = start;
  }
  auto all_done = [&]() {
    bool d = true;
#pragma unroll
    for (int k = 0; k < kPX; ++k) d = d && !(lane_of(p[k >> 1].W, k) >= kWStop);
    return d;
  };
  // REC: this warp's list of the entries some pixel of its 16x8 strip
  // composited, appended after each batch from warp-uniform bit masks
  const int64_t lslot = ((int64_t)v * G.tiles_x * G.tiles_y + tile) * kRasterWarps + w;
  // the warp's list base lives in shared memory: recomputing the 64-bit
  // address from the block indices at every batch's write-out cost ~40
  // instructions (the registers are all taken by the pixel state)
  __shared__ int32_t* s_tl[kRasterWarps];
  if (REC && lane == 0) s_tl[w] = tile_list + lslot * tile_cap;
#if SSS_FWD_SMEM_PTRS
  // the same for the staging's per-view bases (ids, tail, records, masks)
  __shared__ const void* s_ptr[5];
  if (threadIdx.x == 0) {
    s_ptr[0] = BL.ids;
    s_ptr[1] = BL.tail ? BL.tail + BL.tail0 - BL.mend : nullptr;  // index by the list position
    s_ptr[2] = rv;
    s_ptr[3] = cv;
    s_ptr[4] = tmv;
  }
#endif
  int32_t n_rec = 0;
  for (int32_t b0 = start; b0 < end; b0 += kBatch) {
    if (__syncthreads_count(!all_done()) == 0) break;
    if (threadIdx.x == 0) SSS_COUNT(0, 1);
    static_assert(kBatch == 64, "one 64-bit composited mask per batch");
    unsigned long long cm = 0ull;  // REC: this warp's composited entries (warp-uniform bits)
    const int32_t pos = b0 + (int32_t)threadIdx.x;
    bool ok = (int)threadIdx.x < kBatch && pos < end;
#if SSS_FWD_SMEM_PTRS
    const int32_t id = !ok ? 0 : pos < BL.mend ? __ldg(static_cast<const int32_t*>(s_ptr[0]) + pos)
                                               : __ldg(static_cast<const int32_t*>(s_ptr[1]) + pos);
    const uint16_t* tmv_s = static_cast<const uint16_t*>(s_ptr[4]);
#else
    const int32_t id = ok ? BL.id(pos) : 0;
    const uint16_t* tmv_s = tmv;
#endif
    int slot, nb;
    // the truncated list's tail is the depth-sorted visible set: always filtered
    if (FILTER || end > BL.mend) {
      if (ok && (FILTER || pos >= BL.mend)) ok = entry_in_tile(G, tmv_s, pos, BL.mend, id, rcv, tx, ty);
      const unsigned bal = __ballot_sync(0xffffffffu, ok);
      if (lane == 0) wcnt[w] = __popc(bal);
      __syncthreads();
      int off = 0, tot = 0;
#pragma unroll
      for (int k = 0; k < kRasterWarps; ++k) {
        const int c = wcnt[k];
        off += k < w ? c : 0;
        tot += c;
      }
      slot = off + __popc(bal & lt);
      nb = tot;
    } else {
      slot = threadIdx.x;
      nb = min(kBatch, end - b0);
    }
    if (ok) {
#if SSS_FWD_SMEM_PTRS
      const float4* rvs = static_cast<const float4*>(s_ptr[2]);
      const float4* cvs = static_cast<const float4*>(s_ptr[3]);
#else
      const float4* rvs = rv;
      const float4* cvs = cv;
#endif
      SPOS(slot) = pos;
      SA(slot) = rvs[(int64_t)id * 2 + 0];
      SB(slot) = rvs[(int64_t)id * 2 + 1];
      SC(slot) = cvs[id];
    }
    __syncthreads();
    if (threadIdx.x == 0) SSS_COUNT(6, nb);
    const int nb_w = __all_sync(0xffffffffu, all_done()) ? 0 : nb;  // warp already finished
    for (int j = 0; j < nb_w; ++j) {
      if (lane == 0) SSS_COUNT(1, 1);
      const float4 a = SA(j);
      const float4 b = SB(j);  // {C, hmax, o, inv_nu}
      const float dy = __fsub_rn(py, a.y);
      const float bdy = __fmul_rn(a.w, dy);
      const float cdy2 = __fmul_rn(__fmul_rn(b.x, dy), dy);
      float2 h[kPairs];
      bool inc[kPX];
      bool any = false;
#pragma unroll
      for (int k = 0; k < kPairs; ++k) {
        float2 dx;
        h[k] = h_f32_pair(px[k], a.x, a.z, bdy, cdy2, dx);
        inc[2 * k] = h[k].x <= b.y;  // false for stopped pixels (px NaN)
        inc[2 * k + 1] = h[k].y <= b.y;
        any = any || inc[2 * k] || inc[2 * k + 1];
      }
#ifdef SSS_COUNTERS
      {
        const unsigned ba = __ballot_sync(0xffffffffu, any);
        int ninc = 0, nlive = 0;
        for (int k = 0; k < kPX; ++k) {
          ninc += __popc(__ballot_sync(0xffffffffu, inc[k]));
          nlive += __popc(__ballot_sync(0xffffffffu, lane_of(p[k >> 1].W, k) >= kWStop));
        }
        if (lane == 0) { SSS_COUNT(3, ba != 0); SSS_COUNT(4, ninc); SSS_COUNT(5, nlive); }
      }
#endif
      if (__any_sync(0xffffffffu, any)) {  // warp-uniform; pixels predicated
        if (REC) cm |= 1ull << j;
        const float4 c = SC(j);  // {e, r, g, b}
        const int32_t pj1 = SPOS(j) + 1;
        if (fabsf(b.z) > 0.989f || b.w < (1.f / 32.f)) {  // warp-uniform, rare
#pragma unroll
          for (int k = 0; k < kPairs; ++k) composite2<true>(p[k], h[k], b, c, inc[2 * k], inc[2 * k + 1]);
        } else {
#pragma unroll
          for (int k = 0; k < kPairs; ++k) composite2<false>(p[k], h[k], b, c, inc[2 * k], inc[2 * k + 1]);
        }
#pragma unroll
        for (int k = 0; k < kPX; ++k) {
          lastc[k] = inc[k] ? pj1 : lastc[k];
          if (COUNT) cnt[k] += inc[k] ? 1 : 0;
          // R11: the pixel stops after the component that drives W below 1e-4
          float& xk = lane_of(px[k >> 1], k);
          xk = lane_of(p[k >> 1].W, k) >= kWStop ? xk : __int_as_float(0x7fffffff);
        }
      }
      if ((j & 7) == 7 && __all_sync(0xffffffffu, all_done())) break;
    }
    if (REC) {  // spos is rewritten only after the next top barrier
#pragma unroll
      for (int q = 0; q < kBatch / 32; ++q) {
        const unsigned cq = (unsigned)(cm >> (32 * q));
        const int slot = n_rec + __popc(cq & lt);
        if (((cq >> lane) & 1u) && slot < tile_cap) s_tl[w][slot] = SPOS(q * 32 + lane);
        n_rec += __popc(cq);
      }
    }
  }
  if (REC && lane == 0) tile_count[lslot] = n_rec;
  if (G.used) {  // adaptive truncation: how much of the bin list this tile needed
    const bool done = __syncthreads_and(all_done());
    int32_t mx = lastc[0];
#pragma unroll
    for (int k = 1; k < kPX; ++k) mx = max(mx, lastc[k]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) atomicMax(&G.used[(int64_t)v * G.n_bins + bin], done ? mx - start : (1 << 30));
  }
  const int64_t HW = (int64_t)G.width * G.height;
#pragma unroll
  for (int k = 0; k < kPX; ++k) {
    if (!(x0 + k < G.width && y < G.height)) continue;
    const int64_t pix = (int64_t)y * G.width + x0 + k;
    float* o = rgb + (int64_t)v * 3 * HW + pix;
    PixF2& pp = p[k >> 1];
    const float W = lane_of(pp.W, k);
    o[0] = lane_of(pp.C0, k) + bg0 * W;
    o[HW] = lane_of(pp.C1, k) + bg1 * W;
    o[2 * HW] = lane_of(pp.C2, k) + bg2 * W;
    final_T[(int64_t)v * HW + pix] = W;
    if (COUNT) n_contrib[(int64_t)v * HW + pix] = cnt[k];
    last[(int64_t)v * HW + pix] = lastc[k];
  }
}

}  // namespace

bool raster_geom(const sss_projected* pr, const sss_bins* bins, const sss_camera* cams, int n_views,
                 RasterGeom& G) {
  G.width = cams[0].width;
  G.height = cams[0].height;
  G.tiles_x = div_up(G.width, kTile);
  G.tiles_y = div_up(G.height, kTile);
  G.shift = bins->bin_shift;
  G.bins_x = div_up(G.tiles_x, 1 << G.shift);
  G.n_bins = G.bins_x * div_up(G.tiles_y, 1 << G.shift);
  G.n = pr->n;
  G.capacity = bins->capacity;
  const bool trunc = bins->max_per_bin > 0 || bins->used;
  G.sorted = trunc ? bins->sorted : nullptr;
  G.n_vis = trunc ? bins->n_vis : nullptr;
  G.resume = trunc ? bins->resume : nullptr;
  G.used = bins->used;
  G.tmask = (bins->tmask && bins->bin_shift <= 2) ? bins->tmask : nullptr;
  if (trunc && (!bins->sorted || !bins->n_vis || !bins->resume)) return false;
  return G.n_bins <= SSS_MAX_BINS && pr->n_views == n_views && bins->n_views == n_views;
}

}  // namespace sss

using namespace sss;

SSS_COUNTER_ACCESSOR(sss_dev_counters_fwd)

extern "C" sss_status sss_render_fwd(const sss_projected* pr, const sss_bins* bins, const sss_camera* cams,
                                     int32_t n_views, const float* bg, sss_frame* out, void* stream) {
  sss_status st;
  if (!pr || !bins || !out || !bg) { set_error("sss_render_fwd: null argument"); return SSS_ERR_ARG; }
  if ((st = validate_cams(cams, n_views, "sss_render_fwd")) != SSS_OK) return st;
  RasterGeom G;
  if (!raster_geom(pr, bins, cams, n_views, G)) { set_error("sss_render_fwd: geometry mismatch"); return SSS_ERR_SHAPE; }
  if (!out->rgb || !out->final_T || !out->last || !bins->ranges ||
      (pr->n > 0 && (!pr->rec || !pr->col || !pr->rect)) || (bins->capacity > 0 && !bins->ids)) {
    set_error("sss_render_fwd: null buffer");
    return SSS_ERR_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const dim3 grid(G.tiles_x * G.tiles_y, n_views);
#define SSS_FWD_LAUNCH(F, N, R)                                                                         \
  render_fwd_kernel<F, N, R><<<grid, kRasterThreads, 0, s>>>(                                             \
      (const float4*)pr->rec, (const float4*)pr->col, (const short4*)pr->rect, bins->ids, bins->ranges, G,  \
      bg[0], bg[1], bg[2],                                                                                 \
      out->rgb, out->final_T, out->n_contrib, out->last, out->tile_list, out->tile_count, out->tile_cap)
#define SSS_FWD_LAUNCH_R(F, N)                 \
  do {                                         \
    if (recl) SSS_FWD_LAUNCH(F, N, true);      \
    else SSS_FWD_LAUNCH(F, N, false);          \
  } while (0)
  const bool cnt = out->n_contrib != nullptr;
  const bool recl = out->tile_list != nullptr && out->tile_count != nullptr && out->tile_cap > 0;
  if (G.shift > 0) {
    if (cnt) SSS_FWD_LAUNCH_R(true, true); else SSS_FWD_LAUNCH_R(true, false);
  } else {
    if (cnt) SSS_FWD_LAUNCH_R(false, true); else SSS_FWD_LAUNCH_R(false, false);
  }
#undef SSS_FWD_LAUNCH_R
#undef SSS_FWD_LAUNCH
  count_launch();
  return check_launch("sss_render_fwd");
}
