// a3 — sss_render_fwd: signed front-to-back compositing (Eq. 7,
// PAPER.md:131-135, 1224-1228) of the 2D t kernels of Eq. 4
// (T2D = [1 + h/nu]^-(nu+2)/2).
//
// B200 design: one CTA per 16x16 tile and view (grid = tiles x V), one
// thread per pixel.  The tile's bin list is streamed through shared memory
// in batches of 256 entries; for bins coarser than a tile (bin_shift > 0) the
// batch is filtered by the component's tile rect and compacted in order
// (warp ballots) before the 48-byte records are staged.  Every pixel then
// walks the batch with broadcast shared-memory reads.  A pixel stops after
// the component that drives W below 1e-4 (R11); the CTA leaves as soon as no
// pixel is live (__syncthreads_count).  The hot loop is FP32-pipe bound
// (~8 ops per h test, ~12 more + 2 MUFU per composited pair).
#include "raster.cuh"

namespace sss {
namespace {

template <bool FILTER>
__global__ void __launch_bounds__(kRasterThreads) render_fwd_kernel(
    const float4* __restrict__ rec, const short4* __restrict__ rect, const int32_t* __restrict__ ids,
    const int32_t* __restrict__ ranges, RasterGeom G, float bg0, float bg1, float bg2,
    float* __restrict__ rgb, float* __restrict__ final_T, int32_t* __restrict__ n_contrib,
    int32_t* __restrict__ last) {
  __shared__ float4 sa[kBatch], sb[kBatch], sc[kBatch];
  __shared__ int32_t spos[kBatch];
  __shared__ int32_t wcnt[kRasterThreads / 32];
  const int v = blockIdx.y;
  const int tile = blockIdx.x;
  const int tx = tile % G.tiles_x, ty = tile / G.tiles_x;
  const int bin = (ty >> G.shift) * G.bins_x + (tx >> G.shift);
  const int32_t start = ranges[((int64_t)v * G.n_bins + bin) * 2 + 0];
  const int32_t end = ranges[((int64_t)v * G.n_bins + bin) * 2 + 1];
  int lx, ly;
  pixel_of(threadIdx.x, lx, ly);
  const int x = tx * kTile + lx, y = ty * kTile + ly;
  const bool inside = x < G.width && y < G.height;
  const float px = (float)x + 0.5f, py = (float)y + 0.5f;
  const int w = threadIdx.x >> 5, lane = lane_id();
  const unsigned lt = (1u << lane) - 1u;

  const int32_t* idv = ids + (int64_t)v * G.capacity;
  const float4* rv = rec + (int64_t)v * G.n * 3;
  const short4* rcv = rect + (int64_t)v * G.n;

  float W = 1.f, C0 = 0.f, C1 = 0.f, C2 = 0.f;
  int32_t cnt = 0, lastp = start;
  bool done = !inside;
  for (int32_t b0 = start; b0 < end; b0 += kBatch) {
    if (__syncthreads_count(!done) == 0) break;
    const int32_t pos = b0 + (int32_t)threadIdx.x;
    bool ok = pos < end;
    const int32_t id = ok ? idv[pos] : 0;
    int slot, nb;
    if (FILTER) {
      if (ok) {
        const short4 r = rcv[id];
        ok = tx >= r.x && tx <= r.z && ty >= r.y && ty <= r.w;
      }
      const unsigned bal = __ballot_sync(0xffffffffu, ok);
      if (lane == 0) wcnt[w] = __popc(bal);
      __syncthreads();
      int off = 0, tot = 0;
#pragma unroll
      for (int k = 0; k < kRasterThreads / 32; ++k) {
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
      spos[slot] = pos;
      sa[slot] = rv[(int64_t)id * 3 + 0];
      sb[slot] = rv[(int64_t)id * 3 + 1];
      sc[slot] = rv[(int64_t)id * 3 + 2];
    }
    __syncthreads();
    if (!done) {
      for (int j = 0; j < nb; ++j) {
        const float4 a = sa[j];
        const float4 b = sb[j];  // {C, hmax, o, inv_nu}
        const float h = h_f32(px, py, a, b.x);
        if (h <= b.y) {
          const float4 c = sc[j];  // {e, r, g, b}
          const float t = fmaxf(h, 0.f) * b.w;
          const float T = ex2_approx(c.x * log2_1p(t, b.w < (1.f / 32.f)));
          const float alpha = fminf(fmaxf(b.z * T, -kAlphaMax), kAlphaMax);
          const float aw = alpha * W;
          C0 = fmaf(c.y, aw, C0);
          C1 = fmaf(c.z, aw, C1);
          C2 = fmaf(c.w, aw, C2);
          W = fmaf(-alpha, W, W);
          ++cnt;
          lastp = spos[j] + 1;
          if (W < kWStop) {
            done = true;
            break;
          }
        }
      }
    }
  }
  if (inside) {
    const int64_t HW = (int64_t)G.width * G.height;
    const int64_t pix = (int64_t)y * G.width + x;
    float* o = rgb + (int64_t)v * 3 * HW + pix;
    o[0] = C0 + bg0 * W;
    o[HW] = C1 + bg1 * W;
    o[2 * HW] = C2 + bg2 * W;
    final_T[(int64_t)v * HW + pix] = W;
    n_contrib[(int64_t)v * HW + pix] = cnt;
    last[(int64_t)v * HW + pix] = lastp;
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
  return G.n_bins <= SSS_MAX_BINS && pr->n_views == n_views && bins->n_views == n_views;
}

}  // namespace sss

using namespace sss;

extern "C" sss_status sss_render_fwd(const sss_projected* pr, const sss_bins* bins, const sss_camera* cams,
                                     int32_t n_views, const float* bg, sss_frame* out, void* stream) {
  sss_status st;
  if (!pr || !bins || !out || !bg) { set_error("sss_render_fwd: null argument"); return SSS_ERR_ARG; }
  if ((st = validate_cams(cams, n_views, "sss_render_fwd")) != SSS_OK) return st;
  RasterGeom G;
  if (!raster_geom(pr, bins, cams, n_views, G)) { set_error("sss_render_fwd: geometry mismatch"); return SSS_ERR_SHAPE; }
  if (!out->rgb || !out->final_T || !out->n_contrib || !out->last || !bins->ranges ||
      (pr->n > 0 && (!pr->rec || !pr->rect)) || (bins->capacity > 0 && !bins->ids)) {
    set_error("sss_render_fwd: null buffer");
    return SSS_ERR_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const dim3 grid(G.tiles_x * G.tiles_y, n_views);
  if (G.shift > 0)
    render_fwd_kernel<true><<<grid, kRasterThreads, 0, s>>>((const float4*)pr->rec, (const short4*)pr->rect,
                                                            bins->ids, bins->ranges, G, bg[0], bg[1], bg[2],
                                                            out->rgb, out->final_T, out->n_contrib, out->last);
  else
    render_fwd_kernel<false><<<grid, kRasterThreads, 0, s>>>((const float4*)pr->rec, (const short4*)pr->rect,
                                                             bins->ids, bins->ranges, G, bg[0], bg[1], bg[2],
                                                             out->rgb, out->final_T, out->n_contrib, out->last);
  count_launch();
  return check_launch("sss_render_fwd");
}
