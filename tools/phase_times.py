"""Per-phase CUDA-event timing of the hot path on one config (dev tool)."""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2503_10148_b200 as P
from paper_2503_10148_b200 import api as A
from sss_synth import make_scene, make_targets

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--views", type=int, default=None)
ap.add_argument("--shift", type=int, default=0)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--no-count", action="store_true", help="forward without the n_contrib diagnostic")
ap.add_argument("--tile-cap", type=int, default=None)
ap.add_argument("--adaptive", action="store_true", help="adaptive bin caps (sss_bins.used), after one warm round")
ap.add_argument("--tmask", type=int, default=1, help="per-entry tile masks (sss_bins.tmask)")
a = ap.parse_args()
sc = make_scene(a.config, n_views=a.views)
cams = sc.cameras
V = len(cams)
params = P.Params(torch.from_numpy(sc.params).cuda(), sc.sh_degree)
tgt = torch.from_numpy(make_targets(sc)).cuda()
pr = P.sss_project(params, cams)
bins = P.sss_bin_sort(pr, cams, bin_shift=a.shift)
if a.adaptive:
    bins = A.Bins.empty(V, bins.ranges.shape[1], bins.capacity, a.shift, False, "cuda", 0, params.n, adaptive=True,
                        tile_masks=bool(a.tmask) and 1 <= a.shift <= 2)
    P.sss_bin_sort(pr, cams, bin_shift=a.shift, out=bins)
    P.sss_render_fwd(pr, bins, cams, out=P.Frame.empty(V, cams[0].height, cams[0].width))
    used0 = bins.used.clone()  # every timed bin_sort starts from the warm round's consumption
fr = P.sss_render_fwd(pr, bins, cams, out=P.Frame.empty(V, cams[0].height, cams[0].width, **({} if a.tile_cap is None else {"tile_cap": a.tile_cap})))
fr_nc = P.Frame(fr.rgb, fr.final_T, None, fr.last, fr.tile_list, fr.tile_count)
ws_g2d = torch.zeros(A.render_bwd_workspace_bytes(params.n, V), dtype=torch.uint8, device="cuda")
ws_bin = torch.empty(A.bin_sort_workspace_bytes(params.n, cams, a.shift), dtype=torch.uint8, device="cuda")
grad = P.Params.zeros_like(params)
loss = torch.zeros(1, device="cuda")
cc = A.cameras_c(cams)
phases = {
  "project": lambda: P.sss_project(params, cams, out=pr, cams_c=cc),
  "bin_sort": lambda: (bins.used.copy_(used0) if a.adaptive else None,
                       P.sss_bin_sort(pr, cams, bin_shift=a.shift, ws=ws_bin, out=bins, cams_c=cc)),
  "render_fwd": lambda: P.sss_render_fwd(pr, bins, cams, out=fr_nc if a.no_count else fr, cams_c=cc),
  "render_bwd": lambda: P.sss_render_bwd(params, pr, bins, cams, fr, target=tgt, grad=grad, loss=loss, ws=ws_g2d, cams_c=cc),
}
res = {}
for name, f in phases.items():
    f(); torch.cuda.synchronize()
    ts = []
    for _ in range(a.reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    res[name] = min(ts)
tot = bins.totals.cpu().numpy()
tail_bins = complete_bins = 0
if a.adaptive:  # bins whose tiles needed more than the bin kept (read the tail)
    bins.used.copy_(used0)
    P.sss_bin_sort(pr, cams, bin_shift=a.shift, out=bins)
    P.sss_render_fwd(pr, bins, cams, out=fr)
    torch.cuda.synchronize()
    lens = bins.ranges[..., 1] - bins.ranges[..., 0]
    complete_bins = int((bins.used >= (1 << 30)).sum().item())  # some pixel never stops: complete list
    tail_bins = int(((bins.used > lens) & (bins.used < (1 << 30))).sum().item())  # read the virtual tail
nc = fr.n_contrib.float()
tcs = fr.tile_count.float() if fr.tile_count is not None else torch.zeros(1, device="cuda")
cap = fr.tile_list.shape[-1] if fr.tile_list is not None else 0
out = dict(config=a.config, views=V, shift=a.shift, ms=res, total_ms=sum(res.values()),
           tile_count=dict(mean=float(tcs.mean()), max=float(tcs.max()), cap=int(cap),
                           over=float((tcs > cap).float().mean())),
           instances_per_view=float(tot.mean()), capacity=bins.capacity, tail_bins=tail_bins, complete_bins=complete_bins,
           pairs_per_view=float(nc.sum().item()/V), mean_contrib=float(nc.mean().item()),
           mpix_per_s=V*cams[0].width*cams[0].height/sum(res.values())/1e3)
print(json.dumps(out))
