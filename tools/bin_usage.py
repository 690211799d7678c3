"""Dev tool: how much of each per-bin list the raster consumes (config 5).

For every tile: the bin list length (ranges), the furthest list position any
of its pixels composited (`last`), and whether every pixel of the tile
saturated (final_T < 1e-4: the forward then stops reading the list).  A tile
with a live pixel reads its whole bin list.  Prints one JSON line."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2503_10148_b200 as P
from sss_synth import make_scene

views = int(sys.argv[1]) if len(sys.argv) > 1 else 8
shift = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = int(sys.argv[3]) if len(sys.argv) > 3 else 5
P.load()
sc = make_scene(cfg, n_views=views)
cams = sc.cameras
params = P.Params(torch.from_numpy(sc.params).cuda(), sc.sh_degree)
pr = P.sss_project(params, cams)
bins = P.sss_bin_sort(pr, cams, bin_shift=shift)
fr = P.sss_render_fwd(pr, bins, cams)
torch.cuda.synchronize()
W, H = cams[0].width, cams[0].height
tx, ty = (W + 15) // 16, (H + 15) // 16
bx = (tx + (1 << shift) - 1) >> shift
rng = bins.ranges.cpu().numpy()  # [V][nb][2]
last = fr.last.cpu().numpy()     # [V][H][W]
fT = fr.final_T.cpu().numpy()
vis = (pr.rect[..., 0] <= pr.rect[..., 2]).sum(1).cpu().numpy()
out = {"views": views, "shift": shift, "n": sc.n, "n_vis_mean": float(vis.mean()),
       "instances_per_view": float(bins.totals.float().mean().item())}
cons, lens, sat = [], [], []
for v in range(views):
    Lp = np.full((ty * 16, tx * 16), -1, np.int64)
    Lp[:H, :W] = last[v]
    S = np.ones((ty * 16, tx * 16), bool)
    S[:H, :W] = fT[v] < 1e-4
    Lt = Lp.reshape(ty, 16, tx, 16).max(axis=(1, 3))
    St = S.reshape(ty, 16, tx, 16).all(axis=(1, 3))
    for j in range(ty):
        for i in range(tx):
            b = (j >> shift) * bx + (i >> shift)
            s0, s1 = rng[v, b]
            n = s1 - s0
            c = (Lt[j, i] - s0) if St[j, i] else n
            cons.append(c); lens.append(n); sat.append(St[j, i])
cons, lens, sat = np.array(cons), np.array(lens), np.array(sat)
# per bin (view-major): full length, max consumption over its tiles, all saturated
nbv = rng.shape[1]
bl = rng[..., 1] - rng[..., 0]
bcons = np.zeros((views, nbv), np.int64)
bsat = np.ones((views, nbv), bool)
k = 0
for v in range(views):
    for j in range(ty):
        for i in range(tx):
            b = (j >> shift) * bx + (i >> shift)
            bcons[v, b] = max(bcons[v, b], cons[k])
            bsat[v, b] &= sat[k]
            k += 1
pol = {}
for K in (4096, 8192, 16384, 32768):
    over = cons > K  # tiles that would read the tail (their bin is longer than K)
    pol[f"static_{K}"] = {"materialised_per_view": float(np.minimum(bl, K).sum() / views),
                          "tiles_in_tail": int(over.sum()),
                          "unsat_tiles_in_tail": int((over & ~sat).sum())}
adapt = np.where(bsat, np.minimum(bl, (1.5 * bcons).astype(np.int64) + 256), bl)
out["policy_adaptive_1p5"] = {"materialised_per_view": float(adapt.sum() / views),
                              "bins_complete_unsat": int((~bsat & (bl > 4096)).sum()),
                              "their_len_per_view": float(bl[~bsat & (bl > 4096)].sum() / views)}
out["policies"] = pol
out["full_per_view"] = float(bl.sum() / views)
# per bin: the furthest any of its tiles reads
out.update({
    "tiles": int(len(cons)), "frac_tiles_saturated": float(sat.mean()),
    "list_len_mean": float(lens.mean()), "list_len_max": int(lens.max()),
    "consumed_mean": float(cons.mean()), "consumed_p50": float(np.percentile(cons, 50)),
    "consumed_p90": float(np.percentile(cons, 90)), "consumed_p99": float(np.percentile(cons, 99)),
    "consumed_max": int(cons.max()),
    "consumed_sum_over_len_sum": float(cons.sum() / max(lens.sum(), 1)),
    "unsat_tiles_list_len_mean": float(lens[~sat].mean()) if (~sat).any() else 0.0,
})
print(json.dumps(out), flush=True)
