"""Dev tool: adaptive caps at config 5 -- how many bins keep their complete
list (a pixel of theirs never stops), how many instances those hold, and
what share of the chunks the scatter cannot skip."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2503_10148_b200 as P
from paper_2503_10148_b200 import api as A
from sss_synth import make_scene

P.load()
sc = make_scene(5, n_views=64)
cams = sc.cameras[:8]
V = len(cams)
params = P.Params(torch.from_numpy(sc.params).cuda(), sc.sh_degree)
pr = P.sss_project(params, cams)
full = P.sss_bin_sort(pr, cams, bin_shift=2)
b = A.Bins.empty(V, full.ranges.shape[1], full.capacity, 2, False, "cuda", 0, params.n, adaptive=True)
P.sss_bin_sort(pr, cams, bin_shift=2, out=b)
P.sss_render_fwd(pr, b, cams, out=P.Frame.empty(V, cams[0].height, cams[0].width))
P.sss_bin_sort(pr, cams, bin_shift=2, out=b)  # steady-state caps from the warm forward
P.sss_render_fwd(pr, b, cams, out=P.Frame.empty(V, cams[0].height, cams[0].width))
torch.cuda.synchronize()
used = b.used.clone()  # this forward's consumption (bin_sort resets it)
lens_full = (full.ranges[..., 1] - full.ranges[..., 0]).long()
kept = (b.ranges[..., 1] - b.ranges[..., 0]).long()
complete = used >= (1 << 30)
print(json.dumps({"bins_per_view": int(used.shape[1]), "complete_bins_per_view": float(complete.sum() / V),
                  "kept_per_view": float(kept.sum() / V), "kept_in_complete_per_view": float(kept[complete].sum() / V),
                  "full_len_complete_mean": float(lens_full[complete].float().mean()) if complete.any() else 0,
                  "n_vis_mean": float(b.n_vis.float().mean())}))
