"""Dev tool: distribution of tile-rect sizes (config 5, a few views) and the
share of bin-list instances whose component rect exceeds 8x8 tiles."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2503_10148_b200 as P
from sss_synth import make_scene

P.load()
sc = make_scene(5, n_views=64)
cams = sc.cameras[:4]
params = P.Params(torch.from_numpy(sc.params).cuda(), sc.sh_degree)
pr = P.sss_project(params, cams)
r = pr.rect.view(len(cams), -1, 4).long()
w = r[..., 2] - r[..., 0] + 1
h = r[..., 3] - r[..., 1] + 1
vis = (w > 0) & (h > 0)
inst = (w * h * vis).sum().item()
big = ((w > 8) | (h > 8)) & vis
print(json.dumps({"visible": int(vis.sum()), "big_rects": int(big.sum()), "big_share": float(big.sum() / vis.sum()),
                  "instances_tiles": int(inst), "big_tiles_share": float((w * h * big).sum().item() / inst),
                  "w_hist": torch.bincount(w[vis].clamp(max=20)).tolist()}))
