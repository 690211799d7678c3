"""Dev tool: how much the two 16x8 strips of a tile share their composited
entries (config 5).  For every tile: |L0|, |L1| (the forward's per-strip
lists) and |L0 u L1|.  A one-warp-per-tile backward would replay the union
once instead of each list once per strip.  Prints one JSON line."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2503_10148_b200 as P
from sss_synth import make_scene

views = int(sys.argv[1]) if len(sys.argv) > 1 else 4
P.load()
sc = make_scene(5, n_views=64)
cams = sc.cameras[:views]
params = P.Params(torch.from_numpy(sc.params).cuda(), sc.sh_degree)
pr = P.sss_project(params, cams)
bins = P.sss_bin_sort(pr, cams, bin_shift=2)
fr = P.sss_render_fwd(pr, bins, cams, out=P.Frame.empty(views, cams[0].height, cams[0].width, tile_cap=4096))
torch.cuda.synchronize()
tl = fr.tile_list.cpu().numpy()
tc = fr.tile_count.cpu().numpy()
s_sum = s_union = 0
for v in range(views):
    for t in range(tc.shape[1]):
        a = tl[v, t, 0, :tc[v, t, 0]]
        b = tl[v, t, 1, :tc[v, t, 1]]
        s_sum += len(a) + len(b)
        s_union += len(np.union1d(a, b))
print(json.dumps({"views": views, "strip_entries": int(s_sum), "tile_union_entries": int(s_union),
                  "union_over_sum": s_union / max(s_sum, 1), "overflow": int((tc > 4096).sum())}))
