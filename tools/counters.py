"""Dev tool: raster efficiency counters from a -DSSS_COUNTERS variant build."""
import argparse, ctypes as C, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2503_10148_b200 as P
from paper_2503_10148_b200 import _lib as L
from sss_synth import make_scene, make_targets
ap = argparse.ArgumentParser(); ap.add_argument("--config", type=int, default=3)
ap.add_argument("--views", type=int, default=None); ap.add_argument("--shift", type=int, default=0)
a = ap.parse_args()
sc = make_scene(a.config, n_views=a.views); cams = sc.cameras
lib = L.load()
params = P.Params(torch.from_numpy(sc.params).cuda(), sc.sh_degree)
tgt = torch.from_numpy(make_targets(sc)).cuda()
pr = P.sss_project(params, cams); bins = P.sss_bin_sort(pr, cams, bin_shift=a.shift)
names = ["batches", "warp_entries", "box_culled", "warp_entries_any", "pairs", "live_tests", "entries_loaded", "list_len"]
for nm, call in [("fwd", lambda: P.sss_render_fwd(pr, bins, cams)), ]:
    pass
h = (C.c_ulonglong * 16)()
lib.sss_dev_counters_fwd(h, 1); lib.sss_dev_counters_bwd(h, 1)
fr = P.sss_render_fwd(pr, bins, cams); torch.cuda.synchronize()
lib.sss_dev_counters_fwd(h, 1); f = {n: int(h[i]) for i, n in enumerate(names)}
P.sss_render_bwd(params, pr, bins, cams, fr, target=tgt); torch.cuda.synchronize()
lib.sss_dev_counters_bwd(h, 1); b = {n: int(h[i]) for i, n in enumerate(names)}
print(json.dumps({"config": a.config, "shift": a.shift, "fwd": f, "bwd": b,
                  "pairs_true": int(fr.n_contrib.sum().item()), "pixels": int(fr.n_contrib.numel())}))
