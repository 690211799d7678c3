"""Dev tool: adaptive bin caps over a training run (config 5, the bench's
TrainStep): per step, the step time and the bins whose forward needed more
than the bin kept (read the virtual tail: slow) -- the safety margin of the
cap policy (sss_bins.used; binsort.cu bin_cap_of).  Prints one JSON line."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2503_10148_b200 as P
from paper_2503_10148_b200.step import TrainStep
from sss_synth import make_scene, make_targets, sghmc_params_for

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
P.load()
sc = make_scene(5)
cams = sc.cameras
targets = torch.from_numpy(make_targets(sc, list(range(sc.n_views)))).cuda()
ts = TrainStep(torch.from_numpy(sc.params).cuda(), sc.sh_degree, cams, sghmc_params_for(sc), total_views=sc.n_views,
               bin_shift=2, views_per_batch=64, adaptive_bins=True)
ms, tails, kept = [], [], []
for k in range(steps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ts.step(targets)
    e1.record()
    torch.cuda.synchronize()
    if ts.overflowed():
        ts.grow()
    ms.append(round(e0.elapsed_time(e1), 2))
    b = ts.bins[0]
    used = ts.used[0] if ts.used is not None else b.used
    lens = b.ranges[..., 1] - b.ranges[..., 0]
    tails.append(int(((used > lens) & (used < (1 << 30))).sum().item()))
    kept.append(int(b.totals.sum().item()))
print(json.dumps({"lib": os.environ.get("SSS_LIB", "default"), "ms": ms, "tail_bins": tails,
                  "kept_per_step": kept}))
