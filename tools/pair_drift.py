"""Dev tool: composited pairs per step along the bench's training trajectory
(config 5), to tell a kernel change from training-state drift."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2503_10148_b200 as P
from paper_2503_10148_b200.step import TrainStep
from sss_synth import make_scene, make_targets, sghmc_params_for

views = int(sys.argv[1]) if len(sys.argv) > 1 else 16
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
P.load()
sc = make_scene(5, n_views=views)
cams = sc.cameras
targets = torch.from_numpy(make_targets(sc)).cuda()
ts = TrainStep(torch.from_numpy(sc.params).cuda(), sc.sh_degree, cams, sghmc_params_for(sc),
               total_views=len(cams), bin_shift=2, views_per_batch=len(cams))
out = []
for k in range(steps + 1):
    ts.stats = {"pairs": torch.zeros((), dtype=torch.int64, device="cuda"),
                "instances": torch.zeros((), dtype=torch.int64, device="cuda")}
    loss = ts.forward_backward(targets)
    out.append((int(ts.stats["pairs"].item()), int(ts.stats["instances"].item())))
    ts.stats = None
    if k < steps:
        ts.step(targets)
torch.cuda.synchronize()
print(json.dumps({"lib": os.environ.get("SSS_LIB", "default"), "pairs": [p for p, _ in out],
                  "instances": [i for _, i in out]}))
