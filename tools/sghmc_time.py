"""Dev tool: CUDA-event time of sss_sghmc_step on config-5-sized state."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2503_10148_b200 as P
from sss_synth import SGHMCParams

n, deg = 3_000_000, 3
planes = P.n_planes(deg)
g = torch.Generator(device="cuda").manual_seed(0)
mk = lambda: P.Params(torch.randn((planes, n), device="cuda", generator=g) * 0.1, deg)  # noqa: E731
p, gr, m, v = mk(), mk(), mk(), mk()
v.planes.abs_()
r = torch.zeros((3, n), device="cuda")
hp = SGHMCParams(lr=1e-3, friction=0.1, noise=1e-3, g_adam=True, lr_scale=1e-3, lr_rot=1e-3, lr_nu=1e-3,
                 lr_opacity=1e-3, lr_sh=1e-3, seed=1)
ts = []
for k in range(1, 25):
    hp.step = k
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    P.sss_sghmc_step(p, gr, m, v, r, hp)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = sorted(ts[4:])[len(ts[4:]) // 2]
gb = n * 4 * (planes * 7 + 6) / 1e9
print(json.dumps({"lib": os.environ.get("SSS_LIB", "default"), "ms": round(ms, 4), "GB": round(gb, 3),
                  "GBps": round(gb / ms * 1e3, 1)}))
