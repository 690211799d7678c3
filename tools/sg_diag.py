import sys, os, json
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
import paper_2503_10148_b200 as sss
from oracle import oracle as orc
from sss_synth import make_optimizer_state, make_scene, sghmc_params_for
from test_gpu_parity import _hp32
sss.load()
sc = make_scene(5)
r, m, v = make_optimizer_state(sc, seed=3)
rng = np.random.default_rng(5)
grad = (rng.normal(size=sc.params.shape) * 1e-2).astype(np.float32)
hp = _hp32(sghmc_params_for(sc, step=2, seed=99))
print(hp)
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
params = sss.Params(dev(sc.params), 3)
mm, vv, rr = sss.Params(dev(m), 3), sss.Params(dev(v), 3), dev(r)
sss.sss_sghmc_step(params, sss.Params(dev(grad), 3), mm, vv, rr, hp)
torch.cuda.synchronize()
p_ref, m_ref, v_ref, r_ref = orc.sghmc_step(sc.params, 3, grad, m, v, r, hp)
got = params.planes.cpu().numpy().astype(np.float64)
ulp = np.spacing(np.abs(p_ref).astype(np.float32)).astype(np.float64)
tol = ulp + 1e-5 * np.abs(p_ref - sc.params) + 1e-30
bad = np.abs(got - p_ref) > tol
print("bad", int(bad.sum()), "per plane", [int(x) for x in bad.sum(1)])
ii = np.argwhere(bad)[:10]
for pl, j in ii:
    print(pl, j, got[pl, j], p_ref[pl, j], sc.params[pl, j], (got[pl,j]-p_ref[pl,j])/ulp[pl,j], "o", sc.params[0:3, j] if pl < 3 else "")
