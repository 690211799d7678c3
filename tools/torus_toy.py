"""NEXT-4 experiment: torus scooping toy (Fig. 2) — final L1 of 1+/1- vs 2+
vs 5+ component fits over seeds (GPU, the product's training loop)."""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_10148_b200 import toy

ap = argparse.ArgumentParser()
ap.add_argument("--seeds", type=int, default=10)
ap.add_argument("--iters", type=int, default=1000)
ap.add_argument("--lr-mu", type=float, default=0.1)
ap.add_argument("--lr", type=float, default=0.1)
a = ap.parse_args()
res = []
for seed in range(a.seeds):
    for (p, n) in [(1, 1), (2, 0), (5, 0)]:
        res.append(toy.fit_torus(p, n, seed=seed, iters=a.iters, lr_mu=a.lr_mu, lr=a.lr))
s = toy.summarize(res)
wins = sum(1 for k in range(a.seeds) if res[3 * k].final_loss < res[3 * k + 1].final_loss)
wins5 = sum(1 for k in range(a.seeds) if res[3 * k + 2].final_loss < res[3 * k + 1].final_loss)
print(json.dumps({"iters": a.iters, "lr_mu": a.lr_mu, "lr": a.lr, "summary": s,
                  "pm_beats_2pos": wins, "5pos_beats_2pos": wins5, "seeds": a.seeds,
                  "ms_per_iter": res[0].ms_per_iter}))
