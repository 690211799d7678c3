"""Dev tool: of the bin-list entries a forward tile visits (rect test passed,
up to the batch where all its pixels stopped), how many have an ellipse
(h <= hmax) that misses the whole tile / one of its 16x8 strips?  Exact
continuous test in numpy float64 (the kernel would use a conservative fp32
version).  Prints one JSON line."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2503_10148_b200 as P
from sss_synth import make_scene

views = int(sys.argv[1]) if len(sys.argv) > 1 else 2
P.load()
sc = make_scene(5, n_views=64)
cams = sc.cameras[:views]
params = P.Params(torch.from_numpy(sc.params).cuda(), sc.sh_degree)
pr = P.sss_project(params, cams)
bins = P.sss_bin_sort(pr, cams, bin_shift=2)
fr = P.sss_render_fwd(pr, bins, cams)
torch.cuda.synchronize()
W, H = cams[0].width, cams[0].height
tx_n, ty_n = (W + 15) // 16, (H + 15) // 16
bx_n = (tx_n + 3) // 4


def box_min(mx, my, A, B2, C, X0, X1, Y0, Y1):
    """min of h over the box, vectorised (exact quadratic, float64)."""
    dx0, dx1, dy0, dy1 = X0 - mx, X1 - mx, Y0 - my, Y1 - my
    inside = (dx0 <= 0) & (dx1 >= 0) & (dy0 <= 0) & (dy1 >= 0)
    q = lambda dx, dy: A * dx * dx + B2 * dx * dy + C * dy * dy  # noqa: E731
    hB = 0.5 * B2
    ya = np.clip(-hB * dx0 / C, dy0, dy1); yb = np.clip(-hB * dx1 / C, dy0, dy1)
    xa = np.clip(-hB * dy0 / A, dx0, dx1); xb = np.clip(-hB * dy1 / A, dx0, dx1)
    m = np.minimum(np.minimum(q(dx0, ya), q(dx1, yb)), np.minimum(q(xa, dy0), q(xb, dy1)))
    return np.where(inside, 0.0, m)


tot = miss_tile = miss_one_strip = 0
for v in range(views):
    rec = pr.rec[v].cpu().numpy().astype(np.float64)
    rect = pr.rect[v].cpu().numpy()
    ids = bins.ids[v].cpu().numpy()
    rg = bins.ranges[v].cpu().numpy()
    last = fr.last[v].cpu().numpy()
    fT = fr.final_T[v].cpu().numpy()
    for ty in range(ty_n):
        for tx in range(tx_n):
            b = (ty >> 2) * bx_n + (tx >> 2)
            s0, s1 = rg[b]
            lt = last[ty * 16:(ty + 1) * 16, tx * 16:(tx + 1) * 16]
            sat = (fT[ty * 16:(ty + 1) * 16, tx * 16:(tx + 1) * 16] < 1e-4).all()
            stop = s1 if not sat else min(s1, s0 + ((lt.max() - s0 + 63) // 64) * 64)
            e = ids[s0:stop]
            r = rect[e]
            ok = (r[:, 0] <= tx) & (r[:, 2] >= tx) & (r[:, 1] <= ty) & (r[:, 3] >= ty)
            e = e[ok]
            if len(e) == 0:
                continue
            mx, my, A, B2 = rec[e, 0], rec[e, 1], rec[e, 2], rec[e, 3]
            C, hm = rec[e, 4], rec[e, 5]
            X0, X1 = tx * 16 + 0.5, tx * 16 + 15.5
            Y0 = ty * 16 + 0.5
            mt = box_min(mx, my, A, B2, C, X0, X1, Y0, Y0 + 15) > hm
            m0 = box_min(mx, my, A, B2, C, X0, X1, Y0, Y0 + 7) > hm
            m1 = box_min(mx, my, A, B2, C, X0, X1, Y0 + 8, Y0 + 15) > hm
            tot += len(e)
            miss_tile += int(mt.sum())
            miss_one_strip += int((m0 ^ m1).sum())
print(json.dumps({"views": views, "visited_entries": tot, "ellipse_misses_tile": miss_tile / max(tot, 1),
                  "ellipse_misses_exactly_one_strip": miss_one_strip / max(tot, 1)}))
