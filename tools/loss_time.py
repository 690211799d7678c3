"""Dev tool: CUDA-event time of sss_image_loss (Eq. 8 image part) on 64 views of 1297x840."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2503_10148_b200 as P
from paper_2503_10148_b200 import api as A

V, H, W = 64, 840, 1297
g = torch.Generator(device="cuda").manual_seed(0)
rgb = torch.rand((V, 3, H, W), device="cuda", generator=g)
tgt = torch.rand((V, 3, H, W), device="cuda", generator=g)
d = torch.empty_like(rgb)
ws = torch.empty(max(A.image_loss_workspace_bytes(V, H, W), 4), dtype=torch.uint8, device="cuda")
loss = torch.zeros(1, device="cuda")
ts = []
for k in range(12):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    loss.zero_()
    e0.record()
    P.sss_image_loss(rgb, tgt, 0.2, d_rgb=d, loss=loss, ws=ws)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(json.dumps({"lib": os.environ.get("SSS_LIB", "default"), "ms": round(sorted(ts[2:])[len(ts[2:]) // 2], 4),
                  "loss": float(loss.item())}))
