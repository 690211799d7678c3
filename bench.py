#!/usr/bin/env python
"""SSS hot-path benchmark (BASELINE.json metric) — one JSON line on rank 0.

Workload (default): BASELINE config 5, the full training-step loop:
3,000,000 components (SH degree 3), 64 views at 1297x840 on a hemisphere,
per iteration project -> bin/sort -> composite -> fused-L1 backward over all
views, NCCL all-reduce of the parameter gradients (N > 1), SGHMC/Adam step.
A "step" is one such iteration.  `value` is whole-job training iterations/s
with inputs resident in HBM; `e2e` is the same metric through the public API
with the step's target images copied host->device (pinned) and the loss read
back every step.  Views are sharded round-robin over ranks (strong scaling:
the 64-view iteration is fixed, R ranks share it).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "fwd+bwd Mpixel/s and train iters/s at 1/2/4/8 B200; % of FP32/HBM roofline"

# Algorithmic work per unit: FP32 lane-ops per composited
# pair (forward / backward raster) and bytes per component-view (HBM kernels).
FWD_OPS_PER_PAIR = 19  # DESIGN.md §5 derivation
BWD_OPS_PER_PAIR = 58  # DESIGN.md §5 derivation


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--bin-shift", type=int, default=None,
                    help="default per config (measured best): 0 for configs 1-2, 1 for 4, 2 for 3 and 5")
    ap.add_argument("--views-per-batch", type=int, default=64)
    ap.add_argument("--max-per-bin", type=int, default=0,
                    help="truncated bin lists (sss.h sss_bins.max_per_bin); 0 = complete lists")
    ap.add_argument("--overlap-blocks", type=int, default=4,
                    help="N > 1: component blocks of the gradient exchange overlapped with the "
                         "projection backward (0 = one reduce-scatter after it)")
    ap.add_argument("--bins", default="adaptive", choices=["adaptive", "complete"],
                    help="adaptive: per-bin caps from the previous forward's consumption (sss.h sss_bins.used)")
    ap.add_argument("--tile-masks", type=int, default=None,
                    help="1: per-entry tile masks in the bin lists (sss.h sss_bins.tmask; default: on for "
                         "bin_shift 1-2)")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--graph", type=int, default=None,
                    help="1: replay each iteration as one CUDA graph (default: on for the launch-bound "
                         "configs 1-4, off for config 5; one process only)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-next", action="store_true", help="skip the NEXT-row timings")
    ap.add_argument("--cpu-budget-s", type=float, default=20.0)
    # NEXT-1: the full Eq. 8 objective (default: the BASELINE config's L1)
    ap.add_argument("--eps-dssim", type=float, default=0.0)
    ap.add_argument("--eps-o", type=float, default=0.0)
    ap.add_argument("--eps-sigma", type=float, default=0.0)
    a = ap.parse_args()
    if a.bin_shift is None:
        a.bin_shift = {1: 0, 2: 0, 3: 2, 4: 1, 5: 2}.get(a.config, 2)
    return a


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    d = {}
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
    return {"hbm_gbs": float(d.get("hbm_gbs", 6650.0)), "sm_max_mhz": float(d.get("sm_max_mhz", 1965.0)),
            "source": "measured" if d else "fallback"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.idx)], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except (OSError, ValueError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.th.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def ncu_traffic(kernel, views_per_launch):
    """dram read+write bytes per launch of `kernel` from the committed ncu
    capture (profiles/traffic.json), scaled to this run's launch size."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    b = d.get("bytes_per_launch", {}).get(kernel)
    if b is None:
        return None
    return int(b * views_per_launch / d.get("views_per_launch", views_per_launch))


def alu_peaks():
    """Measured FP32-pipe and MUFU rates of this GPU (sss_alu_peaks
    microbenchmark) next to the nominal SMs x 128 lanes x
    max clock."""
    import ctypes as C

    from paper_2503_10148_b200 import _lib as L

    out = (C.c_double * 7)()
    if L.load().sss_alu_peaks(out) != 0:
        return None
    sms, clk_khz = int(out[5]), out[6]
    return {"ffma_lane_ops_per_s": out[0], "ffma2_lane_ops_per_s": out[1],
            "fp32_lane_ops_per_s": max(out[0], out[1]),
            "mufu_ex2_per_s": out[2], "mufu_lg2_per_s": out[3], "mufu_rcp_per_s": out[4],
            "sm_count": sms, "sm_clock_mhz_attr": clk_khz / 1e3,
            "how": "independent FFMA / FFMA2 / MUFU chains, 8 per thread, 8 CTAs x 256 threads per SM, best of 5"}


def roofline_for(phase_ms, counts, n, views, pk, steps, views_per_launch=16, kernel=None):
    """Roofline entry of the dominant kernel (largest share of the timed step),
    or of `kernel` if given."""
    lane_peak = pk["lane_peak"]  # FP32 lane-ops/s: measured (alu_peaks) or nominal
    hbm_peak = pk["hbm_gbs"] * 1e9
    table = {}
    pairs = counts["pairs"]
    table["render_fwd"] = ("alu", pairs * FWD_OPS_PER_PAIR, lane_peak, "Glane-op/s")
    table["render_bwd_raster"] = ("alu", pairs * BWD_OPS_PER_PAIR, lane_peak, "Glane-op/s")
    P = counts["planes"]
    # projection: params read once per launch (<=views_per_batch views) + 60 B/view written
    table["project"] = ("hbm", counts["launches_per_step"] * n * 4 * P + views * n * 60, hbm_peak, "GB/s")
    # bin/sort: 16 B per comp-view (4 B depth + 8 B rect read, 4 B sorted id written)
    # + 4 B id written per materialised instance (+ 4 B id and 24 B record read, 2 B mask written
    # with tile masks)
    table["bin_sort"] = ("hbm", views * n * 16 + counts["instances"] * (34 if counts.get("tile_masks") else 4),
                         hbm_peak, "GB/s")
    # projection backward: g2d 40 B read per comp-view + params 240 B + grad RMW 480 B per launch
    table["render_bwd_projection"] = ("hbm", views * n * 40 + counts["launches_per_step"] * n * 4 * P * 3,
                                      hbm_peak, "GB/s")
    Pu = counts.get("sghmc_planes", P)  # this rank's planes (ZeRO-1 shard for R > 1)
    table["sghmc"] = ("hbm", counts.get("steps", 1) * n * 4 * (Pu * 7 + 6), hbm_peak, "GB/s")
    # image loss (L1 + D-SSIM): 132 B per pixel
    table["image_loss"] = ("hbm", counts.get("pixels", 0) * 132, hbm_peak, "GB/s")
    dom = kernel or max((k for k in phase_ms if k in table), key=lambda k: phase_ms[k])
    bound, work, peak, unit = table[dom]
    t = phase_ms[dom] / 1e3 / steps  # seconds per step in that kernel (all its launches)
    achieved = work / t
    return dom, {"kernel": dom, "bound": bound, "achieved": round(achieved / 1e9, 2),
                 "peak": round(peak / 1e9, 2), "unit": unit, "frac": round(achieved / peak, 4),
                 "traffic": ncu_traffic(dom, views_per_launch),
                 "traffic_unit": "dram bytes per launch (ncu --set full, profiles/traffic.json)",
                 "peak_source": (pk["lane_peak_source"] if bound == "alu" else pk["source"] + " hbm_gbs"),
                 "share_of_step": round(phase_ms[dom] / sum(phase_ms.values()), 3)}


def time_next_rows(ts, targets, pk):
    """NEXT-1 image loss (L1 + D-SSIM, eps 0.2) on the last view batch's
    frames, and one NEXT-2 recycling pass (5% cap) on a copy of the step's
    parameters, each timed with CUDA events on the launching stream."""
    import torch

    import paper_2503_10148_b200 as P
    from paper_2503_10148_b200 import api as A

    def timed(fn, reps=5, setup=None):
        if setup:
            setup()
        fn()
        ts_ = []
        for _ in range(reps):
            if setup:
                setup()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts_.append(e0.elapsed_time(e1))
        return sorted(ts_)[len(ts_) // 2]

    out = {}
    nv = len(ts.batches[-1])
    fr = ts.frame.rgb[:nv]
    tg = targets[ts.batches[-1][0]:ts.batches[-1][-1] + 1]
    if tg.dtype != torch.float32:  # the D-SSIM kernel reads fp32 targets (conversion untimed)
        tg = tg.float() / 255.0
    V, _, H, W = fr.shape
    d = torch.empty_like(fr)
    ws = torch.empty(max(A.image_loss_workspace_bytes(V, H, W), 4), dtype=torch.uint8, device=fr.device)
    ms = timed(lambda: P.sss_image_loss(fr, tg, 0.2, d_rgb=d, ws=ws))
    gbs = V * H * W * 132 / (ms / 1e3) / 1e9
    out["image_loss"] = {"ms": round(ms, 3), "views": V, "bound": "hbm", "achieved_gbs": round(gbs, 1),
                         "peak_gbs": pk["hbm_gbs"], "frac": round(gbs / pk["hbm_gbs"], 4),
                         "bytes_per_pixel": 132}
    planes = ts.params.planes.clone()
    params = P.Params(planes, ts.params.sh_degree)
    # 2% dead components (the bench scene has ~0.5%), restored before every pass
    g = torch.Generator(device=planes.device)
    g.manual_seed(7)
    kill = torch.rand(params.n, device=planes.device, generator=g) < 0.02
    planes[11][kill] = 0.0
    snap = planes.clone()
    m, v = P.Params(torch.zeros_like(planes), params.sh_degree), P.Params(torch.zeros_like(planes), params.sh_degree)
    r = torch.zeros((3, params.n), device=planes.device)
    ws_r = torch.empty(A.relocate_workspace_bytes(params.n), dtype=torch.uint8, device=planes.device)
    moved = torch.zeros(1, dtype=torch.int64, device=planes.device)
    ms_r = timed(lambda: P.sss_relocate(params, m, v, r, seed=1, step=1, n_moved=moved, ws=ws_r),
                 setup=lambda: planes.copy_(snap))
    out["relocate"] = {"ms": round(ms_r, 3), "n": params.n, "moved": int(moved.item()),
                       "note": "one recycling pass (dead |o| < 0.005, 5% cap, n_max 32) with 2% of the "
                               "step's components set dead"}
    del planes, snap, params, m, v, r, ws_r
    return out


def cpu_baseline_sample(scene, targets_np, budget_s, views_total):
    """Time the fp64 oracle (as it stands) on a bounded sample of the workload
    on this host's cores and extrapolate to it/s (rank 0 only)."""
    import numpy as np

    from oracle import oracle as O

    cores = len(os.sched_getaffinity(0))
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    cam = scene.cameras[0]
    n = scene.n
    P_ = cam.width * cam.height
    import ctypes

    t0 = time.time()
    pp = O._P(scene.params, scene.sh_degree)
    cc = O._cam(cam)
    tw, th = O.tiles_of(cam)
    counts = np.zeros(tw * th, np.int32)
    O.lib().orc_bin(pp.ref, ctypes.byref(cc), O._ptr(counts), None, None)  # project + bin
    t_bin = time.time() - t0
    rng = np.random.default_rng(0)
    npx = 65536  # ~6% of the view: enough pixel work to rise above the re-binning noise
    px = rng.choice(P_, npx, replace=False).astype(np.int32)
    # each oracle call re-projects and re-bins the view; subtract a 1-pixel call
    one = px[:1]
    t0 = time.time()
    O.render(scene.params, scene.sh_degree, cam, mode="tiled", pixels=one)
    t_fix_f = time.time() - t0
    t0 = time.time()
    fr = O.render(scene.params, scene.sh_degree, cam, mode="tiled", pixels=px)
    t_fwd = time.time() - t0 - t_fix_f
    tgt = targets_np[:, px // cam.width, px % cam.width]
    d = np.sign(fr.rgb - tgt) / (3 * P_)
    t0 = time.time()
    O.backward(scene.params, scene.sh_degree, cam, d[:, :1].copy(), mode="tiled", pixels=one)
    t_fix_b = time.time() - t0
    t0 = time.time()
    O.backward(scene.params, scene.sh_degree, cam, d, mode="tiled", pixels=px)
    t_bwd = time.time() - t0 - t_fix_b
    t_raster = max(t_fwd, 0.0) + max(t_bwd, 0.0)
    nsub = min(n, 100000)
    from sss_synth import make_optimizer_state, sghmc_params_for

    sub = scene.params[:, :nsub]
    r, m, v = make_optimizer_state(scene, zero=True)
    t0 = time.time()
    O.sghmc_step(sub, scene.sh_degree, np.zeros_like(sub), m[:, :nsub], v[:, :nsub], r[:, :nsub],
                 sghmc_params_for(scene))
    t_sg = (time.time() - t0) * n / nsub
    t_iter = views_total * (t_bin + t_raster * P_ / npx) + t_sg
    return {"value": round(1.0 / t_iter, 8), "unit": "it/s", "cores": cores, "kind": "oracle",
            "sample": (f"fp64 C++ oracle on host cores: project+bin of 1 view ({t_bin:.1f}s), "
                       f"fwd+bwd of {npx} random pixels of that view ({t_raster:.1f}s, scaled x{P_ // npx}), "
                       f"SGHMC on {nsub} comps (scaled x{n / nsub:.0f}); x{views_total} views; extrapolated"),
            "seconds_per_iter": round(t_iter, 1)}


def l2_flush_needed(config: int) -> bool:
    """Configs 1-2 fit the 126 MB L2 (config 2: ~110 MB of parameters, moments
    and per-view buffers): flush it between timed iterations."""
    return config <= 2


def arm_config(a, sc, world):
    """The workload's config (both arms print the same one)."""
    from sss_synth import CONFIG_NAMES

    cam = sc.cameras[0]
    return {"workload": CONFIG_NAMES[a.config], "n_components": sc.n, "views": sc.n_views,
            "width": cam.width, "height": cam.height, "sh_degree": sc.sh_degree,
            "bin_shift": a.bin_shift, "views_per_batch": a.views_per_batch, "max_per_bin": a.max_per_bin, "bins": a.bins,
            "tile_masks": bool(a.tile_masks) if a.tile_masks is not None else 1 <= a.bin_shift <= 2,
            "loss": ("eq8: (1-eps_D) L1 + eps_D D-SSIM + eps_o sum|o| + eps_S sum sqrt(lambda)"
                     if (a.eps_dssim or a.eps_o or a.eps_sigma) else "L1"),
            "eps_dssim": a.eps_dssim, "eps_o": a.eps_o, "eps_sigma": a.eps_sigma,
            "targets": "fp32" if a.eps_dssim > 0.0 else "uint8 images, read as u/255 (SSS_BWD_TARGET_U8)",
            "parallelism": f"view-dp{world}",
            "l2": ("flushed between timed iterations (512 MB write outside the per-iteration events)"
                   if l2_flush_needed(a.config) else
                   "no flush: inputs > L2 (parameters + moments + per-view records and bins exceed 126 MB)")}


def run_reference(a):
    """--impl reference: the oracle, timed as it stands, on bounded samples."""
    rank, world, local = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), 0
    if rank != 0:
        return 0
    from sss_synth import CONFIG_NAMES, make_scene, make_targets

    sc = make_scene(a.config)
    tg = make_targets(sc, [0])[0]
    vals = []
    for k in range(a.warmup + a.steps):
        cb = cpu_baseline_sample(sc, tg, a.cpu_budget_s, sc.n_views)
        if k >= a.warmup:
            vals.append(cb["value"])
    v = sum(vals) / len(vals)
    cb["value"] = v
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "it/s", "n_gpus": a.gpus,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(1e3 / v, 1),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": arm_config(a, sc, a.gpus),
            "cpu_baseline": cb,
            "e2e": {"value": v, "unit": "it/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def main():
    a = parse()
    if a.impl == "reference":
        return run_reference(a)
    import numpy as np
    import torch

    import paper_2503_10148_b200 as P
    from paper_2503_10148_b200 import dist as D
    from paper_2503_10148_b200.step import TrainStep
    from sss_synth import CONFIG_NAMES, make_scene, make_targets, make_targets_u8, sghmc_params_for

    if int(os.environ.get("WORLD_SIZE", "1")) > 1:  # communicator lines (comm_nranks) on stderr
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    rank, world, local = D.init()
    torch.cuda.set_device(local)
    P.load()
    ap_meas = alu_peaks()
    sc = make_scene(a.config)
    V = sc.n_views
    mine = D.shard_views(V, rank, world)
    cams = [sc.cameras[v] for v in mine]
    # 8-bit target images (as the paper's datasets), read by the fused-L1
    # backward as u / 255 (sss.h SSS_BWD_TARGET_U8); the D-SSIM loss reads fp32
    tg_np = make_targets(sc, mine) if a.eps_dssim > 0.0 else make_targets_u8(sc, mine)
    tg_f32 = tg_np if tg_np.dtype == np.float32 else tg_np.astype(np.float32) / np.float32(255.0)
    targets = torch.from_numpy(tg_np).cuda()
    planes = torch.from_numpy(sc.params).cuda()
    hp = sghmc_params_for(sc, eps_o=a.eps_o, eps_sigma=a.eps_sigma)
    ts = TrainStep(planes, sc.sh_degree, cams, hp, total_views=V, bin_shift=a.bin_shift,
                   views_per_batch=a.views_per_batch, eps_dssim=a.eps_dssim, max_per_bin=a.max_per_bin,
                   adaptive_bins=a.bins == "adaptive", overlap_blocks=a.overlap_blocks if world > 1 else 0,
                   tile_masks=None if a.tile_masks is None else bool(a.tile_masks))
    for _ in range(a.warmup):
        ts.step(targets)
        if ts.overflowed():
            ts.grow()
    torch.cuda.synchronize()
    D.barrier()
    # ---- timed region: device-resident inputs
    cvd = [x for x in os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",") if x.strip().isdigit()]
    clk = ClockSampler(int(cvd[local]) if local < len(cvd) else local)
    clk.start()
    snap = ts.params.planes.clone()  # the first timed state (pair counts below)
    torch.cuda.synchronize()
    P.launch_count(reset=True)
    # configs 1-4 are host/launch-bound at one GPU (e2e config 3: +19 % with the
    # graph); config 5's 103 ms step gains 0.2 % and keeps its eager per-phase
    # CUDA-event split inside the timed region
    use_graph = (a.config <= 4 if a.graph is None else bool(a.graph)) and world == 1
    if use_graph:  # one eager warm-up iteration + the capture: both count the launches
        P.launch_count(reset=True)
        ts.capture(targets)
        per_step_launches = P.launch_count(reset=True) // 2
        torch.cuda.synchronize()
    else:
        ts.prof = []
    torch.cuda.synchronize()
    D.barrier()
    # small working sets (configs 1-2: < the 126 MB L2): flush L2 between the
    # timed iterations (a 512 MB write outside the per-iteration events)
    flush = l2_flush_needed(a.config)
    fbuf = torch.empty(512 << 20, dtype=torch.uint8, device="cuda") if flush else None
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
    e0.record()
    for k in range(a.steps):
        if flush:
            fbuf.fill_(k & 255)
            ev[k][0].record()
        if use_graph:
            ts.replay()
        else:
            ts.step(targets)
        if flush:
            ev[k][1].record()
    e1.record()
    torch.cuda.synchronize()
    D.barrier()
    launches = P.launch_count(reset=True)
    if use_graph:
        launches = per_step_launches * a.steps  # replayed from the graph (no host launches)
        ts.prof = []  # the phase split from a few eager iterations after the timed region
        nph = max(2, min(a.steps, 5))
        for _ in range(nph):
            ts.step(targets)
        torch.cuda.synchronize()
    clocks = clk.stop()
    # bitwise checksum of the parameters over ranks after the timed steps
    identical = D.replicas_identical(ts.params.planes)
    ms = sum(b.elapsed_time(c) for b, c in ev) if flush else e0.elapsed_time(e1)
    ms_max = D.allreduce_max(ms, device=torch.device("cuda", local))
    del fbuf
    phases = ts.phase_ms()
    if use_graph:  # scale the eager split to the graph-timed step
        tot = sum(phases.values())
        phases = {k: v / tot * ms_max for k, v in phases.items()} if tot > 0 else phases
    ts.prof = None
    overflow = ts.overflowed()
    it_s = a.steps / (ms_max / 1e3)
    H, W = sc.cameras[0].height, sc.cameras[0].width
    mpix = it_s * V * H * W / 1e6
    # ---- counts for the roofline: composited pairs and instances of the
    # timed states, measured (untimed) at the first and the last timed state
    # and averaged (the counts drift slowly along the training trajectory)
    dev = torch.device("cuda", local)

    def count_state():
        ts.stats = {"pairs": torch.zeros((), dtype=torch.int64, device=dev),
                    "instances": torch.zeros((), dtype=torch.int64, device=dev)}
        ts.forward_backward(targets)
        r = float(ts.stats["pairs"].item()), float(ts.stats["instances"].item())
        ts.stats = None
        return r

    final = ts.params.planes.clone()
    p_last, i_last = count_state()
    ts.params.planes.copy_(snap)
    p_first, i_first = count_state()
    ts.params.planes.copy_(final)
    del snap, final
    pairs, inst = 0.5 * (p_first + p_last), 0.5 * (i_first + i_last)
    counts = {"steps": a.steps, "sghmc_planes": (ts.p1 - ts.p0) if ts.shard else sc.params.shape[0],
              "pairs": pairs * a.steps, "instances": inst * a.steps, "planes": sc.params.shape[0],
              "tile_masks": bool(ts.tile_masks),
              "launches_per_step": len(ts.batches) * a.steps,
              "pixels": len(mine) * a.steps * sc.cameras[0].width * sc.cameras[0].height}
    pk = peaks()
    sms = ap_meas["sm_count"] if ap_meas else torch.cuda.get_device_properties(local).multi_processor_count
    nominal = sms * 128 * pk["sm_max_mhz"] * 1e6
    if ap_meas:
        pk["lane_peak"] = ap_meas["fp32_lane_ops_per_s"]
        pk["lane_peak_source"] = (f"measured (sss_alu_peaks: max of FFMA / FFMA2 lane-op rates; nominal "
                                  f"{sms} SMs x 128 lanes x {pk['sm_max_mhz']:.0f} MHz = {nominal / 1e12:.2f} T)")
    else:
        pk["lane_peak"] = nominal
        pk["lane_peak_source"] = f"nominal ({sms} SMs x 128 FP32 lanes x sm_max_mhz)"
    dom, roof = roofline_for(phases, counts, sc.n, len(mine) * a.steps, pk, 1,
                             views_per_launch=len(ts.batches[0]))
    # every timed phase against its own bound (informational; `roofline` is
    # the dominant one)
    all_roof = {}
    for ph in phases:
        try:
            r = roofline_for(phases, counts, sc.n, len(mine) * a.steps, pk, 1,
                             views_per_launch=len(ts.batches[0]), kernel=ph)[1]
        except KeyError:
            continue
        all_roof[ph] = {k: r[k] for k in ("bound", "achieved", "peak", "unit", "frac", "share_of_step")}
    extra_roof = {}
    if "image_loss" in phases:
        extra_roof["image_loss"] = roofline_for(phases, counts, sc.n, len(mine) * a.steps, pk, 1,
                                                views_per_launch=len(ts.batches[0]),
                                                kernel="image_loss")[1]
    # ---- end to end through the public API: H2D targets + loss read back
    e2e_steps = a.e2e_steps or a.steps
    # Each step's targets are copied host->device (pinned) inside the timed
    # region; the copy for step k+1 runs on a copy stream while step k
    # computes (double-buffered, as a training input pipeline would), and
    # every step's loss is read back to the host.
    host_t = torch.from_numpy(tg_np).pin_memory()
    bufs = [torch.empty_like(targets), torch.empty_like(targets)]
    copy_s = torch.cuda.Stream()
    comp_s = torch.cuda.current_stream()
    copied = [torch.cuda.Event(), torch.cuda.Event()]
    used = [torch.cuda.Event(), torch.cuda.Event()]
    got = [torch.cuda.Event(), torch.cuda.Event()]
    loss_host = torch.zeros(2, dtype=torch.float32).pin_memory()
    losses_e2e = []
    torch.cuda.synchronize()
    D.barrier()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    copy_s.wait_stream(comp_s)
    with torch.cuda.stream(copy_s):
        bufs[0].copy_(host_t, non_blocking=True)
        copied[0].record()
    for k in range(e2e_steps):
        cur, nxt = k % 2, (k + 1) % 2
        if k + 1 < e2e_steps:
            with torch.cuda.stream(copy_s):
                if k >= 1:
                    copy_s.wait_event(used[nxt])  # step k-1 is done with that buffer
                bufs[nxt].copy_(host_t, non_blocking=True)
                copied[nxt].record()
        comp_s.wait_event(copied[cur])
        loss = ts.replay(bufs[cur]) if use_graph else ts.step(bufs[cur])
        used[cur].record()
        # every step's loss goes device->host (pinned); the host reads step
        # k's value while step k+1 runs (the GPU never waits for the host)
        loss_host[cur:cur + 1].copy_(loss, non_blocking=True)
        got[cur].record()
        if k >= 1:
            got[nxt].synchronize()
            losses_e2e.append(float(loss_host[nxt]))
    s1.record()
    got[(e2e_steps - 1) % 2].synchronize()
    losses_e2e.append(float(loss_host[(e2e_steps - 1) % 2]))
    torch.cuda.synchronize()
    e2e_ms = D.allreduce_max(s0.elapsed_time(s1), device=torch.device("cuda", local))
    e2e = {"value": round(e2e_steps / (e2e_ms / 1e3), 4), "unit": "it/s",
           "h2d_bytes_per_step": int(host_t.numel() * host_t.element_size()), "d2h_bytes_per_step": 4,
           "pipeline": ("next step's targets copied (pinned H2D) on a second stream during the current step; "
                        "each step's loss copied D2H (pinned) and read by the host while the next step runs"),
           "losses_read": len(losses_e2e)}
    del bufs, host_t
    # ---- NEXT rows, timed outside the step (CUDA events, 5 repeats, median)
    next_rows = {}
    if not a.no_next:
        next_rows = time_next_rows(ts, targets, pk)
    if rank == 0:
        cb = None
        if world == 1 and not a.no_cpu_baseline:
            try:
                cb = cpu_baseline_sample(sc, tg_f32[0], a.cpu_budget_s, V)
            except Exception as ex:  # noqa: BLE001
                cb = {"error": str(ex)}
        line = {
            "metric": METRIC, "value": round(it_s, 4), "unit": "it/s", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(ms_max / a.steps, 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": arm_config(a, sc, world),
            "mpix_per_s_fwd_bwd": round(mpix, 2),
            "phase_ms_per_step": {k: round(v / a.steps, 3) for k, v in phases.items()},
            "roofline": roof,
            "roofline_all_phases": all_roof,
            **({"roofline_next": extra_roof} if extra_roof else {}),
            "cpu_baseline": cb,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "next_rows": next_rows,
            "clocks": clocks,
            "alu_peaks": ap_meas,
            "cuda_graph": bool(use_graph),
            "bin_overflow": bool(overflow),
            "replicas_identical": bool(identical),
            "exchange": {"scheme": ("zero1-blocked-overlap" if ts.shard and ts.blocks else
                                    "zero1" if ts.shard else "replicated" if world > 1 else "none"),
                         "blocks": ts.blocks, "world": world,
                         "backend": (torch.distributed.get_backend() if world > 1 else None)},
            "counts_per_step": {"pairs_first": p_first, "pairs_last": p_last, "instances_first": i_first,
                                "instances_last": i_last},
        }
        print(json.dumps(line), flush=True)
    D.barrier()
    return 0


if __name__ == "__main__":
    sys.exit(main())
