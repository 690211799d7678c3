"""One SSS training iteration on the CUDA path (SURVEY.md §3 call stack 2).

For each batch of this rank's views: sss_project -> sss_bin_sort ->
sss_render_fwd -> sss_render_bwd (fused L1, gradients accumulated over
views); then the NCCL all-reduce of the flat gradient buffer (R > 1) and
sss_sghmc_step with grad_scale = 1/V (R26).  All calls are asynchronous on
one stream; the only host synchronisation is the loss / overflow read-back
the caller asks for.  Buffers are allocated once and reused; the bin
capacity is sized from a measured instance count with headroom.

Bin overflow (an iteration needs more instances than the capacity): the
overflow flag is sticky on the device and the sampler step is told to skip
its update when it is set (sss_sghmc_hparams.skip_if; all-reduced over
ranks first, so replicas never diverge), so an overflowed iteration never
moves parameters, moments or momentum.  step(check=True) reads the flag
(one host sync), grows the capacity and replays the iteration;
step(check=False) leaves the check to the caller (overflowed() after a run
sees every overflow since the last reset_overflow()).

Loss: step() returns this rank's device float[1] sum over its views of the
per-view mean L1 (sss_render_bwd's loss_out); the objective of R26 is that
sum over all ranks divided by total_views (see mean_loss()).
"""
from __future__ import annotations

from typing import List, Optional, Sequence

import torch

from . import api as A
from . import dist as D


class TrainStep:
    def __init__(self, planes: torch.Tensor, sh_degree: int, cameras: Sequence, hp,
                 total_views: Optional[int] = None, bin_shift: int = 0,
                 views_per_batch: int = 16, bg=(0.0, 0.0, 0.0), headroom: float = 1.25,
                 group=None, momentum: Optional[torch.Tensor] = None,
                 adam_m: Optional[torch.Tensor] = None, adam_v: Optional[torch.Tensor] = None,
                 eps_dssim: float = 0.0, variant: int = 0, shard_update: Optional[bool] = None,
                 max_per_bin: int = 0, adaptive_bins: bool = False, overlap_blocks: int = 0,
                 tile_masks: Optional[bool] = None):
        dev = planes.device
        world = D.dist.get_world_size(group) if D.dist.is_initialized() else 1
        # ZeRO-1 sharded sampler step for R > 1 (dist.py): plane buffers padded
        # to R * ceil(P / R) planes; the Params views cover the first P.
        # shard_update=True forces it on any initialised group (tests run the
        # NCCL path with one rank)
        if shard_update is None:
            self.shard = world > 1
        else:
            self.shard = bool(shard_update) and D.dist.is_initialized()
        P = planes.shape[0]
        self.world = world
        if self.shard:
            self.rank = D.dist.get_rank(group)
            pr, (self.p0, self.p1) = D.plane_shard(P, self.rank, world)
            pad = torch.zeros((pr * world, planes.shape[1]), dtype=planes.dtype, device=dev)
            pad[:P].copy_(planes)
            self.params_pad = pad
            self.grad_pad = torch.zeros_like(pad)
            self.scratch = torch.empty((pr, planes.shape[1]), dtype=planes.dtype, device=dev)
            self.params = A.Params(pad[:P], sh_degree, variant)
            self.grad = A.Params(self.grad_pad[:P], sh_degree, variant)
            # overlapped exchange: component-blocked gradient, one reduce-scatter
            # per block as soon as the projection backward has finished it
            self.blocks = int(overlap_blocks)
            if self.blocks > 0:
                self.grad_blk = A.BlockedParams.zeros(planes.shape[1], sh_degree, self.blocks, pr * world, dev,
                                                      variant)
                self.comm = torch.cuda.Stream(device=dev) if dev.type == "cuda" else None
        else:
            self.params = A.Params(planes, sh_degree, variant)
            self.grad = A.Params.zeros_like(self.params)
            self.blocks = 0
        self.m = A.Params(adam_m if adam_m is not None else torch.zeros_like(planes), sh_degree, variant)
        self.v = A.Params(adam_v if adam_v is not None else torch.zeros_like(planes), sh_degree, variant)
        n = self.params.n
        self.r = momentum if momentum is not None else torch.zeros((3, n), device=dev)
        self.hp = hp
        self.cams = list(cameras)
        self.total_views = int(total_views if total_views is not None else len(self.cams))
        self.bin_shift = int(bin_shift)
        self.max_per_bin = int(max_per_bin)  # > 0: truncated bin lists (sss.h sss_bins)
        # adaptive truncation: each view batch keeps its bins' consumption from
        # the previous iteration's forward (sss.h sss_bins.used; -1 = complete)
        self.adaptive_bins = bool(adaptive_bins)
        # per-entry tile masks (sss.h sss_bins.tmask): on by default for bins of 2x2 / 4x4 tiles
        self.tile_masks = (1 <= self.bin_shift <= 2) if tile_masks is None else bool(tile_masks)
        self.bg = tuple(float(x) for x in bg)
        self.headroom = headroom
        self.group = group
        self.t = int(getattr(hp, "step", 1))
        vb = max(1, min(int(views_per_batch), len(self.cams)))
        self.batches: List[List[int]] = [list(range(i, min(i + vb, len(self.cams))))
                                         for i in range(0, len(self.cams), vb)]
        self.cams_c = [A.cameras_c([self.cams[v] for v in b]) for b in self.batches]
        W, H = int(self.cams[0].width), int(self.cams[0].height)
        self.W, self.H = W, H
        self.proj = A.Projected.empty(n, vb, dev)
        self.frame = A.Frame.empty(vb, H, W, dev)
        self.n_bins = A.n_bins_of(W, H, self.bin_shift)
        need = max(A.bin_sort_workspace_bytes(n, [self.cams[0]] * vb, self.bin_shift), 1)
        self.ws_bin = torch.empty(need, dtype=torch.uint8, device=dev)
        self.ws_g2d = torch.zeros(max(A.render_bwd_workspace_bytes(n, vb), 4), dtype=torch.uint8,
                                  device=dev)
        self.loss = torch.zeros(1, device=dev)
        # Eq. 8 image loss: eps_dssim = 0 keeps the fused-L1 backward (BASELINE
        # configs); > 0 forms (1 - eps) L1 + eps D-SSIM and its image gradient
        # with sss_image_loss, then runs the backward on that gradient.  The
        # regularizer weights travel in hp (eps_o, eps_sigma).
        self.eps_dssim = float(eps_dssim)
        if self.eps_dssim > 0.0:
            self.d_rgb = torch.empty((vb, 3, H, W), dtype=torch.float32, device=dev)
            self.ws_loss = torch.empty(max(A.image_loss_workspace_bytes(vb, H, W), 4),
                                       dtype=torch.uint8, device=dev)
        self.bins: List[A.Bins] = []
        self.used = ([torch.full((len(b), self.n_bins), -1, dtype=torch.int32, device=dev) for b in self.batches]
                     if self.adaptive_bins else None)
        self.prof = None  # list of (phase, cuda event) when timing phases
        self.stats = None  # dict of device counters (pairs, instances) when counting
        self._size_bins()

    def _mark(self, name: str):
        if self.prof is not None:
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            self.prof.append((name, e))

    # -- bin capacity ------------------------------------------------------
    def _size_bins(self, factor: float = 1.0):
        """Measure the per-view instance count of every batch (host sync)."""
        cap = 0
        for bi, b in enumerate(self.batches):
            cams = [self.cams[v] for v in b]
            pv = self._proj_view(len(b))
            A.sss_project(self.params, cams, out=pv, cams_c=self.cams_c[bi])
            probe = A.Bins.empty(len(b), self.n_bins, 0, self.bin_shift, False, self.params.planes.device,
                                 self.max_per_bin, self.params.n)
            A.sss_bin_sort(pv, cams, bin_shift=self.bin_shift, ws=self.ws_bin, out=probe,
                           cams_c=self.cams_c[bi])
            cap = max(cap, int(probe.totals.max().item()))
        cap = int(cap * self.headroom * factor) + 4096
        vb = len(self.batches[0])
        self.bins = [A.Bins.empty(vb, self.n_bins, cap, self.bin_shift, False,
                                  self.params.planes.device, self.max_per_bin, self.params.n,
                                  adaptive=self.adaptive_bins, tile_masks=self.tile_masks)]
        self.capacity = cap

    def _proj_view(self, nv: int) -> A.Projected:
        return A.Projected(self.proj.rec[:nv], self.proj.depth[:nv], self.proj.rect[:nv], self.proj.col[:nv])

    def _frame_view(self, nv: int) -> A.Frame:
        # n_contrib is a diagnostic the backward does not read: counted only
        # when the caller collects statistics
        f = self.frame
        nc = f.n_contrib[:nv] if self.stats is not None else None
        return A.Frame(f.rgb[:nv], f.final_T[:nv], nc, f.last[:nv],
                       f.tile_list[:nv] if f.tile_list is not None else None,
                       f.tile_count[:nv] if f.tile_count is not None else None)

    def _bins_view(self, nv: int) -> A.Bins:
        return self.bins[0].view(nv)

    # -- the iteration -----------------------------------------------------
    def forward_backward(self, targets: torch.Tensor, exchange: bool = False) -> None:
        """Render this rank's views and accumulate grad (no optimizer step).
        targets: [V_local][3][H][W] fp32 device tensor.  exchange (overlapped
        ZeRO-1 mode): the last view batch's projection backward runs block by
        block and each block's reduce-scatter is issued on the communication
        stream right after it (step() waits for them)."""
        blocked = self.blocks > 0
        if blocked:
            self.grad_blk.buf.zero_()
        # plain layout: the first batch's backward assigns the gradient
        # (SSS_BWD_GRAD_ASSIGN), later batches accumulate -- no zeroing pass
        self.loss.zero_()
        self._mark("start")
        for bi, b in enumerate(self.batches):
            nv = len(b)
            cams = [self.cams[v] for v in b]
            cc = self.cams_c[bi]
            pv, fv, bv = self._proj_view(nv), self._frame_view(nv), self._bins_view(nv)
            if self.used is not None:
                bv.used = self.used[bi]
            tg = targets[b[0]:b[-1] + 1]
            A.sss_project(self.params, cams, out=pv, cams_c=cc)
            self._mark("project")
            A.sss_bin_sort(pv, cams, bin_shift=self.bin_shift, ws=self.ws_bin, out=bv, cams_c=cc)
            self._mark("bin_sort")
            A.sss_render_fwd(pv, bv, cams, bg=self.bg, out=fv, cams_c=cc)
            self._mark("render_fwd")
            if self.stats is not None:
                self.stats["pairs"] += fv.n_contrib.sum(dtype=torch.int64)
                self.stats["instances"] += bv.totals.sum()
            d_rgb = None
            if self.eps_dssim > 0.0:
                assert tg.dtype == torch.float32, "the D-SSIM loss reads fp32 targets"
                d_rgb = A.sss_image_loss(fv.rgb, tg, self.eps_dssim, d_rgb=self.d_rgb[:nv],
                                         loss=self.loss, ws=self.ws_loss)
                self._mark("image_loss")
            kw = dict(bg=self.bg, target=None if d_rgb is not None else tg, d_rgb=d_rgb,
                      grad=self.grad_blk if blocked else self.grad, loss=self.loss, ws=self.ws_g2d, cams_c=cc,
                      assign=not blocked and bi == 0)
            if blocked and exchange and bi == len(self.batches) - 1:
                A.sss_render_bwd(self.params, pv, bv, cams, fv, half="raster", **kw)
                self._mark("render_bwd_raster")
                comp = torch.cuda.current_stream()
                for k in range(self.blocks):
                    i0, i1 = self.grad_blk.block_range(k)
                    A.sss_project_bwd_range(self.params, cams, self.ws_g2d, self.grad_blk, i0, i1, cams_c=cc)
                    ev = torch.cuda.Event()
                    ev.record(comp)
                    self.comm.wait_event(ev)
                    with torch.cuda.stream(self.comm):
                        D.reduce_scatter_block_(self.grad_blk.buf[k], self.group)
                self._mark("render_bwd_projection")
            elif self.prof is None:
                A.sss_render_bwd(self.params, pv, bv, cams, fv, **kw)
            else:  # same two kernels, split so each can be timed
                A.sss_render_bwd(self.params, pv, bv, cams, fv, half="raster", **kw)
                self._mark("render_bwd_raster")
                A.sss_render_bwd(self.params, pv, bv, cams, fv, half="projection", **kw)
                self._mark("render_bwd_projection")

    def step(self, targets: torch.Tensor, check: bool = False) -> torch.Tensor:
        """One full iteration; returns this rank's device loss sum (see the
        module docstring).  check=True: synchronise on the overflow flag and
        replay the iteration with grown bins until it fits."""
        overlap = self.shard and self.blocks > 0
        self.forward_backward(targets, exchange=overlap)
        while check and self.overflowed():
            self.grow()
            self.forward_backward(targets, exchange=overlap)
        flag = self.bins[0].overflow
        if self.world > 1:  # any rank's overflow skips every rank's update
            D.allreduce_max_(flag, self.group)
        self.hp.skip_if = flag
        self.hp.step = self.t
        self.hp.grad_scale = 1.0 / self.total_views
        if overlap:  # the blocks' reduce-scatters were issued during the projection backward
            torch.cuda.current_stream().wait_stream(self.comm)
            self._mark("allreduce")
            self.hp.plane_begin, self.hp.plane_end = self.p0, self.p1
            if self.p1 > self.p0:
                A.sss_sghmc_step(self.params, self.grad_blk, self.m, self.v, self.r, self.hp)
            self._mark("sghmc")
            D.all_gather_planes_(self.params_pad, self.scratch, self.group)
            self._mark("allgather")
        elif self.shard:
            D.reduce_scatter_planes_(self.grad_pad, self.scratch, self.group)
            self._mark("allreduce")
            self.hp.plane_begin, self.hp.plane_end = self.p0, self.p1
            if self.p1 > self.p0:
                A.sss_sghmc_step(self.params, self.grad, self.m, self.v, self.r, self.hp)
            self._mark("sghmc")
            D.all_gather_planes_(self.params_pad, self.scratch, self.group)
            self._mark("allgather")
        else:
            D.allreduce_sum_(self.grad.planes, self.group)
            self._mark("allreduce")
            self.hp.plane_begin, self.hp.plane_end = 0, 0
            A.sss_sghmc_step(self.params, self.grad, self.m, self.v, self.r, self.hp)
            self._mark("sghmc")
        self.t += 1
        return self.loss

    # -- CUDA graph of one iteration (launch-bound small scenes, config 2) ---
    def capture(self, targets: torch.Tensor) -> None:
        """Capture one whole iteration (every view batch, the sampler step) in
        a CUDA graph; replay() then runs an iteration with one launch.  The
        step counter moves to the device (sss_step_state), the targets to a
        static buffer.  One process (the NCCL exchange is not captured)."""
        assert self.world == 1 and self.prof is None and self.stats is None
        dev = self.params.planes.device
        self.hp.step_state = A.step_state(self.t, dev)
        self.g_targets = targets.clone()
        side = torch.cuda.Stream(device=dev)
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):  # warm-up iteration (a real one) on the capture stream
            self.step(self.g_targets)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.step(self.g_targets)
        self.t -= 1  # the capture launched nothing

    def replay(self, targets: Optional[torch.Tensor] = None) -> torch.Tensor:
        """One captured iteration; `targets` (if given and not the static
        buffer) is copied into the static buffer first."""
        if targets is not None and targets.data_ptr() != self.g_targets.data_ptr():
            self.g_targets.copy_(targets, non_blocking=True)
        self.graph.replay()
        self.t += 1
        return self.loss

    def phase_ms(self) -> dict:
        """Per-phase milliseconds of the recorded events (after a sync)."""
        out = {}
        if not self.prof:
            return out
        prev = self.prof[0][1]
        for name, e in self.prof[1:]:
            if name == "start":
                prev = e
                continue
            out[name] = out.get(name, 0.0) + prev.elapsed_time(e)
            prev = e
        return out

    def overflowed(self) -> bool:
        """Synchronising check of the (sticky) bin overflow flag."""
        return bool(self.bins[0].overflow.item())

    def reset_overflow(self):
        self.bins[0].overflow.zero_()

    def grow(self):
        """Re-measure the instance counts and re-size the bins (x1.5 headroom
        on top of the usual); the new buffers start with a clear flag."""
        self._size_bins(factor=1.5)

    def mean_loss(self, loss: torch.Tensor = None) -> float:
        """The R26 objective (1/V) sum_v L1_v over all ranks (host sync)."""
        t = (self.loss if loss is None else loss).clone()
        D.allreduce_sum_(t, self.group)
        return float(t.item()) / self.total_views
