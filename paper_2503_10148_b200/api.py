"""Thin torch binding of the C ABI (include/sss.h), same names as the ABI.

PyTorch supplies device memory and streams only; each function marshals
pointers and calls one libsss.so entry point.  Shapes follow sss.h exactly.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence

import torch

from . import _lib as L


def _stream_ptr(stream: Optional[torch.cuda.Stream]):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _ptr(t: Optional[torch.Tensor]):
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)


def n_planes(sh_degree: int) -> int:
    return 12 + 3 * (sh_degree + 1) ** 2


# ------------------------------------------------------------------ params
class Params:
    """Component parameters as one flat [P][n] fp32 device tensor (SoA planes).

    Gradients and Adam moments use the same class (identical layout), so the
    whole gradient is one contiguous buffer for the NCCL all-reduce."""

    def __init__(self, planes: torch.Tensor, sh_degree: int, variant: int = 0):
        assert planes.dtype == torch.float32 and planes.is_contiguous() and planes.dim() == 2
        assert planes.shape[0] == n_planes(sh_degree), (planes.shape, sh_degree)
        self.planes = planes
        self.sh_degree = int(sh_degree)
        self.variant = int(variant)  # SSS_VARIANT_* flags (NEXT-3 ablations); 0 = SSS

    @property
    def n(self) -> int:
        return int(self.planes.shape[1])

    @classmethod
    def zeros_like(cls, other: "Params") -> "Params":
        return cls(torch.zeros_like(other.planes), other.sh_degree, other.variant)

    def c(self) -> L.sss_params:
        b = self.planes.data_ptr()
        n = self.n
        off = lambda p: C.c_void_p(b + 4 * p * n)  # noqa: E731
        return L.sss_params(n, self.sh_degree, self.variant, off(0), off(3), off(6), off(10), off(11),
                            off(12), 0, 0, 0)


class BlockedParams:
    """A component-blocked parameter-shaped set (gradients of the overlapped
    multi-GPU exchange, sss.h sss_params.block): one flat [n_blocks][P_pad][B]
    fp32 tensor; block k holds components [k B, (k + 1) B), plane p at row p.
    A block is contiguous, so it can be exchanged while later blocks are
    still being computed."""

    def __init__(self, buf: torch.Tensor, n: int, sh_degree: int, variant: int = 0):
        assert buf.dtype == torch.float32 and buf.is_contiguous() and buf.dim() == 3
        assert buf.shape[1] >= n_planes(sh_degree) and buf.shape[0] * buf.shape[2] >= n
        self.buf = buf
        self.n = int(n)
        self.sh_degree = int(sh_degree)
        self.variant = int(variant)

    @property
    def block(self) -> int:
        return int(self.buf.shape[2])

    @classmethod
    def zeros(cls, n: int, sh_degree: int, n_blocks: int, planes: int, device, variant: int = 0):
        B = -(-n // n_blocks)
        return cls(torch.zeros((n_blocks, planes, B), dtype=torch.float32, device=device), n, sh_degree,
                   variant)

    def block_range(self, k: int):
        B = self.block
        return k * B, min(self.n, (k + 1) * B)

    def to_planes(self) -> torch.Tensor:
        """The plain [P][n] layout (a copy; host-side inspection / tests)."""
        P = n_planes(self.sh_degree)
        return self.buf[:, :P, :].permute(1, 0, 2).reshape(P, -1)[:, :self.n].contiguous()

    def c(self) -> L.sss_params:
        z = C.c_void_p(0)
        return L.sss_params(self.n, self.sh_degree, self.variant, C.c_void_p(self.buf.data_ptr()), z, z, z, z, z,
                            self.block, int(self.buf.shape[1]), 0)


def camera_c(cam) -> L.sss_camera:
    c = L.sss_camera()
    R = [float(x) for x in torch.as_tensor(cam.R, dtype=torch.float32).reshape(9).tolist()]
    t = [float(x) for x in torch.as_tensor(cam.t, dtype=torch.float32).reshape(3).tolist()]
    for k in range(9):
        c.rot[k] = R[k]
    for k in range(3):
        c.trans[k] = t[k]
    c.fx, c.fy, c.cx, c.cy = float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy)
    c.width, c.height = int(cam.width), int(cam.height)
    c.z_near = float(cam.z_near)
    return c


def cameras_c(cams: Sequence) -> C.Array:
    arr = (L.sss_camera * len(cams))()
    for i, cam in enumerate(cams):
        arr[i] = camera_c(cam)
    return arr


def tiles_of(width: int, height: int):
    return (width + 15) // 16, (height + 15) // 16


def n_bins_of(width: int, height: int, bin_shift: int) -> int:
    tx, ty = tiles_of(width, height)
    s = 1 << bin_shift
    return ((tx + s - 1) // s) * ((ty + s - 1) // s)


# ----------------------------------------------------------------- outputs
@dataclass
class Projected:
    rec: torch.Tensor    # [V][n][8] f32 {mx, my, A, B2, C, hmax, o, inv_nu}
    depth: torch.Tensor  # [V][n] f32
    rect: torch.Tensor   # [V][n][4] i16
    col: torch.Tensor    # [V][n][4] f32 {e, r, g, b}

    @classmethod
    def empty(cls, n: int, V: int, device="cuda") -> "Projected":
        return cls(torch.empty((V, n, L.SSS_REC_FLOATS), dtype=torch.float32, device=device),
                   torch.empty((V, n), dtype=torch.float32, device=device),
                   torch.empty((V, n, 4), dtype=torch.int16, device=device),
                   torch.empty((V, n, L.SSS_COL_FLOATS), dtype=torch.float32, device=device))

    @property
    def n(self):
        return int(self.depth.shape[1])

    @property
    def n_views(self):
        return int(self.depth.shape[0])

    def c(self) -> L.sss_projected:
        return L.sss_projected(self.n, self.n_views, 0, _ptr(self.rec), _ptr(self.depth),
                               _ptr(self.rect), _ptr(self.col))


@dataclass
class Bins:
    bin_shift: int
    capacity: int
    ids: torch.Tensor               # [V][capacity] i32
    keys: Optional[torch.Tensor]    # [V][capacity] i64 (bit pattern of u64) or None
    ranges: torch.Tensor            # [V][n_bins][2] i32
    totals: torch.Tensor            # [V] i64
    overflow: torch.Tensor          # [1] i32 (sticky: zeroed by the caller)
    max_per_bin: int = 0            # 0: complete lists; > 0: truncated (sss.h)
    sorted: Optional[torch.Tensor] = None  # [V][n] i32 depth-sorted visible ids
    n_vis: Optional[torch.Tensor] = None   # [V] i32
    resume: Optional[torch.Tensor] = None  # [V][n_bins] i32
    used: Optional[torch.Tensor] = None    # [V][n_bins] i32: adaptive truncation (sss.h)
    tmask: Optional[torch.Tensor] = None   # [V][capacity] i16: per-entry tile masks (sss.h)

    @classmethod
    def empty(cls, V: int, n_bins: int, capacity: int, bin_shift: int, keys: bool,
              device="cuda", max_per_bin: int = 0, n: int = 0, adaptive: bool = False,
              tile_masks: bool = False) -> "Bins":
        """n: components (needed for the sorted array when truncating).
        adaptive: per-bin caps from the previous forward's consumption (the
        first call, with used = -1, builds complete lists)."""
        cap = max(int(capacity), 1)
        trunc = int(max_per_bin) > 0 or adaptive
        return cls(bin_shift, int(capacity),
                   torch.empty((V, cap), dtype=torch.int32, device=device),
                   torch.empty((V, cap), dtype=torch.int64, device=device) if keys else None,
                   torch.empty((V, n_bins, 2), dtype=torch.int32, device=device),
                   torch.zeros((V,), dtype=torch.int64, device=device),
                   torch.zeros((1,), dtype=torch.int32, device=device),
                   int(max_per_bin),
                   torch.empty((V, max(int(n), 1)), dtype=torch.int32, device=device) if trunc else None,
                   torch.zeros((V,), dtype=torch.int32, device=device) if trunc else None,
                   torch.empty((V, n_bins), dtype=torch.int32, device=device) if trunc else None,
                   torch.full((V, n_bins), -1, dtype=torch.int32, device=device) if adaptive else None,
                   torch.empty((V, cap), dtype=torch.int16, device=device) if tile_masks else None)

    def c(self) -> L.sss_bins:
        return L.sss_bins(self.bin_shift, int(self.totals.shape[0]), self.capacity, _ptr(self.ids),
                          _ptr(self.keys), _ptr(self.ranges), _ptr(self.totals),
                          _ptr(self.overflow), int(self.max_per_bin), 0, _ptr(self.sorted),
                          _ptr(self.n_vis), _ptr(self.resume), _ptr(self.used), _ptr(self.tmask))

    def view(self, nv: int) -> "Bins":
        """The first nv views (shared storage)."""
        return Bins(self.bin_shift, self.capacity, self.ids[:nv],
                    self.keys[:nv] if self.keys is not None else None, self.ranges[:nv],
                    self.totals[:nv], self.overflow, self.max_per_bin,
                    self.sorted[:nv] if self.sorted is not None else None,
                    self.n_vis[:nv] if self.n_vis is not None else None,
                    self.resume[:nv] if self.resume is not None else None,
                    self.used[:nv] if self.used is not None else None,
                    self.tmask[:nv] if self.tmask is not None else None)


TILE_CAP = 3072  # composited entries per 16x8 strip the forward records for the backward (config 5: max 2584;
#                  1536 left 1.1 % of the strips to the slower unlisted replay: +0.6 ms per step)


@dataclass
class Frame:
    rgb: torch.Tensor        # [V][3][H][W] f32
    final_T: torch.Tensor    # [V][H][W] f32
    n_contrib: Optional[torch.Tensor]  # [V][H][W] i32; None = not counted (diagnostic)
    last: torch.Tensor       # [V][H][W] i32
    tile_list: Optional[torch.Tensor] = None   # private [V][tiles][SSS_TILE_LISTS][cap] i32 (None: full replay)
    tile_count: Optional[torch.Tensor] = None  # private [V][tiles][SSS_TILE_LISTS] i32

    @classmethod
    def empty(cls, V: int, H: int, W: int, device="cuda", tile_cap: int = TILE_CAP) -> "Frame":
        tiles = ((W + L.SSS_TILE - 1) // L.SSS_TILE) * ((H + L.SSS_TILE - 1) // L.SSS_TILE)
        tl = tc = None
        if tile_cap > 0:
            tl = torch.empty((V, tiles, L.SSS_TILE_LISTS, tile_cap), dtype=torch.int32, device=device)
            tc = torch.empty((V, tiles, L.SSS_TILE_LISTS), dtype=torch.int32, device=device)
        return cls(torch.empty((V, 3, H, W), dtype=torch.float32, device=device),
                   torch.empty((V, H, W), dtype=torch.float32, device=device),
                   torch.empty((V, H, W), dtype=torch.int32, device=device),
                   torch.empty((V, H, W), dtype=torch.int32, device=device), tl, tc)

    def c(self) -> L.sss_frame:
        cap = int(self.tile_list.shape[-1]) if self.tile_list is not None else 0
        return L.sss_frame(_ptr(self.rgb), _ptr(self.final_T), _ptr(self.n_contrib),
                           _ptr(self.last), _ptr(self.tile_list), _ptr(self.tile_count), cap, 0)


def hparams_c(hp) -> L.sss_sghmc_hparams:
    return L.sss_sghmc_hparams(hp.lr, hp.friction, hp.noise, hp.gate_k, hp.gate_t,
                               int(hp.burn_in), int(hp.g_adam), hp.lr_scale, hp.lr_rot, hp.lr_nu,
                               hp.lr_opacity, hp.lr_sh, hp.beta1, hp.beta2, hp.adam_eps,
                               hp.grad_scale, int(hp.step), int(hp.seed),
                               float(getattr(hp, "eps_o", 0.0)), float(getattr(hp, "eps_sigma", 0.0)),
                               int(getattr(hp, "mu_mode", 0)), int(getattr(hp, "plane_begin", 0)),
                               int(getattr(hp, "plane_end", 0)), 0,
                               _ptr(getattr(hp, "skip_if", None)), _ptr(getattr(hp, "step_state", None)))


# ------------------------------------------------------------- entry points
def sss_project(params: Params, cams: Sequence, out: Optional[Projected] = None,
                stream=None, cams_c=None) -> Projected:
    lib = L.load()
    V = len(cams)
    out = out if out is not None else Projected.empty(params.n, V, params.planes.device)
    cc = cams_c if cams_c is not None else cameras_c(cams)
    p, o = params.c(), out.c()
    L.check(lib.sss_project(C.byref(p), cc, V, C.byref(o), _stream_ptr(stream)), "sss_project")
    return out


def bin_sort_workspace_bytes(n: int, cams: Sequence, bin_shift: int, cams_c=None) -> int:
    lib = L.load()
    cc = cams_c if cams_c is not None else cameras_c(cams)
    return int(lib.sss_bin_sort_workspace(n, len(cams), cc, bin_shift))


def sss_bin_sort(proj: Projected, cams: Sequence, bin_shift: int = 0,
                 capacity: Optional[int] = None, keys: bool = False,
                 ws: Optional[torch.Tensor] = None, out: Optional[Bins] = None, stream=None,
                 cams_c=None, headroom: float = 1.25, max_per_bin: int = 0,
                 tile_masks: bool = False) -> Bins:
    """Bin and depth-sort.  With capacity=None the instance count is measured
    first (one host sync) and the output sized with `headroom`.
    max_per_bin > 0: truncated lists (sss.h sss_bins)."""
    lib = L.load()
    V = len(cams)
    cc = cams_c if cams_c is not None else cameras_c(cams)
    W, H = int(cams[0].width), int(cams[0].height)
    nb = n_bins_of(W, H, bin_shift)
    dev = proj.depth.device
    need = bin_sort_workspace_bytes(proj.n, cams, bin_shift, cams_c=cc)
    if ws is None or ws.numel() < need:
        ws = torch.empty(need, dtype=torch.uint8, device=dev)
    if out is None:
        if capacity is None:
            probe = Bins.empty(V, nb, 0, bin_shift, False, dev, max_per_bin, proj.n)
            pc, prc = probe.c(), proj.c()
            L.check(lib.sss_bin_sort(C.byref(prc), cc, V, _ptr(ws), ws.numel(), C.byref(pc),
                                     _stream_ptr(stream)), "sss_bin_sort(probe)")
            capacity = int(int(probe.totals.max().item()) * headroom) + 1024
        out = Bins.empty(V, nb, capacity, bin_shift, keys, dev, max_per_bin, proj.n, tile_masks=tile_masks)
    bc, prc = out.c(), proj.c()
    L.check(lib.sss_bin_sort(C.byref(prc), cc, V, _ptr(ws), ws.numel(), C.byref(bc),
                             _stream_ptr(stream)), "sss_bin_sort")
    return out


def sss_check_overflow(bins: Bins, stream=None) -> bool:
    lib = L.load()
    b = bins.c()
    st = lib.sss_check_overflow(C.byref(b), _stream_ptr(stream))
    if st == L.SSS_ERR_CAPACITY:
        return True
    L.check(st, "sss_check_overflow")
    return False


def sss_render_fwd(proj: Projected, bins: Bins, cams: Sequence, bg=(0.0, 0.0, 0.0),
                   out: Optional[Frame] = None, stream=None, cams_c=None) -> Frame:
    lib = L.load()
    V = len(cams)
    cc = cams_c if cams_c is not None else cameras_c(cams)
    H, W = int(cams[0].height), int(cams[0].width)
    out = out if out is not None else Frame.empty(V, H, W, proj.depth.device)
    bgc = (C.c_float * 3)(*[float(x) for x in bg])
    prc, bc, fc = proj.c(), bins.c(), out.c()
    L.check(lib.sss_render_fwd(C.byref(prc), C.byref(bc), cc, V, bgc, C.byref(fc),
                               _stream_ptr(stream)), "sss_render_fwd")
    return out


def render_bwd_workspace_bytes(n: int, V: int) -> int:
    return int(L.load().sss_render_bwd_workspace(n, V))


def sss_render_bwd(params: Params, proj: Projected, bins: Bins, cams: Sequence, frame: Frame,
                   bg=(0.0, 0.0, 0.0), d_rgb: Optional[torch.Tensor] = None,
                   target: Optional[torch.Tensor] = None, grad: Optional[Params] = None,
                   loss: Optional[torch.Tensor] = None, ws: Optional[torch.Tensor] = None,
                   nu_grad_paper: bool = False, stream=None, cams_c=None,
                   half: Optional[str] = None, assign: bool = False) -> Params:
    """grad += d(L)/d(params) (assign: grad = d(L)/d(params), the old contents
    unread).  `ws` (zeroed, reusable) holds the screen-space gradient records;
    it is left zero by the call.  half = "raster" / "projection" runs one of
    the two kernels (timing instrumentation)."""
    lib = L.load()
    V = len(cams)
    cc = cams_c if cams_c is not None else cameras_c(cams)
    grad = grad if grad is not None else Params.zeros_like(params)
    need = render_bwd_workspace_bytes(params.n, V)
    if ws is None:
        ws = torch.zeros(max(need, 4), dtype=torch.uint8, device=params.planes.device)
    assert ws.numel() >= need
    if d_rgb is not None:
        assert d_rgb.is_contiguous() and d_rgb.dtype == torch.float32
    if target is not None:  # fp32, or uint8 images (value u / 255, sss.h SSS_BWD_TARGET_U8)
        assert target.is_contiguous() and target.dtype in (torch.float32, torch.uint8)
    bgc = (C.c_float * 3)(*[float(x) for x in bg])
    pc, prc, bc, fc, gc = params.c(), proj.c(), bins.c(), frame.c(), grad.c()
    flags = (L.SSS_BWD_NU_GRAD_PAPER if nu_grad_paper else 0) | (L.SSS_BWD_GRAD_ASSIGN if assign else 0)
    if target is not None and target.dtype == torch.uint8:
        flags |= L.SSS_BWD_TARGET_U8
    if half == "raster":
        flags |= L.SSS_BWD_RASTER_ONLY
    elif half == "projection":
        flags |= L.SSS_BWD_PROJECTION_ONLY
    L.check(lib.sss_render_bwd(C.byref(pc), C.byref(prc), C.byref(bc), cc, V, bgc, C.byref(fc),
                               _ptr(d_rgb), _ptr(target), _ptr(loss), C.byref(gc), _ptr(ws),
                               ws.numel(), flags, _stream_ptr(stream)), "sss_render_bwd")
    return grad


def sss_project_bwd_range(params: Params, cams: Sequence, ws: torch.Tensor, grad, i0: int, i1: int,
                          stream=None, cams_c=None) -> None:
    """The projection backward (a5) for components [i0, i1) only (sss.h):
    consumes the screen-space records a raster-only sss_render_bwd left in
    ws; grad is a Params or BlockedParams."""
    lib = L.load()
    cc = cams_c if cams_c is not None else cameras_c(cams)
    pc, gc = params.c(), grad.c()
    L.check(lib.sss_project_bwd_range(C.byref(pc), cc, len(cams), _ptr(ws), ws.numel(), C.byref(gc),
                                      int(i0), int(i1), _stream_ptr(stream)), "sss_project_bwd_range")


def image_loss_workspace_bytes(V: int, H: int, W: int) -> int:
    return int(L.load().sss_image_loss_workspace(V, H, W))


def sss_image_loss(rgb: torch.Tensor, target: torch.Tensor, eps_dssim: float,
                   d_rgb: Optional[torch.Tensor] = None, loss: Optional[torch.Tensor] = None,
                   ws: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """Image part of Eq. 8 for [V][3][H][W] renders: writes dL/dC into d_rgb
    (returned) and adds sum_v L_v to `loss` (device float[1]) if given."""
    lib = L.load()
    assert rgb.shape == target.shape and rgb.dim() == 4 and rgb.shape[1] == 3
    for t in (rgb, target):
        assert t.is_contiguous() and t.dtype == torch.float32
    V, _, H, W = rgb.shape
    d_rgb = d_rgb if d_rgb is not None else torch.empty_like(rgb)
    need = image_loss_workspace_bytes(V, H, W)
    if ws is None:
        ws = torch.empty(max(need, 4), dtype=torch.uint8, device=rgb.device)
    L.check(lib.sss_image_loss(_ptr(rgb), _ptr(target), V, H, W, float(eps_dssim), _ptr(d_rgb),
                               _ptr(loss), _ptr(ws), ws.numel(), _stream_ptr(stream)),
            "sss_image_loss")
    return d_rgb


def relocate_workspace_bytes(n: int) -> int:
    return int(L.load().sss_relocate_workspace(n))


def sss_relocate(params: Params, adam_m: Params, adam_v: Params, momentum: torch.Tensor,
                 threshold: float = 0.005, cap_frac: float = 0.05, n_max: int = 32, seed: int = 0,
                 step: int = 1, target_of: Optional[torch.Tensor] = None,
                 n_moved: Optional[torch.Tensor] = None, ws: Optional[torch.Tensor] = None,
                 stream=None) -> torch.Tensor:
    """One recycling pass in place (NEXT-2); returns the device int64[1]
    count of relocated components (no host sync)."""
    lib = L.load()
    dev = params.planes.device
    n_moved = n_moved if n_moved is not None else torch.zeros(1, dtype=torch.int64, device=dev)
    need = relocate_workspace_bytes(params.n)
    if ws is None:
        ws = torch.empty(max(need, 4), dtype=torch.uint8, device=dev)
    rp = L.sss_relocate_params(float(threshold), float(cap_frac), int(n_max), 0, int(seed), int(step))
    pc, mc, vc = params.c(), adam_m.c(), adam_v.c()
    L.check(lib.sss_relocate(C.byref(pc), C.byref(mc), C.byref(vc), _ptr(momentum), C.byref(rp),
                             _ptr(target_of), _ptr(n_moved), _ptr(ws), ws.numel(),
                             _stream_ptr(stream)), "sss_relocate")
    return n_moved


def grow(planes: torch.Tensor, sh_degree: int, frac: float = 0.05) -> torch.Tensor:
    """Adds floor(frac * n) components with zero opacity ("we
    add 5% new components with zero opacity and then recycle them"): a new
    flat [P][n'] buffer whose new columns are identity rotations with
    raw_opacity 0, i.e. dead for the next sss_relocate pass.  Host-side
    memory management only (no method arithmetic)."""
    P, n = planes.shape
    add = int(frac * n)
    extra = torch.zeros((P, add), dtype=planes.dtype, device=planes.device)
    extra[6] = 1.0  # quaternion w
    return torch.cat([planes, extra], dim=1).contiguous()


def step_state(first_step: int, device="cuda") -> torch.Tensor:
    """A device sss_step_state (sss.h) starting at `first_step`: set it as
    hp.step_state to make sss_sghmc_step graph-capturable."""
    t = torch.zeros(4, dtype=torch.int64, device=device)  # 32 bytes
    t[0] = int(first_step)
    return t


def sss_sghmc_step(params: Params, grad: Params, adam_m: Params, adam_v: Params,
                   momentum: torch.Tensor, hp, stream=None) -> None:
    lib = L.load()
    h = hparams_c(hp)
    pc, gc, mc, vc = params.c(), grad.c(), adam_m.c(), adam_v.c()
    L.check(lib.sss_sghmc_step(C.byref(pc), C.byref(gc), C.byref(mc), C.byref(vc),
                               _ptr(momentum), C.byref(h), _stream_ptr(stream)),
            "sss_sghmc_step")


def launch_count(reset: bool = False) -> int:
    return int(L.load().sss_launch_count(1 if reset else 0))
