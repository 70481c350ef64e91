"""Device gradient cache for one image subset and the products on it.

`CacheSet` is the B200 counterpart of the reference's per-view
`GradientCache` (ref: jacobian.py:46-84) generalised to the multi-view batch
that PCG sums over.  Building it runs, per view: fp64 projection,
(depth, gid) sort, tile binning, COUNT raster pass (+ per (tile instance,
pixel row) entry counts), residual weights; then per subset: pixel offsets and
(view, gaussian) pairs; then per view: row-major run offsets and the FILL
raster pass, which writes BOTH record streams -- pixel order and gaussian
order (sortCacheByGaussians) -- without any sort.

Everything here is host orchestration of libsplatlm_b200 kernels on the
current torch stream; torch only allocates memory.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import call, ptr, stream_ptr
from .errors import ImageSizeError
from .scene import Camera, GaussianScene, cameras_struct_tensor, num_coefficients

TILE = 16
CHUNK = 128


@dataclass(frozen=True)
class LossConfig:
    """Residual settings of compute_residuals (ref: residuals.py:249-252)."""
    lambda1: float = 0.8
    lambda2: float = 0.2
    mode: str = "l1ssim"
    window: int = 11
    sigma: float = 1.5
    eps_den: float = 1e-8


def rast_cfg_struct(cfg, background) -> _lib.SlmRastCfg:
    s = _lib.SlmRastCfg()
    s.alpha_min, s.t_stop, s.alpha_clamp = float(cfg.alpha_min), float(cfg.t_stop), float(cfg.alpha_clamp)
    s.cov_eps, s.z_near = float(cfg.cov_eps), float(cfg.z_near)
    s.cull_sigma = float(cfg.cull_sigma) if cfg.cull_sigma is not None else -1.0
    # same expression as ref: rasterizer.py:275-279
    s.reach_fac = float(np.sqrt(np.maximum(0.0, 2.0 * np.log(1.0 / cfg.alpha_min)))) if cfg.alpha_min > 0 else -1.0
    for i in range(3):
        s.bg[i] = float(background[i])
    return s


def _bits(n: int) -> int:
    return max(1, int(n - 1).bit_length()) if n > 1 else 1


def _empty(n, dtype, dev):
    return torch.empty(max(int(n), 1), dtype=dtype, device=dev)


def scan_i64(inp: torch.Tensor, out: torch.Tensor):
    n = inp.numel()
    ws = _empty(_lib.load().slm_scan_i64_workspace(n), torch.uint8, inp.device)
    call("slm_scan_i64", ptr(ws), ws.numel(), ptr(inp), ptr(out), n, stream_ptr())


def scan_i32(inp: torch.Tensor, out: torch.Tensor):
    n = inp.numel()
    ws = _empty(_lib.load().slm_scan_i32_workspace(n), torch.uint8, inp.device)
    call("slm_scan_i32", ptr(ws), ws.numel(), ptr(inp), ptr(out), n, stream_ptr())


def sort_u64(kin, kout, vin, vout, n, begin_bit, end_bit):
    ws = _empty(_lib.load().slm_sort_pairs_u64_workspace(n), torch.uint8, kin.device)
    call("slm_sort_pairs_u64", ptr(ws), ws.numel(), ptr(kin), ptr(kout), ptr(vin), ptr(vout), n, begin_bit,
         end_bit, stream_ptr())


def sort_u32(kin, kout, vin, vout, n, begin_bit, end_bit):
    ws = _empty(_lib.load().slm_sort_pairs_u32_workspace(n), torch.uint8, kin.device)
    call("slm_sort_pairs_u32", ptr(ws), ws.numel(), ptr(kin), ptr(kout), ptr(vin), ptr(vout), n, begin_bit,
         end_bit, stream_ptr())


def ssim_host_tables(H, W, window, sigma):
    """Taps and center self weights exactly as ref: residuals.py:49-91."""
    off = np.arange(window) - window // 2
    k = np.exp(-0.5 * (off / sigma) ** 2)
    k = k / k.sum()
    half = window // 2

    def cw(n):
        pos = np.arange(n)
        acc = np.zeros(n)
        for tap, w in zip(range(-half, half + 1), k):
            i = pos + tap
            i = np.where(i < 0, -i - 1, i)
            i = np.where(i >= n, 2 * n - i - 1, i)
            acc += w * (i == pos)
        return acc
    return k, cw(H), cw(W)


class PhaseTimer:
    """CUDA-event phase accounting on the current stream: tick(name) charges the
    time since the previous tick to `name`."""

    def __init__(self):
        self.events = []

    def tick(self, name):
        e = torch.cuda.Event(enable_timing=True)
        e.record(torch.cuda.current_stream())
        self.events.append((name, e))

    def summary(self) -> dict:
        torch.cuda.synchronize()
        out = {}
        for (_, a), (name, b) in zip(self.events, self.events[1:]):
            out[name] = out.get(name, 0.0) + a.elapsed_time(b)
        return out


class _NoTimer:
    def tick(self, name):
        pass


class ViewFrame:
    """Per-view products of the COUNT phase (splats, tile lists, image)."""

    def __init__(self, cam: Camera, pix_base: int):
        self.cam = cam
        self.pix_base = pix_base
        self.splats = None       # uint8 [G*96]
        self.inst_gid = None     # int32 [n_inst]
        self.ranges = None       # int32 [2*n_tiles]
        self.rgb = None          # float64 [HW*3]
        self.t_final = None      # float64 [HW]
        self.tiles_x = (cam.width + TILE - 1) // TILE
        self.tiles_y = (cam.height + TILE - 1) // TILE
        self.n_inst = 0
        self.energy_part = None
        self.sorted_gid = None   # int32 [G] depth order
        self.inst_off = None     # int64 [G+1] instances per depth rank (pre-sort order)
        self.post_of_pre = None  # int32 [n_inst]
        self.rowcnt = None       # uint8 [n_inst*16] entries per (instance, pixel row)


def project_and_bin(scene: GaussianScene, frame: ViewFrame, cfg_s: _lib.SlmRastCfg, err: torch.Tensor,
                    depth_only: bool = False):
    """fp64 projection + (depth, gid) order + tile binning for one view."""
    dev = scene.device
    G = scene.num_gaussians
    cam_s = frame.cam.to_struct(frame.pix_base)
    splats = torch.empty(G * _lib.SPLAT_BYTES, dtype=torch.uint8, device=dev)
    keys = torch.empty(G, dtype=torch.int64, device=dev)
    vals = torch.empty(G, dtype=torch.int32, device=dev)
    call("slm_preprocess", ptr(scene.x), G, scene.sh_degree, _lib.byref(cam_s), _lib.byref(cfg_s), ptr(splats),
         ptr(keys), ptr(vals), ptr(err), stream_ptr())
    frame.splats = splats
    skeys = torch.empty_like(keys)
    sgid = torch.empty_like(vals)
    sort_u64(keys, skeys, vals, sgid, G, 0, 64)
    if depth_only:
        return skeys, sgid
    n_inst = torch.zeros(G + 1, dtype=torch.int64, device=dev)
    call("slm_tile_count", ptr(sgid), ptr(skeys), G, ptr(splats), frame.tiles_x, frame.tiles_y, ptr(n_inst),
         stream_ptr())
    inst_off = torch.empty_like(n_inst)
    scan_i64(n_inst, inst_off)
    total = int(inst_off[G].item())
    frame.n_inst = total
    n_tiles = frame.tiles_x * frame.tiles_y
    rank_bits = _bits(G)
    tile_bits = _bits(n_tiles)
    ik = _empty(total, torch.int64, dev)
    iv = _empty(total, torch.int32, dev)
    ig = _empty(total, torch.int32, dev)
    call("slm_tile_emit", ptr(sgid), ptr(inst_off), G, ptr(splats), frame.tiles_x, frame.tiles_y, rank_bits,
         ptr(ik), ptr(iv), ptr(ig), stream_ptr())
    sk = torch.empty_like(ik)
    sv = torch.empty_like(iv)
    sort_u64(ik, sk, iv, sv, total, 0, rank_bits + tile_bits)
    ranges = torch.empty(2 * n_tiles, dtype=torch.int32, device=dev)
    call("slm_tile_ranges", ptr(sk), total, rank_bits, ptr(ranges), n_tiles, stream_ptr())
    inst_gid = _empty(total, torch.int32, dev)
    post_of_pre = _empty(total, torch.int32, dev)
    call("slm_tile_post", ptr(sv), ptr(ig), total, ptr(inst_gid), ptr(post_of_pre), stream_ptr())
    frame.inst_gid = inst_gid
    frame.ranges = ranges
    frame.sorted_gid = sgid
    frame.inst_off = inst_off
    frame.post_of_pre = post_of_pre
    return skeys, sgid


def inst_base(scene: GaussianScene, frame: ViewFrame, pair_cnt=None, base_out=None):
    """Per-(view, gaussian) entry counts and/or the row-major run offsets of
    each (tile instance, pixel row) inside its gaussian-order pair block."""
    call("slm_inst_base", ptr(frame.sorted_gid), ptr(frame.inst_off), scene.num_gaussians, ptr(frame.splats),
         frame.tiles_x, frame.tiles_y, ptr(frame.post_of_pre), ptr(frame.rowcnt), ptr(base_out), ptr(pair_cnt),
         stream_ptr())


def raster_args(frame: ViewFrame, cfg_s) -> _lib.SlmRasterArgs:
    a = _lib.SlmRasterArgs()
    a.tile_range = ptr(frame.ranges)
    a.inst_gid = ptr(frame.inst_gid)
    a.splats = ptr(frame.splats)
    a.W, a.H, a.tiles_x = frame.cam.width, frame.cam.height, frame.tiles_x
    a.pix_base = frame.pix_base
    a.cfg = cfg_s
    return a


def residual_pass(frame: ViewFrame, gt: torch.Tensor, loss: LossConfig, gradr: torch.Tensor,
                  cgrad: torch.Tensor, exports: dict | None = None):
    """Residual weights of one view into gradr/cgrad (float4 per pixel)."""
    cam = frame.cam
    H, W = cam.height, cam.width
    if tuple(gt.shape) != (H, W, 3):
        raise ImageSizeError(f"image shapes differ: {(H, W, 3)} vs {tuple(gt.shape)}")
    if loss.mode not in ("l1ssim", "l2"):
        raise ValueError(f"unknown loss mode {loss.mode!r}")
    if loss.mode == "l1ssim" and (loss.lambda1 < 0 or loss.lambda2 < 0):
        raise ValueError("loss weights must be >= 0")
    dev = gt.device
    gt = gt.contiguous()
    taps, cwy, cwx = ssim_host_tables(H, W, loss.window, loss.sigma)
    taps_t = torch.from_numpy(taps).to(dev)
    cwy_t = torch.from_numpy(cwy).to(dev)
    cwx_t = torch.from_numpy(cwx).to(dev)
    need_ssim = loss.mode == "l1ssim" and loss.lambda2 > 0
    tmp = _empty(H * W * 15 if need_ssim else 1, torch.float64, dev)
    blocks = int(min(max((H * W + 255) // 256, 1), 148 * 8))
    part = torch.empty(blocks, dtype=torch.float64, device=dev)
    a = _lib.SlmResidArgs()
    a.img = ptr(frame.rgb)
    a.gt = ptr(gt)
    a.gt_f32 = 1 if gt.dtype == torch.float32 else 0
    if gt.dtype not in (torch.float32, torch.float64):
        raise ValueError("ground truth must be float32 or float64")
    a.W, a.H = W, H
    a.lambda1, a.lambda2, a.eps_den = float(loss.lambda1), float(loss.lambda2), float(loss.eps_den)
    a.ssim_c1, a.ssim_c2 = 0.01 ** 2, 0.03 ** 2
    a.mode = 0 if loss.mode == "l1ssim" else 1
    a.win = int(loss.window)
    a.taps, a.cw_y, a.cw_x, a.tmp = ptr(taps_t), ptr(cwy_t), ptr(cwx_t), ptr(tmp)
    a.gradr = C.c_void_p(gradr.data_ptr() + frame.pix_base * 16)
    a.cgrad = C.c_void_p(cgrad.data_ptr() + frame.pix_base * 16)
    a.energy_part = ptr(part)
    if exports is not None:
        for k in ("gradr", "cgrad", "rabs", "rssim", "drabs", "drssim"):
            exports[k] = torch.empty(H * W * 3, dtype=torch.float64, device=dev)
        a.o_gradr, a.o_cgrad = ptr(exports["gradr"]), ptr(exports["cgrad"])
        a.o_rabs, a.o_drabs = ptr(exports["rabs"]), ptr(exports["drabs"])
        a.o_rssim, a.o_drssim = ptr(exports["rssim"]), ptr(exports["drssim"])
    call("slm_residuals", _lib.byref(a), blocks, stream_ptr())
    frame.energy_part = part
    keep = (taps_t, cwy_t, cwx_t, tmp)  # noqa: F841 -- alive until the kernels are queued
    return part


class CacheSet:
    """Gradient cache of one image subset on the device (both record orders).

    Args:
        scene: scene at the current parameters.
        cameras: the subset's views.
        gts: ground-truth images (H, W, 3) float64/float32 device tensors; when
            None the cache is built without residual weights (products only).
        config: RenderConfig.
        loss: LossConfig.
        keep_source_index: also keep the gaussian-order -> pixel-order
            permutation (the reference's source_index) for parity exports.
    """

    def __init__(self, scene: GaussianScene, cameras: list[Camera], gts=None, config=None, loss=LossConfig(),
                 keep_source_index: bool = False, residual_exports: bool = False, weights=None, timer=None):
        from .rasterizer import DEFAULT_CONFIG
        self.scene = scene
        self.config = config if config is not None else DEFAULT_CONFIG
        self.loss = loss
        self.cameras = list(cameras)
        if not self.cameras:
            raise ValueError("a cache needs at least one view")
        dev = scene.device
        self.device = dev
        G = scene.num_gaussians
        V = len(self.cameras)
        self.G, self.V = G, V
        self.P = scene.params_per_gaussian
        self.K = num_coefficients(scene.sh_degree)
        self.cams_dev, self.pix_bases = cameras_struct_tensor(self.cameras, dev)
        self.N = sum(c.num_pixels for c in self.cameras)
        views = (_lib.SlmView * V)()
        for i, c in enumerate(self.cameras):
            views[i].pix_base, views[i].W, views[i].H = self.pix_bases[i], c.width, c.height
        self.views_dev = torch.frombuffer(bytearray(bytes(C.string_at(C.addressof(views), C.sizeof(views)))),
                                          dtype=torch.uint8).to(dev)
        cfg_s = rast_cfg_struct(self.config, scene.background)
        self.cfg_s = cfg_s
        err = torch.zeros(1, dtype=torch.int32, device=dev)
        T = timer if timer is not None else _NoTimer()
        T.tick("start")

        # ---- COUNT phase (per view) --------------------------------------
        self.px_count = torch.zeros(self.N + 1, dtype=torch.int32, device=dev)
        self.pair_cnt = torch.zeros(V * G, dtype=torch.int32, device=dev)
        have_res = gts is not None
        have_w = have_res or weights is not None
        self.gradr = torch.zeros(self.N * 4, dtype=torch.float32, device=dev) if have_w else None
        self.cgrad = torch.zeros(self.N * 4, dtype=torch.float32, device=dev) if have_w else None
        if weights is not None:  # precomputed ResidualBundles (build_cache API)
            for v, (g4, c4) in enumerate(weights):
                b0 = self.pix_bases[v] * 4
                self.gradr[b0:b0 + g4.numel()].copy_(g4)
                self.cgrad[b0:b0 + c4.numel()].copy_(c4)
        self.frames: list[ViewFrame] = []
        self.residual_exports = [] if residual_exports else None
        energy_parts = []
        for v, cam in enumerate(self.cameras):
            fr = ViewFrame(cam, self.pix_bases[v])
            project_and_bin(scene, fr, cfg_s, err)
            T.tick("project_sort_bin")
            hw = cam.num_pixels
            fr.rgb = torch.empty(hw * 3, dtype=torch.float64, device=dev)
            fr.t_final = torch.empty(hw, dtype=torch.float64, device=dev)
            fr.rowcnt = torch.zeros(max(fr.n_inst, 1) * TILE, dtype=torch.uint8, device=dev)
            a = raster_args(fr, cfg_s)
            a.px_count = C.c_void_p(self.px_count.data_ptr() + fr.pix_base * 4)
            a.rgb, a.t_final, a.rowcnt = ptr(fr.rgb), ptr(fr.t_final), ptr(fr.rowcnt)
            call("slm_raster_count", _lib.byref(a), stream_ptr())
            inst_base(scene, fr, pair_cnt=self.pair_cnt[v * G:(v + 1) * G])
            T.tick("raster_count")
            if have_res:
                ex = {} if residual_exports else None
                energy_parts.append(residual_pass(fr, gts[v], loss, self.gradr, self.cgrad, ex))
                if residual_exports:
                    self.residual_exports.append(ex)
                T.tick("residuals")
            self.frames.append(fr)
        e = int(err.item())
        if e & 1:
            raise ValueError("scene contains non-finite parameters")
        if e & 2:
            raise ValueError("quaternion with (near-)zero norm")
        self.energies = [float(p.sum().item()) for p in energy_parts] if have_res else None

        # ---- pixel segments ----------------------------------------------
        N = self.N
        cnt64 = torch.empty(N + 1, dtype=torch.int64, device=dev)
        nonempty = torch.empty(N + 1, dtype=torch.int32, device=dev)
        call("slm_px_prepare", ptr(self.px_count), N + 1, ptr(cnt64), ptr(nonempty), stream_ptr())
        self.pix_off = torch.empty(N + 1, dtype=torch.int64, device=dev)
        scan_i64(cnt64, self.pix_off)
        seg_idx = torch.empty(N + 1, dtype=torch.int32, device=dev)
        scan_i32(nonempty, seg_idx)
        bases = torch.tensor(self.pix_bases + [N], dtype=torch.int64, device=dev)
        view_off = self.pix_off[bases].cpu().tolist()
        self.E = int(view_off[-1])
        self.view_entry_base = view_off
        self.n_seg = int(seg_idx[N].item())
        self.seg_info = _empty(self.n_seg * 2, torch.int32, dev)
        call("slm_px_segments", ptr(self.px_count), ptr(seg_idx), N, ptr(self.cams_dev), V, ptr(self.seg_info),
             stream_ptr())
        del cnt64, nonempty

        # ---- pairs -----------------------------------------------------------
        VG = V * G
        cntV = torch.zeros(VG + 1, dtype=torch.int64, device=dev)
        flagV = torch.zeros(VG + 1, dtype=torch.int32, device=dev)
        flagT = torch.zeros(VG + 1, dtype=torch.int32, device=dev)
        call("slm_pairs_prepare", ptr(self.pair_cnt), V, G, ptr(cntV), ptr(flagV), ptr(flagT), stream_ptr())
        vscan = torch.empty_like(cntV)
        scan_i64(cntV, vscan)
        pair_of = torch.empty_like(flagV)
        scan_i32(flagV, pair_of)
        tscan = torch.empty_like(flagT)
        scan_i32(flagT, tscan)
        self.n_pairs = int(pair_of[VG].item())
        if int(vscan[VG].item()) != self.E:
            raise RuntimeError("cache entry count mismatch between pixel and pair counts")
        Pn = self.n_pairs
        self.pair_off = torch.empty(Pn + 1, dtype=torch.int64, device=dev)
        self.pair_gid = _empty(Pn, torch.int32, dev)
        self.pair_vm = _empty(Pn, torch.int32, dev)
        self.pair_geo = _empty(Pn * _lib.PAIR_GEO_BYTES, torch.uint8, dev)
        pidx = torch.empty(VG, dtype=torch.int32, device=dev)
        self.gpo = torch.empty(G + 1, dtype=torch.int32, device=dev)
        self.gp_list = _empty(Pn, torch.int32, dev)
        splats_all = torch.cat([f.splats for f in self.frames])
        call("slm_pairs_emit", ptr(self.pair_cnt), V, G, ptr(pair_of), ptr(vscan), ptr(tscan), ptr(splats_all),
             ptr(self.pair_off), ptr(self.pair_gid), ptr(self.pair_vm), ptr(self.pair_geo), ptr(pidx), ptr(self.gpo),
             ptr(self.gp_list), Pn, self.E, stream_ptr())
        # first pair of each view (pairs are view-major)
        self.view_pair_base = [int(x) for x in pair_of[torch.tensor([v * G for v in range(V)] + [VG],
                                                                     device=dev)].cpu().tolist()]
        del cntV, flagV, flagT, vscan, pair_of, tscan, splats_all

        T.tick("segments_pairs")
        # ---- FILL phase: pixel-order records, then gaussian order ------------
        E = self.E
        n_chunks = (E + CHUNK - 1) // CHUNK
        self.n_chunks = n_chunks
        f32 = torch.float32

        def stream6():
            return ([_empty(E, torch.int32, dev)] + [_empty(E, f32, dev) for _ in range(5)])
        self.pix_rec = stream6()
        self.gau_rec = stream6()
        self.chunk_seg_pix = _empty(n_chunks, torch.int32, dev)
        self.chunk_seg_gau = _empty(n_chunks, torch.int32, dev)
        self.g_src = _empty(E, torch.int32, dev) if keep_source_index else None
        for v, fr in enumerate(self.frames):
            e0 = view_off[v]
            base = _empty(fr.n_inst * TILE, torch.int32, dev)
            inst_base(scene, fr, base_out=base)
            T.tick("gauss_order")
            a = raster_args(fr, cfg_s)
            a.rgb = ptr(fr.rgb)
            a.pix_off, a.pidx, a.seg_idx = ptr(self.pix_off), C.c_void_p(pidx.data_ptr() + v * G * 4), ptr(seg_idx)
            a.pair_off, a.inst_base = ptr(self.pair_off), ptr(base)
            (a.rec_idx, a.rec_ae, a.rec_at, a.rec_d0, a.rec_d1, a.rec_d2) = [ptr(t) for t in self.pix_rec]
            a.chunk_seg = ptr(self.chunk_seg_pix)
            (a.g_idx, a.g_ae, a.g_at, a.g_d0, a.g_d1, a.g_d2) = [ptr(t) for t in self.gau_rec]
            a.g_chunk_seg = ptr(self.chunk_seg_gau)
            a.g_src = ptr(self.g_src) if self.g_src is not None else None
            a.view_entry_base = e0
            call("slm_raster_fill", _lib.byref(a), stream_ptr())
            T.tick("raster_fill")
            del base
        del pidx, seg_idx
        for fr in self.frames:  # keep images for exports; tile lists are not needed any more
            fr.inst_gid = fr.ranges = fr.rowcnt = fr.post_of_pre = fr.inst_off = fr.sorted_gid = None
        # product scratch
        self.u = torch.empty(self.N * 4, dtype=f32, device=dev)
        self.pm = _empty(Pn * 12, f32, dev)
        self.pacc = _empty(Pn * 9, f32, dev)
        self._carry = {}
        self._b = None
        self._M = None

    # ------------------------------------------------------------------
    @property
    def nbytes(self) -> int:
        """Bytes of both record streams (budget accounting, ref: jacobian.py:76-80)."""
        return 2 * 24 * self.E

    def _carries(self, D):
        if D not in self._carry:
            nb = _lib.load().slm_carry_bytes(D) * max(self.n_chunks, 1)
            self._carry[D] = (torch.empty(nb, dtype=torch.uint8, device=self.device),
                              torch.empty(nb, dtype=torch.uint8, device=self.device))
        return self._carry[D]

    def _stream(self, which: str, D: int) -> _lib.SlmWsrStream:
        rec = self.pix_rec if which == "pixel" else self.gau_rec
        s = _lib.SlmWsrStream()
        s.idx, s.ae, s.at, s.d0, s.d1, s.d2 = [ptr(t) for t in rec]
        s.E = self.E
        s.chunk_seg = ptr(self.chunk_seg_pix if which == "pixel" else self.chunk_seg_gau)
        h, t = self._carries(D)
        s.head, s.tail = ptr(h), ptr(t)
        return s

    def pair_forward(self, p: torch.Tensor, gaussian_major: bool = False):
        G, P = self.G, self.P
        sa, sg = (1, P) if gaussian_major else (G, 1)
        call("slm_pair_forward", ptr(self.scene.x32()), G, self.scene.sh_degree, ptr(self.pair_gid),
             ptr(self.pair_vm), ptr(self.cams_dev), self.n_pairs, ptr(p), sa, sg, ptr(self.pm), stream_ptr())

    def apply_j_raw(self, weighted: bool) -> torch.Tensor:
        """u (or u_hat) into self.u from the pair forward chain in self.pm."""
        if weighted and self.gradr is None:
            raise ValueError("cache was built without residual weights")
        s = self._stream("pixel", 3)
        call("slm_apply_j", _lib.byref(s), ptr(self.seg_info), ptr(self.pair_geo), ptr(self.pm),
             ptr(self.gradr) if weighted else None, ptr(self.u), stream_ptr())
        return self.u

    def apply_jt_raw(self, u: torch.Tensor, out: torch.Tensor, scale: float = 1.0, p=None, M=None, lam=0.0,
                     dot_part=None):
        s = self._stream("gaussian", 9)
        call("slm_apply_jt_pairs", _lib.byref(s), ptr(self.pair_geo), ptr(self.pair_vm), ptr(self.views_dev), ptr(u),
             ptr(self.pacc), stream_ptr())
        call("slm_pair_backward", ptr(self.scene.x32()), self.G, self.scene.sh_degree, ptr(self.gpo), ptr(self.gp_list),
             ptr(self.pair_vm), ptr(self.cams_dev), ptr(self.pacc), 0, float(scale), ptr(p), ptr(M), float(lam),
             ptr(out), ptr(dot_part), stream_ptr())
        return out

    def jtwj(self, p: torch.Tensor, out: torch.Tensor, lam: float = 0.0, M=None, dot_part=None):
        """out = J^T W J p (+ lam * max(M, 1e-12) * p); attribute-major fp32."""
        self.pair_forward(p)
        self.apply_j_raw(weighted=True)
        return self.apply_jt_raw(self.u, out, 1.0, p, M if lam != 0.0 else None, lam, dot_part)

    def rhs(self) -> torch.Tensor:
        """b = -J^T color_grad, summed over the subset's views (ref: jacobian.py:411-413)."""
        if self._b is None:
            if self.cgrad is None:
                raise ValueError("cache was built without residuals")
            b = torch.empty(self.G * self.P, dtype=torch.float32, device=self.device)
            self.apply_jt_raw(self.cgrad, b, -1.0)
            self._b = b
        return self._b

    def diag(self) -> torch.Tensor:
        """M = diag(J^T W J), attribute-major (ref: jacobian.py:486-512)."""
        if self._M is None:
            if self.gradr is None:
                raise ValueError("cache was built without residual weights")
            mom = _empty(self.n_pairs * _lib.DIAG_D, torch.float32, self.device)
            s = self._stream("gaussian", _lib.DIAG_D)
            call("slm_diag_pairs", _lib.byref(s), ptr(self.pair_geo), ptr(self.pair_vm), ptr(self.views_dev),
                 ptr(self.gradr), ptr(mom), stream_ptr())
            M = torch.empty(self.G * self.P, dtype=torch.float32, device=self.device)
            call("slm_pair_backward", ptr(self.scene.x32()), self.G, self.scene.sh_degree, ptr(self.gpo), ptr(self.gp_list),
                 ptr(self.pair_vm), ptr(self.cams_dev), ptr(mom), 1, 1.0, None, None, 0.0, ptr(M), None,
                 stream_ptr())
            del self._carry[_lib.DIAG_D]
            self._M = M
        return self._M

    # ------------------------------------------------------------------
    # parity exports (test infrastructure; host copies)
    # ------------------------------------------------------------------
    def image(self, v: int) -> torch.Tensor:
        c = self.cameras[v]
        return self.frames[v].rgb.view(c.height, c.width, 3)

    def export_view(self, v: int) -> dict:
        """Reference-shaped arrays of view v (pixel-sorted cache fields plus
        the gaussian-order sequence of the same view)."""
        cam = self.cameras[v]
        e0, e1 = self.view_entry_base[v], self.view_entry_base[v + 1]
        pr = [t[e0:e1].cpu() for t in self.pix_rec]
        idx = pr[0].numpy().view(np.uint32)
        pair = (idx & 0x7FFFFFFF).astype(np.int64)
        pair_gid = self.pair_gid[: self.n_pairs].cpu().numpy()
        pair_vm = self.pair_vm[: self.n_pairs].cpu().numpy().view(np.uint32)
        gid = pair_gid[pair] if pair.size else np.zeros(0, np.int64)
        b0 = self.pix_bases[v]
        pix_off = self.pix_off[b0:b0 + cam.num_pixels + 1].cpu().numpy() - e0
        counts = np.diff(pix_off)
        pixel = np.repeat(np.arange(cam.num_pixels), counts)
        ae = pr[1].numpy().astype(np.float64)
        at = pr[2].numpy().astype(np.float64)
        alpha = np.where(ae == 0.0, self.config.alpha_clamp, ae)
        T = at / alpha
        dcda = np.stack([pr[3].numpy(), pr[4].numpy(), pr[5].numpy()], 1).astype(np.float64)
        out = dict(pixel_ids=pixel, gaussian_ids=gid.astype(np.int64), alphas=alpha, alpha_eff=ae,
                   transmittances=T, dc_dalpha=dcda, dc_dcs=at, offsets=pix_off, head=(idx >> 31).astype(bool))
        # gaussian order of this view: its pairs' blocks in pair (= gid) order
        pv = np.arange(self.view_pair_base[v], self.view_pair_base[v + 1])   # pairs are view-major
        assert np.all((pair_vm[pv] & 0xFFFF) == v)
        poff = self.pair_off[: self.n_pairs + 1].cpu().numpy()
        sel = np.arange(poff[pv[0]], poff[pv[-1] + 1]) if pv.size else np.zeros(0, np.int64)
        selt = torch.from_numpy(sel).to(self.device)
        gr = [t[selt].cpu().numpy() for t in self.gau_rec] if sel.size else [np.zeros(0)] * 6
        gidx = gr[0].view(np.uint32) if sel.size else np.zeros(0, np.uint32)
        gx = (gidx & 0xFFFF).astype(np.int64)
        gy = ((gidx >> 16) & 0x7FFF).astype(np.int64)
        g_gid = np.repeat(pair_gid[pv], np.diff(poff)[pv]) if pv.size else np.zeros(0, np.int64)
        goff = np.zeros(self.G + 1, np.int64)
        np.add.at(goff, pair_gid[pv] + 1, np.diff(poff)[pv])
        out.update(g_pixel_ids=gy * cam.width + gx, g_gaussian_ids=g_gid, g_offsets=np.cumsum(goff),
                   g_alpha_eff=gr[1].astype(np.float64) if sel.size else np.zeros(0),
                   g_dc_dcs=gr[2].astype(np.float64) if sel.size else np.zeros(0),
                   g_dc_dalpha=np.stack(gr[3:6], 1).astype(np.float64) if sel.size else np.zeros((0, 3)),
                   g_head=(gidx >> 31).astype(bool))
        if self.g_src is not None and sel.size:
            out["g_source_index"] = self.g_src[selt].cpu().numpy().astype(np.int64)
        return out
