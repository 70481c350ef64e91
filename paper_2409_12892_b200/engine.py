"""Device gradient cache for one image subset and the products on it.

`CacheSet` is the B200 counterpart of the reference's per-view
`GradientCache` (ref: jacobian.py:46-84) generalised to the multi-view batch
that PCG sums over.

Build, per view: fp64 projection, (depth, gid) sort, tile binning, COUNT
raster pass (image, per-(tile, splat) keep masks), residual weights.  Per
subset: instance counts -> runs (a run = one (tile, splat) with >= 1 kept
pixel, numbered (view, tile, depth)), (view, gaussian) pairs, pair -> runs
CSR.  Per view: FILL raster pass writing each run's entries contiguously.
There is no sort of the cache and no second record stream: the pixel-sorted
and gaussian-sorted orders of the reference (jacobian.py:93-121) are both
views of this run order (see export_view).

Everything here is host orchestration of libsplatlm_b200 kernels on the
current torch stream; torch only allocates memory.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import call, off, ptr, stream_ptr
from .errors import ImageSizeError
from .scene import Camera, GaussianScene, cameras_struct_tensor, num_coefficients

TILE = 16
MASK_WORDS = TILE * TILE // 32
CHUNK_RUNS = 64   # SLM_CHUNK_RUNS: max runs per streaming chunk (bytes of schedule per chunk)


# below this many entries per run the J^T pass uses 4 lanes per run (stream.cu)
JT4_ENTRIES_PER_RUN = 18


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


def sort_u32(kin, kout, vin, vout, n, begin_bit, end_bit):
    ws = _empty(_lib.load().slm_sort_pairs_u32_workspace(n), torch.uint8, kin.device)
    call("slm_sort_pairs_u32", ptr(ws), ws.numel(), ptr(kin), ptr(kout), ptr(vin), ptr(vout), n, begin_bit,
         end_bit, stream_ptr())


def sort_u64(kin, kout, vin, vout, n, begin_bit, end_bit):
    ws = _empty(_lib.load().slm_sort_pairs_u64_workspace(n), torch.uint8, kin.device)
    call("slm_sort_pairs_u64", ptr(ws), ws.numel(), ptr(kin), ptr(kout), ptr(vin), ptr(vout), n, begin_bit,
         end_bit, stream_ptr())


def ssim_host_tables(H, W, window, sigma):
    """Taps and center self weights exactly as ref: residuals.py:49-91."""
    offs = np.arange(window) - window // 2
    k = np.exp(-0.5 * (offs / sigma) ** 2)
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


_SSIM_CACHE: dict = {}


def _ssim_tables(H, W, window, sigma, dev):
    """Device copies of the SSIM taps / centre weights, cached per shape."""
    key = (H, W, window, float(sigma), str(dev))
    t = _SSIM_CACHE.get(key)
    if t is None:
        taps, cwy, cwx = ssim_host_tables(H, W, window, sigma)
        t = tuple(torch.from_numpy(a).to(dev) for a in (taps, cwy, cwx))
        _SSIM_CACHE[key] = t
    return t


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
    """Per-view products of projection, binning and the COUNT pass."""

    def __init__(self, cam: Camera, pix_base: int):
        self.cam = cam
        self.pix_base = pix_base
        self.splats = None       # uint8 [G*96]
        self.inst_gid = None     # int32 [n_inst] gid of each (tile, depth) instance
        self.ranges = None       # int32 [2*n_tiles]
        self.rgb = None          # float64 [HW*3]
        self.t_final = None      # float64 [HW]
        self.tiles_x = (cam.width + TILE - 1) // TILE
        self.tiles_y = (cam.height + TILE - 1) // TILE
        self.n_inst = 0
        self.sorted_gid = None   # int32 [G] depth order
        self.inst_off = None     # int64 [G+1] instances per depth rank (pre-sort order)
        self.inst_mask = None    # int32 [n_inst*8] keep mask per instance
        self.inst_start = None   # int64 [n_inst] first entry of the instance's run

    @property
    def n_tiles(self):
        return self.tiles_x * self.tiles_y


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
    n_tiles = frame.n_tiles
    ik = _empty(total, torch.int32, dev)
    iv = _empty(total, torch.int32, dev)
    call("slm_tile_emit", ptr(sgid), ptr(inst_off), G, ptr(splats), frame.tiles_x, frame.tiles_y,
         ptr(ik), ptr(iv), stream_ptr())
    sk = torch.empty_like(ik)
    inst_gid = _empty(total, torch.int32, dev)   # the sorted values: each tile's splats in depth order
    sort_u32(ik, sk, iv, inst_gid, total, 0, _bits(n_tiles))   # stable: depth order within a tile
    ranges = torch.empty(2 * n_tiles, dtype=torch.int32, device=dev)
    call("slm_tile_ranges", ptr(sk), total, ptr(ranges), n_tiles, stream_ptr())
    frame.inst_gid = inst_gid
    frame.ranges = ranges
    frame.sorted_gid = sgid
    frame.inst_off = inst_off
    return skeys, sgid


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
    if gt.dtype not in (torch.float32, torch.float64):
        raise ValueError("ground truth must be float32 or float64")
    dev = gt.device
    gt = gt.contiguous()
    taps_t, cwy_t, cwx_t = _ssim_tables(H, W, loss.window, loss.sigma, dev)
    blocks = int(max(((W + 15) // 16) * ((H + 15) // 16), 1))  # one 16x16 tile per block
    part = torch.empty(blocks, dtype=torch.float64, device=dev)
    a = _lib.SlmResidArgs()
    a.img = ptr(frame.rgb)
    a.gt = ptr(gt)
    a.gt_f32 = 1 if gt.dtype == torch.float32 else 0
    a.W, a.H = W, H
    a.lambda1, a.lambda2, a.eps_den = float(loss.lambda1), float(loss.lambda2), float(loss.eps_den)
    a.ssim_c1, a.ssim_c2 = 0.01 ** 2, 0.03 ** 2
    a.mode = 0 if loss.mode == "l1ssim" else 1
    a.win = int(loss.window)
    a.taps, a.cw_y, a.cw_x = ptr(taps_t), ptr(cwy_t), ptr(cwx_t)
    a.gradr = off(gradr, frame.pix_base * 4)
    a.cgrad = off(cgrad, frame.pix_base * 4)
    a.energy_part = ptr(part)
    if exports is not None:
        for k in ("gradr", "cgrad", "rabs", "rssim", "drabs", "drssim"):
            exports[k] = torch.empty(H * W * 3, dtype=torch.float64, device=dev)
        a.o_gradr, a.o_cgrad = ptr(exports["gradr"]), ptr(exports["cgrad"])
        a.o_rabs, a.o_drabs = ptr(exports["rabs"]), ptr(exports["drabs"])
        a.o_rssim, a.o_drssim = ptr(exports["rssim"]), ptr(exports["drssim"])
    call("slm_residuals", _lib.byref(a), blocks, stream_ptr())
    keep = (taps_t, cwy_t, cwx_t)  # noqa: F841 -- alive until the kernels are queued
    return part


class CacheSet:
    """Gradient cache of one image subset on the device (run order).

    Args:
        scene: scene at the current parameters.
        cameras: the subset's views.
        gts: ground-truth images (H, W, 3) float64/float32 device tensors; when
            None the cache is built without residual weights (products only).
        config: RenderConfig.
        loss: LossConfig.
        weights: precomputed per-view (grad_r_sq4, color_grad4) instead of gts.
        timer: optional PhaseTimer.
        offload: cache offload ("CPU offloading of cache
            parts"): None / 0 keeps every record in HBM; a fraction f places
            the last ~f of the record streams (from a chunk boundary) in
            host-pinned, device-mapped memory that FILL writes and the
            streaming kernels' TMA reads over the host link; "auto" offloads
            only what does not fit in the device's free memory next to the
            product scratch.
    """

    def __init__(self, scene: GaussianScene, cameras: list[Camera], gts=None, config=None, loss=LossConfig(),
                 residual_exports: bool = False, weights=None, timer=None, offload=None):
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
        if V > 255:
            raise ValueError("at most 255 views per cache subset")
        self.G, self.V = G, V
        self.P = scene.params_per_gaussian
        self.K = num_coefficients(scene.sh_degree)
        self.cams_dev, self.pix_bases = cameras_struct_tensor(self.cameras, dev)
        self.camf = torch.empty(max(len(self.cameras), 1) * 20, dtype=torch.float32, device=dev)
        call("slm_cameras_f32", ptr(self.cams_dev), len(self.cameras), ptr(self.camf), stream_ptr())
        self.N = sum(c.num_pixels for c in self.cameras)
        views = (_lib.SlmView * V)()
        for i, c in enumerate(self.cameras):
            views[i].pix_base, views[i].W, views[i].H = self.pix_bases[i], c.width, c.height
        self.views_dev = _lib.struct_tensor(views, dev)
        cfg_s = rast_cfg_struct(self.config, scene.background)
        self.cfg_s = cfg_s
        self._b = None
        self._M = None
        if G == 0:
            self._init_empty(gts, weights, loss, residual_exports)
            return
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
        # ---- subset-batched projection, (view, depth, gid) order, binning ----
        VG = V * G
        tbases, nt = [], 0
        for c in self.cameras:
            tbases.append(nt)
            nt += ((c.width + TILE - 1) // TILE) * ((c.height + TILE - 1) // TILE)
        self.n_tiles_total = nt
        self.view_tile_base = tbases + [nt]
        self.view_tile_base_dev = torch.tensor(self.view_tile_base, dtype=torch.int32, device=dev)
        splats_all = torch.empty(VG * _lib.SPLAT_BYTES, dtype=torch.uint8, device=dev)
        keys = torch.empty(VG, dtype=torch.int64, device=dev)
        vals = torch.empty(VG, dtype=torch.int32, device=dev)
        call("slm_preprocess_views", ptr(scene.x), G, scene.sh_degree, ptr(self.cams_dev), V, _lib.byref(cfg_s),
             ptr(splats_all), ptr(keys), ptr(vals), ptr(err), stream_ptr())
        skeys = torch.empty_like(keys)
        sv0 = torch.empty_like(vals)
        sort_u64(keys, skeys, vals, sv0, VG, 0, 64)           # depth (fp64 bits), ties by (view, gid)
        del keys, vals, skeys
        sv = torch.empty_like(sv0)
        ws = _empty(_lib.load().slm_sort_keys_u32_workspace(VG), torch.uint8, dev)
        call("slm_sort_keys_u32", ptr(ws), ws.numel(), ptr(sv0), ptr(sv), VG, 24, 32, stream_ptr())  # by view (stable)
        del sv0, ws
        n_inst = torch.zeros(VG + 1, dtype=torch.int64, device=dev)
        call("slm_tile_count_v", ptr(sv), VG, G, ptr(splats_all), ptr(self.views_dev), ptr(n_inst), stream_ptr())
        inst_off = torch.empty_like(n_inst)
        scan_i64(n_inst, inst_off)
        del n_inst
        ni = int(inst_off[VG].item())
        self.n_inst_total = ni
        ik = _empty(ni, torch.int32, dev)
        iv = _empty(ni, torch.int32, dev)
        call("slm_tile_emit_v", ptr(sv), ptr(inst_off), VG, G, ptr(splats_all), ptr(self.views_dev),
             ptr(self.view_tile_base_dev), ptr(ik), ptr(iv), stream_ptr())
        sk = torch.empty_like(ik)
        inst_gid = _empty(ni, torch.int32, dev)      # sorted values: global splat v * G + g per instance
        sort_u32(ik, sk, iv, inst_gid, ni, 0, _bits(nt))   # stable: (view, depth) emission order within a tile
        del ik, iv
        ranges = torch.empty(2 * nt, dtype=torch.int32, device=dev)
        call("slm_tile_ranges", ptr(sk), ni, ptr(ranges), nt, stream_ptr())
        del sk
        inst_mask = torch.zeros(max(ni, 1) * MASK_WORDS, dtype=torch.int32, device=dev)
        T.tick("project_sort_bin")

        # ---- COUNT pass (all views, one launch) + residuals per view -----------
        self.rgb_all = torch.empty(self.N * 3, dtype=torch.float64, device=dev)
        self.t_final_all = torch.empty(self.N, dtype=torch.float64, device=dev)

        def batched_args():
            a = _lib.SlmRasterArgs()
            a.tile_range, a.inst_gid, a.splats = ptr(ranges), ptr(inst_gid), ptr(splats_all)
            a.cfg = cfg_s
            a.views, a.view_tile_base, a.n_views, a.n_tiles = ptr(self.views_dev), ptr(self.view_tile_base_dev), V, nt
            a.rgb, a.inst_mask = ptr(self.rgb_all), ptr(inst_mask)
            return a
        a = batched_args()
        a.px_count, a.t_final = ptr(self.px_count), ptr(self.t_final_all)
        call("slm_raster_count", _lib.byref(a), stream_ptr())
        T.tick("raster_count")
        for v, cam in enumerate(self.cameras):
            fr = ViewFrame(cam, self.pix_bases[v])
            hw = cam.num_pixels
            fr.rgb = self.rgb_all[fr.pix_base * 3:(fr.pix_base + hw) * 3]
            fr.t_final = self.t_final_all[fr.pix_base:fr.pix_base + hw]
            if have_res:
                ex = {} if residual_exports else None
                energy_parts.append(residual_pass(fr, gts[v], loss, self.gradr, self.cgrad, ex))
                if residual_exports:
                    self.residual_exports.append(ex)
            self.frames.append(fr)
        T.tick("residuals")
        # ---- instances -> runs ---------------------------------------------
        inst_cnt = torch.zeros(ni + 1, dtype=torch.int64, device=dev)
        inst_used = torch.zeros(ni + 1, dtype=torch.int32, device=dev)
        call("slm_inst_count", ptr(inst_mask), ptr(inst_gid), ni, ptr(inst_cnt), ptr(inst_used), ptr(self.pair_cnt),
             stream_ptr())
        ent_of = torch.empty_like(inst_cnt)
        scan_i64(inst_cnt, ent_of)
        run_of = torch.empty_like(inst_used)
        scan_i32(inst_used, run_of)
        del inst_cnt

        # ---- pairs (view, gaussian) ------------------------------------------
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
        # ONE host sync for the error flags, the per-view energies and the
        # entry / run / pair counts the next allocations need
        sums = [err.to(torch.float64).reshape(1), ent_of[ni].to(torch.float64).reshape(1),
                run_of[ni].to(torch.float64).reshape(1), pair_of[VG].to(torch.float64).reshape(1)] + \
            [p.sum().reshape(1) for p in energy_parts]
        host = torch.cat(sums).cpu().tolist()
        e = int(host[0])
        if e & 1:
            raise ValueError("scene contains non-finite parameters")
        if e & 2:
            raise ValueError("quaternion with (near-)zero norm")
        self.E, self.R, self.n_pairs = int(host[1]), int(host[2]), int(host[3])
        self.energies = host[4:] if have_res else None
        Pn = self.n_pairs
        self.pair_off = torch.empty(Pn + 1, dtype=torch.int64, device=dev)   # entries per pair (stats)
        self.pair_gid = _empty(Pn, torch.int32, dev)
        self.pair_vm = _empty(Pn, torch.int32, dev)
        self.pair_geo = _empty(Pn * _lib.PAIR_GEO_BYTES, torch.uint8, dev)
        pidx = torch.empty(VG, dtype=torch.int32, device=dev)
        self.gpo = torch.empty(G + 1, dtype=torch.int32, device=dev)
        call("slm_pairs_emit", ptr(self.pair_cnt), V, G, ptr(pair_of), ptr(vscan), ptr(tscan), ptr(splats_all),
             ptr(self.pair_off), ptr(self.pair_gid), ptr(self.pair_vm), ptr(self.pair_geo), ptr(pidx), ptr(self.gpo),
             Pn, self.E, stream_ptr())
        del cntV, flagV, flagT, vscan, pair_of, tscan

        # ---- run table, runs per tile, pair -> runs ----------------------------
        R = self.R
        self.run_start = torch.zeros(R + 3, dtype=torch.int64, device=dev)  # +2: 16 B-granular TMA copies
        self.run_q = _empty(R + 8, torch.int32, dev)   # +8: 16-byte granular TMA copies (diag)
        self.run_tile = _empty(R, torch.int32, dev)
        pair_nruns = torch.zeros(Pn + 1, dtype=torch.int32, device=dev)
        tile_nruns = torch.zeros(nt + 1, dtype=torch.int32, device=dev)
        inst_start = _empty(ni, torch.int64, dev)
        call("slm_runs_emit", ptr(inst_mask), ptr(inst_gid), ptr(inst_used), ptr(run_of), ptr(ent_of), 0, ni,
             ptr(pidx), ptr(self.run_start), ptr(self.run_q), None, ptr(pair_nruns), ptr(inst_start),
             stream_ptr())
        call("slm_tile_runs", ptr(ranges), nt, ptr(inst_used), ptr(run_of), 0, 0, ptr(tile_nruns), ptr(self.run_tile),
             ptr(self.view_tile_base_dev), V, stream_ptr())
        self.run_start[R:].fill_(self.E)
        self.tile_run_off = torch.empty_like(tile_nruns)
        scan_i32(tile_nruns, self.tile_run_off)
        # chunk table for the streaming product kernel (<= 64 runs / 896 entries per chunk)
        tile_nch = torch.zeros(nt + 1, dtype=torch.int32, device=dev)
        call("slm_tile_chunks", ptr(self.tile_run_off), nt, ptr(self.run_start), None, ptr(tile_nch), None, 0,
             stream_ptr())
        self.tile_chunk_off = torch.empty_like(tile_nch)
        scan_i32(tile_nch, self.tile_chunk_off)
        self.n_chunks = int(self.tile_chunk_off[nt].item())
        self.chunk_run = torch.empty(self.n_chunks + 1, dtype=torch.int32, device=dev)
        self.chunk_perm = torch.empty((self.n_chunks + 1) * CHUNK_RUNS, dtype=torch.uint8, device=dev)
        call("slm_tile_chunks", ptr(self.tile_run_off), nt, ptr(self.run_start), ptr(self.tile_chunk_off),
             ptr(self.chunk_run), ptr(self.chunk_perm), 1, stream_ptr())
        self.chunk_run[self.n_chunks:].fill_(R)
        self.run_fn = _empty(R + 8, torch.int32, dev)   # +8: 16-byte granular TMA copies stay in bounds
        call("slm_chunk_perm", ptr(self.chunk_run), self.n_chunks, ptr(self.run_start), ptr(self.chunk_perm),
             ptr(self.run_fn), stream_ptr())
        del tile_nch
        self.pair_run_off = torch.empty_like(pair_nruns)
        scan_i32(pair_nruns, self.pair_run_off)
        # pair -> runs CSR: a stable radix sort of the runs by pair.  Runs are
        # in (global tile, depth) order, so each pair's runs come out in tile
        # row-major order -- the (tile row, tile column) order of the
        # reference's bbox walk (rasterizer.py:283-287).  run_slot: each run's
        # position in pair_runs (the J^T kernels write run partials there so
        # the backward reads a gaussian's runs contiguously)
        self.pair_runs = _empty(R, torch.int32, dev)
        self.run_slot = torch.empty(max(R, 1), dtype=torch.int32, device=dev)
        self.tile_counter = torch.zeros(1, dtype=torch.int32, device=dev)  # dynamic tile scheduling scratch
        if R > 0:
            rid = _empty(R, torch.int32, dev)
            call("slm_iota_u32", ptr(rid), R, stream_ptr())
            qk = _empty(R, torch.int32, dev)
            ws = _empty(_lib.load().slm_sort_pairs_u32_workspace(R), torch.uint8, dev)
            call("slm_sort_pairs_u32", ptr(ws), ws.numel(), ptr(self.run_q), ptr(qk), ptr(rid), ptr(self.pair_runs),
                 R, 0, _bits(Pn), stream_ptr())
            del ws, qk, rid
            call("slm_invert_perm", ptr(self.pair_runs), R, ptr(self.run_slot), stream_ptr())
        del sv, inst_off
        del pidx, pair_nruns, tile_nruns, inst_used, run_of, ent_of
        T.tick("runs_pairs")

        # ---- FILL phase: run-ordered records ------------------------------------
        E = self.E
        f32 = torch.float32
        # {alpha_eff, alpha*T, dc/dalpha_r, dc/dalpha_g}, dc/dalpha_b, tile-local
        # pixel; +16 slots so the 16-byte-granular TMA chunk copies of the
        # product kernels stay in bounds
        # every entry is written by the FILL pass; the +16 tail slots are only
        # over-read by the 16-byte-granular copies and never used
        split = self._offload_split(offload)
        self.e_split, self.e_hbase = split, split & ~15
        self.rec4 = torch.empty((split + 16) * 4, dtype=f32, device=dev)
        self.rec_d2 = torch.empty(split + 16, dtype=f32, device=dev)
        self.rec_pix = torch.empty(split + 16, dtype=torch.uint8, device=dev)
        self.rec4_h = self.rec_d2_h = self.rec_pix_h = None
        if split < E:
            nh = E - self.e_hbase + 16
            self.rec4_h = torch.empty(nh * 4, dtype=f32, pin_memory=True)
            self.rec_d2_h = torch.empty(nh, dtype=f32, pin_memory=True)
            self.rec_pix_h = torch.empty(nh, dtype=torch.uint8, pin_memory=True)
        a = batched_args()
        a.inst_start = ptr(inst_start)
        a.rec4, a.rec_d2, a.rec_pix = ptr(self.rec4), ptr(self.rec_d2), ptr(self.rec_pix)
        self._offload_args(a, "rec_d2_h", "rec_pix_h")
        call("slm_raster_fill", _lib.byref(a), stream_ptr())
        T.tick("raster_fill")
        del inst_mask, inst_start, inst_gid, ranges, splats_all
        # product scratch: J^T run partials 0-7 (32-byte records) then partial 8
        self.u = torch.empty(self.N * 4, dtype=f32, device=dev)
        self.run_acc = _empty(R * _lib.JT_D, f32, dev)
        self.run_static = _empty(R * 8, f32, dev)
        self.warp_g0 = torch.empty((Pn >> 5) + 2, dtype=torch.int32, device=dev)
        self.gm = torch.empty(G * self.P, dtype=torch.float32, device=dev)
        call("slm_warp_bounds", ptr(self.gpo), G, Pn, ptr(self.warp_g0), stream_ptr())
        self.pm = _empty(Pn * 12, f32, dev)
        # per-gaussian chain rows: view-independent chain constants, position,
        # SH coefficients (the scene is fixed for the cache)
        self.gtab = torch.empty(G * _lib.load().slm_gauss_tab_floats(scene.sh_degree), dtype=f32, device=dev)
        call("slm_gauss_tab", ptr(scene.x32()), G, scene.sh_degree, ptr(self.gtab), stream_ptr())
        call("slm_run_static", _lib.byref(self._tile_args()), R, ptr(self.run_slot), ptr(self.run_static),
             stream_ptr())

    # ------------------------------------------------------------------
    # cache offload
    # ------------------------------------------------------------------
    @property
    def offloaded_entries(self) -> int:
        return self.E - self.e_split if self.rec4_h is not None else 0

    def _offload_split(self, offload) -> int:
        """First entry of the host-resident tail: a chunk boundary (a chunk's
        records are streamed from one place), E when nothing is offloaded."""
        E = self.E
        if not offload or E == 0 or self.n_chunks == 0:
            return E
        if offload == "auto":
            free, _ = torch.cuda.mem_get_info(self.device)
            st = torch.cuda.memory_stats(self.device)
            free += st.get("reserved_bytes.all.current", 0) - st.get("allocated_bytes.all.current", 0)
            # product / diag / PCG scratch allocated after FILL, plus 2 GB
            scratch = (16 * self.N + 100 * self.R + 250 * self.n_pairs + 700 * self.G * 1 + (2 << 30))
            cap = (free - scratch) // 21
            if E <= cap:
                return E
            target = max(0, int(cap))
        else:
            f = float(offload)
            if not 0.0 < f <= 1.0:
                raise ValueError("offload must be None, 'auto' or a fraction in (0, 1]")
            target = int(E * (1.0 - f))
        starts = self.run_start[self.chunk_run[:self.n_chunks].long()]
        k = int(torch.searchsorted(starts, torch.tensor([target], dtype=starts.dtype, device=starts.device)).item())
        return int(starts[k].item()) if k < self.n_chunks else E

    def _offload_args(self, a, d2_name: str, pix_name: str):
        """Fill the offload fields of a raster / tile argument struct."""
        if self.rec4_h is None:
            return
        a.rec4_h = ptr(self.rec4_h)
        setattr(a, d2_name, ptr(self.rec_d2_h))
        setattr(a, pix_name, ptr(self.rec_pix_h))
        a.e_split, a.e_hbase = self.e_split, self.e_hbase

    def _records(self, e0: int, e1: int):
        """Host copies (rec4 [n, 4], d2 [n], pix [n]) of entries [e0, e1),
        from the device streams and the offloaded tail."""
        parts = []
        s = min(e1, self.e_split)
        if e0 < s:
            parts.append((self.rec4[4 * e0:4 * s].view(-1, 4).cpu(), self.rec_d2[e0:s].cpu(), self.rec_pix[e0:s].cpu()))
        if self.rec4_h is not None and e1 > self.e_split:
            h0, h1 = max(e0, self.e_split) - self.e_hbase, e1 - self.e_hbase
            parts.append((self.rec4_h[4 * h0:4 * h1].view(-1, 4), self.rec_d2_h[h0:h1], self.rec_pix_h[h0:h1]))
        if not parts:
            return np.zeros((0, 4), np.float32), np.zeros(0, np.float32), np.zeros(0, np.uint8)
        return tuple(torch.cat([p[i] for p in parts]).numpy() for i in range(3))

    def _init_empty(self, gts, weights, loss, residual_exports):
        """G = 0: background images, no entries; b and M are
        empty and every product is the zero map."""
        dev, N = self.device, self.N
        self.E = self.R = self.n_pairs = self.n_chunks = self.n_inst_total = 0
        self.rec4_h, self.e_split, self.e_hbase = None, 0, 0
        bg = torch.tensor(self.scene.background, dtype=torch.float64, device=dev)
        self.rgb_all = bg.repeat(N)
        self.t_final_all = torch.ones(N, dtype=torch.float64, device=dev)
        have_w = gts is not None or weights is not None
        self.gradr = torch.zeros(N * 4, dtype=torch.float32, device=dev) if have_w else None
        self.cgrad = torch.zeros(N * 4, dtype=torch.float32, device=dev) if have_w else None
        self.u = torch.zeros(N * 4, dtype=torch.float32, device=dev)
        self.frames, parts = [], []
        self.residual_exports = [] if residual_exports else None
        for v, cam in enumerate(self.cameras):
            fr = ViewFrame(cam, self.pix_bases[v])
            hw = cam.num_pixels
            fr.rgb = self.rgb_all[fr.pix_base * 3:(fr.pix_base + hw) * 3]
            fr.t_final = self.t_final_all[fr.pix_base:fr.pix_base + hw]
            if weights is not None:
                g4, c4 = weights[v]
                self.gradr[fr.pix_base * 4:fr.pix_base * 4 + g4.numel()].copy_(g4)
                self.cgrad[fr.pix_base * 4:fr.pix_base * 4 + c4.numel()].copy_(c4)
            elif gts is not None:
                ex = {} if residual_exports else None
                parts.append(residual_pass(fr, gts[v].to(dev), loss, self.gradr, self.cgrad, ex))
                if residual_exports:
                    self.residual_exports.append(ex)
            self.frames.append(fr)
        self.energies = [float(p.sum().item()) for p in parts] if gts is not None else None

    # ------------------------------------------------------------------
    @property
    def nbytes(self) -> int:
        """Bytes of the record stream (budget accounting, ref: jacobian.py:76-80)."""
        return 21 * self.E + 48 * self.R + 36 * self.n_chunks

    @property
    def host_nbytes(self) -> int:
        """Bytes of the offloaded (host-resident) record tail."""
        return 21 * self.offloaded_entries

    def pair_forward(self, p: torch.Tensor, gaussian_major: bool = False, p_gm: torch.Tensor | None = None):
        """Forward chain m = dy/dx p per pair into self.pm (48 B per pair); the
        J / fused product kernels gather it per run.  p_gm: the padded
        gaussian-major copy of p (stride slm_gm_stride(P)) written by the PCG
        p kernels, read with 16-byte row loads."""
        G, P = self.G, self.P
        if G == 0:
            return
        a = _lib.SlmFwdArgs()
        a.xs, a.G = ptr(self.scene.x32()), G
        a.camf = ptr(self.camf)
        a.pair_gid, a.pair_vm, a.cams, a.n_pairs = ptr(self.pair_gid), ptr(self.pair_vm), ptr(self.cams_dev), \
            self.n_pairs
        if p_gm is not None:   # written by slm_pcg_p* / gm_pack with this cache's chain rows
            a.p, a.sa, a.sg, a.dsig = ptr(p_gm), 1, _lib.load().slm_gm_stride(P), 1
        else:
            a.p = ptr(p)
            a.sa, a.sg = (1, P) if gaussian_major else (G, 1)
        a.pm, a.gtab = ptr(self.pm), ptr(self.gtab)
        call("slm_pair_forward", _lib.byref(a), self.scene.sh_degree, stream_ptr())

    @property
    def gtab_stride(self) -> int:
        return _lib.load().slm_gauss_tab_floats(self.scene.sh_degree)

    def gm_pack(self, p: torch.Tensor) -> torch.Tensor:
        """The padded gaussian-major copy of an attribute-major p with its
        world-covariance perturbation, as the PCG p kernels write it."""
        out = torch.empty(self.G * _lib.load().slm_gm_stride(self.P), dtype=torch.float32, device=self.device)
        call("slm_gm_pack", ptr(p), ptr(out), self.G, self.P, ptr(self.gtab), self.gtab_stride, stream_ptr())
        return out

    def _tile_args(self, with_m: bool = False) -> _lib.SlmTileArgs:
        a = _lib.SlmTileArgs()
        a.views, a.view_tile_base, a.n_views = ptr(self.views_dev), ptr(self.view_tile_base_dev), self.V
        a.n_tiles = self.n_tiles_total
        a.tile_run_off, a.tile_chunk_off, a.chunk_run = ptr(self.tile_run_off), ptr(self.tile_chunk_off), \
            ptr(self.chunk_run)
        a.chunk_perm, a.run_slot = ptr(self.chunk_perm), ptr(self.run_slot)
        a.run_start, a.run_q, a.run_tile, a.run_static = ptr(self.run_start), ptr(self.run_q), ptr(self.run_tile), \
            ptr(self.run_static)
        a.run_fn = ptr(self.run_fn)
        a.pm = ptr(self.pm) if with_m else None
        a.geo = ptr(self.pair_geo)
        a.rec4, a.d2 = ptr(self.rec4), ptr(self.rec_d2)
        a.pix = ptr(self.rec_pix)
        a.jt_lanes = 4 if self.R > 0 and self.E < JT4_ENTRIES_PER_RUN * self.R else 8
        self._offload_args(a, "d2_h", "pix_h")
        a.tile_counter = ptr(self.tile_counter)
        return a

    def _backward(self, run_acc, out, mode, scale=1.0, p=None, M=None, lam=0.0, dot_part=None, lam_out=True):
        """run partials (pair-run-slot order, as the J^T / diag streaming
        kernels write them) -> per-gaussian chain, attribute-major out."""
        a = _lib.SlmBackArgs()
        a.pacc, a.pair_run_off = ptr(run_acc), ptr(self.pair_run_off)
        if mode == 0:
            a.pacc1 = off(run_acc, 8 * self.R)
        a.xs, a.G = ptr(self.scene.x32()), self.G
        a.gpo, a.pair_vm, a.cams, a.camf = ptr(self.gpo), ptr(self.pair_vm), ptr(self.cams_dev), ptr(self.camf)
        a.gtab = ptr(self.gtab)
        a.warp_g0, a.pair_gid, a.n_pairs = ptr(self.warp_g0), ptr(self.pair_gid), self.n_pairs
        a.gm = ptr(self.gm)
        a.scale, a.p, a.Mdiag, a.lam = float(scale), ptr(p), ptr(M), float(lam)
        a.lam_out = 1 if lam_out else 0
        a.out, a.dot_part = ptr(out), ptr(dot_part)
        call("slm_pair_backward", _lib.byref(a), mode, self.scene.sh_degree, stream_ptr())

    def apply_j_raw(self, weighted: bool) -> torch.Tensor:
        """u (or u_hat) into self.u from the run records written by pair_forward."""
        if weighted and self.gradr is None:
            raise ValueError("cache was built without residual weights")
        if self.G == 0:
            return self.u.zero_()
        a = self._tile_args(with_m=True)
        a.gradr = ptr(self.gradr) if weighted else None
        a.u_out = ptr(self.u)
        call("slm_apply_j", _lib.byref(a), stream_ptr())
        return self.u

    def apply_jt_raw(self, u: torch.Tensor, out: torch.Tensor, scale: float = 1.0, p=None, M=None, lam=0.0,
                     dot_part=None):
        if self.G == 0:
            return out
        ra = self._tile_args()
        ra.u, ra.out, ra.out1 = ptr(u), ptr(self.run_acc), off(self.run_acc, 8 * self.R)
        call("slm_apply_jt_runs", _lib.byref(ra), stream_ptr())
        self._backward(self.run_acc, out, 0, scale, p, M, lam, dot_part)
        return out

    def jtwj(self, p: torch.Tensor, out: torch.Tensor, lam: float = 0.0, M=None, dot_part=None,
             lam_out: bool = True, p_gm: torch.Tensor | None = None):
        """out = J^T W J p (+ lam * max(M, 1e-12) * p when lam_out); attribute-major
        fp32.  dot_part receives fp64 block partials of p.(J^T W J p + lam Mf p).

        Four launches: pair forward chain (+ run records), the fused per-tile
        J / W / J^T streaming kernel (u never leaves shared memory), per-pair
        sums, per-gaussian backward chain."""
        if self.gradr is None:
            raise ValueError("cache was built without residual weights")
        if self.G == 0:
            if dot_part is not None:
                dot_part.zero_()
            return out
        self.pair_forward(p, p_gm=p_gm)
        a = self._tile_args(with_m=True)
        a.gradr, a.out, a.out1 = ptr(self.gradr), ptr(self.run_acc), off(self.run_acc, 8 * self.R)
        call("slm_jtwj_runs", _lib.byref(a), stream_ptr())
        self._backward(self.run_acc, out, 0, 1.0, p, M if lam != 0.0 else None, lam, dot_part, lam_out)
        return out

    def rhs(self) -> torch.Tensor:
        """b = -J^T color_grad, summed over the subset's views (ref: jacobian.py:411-413).
        With residual weights it comes from the same cache sweep as diag()."""
        if self._b is None:
            if self.cgrad is None:
                raise ValueError("cache was built without residuals")
            if self.gradr is not None:
                self._diag_and_rhs()
            else:
                b = torch.empty(self.G * self.P, dtype=torch.float32, device=self.device)
                self.apply_jt_raw(self.cgrad, b, -1.0)
                self._b = b
        return self._b

    def diag(self) -> torch.Tensor:
        """M = diag(J^T W J), attribute-major (ref: jacobian.py:486-512)."""
        if self._M is None:
            if self.gradr is None:
                raise ValueError("cache was built without residual weights")
            self._diag_and_rhs()
        return self._M

    def _diag_and_rhs(self):
        """One sweep of the streaming kernel over the cache: the diag moments
        per run and (with a colour gradient) the rhs J^T partials; then the
        two per-gaussian backward chains."""
        dev, n = self.device, self.G * self.P
        if self.G == 0:
            self._M = torch.empty(0, dtype=torch.float32, device=dev)
            if self.cgrad is not None:
                self._b = torch.empty(0, dtype=torch.float32, device=dev)
            return
        moments = _empty(self.R * _lib.DIAG_M, torch.float32, dev)
        want_b = self.cgrad is not None and self._b is None
        ra = self._tile_args()
        ra.gradr, ra.out = ptr(self.gradr), ptr(moments)
        if want_b:
            ra.u, ra.rhs8, ra.rhs1 = ptr(self.cgrad), ptr(self.run_acc), off(self.run_acc, 8 * self.R)
        call("slm_diag_stream", _lib.byref(ra), stream_ptr())
        if self._M is None:
            M = torch.empty(n, dtype=torch.float32, device=dev)
            self._backward(moments, M, 1)
            self._M = M
        if want_b:
            b = torch.empty(n, dtype=torch.float32, device=dev)
            self._backward(self.run_acc, b, 0, -1.0)
            self._b = b

    # ------------------------------------------------------------------
    # parity exports (test infrastructure; host-side reconstruction)
    # ------------------------------------------------------------------
    def image(self, v: int) -> torch.Tensor:
        c = self.cameras[v]
        return self.frames[v].rgb.view(c.height, c.width, 3)

    def export_view(self, v: int) -> dict:
        """Reference-shaped arrays of view v: the pixel-sorted cache
        (ref: jacobian.py:401-409) and its gaussian-sorted permutation
        (ref: jacobian.py:93-105).  Both orders are computed on the device from
        the run order (slm_export_view); the record values are then placed
        with that device-computed permutation."""
        cam = self.cameras[v]
        if self.G == 0:
            e, f = np.zeros(0, np.int64), np.zeros(0)
            return dict(pixel_ids=e, gaussian_ids=e, alphas=f, alpha_eff=f, transmittances=f,
                        dc_dalpha=np.zeros((0, 3)), dc_dcs=f, offsets=np.zeros(cam.num_pixels + 1, np.int64),
                        g_pixel_ids=e, g_gaussian_ids=e, g_offsets=np.zeros(1, np.int64), g_source_index=e,
                        g_dc_dalpha=np.zeros((0, 3)), g_alpha_eff=f, g_dc_dcs=f)
        dev, i64 = self.device, torch.int64
        t0, t1 = self.view_tile_base[v], self.view_tile_base[v + 1]
        r0, r1 = (int(x) for x in self.tile_run_off[[t0, t1]].tolist())
        e0, e1 = (int(x) for x in self.run_start[[r0, r1]].tolist())
        Ev, hw, G = e1 - e0, cam.num_pixels, self.G
        pb = self.pix_bases[v]
        px_cnt = torch.zeros(hw + 1, dtype=i64, device=dev)
        px_cnt[:hw] = self.px_count[pb:pb + hw]
        px_off = torch.empty_like(px_cnt)
        scan_i64(px_cnt, px_off)
        g_cnt = torch.zeros(G + 1, dtype=i64, device=dev)
        g_cnt[:G] = self.pair_cnt[v * G:(v + 1) * G]
        g_off = torch.empty_like(g_cnt)
        scan_i64(g_cnt, g_off)
        out = {k: _empty(Ev, i64, dev) for k in ("pos_pix", "pixel_ids", "gaussian_ids", "g_pixel_ids",
                                                  "g_gaussian_ids", "g_source_index")}
        r4, d2, pxb = self._records(e0, e1)
        pix_v = torch.from_numpy(np.concatenate([pxb, np.zeros(16, np.uint8)])).to(dev)  # the view's pixel bytes
        pix_ptr = C.c_void_p(pix_v.data_ptr() - e0)   # the kernel indexes entries globally
        call("slm_export_view", ptr(self.tile_run_off), t0, t1 - t0, (cam.width + TILE - 1) // TILE, cam.width,
             ptr(self.run_start), ptr(self.run_q), ptr(self.run_tile), ptr(self.pair_gid), ptr(self.pair_vm),
             ptr(self.pair_run_off), ptr(self.pair_runs), self.n_pairs, v, pix_ptr, ptr(px_off),
             ptr(g_off), e0, ptr(out["pos_pix"]), ptr(out["pixel_ids"]), ptr(out["gaussian_ids"]),
             ptr(out["g_pixel_ids"]), ptr(out["g_gaussian_ids"]), ptr(out["g_source_index"]), stream_ptr())
        h = {k: t[:Ev].cpu().numpy() for k, t in out.items()}
        pos, src = h["pos_pix"], h["g_source_index"]
        r4, d2 = r4.astype(np.float64), d2.astype(np.float64)
        ae, at = np.empty(Ev), np.empty(Ev)
        dcda = np.empty((Ev, 3))
        ae[pos], at[pos] = r4[:, 0], r4[:, 1]
        dcda[pos] = np.stack([r4[:, 2], r4[:, 3], d2], 1)
        alpha = np.where(ae == 0.0, self.config.alpha_clamp, ae)
        return dict(pixel_ids=h["pixel_ids"], gaussian_ids=h["gaussian_ids"], alphas=alpha, alpha_eff=ae,
                    transmittances=at / alpha, dc_dalpha=dcda, dc_dcs=at, offsets=px_off.cpu().numpy(),
                    g_pixel_ids=h["g_pixel_ids"], g_gaussian_ids=h["g_gaussian_ids"], g_offsets=g_off.cpu().numpy(),
                    g_source_index=src, g_dc_dalpha=dcda[src], g_alpha_eff=ae[src], g_dc_dcs=at[src])
