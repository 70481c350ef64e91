"""PCG inner solver, Eq. 7 combine and the LM direction (SPEC-only in the
reference: pcg_solve SPEC:391-399, solve_normal_equations_batched SPEC:400-408;
Alg. 1; Eq. 7).

Vectors are attribute-major device tensors: the search direction p and the
product output are float32 (the products are fp32 kernels), the iterate x and
the residual r are float64 (x0 = b / Mf makes |A x0| >> |b|, so an fp32
residual recurrence would cancel), scalars are fp64 and stay on the device
(one 8-byte read per iteration for the exit test).  Multi-GPU: image
subsets are sharded round-robin over ranks; each rank accumulates
num = sum M_i * Delta_i and den = sum M_i, then ONE all_reduce(SUM) of the
packed [num; den] over NCCL combines them.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import torch

from . import _lib
from ._lib import call, ptr, stream_ptr
from .engine import CacheSet, LossConfig, _NoTimer
from .errors import NonSPDError
from .scene import Layout, ParamVector

ST_RZ, ST_PG, ST_BB, ST_RR, ST_ALPHA, ST_BETA, ST_FLAGS, ST_ITERS, ST_STOP = 0, 2, 3, 4, 5, 6, 7, 8, 9


@dataclass(frozen=True)
class BatchSchedule:
    """ref SPEC:379-380 (BatchSchedule); strided selection SPEC:477."""
    n_batches: int = 1
    selection: str = "strided"

    def batches(self, n_views: int) -> list[list[int]]:
        if self.n_batches < 1:
            raise ValueError("n_b must be >= 1")
        return [list(range(j, n_views, self.n_batches)) for j in range(self.n_batches)]

    def shard(self, n_views: int, rank: int, world: int) -> list[tuple[int, list[int]]]:
        """Subsets owned by `rank`: subset j -> rank j mod world."""
        return [(j, v) for j, v in enumerate(self.batches(n_views)) if j % world == rank and v]


def allreduce_sum_(buf: torch.Tensor, group=None) -> torch.Tensor:
    """In-place SUM all_reduce when a process group with >1 rank is up
    (NCCL on GPU boxes, gloo in the CPU tests); no-op otherwise."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
    return buf


_STOP_HOST = []


def _pinned_stop() -> torch.Tensor:
    """Process-wide pinned 2-slot buffer (a pinned allocation per solve would
    cost a synchronising cudaHostAlloc)."""
    if not _STOP_HOST:
        _STOP_HOST.append(torch.zeros(2, dtype=torch.float64).pin_memory())
    return _STOP_HOST[0]


@dataclass
class PCGWorkspace:
    """x, r (fp64), p, g (fp32) vectors + device scalar block (SPEC PCGWorkspace).
    With G, P given, also the padded gaussian-major copy p_gm of p that the
    forward chain of the product reads with 16-byte row loads."""
    n: int
    device: torch.device
    G: int = 0
    P: int = 0
    x: torch.Tensor = field(init=False)
    r: torch.Tensor = field(init=False)
    p: torch.Tensor = field(init=False)
    g: torch.Tensor = field(init=False)
    st: torch.Tensor = field(init=False)
    part: torch.Tensor = field(init=False)

    def __post_init__(self):
        f = torch.float32
        self.x = torch.empty(self.n, dtype=torch.float64, device=self.device)
        self.r = torch.empty(self.n, dtype=torch.float64, device=self.device)
        self.p = torch.empty(self.n, dtype=f, device=self.device)
        self.g = torch.empty(self.n, dtype=f, device=self.device)
        self.p_gm = None
        if self.G > 0 and self.G * self.P == self.n:
            self.p_gm = torch.empty(self.G * _lib.load().slm_gm_stride(self.P), dtype=f, device=self.device)
        self.st = torch.zeros(16, dtype=torch.float64, device=self.device)
        self.part = torch.zeros(3 * _lib.load().slm_vec_blocks(), dtype=torch.float64, device=self.device)
        # pinned copies of the stop flag, one per in-flight iteration
        self.stop_host = _pinned_stop()
        self.stop_ev = [torch.cuda.Event(), torch.cuda.Event()]


def pcg_run(cache: CacheSet, b: torch.Tensor, M: torch.Tensor, lam: float, max_iters: int,
            ws: PCGWorkspace | None = None, stats: dict | None = None, timer=None) -> torch.Tensor:
    """Alg. 1 on the device; returns x (attribute-major fp64, owned by ws).

    Raises NonSPDError when p^T g <= 0."""
    n = b.numel()
    if n == 0:                        # empty scene: nothing to solve
        if stats is not None:
            stats.update(products=0, iterations=0, rr=0.0, bb=0.0)
        return torch.zeros(0, dtype=torch.float64, device=b.device)
    ws = ws or PCGWorkspace(n, b.device, cache.G, cache.P)
    G, P = (cache.G, cache.P) if cache.G * cache.P == n else (n, 1)
    nb = _lib.load().slm_backward_blocks(cache.G)
    dot_part = torch.zeros(nb, dtype=torch.float64, device=b.device)
    s = stream_ptr()
    ws.st.zero_()
    # p := b / Mf  (= x0, Alg. 1 line 4); g0 = A x0
    gt, gts = (cache.gtab, cache.gtab_stride) if ws.p_gm is not None and cache.G > 0 else (None, 0)
    call("slm_pcg_pinit", ptr(ws.p), ptr(ws.p_gm), ptr(b), ptr(M), G, P, ptr(gt), gts, s)
    _product(cache, ws.p, ws.g, lam, M, dot_part, timer, ws.p_gm)
    call("slm_pcg_update", 0, ptr(ws.x), ptr(ws.r), ptr(ws.p), ptr(ws.g), ptr(b), ptr(M), float(lam),
         ptr(ws.st), ptr(dot_part), nb, ptr(ws.part), n, s)
    call("slm_pcg_finalize", 0, ptr(ws.st), ptr(ws.part), s)
    # Iterations are queued one ahead of the host's exit check: the device
    # keeps a sticky stop flag (b = 0, converged, non-SPD) that turns the
    # vector kernels into no-ops, and the host reads iteration i-1's flag
    # (async copy + event) only after iteration i is queued, so the GPU never
    # drains between iterations; on an early exit the one product queued
    # ahead runs but its result is discarded by the gated update.
    for it in range(max_iters):
        call("slm_pcg_pupdate", ptr(ws.p), ptr(ws.p_gm), ptr(ws.r), ptr(M), ptr(ws.st), G, P, ptr(gt), gts, s)
        _product(cache, ws.p, ws.g, lam, M, dot_part, timer, ws.p_gm)
        call("slm_pcg_update", 1, ptr(ws.x), ptr(ws.r), ptr(ws.p), ptr(ws.g), ptr(b), ptr(M), float(lam),
             ptr(ws.st), ptr(dot_part), nb, ptr(ws.part), n, s)
        call("slm_pcg_finalize", 1, ptr(ws.st), ptr(ws.part), s)
        ws.stop_host[it % 2].copy_(ws.st[ST_STOP], non_blocking=True)
        ws.stop_ev[it % 2].record()
        if it > 0:
            ws.stop_ev[(it - 1) % 2].synchronize()
            if ws.stop_host[(it - 1) % 2] != 0.0:
                break
    st_h = ws.st.cpu()
    iters = int(st_h[ST_ITERS])
    if int(st_h[ST_FLAGS]) & 1:
        raise NonSPDError(f"p^T g = {float(st_h[ST_PG])} <= 0 at PCG iteration {iters}")
    if stats is not None:
        # b = 0: x = x0 = 0 and the reference makes no product; the
        # product of the zero x0 is still launched here but its result is unused
        stats["products"] = 1 + iters if float(st_h[ST_BB]) > 0.0 else 0
        stats["iterations"] = iters
        stats["rr"] = float(st_h[ST_RR])
        stats["bb"] = float(st_h[ST_BB])
    return ws.x


def _product(cache, p, g, lam, M, dot_part, timer, p_gm=None):
    """g = J^T W J p (fp32); dot_part = fp64 partials of p.(g + lam Mf p)."""
    if timer is None:
        cache.jtwj(p, g, lam, M, dot_part, lam_out=False, p_gm=p_gm)
    else:
        with timer:
            cache.jtwj(p, g, lam, M, dot_part, lam_out=False, p_gm=p_gm)


def pcg_solve(scene, cache, b: ParamVector, M_diag: ParamVector, lambda_reg: float, max_iters: int,
              stats: dict | None = None) -> ParamVector:
    """SPEC:391-399 signature. cache: CacheSet or jacobian.GradientCache."""
    cs = getattr(cache, "cacheset", cache)
    b.require_layout(Layout.ATTRIBUTE_MAJOR)
    M_diag.require_layout(Layout.ATTRIBUTE_MAJOR)
    bv = b.values.float().contiguous()
    Mv = M_diag.values.float().contiguous()
    x = pcg_run(cs, bv, Mv, float(lambda_reg), int(max_iters), stats=stats)
    return ParamVector(x.clone(), Layout.ATTRIBUTE_MAJOR, scene.num_gaussians, scene.params_per_gaussian)


class Combiner:
    """Eq. 7 accumulator in fp64: num += M * Delta, den += M; finalize
    num / max(den, 1e-12) to the fp32 direction.  The buffer is packed
    [num (n); den (n); energy; accepted batches] so that one all_reduce
    combines everything a rank contributes to the LM step."""

    def __init__(self, n: int, device):
        self.buf = torch.zeros(2 * n + 2, dtype=torch.float64, device=device)
        self.n = n
        self.accepted = 0
        self.energy = 0.0

    @property
    def num(self):
        return self.buf[: self.n]

    @property
    def den(self):
        return self.buf[self.n:2 * self.n]

    def add(self, delta: torch.Tensor, M: torch.Tensor):
        call("slm_combine_acc", ptr(self.num), ptr(self.den), ptr(delta), ptr(M), self.n, stream_ptr())
        self.accepted += 1

    def allreduce(self, group=None, world_size: int | None = None):
        """ONE packed all_reduce of [num; den; energy; accepted] when the
        subsets are sharded over several ranks (world_size > 1)."""
        import torch.distributed as dist
        if not (dist.is_available() and dist.is_initialized()):
            return
        w = dist.get_world_size(group) if world_size is None else world_size
        if w <= 1:
            return
        self.buf[2 * self.n:].copy_(torch.tensor([self.energy, float(self.accepted)], dtype=torch.float64))
        allreduce_sum_(self.buf, group)
        e, a = self.buf[2 * self.n:].tolist()
        self.energy, self.accepted = e, int(round(a))

    def finalize(self) -> torch.Tensor:
        out = torch.empty(self.n, dtype=torch.float32, device=self.buf.device)
        call("slm_combine_fin", ptr(out), ptr(self.num), ptr(self.den), self.n, stream_ptr())
        return out


class _GtPrefetch:
    """Host -> device copies of the next subset's ground-truth images on a side
    stream into one of two persistent device buffers (double buffering: a
    buffer is refilled only after the compute stream has consumed it, i.e.
    after the build of the subset two steps back).  Device-resident images
    pass through untouched."""

    def __init__(self, gts, device, shards):
        self.gts, self.device = gts, device
        self.host = any(not g.is_cuda for g in gts)
        self.pending = None
        if self.host:
            need = max((sum(self._nbytes(gts[i]) for i in views) for _, views in shards), default=0)
            self.buf = [torch.empty(max(need, 1), dtype=torch.uint8, device=device) for _ in range(2)]
            self.free = [None, None]
            self.stream = torch.cuda.Stream(device)

    @staticmethod
    def _nbytes(g):
        return 0 if g.is_cuda else (g.numel() * g.element_size() + 255) // 256 * 256

    def start(self, k, views):
        if not self.host:
            self.pending = ([self.gts[i] for i in views], None, None)
            return
        b = k % 2
        out, off = [], 0
        with torch.cuda.stream(self.stream):
            if self.free[b] is not None:
                self.stream.wait_event(self.free[b])
            for i in views:
                g = self.gts[i]
                if g.is_cuda:
                    out.append(g)
                    continue
                nb = g.numel() * g.element_size()
                dst = self.buf[b][off:off + nb].view(g.dtype).view(g.shape)
                dst.copy_(g, non_blocking=True)
                out.append(dst)
                off += self._nbytes(g)
            ev = torch.cuda.Event()
            ev.record(self.stream)
        self.pending = (out, ev, b)

    def take(self):
        out, ev, b = self.pending
        self.pending = None
        if ev is not None:
            torch.cuda.current_stream(self.device).wait_event(ev)
        return out, b

    def release(self, b):
        """The compute stream is done with buffer b once the queued work so far ran."""
        if b is not None:
            e = torch.cuda.Event()
            e.record(torch.cuda.current_stream(self.device))
            self.free[b] = e


@dataclass
class StepReport:
    delta: torch.Tensor
    energy: float
    batches_accepted: int
    entries: list
    pcg: list
    product_ms: list
    observed: torch.Tensor | None = None   # device count of gaussians with sum_i M_i(opacity) > 0
    n_gaussians: int = 0
    phases: dict | None = None             # per-phase ms (phase_timer given)

    @property
    def observed_fraction(self) -> float | None:
        """Fraction of gaussians observed by the step's subsets (nonzero
        opacity curvature in the combined den = sum_i M_i; one host read)."""
        if self.observed is None or self.n_gaussians == 0:
            return None
        return float(self.observed.item()) / self.n_gaussians


def lm_direction(scene, cameras, gts, schedule: BatchSchedule = BatchSchedule(), lambda_reg: float = 1e-4,
                 n_iters: int = 8, config=None, loss: LossConfig = LossConfig(), rank: int = 0,
                 world_size: int = 1, product_timer=None, keep_caches: bool = False,
                 phase_timer=None, offload=None) -> StepReport:
    """One LM update direction: per subset cache build, b, M, PCG, Eq. 7
    combine; subsets are sharded round-robin over ranks.

    Ground-truth images may live in (pinned) host memory: each subset's images
    are then copied on a side stream while the previous subset is solved."""
    n = scene.param_count
    T = phase_timer if phase_timer is not None else _NoTimer()
    T.tick("start")
    comb = Combiner(n, scene.device)
    ws = PCGWorkspace(n, scene.device, scene.num_gaussians, scene.params_per_gaussian)
    entries, pcg_stats, offloaded = [], [], []
    caches = []
    shards = list(schedule.shard(len(cameras), rank, world_size))
    fetch = _GtPrefetch(gts, scene.device, shards)
    if shards:
        fetch.start(0, shards[0][1])
    for k, (j, views) in enumerate(shards):
        gts_sub, buf = fetch.take()
        if k + 1 < len(shards):
            fetch.start(k + 1, shards[k + 1][1])
        cs = CacheSet(scene, [cameras[i] for i in views], gts_sub, config, loss, timer=phase_timer, offload=offload)
        offloaded.append(cs.offloaded_entries)
        T.tick("cache_tables")
        fetch.release(buf)  # the images are only read by the build's residual pass
        del gts_sub
        comb.energy += sum(cs.energies)
        entries.append(cs.E)
        b = cs.rhs()
        T.tick("rhs")
        M = cs.diag()
        T.tick("diag")
        st = {}
        try:
            d = pcg_run(cs, b, M, lambda_reg, n_iters, ws, stats=st, timer=product_timer)
        except NonSPDError:
            pcg_stats.append({"rejected": True})
            continue
        T.tick("pcg")
        pcg_stats.append(st)
        comb.add(d, M)
        T.tick("combine")
        if keep_caches and not caches:  # the first accepted batch (rho's frozen caches)
            cs.view_ids = list(views)
            caches.append(cs)
        del cs
    comb.allreduce(world_size=world_size)
    T.tick("allreduce")
    if comb.accepted == 0:
        raise NonSPDError("all batches rejected by PCG failure")
    # energy: the global sum over all subsets' views (every rank gets it)
    G = scene.num_gaussians
    rep = StepReport(comb.finalize(), comb.energy, comb.accepted, entries, pcg_stats, [],
                     (comb.den[10 * G:11 * G] > 0).sum() if G else None, G)
    T.tick("finalize")
    rep.offloaded_entries = offloaded
    if phase_timer is not None:
        rep.phases = phase_timer.summary()
    rep.caches = caches
    return rep


def solve_normal_equations_batched(scene, dataset, schedule: BatchSchedule, lambda_reg: float, n_iters: int = 8,
                                   config=None, loss: LossConfig = LossConfig()) -> ParamVector:
    """SPEC:400-408; dataset = (cameras, gt images)."""
    cameras, gts = dataset
    rep = lm_direction(scene, cameras, gts, schedule, lambda_reg, n_iters, config, loss)
    return ParamVector(rep.delta, Layout.ATTRIBUTE_MAJOR, scene.num_gaussians, scene.params_per_gaussian)
