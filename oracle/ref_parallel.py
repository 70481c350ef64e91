"""Multi-process driver of the REFERENCE's own products (TEST / BASELINE
INFRASTRUCTURE ONLY -- never imported by the product path).

Same algorithm as `ref_driver.lm_direction` (Alg. 1, PAPER:211-252 with the
SPEC:394-395 exit/abort rules and the SPEC:474 floors; Eq. 7, PAPER:323 /
SPEC:403; strided subsets SPEC:477), but the per-view work is spread over
worker processes so that every host core runs the reference's numpy code:

* each worker owns a fixed set of views (round-robin) and keeps their
  reference `GradientCache`s and `ResidualBundle`s alive between products
  (ref jacobian.py:360-416 build_cache, :93-121 sort_cache_by_gaussians);
* b (ref jacobian.py:411-413) and diag(J^T J) (ref :486-512) are summed over
  views by the parent in a FIXED view order, so the result does not depend on
  the worker count;
* one product A p = sum_views apply_jt(weight_residuals(apply_j(sort_x(p))))
  (ref jacobian.py:419-483) is evaluated view-parallel, the parent
  again summing per-view outputs in view order.

The products and the PCG arithmetic are therefore bit-identical to the
single-process `ref_driver` for any worker count.  Vectors travel through
POSIX shared memory (one [M] slot per view for the outputs), not pickles.
"""

from __future__ import annotations

import hashlib
import multiprocessing as mp
import os
import time
from multiprocessing import shared_memory

import numpy as np

from .ref_driver import import_reference

M_FLOOR = 1e-12


def digest(a) -> str:
    """sha256 of an index array as little-endian int64 (bit-exact index checks
    against fixtures without storing the arrays)."""
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a), dtype="<i8").tobytes()).hexdigest()


def cache_digests(cache, gc) -> dict:
    """Digests of the reference's pixel-sorted cache (ref jacobian.py:401-409)
    and of its gaussian-sorted permutation (ref jacobian.py:93-105)."""
    return dict(offsets=digest(cache.offsets), pixel_ids=digest(cache.pixel_ids),
                gaussian_ids=digest(cache.gaussian_ids), g_offsets=digest(gc.offsets),
                g_pixel_ids=digest(gc.pixel_ids), g_gaussian_ids=digest(gc.gaussian_ids),
                g_source_index=digest(gc.source_index))


def _worker(conn, views, scene_state, cams, gts, shm_in, shm_out, n):
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    R = import_reference()
    S, RA, RE, J = R["scene"], R["rasterizer"], R["residuals"], R["jacobian"]
    R["parallel"].set_num_threads(1)
    scene = S.GaussianScene(*scene_state)
    G, P = scene.num_gaussians, scene.params_per_gaussian
    sin = shared_memory.SharedMemory(name=shm_in)
    sout = shared_memory.SharedMemory(name=shm_out)
    pin = np.ndarray((n,), np.float64, buffer=sin.buf)
    out = np.ndarray((len(cams), n), np.float64, buffer=sout.buf)
    caches = {}
    try:
        while True:
            msg = conn.recv()
            op = msg[0]
            if op == "build":
                ph = {"render": 0.0, "residuals": 0.0, "build_cache": 0.0, "sort": 0.0}
                res = {}
                for v in views:
                    t0 = time.perf_counter()
                    rr = RA.render(scene, cams[v])
                    ph["render"] += time.perf_counter() - t0
                    t0 = time.perf_counter()
                    bundle = RE.compute_residuals(rr.image.rgb, gts[v])
                    ph["residuals"] += time.perf_counter() - t0
                    t0 = time.perf_counter()
                    bv, cache = J.build_cache(scene, cams[v], bundle, render_result=rr, view_id=v)
                    ph["build_cache"] += time.perf_counter() - t0
                    t0 = time.perf_counter()
                    gc = J.sort_cache_by_gaussians(cache)
                    ph["sort"] += time.perf_counter() - t0
                    caches[v] = (gc, bundle)
                    out[v] = bv.values
                    res[v] = (gc.entry_count, float(bundle.energy), cache_digests(cache, gc))
                conn.send((res, ph))
            elif op == "diag":
                t0 = time.perf_counter()
                for v in views:
                    out[v] = J.diag_jtj(scene, caches[v][0]).values
                conn.send(time.perf_counter() - t0)
            elif op == "product":
                t0 = time.perf_counter()
                pg = S.sort_x(S.ParamVector(pin.copy(), S.Layout.ATTRIBUTE_MAJOR, G, P))
                for v in views:
                    gc, bundle = caches[v]
                    u = J.weight_residuals(J.apply_j(pg, scene, gc), bundle)
                    out[v] = J.apply_jt(u, scene, gc).values
                conn.send(time.perf_counter() - t0)
            elif op == "energy":
                # energy of the scene x + gamma * delta (delta in pin, AM) per view
                gamma = msg[1]
                x = S.flatten(scene).values + gamma * pin
                sc = S.unflatten(S.ParamVector(x, S.Layout.ATTRIBUTE_MAJOR, G, P), scene.sh_degree,
                                 scene.background)
                res = {}
                for v in views:
                    rr = RA.render(sc, cams[v])
                    res[v] = float(RE.compute_residuals(rr.image.rgb, gts[v]).energy)
                conn.send(res)
            elif op == "stop":
                conn.send(None)
                break
    finally:
        sin.close()
        sout.close()


class RefPool:
    """Worker pool holding one image batch's reference caches."""

    def __init__(self, ref_scene, ref_cams, gts, workers: int | None = None):
        self.n = ref_scene.param_count
        self.V = len(ref_cams)
        self.workers = max(1, min(workers or os.cpu_count() or 1, self.V))
        self.shm_in = shared_memory.SharedMemory(create=True, size=max(8 * self.n, 8))
        self.shm_out = shared_memory.SharedMemory(create=True, size=max(8 * self.n * self.V, 8))
        self.pin = np.ndarray((self.n,), np.float64, buffer=self.shm_in.buf)
        self.out = np.ndarray((self.V, self.n), np.float64, buffer=self.shm_out.buf)
        st = (ref_scene.positions, ref_scene.rotations, ref_scene.log_scales, ref_scene.opacity_logits,
              ref_scene.sh_coeffs, ref_scene.sh_degree, ref_scene.background)
        ctx = mp.get_context("fork")
        self.procs, self.conns = [], []
        for w in range(self.workers):
            views = list(range(w, self.V, self.workers))
            a, b = ctx.Pipe()
            p = ctx.Process(target=_worker, args=(b, views, st, ref_cams, gts, self.shm_in.name,
                                                  self.shm_out.name, self.n), daemon=True)
            p.start()
            self.procs.append(p)
            self.conns.append(a)

    def _all(self, msg):
        for c in self.conns:
            c.send(msg)
        return [c.recv() for c in self.conns]

    def _sum_views(self):
        acc = np.zeros(self.n)
        for v in range(self.V):                   # fixed view order
            acc += self.out[v]
        return acc

    def build(self):
        """Returns (b, entries per view, energies per view, phase seconds);
        self.digests holds the per-view index digests."""
        res = self._all(("build",))
        ent, en, ph = [0] * self.V, [0.0] * self.V, {}
        self.digests = [None] * self.V
        for r, p in res:
            for v, (e, E, d) in r.items():
                ent[v], en[v], self.digests[v] = e, E, d
            for k, t in p.items():
                ph[k] = max(ph.get(k, 0.0), t)
        return self._sum_views(), ent, en, ph

    def diag(self):
        self._all(("diag",))
        return self._sum_views()

    def product(self, p):
        self.pin[:] = p
        self._all(("product",))
        return self._sum_views()

    def energies(self, delta, gamma):
        self.pin[:] = delta
        res = self._all(("energy", float(gamma)))
        out = [0.0] * self.V
        for r in res:
            for v, e in r.items():
                out[v] = e
        return out

    def close(self):
        try:
            self._all(("stop",))
        except Exception:
            pass
        for p in self.procs:
            p.join(timeout=10)
        self.shm_in.close()
        self.shm_out.close()
        self.shm_in.unlink()
        self.shm_out.unlink()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def pcg(A, b, M, lam, n_iters, stats=None):
    """Alg. 1, SPEC:394-395 exit/abort, SPEC:474 floors --
    identical arithmetic to lm_oracle.pcg / ref_driver.lm_direction."""
    Mf = np.maximum(M, M_FLOOR)
    bb = float(b @ b)
    x = b / Mf
    n_prod = 0
    if bb == 0.0:
        if stats is not None:
            stats.update(products=0, ok=True)
        return x, True
    r = b - (A(x) + lam * Mf * x)
    n_prod += 1
    z = r / Mf
    p = z.copy()
    rz = float(r @ z)
    ok = True
    for _ in range(n_iters):
        g = A(p) + lam * Mf * p
        n_prod += 1
        pg = float(p @ g)
        if not pg > 0.0:
            ok = False
            break
        a = rz / pg
        x = x + a * p
        r = r - a * g
        z = r / Mf
        rz_new = float(r @ z)
        p = z + (rz_new / rz) * p
        rz = rz_new
        if float(r @ r) < 0.01 * bb:
            break
    if stats is not None:
        stats.update(products=n_prod, ok=ok, rr=float(r @ r), bb=bb)
    return x, ok


def lm_direction(R, scene, cameras, gts, n_batches=1, lam=1e-4, n_iters=8, workers=None, trace=None,
                 phases=None):
    """Eq. 7 over strided batches with the reference's products (view-parallel).
    Returns (delta AM float64, total entries, phases)."""
    n = scene.param_count
    num, den = np.zeros(n), np.zeros(n)
    entries = 0
    ph = phases if phases is not None else {}
    for j in range(n_batches):
        views = list(range(j, len(cameras), n_batches))
        if not views:
            continue
        with RefPool(scene, [cameras[v] for v in views], [gts[v] for v in views], workers) as pool:
            t0 = time.perf_counter()
            b, ent, en, bph = pool.build()
            ph["build"] = ph.get("build", 0.0) + time.perf_counter() - t0
            t0 = time.perf_counter()
            M = pool.diag()
            ph["diag"] = ph.get("diag", 0.0) + time.perf_counter() - t0
            entries += sum(ent)
            st = {}
            t0 = time.perf_counter()
            x, ok = pcg(pool.product, b, M, lam, n_iters, st)
            ph["pcg"] = ph.get("pcg", 0.0) + time.perf_counter() - t0
            if trace is not None:
                trace.setdefault("batches", []).append(dict(views=views, b=b, M=M, x=x, stats=st, entries=ent,
                                                            energies=en, digests=pool.digests))
                if "pool_hook" in trace:
                    trace["pool_hook"](j, pool, x)
        if not ok:
            continue
        num += M * x
        den += M
    return num / np.maximum(den, M_FLOOR), entries, ph
