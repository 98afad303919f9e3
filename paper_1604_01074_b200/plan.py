"""Device plan: one (model, tree, factor, scaling) resident in HBM.

A :class:`DevicePlan` owns a native ``tsmpc_plan`` (``include/tsmpc.h``).
Creating it uploads the fused operator blocks, bounds, scaling and tree arrays
once and lets the native runtime cut the tree into segments / levels / tiles
(``csrc/tsmpc_capi.cu:decompose``).  Per forecast only the stage cache moves
(``set_cache``); per solve only p (and an optional warm dual) go up and the
report comes down.
"""

from __future__ import annotations

import ctypes
import warnings
import weakref

import numpy as np

from . import _native as nat
from .errors import DeviceError, DimensionError, ValidationError
from .points import DualPoint, PrimalPoint

__all__ = ["DevicePlan", "plan_for", "tuned_plan"]


def _c(a, dtype=np.float64):
    return np.ascontiguousarray(np.asarray(a, dtype=dtype))


class DevicePlan:
    """``shard=(rank, world, nccl_id)`` creates one rank's plan of a tree split
    across GPUs (see ``shard.py``); results then cover ``edges()`` only."""

    def __init__(self, model, tree, factor, scaling=None, device: int = 0, shard=None,
                 warn_dense: bool = True):
        lib = nat.load_library()
        pb, keep = self._problem(model, tree, factor, scaling, warn_dense)
        if shard is None:
            handle = lib.tsmpc_plan_create(ctypes.byref(pb), int(device))
        else:
            rank, world, nid = shard
            idbuf = None if nid is None else (ctypes.c_uint8 * 128).from_buffer_copy(bytes(nid))
            handle = lib.tsmpc_plan_create_shard(ctypes.byref(pb), int(device), int(rank), int(world),
                                                 idbuf)
        if not handle:
            nat.check(nat.ERR_CUDA if "CUDA" in nat.last_error() or "device" in nat.last_error()
                      else nat.ERR_VALIDATION, "tsmpc_plan_create")
        self._bind(lib, handle, model, tree, factor, scaling, shard)

    def _problem(self, model, tree, factor, scaling, warn_dense=True):
        """The tsmpc_problem of (model, tree, factor, scaling) and the arrays it points at."""
        n_x, n_u, n_v = factor.n_x, factor.n_u, factor.n_v
        E = np.asarray(model.E, dtype=float)
        n_e = E.shape[0]
        pinv = E.T @ np.linalg.inv(E @ E.T)
        keep = {
            "A": _c(factor.A), "B": _c(model.B), "L": _c(factor.L), "Bbar": _c(factor.Bbar),
            "Phi": _c(factor.Phi), "Psi": _c(factor.Psi), "Wu": _c(model.Wu), "E": _c(E),
            "E_pinvT": _c(pinv.T), "u_min": _c(model.u_min), "u_max": _c(model.u_max),
            "x_min": _c(model.x_min), "x_max": _c(model.x_max), "x_s": _c(model.x_s),
            "stage_starts": _c(tree.stage_starts, np.int64), "anc": _c(tree.anc, np.int64),
            "child_start": _c(tree.child_start, np.int64),
            "child_stop": _c(tree.child_stop, np.int64), "prob": _c(tree.prob),
        }
        self.structured = None
        self.structured_error = None
        if np.count_nonzero(np.asarray(factor.A) - np.diag(np.diag(factor.A))) == 0:
            from .precompute import structured_basis
            try:
                sb = structured_basis(model, _BasisView(factor.L))
            except (ValidationError, np.linalg.LinAlgError) as exc:
                # the plan runs the dense fused-operator kernel; say why (plan.info()["path"])
                self.structured_error = f"{type(exc).__name__}: {exc}"
                if warn_dense:
                    warnings.warn(f"structured kernel basis unavailable ({self.structured_error}); "
                                  "the plan uses the dense DMMA kernel", RuntimeWarning, stacklevel=3)
            else:
                keep["Ls"], keep["lam_s"], keep["Ms"] = _c(sb.Ls), _c(sb.lam), _c(sb.M)
                self.structured = sb
        if scaling is not None:
            keep["sig_stage"] = _c(scaling.sig_stage)
            keep["zeta_stage"] = _c(scaling.zeta_stage)
            keep["psi_stage"] = _c(scaling.psi_stage)
        pb = nat.Problem()
        pb.n_x, pb.n_u, pb.n_v = n_x, n_u, n_v
        pb.n_d, pb.n_e, pb.N, pb.n_nodes = int(model.Gd.shape[1]), n_e, int(tree.N), int(tree.n_nodes)
        pb.W_alpha, pb.Wx, pb.gamma_d = float(model.W_alpha), float(model.Wx), float(model.gamma_d)
        for name, arr in keep.items():
            setattr(pb, name, nat.iptr(arr) if arr.dtype == np.int64 else nat.dptr(arr))
        return pb, keep

    def _bind(self, lib, handle, model, tree, factor, scaling, shard):
        self.shard = shard
        self._lib = lib
        self._h = ctypes.c_void_p(handle)
        self._fin = weakref.finalize(self, lib.tsmpc_plan_destroy, ctypes.c_void_p(handle))
        self.model, self.tree, self.factor, self.scaling = model, tree, factor, scaling
        self.n_x, self.n_u, self.n_v = factor.n_x, factor.n_u, factor.n_v
        self.n_nodes, self.n_edges = int(tree.n_nodes), int(tree.n_edges)
        self._cache_key = None

    @classmethod
    def create_multi(cls, model, tree, factor, scaling, devices) -> list["DevicePlan"]:
        """Rank r's shard plan on devices[r] for every r, NCCL communicators from
        ncclCommInitAll (one process drives all GPUs; tsmpc_plans_create_multi)."""
        lib = nat.load_library()
        head = cls.__new__(cls)
        pb, keep = head._problem(model, tree, factor, scaling)
        n = len(devices)
        devs = (ctypes.c_int32 * n)(*[int(d) for d in devices])
        handles = (ctypes.c_void_p * n)()
        nat.check(lib.tsmpc_plans_create_multi(ctypes.byref(pb), devs, n, handles), "tsmpc_plans_create_multi")
        plans = []
        for r in range(n):
            pl = head if r == 0 else cls.__new__(cls)
            if r:
                pl.structured, pl.structured_error = head.structured, head.structured_error
            pl._bind(lib, handles[r], model, tree, factor, scaling, (r, n, None))
            plans.append(pl)
        return plans

    # -- introspection -------------------------------------------------------
    def info(self) -> dict:
        keys = ("levels", "ctas", "tiles", "segments", "smem_bytes", "diag_A", "threads",
                "tile_rows", "sms", "collapsed", "trunk_edges", "sparse", "resident_ctas",
                "sharded", "rank", "world", "owned_chain_edges", "total_chains", "trunk_ctas",
                "wide", "exchange_doubles", "fill_rows_hbm", "peer_exchange")
        buf = np.zeros(len(keys), dtype=np.int64)
        nat.check(self._lib.tsmpc_plan_info(self._h, nat.iptr(buf), len(keys)), "tsmpc_plan_info")
        d = dict(zip(keys, (int(v) for v in buf)))
        d["path"] = self._lib.tsmpc_plan_path(self._h).decode()
        return d

    # -- in-kernel cut exchange over peer memory (shard plans) ------------------
    PEER_BLOB_BYTES = 160  # include/tsmpc.h TSMPC_PEER_BLOB_BYTES

    def peer_handles(self) -> bytes:
        """This rank's exchange blob (CUDA IPC handles of its receive rows and arrival
        counter, tsmpc_plan_peer_handles); all-gather it across the ranks."""
        buf = (ctypes.c_uint8 * self.PEER_BLOB_BYTES)()
        nat.check(self._lib.tsmpc_plan_peer_handles(self._h, buf), "tsmpc_plan_peer_handles")
        return bytes(buf)

    def peer_open(self, blobs) -> None:
        """Map every rank's exchange buffers (blobs in rank order); the solves then run
        both phases and the cut exchange in one launch (tsmpc_plan_peer_open)."""
        blob = b"".join(bytes(b) for b in blobs)
        buf = (ctypes.c_uint8 * len(blob)).from_buffer_copy(blob)
        nat.check(self._lib.tsmpc_plan_peer_open(self._h, buf, len(blobs)), "tsmpc_plan_peer_open")

    def peer_close(self) -> None:
        """Back to two launches and an ncclAllReduce per iteration."""
        nat.check(self._lib.tsmpc_plan_peer_close(self._h), "tsmpc_plan_peer_close")

    def edges(self, which: int = 0) -> np.ndarray:
        """Edge ids whose rows this plan computes (which=0) or the trunk edges (1)."""
        n = self._lib.tsmpc_plan_edges(self._h, int(which), None, 0)
        if n < 0:
            nat.check(n, "tsmpc_plan_edges")
        buf = np.zeros(max(n, 1), dtype=np.int64)
        self._lib.tsmpc_plan_edges(self._h, int(which), nat.iptr(buf), n)
        return buf[:n]

    def trial(self, iters: int = 40) -> float:
        """CUDA-event ms of `iters` iterations of the plan's kernel (timing trial)."""
        ms = ctypes.c_double()
        nat.check(self._lib.tsmpc_plan_trial(self._h, int(iters), ctypes.byref(ms)), "tsmpc_plan_trial")
        return ms.value

    def debug_timers(self) -> np.ndarray:
        """Phase cycle counters of CTA 0 since the last call (timer builds only)."""
        buf = (ctypes.c_uint64 * 16)()
        nat.check(self._lib.tsmpc_debug_timers(self._h, buf, 16), "tsmpc_debug_timers")
        return np.array(buf[:], dtype=np.uint64)

    # -- uploads -------------------------------------------------------------
    def set_cache(self, cache, model=None):
        """Upload a StageCache (+ the gap's prices / junction rhs / Gd d terms)."""
        key = (id(cache), id(cache.beta), id(cache.uhat), id(cache.evec))
        if key == self._cache_key:
            return
        E, m = self.n_edges, model if model is not None else self.model
        if cache.beta.shape != (E, self.n_v):
            raise DimensionError("stage cache does not match the tree shape")
        prices = jrhs = gdd = None
        demands = np.asarray(cache.demands, dtype=float)
        if getattr(m, "gap_inputs", True):
            prices = _c(np.stack([m.price(cache.k + j) for j in range(self.tree.N)]))
            jrhs = _c(-(demands @ np.asarray(m.Ed, dtype=float).T))
            gdd = _c(demands @ np.asarray(m.Gd, dtype=float).T)
        arrs = [_c(cache.beta), _c(cache.uhat), _c(cache.evec), _c(cache.q), prices, jrhs, gdd]
        nat.check(self._lib.tsmpc_set_cache(self._h, *map(nat.dptr, arrs)), "tsmpc_set_cache")
        self._cache_key = key
        self._cache_ref = cache

    def set_forecast(self, forecast, q, basis, model=None):
        """Build the stage cache of ``forecast`` on the device (reference
        ``elimination.py:114-158`` / ``tree.py:319-331``): only dhat (N x n_d), the
        stage prices, the reduced prices and q are uploaded."""
        m = model if model is not None else self.model
        tree = self.tree
        N = tree.N
        dhat = _c(forecast.dhat)
        if dhat.shape != (N, m.n_d):
            raise DimensionError(f"forecast dhat: shape {dhat.shape}, expected ({N}, {m.n_d})")
        q = _c(q)
        if q.shape != (self.n_u,):
            raise DimensionError(f"q: shape {q.shape}, expected ({self.n_u},)")
        if not getattr(self, "_cache_ops", False):
            pe = np.asarray(tree.edge_prob, dtype=float)
            pa = np.asarray(tree.parent_edge())
            pbar = pe.copy()
            inner = pa >= 0
            np.add.at(pbar, pa[inner], pe[inner])
            ops = [_c(basis.part_map), _c(m.Gd), _c(m.Ed), _c(basis.Rhat), _c(tree.edge_eps), _c(pbar)]
            nat.check(self._lib.tsmpc_set_cache_operators(self._h, int(m.n_d), *map(nat.dptr, ops)),
                      "tsmpc_set_cache_operators")
            self._cache_ops = True
            self._basis_L = np.asarray(basis.L)
        k = int(forecast.k)
        prices = _c(np.stack([m.price(k + j) for j in range(N)]))
        abar = _c(m.W_alpha * (prices @ self._basis_L))
        nat.check(self._lib.tsmpc_set_forecast(self._h, nat.dptr(dhat), nat.dptr(q), nat.dptr(prices),
                                               nat.dptr(abar)), "tsmpc_set_forecast")
        self._cache_key = ("forecast", id(forecast), k)
        self._cache_ref = None

    def get_cache(self):
        """(beta, uhat, evec) currently on the device (tests)."""
        E = self.n_edges
        beta, uhat, evec = np.empty((E, self.n_v)), np.empty((E, self.n_u)), np.empty((E, self.n_x))
        nat.check(self._lib.tsmpc_get_cache(self._h, nat.dptr(beta), nat.dptr(uhat), nat.dptr(evec)),
                  "tsmpc_get_cache")
        return beta, uhat, evec

    # -- solver entry points ---------------------------------------------------
    def solve(self, p, iters: int, lam: float, warm: DualPoint | None = None,
              theta=None, coef=None, record_residuals: bool = False,
              skip_gap: bool = False, keep_device: bool = False,
              warm_device: bool = False, tol: float | None = None,
              check_every: int = 25, gap_trace: bool = False) -> dict:
        """One APG solve (engine.py:485-601).  ``keep_device``: leave the iterates in
        HBM (only u0, residual and gap come back); ``warm_device``: start from the
        previous solve's final dual, still in HBM (closed-loop warm start);
        ``gap_trace``: also the duality gap after every iteration (implies
        ``record_residuals``; engine.py:577-582)."""
        record_residuals = record_residuals or gap_trace
        out, res, trace = self._result_buffers(iters, keep_device, record_residuals)
        gtrace = np.empty(iters) if gap_trace else None
        res.gap_trace = nat.dptr(gtrace)
        flags = ((nat.RECORD_RESIDUALS if record_residuals else 0)
                 | (nat.SKIP_GAP if skip_gap else 0) | (nat.KEEP_DEVICE if keep_device else 0)
                 | (nat.WARM_DEVICE if warm_device else 0) | (nat.GAP_TRACE if gap_trace else 0))
        ws = wz = wp = None
        if warm is not None:
            ws, wz, wp = _c(warm.sig), _c(warm.zeta), _c(warm.psi)
        th = _c(theta) if theta is not None else None
        cf = _c(coef) if coef is not None else None
        pv = _c(p)
        nat.check(self._lib.tsmpc_set_stopping(self._h, float(tol) if tol else 0.0, int(check_every)),
                  "tsmpc_set_stopping")
        rc = self._lib.tsmpc_solve(self._h, nat.dptr(pv), int(iters), float(lam),
                                   nat.dptr(ws), nat.dptr(wz), nat.dptr(wp),
                                   nat.dptr(th), nat.dptr(cf), flags, ctypes.byref(res))
        nat.check(rc, "tsmpc_solve")
        d = self._result_dict(out, res, trace)
        n = d["iterations"]
        if trace is not None and n < iters:  # stopped early: the trace covers n iterations
            d["resid_trace"] = trace[:n]
        d["gap_trace"] = gtrace
        return d

    def _result_buffers(self, iters: int, keep_device: bool, record_residuals: bool):
        E, n_x, n_u, n = self.n_edges, self.n_x, self.n_u, self.n_nodes
        shapes = {"u0": (n_u,)}
        if not keep_device:
            shapes.update({"x": (n, n_x), "u": (E, n_u), "x_avg": (n, n_x), "u_avg": (E, n_u),
                           "dual_sig": (E, n_x), "dual_zeta": (E, n_x), "dual_psi": (E, n_u)})
        # result arrays in page-locked memory (pooled) when available
        arrs = nat.PINNED.arrays(list(shapes.values()))
        if arrs is None:
            arrs = [np.empty(sh) for sh in shapes.values()]
        out = dict(zip(shapes, arrs))
        if keep_device:
            out.update({"x": np.empty((n, n_x)), "u": np.empty((E, n_u)),
                        "x_avg": np.empty((n, n_x)), "u_avg": np.empty((E, n_u)),
                        "dual_sig": np.empty((E, n_x)), "dual_zeta": np.empty((E, n_x)),
                        "dual_psi": np.empty((E, n_u))})
        res = nat.Result()
        res.u0 = nat.dptr(out["u0"])
        if not keep_device:
            for k, v in out.items():
                setattr(res, k, nat.dptr(v))
        trace = np.empty(iters) if record_residuals else None
        res.resid_trace = nat.dptr(trace)
        return out, res, trace

    @staticmethod
    def _result_dict(out: dict, res, trace) -> dict:
        out.update(residual_inf=float(res.residual_inf), gap=float(res.gap),
                   device_ms=float(res.device_ms), iterations=int(res.iterations),
                   device_total_ms=float(res.device_total_ms),
                   kernel_launches=int(res.kernel_launches),
                   resid_trace=trace)
        return out

    def solve_step(self, w: DualPoint, p) -> PrimalPoint:
        x = np.empty((self.n_nodes, self.n_x))
        u = np.empty((self.n_edges, self.n_u))
        args = [_c(w.sig), _c(w.zeta), _c(w.psi), _c(p)]
        nat.check(self._lib.tsmpc_solve_step(self._h, *map(nat.dptr, args), nat.dptr(x),
                                             nat.dptr(u)), "tsmpc_solve_step")
        return PrimalPoint(x, u)

    def prox(self, t, lam: float, scaled: bool):
        rows = t.sig.shape[0]
        o = [np.empty_like(_c(t.sig)), np.empty_like(_c(t.zeta)), np.empty_like(_c(t.psi))]
        args = [_c(t.sig), _c(t.zeta), _c(t.psi)]
        nat.check(self._lib.tsmpc_prox(self._h, int(rows), *map(nat.dptr, args), float(lam),
                                       1 if scaled else 0, *map(nat.dptr, o)), "tsmpc_prox")
        return o

    def dual_operator_begin(self, beta0):
        nat.check(self._lib.tsmpc_dual_operator_begin(self._h, nat.dptr(_c(beta0))),
                  "tsmpc_dual_operator_begin")
        nat.check(self._lib.tsmpc_dual_operator_set_ones(self._h), "tsmpc_dual_operator_set_ones")

    def dual_operator_step(self):
        v = [ctypes.c_double(), ctypes.c_double(), ctypes.c_double()]
        rc = self._lib.tsmpc_dual_operator_step(self._h, *(ctypes.byref(x) for x in v))
        if rc != nat.OK and v[2].value == 0.0:
            nat.check(nat.ERR_VALIDATION, "power iteration")
        nat.check(rc, "tsmpc_dual_operator_step")
        return v[0].value, v[1].value, v[2].value


class _BasisView:
    """The slice of EliminationBasis that structured_basis reads."""

    def __init__(self, L):
        self.L = np.asarray(L)
        self.n_v = self.L.shape[1]


_PLANS: dict = {}
_MAX_PLANS = 6


def describe_tree(tree, max_ctas: int = 148, collapse: bool = True) -> dict:
    """Host-only view of the device decomposition of ``tree`` (no GPU needed).

    Returns levels, ctas, tiles, segments, rows, trunk_edges, max_rows_per_cta,
    max_tiles_per_cta and max_trunk_path as ``tsmpc_plan_create`` would build
    them with ``max_ctas`` CTAs (``collapse``: diagonal-A collapsed-trunk mode).
    """
    lib = nat.load_library()
    keep = {"stage_starts": _c(tree.stage_starts, np.int64), "anc": _c(tree.anc, np.int64),
            "child_start": _c(tree.child_start, np.int64),
            "child_stop": _c(tree.child_stop, np.int64), "prob": _c(tree.prob)}
    pb = nat.Problem()
    pb.N, pb.n_nodes = int(tree.N), int(tree.n_nodes)
    for name, arr in keep.items():
        setattr(pb, name, nat.iptr(arr) if arr.dtype == np.int64 else nat.dptr(arr))
    buf = np.zeros(9, dtype=np.int64)
    nat.check(lib.tsmpc_describe_tree(ctypes.byref(pb), int(max_ctas), 1 if collapse else 0,
                                      nat.iptr(buf), 9), "tsmpc_describe_tree")
    keys = ("levels", "ctas", "tiles", "segments", "rows", "trunk_edges", "max_rows_per_cta",
            "max_tiles_per_cta", "max_trunk_path")
    return dict(zip(keys, (int(v) for v in buf)))


def describe_sparse(model, tree, factor, max_ctas: int = 148, smem_limit: int = 232448) -> dict:
    """Host-only view of the structured-basis kernel plan (no GPU needed)."""
    from .precompute import structured_basis
    lib = nat.load_library()
    sb = structured_basis(model, _BasisView(factor.L))
    keep = {"stage_starts": _c(tree.stage_starts, np.int64), "anc": _c(tree.anc, np.int64),
            "child_start": _c(tree.child_start, np.int64),
            "child_stop": _c(tree.child_stop, np.int64), "prob": _c(tree.prob),
            "B": _c(model.B), "Ls": _c(sb.Ls), "lam_s": _c(sb.lam)}
    pb = nat.Problem()
    pb.n_x, pb.n_u, pb.n_v = factor.n_x, factor.n_u, factor.n_v
    pb.N, pb.n_nodes = int(tree.N), int(tree.n_nodes)
    for name, arr in keep.items():
        setattr(pb, name, nat.iptr(arr) if arr.dtype == np.int64 else nat.dptr(arr))
    keys = ("ctas", "tiles", "chains", "trunk_edges", "resident_ctas", "max_rows", "max_needs",
            "smem_bytes", "trunk_ctas", "wide", "tile_rows")
    buf = np.zeros(len(keys), dtype=np.int64)
    nat.check(lib.tsmpc_describe_sparse(ctypes.byref(pb), int(max_ctas), int(smem_limit),
                                        nat.iptr(buf), len(keys)), "tsmpc_describe_sparse")
    return dict(zip(keys, (int(v) for v in buf)))


def describe_shard(model, tree, factor, rank: int, world: int, max_ctas: int = 148,
                   smem_limit: int = 232448) -> dict:
    """Host-only view of one shard of the structured-basis plan (no GPU needed):
    the chain partition, the trunk positions this rank computes, and the size of
    the per-iteration cut exchange."""
    from .precompute import structured_basis
    lib = nat.load_library()
    sb = structured_basis(model, _BasisView(factor.L))
    keep = {"stage_starts": _c(tree.stage_starts, np.int64), "anc": _c(tree.anc, np.int64),
            "child_start": _c(tree.child_start, np.int64),
            "child_stop": _c(tree.child_stop, np.int64), "prob": _c(tree.prob),
            "B": _c(model.B), "Ls": _c(sb.Ls), "lam_s": _c(sb.lam)}
    pb = nat.Problem()
    pb.n_x, pb.n_u, pb.n_v = factor.n_x, factor.n_u, factor.n_v
    pb.N, pb.n_nodes = int(tree.N), int(tree.n_nodes)
    for name, arr in keep.items():
        setattr(pb, name, nat.iptr(arr) if arr.dtype == np.int64 else nat.dptr(arr))
    keys = ("ctas", "owned_chains", "owned_rows", "trunk_edges", "total_chains",
            "owned_trunk_nodes", "smem_bytes", "own_trunk_positions", "mixed_positions",
            "cut_positions", "exchange_rows", "exchange_doubles", "result_rows")
    buf = np.zeros(len(keys), dtype=np.int64)
    edges = np.zeros(max(1, tree.n_edges), dtype=np.int64)
    nat.check(lib.tsmpc_describe_shard(ctypes.byref(pb), int(max_ctas), int(smem_limit), int(rank),
                                       int(world), nat.iptr(buf), len(keys), nat.iptr(edges),
                                       tree.n_edges), "tsmpc_describe_shard")
    d = dict(zip(keys, (int(v) for v in buf)))
    d["edges"] = edges[:d["result_rows"]]  # rows this shard computes: its chains, own + mixed trunk
    return d


def tuned_plan(model, tree, factor, scaling=None, device: int = 0, candidates: int = 4,
               trial_iters: int = 40) -> DevicePlan:
    """A plan whose device buffers sit at a fast placement.

    The wide kernels' iteration time depends on where the plan's buffers land in
    device memory (identical SMPC8 plans at different addresses ran 57-70
    us/iteration, reproducibly per plan: L2 set / DRAM bank conflicts between rows
    read back to back; tools/layout_probe.py).  For wide plans this creates
    `candidates` plans (kept alive together, so each lands elsewhere), times a short
    trial of each (tsmpc_plan_trial; the cost does not depend on the data) and keeps
    the fastest.  Other plans are returned as created.  TSMPC_NO_LAYOUT_TUNE=1
    disables the search."""
    import os
    first = DevicePlan(model, tree, factor, scaling, device)
    info = first.info()
    if not (info["sparse"] and info["wide"]) or info["sharded"] or candidates <= 1 \
            or os.environ.get("TSMPC_NO_LAYOUT_TUNE"):
        return first
    plans = [first] + [DevicePlan(model, tree, factor, scaling, device) for _ in range(candidates - 1)]
    times = []
    for pl in plans:
        pl.trial(trial_iters)  # warm-up
        times.append(min(pl.trial(trial_iters) for _ in range(2)))
    best = int(np.argmin(times))
    keep = plans[best]
    keep.layout_trials_ms = times
    del plans
    return keep


def plan_for(model, tree, factor, scaling=None, device: int = 0) -> DevicePlan:
    """Cached plan per (model, tree, factor, scaling) object identity."""
    key = (id(model), id(tree), id(factor), id(scaling), device)
    hit = _PLANS.get(key)
    if hit is not None and hit.model is model and hit.tree is tree and hit.factor is factor \
            and hit.scaling is scaling:
        _PLANS[key] = _PLANS.pop(key)  # LRU touch
        return hit
    if len(_PLANS) >= _MAX_PLANS:
        _PLANS.pop(next(iter(_PLANS)))
    plan = tuned_plan(model, tree, factor, scaling, device)
    _PLANS[key] = plan
    return plan


def release_plans():
    _PLANS.clear()


def require_device():
    if nat.device_count() < 1:
        raise DeviceError("no CUDA device visible to libtsmpc")
