"""TEST INFRASTRUCTURE ONLY — Python (ctypes) front end of the CPU oracles.

Two oracles, both CPU, both used only by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs:

* ``Ref``  — oracle/_ref/libtreereg_ref.so: the reference's OWN sources
  (/root/reference/proj/core/src) compiled with the Eigen test shim
  (oracle/Makefile).  This is the parity anchor.
* ``Port`` — oracle/_port/libtrg_oracle.so: the plain-C restatement
  (oracle/trg_oracle.c), pinned bit-for-bit to ``Ref`` by
  tests/test_oracle_port.py.

Trees cross as dicts of numpy arrays (row-major 3x3 blocks):
weight[J], mean[J,3], cov[J,3,3], lambdas[J,3], axes[J,3,3], log_norm[J],
parent[J], first_child[J], child_count[J], level[J], max_level.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libtreereg_ref.so")
PORT_SO = os.path.join(HERE, "_port", "libtrg_oracle.so")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_u64p = C.POINTER(C.c_uint64)


def _d(a):
    return a.ctypes.data_as(_dp)


def _i(a):
    return a.ctypes.data_as(_ip)


def _u(a):
    return a.ctypes.data_as(_u64p)


def tree_capacity(max_level: int) -> int:
    return sum(8 ** (l + 1) for l in range(max_level))


def empty_tree(cap: int, max_level: int) -> dict:
    return dict(
        weight=np.zeros(cap), mean=np.zeros((cap, 3)), cov=np.zeros((cap, 3, 3)),
        lambdas=np.zeros((cap, 3)), axes=np.zeros((cap, 3, 3)), log_norm=np.zeros(cap),
        parent=np.zeros(cap, np.int32), first_child=np.zeros(cap, np.int32),
        child_count=np.zeros(cap, np.int32), level=np.zeros(cap, np.int32),
        max_level=max_level)


def trim_tree(t: dict, n: int) -> dict:
    out = {k: (v[:n].copy() if isinstance(v, np.ndarray) else v) for k, v in t.items()}
    return out


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"oracle error {code}: {msg}")
        self.code = code


@dataclass
class Moments:
    m0: np.ndarray
    m1: np.ndarray
    m2: np.ndarray | None
    total_points: int
    outliers: int
    density_evaluations: int
    total_mass: float


class Ref:
    """The reference implementation itself (shimmed build)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref`")
        L = C.CDLL(path)
        self.L = L
        L.ref_last_error.restype = C.c_char_p
        L.ref_bbox_diagonal.restype = C.c_double
        L.ref_tree_calibration_drift.restype = C.c_double
        L.ref_synthetic.argtypes = [C.c_char_p, C.c_size_t, C.c_uint64, _dp]
        L.ref_unit_normalized.argtypes = [_dp, C.c_size_t]
        L.ref_bbox_diagonal.argtypes = [_dp, C.c_size_t]
        L.ref_random_rigid_transform.argtypes = [C.c_double, C.c_double, C.c_uint64, C.c_int, _dp, _dp]
        L.ref_subsample.argtypes = [_dp, C.c_size_t, C.c_size_t, C.c_uint64, _dp]
        L.ref_build_tree.argtypes = [_dp, C.c_size_t, C.c_int, C.c_int, C.c_size_t, C.c_double,
                                     C.c_double, C.POINTER(C.c_void_p)]
        L.ref_build_flat_gmm.argtypes = [_dp, C.c_size_t, C.c_size_t, C.c_int, C.c_int, C.c_double,
                                         C.c_double, C.c_uint64, C.POINTER(C.c_void_p)]
        L.ref_responsibilities_dense.argtypes = [C.c_void_p, _dp, C.c_size_t, _dp, _dp, C.c_double,
                                                 _dp, _dp, _dp, _u64p, _dp]
        L.ref_read_cloud.argtypes = [C.c_char_p, C.c_int, _dp, C.c_size_t]
        L.ref_read_cloud.restype = C.c_longlong
        L.ref_tree_free.argtypes = [C.c_void_p]
        for f in ("ref_tree_size", "ref_tree_max_level", "ref_tree_calibration_drift",
                  "ref_tree_num_traces"):
            getattr(L, f).argtypes = [C.c_void_p]
        L.ref_tree_trace.argtypes = [C.c_void_p, C.c_int, _dp, C.c_int]
        L.ref_tree_export.argtypes = [C.c_void_p, _dp, _dp, _dp, _dp, _dp, _dp, _ip, _ip, _ip, _ip]
        L.ref_tree_import.argtypes = [C.c_int, C.c_int, _dp, _dp, _dp, _dp, _dp, _dp, _ip, _ip,
                                      _ip, _ip, C.POINTER(C.c_void_p)]
        L.ref_associate.argtypes = [C.c_void_p, _dp, C.c_size_t, _dp, _dp, C.c_double, C.c_int,
                                    _dp, _dp, _dp, _u64p, _dp]
        L.ref_associate_points.argtypes = [C.c_void_p, _dp, C.c_size_t, _dp, _dp, C.c_double,
                                           _ip, _dp]
        L.ref_solve_mstep.argtypes = [C.c_void_p, _dp, _dp, C.c_uint64, _dp, _dp, _dp, _dp, _dp, _ip]
        L.ref_register_with_tree.argtypes = [C.c_void_p, _dp, C.c_size_t, C.c_int, C.c_double,
                                             C.c_int, C.c_double, C.c_double, C.c_double, _dp, _dp,
                                             _ip, _ip, _dp, _dp, _u64p, _dp]
        L.ref_register_clouds.argtypes = [_dp, C.c_size_t, _dp, C.c_size_t, C.c_int, C.c_int,
                                          C.c_double, C.c_int, _dp, _dp, _ip, _ip, _dp, _dp]
        L.ref_eig_sym3.argtypes = [_dp, C.c_int, C.c_double, _dp, _dp]
        L.ref_set_threads.argtypes = [C.c_uint]
        L.ref_save_tree.argtypes = [C.c_void_p, C.c_char_p]
        L.ref_load_tree.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]

    def _chk(self, rc):
        if rc != 0:
            raise OracleError(rc, self.L.ref_last_error().decode())

    def set_threads(self, n: int):
        self.L.ref_set_threads(n)

    # ---- inputs (reference generators) ----
    def synthetic(self, kind: str, n: int, seed: int) -> np.ndarray:
        out = np.zeros((n, 3))
        self._chk(self.L.ref_synthetic(kind.encode(), n, seed, _d(out)))
        return out

    def unit_normalized(self, pts: np.ndarray) -> np.ndarray:
        p = np.ascontiguousarray(pts, dtype=np.float64).copy()
        self._chk(self.L.ref_unit_normalized(_d(p), len(p)))
        return p

    def bbox_diagonal(self, pts: np.ndarray) -> float:
        p = np.ascontiguousarray(pts, dtype=np.float64)
        return self.L.ref_bbox_diagonal(_d(p), len(p))

    def random_rigid_transform(self, rot_deg: float, trans: float, seed: int, trial: int = 0):
        R = np.zeros((3, 3))
        t = np.zeros(3)
        self._chk(self.L.ref_random_rigid_transform(rot_deg, trans, seed, trial, _d(R), _d(t)))
        return R, t

    # ---- tree ----
    def build_tree(self, pts, max_level=3, em_iters=8, min_points=32, eps=1e-4, abs_floor=1e-12):
        p = np.ascontiguousarray(pts, dtype=np.float64)
        h = C.c_void_p()
        self._chk(self.L.ref_build_tree(_d(p), len(p), max_level, em_iters, min_points, eps,
                                        abs_floor, C.byref(h)))
        try:
            t = self._export(h)
            t["calibration_drift"] = self.L.ref_tree_calibration_drift(h)
            traces = []
            buf = np.zeros(256)
            for i in range(self.L.ref_tree_num_traces(h)):
                k = self.L.ref_tree_trace(h, i, _d(buf), 256)
                traces.append(buf[:k].copy())
            t["ll_traces"] = traces
        finally:
            self.L.ref_tree_free(h)
        return t

    def build_flat_gmm(self, pts, j, max_level=3, em_iters=8, eps=1e-4, abs_floor=1e-12, seed=0):
        p = np.ascontiguousarray(pts, dtype=np.float64)
        h = C.c_void_p()
        self._chk(self.L.ref_build_flat_gmm(_d(p), len(p), j, max_level, em_iters, eps, abs_floor,
                                            C.c_uint64(seed), C.byref(h)))
        try:
            t = self._export(h)
            buf = np.zeros(4096)
            k = self.L.ref_tree_trace(h, 0, _d(buf), 4096) if self.L.ref_tree_num_traces(h) else 0
            t["ll_trace"] = buf[:k].copy()
        finally:
            self.L.ref_tree_free(h)
        return t

    def responsibilities_dense(self, comps, pts, R=None, t=None, floor=1e-300) -> Moments:
        R = np.eye(3) if R is None else np.ascontiguousarray(R, dtype=np.float64)
        t = np.zeros(3) if t is None else np.ascontiguousarray(t, dtype=np.float64)
        p = np.ascontiguousarray(pts, dtype=np.float64)
        J = len(comps["weight"])
        m0, m1, m2 = np.zeros(J), np.zeros((J, 3)), np.zeros((J, 3, 3))
        cnt = np.zeros(3, np.uint64)
        tm = np.zeros(1)
        h = self._import(comps)
        try:
            self._chk(self.L.ref_responsibilities_dense(h, _d(p), len(p), _d(R), _d(t), floor,
                                                        _d(m0), _d(m1), _d(m2), _u(cnt), _d(tm)))
        finally:
            self.L.ref_tree_free(h)
        return Moments(m0, m1, m2, int(cnt[0]), int(cnt[1]), int(cnt[2]), float(tm[0]))

    def read_cloud(self, path, fmt=0):
        n = self.L.ref_read_cloud(str(path).encode(), fmt, None, 0)
        if n < 0:
            raise RuntimeError(self.L.ref_last_error().decode())
        out = np.zeros((n, 3))
        self.L.ref_read_cloud(str(path).encode(), fmt, _d(out), n)
        return out

    def subsample(self, pts, n, seed):
        p = np.ascontiguousarray(pts, dtype=np.float64)
        out = np.zeros((int(n), 3))
        if self.L.ref_subsample(_d(p), len(p), int(n), int(seed), _d(out)) != 0:
            raise RuntimeError(self.L.ref_last_error().decode())
        return out

    def save_tree(self, tree: dict, path):
        """gmm.cpp:769-796 save_tree of a host tree (exported layout)."""
        h = self._import(tree)
        try:
            self._chk(self.L.ref_save_tree(h, str(path).encode()))
        finally:
            self.L.ref_tree_free(h)

    def load_tree(self, path) -> dict:
        """gmm.cpp:798-896 load_tree; raises OracleError (code 1/3) like the reference."""
        h = C.c_void_p()
        self._chk(self.L.ref_load_tree(str(path).encode(), C.byref(h)))
        try:
            return self._export(h)
        finally:
            self.L.ref_tree_free(h)

    def _export(self, h):
        n = self.L.ref_tree_size(h)
        t = empty_tree(n, self.L.ref_tree_max_level(h))
        self.L.ref_tree_export(h, _d(t["weight"]), _d(t["mean"]), _d(t["cov"]), _d(t["lambdas"]),
                               _d(t["axes"]), _d(t["log_norm"]), _i(t["parent"]),
                               _i(t["first_child"]), _i(t["child_count"]), _i(t["level"]))
        return t

    def _import(self, t):
        h = C.c_void_p()
        a = {k: np.ascontiguousarray(v) for k, v in t.items() if isinstance(v, np.ndarray)}
        self._chk(self.L.ref_tree_import(
            len(a["weight"]), int(t["max_level"]), _d(a["weight"]), _d(a["mean"]), _d(a["cov"]),
            _d(a["lambdas"]), _d(a["axes"]), _d(a["log_norm"]), _i(a["parent"]),
            _i(a["first_child"]), _i(a["child_count"]), _i(a["level"]), C.byref(h)))
        return h

    def associate(self, tree, pts, R=None, t=None, lambda_c=0.01, max_level=0) -> Moments:
        R = np.eye(3) if R is None else np.ascontiguousarray(R, dtype=np.float64)
        t = np.zeros(3) if t is None else np.ascontiguousarray(t, dtype=np.float64)
        p = np.ascontiguousarray(pts, dtype=np.float64)
        J = len(tree["weight"])
        m0, m1, m2 = np.zeros(J), np.zeros((J, 3)), np.zeros((J, 3, 3))
        cnt = np.zeros(3, np.uint64)
        tm = np.zeros(1)
        h = self._import(tree)
        try:
            self._chk(self.L.ref_associate(h, _d(p), len(p), _d(R), _d(t), lambda_c, max_level,
                                           _d(m0), _d(m1), _d(m2), _u(cnt), _d(tm)))
        finally:
            self.L.ref_tree_free(h)
        return Moments(m0, m1, m2, int(cnt[0]), int(cnt[1]), int(cnt[2]), float(tm[0]))

    def associate_points(self, tree, pts, R=None, t=None, lambda_c=0.01):
        R = np.eye(3) if R is None else np.ascontiguousarray(R, dtype=np.float64)
        t = np.zeros(3) if t is None else np.ascontiguousarray(t, dtype=np.float64)
        p = np.ascontiguousarray(pts, dtype=np.float64)
        node = np.zeros(len(p), np.int32)
        w = np.zeros(len(p))
        h = self._import(tree)
        try:
            self._chk(self.L.ref_associate_points(h, _d(p), len(p), _d(R), _d(t), lambda_c,
                                                  _i(node), _d(w)))
        finally:
            self.L.ref_tree_free(h)
        return node, w

    def solve_mstep(self, tree, m0, m1, total_points):
        h = self._import(tree)
        om, tr, dR, dt, sc = np.zeros(3), np.zeros(3), np.zeros((3, 3)), np.zeros(3), np.zeros(3)
        nv = C.c_int()
        m0 = np.ascontiguousarray(m0, dtype=np.float64)
        m1 = np.ascontiguousarray(m1, dtype=np.float64)
        try:
            self._chk(self.L.ref_solve_mstep(h, _d(m0), _d(m1), total_points, _d(om), _d(tr),
                                             _d(dR), _d(dt), _d(sc), C.byref(nv)))
        finally:
            self.L.ref_tree_free(h)
        return dict(omega=om, translation=tr, R=dR, t=dt, criterion_before=sc[0],
                    criterion_after=sc[1], condition=sc[2], n_vps=nv.value)

    def register_with_tree(self, tree, src, variant="adaptive", lambda_c=0.01, max_iters=50,
                           rot_tol=1e-5, trans_tol=1e-5, target_diag=0.0):
        h = self._import(tree)
        p = np.ascontiguousarray(src, dtype=np.float64)
        R, t = np.zeros((3, 3)), np.zeros(3)
        it, conv = C.c_int(), C.c_int()
        cb, ca = np.zeros(max_iters), np.zeros(max_iters)
        ev = np.zeros(max_iters, np.uint64)
        es = np.zeros(1)
        try:
            self._chk(self.L.ref_register_with_tree(
                h, _d(p), len(p), 1 if variant == "tree" else 0, lambda_c, max_iters, rot_tol,
                trans_tol, target_diag, _d(R), _d(t), C.byref(it), C.byref(conv), _d(cb), _d(ca),
                _u(ev), _d(es)))
        finally:
            self.L.ref_tree_free(h)
        n = it.value
        return dict(R=R, t=t, iterations=n, converged=bool(conv.value),
                    criterion_before=cb[:n].copy(), criterion_after=ca[:n].copy(),
                    eval_counts=ev[:n].copy(), em_seconds=float(es[0]))

    def register_clouds(self, tgt, src, level=3, variant="adaptive", lambda_c=0.01, max_iters=50):
        a = np.ascontiguousarray(tgt, dtype=np.float64)
        b = np.ascontiguousarray(src, dtype=np.float64)
        R, t = np.zeros((3, 3)), np.zeros(3)
        it, conv = C.c_int(), C.c_int()
        bs, es = np.zeros(1), np.zeros(1)
        self._chk(self.L.ref_register_clouds(_d(a), len(a), _d(b), len(b),
                                             {"adaptive": 0, "tree": 1, "flat": 2, "icp": 3}[variant], level,
                                             lambda_c,
                                             max_iters, _d(R), _d(t), C.byref(it), C.byref(conv),
                                             _d(bs), _d(es)))
        return dict(R=R, t=t, iterations=it.value, converged=bool(conv.value),
                    build_seconds=float(bs[0]), em_seconds=float(es[0]))

    def eig_sym3(self, m, floored=False, floor_value=0.0):
        m = np.ascontiguousarray(m, dtype=np.float64)
        lam, ax = np.zeros(3), np.zeros((3, 3))
        self._chk(self.L.ref_eig_sym3(_d(m), 1 if floored else 0, floor_value, _d(lam), _d(ax)))
        return lam, ax


class _TrgoTree(C.Structure):
    _fields_ = [("n_nodes", C.c_int), ("max_level", C.c_int), ("capacity", C.c_int),
                ("weight", _dp), ("mean", _dp), ("cov", _dp), ("lambdas", _dp), ("axes", _dp),
                ("log_norm", _dp), ("parent", _ip), ("first_child", _ip), ("child_count", _ip),
                ("level", _ip)]


class _TrgoCfg(C.Structure):
    _fields_ = [("max_level", C.c_int), ("em_iterations_per_node", C.c_int),
                ("min_points_per_node", C.c_size_t), ("eps", C.c_double),
                ("abs_floor", C.c_double)]


class _TrgoStats(C.Structure):
    _fields_ = [("entries_per_round", C.c_uint64 * 8), ("expanded_per_round", C.c_int * 8),
                ("calibration_passes", C.c_int), ("calibration_drift", C.c_double),
                ("calib_density_evals", C.c_uint64)]


class Port:
    """The plain-C restatement (oracle/trg_oracle.c)."""

    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle port`")
        L = C.CDLL(path)
        self.L = L
        L.trgo_last_error.restype = C.c_char_p
        L.trgo_bbox_diagonal.restype = C.c_double
        L.trgo_bbox_diagonal.argtypes = [_dp, C.c_size_t]
        L.trgo_build_tree.argtypes = [_dp, C.c_size_t, C.POINTER(_TrgoCfg), C.POINTER(_TrgoTree),
                                      C.POINTER(_TrgoStats)]
        L.trgo_associate.argtypes = [C.POINTER(_TrgoTree), _dp, C.c_size_t, _dp, _dp, C.c_double,
                                     C.c_int, _dp, _dp, _dp, _u64p, _dp, _ip, _dp]
        L.trgo_solve_mstep.argtypes = [C.POINTER(_TrgoTree), _dp, _dp, C.c_uint64, _dp, _dp, _dp,
                                       _dp, _dp, _ip]
        L.trgo_register_with_tree.argtypes = [C.POINTER(_TrgoTree), _dp, C.c_size_t, C.c_int,
                                              C.c_double, C.c_int, C.c_double, C.c_double,
                                              C.c_double, _dp, _dp, _ip, _ip, _dp, _dp, _u64p]
        L.trgo_eig_sym3.argtypes = [_dp, C.c_int, C.c_double, _dp, _dp]

    def _chk(self, rc):
        if rc != 0:
            raise OracleError(rc, self.L.trgo_last_error().decode())

    @staticmethod
    def _struct(t):
        s = _TrgoTree()
        s.n_nodes = len(t["weight"])
        s.max_level = int(t["max_level"])
        s.capacity = len(t["weight"])
        for k in ("weight", "mean", "cov", "lambdas", "axes", "log_norm"):
            setattr(s, k, _d(t[k]))
        for k in ("parent", "first_child", "child_count", "level"):
            setattr(s, k, _i(t[k]))
        return s

    def build_tree(self, pts, max_level=3, em_iters=8, min_points=32, eps=1e-4, abs_floor=1e-12,
                   stats_out: dict | None = None):
        p = np.ascontiguousarray(pts, dtype=np.float64)
        cap = tree_capacity(max_level)
        t = empty_tree(cap, max_level)
        s = self._struct(t)
        s.n_nodes = 0
        cfg = _TrgoCfg(max_level, em_iters, min_points, eps, abs_floor)
        st = _TrgoStats()
        self._chk(self.L.trgo_build_tree(_d(p), len(p), C.byref(cfg), C.byref(s), C.byref(st)))
        out = trim_tree(t, s.n_nodes)
        out["calibration_drift"] = st.calibration_drift
        if stats_out is not None:
            stats_out.update(entries_per_round=list(st.entries_per_round)[:max_level],
                             expanded_per_round=list(st.expanded_per_round)[:max_level],
                             calibration_passes=st.calibration_passes,
                             calib_density_evals=st.calib_density_evals)
        return out

    def associate(self, tree, pts, R=None, t=None, lambda_c=0.01, max_level=0, per_point=False):
        R = np.eye(3) if R is None else np.ascontiguousarray(R, dtype=np.float64)
        t = np.zeros(3) if t is None else np.ascontiguousarray(t, dtype=np.float64)
        p = np.ascontiguousarray(pts, dtype=np.float64)
        J = len(tree["weight"])
        m0, m1, m2 = np.zeros(J), np.zeros((J, 3)), np.zeros((J, 3, 3))
        cnt = np.zeros(3, np.uint64)
        tm = np.zeros(1)
        node = np.zeros(len(p), np.int32) if per_point else None
        w = np.zeros(len(p)) if per_point else None
        s = self._struct(tree)
        self._chk(self.L.trgo_associate(C.byref(s), _d(p), len(p), _d(R), _d(t), lambda_c,
                                        max_level, _d(m0), _d(m1), _d(m2), _u(cnt), _d(tm),
                                        _i(node) if per_point else None,
                                        _d(w) if per_point else None))
        m = Moments(m0, m1, m2, int(cnt[0]), int(cnt[1]), int(cnt[2]), float(tm[0]))
        return (m, node, w) if per_point else m

    def solve_mstep(self, tree, m0, m1, total_points):
        s = self._struct(tree)
        om, tr, dR, dt, sc = np.zeros(3), np.zeros(3), np.zeros((3, 3)), np.zeros(3), np.zeros(3)
        nv = C.c_int()
        m0 = np.ascontiguousarray(m0, dtype=np.float64)
        m1 = np.ascontiguousarray(m1, dtype=np.float64)
        self._chk(self.L.trgo_solve_mstep(C.byref(s), _d(m0), _d(m1), total_points, _d(om),
                                          _d(tr), _d(dR), _d(dt), _d(sc), C.byref(nv)))
        return dict(omega=om, translation=tr, R=dR, t=dt, criterion_before=sc[0],
                    criterion_after=sc[1], condition=sc[2], n_vps=nv.value)

    def register_with_tree(self, tree, src, variant="adaptive", lambda_c=0.01, max_iters=50,
                           rot_tol=1e-5, trans_tol=1e-5, target_diag=0.0):
        s = self._struct(tree)
        p = np.ascontiguousarray(src, dtype=np.float64)
        R, t = np.zeros((3, 3)), np.zeros(3)
        it, conv = C.c_int(), C.c_int()
        cb, ca = np.zeros(max_iters), np.zeros(max_iters)
        ev = np.zeros(max_iters, np.uint64)
        self._chk(self.L.trgo_register_with_tree(
            C.byref(s), _d(p), len(p), 1 if variant == "tree" else 0, lambda_c, max_iters,
            rot_tol, trans_tol, target_diag, _d(R), _d(t), C.byref(it), C.byref(conv), _d(cb),
            _d(ca), _u(ev)))
        n = it.value
        return dict(R=R, t=t, iterations=n, converged=bool(conv.value),
                    criterion_before=cb[:n].copy(), criterion_after=ca[:n].copy(),
                    eval_counts=ev[:n].copy())

    def eig_sym3(self, m, floored=False, floor_value=0.0):
        m = np.ascontiguousarray(m, dtype=np.float64)
        lam, ax = np.zeros(3), np.zeros((3, 3))
        self._chk(self.L.trgo_eig_sym3(_d(m), 1 if floored else 0, floor_value, _d(lam), _d(ax)))
        return lam, ax

    def bbox_diagonal(self, pts):
        p = np.ascontiguousarray(pts, dtype=np.float64)
        return self.L.trgo_bbox_diagonal(_d(p), len(p))


TREE_KEYS = ("weight", "mean", "cov", "lambdas", "axes", "log_norm", "parent", "first_child",
             "child_count", "level")
