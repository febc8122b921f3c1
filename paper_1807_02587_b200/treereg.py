"""Host-side mirror of the reference's hot-path API (namespace treereg).

Same names, argument meaning and error behaviour as
/root/reference/proj/core/include/treereg/{gmm,association,mstep,registration}.hpp,
so parity tests read like the reference's own tests.  Every call goes
through the C-ABI of libtrg_cuda.so (include/treereg_b200.h) and runs on the
GPU; nothing here computes on the CPU beyond argument packing.

Exceptions mirror the reference's C++ types:
  std::invalid_argument   -> InvalidArgument (ValueError)
  std::domain_error       -> DomainError (ArithmeticError)
  std::runtime_error      -> RuntimeError
  std::out_of_range       -> IndexError
  DegenerateGeometryError -> DegenerateGeometryError (RuntimeError)
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import (AssocConfigC, BuildDiagC, MomentsC, MStepSolutionC, ModelConfigC, RegConfigC,
                   RegResultC, TreeC, dp, ip, u64p)


class InvalidArgument(ValueError):
    pass


class DomainError(ArithmeticError):
    pass


class DegenerateGeometryError(RuntimeError):
    pass


class CudaError(RuntimeError):
    pass


def _raise(rc: int, host: bool = False):
    msg = _lib.host_last_error() if host else _lib.last_error()
    if rc == _lib.TRG_EINVAL:
        raise InvalidArgument(msg)
    if rc == _lib.TRG_EDOMAIN:
        raise DomainError(msg)
    if rc == _lib.TRG_ERANGE:
        raise IndexError(msg)
    if rc == _lib.TRG_EDEGENERATE:
        raise DegenerateGeometryError(msg)
    if rc in (_lib.TRG_ECUDA, _lib.TRG_ENCCL):
        raise CudaError(msg)
    raise RuntimeError(msg)


def _chk(rc: int):
    if rc != 0:
        _raise(rc)


def _chk_host(rc: int):
    if rc != 0:
        _raise(rc, host=True)


def _d(a: np.ndarray):
    return a.ctypes.data_as(dp)


def _i(a: np.ndarray):
    return a.ctypes.data_as(ip)


# ------------------------------------------------------------------ context
class Context:
    """One CUDA device + stream + workspace (trg_ctx)."""

    def __init__(self, device: int = 0):
        self.h = C.c_void_p()
        _chk(_lib.lib().trg_ctx_create(device, C.byref(self.h)))
        self.device = device

    def close(self):
        if self.h:
            _lib.lib().trg_ctx_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def sms(self) -> int:
        return _lib.lib().trg_device_sms(self.h)

    def set_sm_budget(self, sms: int) -> None:
        """Limit this context's persistent grids to `sms` SMs (0 = all)."""
        _chk(_lib.lib().trg_ctx_set_sm_budget(self.h, int(sms)))

    @property
    def kernel_launches(self) -> int:
        return int(_lib.lib().trg_kernel_launches(self.h))

    def transfer_bytes(self):
        """(host->device, device->host) bytes copied by this context so far."""
        a, b = C.c_uint64(), C.c_uint64()
        _lib.lib().trg_ctx_transfer_bytes(self.h, C.byref(a), C.byref(b))
        return int(a.value), int(b.value)

    @property
    def stream(self) -> int:
        return int(_lib.lib().trg_ctx_stream(self.h) or 0)


_DEFAULT: Context | None = None


def default_context() -> Context:
    global _DEFAULT
    if _DEFAULT is None:
        _DEFAULT = Context(0)
    return _DEFAULT


# ------------------------------------------------------------------ configs
@dataclass
class ModelConfig:  # gmm.hpp:34-41
    em_iterations_per_node: int = 8
    min_points_per_node: int = 32
    cov_regularization_epsilon: float = 1e-4
    cov_regularization_absolute: float = 1e-12
    rng_seed: int = 0
    max_level: int = 3

    def c(self) -> ModelConfigC:
        return ModelConfigC(self.em_iterations_per_node, self.min_points_per_node,
                            self.cov_regularization_epsilon, self.cov_regularization_absolute,
                            self.rng_seed, self.max_level)


@dataclass
class AssocConfig:  # association.hpp:34-40
    lambda_c: float = 0.01
    max_level: int = 0
    outlier_floor: float = 1e-300
    deterministic: bool = True

    def c(self) -> AssocConfigC:
        return AssocConfigC(self.lambda_c, self.max_level, self.outlier_floor,
                            1 if self.deterministic else 0)


@dataclass
class Variant:  # registration.hpp:17-25
    kind: str = "adaptive"  # "adaptive" | "tree" | "flat" | "icp"
    param: int = 3

    @staticmethod
    def parse(text: str) -> "Variant":
        head, _, tail = text.partition(":")
        if head == "icp" and not tail:
            return Variant("icp", 0)
        if head not in ("adaptive", "tree", "flat"):
            raise InvalidArgument(f"unsupported variant '{text}' (adaptive:L, tree:L, flat:J, icp)")
        if not tail:
            raise InvalidArgument(f"variant '{head}' needs a parameter, e.g. {head}:3")
        try:
            p = int(tail)
        except ValueError:
            raise InvalidArgument(f"bad variant parameter in '{text}'") from None
        if p < 1:
            raise InvalidArgument("variant parameter must be >= 1")
        return Variant(head, p)

    def name(self) -> str:
        if self.kind == "icp":
            return "ICP"
        if self.kind == "flat":
            return f"GMM J={self.param}"
        return ("Adaptive L" if self.kind == "adaptive" else "GMM-Tree L") + str(self.param)


@dataclass
class RigidTransform:  # geometry.hpp:26-56
    rotation: np.ndarray = field(default_factory=lambda: np.eye(3))
    translation: np.ndarray = field(default_factory=lambda: np.zeros(3))

    @staticmethod
    def identity() -> "RigidTransform":
        return RigidTransform()

    def __call__(self, p):
        return np.asarray(p) @ self.rotation.T + self.translation

    def __mul__(self, rhs: "RigidTransform") -> "RigidTransform":
        return RigidTransform(self.rotation @ rhs.rotation,
                              self.rotation @ rhs.translation + self.translation)

    def inverse(self) -> "RigidTransform":
        rt = self.rotation.T
        return RigidTransform(rt, -(rt @ self.translation))

    def rotation_angle(self) -> float:
        c = np.clip((np.trace(self.rotation) - 1.0) * 0.5, -1.0, 1.0)
        return float(np.arccos(c))


@dataclass
class RegistrationConfig:  # registration.hpp:27-36
    variant: Variant = field(default_factory=Variant)
    lambda_c: float = 0.01
    max_em_iterations: int = 50
    rotation_tol: float = 1e-5
    translation_tol: float = 1e-5
    initial_transform: RigidTransform = field(default_factory=RigidTransform)
    model_config: ModelConfig = field(default_factory=ModelConfig)
    deterministic: bool = True
    # not in the reference: FP32 association scoring in the EM (SURVEY 7.2 fast
    # path; off = the reference's FP64 parity mode)
    fast_scoring: bool = False

    def c(self) -> RegConfigC:
        r = RegConfigC()
        r.variant_kind = {"adaptive": 0, "tree": 1, "flat": 2, "icp": 3}[self.variant.kind]
        r.variant_param = self.variant.param
        r.lambda_c = self.lambda_c
        r.max_em_iterations = self.max_em_iterations
        r.rotation_tol = self.rotation_tol
        r.translation_tol = self.translation_tol
        R = np.ascontiguousarray(self.initial_transform.rotation, dtype=np.float64).ravel()
        for k in range(9):
            r.initial_R[k] = R[k]
        for k in range(3):
            r.initial_t[k] = float(self.initial_transform.translation[k])
        r.model_config = self.model_config.c()
        r.fast_scoring = 1 if self.fast_scoring else 0
        return r


# ------------------------------------------------------------------ clouds
def _points(cloud) -> np.ndarray:
    p = np.ascontiguousarray(cloud, dtype=np.float64)
    if p.ndim != 2 or p.shape[1] != 3:
        raise InvalidArgument("point cloud must be an (N, 3) array")
    return p


def _cloud_ptr(cloud, ctx):
    """(pointer, n, on_device) for a numpy (host) or torch CUDA tensor.  A
    CUDA tensor may still be in production on torch's current stream: the
    context's stream waits for it (trg_ctx_wait_stream) before any kernel of
    the call reads it."""
    if hasattr(cloud, "is_cuda") and cloud.is_cuda:
        if cloud.dtype.__str__() != "torch.float64" or cloud.dim() != 2 or cloud.shape[1] != 3:
            raise InvalidArgument("device point cloud must be a contiguous (N, 3) float64 tensor")
        if not cloud.is_contiguous():
            raise InvalidArgument("device point cloud must be contiguous")
        import torch
        _chk(_lib.lib().trg_ctx_wait_stream(ctx.h, C.c_void_p(torch.cuda.current_stream(cloud.device).cuda_stream)))
        return C.c_void_p(cloud.data_ptr()), int(cloud.shape[0]), 1, cloud
    p = _points(cloud)
    return p.ctypes.data_as(C.c_void_p), len(p), 0, p


# ------------------------------------------------------------------ model
class GmmTree:
    """Device-resident GMM tree (gmm.hpp:56-67).  Host arrays are fetched
    lazily (``.host()``) for inspection and parity checks."""

    def __init__(self, handle: C.c_void_p, ctx: Context):
        self.h = handle
        self.ctx = ctx
        self._host = None

    def __del__(self):
        try:
            if self.h:
                _lib.lib().trg_tree_free(self.ctx.h, self.h)
                self.h = C.c_void_p()
        except Exception:
            pass

    def size(self) -> int:
        return _lib.lib().trg_tree_size(self.h)

    def host(self) -> dict:
        if self._host is None:
            J = self.size()
            t = dict(weight=np.zeros(J), mean=np.zeros((J, 3)), cov=np.zeros((J, 3, 3)),
                     lambdas=np.zeros((J, 3)), axes=np.zeros((J, 3, 3)), log_norm=np.zeros(J),
                     parent=np.zeros(J, np.int32), first_child=np.zeros(J, np.int32),
                     child_count=np.zeros(J, np.int32), level=np.zeros(J, np.int32))
            s = _tree_struct(t, 0, J)
            _chk(_lib.lib().trg_tree_download(self.ctx.h, self.h, C.byref(s)))
            t["max_level"] = s.max_level
            self._host = t
        return self._host

    @property
    def max_level(self) -> int:
        return int(self.host()["max_level"])

    @staticmethod
    def from_host(t: dict, ctx: Context | None = None) -> "GmmTree":
        """Upload a host tree (e.g. an oracle tree or a load_tree() result)."""
        ctx = ctx or default_context()
        a = {k: np.ascontiguousarray(v) for k, v in t.items() if isinstance(v, np.ndarray)}
        a["level"] = a["level"].astype(np.int32)
        for k in ("parent", "first_child", "child_count"):
            a[k] = a[k].astype(np.int32)
        s = _tree_struct(a, int(t["max_level"]), len(a["weight"]))
        s.n_nodes = len(a["weight"])
        h = C.c_void_p()
        _chk(_lib.lib().trg_tree_upload(ctx.h, C.byref(s), C.byref(h)))
        return GmmTree(h, ctx)


# ------------------------------------------------------------------ model files
def save_tree(tree, path) -> None:
    """gmm.cpp:769-796 save_tree (trg_save_tree / trg_save_tree_host): the
    reference's JSON model file, byte for byte.  `tree` is a GmmTree or a
    host dict in the .host() layout."""
    if isinstance(tree, GmmTree):
        _chk(_lib.lib().trg_save_tree(tree.ctx.h, tree.h, str(path).encode()))
        return
    a = {k: np.ascontiguousarray(v) for k, v in tree.items() if isinstance(v, np.ndarray)}
    for k in ("parent", "first_child", "child_count", "level"):
        a[k] = a[k].astype(np.int32)
    s = _tree_struct(a, int(tree["max_level"]), len(a["weight"]))
    s.n_nodes = len(a["weight"])
    _chk(_lib.lib().trg_save_tree_host(C.byref(s), str(path).encode()))


def _empty_host_tree(J: int) -> dict:
    return dict(weight=np.zeros(J), mean=np.zeros((J, 3)), cov=np.zeros((J, 3, 3)),
                lambdas=np.zeros((J, 3)), axes=np.zeros((J, 3, 3)), log_norm=np.zeros(J),
                parent=np.zeros(J, np.int32), first_child=np.zeros(J, np.int32),
                child_count=np.zeros(J, np.int32), level=np.zeros(J, np.int32))


def parse_tree_file(path) -> dict:
    """The host half of load_tree (gmm.cpp:798-887; trg_load_tree_host): JSON
    parse and every structural check with the reference's messages.  Returns
    weight / mean / cov / topology (eigen fields unset)."""
    L = _lib.lib()
    s = _tree_struct(_empty_host_tree(0), 0, 0)
    rc = L.trg_load_tree_host(str(path).encode(), C.byref(s))
    if rc != _lib.TRG_ERANGE:
        _chk(rc if rc != 0 else _lib.TRG_EINVAL)
    t = _empty_host_tree(s.n_nodes)
    s = _tree_struct(t, 0, s.n_nodes)
    _chk(L.trg_load_tree_host(str(path).encode(), C.byref(s)))
    t["max_level"] = s.max_level
    return t


def load_tree(path, ctx: Context | None = None) -> "GmmTree":
    """gmm.cpp:798-896 load_tree onto the device (trg_load_tree): host parse
    and validation, then refresh_eig of every node on the GPU.  Bad files
    raise RuntimeError("bad model file <path>: ...") like the reference; a
    covariance eig_sym3 rejects raises InvalidArgument."""
    ctx = ctx or default_context()
    h = C.c_void_p()
    _chk(_lib.lib().trg_load_tree(ctx.h, str(path).encode(), C.byref(h)))
    return GmmTree(h, ctx)


def _tree_struct(t: dict, max_level: int, cap: int) -> TreeC:
    s = TreeC()
    s.n_nodes = 0
    s.max_level = max_level
    s.capacity = cap
    for k in ("weight", "mean", "cov", "lambdas", "axes", "log_norm"):
        setattr(s, k, _d(t[k]))
    for k in ("parent", "first_child", "child_count", "level"):
        setattr(s, k, _i(t[k]))
    return s


@dataclass
class BuildDiagnostics:  # gmm.hpp:43-49 (+ device counters)
    calibration_drift: float = 0.0
    calibration_passes: int = 0
    entries_per_round: list = field(default_factory=list)
    expanded_per_round: list = field(default_factory=list)
    calib_density_evaluations: int = 0
    node_ll_traces: list = field(default_factory=list)


def build_tree(cloud, config: ModelConfig = ModelConfig(),
               diagnostics: BuildDiagnostics | None = None,
               ctx: Context | None = None) -> GmmTree:
    """gmm.hpp:69-70 build_tree, on the GPU."""
    ctx = ctx or default_context()
    ptr, n, on_dev, _keep = _cloud_ptr(cloud, ctx)
    cfg = config.c()
    h = C.c_void_p()
    d = BuildDiagC()
    I1 = config.em_iterations_per_node + 1
    cap = sum(8 ** l for l in range(config.max_level))  # expansions <= internal nodes + root
    traces = np.zeros((cap, I1))
    if diagnostics is not None:
        d.ll_traces = _d(traces)
        d.ll_trace_capacity = cap
    _chk(_lib.lib().trg_build_tree(ctx.h, ptr, n, on_dev, C.byref(cfg), C.byref(h), C.byref(d)))
    if diagnostics is not None:
        diagnostics.calibration_drift = d.calibration_drift
        diagnostics.calibration_passes = d.calibration_passes
        L = config.max_level
        diagnostics.entries_per_round = list(d.entries_per_round)[:L]
        diagnostics.expanded_per_round = list(d.expanded_per_round)[:L]
        diagnostics.calib_density_evaluations = int(d.calib_density_evaluations)
        diagnostics.node_ll_traces = [traces[e].copy() for e in range(min(d.n_expansions, cap))]
    return GmmTree(h, ctx)


# ------------------------------------------------------------------ E-step
@dataclass
class MomentSet:  # association.hpp:14-32
    m0: np.ndarray
    m1: np.ndarray
    m2: np.ndarray | None
    total_points: int = 0
    total_mass: float = 0.0
    outliers: int = 0
    density_evaluations: int = 0

    def components(self) -> int:
        return len(self.m0)


def associate_adaptive(cloud, tree: GmmTree, t: RigidTransform = None,
                       config: AssocConfig = AssocConfig(), with_m2: bool = True,
                       per_point: bool = False):
    """association.hpp:54-56 associate_adaptive on the GPU.  With
    ``per_point`` also returns each point's (deposit node, path weight)."""
    t = t or RigidTransform.identity()
    ptr, n, on_dev, _keep = _cloud_ptr(cloud, tree.ctx)
    J = tree.size()
    m0, m1 = np.zeros(J), np.zeros((J, 3))
    m2 = np.zeros((J, 3, 3)) if with_m2 else None
    mc = MomentsC()
    mc.m0, mc.m1 = _d(m0), _d(m1)
    mc.m2 = _d(m2) if with_m2 else None
    R = np.ascontiguousarray(t.rotation, dtype=np.float64)
    tr = np.ascontiguousarray(t.translation, dtype=np.float64)
    cfg = config.c()
    node = np.zeros(n, np.int32) if per_point else None
    w = np.zeros(n) if per_point else None
    _chk(_lib.lib().trg_associate(tree.ctx.h, tree.h, ptr, n, on_dev, _d(R), _d(tr), C.byref(cfg),
                                  C.byref(mc), _i(node) if per_point else None,
                                  _d(w) if per_point else None))
    ms = MomentSet(m0, m1, m2, int(mc.total_points), float(mc.total_mass), int(mc.outliers),
                   int(mc.density_evaluations))
    return (ms, node, w) if per_point else ms


# ------------------------------------------------------------------ M-step
@dataclass
class VirtualPointSet:  # mstep.hpp:21-32
    """The virtual points make_virtual_points produced on the device: per
    point pi* and mu* and the index of its component in ``tree`` (the
    reference's VirtualPoint::component), plus the moments they came from."""
    moments: MomentSet
    tree: GmmTree
    index: np.ndarray = None    # [n] component (node) index
    pi_star: np.ndarray = None  # [n]
    mu_star: np.ndarray = None  # [n, 3]

    def size(self) -> int:
        return 0 if self.index is None else len(self.index)

    def empty(self) -> bool:
        return self.size() == 0


@dataclass
class MStepSolution:  # mstep.hpp:54-61
    omega: np.ndarray
    translation: np.ndarray
    delta: RigidTransform
    criterion_before: float
    criterion_after: float
    condition_estimate: float
    n_virtual_points: int


def make_virtual_points(moments: MomentSet, tree: GmmTree) -> VirtualPointSet:
    """mstep.hpp:46-47 on the GPU (trg_make_virtual_points, k_make_vps): the
    order-preserving filter m0 > 1e-8 N with pi* = m0 / N, mu* = m1 / m0
    (mstep.cpp:8-30); validation mirrors mstep.cpp:11-17."""
    if moments.components() != tree.size():
        raise InvalidArgument("make_virtual_points: moment/component count mismatch")
    if moments.total_points == 0:
        raise InvalidArgument("make_virtual_points: no points were associated")
    J = moments.components()
    m0 = np.ascontiguousarray(moments.m0, dtype=np.float64)
    m1 = np.ascontiguousarray(moments.m1, dtype=np.float64)
    idx = np.zeros(J, np.int32)
    pi = np.zeros(J)
    mu = np.zeros((J, 3))
    n = C.c_int(0)
    _chk(_lib.lib().trg_make_virtual_points(tree.ctx.h, J, _d(m0), _d(m1), int(moments.total_points),
                                            idx.ctypes.data_as(_lib.ip), _d(pi), _d(mu), C.byref(n)))
    k = int(n.value)
    return VirtualPointSet(moments, tree, idx[:k].copy(), pi[:k].copy(), mu[:k].copy())


def solve_mstep(vps: VirtualPointSet) -> MStepSolution:
    """mstep.hpp:67 solve_mstep on the GPU (single thread-block)."""
    m = vps.moments
    out = MStepSolutionC()
    m0 = np.ascontiguousarray(m.m0, dtype=np.float64)
    m1 = np.ascontiguousarray(m.m1, dtype=np.float64)
    _chk(_lib.lib().trg_solve_mstep(vps.tree.ctx.h, vps.tree.h, _d(m0), _d(m1), m.total_points,
                                    C.byref(out)))
    R = np.array(out.delta_R[:]).reshape(3, 3)
    return MStepSolution(np.array(out.omega[:]), np.array(out.translation[:]),
                         RigidTransform(R, np.array(out.delta_t[:])), out.criterion_before,
                         out.criterion_after, out.condition_estimate, out.n_virtual_points)


# ------------------------------------------------------------------ driver
@dataclass
class RegistrationResult:  # registration.hpp:38-48
    transform: RigidTransform
    iterations: int
    converged: bool
    criterion_trace: np.ndarray
    criterion_after_trace: np.ndarray
    eval_counts: np.ndarray
    model_build_seconds: float
    em_seconds: float
    model_components: int


def _result(r: RegResultC, cb, ca, ev) -> RegistrationResult:
    n = r.iterations
    return RegistrationResult(
        RigidTransform(np.array(r.R[:]).reshape(3, 3), np.array(r.t[:])), n, bool(r.converged),
        cb[:n].copy(), ca[:n].copy(), ev[:n].copy(), r.model_build_seconds, r.em_seconds,
        int(r.model_components))


def _result_buffers(cfg: RegistrationConfig):
    k = max(1, cfg.max_em_iterations)
    cb, ca, ev = np.zeros(k), np.zeros(k), np.zeros(k, np.uint64)
    r = RegResultC()
    r.criterion_trace, r.criterion_after_trace = _d(cb), _d(ca)
    r.eval_counts = ev.ctypes.data_as(u64p)
    r.trace_capacity = k
    return r, cb, ca, ev


def register_with_tree(tree: GmmTree, source, config: RegistrationConfig = RegistrationConfig(),
                       target_diag: float = 0.0) -> RegistrationResult:
    """registration.hpp:59-62, EM loop resident on the GPU."""
    ptr, n, on_dev, _keep = _cloud_ptr(source, tree.ctx)
    r, cb, ca, ev = _result_buffers(config)
    cfg = config.c()
    _chk(_lib.lib().trg_register_with_tree(tree.ctx.h, tree.h, ptr, n, on_dev, C.byref(cfg),
                                           float(target_diag), C.byref(r)))
    return _result(r, cb, ca, ev)


def register_clouds(target, source, config: RegistrationConfig = RegistrationConfig(),
                    ctx: Context | None = None) -> RegistrationResult:
    """registration.hpp:53-55 (adaptive:L / tree:L): build + EM on the GPU."""
    ctx = ctx or default_context()
    pt, nt, dev_t, _k1 = _cloud_ptr(target, ctx)
    ps, ns, dev_s, _k2 = _cloud_ptr(source, ctx)
    if dev_t != dev_s:
        raise InvalidArgument("register_clouds: target and source must live on the same side")
    r, cb, ca, ev = _result_buffers(config)
    cfg = config.c()
    _chk(_lib.lib().trg_register_clouds(ctx.h, pt, nt, ps, ns, dev_t, C.byref(cfg), C.byref(r)))
    return _result(r, cb, ca, ev)


def register_batch(targets, sources, config: RegistrationConfig = RegistrationConfig(),
                   ctx: Context | None = None, streams: int = 0) -> list:
    """Independent frame pairs (BASELINE config C5): pair i registers
    sources[i] to targets[i] exactly as register_clouds would; `streams`
    pairs run concurrently (0 = library default).  No reference counterpart
    (the reference loops over register_clouds)."""
    ctx = ctx or default_context()
    if len(targets) != len(sources):
        raise InvalidArgument("register_batch: targets and sources differ in length")
    n = len(targets)
    keep, sides = [], set()
    tp, tn = (C.c_void_p * max(1, n))(), (C.c_size_t * max(1, n))()
    sp, sn = (C.c_void_p * max(1, n))(), (C.c_size_t * max(1, n))()
    for i in range(n):
        pt, nt, dt, k1 = _cloud_ptr(targets[i], ctx)
        ps, ns, ds, k2 = _cloud_ptr(sources[i], ctx)
        keep += [k1, k2]
        sides |= {dt, ds}
        tp[i], tn[i], sp[i], sn[i] = pt.value, nt, ps.value, ns
    if len(sides) > 1:
        raise InvalidArgument("register_batch: all clouds must live on the same side")
    bufs = [_result_buffers(config) for _ in range(n)]
    arr = (RegResultC * max(1, n))()
    for i, (r, _, _, _) in enumerate(bufs):
        arr[i] = r
    cfg = config.c()
    _chk(_lib.lib().trg_register_batch(ctx.h, n, tp, tn, sp, sn, sides.pop() if sides else 0,
                                       C.byref(cfg), int(streams), arr))
    return [_result(arr[i], cb, ca, ev) for i, (_, cb, ca, ev) in enumerate(bufs)]


def register_sequence(frames, config: RegistrationConfig = RegistrationConfig(),
                      ctx: Context | None = None, streams: int = 0):
    """Frame-to-frame sequence (the reference harness's run_sequence core,
    harness.cpp:334-389): pair k registers frame k (source) to frame k-1
    (target) and the trajectory chains T_k = T_{k-1} * pairwise_k (frame k ->
    frame 0).  All pairs go through register_batch, so the GPU overlaps the
    tree builds and EM loops of consecutive pairs.  Returns (pairwise
    results, trajectory)."""
    if len(frames) < 2:
        raise InvalidArgument("sequence: need at least 2 frames")
    res = register_batch(list(frames[:-1]), list(frames[1:]), config, ctx, streams)
    traj = [RigidTransform.identity()]
    for r in res:
        traj.append(traj[-1] * r.transform)
    return res, traj


# ------------------------------------------------------------------ flat mixture
def build_flat_gmm(cloud, j: int, config: ModelConfig = ModelConfig(),
                   diagnostics: BuildDiagnostics | None = None,
                   ctx: Context | None = None) -> GmmTree:
    """gmm.hpp:74-76 build_flat_gmm on the GPU: the J components come back as
    a depth-1 GmmTree of J roots (``.host()`` gives the component arrays)."""
    ctx = ctx or default_context()
    ptr, n, on_dev, _keep = _cloud_ptr(cloud, ctx)
    cfg = config.c()
    h = C.c_void_p()
    d = BuildDiagC()
    iters = max(1, config.em_iterations_per_node * config.max_level)
    trace = np.zeros(iters)
    if diagnostics is not None:  # one row of em_iterations_per_node + 1 values per capacity unit
        d.ll_traces = _d(trace)
        d.ll_trace_capacity = -(-iters // (config.em_iterations_per_node + 1))
    _chk(_lib.lib().trg_build_flat_gmm(ctx.h, ptr, n, on_dev, int(j), C.byref(cfg), C.byref(h),
                                       C.byref(d)))
    if diagnostics is not None:
        diagnostics.entries_per_round = [int(d.entries_per_round[0])]
        # gmm.cpp:729-734: the flat fit's EM log-likelihood trace
        diagnostics.node_ll_traces = [trace[:d.flat_trace_len].copy()]
    return GmmTree(h, ctx)


def responsibilities_dense(cloud, components: GmmTree, t: "RigidTransform" = None,
                           outlier_floor: float = 1e-300, with_m2: bool = True) -> "MomentSet":
    """association.hpp:44-47 responsibilities_dense: every node of
    `components` (a flat mixture or any tree's nodes) against every point."""
    t = t or RigidTransform.identity()
    ptr, n, on_dev, _keep = _cloud_ptr(cloud, components.ctx)
    J = components.size()
    m0, m1 = np.zeros(J), np.zeros((J, 3))
    m2 = np.zeros((J, 3, 3)) if with_m2 else None
    mc = MomentsC()
    mc.m0, mc.m1 = _d(m0), _d(m1)
    mc.m2 = _d(m2) if with_m2 else None
    R = np.ascontiguousarray(t.rotation, dtype=np.float64)
    tt = np.ascontiguousarray(t.translation, dtype=np.float64)
    _chk(_lib.lib().trg_responsibilities_dense(components.ctx.h, components.h, ptr, n, on_dev,
                                               _d(R), _d(tt), float(outlier_floor),
                                               C.byref(mc)))
    return MomentSet(m0, m1, m2, int(mc.total_points), float(mc.total_mass), int(mc.outliers),
                     int(mc.density_evaluations))


# ------------------------------------------------------------------ sharding
def shard_bounds(n: int, world: int, rank: int) -> tuple:
    """Contiguous block [lo, hi) of an n-point cloud held by `rank` of `world`
    (the block order is the global entry order the sharded build assumes)."""
    if world < 1 or not 0 <= rank < world:
        raise InvalidArgument("shard_bounds: bad rank/world")
    return (n * rank) // world, (n * (rank + 1)) // world


def share_unique_id(dist, make_id) -> bytes:
    """Rank 0 makes the 128-byte communicator id, every rank receives it
    (torch.distributed object broadcast; any backend)."""
    obj = [make_id() if dist.get_rank() == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    uid = obj[0]
    if not isinstance(uid, (bytes, bytearray)) or len(uid) != 128:
        raise InvalidArgument("share_unique_id: malformed id")
    return bytes(uid)


class Comm:
    """Point-sharded communicator (trg_comm).  ``Comm.local(k)``: k shards
    driven by this process on one GPU (fixed-order device reduction);
    ``Comm.nccl(...)`` / ``Comm.from_torch_distributed()``: one shard per
    process over NCCL."""

    def __init__(self, handle, ctx: Context):
        self.h = handle
        self.ctx = ctx

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_ubyte * 128)()
        _chk(_lib.lib().trg_comm_unique_id(buf))
        return bytes(buf)

    @staticmethod
    def local(shards: int, ctx: Context | None = None) -> "Comm":
        ctx = ctx or default_context()
        h = C.c_void_p()
        _chk(_lib.lib().trg_comm_create_local(ctx.h, int(shards), C.byref(h)))
        return Comm(h, ctx)

    @staticmethod
    def nccl(rank: int, world: int, uid: bytes, ctx: Context | None = None) -> "Comm":
        ctx = ctx or default_context()
        buf = (C.c_ubyte * 128).from_buffer_copy(uid)
        h = C.c_void_p()
        _chk(_lib.lib().trg_comm_create_nccl(ctx.h, buf, int(rank), int(world), C.byref(h)))
        return Comm(h, ctx)

    @staticmethod
    def from_torch_distributed(ctx: Context | None = None) -> "Comm":
        import torch.distributed as dist
        uid = share_unique_id(dist, Comm.unique_id)
        return Comm.nccl(dist.get_rank(), dist.get_world_size(), uid, ctx)

    @property
    def rank(self) -> int:
        return _lib.lib().trg_comm_rank(self.h)

    @property
    def world(self) -> int:
        return _lib.lib().trg_comm_world(self.h)

    @property
    def local_shards(self) -> int:
        return _lib.lib().trg_comm_local_shards(self.h)

    def close(self):
        if self.h:
            _lib.lib().trg_comm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _shard_arrays(clouds, comm: Comm):
    if len(clouds) != comm.local_shards:
        raise InvalidArgument(f"expected {comm.local_shards} shard clouds, got {len(clouds)}")
    keep, sides = [], set()
    ptr = (C.c_void_p * len(clouds))()
    cnt = (C.c_size_t * len(clouds))()
    for i, c in enumerate(clouds):
        p, n, d, k = _cloud_ptr(c, comm.ctx)
        keep.append(k)
        sides.add(d)
        ptr[i], cnt[i] = p.value, n
    if len(sides) > 1:
        raise InvalidArgument("all shard clouds must live on the same side")
    return ptr, cnt, sides.pop(), keep


def build_tree_sharded(shards: list, comm: Comm, config: ModelConfig = ModelConfig(),
                       diagnostics: BuildDiagnostics | None = None) -> GmmTree:
    """build_tree over the union of the shards' clouds (this process's local
    shards; contiguous blocks of one cloud in shard order)."""
    ptr, cnt, on_dev, _keep = _shard_arrays(shards, comm)
    cfg = config.c()
    h = C.c_void_p()
    d = BuildDiagC()
    _chk(_lib.lib().trg_build_tree_sharded(comm.h, ptr, cnt, on_dev, C.byref(cfg), C.byref(h),
                                           C.byref(d)))
    if diagnostics is not None:
        diagnostics.calibration_drift = d.calibration_drift
        diagnostics.calibration_passes = d.calibration_passes
        L = config.max_level
        diagnostics.entries_per_round = list(d.entries_per_round)[:L]
        diagnostics.expanded_per_round = list(d.expanded_per_round)[:L]
    return GmmTree(h, comm.ctx)


def register_clouds_sharded(targets: list, sources: list, comm: Comm,
                            config: RegistrationConfig = RegistrationConfig()) -> RegistrationResult:
    """register_clouds over sharded target / source clouds."""
    tp, tn, dt, _k1 = _shard_arrays(targets, comm)
    sp, sn, ds, _k2 = _shard_arrays(sources, comm)
    if dt != ds:
        raise InvalidArgument("register_clouds_sharded: targets and sources on different sides")
    r, cb, ca, ev = _result_buffers(config)
    cfg = config.c()
    _chk(_lib.lib().trg_register_clouds_sharded(comm.h, tp, tn, sp, sn, dt, C.byref(cfg),
                                                C.byref(r)))
    return _result(r, cb, ca, ev)


# ------------------------------------------------------------------ inputs
def read_cloud(path, fmt: str = "auto") -> np.ndarray:
    """cloud_io read_cloud: fmt in auto | ply_ascii | ply_binary | xyz."""
    code = {"auto": 0, "ply_ascii": 1, "ply_binary": 2, "xyz": 3}[fmt]
    p = dp()
    n = C.c_size_t()
    _chk_host(_lib.host_lib().trg_read_cloud(str(path).encode(), code, C.byref(p), C.byref(n)))
    try:
        return np.ctypeslib.as_array(p, shape=(n.value * 3,)).reshape(n.value, 3).copy() \
            if n.value else np.zeros((0, 3))
    finally:
        _lib.host_lib().trg_free_cloud(p)


def subsample(cloud, n: int, seed: int) -> np.ndarray:
    """cloud_io subsample: n points in index order, reference-identical picks."""
    p = _points(cloud)
    out = np.zeros((int(n), 3))
    _chk_host(_lib.host_lib().trg_subsample(_d(p), len(p), int(n), seed, _d(out)))
    return out


def synthetic(kind: str, n: int, seed: int) -> np.ndarray:
    """synthetic.cpp generators (bit-identical restatement)."""
    out = np.zeros((n, 3))
    _chk_host(_lib.host_lib().trg_synthetic(kind.encode(), n, seed, _d(out)))
    return out


def unit_normalized(cloud) -> np.ndarray:
    p = _points(cloud).copy()
    _chk_host(_lib.host_lib().trg_unit_normalize(_d(p), len(p)))
    return p


def bbox_diagonal(cloud) -> float:
    p = _points(cloud)
    return float(_lib.host_lib().trg_bbox_diagonal(_d(p), len(p)))


def random_rigid_transform(rot_range_deg: float, trans_range: float, seed: int,
                           trial: int = 0) -> RigidTransform:
    R, t = np.zeros((3, 3)), np.zeros(3)
    _chk_host(_lib.host_lib().trg_random_rigid_transform(rot_range_deg, trans_range, seed, trial, _d(R),
                                               _d(t)))
    return RigidTransform(R, t)


def kinect_pair(seed: int):
    """C2: 320x240 Kinect-style frame pair -> (target, source, gt source->target)."""
    tg, sr, R, t = np.zeros((76800, 3)), np.zeros((76800, 3)), np.zeros((3, 3)), np.zeros(3)
    _chk_host(_lib.host_lib().trg_synth_kinect_pair(seed, _d(tg), _d(sr), _d(R), _d(t)))
    return tg, sr, RigidTransform(R, t)


def kinect_sequence(seed: int, frames: int, step_rot_deg: float = 2.0, step_trans: float = 0.02):
    """Kinect-style frame sequence -> (frames [F, 76800, 3], gt [F] RigidTransform
    mapping frame k into frame 0)."""
    out = np.zeros((frames, 76800, 3))
    R, t = np.zeros((frames, 3, 3)), np.zeros((frames, 3))
    _chk_host(_lib.host_lib().trg_synth_kinect_sequence(seed, frames, step_rot_deg, step_trans, _d(out), _d(R),
                                              _d(t)))
    return out, [RigidTransform(R[k], t[k]) for k in range(frames)]


def _render_frames(kind: str, seed: int, ctx, noise_scale: float, rot_range_deg: float,
                   trans_range: float):
    import torch
    ctx = ctx or default_context()
    n = 76800 if kind == "kinect" else 72000
    R, t = np.zeros((2, 3, 3)), np.zeros((2, 3))
    noise = np.zeros(2 * n)
    Rg, tg = np.zeros((3, 3)), np.zeros(3)
    H = _lib.host_lib()
    tab = None
    if kind == "kinect":
        _chk_host(H.trg_synth_kinect_pair_plan(seed, rot_range_deg, trans_range, _d(R), _d(t), _d(noise),
                                               _d(Rg), _d(tg)))
    else:
        tab = np.zeros(4564)
        _chk_host(H.trg_synth_lidar_pair_plan(seed, _d(R), _d(t), _d(noise), _d(tab), _d(Rg), _d(tg)))
    dev = torch.device("cuda", ctx.device)
    out = torch.empty((2, n, 3), dtype=torch.float64, device=dev)
    # the buffer's previous users on torch's stream finish first; torch's
    # stream then waits for the render
    _chk(_lib.lib().trg_ctx_wait_stream(ctx.h, C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)))
    if kind == "kinect":
        _chk(_lib.lib().trg_render_kinect_frames(ctx.h, 2, _d(R), _d(t), _d(noise), noise_scale,
                                                 C.c_void_p(out.data_ptr())))
    else:
        _chk(_lib.lib().trg_render_lidar_frames(ctx.h, 2, _d(R), _d(t), _d(noise), _d(tab),
                                                C.c_void_p(out.data_ptr())))
    torch.cuda.current_stream(dev).wait_stream(torch.cuda.ExternalStream(ctx.stream, device=dev))
    return out[0], out[1], RigidTransform(Rg, tg)


def kinect_pair_device(seed: int, ctx: Context | None = None, noise_scale: float = 1.0,
                       rot_range_deg: float = 5.0, trans_range: float = 0.05):
    """kinect_pair rendered on the GPU: the poses and the
    noise draws from the host generator (trg_synth_kinect_pair_plan), the
    76,800 rays per frame cast on the device (trg_render_kinect_frames) ->
    (target, source) as CUDA (N, 3) float64 tensors, bit-identical to
    kinect_pair(seed), and the ground truth."""
    return _render_frames("kinect", seed, ctx, noise_scale, rot_range_deg, trans_range)


def lidar_pair_device(seed: int, ctx: Context | None = None):
    """lidar_pair rendered on the GPU (trg_render_lidar_frames), bit-identical
    to lidar_pair(seed)."""
    return _render_frames("lidar", seed, ctx, 1.0, 0.0, 0.0)


def lidar_pair(seed: int):
    """C3: HDL-32-style sweep pair -> (target, source, gt source->target)."""
    tg, sr, R, t = np.zeros((72000, 3)), np.zeros((72000, 3)), np.zeros((3, 3)), np.zeros(3)
    _chk_host(_lib.host_lib().trg_synth_lidar_pair(seed, _d(tg), _d(sr), _d(R), _d(t)))
    return tg, sr, RigidTransform(R, t)
