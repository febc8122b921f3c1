"""ctypes binding of libtrg_cuda.so (the C-ABI in include/treereg_b200.h).

The library is built in-tree (``make -C paper_1807_02587_b200`` or
``__graft_entry__.build()``).  There is no CPU fallback: if the shared
library is missing or no CUDA device is present, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libtrg_cuda.so")
# host-only companion (include/treereg_b200_host.h): ingest + synthetic inputs
HOST_LIB_PATH = os.path.join(HERE, "libtrg_host.so")

dp = C.POINTER(C.c_double)
ip = C.POINTER(C.c_int)
u64p = C.POINTER(C.c_uint64)

TRG_OK, TRG_EINVAL, TRG_EDOMAIN, TRG_ERUNTIME, TRG_ERANGE, TRG_EDEGENERATE, TRG_ECUDA, TRG_ENCCL = range(8)


class ModelConfigC(C.Structure):
    _fields_ = [("em_iterations_per_node", C.c_int), ("min_points_per_node", C.c_size_t),
                ("cov_regularization_epsilon", C.c_double),
                ("cov_regularization_absolute", C.c_double), ("rng_seed", C.c_uint64),
                ("max_level", C.c_int)]


class AssocConfigC(C.Structure):
    _fields_ = [("lambda_c", C.c_double), ("max_level", C.c_int), ("outlier_floor", C.c_double),
                ("deterministic", C.c_int)]


class RegConfigC(C.Structure):
    _fields_ = [("variant_kind", C.c_int), ("variant_param", C.c_int), ("lambda_c", C.c_double),
                ("max_em_iterations", C.c_int), ("rotation_tol", C.c_double),
                ("translation_tol", C.c_double), ("initial_R", C.c_double * 9),
                ("initial_t", C.c_double * 3), ("model_config", ModelConfigC),
                ("fast_scoring", C.c_int)]


class TreeC(C.Structure):
    _fields_ = [("n_nodes", C.c_int), ("max_level", C.c_int), ("capacity", C.c_int),
                ("weight", dp), ("mean", dp), ("cov", dp), ("lambdas", dp), ("axes", dp),
                ("log_norm", dp), ("parent", ip), ("first_child", ip), ("child_count", ip),
                ("level", ip)]


class MomentsC(C.Structure):
    _fields_ = [("m0", dp), ("m1", dp), ("m2", dp), ("total_points", C.c_uint64),
                ("outliers", C.c_uint64), ("density_evaluations", C.c_uint64),
                ("total_mass", C.c_double)]


class BuildDiagC(C.Structure):
    _fields_ = [("entries_per_round", C.c_uint64 * 8), ("expanded_per_round", C.c_int * 8),
                ("calibration_passes", C.c_int), ("calibration_drift", C.c_double),
                ("calib_density_evaluations", C.c_uint64), ("ll_traces", dp),
                ("ll_trace_capacity", C.c_int), ("n_expansions", C.c_int),
                ("flat_trace_len", C.c_int)]


class MStepSolutionC(C.Structure):
    _fields_ = [("omega", C.c_double * 3), ("translation", C.c_double * 3),
                ("delta_R", C.c_double * 9), ("delta_t", C.c_double * 3),
                ("criterion_before", C.c_double), ("criterion_after", C.c_double),
                ("condition_estimate", C.c_double), ("n_virtual_points", C.c_int)]


class RegResultC(C.Structure):
    _fields_ = [("R", C.c_double * 9), ("t", C.c_double * 3), ("iterations", C.c_int),
                ("converged", C.c_int), ("criterion_trace", dp), ("criterion_after_trace", dp),
                ("eval_counts", u64p), ("trace_capacity", C.c_int),
                ("model_build_seconds", C.c_double), ("em_seconds", C.c_double),
                ("model_components", C.c_size_t)]


# name -> (restype, argtypes); every symbol include/treereg_b200.h declares.
SIGNATURES = {
    "trg_ctx_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "trg_ctx_destroy": (C.c_int, [C.c_void_p]),
    "trg_last_error": (C.c_char_p, []),
    "trg_device_sms": (C.c_int, [C.c_void_p]),
    "trg_ctx_set_sm_budget": (C.c_int, [C.c_void_p, C.c_int]),
    "trg_kernel_launches": (C.c_uint64, [C.c_void_p]),
    "trg_ctx_stream": (C.c_void_p, [C.c_void_p]),
    "trg_ctx_wait_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "trg_ctx_transfer_bytes": (None, [C.c_void_p, u64p, u64p]),
    "trg_tree_capacity": (C.c_int, [C.c_int]),
    "trg_tree_upload": (C.c_int, [C.c_void_p, C.POINTER(TreeC), C.POINTER(C.c_void_p)]),
    "trg_tree_upload_refresh": (C.c_int, [C.c_void_p, C.POINTER(TreeC), C.POINTER(C.c_void_p)]),
    "trg_save_tree": (C.c_int, [C.c_void_p, C.c_void_p, C.c_char_p]),
    "trg_load_tree": (C.c_int, [C.c_void_p, C.c_char_p, C.POINTER(C.c_void_p)]),
    "trg_save_tree_host": (C.c_int, [C.POINTER(TreeC), C.c_char_p]),
    "trg_load_tree_host": (C.c_int, [C.c_char_p, C.POINTER(TreeC)]),
    "trg_tree_download": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(TreeC)]),
    "trg_tree_free": (C.c_int, [C.c_void_p, C.c_void_p]),
    "trg_tree_size": (C.c_int, [C.c_void_p]),
    "trg_build_tree": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int,
                                 C.POINTER(ModelConfigC), C.POINTER(C.c_void_p),
                                 C.POINTER(BuildDiagC)]),
    "trg_associate": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, dp, dp,
                                C.POINTER(AssocConfigC), C.POINTER(MomentsC), ip, dp]),
    "trg_solve_mstep": (C.c_int, [C.c_void_p, C.c_void_p, dp, dp, C.c_uint64,
                                  C.POINTER(MStepSolutionC)]),
    "trg_make_virtual_points": (C.c_int, [C.c_void_p, C.c_int, dp, dp, C.c_uint64, ip, dp, dp,
                                          ip]),
    "trg_solve_mstep_vps": (C.c_int, [C.c_void_p, C.c_int, dp, dp, dp, dp, dp,
                                      C.POINTER(MStepSolutionC)]),
    "trg_register_with_tree": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_int,
                                         C.POINTER(RegConfigC), C.c_double,
                                         C.POINTER(RegResultC)]),
    "trg_build_flat_gmm": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_size_t,
                                     C.c_void_p, C.POINTER(C.c_void_p), C.c_void_p]),
    "trg_responsibilities_dense": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_int,
                                             dp, dp, C.c_double, C.c_void_p]),
    "trg_comm_unique_id": (C.c_int, [C.c_void_p]),
    "trg_comm_create_nccl": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    "trg_comm_create_local": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_void_p)]),
    "trg_comm_destroy": (C.c_int, [C.c_void_p]),
    "trg_comm_rank": (C.c_int, [C.c_void_p]),
    "trg_comm_world": (C.c_int, [C.c_void_p]),
    "trg_comm_local_shards": (C.c_int, [C.c_void_p]),
    "trg_build_tree_sharded": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_size_t), C.c_int,
                                         C.c_void_p, C.POINTER(C.c_void_p), C.c_void_p]),
    "trg_register_clouds_sharded": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_size_t),
                                              C.POINTER(C.c_void_p), C.POINTER(C.c_size_t), C.c_int,
                                              C.c_void_p, C.c_void_p]),
    "trg_render_kinect_frames": (C.c_int, [C.c_void_p, C.c_int, dp, dp, dp, C.c_double, C.c_void_p]),
    "trg_render_lidar_frames": (C.c_int, [C.c_void_p, C.c_int, dp, dp, dp, dp, C.c_void_p]),
    "trg_register_batch": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_void_p), C.POINTER(C.c_size_t),
                                     C.POINTER(C.c_void_p), C.POINTER(C.c_size_t), C.c_int,
                                     C.c_void_p, C.c_int, C.c_void_p]),
    "trg_register_clouds": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p,
                                      C.c_size_t, C.c_int, C.POINTER(RegConfigC),
                                      C.POINTER(RegResultC)]),
    "trg_debug_build_timeline": (C.c_int, [C.c_void_p, u64p, ip, C.c_int]),
    "trg_debug_solve": (C.c_int, [C.c_void_p, dp, C.c_int, dp]),
    "trg_debug_eig": (C.c_int, [C.c_void_p, C.c_int, dp, C.c_int, dp, dp, ip]),
}

HOST_SIGNATURES = {
    "trg_host_last_error": (C.c_char_p, []),
    "trg_synthetic": (C.c_int, [C.c_char_p, C.c_size_t, C.c_uint64, dp]),
    "trg_unit_normalize": (C.c_int, [dp, C.c_size_t]),
    "trg_bbox_diagonal": (C.c_double, [dp, C.c_size_t]),
    "trg_random_rigid_transform": (C.c_int, [C.c_double, C.c_double, C.c_uint64, C.c_int, dp,
                                             dp]),
    "trg_read_cloud": (C.c_int, [C.c_char_p, C.c_int, C.POINTER(dp), C.POINTER(C.c_size_t)]),
    "trg_free_cloud": (None, [dp]),
    "trg_subsample": (C.c_int, [dp, C.c_size_t, C.c_size_t, C.c_uint64, dp]),
    "trg_synth_kinect_sequence": (C.c_int, [C.c_uint64, C.c_int, C.c_double, C.c_double, dp, dp, dp]),
    "trg_synth_kinect_pair": (C.c_int, [C.c_uint64, dp, dp, dp, dp]),
    "trg_synth_kinect_pair_ex": (C.c_int, [C.c_uint64, C.c_double, C.c_double, C.c_double, dp, dp,
                                           dp, dp]),
    "trg_synth_lidar_pair": (C.c_int, [C.c_uint64, dp, dp, dp, dp]),
    "trg_synth_kinect_pair_plan": (C.c_int, [C.c_uint64, C.c_double, C.c_double, dp, dp, dp, dp, dp]),
    "trg_synth_lidar_pair_plan": (C.c_int, [C.c_uint64, dp, dp, dp, dp, dp, dp]),
}

_LIB = None


def lib():
    """Load libtrg_cuda.so once; raise loudly if it is not built."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is not built (run `make -C {HERE}` or __graft_entry__.build()); "
                "the B200 path has no CPU fallback")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = L
    return _LIB


def last_error() -> str:
    return lib().trg_last_error().decode(errors="replace")


_HOST = None


def host_lib():
    """Load libtrg_host.so (no device code) once."""
    global _HOST
    if _HOST is None:
        if not os.path.exists(HOST_LIB_PATH):
            raise ImportError(f"{HOST_LIB_PATH} is not built (run `make -C {HERE}`)")
        L = C.CDLL(HOST_LIB_PATH)
        for name, (res, args) in HOST_SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _HOST = L
    return _HOST


def host_last_error() -> str:
    return host_lib().trg_host_last_error().decode(errors="replace")
