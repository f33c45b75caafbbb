"""ctypes binding of the in-tree C ABI library libdabd_gpu.so (include/dabd_gpu.h).

There is no CPU fallback: if the library is missing this module raises, and
every compute call needs a CUDA device.
"""

from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libdabd_gpu.so")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_up = C.POINTER(C.c_uint32)


class SimParams(C.Structure):
    _fields_ = [("h", C.c_double), ("gravity_x", C.c_double), ("gravity_y", C.c_double),
                ("arap_stiffness", C.c_double), ("barrier_stiffness", C.c_double),
                ("d_hat", C.c_double), ("theta", C.c_double), ("scene_scale", C.c_double)]


class AdaptParams(C.Structure):
    _fields_ = [("beta", C.c_double), ("tau", C.c_double), ("mu", C.c_double),
                ("sigma_min", C.c_double), ("sigma_max", C.c_double), ("adapt_enabled", C.c_int)]


class RunParams(C.Structure):
    _fields_ = [("w_min", C.c_double), ("admm_max_iterations", C.c_int), ("newton_cap", C.c_int),
                ("max_halvings", C.c_int), ("force_split_frames", C.c_int)]


class SolverParams(C.Structure):
    _fields_ = [("pcg_rel_tol", C.c_double), ("pcg_max_iters", C.c_int)]


class BalanceParams(C.Structure):
    _fields_ = [("enabled", C.c_int), ("kp", C.c_double), ("kd", C.c_double),
                ("smoothing", C.c_double), ("dp_max", C.c_double)]


class FrameStats(C.Structure):
    _fields_ = [("committed", C.c_int), ("attempts", C.c_int), ("h", C.c_double),
                ("admm_iterations", C.c_int), ("newton_iterations", C.c_int),
                ("line_search_steps", C.c_int), ("pcg_iterations", C.c_int),
                ("max_contacts", C.c_int), ("max_candidates", C.c_int),
                ("exact_retries", C.c_int), ("capacity_retries", C.c_int),
                ("t_solve", C.c_double), ("t_coll", C.c_double), ("t_sync", C.c_double),
                ("t_frame", C.c_double)]


HaloFn = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p,
                     C.c_void_p, C.c_size_t, C.c_size_t)
AllgatherFn = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_size_t)


class Comm(C.Structure):
    """dabd_gpu_comm (include/dabd_gpu.h)."""
    _fields_ = [("user", C.c_void_p), ("halo", HaloFn), ("allgather", AllgatherFn),
                ("rank", C.c_int), ("world", C.c_int), ("part_offsets", _ip)]


class Sim3dParams(C.Structure):
    """dabd_gpu_sim3d_params (include/dabd_gpu.h)."""
    _fields_ = [("h", C.c_double), ("gravity", C.c_double * 3), ("d_hat", C.c_double),
                ("kappa", C.c_double), ("kappa_arap", C.c_double), ("theta", C.c_double),
                ("scene_scale", C.c_double), ("newton_cap", C.c_int), ("pcg_rel_tol", C.c_double),
                ("pcg_max_iters", C.c_int)]


class Sim3dStats(C.Structure):
    """dabd_gpu_sim3d_stats (include/dabd_gpu.h)."""
    _fields_ = [("newton_iterations", C.c_int), ("line_search_steps", C.c_int),
                ("pcg_iterations", C.c_int), ("max_candidates", C.c_int), ("converged", C.c_int),
                ("min_distance", C.c_double)]


# Every symbol include/dabd_gpu.h declares (checked by tests/test_abi.py).
EXPORTS = [
    "dabd_gpu_version", "dabd_gpu_last_error", "dabd_gpu_scene_create", "dabd_gpu_scene_free",
    "dabd_gpu_scene_set_params", "dabd_gpu_scene_set_planes", "dabd_gpu_scene_set_force_split",
    "dabd_gpu_scene_counts", "dabd_gpu_scene_bodies", "dabd_gpu_ctx_create", "dabd_gpu_ctx_free",
    "dabd_gpu_ctx_set_solver", "dabd_gpu_ctx_set_inexact", "dabd_gpu_ctx_set_stream", "dabd_gpu_broad_phase",
    "dabd_gpu_narrow_phase", "dabd_gpu_ccd_toi", "dabd_gpu_holder_masks", "dabd_gpu_audit", "dabd_gpu_objective",
    "dabd_gpu_newton_solve", "dabd_gpu_run_frames", "dabd_gpu_set_state", "dabd_gpu_get_state",
    "dabd_gpu_get_rho", "dabd_gpu_take_trace", "dabd_gpu_launch_count",
    "dabd_gpu_kernel_timer_enable", "dabd_gpu_kernel_timer_read", "dabd_gpu_kernel_timer_report",
    "dabd_gpu_ctx_pcg_perf", "dabd_gpu_ctx_set_comm", "dabd_gpu_ctx_pcg_phases",
    "dabd_gpu_ctx_list_stats", "dabd_gpu_scene_set_balance", "dabd_gpu_ctx_get_planes",
    "dabd_gpu_ctx_partition_costs", "dabd_gpu_imbalance_metric", "dabd_gpu_pd_update",
    "dabd_gpu_balance_factor", "dabd_gpu_balancer_create", "dabd_gpu_balancer_free",
    "dabd_gpu_balancer_update", "dabd_gpu_contact3d_terms", "dabd_gpu_ccd3d",
    "dabd_gpu_body3d_moments", "dabd_gpu_body3d_terms",
    "dabd_gpu_broad_phase3d", "dabd_gpu_ctx_comm_mode", "dabd_gpu_consensus_step",
    "dabd_gpu_check_stopping", "dabd_gpu_timestep_apply",
    "dabd_gpu_sim3d_create", "dabd_gpu_sim3d_free", "dabd_gpu_sim3d_run", "dabd_gpu_sim3d_get_state",
    "dabd_gpu_sim3d_set_state", "dabd_gpu_sim3d_system",
]

_lib = None


class DabdGpuError(RuntimeError):
    def __init__(self, status: int, message: str) -> None:
        super().__init__(f"[status {status}] {message}")
        self.status = status


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                          "(no CPU fallback exists for the dabd_gpu hot path)")
    lib = C.CDLL(LIB_PATH)
    lib.dabd_gpu_version.restype = C.c_char_p
    lib.dabd_gpu_last_error.restype = C.c_char_p
    lib.dabd_gpu_scene_free.argtypes = [C.c_void_p]
    lib.dabd_gpu_scene_free.restype = None
    lib.dabd_gpu_ctx_free.argtypes = [C.c_void_p]
    lib.dabd_gpu_sim3d_free.argtypes = [C.c_void_p]
    lib.dabd_gpu_sim3d_free.restype = None
    lib.dabd_gpu_ctx_free.restype = None
    lib.dabd_gpu_ctx_set_stream.argtypes = [C.c_void_p, C.c_size_t]
    lib.dabd_gpu_ctx_set_inexact.argtypes = [C.c_void_p, C.c_double, C.c_double]
    lib.dabd_gpu_balancer_free.argtypes = [C.c_void_p]
    lib.dabd_gpu_balancer_free.restype = None
    for fn in ("dabd_gpu_imbalance_metric", "dabd_gpu_pd_update"):
        getattr(lib, fn).restype = C.c_int
    _lib = lib
    return lib


def check(status: int) -> None:
    if status != 0:
        raise DabdGpuError(status, load().dabd_gpu_last_error().decode())
