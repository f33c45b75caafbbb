"""Python mirror of the reference interface for the hot path, over the C ABI.

Names and argument meaning follow proj/include/dabd/{geometry,partition,
objective,newton,sim}.hpp so the parity tests read like the reference's own
tests: `broad_phase`, `narrow_phase`, `ccd_toi_scene`, `body_holder_mask`,
`LocalObjective`-style `objective`, `newton_solve`, `run_reference`,
`run_distributed`. Every call executes the sm_100a kernels of
libdabd_gpu.so; there is no CPU path.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _lib as L
from .scene import SceneData

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_up = C.POINTER(C.c_uint32)


def _d(a):
    return None if a is None else a.ctypes.data_as(_dp)


def _i(a):
    return None if a is None else a.ctypes.data_as(_ip)


def _f64(a, shape=None):
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return arr if shape is None else arr.reshape(shape)


def _i32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def sim_params(p) -> L.SimParams:
    return L.SimParams(p.h, p.gravity[0], p.gravity[1], p.arap_stiffness, p.barrier_stiffness,
                       p.d_hat, p.theta, p.scene_scale)


class Scene:
    """Device-independent scene handle (dabd_gpu_scene): bodies + knobs."""

    def __init__(self, scene: SceneData) -> None:
        lib = L.load()
        self.data = scene
        fl = scene.flat()
        self._fl = fl
        self.n = fl["n_bodies"]
        h = C.c_void_p()
        L.check(lib.dabd_gpu_scene_create(
            self.n, _i(fl["body_loop_start"]), _i(fl["loop_vert_start"]), _d(_f64(fl["verts"])),
            _d(fl["density"]), _i(fl["is_static"]), _d(fl["arap_scale"]), _d(_f64(fl["qdot"])),
            C.byref(h)))
        self.h = h
        a = scene.adapt
        L.check(lib.dabd_gpu_scene_set_params(
            self.h, C.byref(sim_params(scene.params)),
            C.byref(L.AdaptParams(a.beta, a.tau, a.mu, a.sigma_min, a.sigma_max,
                                  int(a.adapt_enabled))),
            C.byref(L.RunParams(scene.w_min, scene.admm_max_iterations, scene.newton_cap,
                                scene.max_halvings, scene.force_split_frames))))
        planes = _f64(fl["planes"]).reshape(-1)
        L.check(lib.dabd_gpu_scene_set_planes(self.h, len(scene.planes),
                                              _d(planes) if planes.size else None))
        bal = scene.balance
        L.check(lib.dabd_gpu_scene_set_balance(self.h, C.byref(L.BalanceParams(
            int(bool(bal.get("enabled", False))), float(bal.get("kp", 0.0)), float(bal.get("kd", 0.0)),
            float(bal.get("smoothing", 0.5)), float(bal.get("dp_max", 0.0))))))
        for body, f in fl["force_split"]:
            L.check(lib.dabd_gpu_scene_set_force_split(self.h, body, C.c_double(f[0]),
                                                       C.c_double(f[1])))
        nb, nv = C.c_int(), C.c_int()
        L.check(lib.dabd_gpu_scene_counts(self.h, C.byref(nb), C.byref(nv)))
        self.nv = nv.value
        self.rest = np.zeros((self.nv, 2))
        self.vert_start = np.zeros(self.n + 1, dtype=np.int32)
        self.q0 = np.zeros((self.n, 6))
        self.mass = np.zeros(self.n)
        self.mass_matrix = np.zeros((self.n, 6, 6))
        L.check(lib.dabd_gpu_scene_bodies(self.h, _d(self.rest), _i(self.vert_start), _d(self.q0),
                                          _d(self.mass), _d(self.mass_matrix)))
        self.qdot0 = _f64(fl["qdot"]).copy()
        self.is_static = fl["is_static"].astype(bool)

    def __del__(self):
        try:
            L.load().dabd_gpu_scene_free(self.h)
        except Exception:
            pass


class Context:
    """One GPU's engine (dabd_gpu_ctx). num_workers=0: run_reference semantics."""

    def __init__(self, scene: Scene, device: int = 0, num_workers: int = 0,
                 part_begin: int = 0, part_end: Optional[int] = None,
                 pcg_rel_tol: Optional[float] = None, pcg_max_iters: Optional[int] = None,
                 inexact: Optional[Tuple[float, float]] = None) -> None:
        lib = L.load()
        self.scene = scene
        if part_end is None:
            part_end = max(num_workers, 1)
        h = C.c_void_p()
        L.check(lib.dabd_gpu_ctx_create(scene.h, device, num_workers, part_begin, part_end,
                                        C.byref(h)))
        self.h = h
        self.n = scene.n
        self.num_workers = num_workers
        if pcg_rel_tol is not None or pcg_max_iters is not None:
            self.set_solver(pcg_rel_tol or 1e-10, pcg_max_iters or 4000)
        if inexact is not None:
            self.set_inexact(*inexact)

    def __del__(self):
        try:
            L.load().dabd_gpu_ctx_free(self.h)
        except Exception:
            pass

    def set_solver(self, rel_tol: float, max_iters: int) -> None:
        L.check(L.load().dabd_gpu_ctx_set_solver(self.h, C.byref(L.SolverParams(rel_tol, max_iters))))

    def set_inexact(self, eta: float, factor: float = 10.0) -> None:
        """Inexact Newton inside frames (dabd_gpu_ctx_set_inexact); eta=0: off."""
        L.check(L.load().dabd_gpu_ctx_set_inexact(self.h, C.c_double(eta), C.c_double(factor)))

    def set_stream(self, stream_handle: int) -> None:
        L.check(L.load().dabd_gpu_ctx_set_stream(self.h, int(stream_handle)))

    def set_comm(self, comm) -> None:
        """Join a partition-per-GPU run (dist.TorchComm, or None to leave)."""
        L.check(L.load().dabd_gpu_ctx_set_comm(self.h, None if comm is None else C.byref(comm.struct)))
        self._comm = comm

    # ---- geometry (geometry.hpp:47-74) -------------------------------------
    def broad_phase(self, q, margin, q_end=None, subset=None) -> np.ndarray:
        q = _f64(q, (self.n, 6))
        qe = None if q_end is None else _f64(q_end, (self.n, 6))
        sub = None if subset is None else _i32(subset)
        cap = 4096
        while True:
            out = np.zeros((cap, 4), dtype=np.int32)
            cnt = C.c_int()
            st = L.load().dabd_gpu_broad_phase(self.h, _d(q), _d(qe), C.c_double(margin), _i(sub),
                                               0 if sub is None else len(sub), _i(out), cap,
                                               C.byref(cnt))
            if st == 3 and cnt.value > cap:
                cap = cnt.value
                continue
            L.check(st)
            return out[: cnt.value].copy()

    def narrow_phase(self, q, cand, d_hat):
        q = _f64(q, (self.n, 6))
        cand = _i32(cand).reshape(-1, 4)
        n = len(cand)
        out = np.zeros((max(n, 1), 4), dtype=np.int32)
        d = np.zeros(max(n, 1))
        cnt = C.c_int()
        L.check(L.load().dabd_gpu_narrow_phase(self.h, _d(q), _i(cand) if n else None, n,
                                               C.c_double(d_hat), _i(out), _d(d), C.byref(cnt)))
        return out[: cnt.value].copy(), d[: cnt.value].copy()

    def ccd_toi(self, q0, q1, subset=None) -> float:
        sub = None if subset is None else _i32(subset)
        t = C.c_double()
        L.check(L.load().dabd_gpu_ccd_toi(self.h, _d(_f64(q0, (self.n, 6))),
                                          _d(_f64(q1, (self.n, 6))), _i(sub),
                                          0 if sub is None else len(sub), C.byref(t)))
        return t.value

    def intersection_test(self, q=None, subset=None) -> bool:
        """geometry.cpp:389-454 on the device (q None: the current state)."""
        return self.audit(q, subset)[0]

    def audit(self, q=None, subset=None, cutoff: float = 0.0):
        """(intersecting, n_violating_pairs, min_distance); see dabd_gpu_audit."""
        res, nv, dm = C.c_int(), C.c_int(), C.c_double()
        sub = None if subset is None else _i32(subset)
        L.check(L.load().dabd_gpu_audit(self.h, None if q is None else _d(_f64(q, (self.n, 6))),
                                        _i(sub), 0 if sub is None else len(sub), C.c_double(cutoff),
                                        C.byref(res), C.byref(nv), C.byref(dm)))
        return bool(res.value), nv.value, dm.value

    def holder_masks(self, q, planes, w) -> np.ndarray:
        planes = _f64(planes).reshape(-1, 4)
        out = np.zeros(self.n, dtype=np.uint32)
        L.check(L.load().dabd_gpu_holder_masks(self.h, _d(_f64(q, (self.n, 6))), len(planes),
                                               _d(planes) if len(planes) else None,
                                               C.c_double(w), out.ctypes.data_as(_up)))
        return out

    # ---- objective / newton (objective.hpp:34-75, newton.hpp:25-26) --------
    def _obj_args(self, local, kappa, q_tilde, anchors, holder_mask, sim):
        local = _i32(local)
        kappa = _f64(kappa)
        q_tilde = _f64(q_tilde, (len(local), 6))
        anchors = anchors or []
        ab = _i32([a[0] for a in anchors]) if anchors else np.zeros(1, np.int32)
        azu = _f64([list(a[1]) + list(a[2]) for a in anchors]) if anchors else np.zeros(12)
        arho = _f64([a[3] for a in anchors]) if anchors else np.zeros(1)
        hm = None if holder_mask is None else np.ascontiguousarray(holder_mask, dtype=np.uint32)
        sp = sim_params(sim)
        self._tmp = (local, kappa, q_tilde, ab, azu, arho, hm, sp)
        return [len(local), _i(local), _d(kappa), _d(q_tilde), len(anchors), _i(ab), _d(azu),
                _d(arho), None if hm is None else hm.ctypes.data_as(_up), C.byref(sp)]

    def objective(self, q, local, kappa, q_tilde, sim, anchors=None, holder_mask=None, mode=0):
        args = self._obj_args(local, kappa, q_tilde, anchors, holder_mask, sim)
        nd = 6 * int(sum(1 for b in local if not self.scene.is_static[b]))
        val = C.c_double()
        grad = np.zeros(max(nd, 1))
        hess = np.zeros((max(nd, 1), max(nd, 1)))
        act, cand = C.c_int(), C.c_int()
        L.check(L.load().dabd_gpu_objective(self.h, *args, _d(_f64(q, (self.n, 6))), mode,
                                            C.byref(val), _d(grad), _d(hess), C.byref(act),
                                            C.byref(cand)))
        return dict(value=val.value, grad=grad[:nd], hess=hess[:nd, :nd], active=act.value,
                    candidates=cand.value)

    def newton_solve(self, q, local, kappa, q_tilde, sim, max_iters, tol, anchors=None,
                     holder_mask=None):
        args = self._obj_args(local, kappa, q_tilde, anchors, holder_mask, sim)
        qq = _f64(q, (self.n, 6)).copy()
        it, conv, ls = C.c_int(), C.c_int(), C.c_int()
        fu = C.c_double()
        L.check(L.load().dabd_gpu_newton_solve(self.h, *args, _d(qq), max_iters, C.c_double(tol),
                                               C.byref(it), C.byref(fu), C.byref(conv),
                                               C.byref(ls)))
        return qq, dict(iterations=it.value, final_update_inf=fu.value,
                        converged=bool(conv.value), line_search_steps=ls.value)

    # ---- stepping ----------------------------------------------------------
    def run_frames(self, n: int) -> List[dict]:
        st = (L.FrameStats * max(n, 1))()
        status = L.load().dabd_gpu_run_frames(self.h, n, st)
        comm = getattr(self, "_comm", None)
        if status != 0 and comm is not None and comm.error is not None:
            err, comm.error = comm.error, None
            raise L.DabdGpuError(status, L.load().dabd_gpu_last_error().decode()) from err
        L.check(status)
        return [{k: getattr(st[i], k) for k, _ in L.FrameStats._fields_} for i in range(n)]

    def state(self):
        q = np.zeros((self.n, 6))
        qd = np.zeros((self.n, 6))
        L.check(L.load().dabd_gpu_get_state(self.h, _d(q), _d(qd)))
        return q, qd

    def set_state(self, q, qd) -> None:
        L.check(L.load().dabd_gpu_set_state(self.h, _d(_f64(q, (self.n, 6))),
                                            _d(_f64(qd, (self.n, 6)))))

    def rho(self) -> np.ndarray:
        out = np.zeros(max(self.n, 1))
        L.check(L.load().dabd_gpu_get_rho(self.h, _d(out)))
        return out[: self.n]

    def comm_mode(self) -> int:
        """0 single process, 1 halo callback, 2 peer-memory halo (CUDA IPC)."""
        m = C.c_int()
        L.check(L.load().dabd_gpu_ctx_comm_mode(self.h, C.byref(m)))
        return m.value

    def planes(self) -> np.ndarray:
        """Interface planes the next frame partitions with ((W-1) x 4)."""
        w = max(self.num_workers - 1, 0)
        out = np.zeros(max(4 * w, 1))
        L.check(L.load().dabd_gpu_ctx_get_planes(self.h, _d(out)))
        return out[: 4 * w].reshape(w, 4)

    def partition_costs(self) -> np.ndarray:
        """Balancer input of the last committed frame (one cost per partition)."""
        out = np.zeros(max(self.num_workers, 1))
        L.check(L.load().dabd_gpu_ctx_partition_costs(self.h, _d(out)))
        return out[: self.num_workers]

    def take_trace(self, cap: int = 1 << 16) -> np.ndarray:
        rows = np.zeros((cap, 8))
        cnt = C.c_int()
        L.check(L.load().dabd_gpu_take_trace(self.h, _d(rows), cap, C.byref(cnt)))
        return rows[: cnt.value].copy()


# ---- PD load balancer (balance.hpp:9-56), host logic over the C ABI -------
def imbalance_metric(tau_i: float, tau_j: float) -> float:
    out = C.c_double()
    L.check(L.load().dabd_gpu_imbalance_metric(C.c_double(tau_i), C.c_double(tau_j), C.byref(out)))
    return out.value


def pd_update(t: float, t_prev: float, kp: float, kd: float, dp_max: float) -> float:
    out = C.c_double()
    L.check(L.load().dabd_gpu_pd_update(C.c_double(t), C.c_double(t_prev), C.c_double(kp),
                                        C.c_double(kd), C.c_double(dp_max), C.byref(out)))
    return out.value


def balance_factor(times) -> float:
    t = _f64(times)
    out = C.c_double()
    L.check(L.load().dabd_gpu_balance_factor(_d(t) if t.size else None, int(t.size), C.byref(out)))
    return out.value


class Balancer:
    """Balancer (balance.hpp:23-53): update(times, planes, w) shifts the
    planes ((n-1) x (px, py, nx, ny), in place) and returns the shifts."""

    def __init__(self, num_workers: int, kp=0.0, kd=0.0, smoothing=0.5, dp_max=0.0) -> None:
        h = C.c_void_p()
        L.check(L.load().dabd_gpu_balancer_create(
            num_workers, C.byref(L.BalanceParams(1, kp, kd, smoothing, dp_max)), C.byref(h)))
        self.h = h
        self.n = num_workers

    def __del__(self):
        try:
            L.load().dabd_gpu_balancer_free(self.h)
        except Exception:
            pass

    def update(self, times, planes: np.ndarray, w: float) -> np.ndarray:
        t = _f64(times)
        if t.size != self.n:
            raise L.DabdGpuError(4, "Balancer: worker count mismatch")
        pl = np.ascontiguousarray(planes, dtype=np.float64).reshape(-1, 4)
        applied = np.zeros(max(len(pl), 1))
        L.check(L.load().dabd_gpu_balancer_update(self.h, _d(t), len(pl), _d(pl) if len(pl) else None,
                                                  C.c_double(w), _d(applied)))
        planes[...] = pl.reshape(planes.shape)
        return applied[: len(pl)]


@dataclass
class Trajectory:
    """sim.hpp:81-85 plus per-frame stats, the ADMM trace and the final rho."""

    q: np.ndarray
    q_dot: np.ndarray
    h: np.ndarray
    stats: List[dict]
    trace: np.ndarray
    rho: np.ndarray


def _run(scene: SceneData, frames: int, workers: int, device: int, **solver) -> Trajectory:
    sc = Scene(scene)
    ctx = Context(sc, device=device, num_workers=workers, **solver)
    qs, qds, hs, stats = [], [], [], []
    for _ in range(frames):
        st = ctx.run_frames(1)[0]
        q, qd = ctx.state()
        qs.append(q)
        qds.append(qd)
        hs.append(st["h"])
        stats.append(st)
    return Trajectory(np.array(qs).reshape(frames, sc.n, 6), np.array(qds).reshape(frames, sc.n, 6),
                      np.array(hs), stats, ctx.take_trace(), ctx.rho())


def run_reference(scene: SceneData, frames: Optional[int] = None, device: int = 0,
                  **solver) -> Trajectory:
    """Single-domain solve (proj/src/sim.cpp:186-249) on the GPU."""
    return _run(scene, scene.frames if frames is None else frames, 0, device, **solver)


def run_distributed(scene: SceneData, workers: int, frames: Optional[int] = None,
                    device: int = 0, **solver) -> Trajectory:
    """Consensus-ADMM runtime semantics (proj/src/runtime.cpp:110-694) with
    `workers` slab partitions, all solved on one GPU in batched kernels."""
    return _run(scene, scene.frames if frames is None else frames, workers, device, **solver)


# ---- snapshot files (proj/src/sim.cpp:34-108, same byte layout as
#      include/dabd_gpu.hpp): [u64 frame][u64 n_dynamic][per dynamic body:
#      u64 id, 6 f64 q, 6 f64 q_dot], bodies ascending by id ----------------
_SNAP_REC = np.dtype([("id", "<u8"), ("q", "<f8", 6), ("q_dot", "<f8", 6)])


def frame_path(out_dir: str, frame: int) -> str:
    return f"{out_dir}/frame_{frame:04d}.bin"


def write_snapshot(path: str, frame: int, is_static, q, q_dot) -> None:
    dyn = np.nonzero(~np.asarray(is_static, dtype=bool))[0]
    rec = np.zeros(len(dyn), dtype=_SNAP_REC)
    rec["id"] = dyn
    rec["q"] = np.asarray(q, dtype=np.float64)[dyn]
    rec["q_dot"] = np.asarray(q_dot, dtype=np.float64)[dyn]
    with open(path, "wb") as f:
        f.write(np.array([frame, len(dyn)], dtype="<u8").tobytes())
        f.write(rec.tobytes())


def read_snapshot(path: str):
    """(frame, ids, q [n][6], q_dot [n][6]); raises on a truncated file."""
    raw = open(path, "rb").read()
    if len(raw) < 16:
        raise L.DabdGpuError(1, f"snapshot: truncated file {path}")
    frame, n = np.frombuffer(raw[:16], dtype="<u8")
    if len(raw) < 16 + int(n) * _SNAP_REC.itemsize:
        raise L.DabdGpuError(1, f"snapshot: truncated file {path}")
    rec = np.frombuffer(raw[16:16 + int(n) * _SNAP_REC.itemsize], dtype=_SNAP_REC)
    return int(frame), rec["id"].astype(np.int64), rec["q"].copy(), rec["q_dot"].copy()


def load_trajectory(out_dir: str, initial_q) -> Trajectory:
    """sim.cpp:53-78: frame_0000.bin, frame_0001.bin, ... until one is missing;
    static bodies keep `initial_q`."""
    import os

    init = np.asarray(initial_q, dtype=np.float64)
    qs, qds = [], []
    while os.path.exists(frame_path(out_dir, len(qs))):
        _, ids, q, qd = read_snapshot(frame_path(out_dir, len(qs)))
        qq, qqd = init.copy(), np.zeros_like(init)
        qq[ids], qqd[ids] = q, qd
        qs.append(qq)
        qds.append(qqd)
    if not qs:
        raise L.DabdGpuError(1, f"load_trajectory: no snapshots in {out_dir}")
    return Trajectory(np.array(qs), np.array(qds), np.zeros(len(qs)), [], np.zeros((0, 8)),
                      np.zeros(0))


# ---- 3D affine-body contact terms (no reference) ----
def contact3d_terms(kind, qa, qb, rest, d_hat: float, kappa: float, weight: float = 1.0,
                    project: bool = True, hessian: bool = True, device: int = 0) -> dict:
    """Per pair: kind 0 point-triangle / 1 edge-edge, qa/qb [n][12], rest
    [n][4][3] -> d, type, value, grad [n][24], hess [n][24][24] (see
    dabd_gpu_contact3d_terms)."""
    kind = _i32(kind).reshape(-1)
    n = len(kind)
    qa = _f64(qa, (n, 12))
    qb = _f64(qb, (n, 12))
    rest = _f64(rest, (n, 4, 3))
    d = np.zeros(max(n, 1))
    t = np.zeros(max(n, 1), dtype=np.int32)
    v = np.zeros(max(n, 1))
    g = np.zeros((max(n, 1), 24))
    h = np.zeros((max(n, 1), 24, 24)) if hessian else None
    L.check(L.load().dabd_gpu_contact3d_terms(device, n, _i(kind), _d(qa), _d(qb), _d(rest),
                                              C.c_double(d_hat), C.c_double(kappa),
                                              C.c_double(weight), int(project), _d(d), _i(t),
                                              _d(v), _d(g), _d(h)))
    out = dict(d=d[:n], type=t[:n], value=v[:n], grad=g[:n])
    if hessian:
        out["hess"] = h[:n]
    return out


def ccd3d(kind, qa0, qa1, qb0, qb1, rest, device: int = 0) -> np.ndarray:
    """Additive CCD per 3D pair (dabd_gpu_ccd3d): toi in [0, 1]."""
    kind = _i32(kind).reshape(-1)
    n = len(kind)
    arrs = [_f64(a, (n, 12)) for a in (qa0, qa1, qb0, qb1)]
    rest = _f64(rest, (n, 4, 3))
    toi = np.zeros(max(n, 1))
    L.check(L.load().dabd_gpu_ccd3d(device, n, _i(kind), *[_d(a) for a in arrs], _d(rest), _d(toi)))
    return toi[:n]


def body3d_moments(verts, tris, density: float = 1000.0):
    """Mass moments of a closed triangle surface (dabd_gpu_body3d_moments):
    (moments10, centroid, volume)."""
    v = _f64(verts).reshape(-1, 3)
    t = _i32(tris).reshape(-1, 3)
    mom, cen, vol = np.zeros(10), np.zeros(3), C.c_double()
    L.check(L.load().dabd_gpu_body3d_moments(len(v), _d(v), len(t), _i(t), C.c_double(density),
                                             _d(mom), _d(cen), C.byref(vol)))
    return mom, cen, vol.value


def body3d_terms(q, qt, moments10, w, scale: float, project: bool = True, hessian: bool = True,
                 device: int = 0) -> dict:
    """Inertia + orthogonality terms of 12-DoF bodies (dabd_gpu_body3d_terms)."""
    q = _f64(q).reshape(-1, 12)
    n = len(q)
    qt = _f64(qt, (n, 12))
    mo = _f64(moments10, (n, 10))
    w = _f64(w).reshape(n)
    v = np.zeros(max(n, 1))
    g = np.zeros((max(n, 1), 12))
    h = np.zeros((max(n, 1), 12, 12)) if hessian else None
    L.check(L.load().dabd_gpu_body3d_terms(device, n, _d(q), _d(qt), _d(mo), _d(w), C.c_double(scale),
                                           int(project), _d(v), _d(g), _d(h)))
    out = dict(value=v[:n], grad=g[:n])
    if hessian:
        out["hess"] = h[:n]
    return out


def broad_phase3d(q, meshes, margin: float, q_end=None, device: int = 0) -> np.ndarray:
    """3D broad phase (dabd_gpu_broad_phase3d). meshes: per body (verts [k][3]
    rest coordinates, tris [t][3], edges [e][2]); returns [m][5] rows (kind,
    a, b, primitive a, primitive b), sorted."""
    n = len(meshes)
    q = _f64(q, (n, 12))
    qe = None if q_end is None else _f64(q_end, (n, 12))
    vs, ts, es = [0], [0], [0]
    V, T, E = [], [], []
    for v, t, e in meshes:
        V.append(np.asarray(v, float).reshape(-1, 3))
        T.append(np.asarray(t, np.int32).reshape(-1, 3))
        E.append(np.asarray(e, np.int32).reshape(-1, 2))
        vs.append(vs[-1] + len(V[-1]))
        ts.append(ts[-1] + len(T[-1]))
        es.append(es[-1] + len(E[-1]))
    V = _f64(np.concatenate(V) if V else np.zeros((0, 3)))
    T = _i32(np.concatenate(T) if T else np.zeros((0, 3)))
    E = _i32(np.concatenate(E) if E else np.zeros((0, 2)))
    vs, ts, es = _i32(vs), _i32(ts), _i32(es)
    cap = 4096
    while True:
        out = np.zeros((cap, 5), dtype=np.int32)
        cnt = C.c_int()
        st = L.load().dabd_gpu_broad_phase3d(device, n, _d(q), _d(qe), _i(vs), _d(V), _i(ts), _i(T), _i(es),
                                             _i(E), C.c_double(margin), _i(out), cap, C.byref(cnt))
        if st == 3 and cnt.value > cap:
            cap = cnt.value
            continue
        L.check(st)
        return out[: cnt.value].copy()


def cube_mesh(half):
    """Closed, outward-oriented box surface about its centroid: verts [8][3],
    tris [12][3], edges [12][2] (half = scalar or (hx, hy, hz))."""
    hx, hy, hz = (half, half, half) if np.isscalar(half) else half
    v = np.array([[x, y, z] for x in (-hx, hx) for y in (-hy, hy) for z in (-hz, hz)], float)
    # vertex index = 4 ix + 2 iy + iz; two triangles per face, outward normals
    quads = [(0, 1, 3, 2), (4, 6, 7, 5), (0, 4, 5, 1), (2, 3, 7, 6), (0, 2, 6, 4), (1, 5, 7, 3)]
    tris = []
    for a, b, c, d in quads:
        tris += [(a, b, c), (a, c, d)]
    edges = sorted({tuple(sorted(e)) for a, b, c, d in quads for e in ((a, b), (b, c), (c, d), (d, a))})
    return v, np.array(tris, np.int32), np.array(edges, np.int32)


class Sim3D:
    """3D affine-body scene stepping on the device (dabd_gpu_sim3d_*; the
    reference's run_reference + newton_solve in 3D). bodies: list of
    (verts [k][3] about the centroid, tris, edges, centre (3,), static)."""

    def __init__(self, bodies, h=1.0 / 60.0, gravity=(0.0, -9.81, 0.0), d_hat=1e-2, kappa=1e3,
                 kappa_arap=1e4, theta=1e-3, scene_scale=1.0, newton_cap=64, pcg_rel_tol=1e-10,
                 pcg_max_iters=4000, density=1000.0, qd0=None, device: int = 0) -> None:
        lib = L.load()
        n = len(bodies)
        vs, ts, es, V, T, E, mom, vol, stat = [0], [0], [0], [], [], [], [], [], []
        q0 = np.zeros((n, 12))
        for i, (v, t, e, centre, static) in enumerate(bodies):
            v = np.asarray(v, float).reshape(-1, 3)
            V.append(v)
            T.append(np.asarray(t, np.int32).reshape(-1, 3))
            E.append(np.asarray(e, np.int32).reshape(-1, 2))
            vs.append(vs[-1] + len(v))
            ts.append(ts[-1] + len(T[-1]))
            es.append(es[-1] + len(E[-1]))
            m, _, vl = body3d_moments(v, T[-1], density)
            mom.append(m)
            vol.append(vl)
            stat.append(1 if static else 0)
            q0[i, :3] = centre
            q0[i, 3:] = np.eye(3).reshape(-1)
        self.n = n
        self.is_static = np.array(stat, bool)
        self._arrays = (_i32(vs), _f64(np.concatenate(V)), _i32(ts), _i32(np.concatenate(T)), _i32(es),
                        _i32(np.concatenate(E)), _i32(stat), _f64(np.array(mom)), _f64(vol))
        qd = np.zeros((n, 12)) if qd0 is None else _f64(qd0, (n, 12))
        p = L.Sim3dParams(h, (C.c_double * 3)(*gravity), d_hat, kappa, kappa_arap, theta, scene_scale,
                          newton_cap, pcg_rel_tol, pcg_max_iters)
        a = self._arrays
        h_ = C.c_void_p()
        L.check(lib.dabd_gpu_sim3d_create(device, n, _i(a[0]), _d(a[1]), _i(a[2]), _i(a[3]), _i(a[4]),
                                          _i(a[5]), _i(a[6]), _d(a[7]), _d(a[8]), _d(_f64(q0)), _d(qd),
                                          C.byref(p), C.byref(h_)))
        self.h = h_
        self.params = p

    def __del__(self):
        try:
            L.load().dabd_gpu_sim3d_free(self.h)
        except Exception:
            pass

    def run(self, frames: int) -> List[dict]:
        st = (L.Sim3dStats * max(frames, 1))()
        L.check(L.load().dabd_gpu_sim3d_run(self.h, frames, st))
        return [{k: getattr(st[i], k) for k, _ in L.Sim3dStats._fields_} for i in range(frames)]

    def state(self):
        q, qd = np.zeros((self.n, 12)), np.zeros((self.n, 12))
        L.check(L.load().dabd_gpu_sim3d_get_state(self.h, _d(q), _d(qd)))
        return q, qd

    def set_state(self, q, qd) -> None:
        L.check(L.load().dabd_gpu_sim3d_set_state(self.h, _d(_f64(q, (self.n, 12))), _d(_f64(qd, (self.n, 12)))))

    def system(self):
        """(H, g, dq) of the next frame's first Newton iteration (dynamic bodies)."""
        N = 12 * self.n
        H, g, dq, rows = np.zeros((N, N)), np.zeros(N), np.zeros(N), C.c_int()
        L.check(L.load().dabd_gpu_sim3d_system(self.h, _d(H), _d(g), _d(dq), C.byref(rows)))
        m = 12 * rows.value
        return H[:m, :m] if m == N else H.reshape(-1)[: m * m].reshape(m, m), g[:m], dq[:m]


def consensus_step(q, u, rho, z_prev, rho0, adapt=None, device: int = 0) -> dict:
    """One consensus / dual / residual / rho-adaptation step for split bodies
    with two replicas (dabd_gpu_consensus_step). q, u: [n][2][6]."""
    from .scene import AdaptParams

    a = adapt or AdaptParams()
    q = _f64(q).reshape(-1, 2, 6)
    n = len(q)
    u = _f64(u, (n, 2, 6))
    rho, zp, r0 = _f64(rho).reshape(n), _f64(z_prev, (n, 6)), _f64(rho0).reshape(n)
    z, un = np.zeros((max(n, 1), 6)), np.zeros((max(n, 1), 2, 6))
    r, s, rn = np.zeros(max(n, 1)), np.zeros(max(n, 1)), np.zeros(max(n, 1))
    L.check(L.load().dabd_gpu_consensus_step(
        device, n, _d(q), _d(u), _d(rho), _d(zp), _d(r0),
        C.byref(L.AdaptParams(a.beta, a.tau, a.mu, a.sigma_min, a.sigma_max, int(a.adapt_enabled))),
        _d(z), _d(un), _d(r), _d(s), _d(rn)))
    return dict(z=z[:n], u=un[:n], r=r[:n], s=s[:n], rho=rn[:n])


def check_stopping(dq: float, r: float, s: float, tois, h: float, l: float, theta: float) -> bool:
    """The controller's stop rule (consensus.cpp:54-64) as the multi-partition
    frame evaluates it (dabd_gpu_check_stopping; host code, no device)."""
    t = _f64(tois).reshape(-1)
    end = C.c_int()
    L.check(L.load().dabd_gpu_check_stopping(
        C.c_double(dq), C.c_double(r), C.c_double(s), _d(t) if len(t) else None, len(t),
        C.c_double(h), C.c_double(l), C.c_double(theta), C.byref(end)))
    return bool(end.value)


def timestep_apply(h0: float, max_halvings: int, events) -> np.ndarray:
    """TimestepController (consensus.hpp:60-87) over frame outcomes
    (0 failed, 1 committed); h after each event (dabd_gpu_timestep_apply)."""
    ev = np.ascontiguousarray(events, dtype=np.int32)
    out = np.zeros(max(len(ev), 1))
    L.check(L.load().dabd_gpu_timestep_apply(C.c_double(h0), int(max_halvings), _i(ev), len(ev), _d(out)))
    return out[: len(ev)]
