"""TEST INFRASTRUCTURE ONLY -- ctypes wrapper of the CPU oracle (liboracle.so).

The oracle is a C++ restatement of the reference hot path (see oracle.hpp).
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
import this module; the product (paper_2605_15875_b200) never does.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "liboracle.so")
_lib = None

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_up = C.POINTER(C.c_uint32)


class OracleError(RuntimeError):
    pass


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = C.CDLL(_LIB_PATH)
        _lib.oracle_last_error.restype = C.c_char_p
        _lib.oracle_scene_new.restype = C.c_void_p
        _lib.oracle_scene_free.argtypes = [C.c_void_p]
    return _lib


def _d(a):
    return None if a is None else a.ctypes.data_as(_dp)


def _i(a):
    return None if a is None else a.ctypes.data_as(_ip)


def _check(rc: int) -> None:
    if rc != 0:
        raise OracleError(lib().oracle_last_error().decode())


def _f64(a, shape=None):
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return arr if shape is None else arr.reshape(shape)


def _i32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


class Scene:
    """Oracle scene built from a paper_2605_15875_b200.scene.SceneData."""

    def __init__(self, scene) -> None:
        L = lib()
        fl = scene.flat()
        self._keep = fl
        self.scene = scene
        self.n = fl["n_bodies"]
        L.oracle_scene_new.argtypes = [C.c_int, _ip, _ip, _dp, _dp, _ip, _dp, _dp]
        h = L.oracle_scene_new(self.n, _i(fl["body_loop_start"]), _i(fl["loop_vert_start"]),
                               _d(_f64(fl["verts"])), _d(fl["density"]), _i(fl["is_static"]),
                               _d(fl["arap_scale"]), _d(_f64(fl["qdot"])))
        if not h:
            raise OracleError(L.oracle_last_error().decode())
        self.h = C.c_void_p(h)
        planes = _f64(fl["planes"]).reshape(-1)
        _check(L.oracle_scene_set_params(
            self.h, _d(scene.params.as_array()), _d(scene.adapt.as_array()),
            int(scene.adapt.adapt_enabled), int(scene.admm_max_iterations),
            int(scene.newton_cap), int(scene.max_halvings), C.c_double(scene.w_min),
            len(scene.planes), _d(planes) if planes.size else None,
            int(scene.force_split_frames)))
        for body, f in fl["force_split"]:
            _check(L.oracle_scene_set_force_split(self.h, body, C.c_double(f[0]),
                                                  C.c_double(f[1])))
        nb, nv = C.c_int(), C.c_int()
        _check(L.oracle_scene_counts(self.h, C.byref(nb), C.byref(nv)))
        self.nv = nv.value
        self.rest = np.zeros((self.nv, 2))
        self.vert_start = np.zeros(self.n + 1, dtype=np.int32)
        self.q0 = np.zeros((self.n, 6))
        self.mass = np.zeros(self.n)
        self.mass_matrix = np.zeros((self.n, 6, 6))
        self.rest_area = np.zeros(self.n)
        _check(L.oracle_scene_bodies(self.h, _d(self.rest), _i(self.vert_start), _d(self.q0),
                                     _d(self.mass), _d(self.mass_matrix), _d(self.rest_area)))
        self.qdot0 = _f64(fl["qdot"]).copy()
        self.is_static = fl["is_static"].astype(bool)

    def __del__(self):
        try:
            lib().oracle_scene_free(self.h)
        except Exception:
            pass

    def set_state(self, q, qdot):
        """Start subsequent run() calls from (q, qdot) instead of the scene's initial state."""
        _check(lib().oracle_scene_set_state(self.h, _d(_f64(q, (self.n, 6))),
                                            _d(_f64(qdot, (self.n, 6)))))

    # -- geometry -----------------------------------------------------------
    def broad_phase(self, q, margin, q_end=None, subset=None):
        q = _f64(q, (self.n, 6))
        qe = None if q_end is None else _f64(q_end, (self.n, 6))
        sub = None if subset is None else _i32(subset)
        cap = 1 << 16
        while True:
            out = np.zeros((cap, 4), dtype=np.int32)
            cnt = C.c_int()
            rc = lib().oracle_broad_phase(self.h, _d(q), _d(qe), C.c_double(margin), _i(sub),
                                          0 if sub is None else len(sub), _i(out), cap,
                                          C.byref(cnt))
            if rc != 0 and cnt.value > cap:
                cap = cnt.value
                continue
            _check(rc)
            return out[: cnt.value].copy()

    def narrow_phase(self, q, cand, d_hat):
        q = _f64(q, (self.n, 6))
        cand = _i32(cand).reshape(-1, 4)
        out = np.zeros((max(len(cand), 1), 4), dtype=np.int32)
        d = np.zeros(max(len(cand), 1))
        cnt = C.c_int()
        _check(lib().oracle_narrow_phase(self.h, _d(q), _i(cand), len(cand), C.c_double(d_hat),
                                         _i(out), _d(d), C.byref(cnt)))
        return out[: cnt.value].copy(), d[: cnt.value].copy()

    def ccd_toi(self, q0, q1, subset=None):
        sub = None if subset is None else _i32(subset)
        t = C.c_double()
        _check(lib().oracle_ccd_toi(self.h, _d(_f64(q0, (self.n, 6))), _d(_f64(q1, (self.n, 6))),
                                    _i(sub), 0 if sub is None else len(sub), C.byref(t)))
        return t.value

    def ccd_toi_pairs(self, q0, q1, cand):
        cand = _i32(cand).reshape(-1, 4)
        t = C.c_double()
        _check(lib().oracle_ccd_toi_pairs(self.h, _d(_f64(q0, (self.n, 6))),
                                          _d(_f64(q1, (self.n, 6))), _i(cand), len(cand),
                                          C.byref(t)))
        return t.value

    def holder_masks(self, q, planes, w):
        planes = _f64(planes).reshape(-1, 4)
        out = np.zeros(self.n, dtype=np.uint32)
        _check(lib().oracle_holder_masks(self.h, _d(_f64(q, (self.n, 6))), len(planes),
                                         _d(planes) if len(planes) else None, C.c_double(w),
                                         out.ctypes.data_as(_up)))
        return out

    def max_vertex_speed(self, qdot):
        out = np.zeros(self.n)
        _check(lib().oracle_max_vertex_speed(self.h, _d(_f64(qdot, (self.n, 6))), _d(out)))
        return out

    def intersection_test(self, q, subset=None):
        sub = None if subset is None else _i32(subset)
        r = C.c_int()
        _check(lib().oracle_intersection_test(self.h, _d(_f64(q, (self.n, 6))), _i(sub),
                                              0 if sub is None else len(sub), C.byref(r)))
        return bool(r.value)

    def min_pair_distance(self, q, subset=None, skip_static_pairs=True):
        sub = None if subset is None else _i32(subset)
        r = C.c_double()
        _check(lib().oracle_min_pair_distance(self.h, _d(_f64(q, (self.n, 6))), _i(sub),
                                              0 if sub is None else len(sub),
                                              int(skip_static_pairs), C.byref(r)))
        return r.value

    def predicted_position(self, q, qdot, f, h):
        out = np.zeros((self.n, 6))
        _check(lib().oracle_predicted_position(self.h, _d(_f64(q, (self.n, 6))),
                                               _d(_f64(qdot, (self.n, 6))),
                                               _d(_f64(f, (self.n, 6))), C.c_double(h), _d(out)))
        return out

    def contact_energy(self, q, a, b, v, e, d_hat, kappa):
        val = C.c_double()
        g = np.zeros(12)
        H = np.zeros((12, 12))
        _check(lib().oracle_contact_energy(self.h, _d(_f64(q, (self.n, 6))), a, b, v, e,
                                           C.c_double(d_hat), C.c_double(kappa), C.byref(val),
                                           _d(g), _d(H)))
        return val.value, g, H

    # -- objective / newton --------------------------------------------------
    def _obj_args(self, local, kappa, q_tilde, anchors, holder_mask, sim):
        local = _i32(local)
        kappa = _f64(kappa)
        q_tilde = _f64(q_tilde, (len(local), 6))
        anchors = anchors or []
        ab = _i32([a[0] for a in anchors]) if anchors else np.zeros(1, np.int32)
        azu = _f64([list(a[1]) + list(a[2]) for a in anchors]) if anchors else np.zeros(12)
        arho = _f64([a[3] for a in anchors]) if anchors else np.zeros(1)
        hm = None if holder_mask is None else np.ascontiguousarray(holder_mask, dtype=np.uint32)
        self._tmp = (local, kappa, q_tilde, ab, azu, arho, hm, sim)
        return [len(local), _i(local), _d(kappa), _d(q_tilde), len(anchors), _i(ab), _d(azu),
                _d(arho), None if hm is None else hm.ctypes.data_as(_up), _d(sim)]

    def objective(self, q, local, kappa, q_tilde, sim, anchors=None, holder_mask=None, mode=0):
        """mode 0 value, 1 value w/o anchors, 2 derivatives, 3 unprojected derivatives."""
        args = self._obj_args(local, kappa, q_tilde, anchors, holder_mask, _f64(sim))
        nd = 6 * int(sum(1 for b in local if not self.is_static[b]))
        val = C.c_double()
        grad = np.zeros(max(nd, 1))
        hess = np.zeros((max(nd, 1), max(nd, 1)))
        ndo, act, cand = C.c_int(), C.c_int(), C.c_int()
        _check(lib().oracle_objective(self.h, *args, _d(_f64(q, (self.n, 6))), mode,
                                      C.byref(val), _d(grad), _d(hess), C.byref(ndo),
                                      C.byref(act), C.byref(cand)))
        return dict(value=val.value, grad=grad[:nd], hess=hess[:nd, :nd], active=act.value,
                    candidates=cand.value)

    def newton_solve(self, q, local, kappa, q_tilde, sim, max_iters, tol, anchors=None,
                     holder_mask=None):
        args = self._obj_args(local, kappa, q_tilde, anchors, holder_mask, _f64(sim))
        qq = _f64(q, (self.n, 6)).copy()
        it, conv, ls = C.c_int(), C.c_int(), C.c_int()
        fu = C.c_double()
        _check(lib().oracle_newton_solve(self.h, *args, _d(qq), max_iters, C.c_double(tol),
                                         C.byref(it), C.byref(fu), C.byref(conv), C.byref(ls)))
        return qq, dict(iterations=it.value, final_update_inf=fu.value,
                        converged=bool(conv.value), line_search_steps=ls.value)

    # -- drivers --------------------------------------------------------------
    def run(self, frames, workers=0):
        """workers=0: run_reference (sim.cpp:186-249); else distributed semantics."""
        n = self.n
        q = np.zeros((frames, n, 6))
        qd = np.zeros((frames, n, 6))
        hh = np.zeros(frames)
        st = np.zeros((frames, 4), dtype=np.int32)
        cap = 300 * frames * 5 + 16
        tr = np.zeros((cap, 8))
        cnt = C.c_int()
        rho = np.zeros(max(n, 1))
        _check(lib().oracle_run(self.h, workers, frames, _d(q), _d(qd), _d(hh), _i(st), _d(tr),
                                cap, C.byref(cnt), _d(rho)))
        return dict(q=q, qdot=qd, h=hh, attempts=st[:, 0], admm=st[:, 1], newton=st[:, 2],
                    ls=st[:, 3], trace=tr[: min(cnt.value, cap)], rho=rho[:n])


def point_edge_distance(p, e0, e1, with_hessian=True):
    x = _f64([p[0], p[1], e0[0], e0[1], e1[0], e1[1]])
    d = C.c_double()
    g = np.zeros(6)
    H = np.zeros((6, 6))
    _check(lib().oracle_point_edge_distance(_d(x), int(with_hessian), C.byref(d), _d(g), _d(H)))
    return d.value, g, H


def barrier_energy(d, d_hat, kappa):
    out = np.zeros(3)
    _check(lib().oracle_barrier(C.c_double(d), C.c_double(d_hat), C.c_double(kappa), _d(out)))
    return out


def inertia_energy(q, qt, M):
    v = C.c_double()
    g = np.zeros(6)
    _check(lib().oracle_inertia_energy(_d(_f64(q)), _d(_f64(qt)), _d(_f64(M)), C.byref(v), _d(g)))
    return v.value, g


def arap_energy(q, kappa, area):
    v = C.c_double()
    g = np.zeros(6)
    H = np.zeros((6, 6))
    _check(lib().oracle_arap_energy(_d(_f64(q)), C.c_double(kappa), C.c_double(area),
                                    C.byref(v), _d(g), _d(H)))
    return v.value, g, H


def clamp_psd(M):
    M = _f64(M)
    n = M.shape[0]
    out = np.zeros_like(M)
    _check(lib().oracle_clamp_psd(n, _d(M), _d(out)))
    return out


def contact3d_value(kind, qa, qb, rest, d_hat, kappa, weight=1.0):
    """oracle/geometry3d.cpp: (d, type, value) of one 3D PT (kind 0) / EE (kind 1) pair."""
    d, t, v = C.c_double(), C.c_int(), C.c_double()
    rc = lib().oracle_contact3d_value(int(kind), _d(_f64(qa)), _d(_f64(qb)), _d(_f64(rest)),
                                      C.c_double(d_hat), C.c_double(kappa), C.c_double(weight),
                                      C.byref(d), C.byref(t), C.byref(v))
    if rc != 0:
        raise OracleError("contact3d: d <= 0")
    return d.value, t.value, v.value


def ccd3d(kind, qa0, qa1, qb0, qb1, rest):
    """oracle/geometry3d.cpp additive CCD of one 3D pair."""
    f = lib().oracle_ccd3d
    f.restype = C.c_double
    return f(int(kind), _d(_f64(qa0)), _d(_f64(qa1)), _d(_f64(qb0)), _d(_f64(qb1)), _d(_f64(rest)))


# ---- 3D affine bodies (test-only restatements, numpy; parity unpinned) ----
def polyhedron_moments_tets(verts, tris, density):
    """Mass moments of a closed, outward-oriented triangle surface by signed
    tetrahedra from the origin (a different decomposition than the library's
    divergence-theorem integrals): (moments10 about the centroid, centroid, V)."""
    v = np.asarray(verts, dtype=np.float64).reshape(-1, 3)
    V, first, second = 0.0, np.zeros(3), np.zeros((3, 3))
    for t in np.asarray(tris).reshape(-1, 3):
        a, b, c = v[t[0]], v[t[1]], v[t[2]]
        vol = np.dot(a, np.cross(b, c)) / 6.0
        V += vol
        first += vol * (a + b + c) / 4.0
        s = a + b + c
        second += vol / 20.0 * (np.outer(a, a) + np.outer(b, b) + np.outer(c, c) + np.outer(s, s))
    cen = first / V
    S = second - V * np.outer(cen, cen)
    mom = density * np.array([V, 0, 0, 0, S[0, 0], S[0, 1], S[0, 2], S[1, 1], S[1, 2], S[2, 2]])
    mom[1:4] = 0.0
    return mom, cen, V


def body3d_value(q, qt, mom, w, scale):
    """1/2 (q - qt)^T M (q - qt) + scale w ||A^T A - I||_F^2 (energy.cpp:7-48 in 3D)."""
    q, qt = np.asarray(q, float), np.asarray(qt, float)
    m, s = mom[0], np.asarray(mom[1:4])
    S = np.array([[mom[4], mom[5], mom[6]], [mom[5], mom[7], mom[8]], [mom[6], mom[8], mom[9]]])
    M = np.zeros((12, 12))
    for r in range(3):
        M[r, r] = m
        M[r, 3 + 3 * r:6 + 3 * r] = s
        M[3 + 3 * r:6 + 3 * r, r] = s
        M[3 + 3 * r:6 + 3 * r, 3 + 3 * r:6 + 3 * r] = S
    dq = q - qt
    A = q[3:].reshape(3, 3)
    G = A.T @ A - np.eye(3)
    return 0.5 * dq @ M @ dq + scale * w * float(np.sum(G * G))


def broad_phase3d(q, meshes, margin, q_end=None):
    """Brute-force 3D broad phase with the library's box rules (test-only):
    every body pair whose inflated boxes overlap; PT both orders (point box
    vs inflated triangle box), EE once with a < b (edge box vs inflated edge
    box of b). World points round like x = ((A0 xb + A1 yb) + A2 zb) + p."""
    q = np.asarray(q, float).reshape(-1, 12)
    qe = None if q_end is None else np.asarray(q_end, float).reshape(-1, 12)

    def world(qq, xb):
        A = qq[3:].reshape(3, 3)
        X = np.empty_like(xb)
        for r in range(3):
            X[:, r] = ((A[r, 0] * xb[:, 0] + A[r, 1] * xb[:, 1]) + A[r, 2] * xb[:, 2]) + qq[r]
        return X

    def box(b, idx):
        xb = np.asarray(meshes[b][0], float).reshape(-1, 3)[list(idx)]
        pts = [world(q[b], xb)] + ([world(qe[b], xb)] if qe is not None else [])
        P = np.vstack(pts)
        return P.min(axis=0), P.max(axis=0)

    def ov(a, b):
        return bool(np.all(a[0] <= b[1]) and np.all(b[0] <= a[1]))

    def infl(bx):
        return (bx[0] - margin, bx[1] + margin)

    n = len(meshes)
    bb = [infl(box(b, range(len(meshes[b][0])))) for b in range(n)]
    out = []
    for a in range(n):
        for b in range(a + 1, n):
            if not ov(bb[a], bb[b]):
                continue
            for pa, tb in ((a, b), (b, a)):
                tris = np.asarray(meshes[tb][1]).reshape(-1, 3)
                tboxes = [infl(box(tb, t)) for t in tris]
                for v in range(len(meshes[pa][0])):
                    pbx = box(pa, [v])
                    for ti, tbx in enumerate(tboxes):
                        if ov(pbx, tbx):
                            out.append((0, pa, tb, v, ti))
            ea = np.asarray(meshes[a][2]).reshape(-1, 2)
            eb = np.asarray(meshes[b][2]).reshape(-1, 2)
            ebx = [infl(box(b, e)) for e in eb]
            for i, e in enumerate(ea):
                abx = box(a, e)
                for j, bx in enumerate(ebx):
                    if ov(abx, bx):
                        out.append((1, a, b, i, j))
    out.sort()
    return np.array(out, dtype=np.int32).reshape(-1, 5)


def consensus_step(q, u, rho, z_prev, rho0, adapt6):
    """oracle/capi.cpp oracle_consensus_step (consensus.cpp:9-52)."""
    q = _f64(q).reshape(-1, 2, 6)
    n = len(q)
    z, un = np.zeros((max(n, 1), 6)), np.zeros((max(n, 1), 2, 6))
    r, s, rn = np.zeros(max(n, 1)), np.zeros(max(n, 1)), np.zeros(max(n, 1))
    _check(lib().oracle_consensus_step(n, _d(q), _d(_f64(u, (n, 2, 6))), _d(_f64(rho)), _d(_f64(z_prev, (n, 6))),
                                       _d(_f64(rho0)), _d(_f64(adapt6)), _d(z), _d(un), _d(r), _d(s), _d(rn)))
    return dict(z=z[:n], u=un[:n], r=r[:n], s=s[:n], rho=rn[:n])


def consensus_update(qu, rho):
    """consensus.cpp:9-21 with per-replica weights (oracle_consensus_update)."""
    qu = _f64(qu).reshape(-1, 6)
    z = np.zeros(6)
    n = len(qu)
    _check(lib().oracle_consensus_update(n, _d(qu), _d(_f64(rho)) if n else None, _d(z)))
    return z


def init_rho(mass, beta):
    out = C.c_double()
    _check(lib().oracle_init_rho(C.c_double(mass), C.c_double(beta), C.byref(out)))
    return out.value


def adapt_rho(rho, r, s, adapt6, rho0):
    out = C.c_double()
    _check(lib().oracle_adapt_rho(C.c_double(rho), C.c_double(r), C.c_double(s),
                                  _d(_f64(adapt6)), C.c_double(rho0), C.byref(out)))
    return out.value


def check_stopping(dq, r, s, tois, h, l, theta):
    t = _f64(tois).reshape(-1)
    end = C.c_int()
    _check(lib().oracle_check_stopping(*(C.c_double(x) for x in (dq, r, s)), _d(t), len(t),
                                       *(C.c_double(x) for x in (h, l, theta)), C.byref(end)))
    return bool(end.value)


def timestep_apply(h0, max_halvings, events):
    ev = np.asarray(events, dtype=np.int32)
    out = np.zeros(max(len(ev), 1))
    _check(lib().oracle_timestep_apply(C.c_double(h0), int(max_halvings), _i(ev), len(ev), _d(out)))
    return out[: len(ev)]


def contact_replication(mask_a, mask_b):
    kc = C.c_int()
    _check(lib().oracle_contact_replication(C.c_uint32(mask_a), C.c_uint32(mask_b), C.byref(kc)))
    return kc.value
