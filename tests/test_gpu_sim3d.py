"""3D scene stepping on the device (include/dabd_gpu.h
dabd_gpu_sim3d_*): run_reference (sim.cpp:186-249) with newton.cpp:7-71 for
12-DoF affine bodies. The reference is 2D, so no reference 3D frame exists;
the checks are analytic (free fall is the predicted position exactly),
structural (the assembled Newton system equals the per-term kernels summed in
numpy, the PCG direction solves it) and physical (a dropped stack stays
penetration-free, every frame converges, the stack comes to rest in order).
"""

import numpy as np
import pytest

from paper_2605_15875_b200 import api

pytestmark = pytest.mark.gpu

H = 1.0 / 60.0
G = (0.0, -9.81, 0.0)
# kappa_arap x volume x h^2 well above the mass: near-rigid cubes
PARAMS = dict(h=H, gravity=G, d_hat=1e-2, kappa=1e4, kappa_arap=1e9, theta=1e-3, scene_scale=1.0)


def _ground():
    v, t, e = api.cube_mesh((2.0, 0.1, 2.0))
    return (v, t, e, (0.0, -0.1, 0.0), True)


def _cube(centre, half=0.1):
    v, t, e = api.cube_mesh(half)
    return (v, t, e, centre, False)


def test_free_fall_is_the_predicted_position():
    """One body, nothing within d_hat: E = 1/2 (q - q~)^T M (q - q~) +
    h^2 w ||A^T A - I||^2 is minimised by q = q~ (A stays I). Newton solves
    (H + eps I) dq = -g with the eps = 1e-8 tr(H)/n of newton.cpp:20-24, so the
    first step stops ~eps/m short of q~; with a Newton tolerance below that
    residual the second step closes it. q_dot = (q - q0) / h."""
    qd0 = np.zeros((1, 12))
    qd0[0, :3] = (0.3, 0.5, -0.2)
    params = dict(PARAMS, theta=1e-9)
    sim = api.Sim3D([_cube((0.0, 1.0, 0.0))], qd0=qd0, pcg_rel_tol=1e-14, **params)
    q0, _ = sim.state()
    st = sim.run(1)[0]
    q, qd = sim.state()
    qt = q0.copy()
    qt[0, :3] += H * qd0[0, :3] + H * H * np.array(G)
    assert st["converged"] and st["newton_iterations"] <= 4, st
    assert np.abs(q - qt).max() < 5e-12  # (eps/m)^2 of the step
    assert np.abs(qd - (q - q0) / H).max() < 1e-9


def _assemble_numpy(sim, bodies):
    """The Newton system of the next frame's first iteration from the per-term
    kernels (dabd_gpu_body3d_terms, dabd_gpu_broad_phase3d, dabd_gpu_contact3d_terms),
    summed on the host."""
    q, qd = sim.state()
    n = len(bodies)
    stat = np.array([b[4] for b in bodies])
    qt = q.copy()
    qt[~stat] += H * qd[~stat]
    qt[~stat, :3] += H * H * np.array(G)
    moms, vols = [], []
    for v, t, e, _, _ in bodies:
        m, _, vl = api.body3d_moments(v, t, 1000.0)
        moms.append(m)
        vols.append(vl)
    bt = api.body3d_terms(q, qt, np.array(moms), PARAMS["kappa_arap"] * np.array(vols), H * H)
    meshes = [(b[0], b[1], b[2]) for b in bodies]
    cand = api.broad_phase3d(q, meshes, PARAMS["d_hat"])
    rows = [i for i in range(n) if not stat[i]]
    idx = {b: k for k, b in enumerate(rows)}
    N = 12 * len(rows)
    Hm, g = np.zeros((N, N)), np.zeros(N)
    for b in rows:
        s = slice(12 * idx[b], 12 * idx[b] + 12)
        Hm[s, s] += bt["hess"][b]
        g[s] += bt["grad"][b]
    if len(cand):
        kind, a, b, pa, pb = cand.T
        rest = np.zeros((len(cand), 4, 3))
        for k in range(len(cand)):
            va, ta, ea = meshes[a[k]][0], meshes[a[k]][1], meshes[a[k]][2]
            vb, tb, eb = meshes[b[k]][0], meshes[b[k]][1], meshes[b[k]][2]
            if kind[k] == 0:
                rest[k] = [va[pa[k]], *vb[tb[pb[k]]]]
            else:
                rest[k] = [*va[ea[pa[k]]], *vb[eb[pb[k]]]]
        ct = api.contact3d_terms(kind, q[a], q[b], rest, PARAMS["d_hat"], PARAMS["kappa"], weight=H * H)
        for k in range(len(cand)):
            for side, body in ((0, a[k]), (1, b[k])):
                if body in idx:
                    s = slice(12 * idx[body], 12 * idx[body] + 12)
                    g[s] += ct["grad"][k][12 * side:12 * side + 12]
            for sa, ba in ((0, a[k]), (1, b[k])):
                for sb, bb in ((0, a[k]), (1, b[k])):
                    if ba in idx and bb in idx:
                        Hm[12 * idx[ba]:12 * idx[ba] + 12, 12 * idx[bb]:12 * idx[bb] + 12] += \
                            ct["hess"][k][12 * sa:12 * sa + 12, 12 * sb:12 * sb + 12]
    Hm += 1e-8 * np.trace(Hm) / N * np.eye(N)
    return Hm, g, len(cand)


def test_assembled_system_and_direction():
    """A cube resting on the ground and a second one in contact with it: the
    device-assembled system equals the per-term kernels summed in numpy (to
    rounding), it is symmetric positive definite, and the PCG direction
    solves it."""
    bodies = [_ground(), _cube((0.0, 0.105, 0.0)), _cube((0.02, 0.312, 0.01))]
    sim = api.Sim3D(bodies, **PARAMS)
    Hd, gd, dq = sim.system()
    Hn, gn, ncand = _assemble_numpy(sim, bodies)
    assert ncand > 0
    scale = np.abs(Hn).max()
    assert np.abs(Hd - Hn).max() < 1e-12 * scale
    assert np.abs(gd - gn).max() < 1e-12 * max(np.abs(gn).max(), 1.0)
    assert np.abs(Hd - Hd.T).max() < 1e-12 * scale
    assert np.linalg.eigvalsh(Hd).min() > 0.0
    ref = np.linalg.solve(Hn, -gn)
    assert np.abs(dq - ref).max() < 1e-6 * np.abs(ref).max()


def _boxes_intersect(qa, qb, half):
    """Exact test for two cubes of the same half size as affine bodies: any
    vertex of one inside the other (A^-1 (x - p) within the half size), both
    ways, or overlapping centres."""
    v = np.array([[x, y, z] for x in (-half, half) for y in (-half, half) for z in (-half, half)])
    for a, b in ((qa, qb), (qb, qa)):
        Aa, Ab = a[3:].reshape(3, 3), b[3:].reshape(3, 3)
        xw = v @ Aa.T + a[:3]
        local = (xw - b[:3]) @ np.linalg.inv(Ab).T
        if np.any(np.all(np.abs(local) < half, axis=1)):
            return True
    return False


def test_dropped_cubes_penetration_free_and_rigid():
    """Three cubes dropped onto the ground with gaps (frictionless, so the
    stack may slide apart): every frame converges, the minimum distance over
    the pairs within d_hat stays positive, and at the end no two cubes
    intersect, every cube is above the ground, A^T A = I to 1e-2 (near-rigid)
    and the cubes have settled vertically."""
    half = 0.1
    bodies = [_ground(), _cube((0.0, 0.15, 0.0)), _cube((0.01, 0.40, -0.01)), _cube((-0.01, 0.65, 0.02))]
    sim = api.Sim3D(bodies, **PARAMS)
    dmins = []
    for f, st in enumerate(sim.run(120)):
        assert st["converged"], (f, st)
        if st["max_candidates"]:
            assert st["min_distance"] > 0.0, (f, st)
            dmins.append(st["min_distance"])
        if f % 20 == 19:
            q, _ = sim.state()
            for i in range(1, 4):
                for j in range(i + 1, 4):
                    assert not _boxes_intersect(q[i], q[j], half), (f, i, j)
    q, qd = sim.state()
    A = q[1:, 3:].reshape(-1, 3, 3)
    assert np.abs(np.einsum("bji,bjk->bik", A, A) - np.eye(3)).max() < 1e-2  # rotations allowed
    corners = np.array([[x, y, z] for x in (-half, half) for y in (-half, half) for z in (-half, half)])
    lowest = min((corners @ A[b].T + q[1 + b, :3])[:, 1].min() for b in range(3))
    assert lowest > 0.0  # above the ground's top face
    assert np.abs(qd[1:, 1]).max() < 0.05  # settled vertically (frictionless: they may still slide)
    assert len(dmins) > 0


def test_single_cube_comes_to_rest_on_the_ground():
    """A cube dropped flat onto the ground lands and rests within d_hat of it,
    unrotated (the contact is symmetric), at rest."""
    sim = api.Sim3D([_ground(), _cube((0.0, 0.16, 0.0))], **PARAMS)
    for st in sim.run(90):
        assert st["converged"]
    q, qd = sim.state()
    assert 0.1 < q[1, 1] < 0.1 + PARAMS["d_hat"]
    assert np.abs(q[1, 3:] - np.eye(3).reshape(-1)).max() < 1e-3
    assert np.abs(qd[1, :3]).max() < 1e-2
