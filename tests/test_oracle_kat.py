"""Pin the CPU oracle against the reference's own known-answer tests.

Each test cites the reference test it ports (proj/tests/*.cpp). These are the
golden values that pin the oracle; the GPU parity tests then
compare the CUDA path against this oracle.
"""

import math

import numpy as np
import pytest

import oracle as O
from support import (Rng, brute_force_active_pairs, default_params, random_convex_polygon,
                     scene_of, square)
from paper_2605_15875_b200.scene import (BodySpec, Plane, SceneData, SimParams,
                                         make_scenario)


# ---------------------------------------------------------------- body (test_body.cpp)

def test_unit_square_mass_matrix():  # test_body.cpp:18-36
    s = O.Scene(scene_of([[square(0.5)]]))
    assert s.mass[0] == pytest.approx(1.0, rel=1e-14)
    M = s.mass_matrix[0]
    assert M[0, 0] == pytest.approx(1.0)
    assert M[1, 1] == pytest.approx(1.0)
    assert M[2, 2] == pytest.approx(1.0 / 12.0)
    assert abs(M[0, 2]) < 1e-15
    assert np.allclose(M, M.T)
    assert np.linalg.eigvalsh(M).max() <= s.mass[0] + 1e-12


def test_lambda_max_bound_random_polygons():  # test_body.cpp:57-65
    rng = Rng(7)
    for trial in range(100):
        poly = random_convex_polygon(rng, 3, 12, 0.05, 1.0)
        dens = rng.uniform(0.1, 1e4)
        s = O.Scene(scene_of([[poly]], density=dens))
        assert np.linalg.eigvalsh(s.mass_matrix[0]).max() <= s.mass[0] * (1 + 1e-10)


def test_degenerate_polygon_rejected():  # test_body.cpp:67-77
    cw = list(reversed(square(0.5)))
    with pytest.raises(O.OracleError):
        O.Scene(scene_of([[cw]]))
    with pytest.raises(O.OracleError):
        O.Scene(scene_of([[[(0.0, 0.0), (1.0, 0.0), (2.0, 0.0)]]]))


def test_recentering():  # test_body.cpp:79-95
    sq = square(0.5, (3.0, -2.0))
    s = O.Scene(scene_of([[sq]], density=2.0))
    assert s.q0[0, 0] == pytest.approx(3.0)
    assert s.q0[0, 1] == pytest.approx(-2.0)
    q = s.q0[0]
    for v in range(4):
        xb = s.rest[v]
        w = ((q[2] * xb[0] + q[3] * xb[1]) + q[0], (q[4] * xb[0] + q[5] * xb[1]) + q[1])
        assert w == pytest.approx(sq[v])


def test_predicted_position():  # test_body.cpp:97-126
    s = O.Scene(scene_of([[square(0.5)]]))
    z = np.zeros((1, 6))
    assert np.allclose(s.predicted_position(s.q0, z, z, 0.01), s.q0)
    qd = z.copy()
    qd[0, 0] = 1.0
    qt = s.predicted_position(z, qd, z, 0.01)
    assert qt[0, 0] == pytest.approx(0.01)
    assert np.linalg.norm(qt[0, 1:]) == pytest.approx(0.0)
    f = z.copy()
    f[0, 1] = s.mass[0] * -10.0
    qt = s.predicted_position(z, z, f, 0.1)
    assert qt[0, 0] == pytest.approx(0.0)
    assert qt[0, 1] == pytest.approx(-0.1)
    assert np.linalg.norm(qt[0, 2:]) == pytest.approx(0.0, abs=1e-15)


def test_max_vertex_speed():  # test_body.cpp:128-138
    s = O.Scene(scene_of([[square(0.5)]]))
    qd = np.zeros((1, 6))
    qd[0, 0] = 3.0
    assert s.max_vertex_speed(qd)[0] == pytest.approx(3.0)
    qd[:] = 0
    qd[0, 2] = 1.0
    qd[0, 5] = 1.0
    assert s.max_vertex_speed(qd)[0] == pytest.approx(math.sqrt(0.5))


# ---------------------------------------------------------------- energy (test_energy.cpp)

def test_inertia_and_arap_known_values():  # test_energy.cpp:29-109
    v, _ = O.inertia_energy(np.ones(6), np.ones(6) - np.array([1.0, 0, 0, 0, 0, 0]), np.eye(6))
    assert v == pytest.approx(0.5)
    q = np.array([0, 0, 1.0, 0, 0, 1.0])
    assert O.arap_energy(q, 1.0, 1.0)[0] == pytest.approx(0.0)
    for ang in (0.3, 1.2, -2.5):
        qr = np.array([0, 0, math.cos(ang), -math.sin(ang), math.sin(ang), math.cos(ang)])
        assert O.arap_energy(qr, 1.0, 1.0)[0] == pytest.approx(0.0, abs=1e-14)
    assert O.arap_energy(np.array([0, 0, 2.0, 0, 0, 2.0]), 1.0, 1.0)[0] == pytest.approx(18.0)


def _fd_grad(f, x, step):
    g = np.zeros_like(x)
    for i in range(len(x)):
        def at(o):
            y = x.copy()
            y[i] += o
            return f(y)
        g[i] = (-at(2 * step) + 8 * at(step) - 8 * at(-step) + at(-2 * step)) / (12 * step)
    return g


def _rel(a, b):
    scale = max(np.abs(a).max(), np.abs(b).max(), 1e-12)
    return np.abs(a - b).max() / scale


def test_arap_fd():  # test_energy.cpp:93-108
    rng = Rng(4)
    for _ in range(50):
        qa = np.array([rng.uniform(-1.5, 1.5) for _ in range(6)])
        v, g, H = O.arap_energy(qa, 3.0, 0.4)
        assert _rel(_fd_grad(lambda x: O.arap_energy(x, 3.0, 0.4)[0], qa, 1e-5), g) < 1e-4
        Hfd = np.stack([_fd_grad(lambda x: O.arap_energy(x, 3.0, 0.4)[1][i], qa, 1e-5)
                        for i in range(6)])
        assert _rel(Hfd, H) < 1e-3


def test_barrier_known_values():  # test_energy.cpp:111-164
    assert O.barrier_energy(1.0, 1.0, 1.0)[0] == 0.0
    assert O.barrier_energy(0.5, 1.0, 1.0)[0] == pytest.approx(0.25 * math.log(2.0))
    prev = 0.0
    for d in (1e-2, 1e-4, 1e-8, 1e-16, 1e-32):
        v = O.barrier_energy(d, 1.0, 1.0)[0]
        assert v > prev
        prev = v
    assert prev > 70.0
    with pytest.raises(O.OracleError):
        O.barrier_energy(0.0, 1.0, 1.0)
    b = O.barrier_energy(1.0 - 1e-7, 1.0, 1.0)
    assert abs(b[0]) < 1e-8 and abs(b[1]) < 1e-6 and abs(b[2]) < 1e-5


def test_contact_energy_fd():  # test_energy.cpp:166-202
    rng = Rng(6)
    s = O.Scene(scene_of([[square(0.5)], [square(0.5)]]))
    checked = 0
    for trial in range(200):
        if checked >= 60:
            break
        q = s.q0.copy()
        q[0, 0] += rng.uniform(-0.2, 0.2)
        q[0, 1] += rng.uniform(0.9, 1.4)
        for i in range(2, 6):
            q[0, i] += rng.uniform(-0.05, 0.05)
            q[1, i] += rng.uniform(-0.05, 0.05)
        v, g, H = s.contact_energy(q, 0, 1, 0, 2, 0.8, 10.0)
        if v <= 0.0:
            continue
        checked += 1
        x = q.reshape(-1).copy()

        def f(y):
            return s.contact_energy(y.reshape(2, 6), 0, 1, 0, 2, 0.8, 10.0)[0]

        assert _rel(_fd_grad(f, x, 1e-6), g) < 1e-4
        Hfd = np.stack([_fd_grad(lambda y: s.contact_energy(y.reshape(2, 6), 0, 1, 0, 2, 0.8,
                                                            10.0)[1][i], x, 1e-6)
                        for i in range(12)])
        assert _rel(Hfd, H) < 1e-3
    assert checked >= 30


# ---------------------------------------------------------------- geometry (test_geometry.cpp)

def test_point_edge_distance_values():  # test_geometry.cpp:32-38
    assert O.point_edge_distance((0, 1), (-1, 0), (1, 0))[0] == pytest.approx(1.0)
    assert O.point_edge_distance((2, 1), (-1, 0), (1, 0))[0] == pytest.approx(math.sqrt(2))
    assert O.point_edge_distance((-3, 0), (-1, 0), (1, 0))[0] == pytest.approx(2.0)
    with pytest.raises(O.OracleError):
        O.point_edge_distance((0, 1), (-1, 0), (-1, 0))


def test_point_edge_distance_fd():  # test_geometry.cpp:40-66
    rng = Rng(11)
    for _ in range(200):
        x = np.array([rng.uniform(-1, 1) for _ in range(6)])
        p, e0, e1 = x[0:2], x[2:4], x[4:6]
        if np.linalg.norm(e1 - e0) < 0.3:
            continue
        d, g, H = O.point_edge_distance(p, e0, e1)
        if d < 1e-3:
            continue
        t = np.dot(p - e0, e1 - e0) / np.dot(e1 - e0, e1 - e0)
        if abs(t) < 1e-2 or abs(t - 1) < 1e-2:
            continue
        f = lambda y: O.point_edge_distance(y[0:2], y[2:4], y[4:6], False)[0]
        assert _rel(_fd_grad(f, x, 1e-6), g) < 1e-5
        Hfd = np.stack([_fd_grad(lambda y: O.point_edge_distance(y[0:2], y[2:4], y[4:6])[1][i],
                                 x, 1e-5) for i in range(6)])
        assert _rel(Hfd, H) < 1e-3


def test_broad_phase_basic():  # test_geometry.cpp:80-98
    s = O.Scene(scene_of([[square(0.5)], [square(0.5, (10, 0))]]))
    assert len(s.broad_phase(s.q0, 0.1)) == 0
    s = O.Scene(scene_of([[square(0.5)], [square(0.5, (0.6, 0.1))]]))
    cand = s.broad_phase(s.q0, 0.1)
    act, _ = brute_force_active_pairs(s, s.q0, 0.1)
    cset = {tuple(r) for r in cand}
    assert all(tuple(r) in cset for r in act)
    assert [tuple(r) for r in cand] == sorted(tuple(r) for r in cand)


def random_scene(rng, nb_lo=2, nb_hi=16, vmin=3, vmax=8, rmin=0.1, rmax=0.4, span=2.0):
    nb = rng.uniform_int(nb_lo, nb_hi)
    loops = []
    for _ in range(nb):
        poly = random_convex_polygon(rng, vmin, vmax, rmin, rmax)
        cx, cy = rng.uniform(-span, span), rng.uniform(-span, span)
        loops.append([[(x + cx, y + cy) for (x, y) in poly]])
    return scene_of(loops)


def test_narrow_equals_brute_force_100_scenes():  # test_geometry.cpp:100-123
    rng = Rng(13)
    for _ in range(100):
        sd = random_scene(rng)
        s = O.Scene(sd)
        d_hat = rng.uniform(0.02, 0.2)
        got, gd = s.narrow_phase(s.q0, s.broad_phase(s.q0, d_hat), d_hat)
        exp, ed = brute_force_active_pairs(s, s.q0, d_hat)
        assert np.array_equal(got, exp)
        assert np.allclose(gd, ed, rtol=1e-12, atol=0)


def test_narrow_trivial():  # test_geometry.cpp:125-133
    s = O.Scene(scene_of([[square(0.5)], [square(0.5, (0, 1.05))]]))
    pairs, d = s.narrow_phase(s.q0, s.broad_phase(s.q0, 0.1), 0.1)
    assert len(pairs) > 0
    assert np.allclose(d, 0.05)


def test_ccd_analytic():  # test_geometry.cpp:135-151
    tri = [(0.0, 1.0), (0.1, 1.2), (-0.1, 1.2)]
    bar = [(-1.0, -0.05), (1.0, -0.05), (1.0, 0.0), (-1.0, 0.0)]
    s = O.Scene(scene_of([[tri], [bar]], static=[False, True]))
    end = s.q0.copy()
    end[0, 1] -= 2.0
    assert s.ccd_toi(s.q0, end) == pytest.approx(0.45, rel=1e-9)


def test_ccd_trivial():  # test_geometry.cpp:153-173
    s = O.Scene(scene_of([[square(0.5)], [square(0.5, (2, 0))]]))
    assert s.ccd_toi(s.q0, s.q0) == 1.0
    end = s.q0.copy()
    end[1, 0] += 5.0
    assert s.ccd_toi(s.q0, end) == 1.0
    t = O.Scene(scene_of([[square(0.5)], [square(0.5, (1.0, 0))]]))
    end = t.q0.copy()
    end[1, 0] -= 0.5
    with pytest.raises(O.OracleError):
        t.ccd_toi(t.q0, end)


def test_intersection_cases():  # test_geometry.cpp:217-245
    assert not O.Scene(scene_of([[square(0.5)], [square(0.5, (2, 0))]])).intersection_test(
        O.Scene(scene_of([[square(0.5)], [square(0.5, (2, 0))]])).q0)
    s = O.Scene(scene_of([[square(0.5)], [square(0.5)]]))
    assert s.intersection_test(s.q0)
    s = O.Scene(scene_of([[square(0.5)], [square(0.5, (0.6, 0.3))]]))
    assert s.intersection_test(s.q0)
    s = O.Scene(scene_of([[square(0.5)], [square(0.5, (1.0, 0))]]))
    assert not s.intersection_test(s.q0)
    hbar = [(-2, -0.1), (2, -0.1), (2, 0.1), (-2, 0.1)]
    vbar = [(-0.1, -2), (0.1, -2), (0.1, 2), (-0.1, 2)]
    s = O.Scene(scene_of([[hbar], [vbar]]))
    assert s.intersection_test(s.q0)


def test_min_pair_distance():  # tests/support/oracles.cpp:153-173
    s = O.Scene(scene_of([[square(0.5)], [square(0.5, (1.5, 0))]]))
    assert s.min_pair_distance(s.q0) == 0.5
    s = O.Scene(scene_of([[square(0.5)], [square(0.5, (1.5, 1.5))]]))
    assert abs(s.min_pair_distance(s.q0) - np.sqrt(0.5)) < 1e-15  # corner to corner
    # two touching statics are skipped unless asked for
    s = O.Scene(scene_of([[square(0.5)], [square(0.5, (1.0, 0))], [square(0.5, (0, 3))]],
                         static=[True, True, False]))
    assert s.min_pair_distance(s.q0, skip_static_pairs=False) == 0.0
    assert s.min_pair_distance(s.q0) == 2.0


# ---------------------------------------------------------------- partition (test_partition.cpp)

MID = np.array([[0.0, 0.0, -1.0, 0.0]])


def test_membership():  # test_partition.cpp:32-58
    s = O.Scene(scene_of([[square(0.2)], [square(0.2, (-2, 0))], [square(0.2, (2, 0))],
                          [square(3.0, (0, 1))]], static=[False, False, False, True]))
    m = s.holder_masks(s.q0, MID, 0.4)
    assert list(m) == [3, 1, 2, 3]


def test_three_worker_chain_and_straddle():  # test_partition.cpp:84-105
    planes = np.array([[-1.0, 0, -1, 0], [1.0, 0, -1, 0]])
    s = O.Scene(scene_of([[square(0.2, (-2, 0))], [square(0.2)], [square(0.2, (2, 0))],
                          [square(0.2, (1, 0))]]))
    assert list(s.holder_masks(s.q0, planes, 0.3)) == [1, 2, 4, 6]
    g = O.Scene(scene_of([[square(1.0)]]))
    with pytest.raises(O.OracleError):
        g.holder_masks(g.q0, np.array([[-0.5, 0, -1, 0], [0.5, 0, -1, 0]]), 0.2)


# ---------------------------------------------------------------- solver (test_solver.cpp)

def _single_domain(s, params):
    n = s.n
    local = list(range(n))
    f = np.zeros((n, 6))
    for b in range(n):
        if not s.is_static[b]:
            f[b, 0] = s.mass[b] * params.gravity[0]
            f[b, 1] = s.mass[b] * params.gravity[1]
    qt = s.predicted_position(s.q0, s.qdot0, f, params.h)
    return local, np.ones(n), qt


def test_newton_one_iteration():  # test_solver.cpp:142-155
    p = default_params(gravity=(0.0, 0.0))
    s = O.Scene(scene_of([[square(0.25)]], density=1000.0, params=p))
    local, kap, qt = _single_domain(s, p)
    q, rep = s.newton_solve(s.q0, local, kap, qt, p.as_array(), 32, 1e-10)
    assert rep["iterations"] == 1 and rep["converged"] and rep["final_update_inf"] < 1e-10


def test_floor_barrier_equilibrium():  # test_solver.cpp:157-202
    p = default_params(arap_stiffness=1e10)
    half, clear0 = 0.25, 0.005
    floor = [(-3.0, -0.2), (3.0, -0.2), (3.0, 0.0), (-3.0, 0.0)]
    s = O.Scene(scene_of([[square(half, (0.0, half + clear0))], [floor]], density=1000.0,
                         static=[False, True], params=p))
    local, kap, qt = _single_domain(s, p)
    q, _ = s.newton_solve(s.q0, local, kap, qt, p.as_array(), 200, 1e-12)
    m = s.mass[0]
    ytilde = s.q0[0, 1] + p.h * p.h * p.gravity[1]

    def residual(c):
        return m * (half + c - ytilde) + p.h * p.h * 2.0 * O.barrier_energy(c, p.d_hat, 1e4)[1]

    lo, hi = 1e-9, p.d_hat - 1e-12
    assert residual(lo) < 0 < residual(hi)
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if residual(mid) < 0:
            lo = mid
        else:
            hi = mid
    c_star = 0.5 * (lo + hi)
    clearance = q[0, 1] - half * q[0, 5]
    assert clearance > 0
    assert q[0, 1] == pytest.approx(half + c_star, rel=1e-6)


def test_dominant_anchor():  # test_solver.cpp:204-225
    p = default_params()
    s = O.Scene(scene_of([[square(0.25)]], density=1000.0, params=p))
    rng = Rng(21)
    z = s.q0[0] + np.array([rng.uniform(-0.05, 0.05) for _ in range(6)])
    u = np.array([rng.uniform(-0.02, 0.02) for _ in range(6)])
    local, kap, qt = _single_domain(s, p)
    q, _ = s.newton_solve(s.q0, local, kap, qt, p.as_array(), 100, 1e-12,
                          anchors=[(0, z, u, 1e6 * s.mass[0])])
    target = z - u
    assert np.linalg.norm(q[0] - target) / np.linalg.norm(target) < 1e-3


def test_monotone_feasible():  # test_solver.cpp:227-252
    p = default_params(d_hat=0.02)
    floor = [(-2.0, -0.2), (2.0, -0.2), (2.0, 0.0), (-2.0, 0.0)]
    vel = [(0, -3.0, 0, 0, 0, 0), (0,) * 6, (0,) * 6]
    s = O.Scene(scene_of([[square(0.2, (0.02, 0.85))], [square(0.2, (0.0, 0.21))], [floor]],
                         density=1000.0, static=[False, False, True], params=p,
                         velocities=vel))
    local, kap, qt = _single_domain(s, p)
    q = s.q0.copy()
    prev = s.objective(q, local, kap, qt, p.as_array())["value"]
    for _ in range(40):
        q, rep = s.newton_solve(q, local, kap, qt, p.as_array(), 1, 1e-9)
        now = s.objective(q, local, kap, qt, p.as_array())["value"]
        assert now <= prev + 1e-12
        assert not s.intersection_test(q)
        prev = now
        if rep["converged"]:
            break


def test_replicated_objective_sum():  # test_consensus.cpp:263-335
    p = SimParams(h=0.01, gravity=(0.0, -10.0), arap_stiffness=1e8, barrier_stiffness=1e4,
                  d_hat=0.05)
    loops = [[square(0.25, (-1.25 + 0.51 * i, 0.26))] for i in range(6)]
    loops.append([square(3.0, (0.0, -0.25))])
    s = O.Scene(scene_of(loops, density=[1000.0] * 6 + [1.0], static=[False] * 6 + [True],
                         params=p))
    masks = s.holder_masks(s.q0, MID, 0.4)
    assert any(bin(int(m)).count("1") == 2 for m in masks[:6])
    local_all, kap1, qt = _single_domain(s, p)
    rng = Rng(41)
    qe = s.q0.copy()
    for i in range(6):
        qe[i, 0] += rng.uniform(-0.005, 0.005)
        qe[i, 1] += rng.uniform(-0.005, 0.005)
        qe[i, 3] += rng.uniform(-0.002, 0.002)
    total = 0.0
    for w in range(2):
        loc = [b for b in range(s.n) if masks[b] & (1 << w)]
        kap = [bin(int(masks[b])).count("1") for b in loc]
        total += s.objective(qe, loc, kap, qt[loc], p.as_array(), holder_mask=masks,
                             mode=1)["value"]
    ref = s.objective(qe, local_all, kap1, qt, p.as_array(), mode=1)
    assert ref["active"] > 0
    assert total == pytest.approx(ref["value"], rel=1e-12)


# ---------------------------------------------------------------- runtime (test_runtime.cpp)

def test_free_fall_closed_form():  # test_runtime.cpp:256-280
    sd = SceneData(name="free-fall", frames=10)
    sd.params = SimParams(h=0.0025, gravity=(0.0, -10.0), arap_stiffness=1.0, scene_scale=1.0)
    sd.bodies.append(BodySpec(loops=[square(0.1)], density=1000.0,
                              velocity=(0.1, 0, 0, 0, 0, 0)))
    t = O.Scene(sd).run(10)
    x, y, vy = 0.0, 0.0, 0.0
    vx = 0.1
    for f in range(10):
        vy += 0.0025 * -10.0
        x += 0.0025 * vx
        y += 0.0025 * vy
        assert abs(t["q"][f, 0, 0] - x) < 1e-10
        assert abs(t["q"][f, 0, 1] - y) < 1e-10
        assert abs(t["qdot"][f, 0, 1] - vy) < 1e-8


def test_rest_equilibrium():  # test_runtime.cpp:282-324
    sd = SceneData(name="rest", frames=50)
    sd.params = SimParams(h=0.01, gravity=(0.0, -10.0), arap_stiffness=1e10,
                          barrier_stiffness=1e4, d_hat=0.01, scene_scale=1.0)
    sd.bodies.append(BodySpec(loops=[square(0.2, (0.0, 0.208))], density=1000.0))
    sd.bodies.append(BodySpec(loops=[[(-2.0, -0.3), (2.0, -0.3), (2.0, 0.0), (-2.0, 0.0)]],
                              density=1000.0, is_static=True))
    s = O.Scene(sd)
    t = s.run(50)
    q = t["q"][-1, 0]
    clearance = q[1] - 0.2 * q[5]
    assert clearance > 0
    assert abs(t["qdot"][-1, 0, 1]) < 1e-6
    assert np.abs(t["q"][49, 0] - t["q"][48, 0]).max() < 1e-6
    m = s.mass[0]
    h = 0.01

    def residual(c):
        return -m * h * h * -10.0 + h * h * 2.0 * O.barrier_energy(c, 0.01, 1e4)[1]

    lo, hi = 1e-9, 0.01 - 1e-12
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if residual(mid) < 0:
            lo = mid
        else:
            hi = mid
    # The reference asserts 1e-3 relative (test_runtime.cpp:323); the fixed point
    # the stepping stalls at is only defined to the Newton resolution
    # theta*h*l = 1e-5 (newton.cpp:30-36), and which point in that band is hit
    # depends on Eigen's rounding, so the restatement is held to that band.
    assert abs(clearance - 0.5 * (lo + hi)) < 1e-3 * 0.01 * 1.0


def test_empty_scene():  # test_runtime.cpp:326-333
    sd = SceneData(name="empty", frames=3)
    s = O.Scene(sd)
    t = s.run(3)
    assert t["q"].shape == (3, 0, 6)


def test_one_worker_equals_reference():  # test_runtime.cpp:33-46 (bitwise)
    sd = make_scenario("funnel-analog")
    s = O.Scene(sd)
    a = s.run(3, workers=0)
    b = s.run(3, workers=1)
    assert np.array_equal(a["q"], b["q"]) and np.array_equal(a["qdot"], b["qdot"])


def test_two_worker_mse_and_blocked_merge():  # test_runtime.cpp:98-115, 146-159
    sd = make_scenario("funnel-analog")
    s = O.Scene(sd)
    ref = s.run(4, workers=0)
    two = s.run(4, workers=2)
    l2 = sd.params.scene_scale ** 2
    dyn = ~s.is_static
    for f in range(4):
        mse = np.mean((two["q"][f][dyn] - ref["q"][f][dyn]) ** 2)
        assert mse < 1e-4 * l2
    assert (two["admm"] >= 2).all()
    bm = O.Scene(make_scenario("blocked-merge"))
    t = bm.run(3, workers=2)
    assert t["attempts"][0] >= 2
    assert t["h"][0] < 0.02
    for f in range(3):
        assert not bm.intersection_test(t["q"][f])


# ---------------------------------------------------------------- consensus (test_consensus.cpp)

ADAPT6 = [1.0, 2.0, 5.0, 1e-3, 1e3, 1.0]  # params.hpp:26-41 defaults


def test_consensus_update_closed_form():  # test_consensus.cpp:30-50
    a, b = np.zeros(6), np.full(6, 4.0)
    assert O.consensus_update([a, b], [2.0, 2.0])[0] == pytest.approx(2.0)
    assert np.allclose(O.consensus_update([a, b], [1.0, 3.0]), 3.0)
    r = np.random.default_rng(31).uniform(-2, 2, 6)
    assert np.abs(O.consensus_update([r], [7.5]) - r).max() == pytest.approx(0.0, abs=1e-15)
    with pytest.raises(O.OracleError):
        O.consensus_update(np.zeros((0, 6)), [])
    with pytest.raises(O.OracleError):
        O.consensus_update([np.zeros(6)], [0.0])


def test_stopping_rule():  # test_consensus.cpp:131-161
    h, l, th = 0.01, 2.0, 1e-3
    assert O.check_stopping(0, 0, 0, [1.0, 1.0], h, l, th)
    assert not O.check_stopping(0, 0, 0, [1.0, 0.7], h, l, th)
    at = th * h * l
    assert not O.check_stopping(0, at, 0, [1.0], h, l, th)
    assert O.check_stopping(0, np.nextafter(at, 0.0), 0, [1.0], h, l, th)
    rng = np.random.default_rng(39)
    for _ in range(200):
        dq, r, s = rng.uniform(0, 2 * at, 3)
        if not O.check_stopping(dq, r, s, [1.0], h, l, th):
            continue
        for m in range(3):
            v = [dq, r, s]
            v[m] *= rng.uniform()
            assert O.check_stopping(*v, [1.0], h, l, th)


def test_penalty_policy():  # test_consensus.cpp:163-187
    assert O.init_rho(100.0, 1.0) == pytest.approx(100.0)
    assert O.init_rho(100.0, 0.01) == pytest.approx(1.0)
    prev = None
    for beta in (0.01, 0.1, 1.0, 10.0, 100.0):
        rho = O.init_rho(50.0, beta)
        if prev:
            assert rho / prev == pytest.approx(10.0)
        prev = rho
    with pytest.raises(O.OracleError):
        O.init_rho(0.0, 1.0)
    assert O.adapt_rho(1.0, 10.0, 1.0, ADAPT6, 1.0) == pytest.approx(2.0)
    assert O.adapt_rho(1.0, 1.0, 10.0, ADAPT6, 1.0) == pytest.approx(0.5)
    assert O.adapt_rho(1.0, 3.0, 3.0, ADAPT6, 1.0) == pytest.approx(1.0)
    top, bottom = ADAPT6[4], ADAPT6[3]
    assert O.adapt_rho(top, 100.0, 0.001, ADAPT6, 1.0) == pytest.approx(top)
    assert O.adapt_rho(bottom, 0.001, 100.0, ADAPT6, 1.0) == pytest.approx(bottom)


def test_adaptive_timestep_controller():  # test_consensus.cpp:246-261
    h = O.timestep_apply(0.02, 4, [0, 0, 1, 1, 1])
    assert list(h) == pytest.approx([0.01, 0.005, 0.01, 0.02, 0.02])
    assert O.timestep_apply(0.02, 4, [0, 0, 0, 0])[-1] == pytest.approx(0.02 / 16)
    with pytest.raises(O.OracleError):
        O.timestep_apply(0.02, 4, [0, 0, 0, 0, 0])


def test_contact_replication_counts():  # test_partition.cpp:107-123
    s = O.Scene(scene_of([[square(0.2, (-2.0, 0.0))], [square(0.2, (-1.8, 0.5))], [square(0.2)],
                          [square(0.2, (0.05, 0.5))], [square(0.2, (2.0, 0.0))]], density=1000.0))
    m = s.holder_masks(s.q0, MID, 0.4)
    assert list(m) == [1, 1, 3, 3, 2]
    assert O.contact_replication(m[0], m[1]) == 1  # both internal to worker 0
    assert O.contact_replication(m[2], m[3]) == 2  # both shared
    assert O.contact_replication(m[0], m[2]) == 1  # internal vs shared
    assert O.contact_replication(m[2], m[4]) == 1  # shared vs internal(1)
    with pytest.raises(O.OracleError):
        O.contact_replication(m[0], m[4])  # disjoint holders
