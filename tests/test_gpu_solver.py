"""Parity of the sm_100a local solve with the CPU oracle.

Continuous quantities match within stated FP64 tolerances: the GPU uses a
block-Jacobi PCG (relative residual 1e-12 here) where the reference uses a
direct LDLT, a rank-6 closed-form projection of the 12x12 contact blocks,
and tree-ordered sums.
"""

import numpy as np
import pytest

import oracle as O
from support import Rng, default_params, scene_of, square
from paper_2605_15875_b200 import api
from paper_2605_15875_b200.scene import BodySpec, SceneData, SimParams, make_scenario

pytestmark = pytest.mark.gpu

# the oracle-parity settings emulate the reference's exact solves: PCG to
# 1e-12 and every Newton direction to it (inexact Newton off)
TIGHT = dict(pcg_rel_tol=1e-12, pcg_max_iters=20000, inexact=(0.0, 10.0))


def _single(o, p):
    n = o.n
    f = np.zeros((n, 6))
    for b in range(n):
        if not o.is_static[b]:
            f[b, 0] = o.mass[b] * p.gravity[0]
            f[b, 1] = o.mass[b] * p.gravity[1]
    return list(range(n)), np.ones(n), o.predicted_position(o.q0, o.qdot0, f, p.h)


def _rel(a, b):
    s = max(np.abs(a).max(initial=0.0), np.abs(b).max(initial=0.0), 1e-300)
    return np.abs(a - b).max(initial=0.0) / s


def _pile_state(name, rng_seed=3, frames=0):
    sd = make_scenario(name)
    o = O.Scene(sd)
    q = o.q0.copy()
    rng = Rng(rng_seed)
    # settle bodies toward contact: shift everything down a bit
    return sd, o, q


def test_objective_value_grad_hess_with_contacts():
    p = default_params(d_hat=0.05)
    sd = scene_of([[square(0.25, (0.0, 0.52))], [square(0.25, (0.1, 0.0))]], density=1000.0,
                  static=[False, True], params=p)
    o = O.Scene(sd)
    ctx = api.Context(api.Scene(sd), **TIGHT)
    local, kap, qt = _single(o, p)
    anchors = [(0, o.q0[0] + np.array([0.01, 0, 0, 0, 0, 0]), np.array([0, 0.002, 0, 0, 0, 0]), 50.0)]
    for mode in (0, 1, 2, 3):
        g = ctx.objective(o.q0, local, kap, qt, p, anchors=anchors, mode=mode)
        e = o.objective(o.q0, local, kap, qt, p.as_array(), anchors=anchors, mode=mode)
        assert g["active"] == e["active"] > 0
        assert g["candidates"] == e["candidates"]
        assert g["value"] == pytest.approx(e["value"], rel=1e-12)
        if mode >= 2:
            assert _rel(g["grad"], e["grad"]) < 1e-12
            assert _rel(g["hess"], e["hess"]) < 1e-10


def test_objective_pile_projected_hessian():
    sd = make_scenario("drop-grid-4")
    o = O.Scene(sd)
    ctx = api.Context(api.Scene(sd), **TIGHT)
    p = sd.params
    local, kap, qt = _single(o, p)
    # bring every box down onto its neighbour to create many active contacts
    q = o.q0.copy()
    rng = Rng(9)
    for b in range(o.n):
        if not o.is_static[b]:
            q[b, 1] -= 0.0
            q[b, 2] += rng.uniform(-1e-3, 1e-3)
    for mode in (2, 3):
        g = ctx.objective(q, local, kap, qt, p, mode=mode)
        e = o.objective(q, local, kap, qt, p.as_array(), mode=mode)
        assert g["active"] == e["active"]
        assert g["value"] == pytest.approx(e["value"], rel=1e-12)
        assert _rel(g["grad"], e["grad"]) < 1e-12
        assert _rel(g["hess"], e["hess"]) < 1e-10


def test_newton_one_iteration():  # test_solver.cpp:142-155
    p = default_params(gravity=(0.0, 0.0))
    sd = scene_of([[square(0.25)]], density=1000.0, params=p)
    o = O.Scene(sd)
    ctx = api.Context(api.Scene(sd), **TIGHT)
    local, kap, qt = _single(o, p)
    q, rep = ctx.newton_solve(o.q0, local, kap, qt, p, 32, 1e-10)
    assert rep["iterations"] == 1 and rep["converged"] and rep["final_update_inf"] < 1e-10


def test_newton_floor_equilibrium_matches_oracle():  # test_solver.cpp:157-202
    p = default_params(arap_stiffness=1e10)
    half, clear0 = 0.25, 0.005
    floor = [(-3.0, -0.2), (3.0, -0.2), (3.0, 0.0), (-3.0, 0.0)]
    sd = scene_of([[square(half, (0.0, half + clear0))], [floor]], density=1000.0,
                  static=[False, True], params=p)
    o = O.Scene(sd)
    ctx = api.Context(api.Scene(sd), **TIGHT)
    local, kap, qt = _single(o, p)
    qg, rg = ctx.newton_solve(o.q0, local, kap, qt, p, 200, 1e-12)
    qo, ro = o.newton_solve(o.q0, local, kap, qt, p.as_array(), 200, 1e-12)
    assert abs(qg[0, 1] - qo[0, 1]) < 1e-9
    assert _rel(qg, qo) < 1e-8


def test_newton_dominant_anchor():  # test_solver.cpp:204-225
    p = default_params()
    sd = scene_of([[square(0.25)]], density=1000.0, params=p)
    o = O.Scene(sd)
    ctx = api.Context(api.Scene(sd), **TIGHT)
    rng = Rng(21)
    z = o.q0[0] + np.array([rng.uniform(-0.05, 0.05) for _ in range(6)])
    u = np.array([rng.uniform(-0.02, 0.02) for _ in range(6)])
    local, kap, qt = _single(o, p)
    q, _ = ctx.newton_solve(o.q0, local, kap, qt, p, 100, 1e-12,
                            anchors=[(0, z, u, 1e6 * o.mass[0])])
    assert np.linalg.norm(q[0] - (z - u)) / np.linalg.norm(z - u) < 1e-3


def test_newton_stack_matches_oracle():  # test_solver.cpp:227-252 scene
    p = default_params(d_hat=0.02)
    floor = [(-2.0, -0.2), (2.0, -0.2), (2.0, 0.0), (-2.0, 0.0)]
    vel = [(0, -3.0, 0, 0, 0, 0), (0,) * 6, (0,) * 6]
    sd = scene_of([[square(0.2, (0.02, 0.85))], [square(0.2, (0.0, 0.21))], [floor]],
                  density=1000.0, static=[False, False, True], params=p, velocities=vel)
    o = O.Scene(sd)
    ctx = api.Context(api.Scene(sd), **TIGHT)
    local, kap, qt = _single(o, p)
    qg, rg = ctx.newton_solve(o.q0, local, kap, qt, p, 32, 1e-9)
    qo, ro = o.newton_solve(o.q0, local, kap, qt, p.as_array(), 32, 1e-9)
    assert rg["iterations"] == ro["iterations"]
    assert _rel(qg, qo) < 1e-7
    assert not o.intersection_test(qg)


def test_run_reference_free_fall():  # test_runtime.cpp:256-280
    sd = SceneData(name="free-fall", frames=10)
    sd.params = SimParams(h=0.0025, gravity=(0.0, -10.0), arap_stiffness=1.0, scene_scale=1.0)
    sd.bodies.append(BodySpec(loops=[square(0.1)], density=1000.0, velocity=(0.1, 0, 0, 0, 0, 0)))
    t = api.run_reference(sd, 10, **TIGHT)
    x = y = vy = 0.0
    for f in range(10):
        vy += 0.0025 * -10.0
        x += 0.0025 * 0.1
        y += 0.0025 * vy
        assert abs(t.q[f, 0, 0] - x) < 1e-10
        assert abs(t.q[f, 0, 1] - y) < 1e-10
        assert abs(t.q_dot[f, 0, 1] - vy) < 1e-8


def test_run_reference_empty_scene():  # test_runtime.cpp:326-333
    t = api.run_reference(SceneData(name="empty", frames=3), 3)
    assert t.q.shape == (3, 0, 6)


@pytest.mark.parametrize("name,frames", [("funnel-analog", 5), ("drop-grid-1", 5)])
def test_run_reference_matches_oracle(name, frames):
    sd = make_scenario(name)
    o = O.Scene(sd)
    ref = o.run(frames, workers=0)
    gpu = api.run_reference(sd, frames, **TIGHT)
    l2 = sd.params.scene_scale ** 2
    dyn = ~o.is_static
    for f in range(frames):
        mse = np.mean((gpu.q[f][dyn] - ref["q"][f][dyn]) ** 2)
        assert mse < 1e-10 * l2, (f, mse)
    assert [s["admm_iterations"] for s in gpu.stats] == list(ref["admm"])


def test_graph_frame_equals_eager_frame(monkeypatch):
    """The captured conditional-graph frame replays exactly the eager frame."""
    sd = make_scenario("drop-grid-1")
    monkeypatch.setenv("DABD_GPU_NO_GRAPH", "1")
    eager = api.run_reference(sd, 6, **TIGHT)
    monkeypatch.setenv("DABD_GPU_NO_GRAPH", "0")
    graph = api.run_reference(sd, 6, **TIGHT)
    assert np.array_equal(eager.q, graph.q) and np.array_equal(eager.q_dot, graph.q_dot)
    assert [s["admm_iterations"] for s in eager.stats] == [s["admm_iterations"] for s in graph.stats]
    assert [s["newton_iterations"] for s in eager.stats] == [s["newton_iterations"] for s in graph.stats]


def test_bench_settings_match_oracle_on_a_pile():
    """The bench's solver settings (PCG to 1e-10, warm-started; the defaults)
    on a contact-rich pile: 100 boxes of the pile-1k recipe dropped into the
    container, 40 frames of run_reference. States match the oracle to the
    north star's 1e-6 relative tolerance (on scene scale l), the per-frame
    ADMM k-counts exactly, and the final state is penetration-free."""
    from paper_2605_15875_b200.scene import lattice_pile

    sd = lattice_pile("pile-100", rows=10, cols_per_slab=10, slabs=1, half=0.05, spacing=0.13,
                      jitter=0.005, seed=11, l=6.0)
    frames = 40
    o = O.Scene(sd)
    ref = o.run(frames, workers=0)
    gpu = api.run_reference(sd, frames)
    dyn = ~o.is_static
    l = sd.params.scene_scale
    err = max(float(np.abs(gpu.q[f][dyn] - ref["q"][f][dyn]).max()) for f in range(frames))
    assert err < 1e-6 * l, err
    assert [s["admm_iterations"] for s in gpu.stats] == list(ref["admm"])
    assert max(s["max_contacts"] for s in gpu.stats) > 100  # contact-rich
    ctx = api.Context(api.Scene(sd))
    hit, _, dmin = ctx.audit(gpu.q[-1], cutoff=sd.params.d_hat)
    assert not hit and dmin > 0.0
