"""Degenerate shapes of the multi-partition frame (runtime.cpp:110-694) on the
device path against the oracle: partitions with no bodies, a scene with no
dynamic body, a lone body that every worker holds (the consensus of identical
replicas), and zero frames. The reference's own empty-scene case is
test_gpu_solver.py::test_run_reference_empty_scene (test_runtime.cpp:326-333).
"""

import numpy as np
import pytest

import oracle as O
from support import scene_of, square
from paper_2605_15875_b200 import api
from paper_2605_15875_b200.scene import BodySpec, Plane, SceneData, SimParams, make_scenario

pytestmark = pytest.mark.gpu

TIGHT = dict(pcg_rel_tol=1e-12, pcg_max_iters=20000, inexact=(0.0, 10.0))


def _compare(sd, workers, frames, state_tol=1e-7):
    o = O.Scene(sd)
    ref = o.run(frames, workers=workers)
    gpu = api.run_distributed(sd, workers, frames, **TIGHT)
    for f in range(frames):
        assert gpu.h[f] == ref["h"][f], f
        assert gpu.stats[f]["attempts"] == ref["attempts"][f], f
        assert gpu.stats[f]["admm_iterations"] == ref["admm"][f], (f, gpu.stats[f], ref["admm"][f])
        scale = max(1.0, np.abs(ref["q"][f]).max()) if ref["q"][f].size else 1.0
        assert np.abs(gpu.q[f] - ref["q"][f]).max(initial=0.0) < state_tol * scale, f
    return gpu, ref


def test_empty_partitions():
    """drop-grid-1 split four ways by planes far to the right of every body:
    partitions 1-3 hold nothing, every frame equals the oracle's and the
    one-worker run's ADMM counts."""
    sd = make_scenario("drop-grid-1")
    sd.planes = [Plane((5.0 + k, 0.0), (-1.0, 0.0)) for k in range(3)]
    gpu, ref = _compare(sd, 4, 8)
    one = api.run_distributed(make_scenario("drop-grid-1"), 1, 8, **TIGHT)
    assert [s["admm_iterations"] for s in gpu.stats] == [s["admm_iterations"] for s in one.stats]
    assert np.abs(gpu.q - one.q).max() < 1e-9


def test_no_dynamic_body():
    """Only static geometry, two workers: frames complete, nothing moves."""
    p = SimParams(h=0.01, gravity=(0.0, -10.0), arap_stiffness=1e8, barrier_stiffness=1e4, d_hat=0.01,
                  theta=1e-3, scene_scale=2.0)
    floor = [(-2.0, -0.2), (2.0, -0.2), (2.0, 0.0), (-2.0, 0.0)]
    sd = scene_of([[floor], [square(0.2, (0.5, 0.5))]], density=1000.0, static=[True, True], params=p)
    sd.planes = [Plane((0.0, 0.0), (-1.0, 0.0))]
    gpu, ref = _compare(sd, 2, 3)
    assert np.array_equal(gpu.q[-1], gpu.q[0])
    assert all(s["committed"] for s in gpu.stats)


def test_lone_body_held_by_both_workers():
    """One square straddling the interface in free fall, no contacts: both
    workers hold a replica, the replicas agree, ADMM stops as the oracle's
    does and the state is the analytic free fall."""
    p = SimParams(h=0.01, gravity=(0.0, -10.0), arap_stiffness=1e8, barrier_stiffness=1e4, d_hat=0.01,
                  theta=1e-3, scene_scale=1.0)
    sd = scene_of([[square(0.1, (0.0, 1.0))]], density=1000.0, static=[False], params=p,
                  velocities=[(0.3, 0.0, 0, 0, 0, 0)])
    sd.planes = [Plane((0.0, 0.0), (-1.0, 0.0))]
    frames = 6
    gpu, ref = _compare(sd, 2, frames)
    vy = y = x = 0.0
    for f in range(frames):
        vy += p.h * -10.0
        x += p.h * 0.3
        y += p.h * vy
    tol = 0.1 * p.theta * p.h * p.scene_scale  # a tenth of the Newton tolerance theta h l
    assert abs(gpu.q[-1][0, 0] - x) < tol and abs(gpu.q[-1][0, 1] - (1.0 + y)) < tol
    shared = ~np.isnan(ref["rho"])
    assert np.array_equal(shared, ~np.isnan(gpu.rho))


def test_zero_frames():
    sd = make_scenario("drop-grid-4")
    ctx = api.Context(api.Scene(sd), num_workers=4)
    q0, qd0 = ctx.state()
    assert ctx.run_frames(0) == []
    q1, qd1 = ctx.state()
    assert np.array_equal(q0, q1) and np.array_equal(qd0, qd1)


def test_run_reference_no_dynamic_body():
    """The captured single-domain frame with zero solver rows: frames
    complete as the oracle's, nothing moves."""
    p = SimParams(h=0.01, gravity=(0.0, -10.0), arap_stiffness=1e8, barrier_stiffness=1e4, d_hat=0.01,
                  theta=1e-3, scene_scale=2.0)
    floor = [(-2.0, -0.2), (2.0, -0.2), (2.0, 0.0), (-2.0, 0.0)]
    sd = scene_of([[floor], [square(0.2, (0.5, 0.5))]], density=1000.0, static=[True, True], params=p)
    ref = O.Scene(sd).run(3, workers=0)
    t = api.run_reference(sd, 3, **TIGHT)
    assert [s["admm_iterations"] for s in t.stats] == list(ref["admm"])
    assert np.array_equal(t.q[-1], t.q[0])


@pytest.mark.parametrize("workers", [0, 2])
def test_fast_box_does_not_tunnel_through_a_thin_wall(workers):
    """A box fired at 20 m/s (0.2 per frame, ten wall thicknesses) at a thin
    static wall, no gravity: the CCD-capped line search (newton.cpp:38-42)
    stops it in front of the wall in the frame it would cross, then the
    barrier pushes it back — single-domain, and with the interface plane
    between box and wall (workers = 2). States and ADMM counts as the
    oracle's; the box's front face never reaches the wall."""
    p = SimParams(h=0.01, gravity=(0.0, 0.0), arap_stiffness=1e8, barrier_stiffness=1e4, d_hat=0.01,
                  theta=1e-3, scene_scale=2.0)
    wall = [(0.5, -0.5), (0.52, -0.5), (0.52, 0.5), (0.5, 0.5)]
    sd = scene_of([[square(0.05, (0.0, 0.0))], [wall]], density=1000.0, static=[False, True], params=p,
                  velocities=[(20.0, 0.0, 0, 0, 0, 0), (0,) * 6])
    frames = 8
    if workers:
        sd.planes = [Plane((0.3, 0.0), (-1.0, 0.0))]
        gpu, ref = _compare(sd, workers, frames, state_tol=1e-6)
        q = gpu.q
    else:
        ref = O.Scene(sd).run(frames, workers=0)
        t = api.run_reference(sd, frames, **TIGHT)
        assert [s["admm_iterations"] for s in t.stats] == list(ref["admm"])
        assert np.abs(t.q - ref["q"]).max() < 1e-6 * p.scene_scale
        q = t.q
    front = q[:, 0, 0] + 0.05  # the box stays axis-aligned (no torque)
    assert front.max() < 0.5
    assert front[2] > 0.5 - p.d_hat  # stopped within d_hat of the wall, not short of it
