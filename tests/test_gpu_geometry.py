"""Bit-exact parity of the sm_100a collision kernels with the CPU oracle.

North-star contract: candidate pair lists, partition masks and CCD
accept/reject decisions are bit-exact on identical inputs.
"""

import numpy as np
import pytest

import oracle as O
from support import Rng, random_convex_polygon, scene_of, square
from test_oracle_kat import random_scene
from paper_2605_15875_b200 import api
from paper_2605_15875_b200._lib import DabdGpuError
from paper_2605_15875_b200.scene import make_scenario

pytestmark = pytest.mark.gpu


def _pair(sd):
    g = api.Scene(sd)
    return api.Context(g), O.Scene(sd)


def _perturb(q, rng, scale, static):
    q = q.copy()
    for b in range(len(q)):
        if static[b]:
            continue
        for k in range(6):
            q[b, k] += rng.uniform(-scale, scale) * (1.0 if k < 2 else 0.2)
    return q


def test_broad_narrow_random_scenes_bitwise():  # test_geometry.cpp:100-123 scenes
    rng = Rng(13)
    for _ in range(100):
        sd = random_scene(rng)
        ctx, o = _pair(sd)
        d_hat = rng.uniform(0.02, 0.2)
        g = ctx.broad_phase(o.q0, d_hat)
        e = o.broad_phase(o.q0, d_hat)
        assert np.array_equal(g, e)
        gp, gd = ctx.narrow_phase(o.q0, g, d_hat)
        ep, ed = o.narrow_phase(o.q0, e, d_hat)
        assert np.array_equal(gp, ep)
        assert np.array_equal(gd, ed)  # bitwise distances


def test_swept_broad_phase_and_ccd_bitwise():
    rng = Rng(17)
    for trial in range(60):
        sd = random_scene(rng, nb_lo=4, nb_hi=24, span=1.5)
        ctx, o = _pair(sd)
        if o.intersection_test(o.q0):
            continue
        q1 = _perturb(o.q0, rng, 0.4, o.is_static)
        for margin in (0.0, 0.01):
            g = ctx.broad_phase(o.q0, margin, q_end=q1)
            e = o.broad_phase(o.q0, margin, q_end=q1)
            assert np.array_equal(g, e)
        try:
            te = o.ccd_toi(o.q0, q1)
        except O.OracleError:
            with pytest.raises(DabdGpuError):
                ctx.ccd_toi(o.q0, q1)
            continue
        assert ctx.ccd_toi(o.q0, q1) == te  # bitwise TOI -> identical accept/reject


def test_ccd_known_answers():  # test_geometry.cpp:135-173
    tri = [(0.0, 1.0), (0.1, 1.2), (-0.1, 1.2)]
    bar = [(-1.0, -0.05), (1.0, -0.05), (1.0, 0.0), (-1.0, 0.0)]
    ctx, o = _pair(scene_of([[tri], [bar]], static=[False, True]))
    end = o.q0.copy()
    end[0, 1] -= 2.0
    assert ctx.ccd_toi(o.q0, end) == o.ccd_toi(o.q0, end)
    assert ctx.ccd_toi(o.q0, end) == pytest.approx(0.45, rel=1e-9)
    ctx, o = _pair(scene_of([[square(0.5)], [square(0.5, (2, 0))]]))
    assert ctx.ccd_toi(o.q0, o.q0) == 1.0
    end = o.q0.copy()
    end[1, 0] += 5.0
    assert ctx.ccd_toi(o.q0, end) == 1.0
    ctx, o = _pair(scene_of([[square(0.5)], [square(0.5, (1.0, 0))]]))
    end = o.q0.copy()
    end[1, 0] -= 0.5
    with pytest.raises(DabdGpuError):
        ctx.ccd_toi(o.q0, end)


@pytest.mark.parametrize("name", ["funnel-analog", "drop-grid-4", "heterogeneous", "cubes-64",
                                  "pile-1k"])
def test_builtin_scenes_bitwise(name):
    sd = make_scenario(name)
    ctx, o = _pair(sd)
    rng = Rng(5)
    q = _perturb(o.q0, rng, 0.01, o.is_static)
    q1 = _perturb(q, rng, 0.05, o.is_static)
    dh = sd.params.d_hat
    for (qa, qb, m) in ((o.q0, None, dh), (q, None, dh), (q, q1, dh), (q, q1, 0.0)):
        assert np.array_equal(ctx.broad_phase(qa, m, q_end=qb), o.broad_phase(qa, m, q_end=qb))
    # subsets (LocalObjective's local_ list)
    sub = [b for b in range(o.n) if b % 3 != 1 or o.is_static[b]]
    assert np.array_equal(ctx.broad_phase(q, dh, subset=sub), o.broad_phase(q, dh, subset=sub))
    # masks on the scene's planes with several widths
    if sd.planes:
        planes = np.array([[p.point[0], p.point[1], p.normal[0], p.normal[1]] for p in sd.planes])
        for w in (sd.w_min, 0.05, 0.3):
            try:
                me = o.holder_masks(q, planes, w)
            except O.OracleError:
                with pytest.raises(DabdGpuError):
                    ctx.holder_masks(q, planes, w)
                continue
            assert np.array_equal(ctx.holder_masks(q, planes, w), me)


def test_masks_known_answers_and_straddle():  # test_partition.cpp:32-105
    mid = np.array([[0.0, 0.0, -1.0, 0.0]])
    ctx, o = _pair(scene_of([[square(0.2)], [square(0.2, (-2, 0))], [square(0.2, (2, 0))],
                             [square(3.0, (0, 1))]], static=[False, False, False, True]))
    assert list(ctx.holder_masks(o.q0, mid, 0.4)) == [3, 1, 2, 3]
    g = scene_of([[square(1.0)]])
    ctx, o = _pair(g)
    with pytest.raises(DabdGpuError):
        ctx.holder_masks(o.q0, np.array([[-0.5, 0, -1, 0], [0.5, 0, -1, 0]]), 0.2)
