"""Device penetration audit vs the oracle: intersection_test
(geometry.cpp:389-454, bit-exact decision, per pair) and the minimum
point-edge distance (tests/support/oracles.cpp:153-173, bitwise)."""

import numpy as np
import pytest

import oracle as O
from support import Rng, scene_of, square
from test_gpu_geometry import _pair, _perturb
from test_oracle_kat import random_scene
from paper_2605_15875_b200 import api
from paper_2605_15875_b200.scene import make_scenario

pytestmark = pytest.mark.gpu

CUTOFF = 1e300  # every pair within reach: the minimum is exact


def _oracle_violations(o, q):
    n = 0
    for i in range(o.n):
        for j in range(i + 1, o.n):
            n += o.intersection_test(q, subset=[i, j])
    return n


def test_intersection_known_cases():  # test_geometry.cpp:217-245 shapes
    hbar = [(-2, -0.1), (2, -0.1), (2, 0.1), (-2, 0.1)]
    vbar = [(-0.1, -2), (0.1, -2), (0.1, 2), (-0.1, 2)]
    cases = [([[square(0.5)], [square(0.5, (2, 0))]], False),
             ([[square(0.5)], [square(0.5)]], True),            # coincident: centroid test
             ([[square(0.5)], [square(0.5, (0.6, 0.3))]], True),
             ([[square(0.5)], [square(0.5, (1.0, 0))]], False),  # touching is not inside
             ([[hbar], [vbar]], True)]                          # crossing without a vertex inside
    for loops, expect in cases:
        ctx, o = _pair(scene_of(loops))
        hit, nv, dmin = ctx.audit(o.q0, cutoff=CUTOFF)
        assert hit == expect == o.intersection_test(o.q0)
        assert nv == int(expect)
        assert dmin == o.min_pair_distance(o.q0)


def test_random_scenes_per_pair_and_distance_bitwise():
    rng = Rng(29)
    hits = 0
    for trial in range(40):
        sd = random_scene(rng, nb_lo=4, nb_hi=20, span=1.2)
        ctx, o = _pair(sd)
        q = _perturb(o.q0, rng, 0.3, o.is_static) if trial % 2 else o.q0
        hit, nv, dmin = ctx.audit(q, cutoff=CUTOFF)
        assert hit == o.intersection_test(q)
        assert nv == _oracle_violations(o, q)
        assert dmin == o.min_pair_distance(q)  # bitwise
        hits += hit
        # a subset audits only its own pairs
        sub = list(range(0, o.n, 2))
        assert ctx.intersection_test(q, subset=sub) == o.intersection_test(q, subset=sub)
    assert 5 <= hits <= 35  # both outcomes exercised


def test_cutoff_bounds_the_distance_search():
    ctx, o = _pair(scene_of([[square(0.5)], [square(0.5, (1.5, 0))], [square(0.5, (5, 0))]]))
    assert ctx.audit(o.q0, cutoff=0.3)[2] == 0.5        # within 2 x cutoff: exact
    assert ctx.audit(o.q0, cutoff=0.1)[2] > 1e300       # nothing within reach
    assert ctx.audit(o.q0, cutoff=0.0)[2] > 1e300       # distance not requested


@pytest.mark.parametrize("name,workers,frames", [("pile-1k", 0, 30), ("cubes-64", 2, 40)])
def test_simulated_pile_stays_penetration_free(name, workers, frames):
    """North-star property: zero interpenetration and a positive minimum
    distance over the whole scene after stepping, audited on the device
    state and cross-checked against the oracle on the downloaded state."""
    sd = make_scenario(name)
    ctx = api.Context(api.Scene(sd), num_workers=workers)
    ctx.run_frames(frames)
    hit, nv, dmin = ctx.audit(None, cutoff=sd.params.d_hat)
    q, _ = ctx.state()
    o = O.Scene(sd)
    assert not hit and nv == 0
    assert not o.intersection_test(q)
    assert 0.0 < dmin < sd.params.d_hat
    assert dmin == o.min_pair_distance(q)


def test_pour_10k_eight_partitions_penetration_free():
    sd = make_scenario("pour-10k")
    ctx = api.Context(api.Scene(sd), num_workers=8)
    ctx.run_frames(3)
    hit, nv, dmin = ctx.audit(None, cutoff=sd.params.d_hat)
    assert not hit and nv == 0
    assert dmin > 0.0
