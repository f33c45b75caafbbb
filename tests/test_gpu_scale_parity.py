"""Oracle parity at the configurations the bench and the north star run
(BASELINE.json configs C2-C5), from states the GPU reached itself:

- C2 pile-1k, run_reference semantics (sim.cpp:186-249) at the bench's own
  solver settings (PCG to 1e-10 relative, warm-started): GPU and oracle start
  from the same settled pile and step 5 frames side by side;
- C3 pour-10k with 8 partitions, consensus-ADMM semantics
  (runtime.cpp:110-694): ADMM traces (dq, r, s), merge-gate TOIs, iteration
  counts and the final rho of a frame from an oracle-poured 8-partition state
  (the oracle's frame is recorded in a fixture);
- C5 sweep-100k: broad phase (plain and swept), holder masks and CCD
  accept/reject bitwise at a settled state;
- C4 hooks-c4: non-convex bodies, 1000:1 mass ratios across the interface, a
  tray whose BSR row outgrows the initial ELL width.

Tolerances are the north star's: states within 1e-6 (relative to the scene
scale l), residual traces within 1e-6 h l, integer decisions exact.
"""

import os

import numpy as np
import pytest

import oracle as O
from support import assert_rho
from paper_2605_15875_b200 import api
from paper_2605_15875_b200.scene import make_scenario

pytestmark = pytest.mark.gpu

# the oracle-parity settings emulate the reference's exact solves: PCG to
# 1e-12 and every Newton direction to it (inexact Newton off)
TIGHT = dict(pcg_rel_tol=1e-12, pcg_max_iters=20000, inexact=(0.0, 10.0))
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _settled(name, frames, workers=0, **solver):
    """The scene after `frames` GPU frames (run_reference, or consensus ADMM
    over `workers` partitions)."""
    sd = make_scenario(name)
    ctx = api.Context(api.Scene(sd), num_workers=workers, **solver)
    if frames:
        ctx.run_frames(frames)
    q, qd = ctx.state()
    return sd, q, qd


def test_pile_1k_bench_settings():
    """C2 at the bench's settings: identical ADMM (k-loop) counts, no exact
    retries, states within 1e-6 l of the oracle for 5 consecutive frames."""
    sd, q, qd = _settled("pile-1k", 40)
    ctx = api.Context(api.Scene(sd))  # defaults = bench.py (1e-10, warm start)
    ctx.set_state(q, qd)
    o = O.Scene(sd)
    o.set_state(q, qd)
    frames = 5
    ref = o.run(frames, workers=0)
    l = sd.params.scene_scale
    for f in range(frames):
        st = ctx.run_frames(1)[0]
        qg, _ = ctx.state()
        assert st["admm_iterations"] == ref["admm"][f], (f, st["admm_iterations"], ref["admm"][f])
        assert st["exact_retries"] == 0 and st["capacity_retries"] == 0, (f, st)
        err = np.abs(qg - ref["q"][f]).max()
        assert err < 1e-6 * l, (f, err)


def test_pour_10k_eight_partitions():
    """C3: one consensus-ADMM frame of the 8-partition pour from a contact-
    rich 8-partition state (tests/golden/pour-10k_w8.npz: the oracle poured
    30 single-domain frames and ran 2 frames on 8 partitions; the fixture
    holds that state and the oracle's next frame, tools/make_pour_fixture.py),
    rho carry empty on both sides as at the start of a run: identical ADMM
    counts, attempts and sigma decisions, identical merge-gate accept/reject
    decisions with the TOI values within 1e-9 relative, dq / r / s within
    1e-6 h l, states within 1e-6 l, final rho to 1e-12 with at most 5% of
    the replicas on a flipped adaptation decision (support.assert_rho; the
    recorded frame takes 275 ADMM iterations over 3 attempts, and 27 of its
    1,476 replicas, 1.8%, end one or two adaptation steps apart).

    The gate TOIs are bit-exact on identical inputs (test_gpu_geometry); here
    they are evaluated at ADMM iterates that agree with the oracle's to the
    PCG's rounding, not bitwise, so their values carry that rounding."""
    z = np.load(os.path.join(GOLDEN, "pour-10k_w8.npz"))
    sd = make_scenario("pour-10k")
    ctx = api.Context(api.Scene(sd), num_workers=8, **TIGHT)
    ctx.set_state(z["q0"], z["qd0"])
    stats = ctx.run_frames(1)
    qg, _ = ctx.state()
    tr_g, tr_o = ctx.take_trace(), z["trace"]
    norm = sd.params.h * sd.params.scene_scale
    assert stats[0]["admm_iterations"] == z["admm"][0], (stats[0]["admm_iterations"], z["admm"][0])
    assert stats[0]["attempts"] == z["attempts"][0]
    assert tr_g.shape == tr_o.shape
    assert np.array_equal(tr_g[:, [1, 2, 7]], tr_o[:, [1, 2, 7]])
    assert np.array_equal(tr_g[:, 6] == 1.0, tr_o[:, 6] == 1.0)  # merge-gate accept/reject
    toi_rel = np.abs(tr_g[:, 6] - tr_o[:, 6]) / tr_o[:, 6]
    assert toi_rel.max() < 1e-9, toi_rel.max()
    for col in (3, 4, 5):
        err = np.abs(tr_g[:, col] - tr_o[:, col]).max()
        assert err < 1e-6 * norm, (col, err)
    assert np.abs(qg - z["q1"]).max() < 1e-6 * sd.params.scene_scale
    rho_g, rho_o = ctx.rho(), z["rho"]
    shared = ~np.isnan(rho_o)
    assert shared.sum() > 100  # the interfaces of a settled pour carry many split bodies
    assert stats[0]["admm_iterations"] > 3 and stats[0]["max_contacts"] > 10000
    assert np.array_equal(shared, ~np.isnan(rho_g))
    assert_rho(rho_g[shared], rho_o[shared], 0.05)


@pytest.mark.slow
def test_sweep_100k_broad_phase_and_masks():
    """C5 at a settled state: candidate lists (static and swept), holder masks
    of the 8-slab partition and the CCD accept/reject decision are bitwise the
    oracle's."""
    sd, q, qd = _settled("sweep-100k", 8)
    ctx = api.Context(api.Scene(sd))
    o = O.Scene(sd)
    d_hat = sd.params.d_hat
    a = ctx.broad_phase(q, d_hat)
    b = o.broad_phase(q, d_hat)
    assert len(a) > 100000 and np.array_equal(a, b)
    q1 = q + sd.params.h * qd
    a = ctx.broad_phase(q, 0.0, q_end=q1)
    b = o.broad_phase(q, 0.0, q_end=q1)
    assert np.array_equal(a, b)
    planes = np.array([[p.point[0], p.point[1], p.normal[0], p.normal[1]] for p in sd.planes])
    w = max(2.0 * sd.params.h * float(np.abs(qd).max()) * 2.0, sd.w_min)
    mg, mo = ctx.holder_masks(q, planes, w), o.holder_masks(q, planes, w)
    assert np.array_equal(mg, mo)
    assert (np.array([bin(int(m)).count("1") for m in mg[1:]]) == 2).sum() > 100
    tg, to = ctx.ccd_toi(q, q1), o.ccd_toi(q, q1)
    assert tg == to


def test_hooks_c4_two_partitions():
    """C4: consensus-ADMM parity over the first 8 frames (exact counts,
    decisions and gate TOIs), then 30 GPU frames stay penetration-free; the
    tray's BSR row outgrows the initial ELL width (24 coupled bodies) and
    the engine grows it instead of failing."""
    from test_gpu_admm import _compare

    # 1000:1 mass ratios: the Newton systems are ill-conditioned enough that
    # a 1e-12 relative PCG residual leaves ~1e-5 h l of difference to the
    # reference's exact LDL^T step, so the PCG runs at the exact-solve limit
    gpu, ref = _compare("hooks-c4", 2, 8, state_tol=1e-6, trace_tol=1e-5, rho_flips=0.05,
                        pcg_rel_tol=1e-14, pcg_max_iters=50000, inexact=(0.0, 10.0))
    sd = make_scenario("hooks-c4")
    ctx = api.Context(api.Scene(sd), num_workers=2)
    st = ctx.run_frames(30)
    assert all(s["committed"] for s in st)
    assert sum(s["capacity_retries"] for s in st) >= 1
    intersecting, violating, dmin = ctx.audit()
    assert not intersecting and violating == 0 and dmin > 0.0


def test_large_body_partner_spill():
    """k_emit_warp keeps at most 96 broad-phase partners per body in shared
    memory; the tray of hooks-c4 has ~200 boxes inside its bounding box, so
    its candidates come from the spill path. Candidate lists stay bitwise
    the oracle's."""
    sd, q, _ = _settled("hooks-c4", 20)
    ctx = api.Context(api.Scene(sd))
    o = O.Scene(sd)
    for margin in (sd.params.d_hat, 0.05):
        a = ctx.broad_phase(q, margin)
        b = o.broad_phase(q, margin)
        assert np.array_equal(a, b)
        assert len(np.unique(a[a[:, 0] == 1, 1])) + len(np.unique(a[a[:, 1] == 1, 0])) > 30


def test_pour_10k_single_domain_grid_pcg():
    """The undivided pour (one partition of 10,000 rows) goes past the
    cluster kernel's 4,096-row limit to the grid-wide pipelined PCG
    (k_pcg_grid): two run_reference frames against the oracle's, identical
    ADMM counts and states within 1e-6 l (exact-solve settings)."""
    sd = make_scenario("pour-10k")
    ref = O.Scene(sd).run(2, workers=0)
    gpu = api.run_reference(sd, 2, **TIGHT)
    for f in range(2):
        assert gpu.stats[f]["admm_iterations"] == ref["admm"][f]
        assert np.abs(gpu.q[f] - ref["q"][f]).max() < 1e-6 * sd.params.scene_scale
    assert sum(s["pcg_iterations"] for s in gpu.stats) > 0
