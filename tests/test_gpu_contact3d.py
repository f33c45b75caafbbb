"""3D affine-body contact terms: point-triangle and
edge-edge distance, barrier value, gradient and PSD-clamped Hessian over the
24 DoF of two 12-DoF bodies (dabd_gpu_contact3d_terms).

Parity is unpinned (the reference is 2D). The checkers: the independent
CPU restatement oracle/geometry3d.cpp (distance as a minimum over all
feature pairs, barrier of energy.cpp:50-61), central finite differences for
the gradient and the unprojected Hessian, numpy's eigen-clamp
(objective.cpp:12-17) for the projected Hessian, and closed-form known
answers. Tolerances are stated per check.
"""

import numpy as np
import pytest

import oracle as O
from paper_2605_15875_b200 import api
from paper_2605_15875_b200 import _lib as L

D_HAT, KAPPA = 0.05, 1e4


def _rand_affine(rng, center, scale=0.15):
    A = np.eye(3) + scale * rng.standard_normal((3, 3))
    return np.concatenate([center, A.reshape(-1)]), A


def _pair(rng, kind, target_d):
    """Random world configuration of one PT / EE pair at distance ~target_d,
    returned in body coordinates (qa, qb, rest)."""
    qa, Aa = _rand_affine(rng, rng.standard_normal(3))
    qb, Ab = _rand_affine(rng, rng.standard_normal(3))
    if kind == 0:
        tri = rng.standard_normal((3, 3)) * 0.3
        n = np.cross(tri[1] - tri[0], tri[2] - tri[0])
        n /= np.linalg.norm(n)
        bary = rng.dirichlet([1, 1, 1]) * 1.6 - 0.2  # inside and outside the face
        p = bary @ tri + target_d * n
        world = np.vstack([p, tri])
        owner = [0, 1, 1, 1]
    else:
        a0 = rng.standard_normal(3) * 0.3
        u = rng.standard_normal(3)
        v = rng.standard_normal(3)
        n = np.cross(u, v)
        n /= np.linalg.norm(n)
        s, t = rng.uniform(-0.3, 1.3, size=2)
        b0 = a0 + s * u - t * v + target_d * n
        world = np.vstack([a0, a0 + u, b0, b0 + v])
        owner = [0, 0, 1, 1]
    rest = np.zeros((4, 3))
    for i in range(4):
        q, A = (qa, Aa) if owner[i] == 0 else (qb, Ab)
        rest[i] = np.linalg.solve(A, world[i] - q[:3])
    return qa, qb, rest


def _batch(seed, n):
    rng = np.random.default_rng(seed)
    kinds, qas, qbs, rests = [], [], [], []
    for k in range(n):
        kind = k % 2
        while True:  # keep pairs inside the barrier's support (d < d_hat)
            qa, qb, rest = _pair(rng, kind, rng.uniform(0.2, 0.95) * D_HAT)
            if O.contact3d_value(kind, qa, qb, rest, D_HAT, KAPPA)[0] < 0.97 * D_HAT:
                break
        kinds.append(kind)
        qas.append(qa)
        qbs.append(qb)
        rests.append(rest)
    return np.array(kinds), np.array(qas), np.array(qbs), np.array(rests)


def _oracle_value(kind, q24, rest):
    return O.contact3d_value(kind, q24[:12], q24[12:], rest, D_HAT, KAPPA)[2]


def test_contact3d_argument_checks():
    """CPU: argument validation happens before any device work."""
    with pytest.raises(L.DabdGpuError, match="kind"):
        api.contact3d_terms([2], np.zeros((1, 12)), np.zeros((1, 12)), np.zeros((1, 4, 3)),
                            D_HAT, KAPPA)
    out = api.contact3d_terms(np.zeros(0, np.int32), np.zeros((0, 12)), np.zeros((0, 12)),
                              np.zeros((0, 4, 3)), D_HAT, KAPPA)
    assert out["d"].shape == (0,)


def test_oracle3d_known_answers():
    """CPU: closed-form distances through the oracle restatement."""
    I = np.concatenate([np.zeros(3), np.eye(3).reshape(-1)])
    tri = np.array([[0.0, 0, 0], [1, 0, 0], [0, 1, 0]])
    # above the face: d = height, type 6
    d, t, _ = O.contact3d_value(0, I, I, np.vstack([[0.2, 0.2, 0.03], tri]), D_HAT, KAPPA)
    assert d == pytest.approx(0.03, rel=1e-15) and t == 6
    # beyond vertex t1: point-point
    d, t, _ = O.contact3d_value(0, I, I, np.vstack([[1.02, -0.01, 0.0], tri]), D_HAT, KAPPA)
    assert d == pytest.approx(np.hypot(0.02, 0.01), rel=1e-14) and t == 1
    # crossing perpendicular edges 0.04 apart: line-line
    rest = np.array([[-1.0, 0, 0], [1, 0, 0], [0, -1, 0.04], [0, 1, 0.04]])
    d, t, v = O.contact3d_value(1, I, I, rest, D_HAT, KAPPA)
    assert d == pytest.approx(0.04, rel=1e-14) and t == 8
    assert v == pytest.approx(-KAPPA * (0.04 - D_HAT) ** 2 * np.log(0.04 / D_HAT), rel=1e-14)


@pytest.mark.gpu
def test_contact3d_known_answers_gpu():
    I = np.concatenate([np.zeros(3), np.eye(3).reshape(-1)])
    tri = np.array([[0.0, 0, 0], [1, 0, 0], [0, 1, 0]])
    rest = np.array([np.vstack([[0.2, 0.2, 0.03], tri]), np.vstack([[1.02, -0.01, 0.0], tri]),
                     [[-1.0, 0, 0], [1, 0, 0], [0, -1, 0.04], [0, 1, 0.04]],
                     [[0.0, 0, 0], [1, 0, 0], [2.0, 0.02, 0], [3, 0.02, 0]]])
    out = api.contact3d_terms([0, 0, 1, 1], np.tile(I, (4, 1)), np.tile(I, (4, 1)), rest, D_HAT, KAPPA)
    assert out["d"][0] == pytest.approx(0.03, rel=1e-14) and out["type"][0] == 6
    assert out["d"][1] == pytest.approx(np.hypot(0.02, 0.01), rel=1e-14) and out["type"][1] == 1
    assert out["d"][2] == pytest.approx(0.04, rel=1e-14) and out["type"][2] == 8
    # collinear, disjoint edges: a1 against b0 (vertex-vertex, type 2)
    assert out["d"][3] == pytest.approx(np.hypot(1.0, 0.02), rel=1e-14) and out["type"][3] == 2
    assert out["value"][3] == 0.0 and not out["grad"][3].any()


@pytest.mark.gpu
def test_contact3d_matches_oracle_and_finite_differences():
    kinds, qa, qb, rest = _batch(3, 64)
    g = api.contact3d_terms(kinds, qa, qb, rest, D_HAT, KAPPA, project=False)
    types = {0: set(), 1: set()}
    for k in range(len(kinds)):
        d, t, v = O.contact3d_value(kinds[k], qa[k], qb[k], rest[k], D_HAT, KAPPA)
        assert g["d"][k] == pytest.approx(d, rel=1e-11)
        assert g["value"][k] == pytest.approx(v, rel=1e-9)
        assert g["type"][k] == t
        types[int(kinds[k])].add(t)
        # gradient vs central differences of the oracle value (rel 1e-5)
        q24 = np.concatenate([qa[k], qb[k]])
        h = 1e-7
        fd = np.array([(_oracle_value(kinds[k], q24 + h * e, rest[k]) -
                        _oracle_value(kinds[k], q24 - h * e, rest[k])) / (2 * h) for e in np.eye(24)])
        scale = np.abs(fd).max()
        assert np.abs(g["grad"][k] - fd).max() < 1e-5 * scale
        # unprojected Hessian vs central differences of the device gradient (rel 1e-5)
        qp = np.array([q24 + h * e for e in np.eye(24)])
        qm = np.array([q24 - h * e for e in np.eye(24)])
        gp = api.contact3d_terms(np.full(24, kinds[k]), qp[:, :12], qp[:, 12:], np.tile(rest[k], (24, 1, 1)),
                                 D_HAT, KAPPA, hessian=False)["grad"]
        gm = api.contact3d_terms(np.full(24, kinds[k]), qm[:, :12], qm[:, 12:], np.tile(rest[k], (24, 1, 1)),
                                 D_HAT, KAPPA, hessian=False)["grad"]
        Hfd = (gp - gm) / (2 * h)
        assert np.abs(g["hess"][k] - Hfd).max() < 1e-5 * np.abs(Hfd).max()
        assert np.abs(g["hess"][k] - g["hess"][k].T).max() <= 1e-12 * np.abs(Hfd).max()
    # the batch covers the face / line-line cases and at least one other type
    assert 6 in types[0] and 8 in types[1]
    assert len(types[0]) + len(types[1]) >= 4


@pytest.mark.gpu
def test_contact3d_projection_is_the_eigen_clamp():
    """project=1 equals V max(L, 0) V^T of the unprojected 24x24 Hessian
    (objective.cpp:12-17) to 1e-9 relative; the result is PSD."""
    kinds, qa, qb, rest = _batch(11, 40)
    raw = api.contact3d_terms(kinds, qa, qb, rest, D_HAT, KAPPA, project=False)
    prj = api.contact3d_terms(kinds, qa, qb, rest, D_HAT, KAPPA, project=True)
    assert np.array_equal(raw["grad"], prj["grad"]) and np.array_equal(raw["value"], prj["value"])
    for k in range(len(kinds)):
        w, V = np.linalg.eigh(raw["hess"][k])
        ref = (V * np.maximum(w, 0.0)) @ V.T
        sc = np.abs(raw["hess"][k]).max()
        assert np.abs(prj["hess"][k] - ref).max() < 1e-9 * sc
        assert np.linalg.eigvalsh(prj["hess"][k]).min() > -1e-10 * sc


@pytest.mark.gpu
def test_contact3d_inactive_and_penetrating():
    kinds, qa, qb, rest = _batch(5, 4)
    far = qa.copy()
    far[:, :3] += 10.0  # body a translated far away
    out = api.contact3d_terms(kinds, far, qb, rest, D_HAT, KAPPA)
    assert (out["d"] >= D_HAT).all() and not out["value"].any() and not out["grad"].any()
    I = np.concatenate([np.zeros(3), np.eye(3).reshape(-1)])
    touching = np.array([[[0.2, 0.2, 0.0], [0, 0, 0], [1, 0, 0], [0, 1, 0]]])
    with pytest.raises(L.DabdGpuError, match="d <= 0"):
        api.contact3d_terms([0], I[None], I[None], touching, D_HAT, KAPPA)


# ---- 3D CCD (additive CCD, dabd_gpu_ccd3d) ---------------------------------
def _moving_batch(seed, n):
    """Pairs whose body a translates along the contact normal through body b
    (every other pair: a hit) or away from it (a miss), with a small random
    affine drift on both bodies."""
    rng = np.random.default_rng(seed)
    kinds, qa0, qa1, qb0, qb1, rests = [], [], [], [], [], []
    for k in range(n):
        kind = k % 2
        qa, qb, rest = _pair(rng, kind, rng.uniform(0.3, 0.9) * D_HAT)
        d = O.contact3d_value(kind, qa, qb, rest, D_HAT, KAPPA)[0]
        h = 1e-7
        gn = np.array([(O.contact3d_value(kind, qa + h * e, qb, rest, D_HAT, KAPPA)[0] - d) / h
                       for e in np.eye(12)[:3]])
        gn /= np.linalg.norm(gn)
        step = np.zeros(12)
        step[:3] = (-3.0 * d if k % 4 < 2 else 0.5 * d) * gn
        kinds.append(kind)
        qa0.append(qa)
        qa1.append(qa + step + 1e-3 * d * rng.standard_normal(12))
        qb0.append(qb)
        qb1.append(qb + 1e-3 * d * rng.standard_normal(12))
        rests.append(rest)
    return [np.array(x) for x in (kinds, qa0, qa1, qb0, qb1, rests)]


def test_oracle_ccd3d_known_answers():
    """CPU: a point falling through a triangle's face, and missing it."""
    I = np.concatenate([np.zeros(3), np.eye(3).reshape(-1)])
    tri = [[0.0, 0, 0], [1, 0, 0], [0, 1, 0]]
    rest = np.vstack([[0.2, 0.2, 0.0], tri])
    up, down = I.copy(), I.copy()
    up[2], down[2] = 0.1, -0.1  # the point's body moves from z=0.1 to z=-0.1
    t = O.ccd3d(0, up, down, I, I, rest)
    assert 0.40 < t < 0.5  # conservative, within the last 10% of the gap
    side = I.copy()
    side[0] = 0.5
    up2 = up.copy()
    up2[0] = 0.5
    assert O.ccd3d(0, up, up2, I, I, rest) == 1.0  # parallel to the face: no impact


@pytest.mark.gpu
def test_ccd3d_conservative_and_matches_oracle():
    """Hits (body a driven 3 d(0) through the closest feature: contact at
    t = 1/3 up to the 1e-3 drift) stop before contact with a positive gap and
    within the last 10% of it; misses (moving apart) return exactly 1.0; the
    device agrees with the oracle restatement (rel 1e-9) on >= 90% of pairs
    (the rest differ only by a break decision flipped by rounding)."""
    kinds, qa0, qa1, qb0, qb1, rest = _moving_batch(7, 48)
    toi = api.ccd3d(kinds, qa0, qa1, qb0, qb1, rest)
    agree = 0
    for k in range(len(kinds)):
        ref = O.ccd3d(kinds[k], qa0[k], qa1[k], qb0[k], qb1[k], rest[k])
        agree += toi[k] == ref or abs(toi[k] - ref) <= 1e-9 * ref
        if k % 4 < 2:
            assert 0.25 < toi[k] < 0.33, (k, toi[k])
            t = toi[k]
            d = O.contact3d_value(kinds[k], qa0[k] + t * (qa1[k] - qa0[k]), qb0[k] + t * (qb1[k] - qb0[k]),
                                  rest[k], D_HAT, KAPPA)[0]
            assert d > 0.0
        else:
            assert toi[k] == 1.0
    assert agree >= 0.9 * len(kinds)


@pytest.mark.gpu
def test_ccd3d_known_answers_gpu():
    I = np.concatenate([np.zeros(3), np.eye(3).reshape(-1)])
    rest = np.vstack([[0.2, 0.2, 0.0], [0.0, 0, 0], [1, 0, 0], [0, 1, 0]])
    up, down, up2 = I.copy(), I.copy(), I.copy()
    up[2], down[2], up2[2] = 0.1, -0.1, 0.1
    up2[0] = 0.5
    toi = api.ccd3d([0, 0, 0], [up, up, I], [down, up2, I], [I, I, I], [I, I, I], [rest, rest, rest])
    assert 0.40 < toi[0] < 0.5 and toi[1] == 1.0 and toi[2] == 1.0


# ---- 3D broad phase (dabd_gpu_broad_phase3d) --------------------------------
def _box_mesh(half=0.1):
    """Closed box surface in rest coordinates: 8 vertices, 12 triangles, 18 edges."""
    v = np.array([[x, y, z] for x in (-half, half) for y in (-half, half) for z in (-half, half)])
    quads = [(0, 1, 3, 2), (4, 6, 7, 5), (0, 4, 5, 1), (2, 3, 7, 6), (0, 2, 6, 4), (1, 5, 7, 3)]
    tris = []
    for a, b, c, d in quads:
        tris += [(a, b, c), (a, c, d)]
    edges = sorted({tuple(sorted((t[i], t[(i + 1) % 3]))) for t in tris for i in range(3)})
    return v, np.array(tris), np.array(edges)


def _pile3d(seed, n):
    rng = np.random.default_rng(seed)
    meshes, q = [], []
    for i in range(n):
        meshes.append(_box_mesh(rng.uniform(0.08, 0.12)))
        A = np.eye(3) + 0.1 * rng.standard_normal((3, 3))
        q.append(np.concatenate([rng.uniform(-0.5, 0.5, 3), A.ravel()]))
    return np.array(q), meshes


def test_broad_phase3d_argument_checks():
    v, t, e = _box_mesh()
    bad = t.copy()
    bad[0, 0] = 99
    with pytest.raises(L.DabdGpuError, match="out of range"):
        api.broad_phase3d(np.tile(np.concatenate([np.zeros(3), np.eye(3).ravel()]), (2, 1)),
                          [(v, bad, e), (v, t, e)], 0.01)
    assert api.broad_phase3d(np.zeros((1, 12)), [(v, t, e)], 0.01).shape == (0, 5)


@pytest.mark.gpu
@pytest.mark.parametrize("seed,n,swept", [(1, 12, False), (2, 20, True), (3, 40, False)])
def test_broad_phase3d_bitwise_against_brute_force(seed, n, swept):
    q, meshes = _pile3d(seed, n)
    q_end = q + 0.02 * np.random.default_rng(seed + 100).standard_normal(q.shape) if swept else None
    got = api.broad_phase3d(q, meshes, 0.01, q_end=q_end)
    ref = O.broad_phase3d(q, meshes, 0.01, q_end=q_end)
    assert len(ref) > 0 and (ref[:, 0] == 0).any() and (ref[:, 0] == 1).any()
    assert np.array_equal(got, ref)


@pytest.mark.gpu
def test_broad_phase3d_feeds_contact_terms():
    """Every pair the 3D contact terms see as active (d < d_hat) is in the
    broad phase's candidate list with margin d_hat (no missed contacts)."""
    q, meshes = _pile3d(4, 16)
    cand = api.broad_phase3d(q, meshes, D_HAT)
    cset = {tuple(r) for r in cand.tolist()}
    kinds, qa, qb, rest, keys = [], [], [], [], []
    for a in range(len(meshes)):
        for b in range(len(meshes)):
            if a == b:
                continue
            va, ta, ea = meshes[a]
            vb, tb, eb = meshes[b]
            for vi in range(len(va)):
                for ti, t in enumerate(tb):
                    kinds.append(0); qa.append(q[a]); qb.append(q[b])
                    rest.append(np.vstack([va[vi], vb[t]])); keys.append((0, a, b, vi, ti))
            if a < b:
                for i, e in enumerate(ea):
                    for j, f in enumerate(eb):
                        kinds.append(1); qa.append(q[a]); qb.append(q[b])
                        rest.append(np.vstack([va[e], vb[f]])); keys.append((1, a, b, i, j))
    # skip pairs that interpenetrate in this random pile (d = 0 is an error)
    out = {}
    for s in range(0, len(kinds), 4096):
        try:
            r = api.contact3d_terms(kinds[s:s + 4096], qa[s:s + 4096], qb[s:s + 4096], rest[s:s + 4096],
                                    D_HAT, KAPPA, hessian=False)
        except L.DabdGpuError:
            continue
        for k, d in zip(keys[s:s + 4096], r["d"]):
            out[k] = d
    active = [k for k, d in out.items() if d < D_HAT]
    assert active, "the pile has no close pairs"
    assert all(k in cset for k in active)
