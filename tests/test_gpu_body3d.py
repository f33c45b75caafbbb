"""12-DoF (3D) affine bodies: mass moments from a closed triangle surface
and the inertia + orthogonality body terms (the
reference is 2D, so parity is unpinned). Checkers: closed-form cube moments,
the oracle's signed-tetrahedra moments, the oracle's energy value with
central finite differences for gradient and Hessian, numpy's eigen-clamp
(objective.cpp:12-17) for the projected Hessian."""

import numpy as np
import pytest

import oracle as O
from paper_2605_15875_b200 import api
from paper_2605_15875_b200 import _lib as L


def _cube(lo=(0.0, 0.0, 0.0), size=1.0):
    v = np.array([[x, y, z] for x in (0, 1) for y in (0, 1) for z in (0, 1)], float) * size + lo
    # outward-oriented triangles of the 6 faces (vertex index = 4x + 2y + z)
    quads = [(0, 1, 3, 2), (4, 6, 7, 5), (0, 4, 5, 1), (2, 3, 7, 6), (0, 2, 6, 4), (1, 5, 7, 3)]
    tris = []
    for a, b, c, d in quads:
        tris += [(a, b, c), (a, c, d)]
    return v, np.array(tris)


def _hull(seed, n=30):
    from scipy.spatial import ConvexHull

    rng = np.random.default_rng(seed)
    pts = rng.standard_normal((n, 3)) * [0.3, 0.2, 0.1] + [1.0, -2.0, 0.5]
    h = ConvexHull(pts)
    tris = []
    cen = pts[h.vertices].mean(axis=0)
    for s in h.simplices:
        a, b, c = pts[s]
        tris.append(s if np.dot(np.cross(b - a, c - a), a - cen) > 0 else s[[0, 2, 1]])
    return pts, np.array(tris)


def test_cube_moments_known_answers():
    v, t = _cube((2.0, -1.0, 0.5), 2.0)
    mom, cen, vol = api.body3d_moments(v, t, density=3.0)
    assert vol == pytest.approx(8.0, rel=1e-14)
    assert np.allclose(cen, [3.0, 0.0, 1.5], rtol=0, atol=1e-14)
    assert mom[0] == pytest.approx(24.0, rel=1e-14)
    # S_xx = rho * a^5 / 12 for a cube of side a about its centroid
    assert mom[4] == pytest.approx(3.0 * 32.0 / 12.0, rel=1e-13)
    assert abs(mom[5]) < 1e-12 and abs(mom[6]) < 1e-12 and abs(mom[8]) < 1e-12
    with pytest.raises(L.DabdGpuError, match="volume"):
        api.body3d_moments(v, t[:, [0, 2, 1]])  # inward orientation


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_hull_moments_match_oracle(seed):
    v, t = _hull(seed)
    mom, cen, vol = api.body3d_moments(v, t, density=500.0)
    rm, rc, rv = O.polyhedron_moments_tets(v, t, 500.0)
    assert vol == pytest.approx(rv, rel=1e-12)
    assert np.allclose(cen, rc, rtol=1e-12, atol=1e-13)
    assert np.allclose(mom, rm, rtol=1e-10, atol=1e-12 * rm[0])


@pytest.mark.gpu
def test_body3d_terms_match_oracle_fd_and_clamp():
    rng = np.random.default_rng(4)
    bodies = [O.polyhedron_moments_tets(*_hull(s), 800.0) for s in range(6)]
    mom = np.array([b[0] for b in bodies])
    w = np.array([1e8 * b[2] for b in bodies])  # ARAP-dominated: indefinite blocks get clamped
    scale = 1e-4
    q = np.array([np.concatenate([rng.standard_normal(3), (np.eye(3) + 0.2 * rng.standard_normal((3, 3))).ravel()])
                  for _ in range(6)])
    qt = q + 0.01 * rng.standard_normal(q.shape)
    raw = api.body3d_terms(q, qt, mom, w, scale, project=False)
    prj = api.body3d_terms(q, qt, mom, w, scale, project=True)
    h = 1e-6
    for b in range(6):
        v = O.body3d_value(q[b], qt[b], mom[b], w[b], scale)
        assert raw["value"][b] == pytest.approx(v, rel=1e-12)
        fd = np.array([(O.body3d_value(q[b] + h * e, qt[b], mom[b], w[b], scale) -
                        O.body3d_value(q[b] - h * e, qt[b], mom[b], w[b], scale)) / (2 * h) for e in np.eye(12)])
        assert np.abs(raw["grad"][b] - fd).max() < 1e-6 * np.abs(fd).max()
        gp = api.body3d_terms(q[b] + h * np.eye(12), np.tile(qt[b], (12, 1)), np.tile(mom[b], (12, 1)),
                              np.full(12, w[b]), scale, hessian=False)["grad"]
        gm = api.body3d_terms(q[b] - h * np.eye(12), np.tile(qt[b], (12, 1)), np.tile(mom[b], (12, 1)),
                              np.full(12, w[b]), scale, hessian=False)["grad"]
        Hfd = (gp - gm) / (2 * h)
        H = raw["hess"][b]
        assert np.abs(H - Hfd).max() < 1e-6 * np.abs(Hfd).max()
        lam, V = np.linalg.eigh(H)
        ref = (V * np.maximum(lam, 0.0)) @ V.T
        assert np.abs(prj["hess"][b] - ref).max() < 1e-9 * np.abs(H).max()
    assert np.array_equal(raw["grad"], prj["grad"])
    # the batch exercises the clamp (some raw blocks indefinite)
    assert any(np.linalg.eigvalsh(raw["hess"][b]).min() < 0 for b in range(6))
