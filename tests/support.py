"""Test-only helpers restating proj/tests/support/oracles.{hpp,cpp}.

Rng is the splitmix64 generator of oracles.hpp:15-36; random_convex_polygon
follows oracles.cpp:130-146; the brute-force active set follows
oracles.cpp:199-230 (vectorised, distances from the same formulas).
"""

from __future__ import annotations

import math

import numpy as np

from paper_2605_15875_b200.scene import BodySpec, SceneData, SimParams

_M = (1 << 64) - 1


class Rng:
    def __init__(self, seed: int) -> None:
        self.state = seed if seed else 0x9E3779B97F4A7C15

    def next_u64(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & _M
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M
        return z ^ (z >> 31)

    def uniform(self, lo: float = 0.0, hi: float = 1.0) -> float:
        u = float(self.next_u64() >> 11) * (2.0 ** -53)
        return lo + u * (hi - lo)

    def uniform_int(self, lo: int, hi: int) -> int:
        return lo + int(self.next_u64() % (hi - lo + 1))


def random_convex_polygon(rng: Rng, min_v, max_v, min_r, max_r):
    while True:
        n = rng.uniform_int(min_v, max_v)
        angles = sorted(rng.uniform(0.0, 2.0 * math.pi) for _ in range(n))
        r = rng.uniform(min_r, max_r)
        loop = [(r * math.cos(a), r * math.sin(a)) for a in angles]
        ok = True
        for i in range(n):
            nxt = angles[(i + 1) % n] + (2.0 * math.pi if i + 1 == n else 0.0)
            if nxt - angles[i] < 1e-3:
                ok = False
                break
        if ok:
            return loop


def square(half, center=(0.0, 0.0)):
    cx, cy = center
    return [(-half + cx, -half + cy), (half + cx, -half + cy), (half + cx, half + cy),
            (-half + cx, half + cy)]


def scene_of(loops_list, density=1.0, static=None, params=None, velocities=None):
    """Scene from a list of per-body loop lists (make_affine_body inputs)."""
    s = SceneData(name="test")
    static = static or [False] * len(loops_list)
    for i, loops in enumerate(loops_list):
        vel = (0.0,) * 6 if velocities is None else tuple(velocities[i])
        dens = density[i] if isinstance(density, (list, tuple)) else density
        s.bodies.append(BodySpec(loops=loops, density=dens, is_static=static[i], velocity=vel))
    if params is not None:
        s.params = params
    return s


def world_points(rest, vert_start, q):
    """x = A xbar + p, unfused (types.hpp:28-30)."""
    out = np.zeros_like(rest)
    nb = len(vert_start) - 1
    for b in range(nb):
        s, e = vert_start[b], vert_start[b + 1]
        xb = rest[s:e]
        qq = q[b]
        out[s:e, 0] = (qq[2] * xb[:, 0] + qq[3] * xb[:, 1]) + qq[0]
        out[s:e, 1] = (qq[4] * xb[:, 0] + qq[5] * xb[:, 1]) + qq[1]
    return out


def edge_next(oscene):
    """Second endpoint (flat index) of each edge, loop wrap-around."""
    nxt = np.zeros(oscene.nv, dtype=np.int64)
    for b, spec in enumerate(oscene.scene.bodies):
        base = oscene.vert_start[b]
        for loop in spec.loops:
            n = len(loop)
            for i in range(n):
                nxt[base + i] = base + (i + 1) % n
            base += n
    return nxt


def pe_distance_np(p, e0, e1):
    """Vectorised point_edge_distance value (geometry.cpp:34-56)."""
    e = e1 - e0
    len2 = e[:, 0] * e[:, 0] + e[:, 1] * e[:, 1]
    w = p - e0
    t = (w[:, 0] * e[:, 0] + w[:, 1] * e[:, 1]) / len2
    u0 = p - e0
    u1 = p - e1
    d0 = np.sqrt(u0[:, 0] * u0[:, 0] + u0[:, 1] * u0[:, 1])
    d1 = np.sqrt(u1[:, 0] * u1[:, 0] + u1[:, 1] * u1[:, 1])
    c = e[:, 0] * w[:, 1] - e[:, 1] * w[:, 0]
    s = np.where(c >= 0.0, 1.0, -1.0)
    di = (s * c) / np.sqrt(len2)
    return np.where(t <= 0.0, d0, np.where(t >= 1.0, d1, di))


def brute_force_active_pairs(oscene, q, d_hat):
    """oracles.cpp:199-230: all ordered cross-body pairs with d < d_hat."""
    X = world_points(oscene.rest, oscene.vert_start, q)
    nxt = edge_next(oscene)
    vs = oscene.vert_start
    rows = []
    nb = oscene.n
    for a in range(nb):
        va = np.arange(vs[a], vs[a + 1])
        for b in range(nb):
            if a == b:
                continue
            eb = np.arange(vs[b], vs[b + 1])
            P = np.repeat(X[va], len(eb), axis=0)
            E0 = np.tile(X[eb], (len(va), 1))
            E1 = np.tile(X[nxt[eb]], (len(va), 1))
            d = pe_distance_np(P, E0, E1)
            idx = np.nonzero(d < d_hat)[0]
            for k in idx:
                rows.append((a, b, int(k // len(eb)), int(k % len(eb)), d[k]))
    rows.sort(key=lambda r: r[:4])
    pairs = np.array([r[:4] for r in rows], dtype=np.int32).reshape(-1, 4)
    ds = np.array([r[4] for r in rows])
    return pairs, ds


def default_params(**kw):
    p = SimParams(h=0.01, gravity=(0.0, -10.0), arap_stiffness=1e8, barrier_stiffness=1e4,
                  d_hat=0.01)
    for k, v in kw.items():
        setattr(p, k, v)
    return p


def assert_rho(rho_g, rho_o, max_flip_frac=0.0):
    """Final per-replica rho (runtime.cpp:481-482). rho only ever changes by
    exact factors of tau (and the sigma clamps), so a replica either carries
    the oracle's value to 1e-12 or one of its adaptation decisions flipped.
    The decision compares r_b with mu s_b (consensus.cpp:44-52); for a
    replica at rest both are at rounding level (~1e-17) and rounding decides
    the comparison, which two implementations whose iterates agree to ~1e-14
    (not bitwise) cannot share. `max_flip_frac` bounds the flipped fraction
    (0: every replica exact)."""
    rho_g, rho_o = np.asarray(rho_g), np.asarray(rho_o)
    same = np.isclose(rho_g, rho_o, rtol=1e-12, atol=0.0)
    flips = ~same
    ratio = rho_g[flips] / rho_o[flips]
    print(f"rho: {same.sum()} of {len(same)} replicas equal, {flips.sum()} decision flips"
          + (f" (ratios {ratio.min():.3g}..{ratio.max():.3g})" if flips.any() else ""))
    allowed = 0 if max_flip_frac <= 0.0 else max(1, int(max_flip_frac * len(same)))
    assert flips.sum() <= allowed, (int(flips.sum()), len(same))
