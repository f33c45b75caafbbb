"""Scene data, builtin scenarios and strict JSON (de)serialisation.

Host-side mirror of the reference's scene layer (proj/include/dabd/scene.hpp:15-56,
proj/src/scene.cpp). A scene is a list of body *specs* (world-space loops plus
density / velocity / static / arap_scale) and every solver knob; the C++ host
library turns the specs into affine bodies (centroid re-centring and exact
polygon moments, proj/src/body.cpp:96-118) when the scene is uploaded.

The builtin generators restate proj/src/scene.cpp:345-564 with the same
splitmix64 jitter stream (scene.cpp:18-32), so `make_scenario(name, seed)`
produces bit-identical geometry. The bench configurations of BASELINE.json
(cubes-64, pile-1k, pour-10k, hetero-1000, sweep-100k) are added as
further builtins following SURVEY.md Appendix B.
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

__all__ = [
    "SimParams",
    "AdaptParams",
    "Plane",
    "BodySpec",
    "SceneData",
    "JitterRng",
    "make_scenario",
    "scenario_names",
    "parse_scene_json",
    "scene_to_json",
]

_MASK64 = (1 << 64) - 1


class SceneError(ValueError):
    """Raised for invalid scene content (mirrors dabd::Error from scene.cpp)."""


@dataclass
class SimParams:
    """proj/include/dabd/params.hpp:8-23 (same field order and defaults)."""

    h: float = 0.01
    gravity: Tuple[float, float] = (0.0, -9.81)
    arap_stiffness: float = 1e6
    barrier_stiffness: float = 1e4
    d_hat: float = 0.01
    theta: float = 1e-3
    scene_scale: float = 1.0

    def validate(self) -> None:
        if self.h <= 0.0:
            raise SceneError("SimParams: h must be > 0")
        if self.d_hat <= 0.0:
            raise SceneError("SimParams: d_hat must be > 0")
        if self.theta <= 0.0:
            raise SceneError("SimParams: theta must be > 0")
        if self.scene_scale <= 0.0:
            raise SceneError("SimParams: scene_scale must be > 0")

    def as_array(self) -> np.ndarray:
        return np.array(
            [self.h, self.gravity[0], self.gravity[1], self.arap_stiffness,
             self.barrier_stiffness, self.d_hat, self.theta, self.scene_scale],
            dtype=np.float64,
        )


@dataclass
class AdaptParams:
    """proj/include/dabd/params.hpp:26-41."""

    beta: float = 1.0
    tau: float = 2.0
    mu: float = 5.0
    sigma_min: float = 1e-3
    sigma_max: float = 1e3
    adapt_enabled: bool = True

    def validate(self) -> None:
        if self.beta <= 0.0:
            raise SceneError("AdaptParams: beta must be > 0")
        if self.tau <= 1.0:
            raise SceneError("AdaptParams: tau must be > 1")
        if self.mu <= 1.0:
            raise SceneError("AdaptParams: mu must be > 1")
        if not (0.0 < self.sigma_min < 1.0 and self.sigma_max > 1.0):
            raise SceneError("AdaptParams: need 0 < sigma_min < 1 < sigma_max")

    def as_array(self) -> np.ndarray:
        return np.array([self.beta, self.tau, self.mu, self.sigma_min, self.sigma_max],
                        dtype=np.float64)


@dataclass
class Plane:
    """Interface plane between workers k and k+1 (partition.hpp:13-16)."""

    point: Tuple[float, float] = (0.0, 0.0)
    normal: Tuple[float, float] = (1.0, 0.0)


@dataclass
class BodySpec:
    """The JSON-level body description of scene.cpp:81-98."""

    loops: List[List[Tuple[float, float]]]
    density: float = 1000.0
    velocity: Tuple[float, ...] = (0.0,) * 6
    is_static: bool = False
    arap_scale: float = 1.0
    force_split: Optional[Tuple[float, float]] = None


@dataclass
class SceneData:
    """proj/include/dabd/scene.hpp:15-56 with body specs instead of built bodies."""

    name: str = "scene"
    bodies: List[BodySpec] = field(default_factory=list)
    params: SimParams = field(default_factory=SimParams)
    adapt: AdaptParams = field(default_factory=AdaptParams)
    planes: List[Plane] = field(default_factory=list)
    w_min: float = 0.1
    frames: int = 100
    admm_max_iterations: int = 300
    newton_cap: int = 32
    max_halvings: int = 4
    force_split_frames: int = -1
    seed: int = 0
    # balance knobs are carried for JSON round trips only (balancer is out of scope)
    balance: Dict[str, float] = field(default_factory=lambda: {
        "enabled": False, "kp": 0.5, "kd": 0.1, "smoothing": 0.5, "dp_max": 0.25})

    def dynamic_count(self) -> int:
        return sum(1 for b in self.bodies if not b.is_static)

    def validate(self) -> None:
        self.params.validate()
        self.adapt.validate()
        if self.frames < 0 or self.admm_max_iterations < 2 or self.newton_cap < 1:
            raise SceneError("scene: invalid iteration limits")

    def flat(self):
        """Flattened spec arrays consumed by the C ABI (dabd_gpu_scene_create)."""
        body_loop_start = [0]
        loop_vert_start = [0]
        verts: List[Tuple[float, float]] = []
        for b in self.bodies:
            for loop in b.loops:
                verts.extend(loop)
                loop_vert_start.append(len(verts))
            body_loop_start.append(len(loop_vert_start) - 1)
        n = len(self.bodies)
        return dict(
            n_bodies=n,
            body_loop_start=np.asarray(body_loop_start, dtype=np.int32),
            loop_vert_start=np.asarray(loop_vert_start, dtype=np.int32),
            verts=np.asarray(verts, dtype=np.float64).reshape(-1, 2),
            density=np.asarray([b.density for b in self.bodies], dtype=np.float64),
            is_static=np.asarray([1 if b.is_static else 0 for b in self.bodies], dtype=np.int32),
            arap_scale=np.asarray([b.arap_scale for b in self.bodies], dtype=np.float64),
            qdot=np.asarray([list(b.velocity) for b in self.bodies], dtype=np.float64).reshape(n, 6),
            planes=np.asarray([[p.point[0], p.point[1], p.normal[0], p.normal[1]]
                               for p in self.planes], dtype=np.float64).reshape(-1, 4),
            force_split=[(i, b.force_split) for i, b in enumerate(self.bodies)
                         if b.force_split is not None],
        )


class JitterRng:
    """splitmix64 jitter source, scene.cpp:18-32."""

    def __init__(self, seed: int) -> None:
        self.state = seed if seed else 0x9E3779B97F4A7C15

    def uniform(self, lo: float, hi: float) -> float:
        self.state = (self.state + 0x9E3779B97F4A7C15) & _MASK64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK64
        z = z ^ (z >> 31)
        u = float(z >> 11) * (2.0 ** -53)
        return lo + u * (hi - lo)


# ----------------------------------------------------------------------------
# geometry helpers (scene.cpp:48-79)
# ----------------------------------------------------------------------------

def box_loop(center, half):
    cx, cy = center
    hx, hy = half
    return [(cx + -hx, cy + -hy), (cx + hx, cy + -hy), (cx + hx, cy + hy), (cx + -hx, cy + hy)]


def ngon_loop(center, radius, sides, phase):
    out = []
    for i in range(sides):
        a = phase + 2.0 * math.pi * i / sides
        out.append((center[0] + radius * math.cos(a), center[1] + radius * math.sin(a)))
    return out


def loop_area(loop) -> float:
    area = 0.0
    n = len(loop)
    for i in range(n):
        ax, ay = loop[i]
        bx, by = loop[(i + 1) % n]
        area += (ax * by - bx * ay) / 2.0
    return area


def thick_segment_loop(a, b, thickness):
    dx, dy = b[0] - a[0], b[1] - a[1]
    nrm = math.sqrt(dx * dx + dy * dy)
    dx, dy = dx / nrm, dy / nrm
    nx, ny = -dy, dx
    s = 0.5 * thickness
    tx, ty = s * nx, s * ny
    loop = [(a[0] - tx, a[1] - ty), (b[0] - tx, b[1] - ty), (b[0] + tx, b[1] + ty),
            (a[0] + tx, a[1] + ty)]
    if loop_area(loop) < 0.0:
        loop.reverse()
    return loop


def rotate_loop(loop, pivot, angle):
    c, s = math.cos(angle), math.sin(angle)
    out = []
    for (x, y) in loop:
        wx, wy = x - pivot[0], y - pivot[1]
        out.append((pivot[0] + (c * wx + (-s) * wy), pivot[1] + (s * wx + c * wy)))
    return out


# ----------------------------------------------------------------------------
# builtin scenarios (scene.cpp:347-564) and the BASELINE.json configs
# ----------------------------------------------------------------------------

def _drop_params(scene: SceneData, l: float, kbar: float = 1e4) -> None:
    scene.params = SimParams(h=0.01, gravity=(0.0, -10.0), arap_stiffness=1e8,
                             barrier_stiffness=kbar, d_hat=0.01, theta=1e-3, scene_scale=l)


def funnel_analog(density: float = 1000.0, seed: int = 7) -> SceneData:
    s = SceneData(name="funnel-analog", frames=100, seed=seed)
    s.params = SimParams(h=0.01, gravity=(0.0, -10.0), arap_stiffness=1e8,
                         barrier_stiffness=1e5, d_hat=0.01, theta=3e-4, scene_scale=4.0)
    s.planes = [Plane((0.0, 0.0), (-1.0, 0.0))]
    s.w_min = 0.5
    s.bodies.append(BodySpec(loops=[box_loop((0.0, -0.06), (1.3, 0.06)),
                                    thick_segment_loop((-1.24, -0.02), (-2.0, 0.78), 0.12),
                                    thick_segment_loop((1.24, -0.02), (2.0, 0.78), 0.12)],
                             density=1000.0, is_static=True))
    rng = JitterRng(seed)
    for r in range(4):
        for c in range(8):
            cx = -0.98 + 0.28 * c
            cy = 0.145 + 0.45 * r
            cx += rng.uniform(-0.012, 0.012)
            cy += rng.uniform(-0.005, 0.005)
            s.bodies.append(BodySpec(loops=[box_loop((cx, cy), (0.12, 0.12))], density=density))
    return s


def drop_grid(slabs: int, seed: int = 11) -> SceneData:
    s = SceneData(name=f"drop-grid-{slabs}", frames=100, seed=seed)
    _drop_params(s, 2.0 * slabs)
    s.w_min = 0.4
    width = 2.0 * slabs
    for k in range(1, slabs):
        s.planes.append(Plane((-width / 2.0 + 2.0 * k, 0.0), (-1.0, 0.0)))
    s.bodies.append(BodySpec(loops=[box_loop((0.0, -0.06), (width / 2.0 + 0.2, 0.06)),
                                    box_loop((-width / 2.0 - 0.14, 0.8), (0.06, 0.8)),
                                    box_loop((width / 2.0 + 0.14, 0.8), (0.06, 0.8))],
                             density=1000.0, is_static=True))
    rng = JitterRng(seed)
    for sl in range(slabs):
        x0 = -width / 2.0 + 2.0 * sl + 0.35
        for r in range(4):
            for c in range(4):
                cx = x0 + 0.43 * c
                cy = 0.35 + 0.42 * r
                cx += rng.uniform(-0.02, 0.02)
                cy += rng.uniform(-0.02, 0.02)
                s.bodies.append(BodySpec(loops=[box_loop((cx, cy), (0.12, 0.12))]))
    return s


def blocked_merge() -> SceneData:
    s = SceneData(name="blocked-merge", frames=3, seed=3)
    s.params = SimParams(h=0.02, gravity=(0.0, -10.0), arap_stiffness=1e8,
                         barrier_stiffness=1e4, d_hat=0.01, theta=1e-3, scene_scale=2.0)
    s.planes = [Plane((0.0, 0.0), (-1.0, 0.0))]
    s.w_min = 0.8
    s.admm_max_iterations = 40
    s.force_split_frames = 1
    s.bodies.append(BodySpec(loops=[box_loop((0.0, -0.06), (1.5, 0.06))], is_static=True))
    s.bodies.append(BodySpec(loops=[box_loop((0.0, 1.0), (0.05, 0.3))], is_static=True))
    s.bodies.append(BodySpec(loops=[box_loop((0.0, 1.7), (0.15, 0.15))],
                             velocity=(0.0, -20.0, 0.0, 0.0, 0.0, 0.0),
                             force_split=(6.0e4, 0.0)))
    return s


def heterogeneous(seed: int = 13, groups=((1.0, 1.0), (100.0, 100.0), (10000.0, 10000.0)),
                  name: str = "heterogeneous") -> SceneData:
    s = SceneData(name=name, frames=100, seed=seed)
    s.params = SimParams(h=0.01, gravity=(0.0, -10.0), arap_stiffness=1e6,
                         barrier_stiffness=1e4, d_hat=0.01, theta=1e-3, scene_scale=4.0)
    s.planes = [Plane((0.0, 0.0), (-1.0, 0.0))]
    s.w_min = 0.4
    s.bodies.append(BodySpec(loops=[box_loop((0.0, -0.06), (2.2, 0.06)),
                                    box_loop((-2.14, 0.8), (0.06, 0.8)),
                                    box_loop((2.14, 0.8), (0.06, 0.8))], is_static=True))
    area = 0.24 * 0.24
    rng = JitterRng(seed)
    placed = 0
    for r in range(3):
        for c in range(8):
            mass, scale = groups[placed % len(groups)]
            cx = -1.47 + 0.42 * c
            cy = 0.35 + 0.45 * r
            cx += rng.uniform(-0.02, 0.02)
            cy += rng.uniform(-0.02, 0.02)
            s.bodies.append(BodySpec(loops=[box_loop((cx, cy), (0.12, 0.12))],
                                     density=mass / area, arap_scale=scale))
            placed += 1
    return s


def _container(width: float, wall_h: float):
    hw = width / 2.0
    return BodySpec(loops=[box_loop((0.0, -0.06), (hw + 0.2, 0.06)),
                           box_loop((-hw - 0.14, wall_h / 2.0), (0.06, wall_h / 2.0)),
                           box_loop((hw + 0.14, wall_h / 2.0), (0.06, wall_h / 2.0))],
                    is_static=True)


def lattice_pile(name: str, rows: int, cols_per_slab: int, slabs: int, half: float,
                 spacing: float, jitter: float, seed: int = 11, slab_width: float = 0.0,
                 l: Optional[float] = None) -> SceneData:
    """Dense lattice of boxes dropped into a floor-and-walls container.

    SURVEY.md Appendix B / 8(d): C2 (pile-1k), C3 (pour-10k), C5 (sweep-100k).
    Slabs of width `slab_width` are separated by interface planes at the slab
    boundaries (normal -x, worker k on the positive side, partition.hpp:10-16);
    each slab holds `cols_per_slab` columns centred in the slab so no body
    meets two interface slabs.
    """
    if slab_width <= 0.0:
        slab_width = cols_per_slab * spacing
    width = slab_width * slabs
    s = SceneData(name=name, frames=100, seed=seed)
    _drop_params(s, l if l is not None else max(2.0, width))
    s.w_min = 0.4
    for k in range(1, slabs):
        s.planes.append(Plane((-width / 2.0 + slab_width * k, 0.0), (-1.0, 0.0)))
    s.bodies.append(_container(width, rows * spacing + 1.0))
    rng = JitterRng(seed)
    y0 = half + 0.02
    for sl in range(slabs):
        x0 = -width / 2.0 + slab_width * sl + 0.5 * (slab_width - (cols_per_slab - 1) * spacing)
        for r in range(rows):
            for c in range(cols_per_slab):
                cx = x0 + spacing * c
                cy = y0 + spacing * r
                cx += rng.uniform(-jitter, jitter)
                cy += rng.uniform(-jitter, jitter)
                s.bodies.append(BodySpec(loops=[box_loop((cx, cy), (half, half))]))
    return s


def cubes_64(seed: int = 11) -> SceneData:
    """C1: drop-grid-4 geometry (64 boxes) on two partitions.

    The reference's mid plane x=0 leaves no body in the slab,
    so the single interface plane runs through the x=0.35 lattice column.
    """
    s = drop_grid(4, seed)
    s.name = "cubes-64"
    s.planes = [Plane((0.35, 0.0), (-1.0, 0.0))]
    return s


def pile_1k(seed: int = 11) -> SceneData:
    """C2: 1,000 boxes (25 rows x 40 columns), half 0.05, spacing 0.13."""
    return lattice_pile("pile-1k", rows=25, cols_per_slab=40, slabs=1, half=0.05,
                        spacing=0.13, jitter=0.005, seed=seed, l=6.0)


def pile_slabs(n: int, seed: int = 11) -> SceneData:
    """Weak-scaling workload: n pile-1k slabs side by side (n x 1,000 boxes),
    one interface plane between neighbouring slabs."""
    return lattice_pile(f"pile-1k-x{n}", rows=25, cols_per_slab=40, slabs=n, half=0.05,
                        spacing=0.13, jitter=0.005, seed=seed, l=6.0)


def pour_10k(seed: int = 11) -> SceneData:
    """C3: 10,000 boxes over 8 slabs (50 rows x 25 columns each)."""
    return lattice_pile("pour-10k", rows=50, cols_per_slab=25, slabs=8, half=0.03,
                        spacing=0.075, jitter=0.004, seed=seed, slab_width=2.0)


def sweep_100k(seed: int = 11) -> SceneData:
    """C5: 100,000 boxes over 8 slabs (125 rows x 100 columns each)."""
    return lattice_pile("sweep-100k", rows=125, cols_per_slab=100, slabs=8, half=0.02,
                        spacing=0.05, jitter=0.002, seed=seed, slab_width=5.2)


def hetero_1000(seed: int = 13) -> SceneData:
    """C4: heterogeneous groups with a 1000:1 mass ratio, arap_scale ~ mass."""
    return heterogeneous(seed, groups=((1.0, 1.0), (31.6227766, 31.6227766), (1000.0, 1000.0)),
                         name="hetero-1000")


def hooks_c4(seed: int = 17) -> SceneData:
    """C4: contact-rich non-convex bodies with 1000:1 mass
    ratios across a two-partition interface. The reference has no 2D
    "interlocking chains"; this uses its multi-loop / non-convex polygon
    bodies (scene.cpp:212-217) instead (parity-unpinned geometry):
      - a heavy U-shaped tray (non-convex, 8 vertices) spanning the x = 0
        interface, so it is split, and whose bounding box holds every box in
        it (> 96 broad-phase partners, > 24 coupled bodies in its BSR row);
      - 200 small boxes in the tray whose densities alternate 1000 and 1
        (1000:1 masses between neighbours), arap_scale proportional to mass
        (1 for the light bodies, as the heterogeneous builtin);
      - six U-hooks (density 1000) carrying one light peg each (density 1)
        dropped onto the pile.
    The U floors are thick enough that every loop centroid lies inside its
    own loop: intersection_test's centroid probe (geometry.cpp:412-427)
    assumes that, and would flag a cup holding a body otherwise.
    """
    s = SceneData(name="hooks-c4", frames=100, seed=seed)
    s.params = SimParams(h=0.01, gravity=(0.0, -10.0), arap_stiffness=1e6,
                         barrier_stiffness=1e4, d_hat=0.01, theta=1e-3, scene_scale=4.0)
    s.planes = [Plane((0.0, 0.0), (-1.0, 0.0))]
    s.w_min = 0.4
    s.bodies.append(_container(4.4, 1.6))

    def u_loop(cx, y0, hw, height, tf, tw):  # counter-clockwise U (cup opening up)
        return [(cx - hw, y0), (cx + hw, y0), (cx + hw, y0 + height), (cx + hw - tw, y0 + height),
                (cx + hw - tw, y0 + tf), (cx - hw + tw, y0 + tf), (cx - hw + tw, y0 + height),
                (cx - hw, y0 + height)]

    tray_y0, tray_tf = 0.015, 0.1
    s.bodies.append(BodySpec(loops=[u_loop(0.0, tray_y0, 1.6, 0.5, tray_tf, 0.06)], density=100.0,
                             arap_scale=1000.0))
    rng = JitterRng(seed)
    half, spacing, cols, rows = 0.03, 0.075, 40, 5
    y_row0 = tray_y0 + tray_tf + 0.015 + half
    for r in range(rows):
        for c in range(cols):
            heavy = (r + c) % 2 == 0
            cx = -0.5 * (cols - 1) * spacing + spacing * c + rng.uniform(-0.002, 0.002)
            cy = y_row0 + spacing * r + rng.uniform(-0.002, 0.002)
            dens = 1000.0 if heavy else 1.0
            s.bodies.append(BodySpec(loops=[box_loop((cx, cy), (half, half))], density=dens,
                                     arap_scale=dens))
    for k in range(6):
        cx = -1.25 + 0.5 * k
        s.bodies.append(BodySpec(loops=[u_loop(cx, 0.7, 0.2, 0.25, 0.09, 0.04)], density=1000.0,
                                 arap_scale=1000.0))
        s.bodies.append(BodySpec(loops=[box_loop((cx, 0.7 + 0.09 + 0.015 + 0.05), (0.05, 0.05))],
                                 density=1.0, arap_scale=1.0))
    return s


_BUILTINS = {
    "funnel-analog": lambda seed: funnel_analog(1000.0, 7 if seed is None else seed),
    "drop-grid-1": lambda seed: drop_grid(1, 11 if seed is None else seed),
    "drop-grid-2": lambda seed: drop_grid(2, 11 if seed is None else seed),
    "drop-grid-4": lambda seed: drop_grid(4, 11 if seed is None else seed),
    "heterogeneous": lambda seed: heterogeneous(13 if seed is None else seed),
    "cubes-64": lambda seed: cubes_64(11 if seed is None else seed),
    "pile-1k": lambda seed: pile_1k(11 if seed is None else seed),
    "pour-10k": lambda seed: pour_10k(11 if seed is None else seed),
    "sweep-100k": lambda seed: sweep_100k(11 if seed is None else seed),
    "hetero-1000": lambda seed: hetero_1000(13 if seed is None else seed),
    "hooks-c4": lambda seed: hooks_c4(17 if seed is None else seed),
}


def scenario_names() -> List[str]:
    """scene.cpp:559-564 plus the BASELINE.json configs."""
    return ["funnel-analog", "drop-grid-1", "drop-grid-2", "drop-grid-4", "density-sweep-10",
            "density-sweep-100", "density-sweep-1000", "density-sweep-10000",
            "density-sweep-100000", "blocked-merge", "heterogeneous", "cubes-64", "pile-1k",
            "pour-10k", "sweep-100k", "hetero-1000", "hooks-c4"]


def make_scenario(name: str, seed: Optional[int] = None) -> SceneData:
    """scene.cpp:538-557."""
    if name == "blocked-merge":
        s = blocked_merge()
        if seed is not None:
            s.seed = seed
        return s
    if name in _BUILTINS:
        return _BUILTINS[name](seed)
    if name.startswith("pile-1k-x"):
        return pile_slabs(int(name[len("pile-1k-x"):]), 11 if seed is None else seed)
    prefix = "density-sweep-"
    if name.startswith(prefix):
        density = float(name[len(prefix):])
        s = funnel_analog(density, 7 if seed is None else seed)
        s.name = name
        return s
    raise SceneError(f"unknown scenario '{name}'")


# ----------------------------------------------------------------------------
# strict JSON (scene.cpp:110-339)
# ----------------------------------------------------------------------------

def _require_keys(obj, where: str, allowed) -> None:
    if not isinstance(obj, dict):
        raise SceneError(f"scene: {where} must be an object")
    for key in obj:
        if key not in allowed:
            raise SceneError(f"scene: unknown key '{key}' in {where}")


def _vec2(v, where: str):
    if not isinstance(v, list) or len(v) != 2:
        raise SceneError(f"scene: {where} must be [x, y]")
    return (float(v[0]), float(v[1]))


def _velocity(v):
    if not isinstance(v, list) or len(v) not in (2, 6):
        raise SceneError("scene: velocity must have 2 or 6 entries")
    out = [0.0] * 6
    for i, x in enumerate(v):
        out[i] = float(x)
    return tuple(out)


def parse_scene_json(text: str) -> SceneData:
    root = json.loads(text)
    _require_keys(root, "root", {"name", "frames", "seed", "params", "adapt", "admm",
                                 "partition", "balance", "bodies", "grids",
                                 "force_split_frames"})
    s = SceneData()
    s.name = root.get("name", "scene")
    s.frames = int(root.get("frames", 100))
    s.seed = int(root.get("seed", 0))
    s.force_split_frames = int(root.get("force_split_frames", -1))
    if "params" in root:
        p = root["params"]
        _require_keys(p, "params", {"h", "gravity", "arap_stiffness", "barrier_stiffness",
                                    "d_hat", "theta", "scene_scale"})
        for k in ("h", "arap_stiffness", "barrier_stiffness", "d_hat", "theta", "scene_scale"):
            if k in p:
                setattr(s.params, k, float(p[k]))
        if "gravity" in p:
            s.params.gravity = _vec2(p["gravity"], "gravity")
    if "adapt" in root:
        a = root["adapt"]
        _require_keys(a, "adapt", {"beta", "tau", "mu", "sigma_min", "sigma_max", "enabled"})
        for k in ("beta", "tau", "mu", "sigma_min", "sigma_max"):
            if k in a:
                setattr(s.adapt, k, float(a[k]))
        if "enabled" in a:
            s.adapt.adapt_enabled = bool(a["enabled"])
    if "admm" in root:
        a = root["admm"]
        _require_keys(a, "admm", {"max_iterations", "newton_cap", "max_halvings"})
        s.admm_max_iterations = int(a.get("max_iterations", s.admm_max_iterations))
        s.newton_cap = int(a.get("newton_cap", s.newton_cap))
        s.max_halvings = int(a.get("max_halvings", s.max_halvings))
    if "partition" in root:
        p = root["partition"]
        _require_keys(p, "partition", {"planes", "w_min"})
        if "w_min" in p:
            s.w_min = float(p["w_min"])
        for pl in p.get("planes", []):
            _require_keys(pl, "plane", {"point", "normal"})
            nx, ny = _vec2(pl["normal"], "plane normal")
            n = math.sqrt(nx * nx + ny * ny)
            s.planes.append(Plane(_vec2(pl["point"], "plane point"), (nx / n, ny / n)))
    if "balance" in root:
        b = root["balance"]
        _require_keys(b, "balance", {"enabled", "kp", "kd", "smoothing", "dp_max"})
        s.balance.update(b)
    for b in root.get("bodies", []):
        _require_keys(b, "body", {"kind", "center", "half_extents", "radius", "sides", "loops",
                                  "density", "velocity", "static", "rotation", "arap_scale",
                                  "force_split", "from", "to", "thickness"})
        spec = BodySpec(loops=[], density=float(b.get("density", 1000.0)),
                        is_static=bool(b.get("static", False)),
                        arap_scale=float(b.get("arap_scale", 1.0)))
        if "velocity" in b:
            spec.velocity = _velocity(b["velocity"])
        if "force_split" in b:
            spec.force_split = _vec2(b["force_split"], "force_split")
        kind = b.get("kind", "box")
        if kind == "box":
            c = _vec2(b["center"], "center")
            loop = box_loop(c, _vec2(b["half_extents"], "half_extents"))
            if "rotation" in b:
                loop = rotate_loop(loop, c, float(b["rotation"]))
            spec.loops = [loop]
        elif kind == "ngon":
            spec.loops = [ngon_loop(_vec2(b["center"], "center"), float(b["radius"]),
                                    int(b["sides"]), float(b.get("rotation", 0.0)))]
        elif kind == "bar":
            spec.loops = [thick_segment_loop(_vec2(b["from"], "from"), _vec2(b["to"], "to"),
                                             float(b["thickness"]))]
        elif kind == "polygon":
            spec.loops = [[_vec2(v, "vertex") for v in loop] for loop in b["loops"]]
        else:
            raise SceneError(f"scene: unknown body kind '{kind}'")
        s.bodies.append(spec)
    if "grids" in root:
        rng = JitterRng(s.seed)
        for g in root["grids"]:
            _require_keys(g, "grid", {"kind", "half_extents", "radius", "sides", "rows", "cols",
                                      "origin", "spacing", "jitter", "density", "velocity",
                                      "arap_scale"})
            rows, cols = int(g["rows"]), int(g["cols"])
            ox, oy = _vec2(g["origin"], "origin")
            sx, sy = _vec2(g["spacing"], "spacing")
            jit = float(g.get("jitter", 0.0))
            kind = g.get("kind", "box")
            for r in range(rows):
                for c in range(cols):
                    spec = BodySpec(loops=[], density=float(g.get("density", 1000.0)),
                                    arap_scale=float(g.get("arap_scale", 1.0)))
                    if "velocity" in g:
                        spec.velocity = _velocity(g["velocity"])
                    cx, cy = ox + c * sx, oy + r * sy
                    cx += rng.uniform(-jit, jit)
                    cy += rng.uniform(-jit, jit)
                    if kind == "box":
                        spec.loops = [box_loop((cx, cy), _vec2(g["half_extents"], "half_extents"))]
                    elif kind == "ngon":
                        spec.loops = [ngon_loop((cx, cy), float(g["radius"]), int(g["sides"]),
                                                rng.uniform(0.0, 2.0 * math.pi))]
                    else:
                        raise SceneError(f"scene: unknown grid kind '{kind}'")
                    s.bodies.append(spec)
    s.validate()
    return s


def scene_to_json(scene: SceneData) -> str:
    """scene.cpp:279-339: bodies are written as world-space polygons."""
    root = {
        "name": scene.name,
        "frames": scene.frames,
        "seed": scene.seed,
        "params": {"h": scene.params.h, "gravity": list(scene.params.gravity),
                   "arap_stiffness": scene.params.arap_stiffness,
                   "barrier_stiffness": scene.params.barrier_stiffness,
                   "d_hat": scene.params.d_hat, "theta": scene.params.theta,
                   "scene_scale": scene.params.scene_scale},
        "adapt": {"beta": scene.adapt.beta, "tau": scene.adapt.tau, "mu": scene.adapt.mu,
                  "sigma_min": scene.adapt.sigma_min, "sigma_max": scene.adapt.sigma_max,
                  "enabled": scene.adapt.adapt_enabled},
        "admm": {"max_iterations": scene.admm_max_iterations, "newton_cap": scene.newton_cap,
                 "max_halvings": scene.max_halvings},
        "partition": {"planes": [{"point": list(p.point), "normal": list(p.normal)}
                                 for p in scene.planes], "w_min": scene.w_min},
        "balance": dict(scene.balance),
        "bodies": [],
    }
    if scene.force_split_frames >= 0:
        root["force_split_frames"] = scene.force_split_frames
    for b in scene.bodies:
        jb = {"kind": "polygon", "loops": [[list(v) for v in loop] for loop in b.loops],
              "density": b.density, "static": b.is_static, "velocity": list(b.velocity)}
        if b.arap_scale != 1.0:
            jb["arap_scale"] = b.arap_scale
        if b.force_split is not None:
            jb["force_split"] = list(b.force_split)
        root["bodies"].append(jb)
    return json.dumps(root, indent=2)
