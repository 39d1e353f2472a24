"""Approach-sampling initialization (defaults) —
specified by the reference but not implemented there.

Per candidate (deterministic per (seed, index), counter-based Philox):
  * a random direction d from the object's centre of mass; the surface point
    p_s is where the ray leaves the zero level set (analytic for primitives,
    bisection on the trilinear grid for grids, the last ray/triangle crossing
    for meshes) and n is the outward normal;
  * palm position p_s + standoff * n, standoff = 1.2 x bounding radius;
  * palm approach axis (+z, assets.cpp:211) anti-parallel to n, roll about it
    uniform in [0, 2 pi);
  * joints at mid-range (hand.cpp:212-216).

This is host-side setup producing the optimizer's INPUT q; the same array is
fed to the GPU and to the oracle.
"""
from __future__ import annotations

import numpy as np

from .model import HandDesc, ObjectDesc


def _grid_phi(o: ObjectDesc, p: np.ndarray) -> np.ndarray:
    """Trilinear value (same node layout as csrc/dgx_geom.h GridSdf), inside the box."""
    u = (p - o.origin) * o.inv_spacing
    n = np.array(o.dims)
    u = np.clip(u, 0.0, n - 1.0)
    i = np.minimum(u.astype(np.int64), n - 2)
    t = u - i
    v = o.values
    def at(di, dj, dk):
        return v[i[..., 2] + dk, i[..., 1] + dj, i[..., 0] + di].astype(np.float64)
    tx, ty, tz = t[..., 0], t[..., 1], t[..., 2]
    c00 = at(0, 0, 0) + (at(1, 0, 0) - at(0, 0, 0)) * tx
    c10 = at(0, 1, 0) + (at(1, 1, 0) - at(0, 1, 0)) * tx
    c01 = at(0, 0, 1) + (at(1, 0, 1) - at(0, 0, 1)) * tx
    c11 = at(0, 1, 1) + (at(1, 1, 1) - at(0, 1, 1)) * tx
    c0 = c00 + (c10 - c00) * ty
    c1 = c01 + (c11 - c01) * ty
    return c0 + (c1 - c0) * tz


def surface_points(o: ObjectDesc, d: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """(p_s [B,3], outward unit normal [B,3]) along the rays com + t d (vectorised)."""
    d = np.atleast_2d(d)
    if o.kind == "sphere":
        return o.center[None, :] + o.radius * d, d.copy()
    if o.kind == "box":
        with np.errstate(divide="ignore"):
            ts = np.where(np.abs(d) > 0, o.half_extents[None, :] / np.abs(d), np.inf)
        k = np.argmin(ts, axis=1)
        t = ts[np.arange(d.shape[0]), k]
        n = np.zeros_like(d)
        n[np.arange(d.shape[0]), k] = np.sign(d[np.arange(d.shape[0]), k])
        return o.center[None, :] + t[:, None] * d, n
    if o.kind == "mesh":
        return _mesh_exit(o, d)
    lo = np.zeros(d.shape[0])
    hi = np.full(d.shape[0], float(np.max(o.spacing * (np.array(o.dims) - 1))))
    for _ in range(60):  # bisection on phi(com + t d) = 0
        mid = 0.5 * (lo + hi)
        inside = _grid_phi(o, o.com[None, :] + mid[:, None] * d) < 0.0
        lo = np.where(inside, mid, lo)
        hi = np.where(inside, hi, mid)
    p = o.com[None, :] + (0.5 * (lo + hi))[:, None] * d
    h = 0.5 * o.spacing
    g = np.stack([_grid_phi(o, p + h * e) - _grid_phi(o, p - h * e) for e in np.eye(3)], axis=1)
    gn = np.linalg.norm(g, axis=1, keepdims=True)
    n = np.where(gn > 0, g / np.where(gn > 0, gn, 1.0), d)
    return p, n


def _mesh_exit(o: ObjectDesc, d: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """Last crossing of the ray com + t d with the mesh (Moller-Trumbore over
    all faces) and that face's outward unit normal."""
    V, F = o.vertices, o.faces
    a, b, c = V[F[:, 0]], V[F[:, 1]], V[F[:, 2]]
    e1, e2 = b - a, c - a
    fn = np.cross(e1, e2)
    fn /= np.linalg.norm(fn, axis=1, keepdims=True)
    p = np.empty_like(d)
    n = np.empty_like(d)
    for k in range(d.shape[0]):
        h = np.cross(d[k][None, :], e2)
        det = np.sum(e1 * h, axis=1)
        ok = np.abs(det) > 1e-18
        f = np.where(ok, 1.0 / np.where(ok, det, 1.0), 0.0)
        s = o.com[None, :] - a
        u = f * np.sum(s * h, axis=1)
        qv = np.cross(s, e1)
        v = f * (qv @ d[k])
        t = f * np.sum(e2 * qv, axis=1)
        hit = ok & (u >= 0) & (v >= 0) & (u + v <= 1) & (t > 0)
        if not np.any(hit):
            raise ValueError("approach_init: ray from the COM misses the mesh")
        j = np.flatnonzero(hit)[np.argmax(t[hit])]
        p[k] = o.com + t[j] * d[k]
        n[k] = fn[j]
    return p, n


def surface_point(o: ObjectDesc, d: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    p, n = surface_points(o, np.asarray(d, np.float64)[None, :])
    return p[0], n[0]


def _quat_from_matrix(R: np.ndarray) -> np.ndarray:
    w = np.sqrt(max(0.0, 1.0 + R[0, 0] + R[1, 1] + R[2, 2])) / 2.0
    x = np.sqrt(max(0.0, 1.0 + R[0, 0] - R[1, 1] - R[2, 2])) / 2.0
    y = np.sqrt(max(0.0, 1.0 - R[0, 0] + R[1, 1] - R[2, 2])) / 2.0
    z = np.sqrt(max(0.0, 1.0 - R[0, 0] - R[1, 1] + R[2, 2])) / 2.0
    x = np.copysign(x, R[2, 1] - R[1, 2])
    y = np.copysign(y, R[0, 2] - R[2, 0])
    z = np.copysign(z, R[1, 0] - R[0, 1])
    q = np.array([w, x, y, z])
    return q / np.linalg.norm(q)


def approach_init(obj: ObjectDesc, hand: HandDesc, B: int, seed: int = 0, standoff_scale: float = 1.2,
                  first: int = 0) -> np.ndarray:
    """[B, 7+J] initial configurations for candidates first..first+B-1."""
    out = np.zeros((B, 7 + hand.num_joints))
    if B == 0:
        return out
    standoff = standoff_scale * obj.bounding_radius()
    mid = hand.mid_range()
    d = np.zeros((B, 3))
    roll = np.zeros(B)
    for b in range(B):
        rng = np.random.Generator(np.random.Philox(key=seed, counter=first + b))
        v = rng.normal(size=3)
        d[b] = v / np.linalg.norm(v)
        roll[b] = rng.uniform(0.0, 2.0 * np.pi)
    p_s, n = surface_points(obj, d)
    for b in range(B):
        z = -n[b]
        a = np.array([1.0, 0.0, 0.0]) if abs(z[0]) < 0.9 else np.array([0.0, 1.0, 0.0])
        x = a - np.dot(a, z) * z
        x /= np.linalg.norm(x)
        y = np.cross(z, x)
        c, s_ = np.cos(roll[b]), np.sin(roll[b])
        xr, yr = c * x + s_ * y, -s_ * x + c * y
        R = np.stack([xr, yr, z], axis=1)  # columns: palm x, y, z in world
        out[b, :3] = p_s[b] + standoff * n[b]
        out[b, 3:7] = _quat_from_matrix(R)
    out[:, 7:] = mid
    return out
