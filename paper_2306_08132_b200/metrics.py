"""Grasp-quality metrics. The reference
specifies this module but has no code for it; behaviour follows SPEC.md:
  * contacts(): GPU contact generation (dgx_contacts_batch): hand samples with
    |rho| <= threshold at the object's canonical pose become contacts at their
    smoothed surface points r*_rho with normal grad rho, and
    contact area = sum of HandModel::sample_areas over contacts,
    for up to 16 thresholds in one launch;
  * wrench_hull_metrics(): per contact `cone_edges` unit forces on the friction
    cone about the inward normal (|f_t| = mu |f_n| before normalisation),
    wrenches (f, lambda (p - com) x f) with lambda = 1 / max |p - com|; epsilon
    = radius of the largest origin-centred ball inside their convex hull (0 if
    the origin is not strictly inside), gws volume = 6-D hull volume; fewer
    than 7 affinely independent wrenches -> (0, 0). The hull
    is Qhull (scipy.spatial), on the host: an evaluation path, correctness over
    speed; above `max_contacts` (default 32) contacts the hull is
    taken over a deterministic farthest-point subset (6-D hull cost grows
    steeply with the point count), None = every contact;
  * threshold_sweep() / top_k(): Fig. 3-style CSV rows and Table 2's "top10
    (ranked by epsilon metric)" aggregation.
Units at the boundary: SPEC reports CA in cm^2 and thresholds in mm.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import api, capi


@dataclass
class Contacts:
    thresholds: np.ndarray   # [T] m
    area: np.ndarray         # [B, T] m^2
    count: np.ndarray        # [B, T]
    n: np.ndarray            # [B] contacts at the largest threshold
    index: np.ndarray        # [B, cap] sample indices (ascending), -1 padded
    rec: np.ndarray          # [B, cap, 7] rho, smoothed point (3), unit gradient (3)

    def at(self, b: int, t: float):
        """(points [K,3], normals [K,3]) of candidate b at threshold t (<= max)."""
        k = min(int(self.n[b]), self.index.shape[1])
        r = self.rec[b, :k]
        sel = np.abs(r[:, 0]) <= t
        return r[sel, 1:4], r[sel, 4:7]


def contacts(ctx: api.Context, hand: api.Hand, obj: api.GraspObject, q, thresholds_mm=(5.0,), cap: int | None = None
             ) -> Contacts:
    hd = hand.desc
    if hd.sample_area is None:
        raise ValueError("hand descriptor has no sample_area (re-export assets with tools/export_assets.py)")
    q = np.ascontiguousarray(q, np.float64).reshape(-1, 7 + hd.num_joints)
    B = q.shape[0]
    thr = np.ascontiguousarray(np.asarray(thresholds_mm, np.float64) * 1e-3)
    T = thr.size
    cap = hd.num_samples if cap is None else int(cap)
    area, count = np.zeros((B, T)), np.zeros((B, T), np.int32)
    n = np.zeros(B, np.int32)
    idx, rec = np.full((B, cap), -1, np.int32), np.zeros((B, cap, 7))
    sa = np.ascontiguousarray(hd.sample_area, np.float64)
    capi.check(ctx.L.dgx_contacts_batch(ctx.h, hand.h, obj.h, B, capi.ptr(q), capi.ptr(sa), T,
                                        thr.ctypes.data_as(capi._dp), cap, capi.ptr(area), capi.ptr(count),
                                        capi.ptr(n), capi.ptr(idx), capi.ptr(rec), 0))
    return Contacts(thr, area, count, n, idx, rec)


def _tangents(n: np.ndarray):
    a = np.where(np.abs(n[:, 0:1]) < 0.9, np.array([[1.0, 0.0, 0.0]]), np.array([[0.0, 1.0, 0.0]]))
    t1 = np.cross(n, a)
    t1 /= np.linalg.norm(t1, axis=1, keepdims=True)
    return t1, np.cross(n, t1)


def contact_wrenches(points, normals, com, mu: float = 1.0, cone_edges: int = 8) -> np.ndarray:
    """[K*E, 6] unit-force cone-edge wrenches."""
    points, normals = np.asarray(points, np.float64).reshape(-1, 3), np.asarray(normals, np.float64).reshape(-1, 3)
    if points.shape[0] == 0:
        return np.zeros((0, 6))
    n_in = -normals / np.linalg.norm(normals, axis=1, keepdims=True)  # force pushes into the object
    t1, t2 = _tangents(n_in)
    ang = 2.0 * np.pi * np.arange(cone_edges) / cone_edges
    f = n_in[:, None, :] + mu * (np.cos(ang)[None, :, None] * t1[:, None, :] + np.sin(ang)[None, :, None] * t2[:, None, :])
    f /= np.linalg.norm(f, axis=2, keepdims=True)
    r = points - np.asarray(com, np.float64)[None, :]
    rmax = float(np.max(np.linalg.norm(r, axis=1)))
    lam = 1.0 / rmax if rmax > 0 else 0.0
    tq = lam * np.cross(r[:, None, :], f)
    return np.concatenate([f, tq], axis=2).reshape(-1, 6)


def farthest_subset(points: np.ndarray, k: int) -> np.ndarray:
    """Deterministic farthest-point subset (starting from contact 0)."""
    n = points.shape[0]
    if n <= k:
        return np.arange(n)
    sel = [0]
    d = np.linalg.norm(points - points[0], axis=1)
    for _ in range(k - 1):
        j = int(np.argmax(d))
        sel.append(j)
        d = np.minimum(d, np.linalg.norm(points - points[j], axis=1))
    return np.sort(np.array(sel))


def wrench_hull_metrics(points, normals, com, mu: float = 1.0, cone_edges: int = 8,
                        max_contacts: int | None = None) -> tuple[float, float]:
    """(epsilon, gws_volume). max_contacts: hull of a
    farthest-point subset of at most that many contacts (6-D Qhull cost grows
    steeply: ~0.2 s at 32 contacts, ~14 s at 250); None = all contacts."""
    if cone_edges < 3:
        raise ValueError("cone_edges must be >= 3")
    points = np.asarray(points, np.float64).reshape(-1, 3)
    normals = np.asarray(normals, np.float64).reshape(-1, 3)
    if max_contacts is not None and points.shape[0] > max_contacts:
        sel = farthest_subset(points, max_contacts)
        points, normals = points[sel], normals[sel]
    w = contact_wrenches(points, normals, com, mu, cone_edges)
    if w.shape[0] < 7 or np.linalg.matrix_rank(w[1:] - w[0], tol=1e-12) < 6:
        return 0.0, 0.0
    from scipy.spatial import ConvexHull
    from scipy.spatial._qhull import QhullError
    try:
        hull = ConvexHull(w)
    except QhullError:
        return 0.0, 0.0
    off = hull.equations[:, 6]             # normal . x + off <= 0 inside, unit normals
    eps = float(np.min(-off)) if np.all(off < 0.0) else 0.0
    return max(eps, 0.0), float(hull.volume)


def evaluate(ctx, hand, obj, q, thresholds_mm=(5.0,), mu: float = 1.0, cone_edges: int = 8,
             hull_thresholds_mm=None, max_contacts: int | None = 32, workers: int | None = None) -> list:
    """Per candidate and threshold: MetricReport-like dicts (CA cm^2, contact
    count, epsilon, gws volume). Contact generation for all
    candidates and thresholds is one GPU launch; the wrench hulls (host Qhull,
    threads) are computed at hull_thresholds_mm (default: all thresholds),
    elsewhere epsilon / gws_volume are None."""
    import os
    from concurrent.futures import ThreadPoolExecutor
    con = contacts(ctx, hand, obj, q, thresholds_mm)
    com = obj.desc.com
    thr = np.asarray(thresholds_mm, np.float64)
    hull_t = set(range(thr.size)) if hull_thresholds_mm is None else \
        {int(np.argmin(np.abs(thr - h))) for h in hull_thresholds_mm}
    jobs = [(b, t) for b in range(con.n.shape[0]) for t in sorted(hull_t)]

    def run(job):
        b, t = job
        p, n = con.at(b, con.thresholds[t])
        return wrench_hull_metrics(p, n, com, mu, cone_edges, max_contacts)

    with ThreadPoolExecutor(workers or os.cpu_count()) as ex:
        res = dict(zip(jobs, ex.map(run, jobs)))
    out = []
    for b in range(con.n.shape[0]):
        rows = []
        for t, tm in enumerate(thr):
            eps, vol = res.get((b, t), (None, None))
            rows.append(dict(threshold_mm=float(tm), contact_area_cm2=float(con.area[b, t] * 1e4),
                             contacts=int(con.count[b, t]), epsilon=eps, gws_volume=vol))
        out.append(rows)
    return out


def threshold_sweep(reports: list, path: str | None = None) -> list:
    """Per-threshold means (CSV columns SPEC.md:519)."""
    T = len(reports[0])
    rows = []
    def mean(col, key):
        v = [c[key] for c in col if c[key] is not None]
        return float(np.mean(v)) if v else None

    for t in range(T):
        col = [r[t] for r in reports]
        rows.append(dict(threshold_mm=col[0]["threshold_mm"], mean_CA_cm2=mean(col, "contact_area_cm2"),
                         mean_eps=mean(col, "epsilon"), mean_vol=mean(col, "gws_volume")))
    if path:
        f = lambda v: "" if v is None else f"{v:.9g}"  # noqa: E731
        with open(path, "w", encoding="utf-8") as fh:
            fh.write("threshold_mm,mean_CA_cm2,mean_eps,mean_vol\n")
            for r in rows:
                fh.write(f"{f(r['threshold_mm'])},{f(r['mean_CA_cm2'])},{f(r['mean_eps'])},{f(r['mean_vol'])}\n")
    return rows


def top_k(reports: list, k: int = 10, threshold_index: int = 0) -> list:
    """Indices of the k grasps with the highest epsilon ("top10")."""
    eps = np.array([r[threshold_index]["epsilon"] for r in reports])
    return [int(i) for i in np.argsort(-eps, kind="stable")[:k]]
