"""Scene pipeline around the batched drop.

The reference implements the physics step (``step_on_table``, sim.cpp:14-94)
but not the pipeline; its behaviour here follows SPEC.md:
  * ``scene_states``: per seed a uniform random orientation and a drop height
    of 2x the bounding-sphere radius (COM at z = 2 r_b over the table origin),
    at rest. Deterministic per (seed) via counter-based Philox.
  * ``generate_scenes``: all seeds dropped in one batched GPU launch
    (``api.drop``) until at rest (contact step with kinetic energy < 1e-6 J) or
    5 s simulated.
  * ``transfer_grasps``: base grasps (canonical object pose) composed with each
    scene's object pose, joints unchanged; rejected if any hand surface point
    is below the table by more than ``table_clearance``.
  * ``export_jsonl``: one JSON-lines file per (hand, object) + a manifest
    (SPEC.md:561-569), 9 significant digits, stable field order.
"""
from __future__ import annotations

import hashlib
import json
import os
from dataclasses import dataclass

import numpy as np

from . import api
from .model import ObjectDesc


def _quat_mul(a, b):
    return np.array([a[0] * b[0] - a[1] * b[1] - a[2] * b[2] - a[3] * b[3],
                     a[0] * b[1] + a[1] * b[0] + a[2] * b[3] - a[3] * b[2],
                     a[0] * b[2] - a[1] * b[3] + a[2] * b[0] + a[3] * b[1],
                     a[0] * b[3] + a[1] * b[2] - a[2] * b[1] + a[3] * b[0]])


def _rot(q):
    w, x, y, z = q
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


def scene_states(obj: ObjectDesc, seeds) -> np.ndarray:
    """[S, 13] initial RigidState rows (x, theta w,x,y,z, xdot, thetadot)."""
    seeds = np.atleast_1d(np.asarray(seeds, np.int64))
    rb = obj.bounding_radius()
    out = np.zeros((seeds.size, 13))
    for k, s in enumerate(seeds):
        rng = np.random.Generator(np.random.Philox(key=int(s), counter=0))
        q = rng.normal(size=4)
        q /= np.linalg.norm(q)
        if q[0] < 0:
            q = -q
        out[k, 0:3] = [0.0, 0.0, 2.0 * rb]
        out[k, 3:7] = q
    return out


@dataclass
class Scenes:
    seeds: np.ndarray
    state: np.ndarray     # [S, 13] rest RigidState
    steps: np.ndarray     # [S] simulated steps
    ke: np.ndarray        # [S] final kinetic energy (J)
    at_rest: np.ndarray   # [S] bool: stopped by the rest rule (not the 5 s cap)
    stats: np.ndarray     # [S, 4] active contacts, corrections, singular, max penetration


def generate_scenes(ctx: api.Context, gobj: api.GraspObject, seeds, params: api.DropParams | None = None,
                    strict: bool = False) -> Scenes:
    """Drop every seed's scene. A scene that hits the step cap is not at rest
    (SPEC.md:541 asks for an error): ``strict=True`` raises RuntimeError naming
    seed, steps and kinetic energy; otherwise it is returned with
    at_rest=False and ``transfer_grasps`` rejects its grasps."""
    params = params or api.DropParams(max_steps=5000, ke_tol=1e-6, measure_residual=True)
    seeds = np.atleast_1d(np.asarray(seeds, np.int64))
    r = api.drop(ctx, gobj, scene_states(gobj.desc, seeds), params)
    at_rest = np.asarray(r["steps"]) < params.max_steps
    if strict and not np.all(at_rest):
        bad = [(int(seeds[k]), int(r["steps"][k]), float(r["ke"][k])) for k in np.nonzero(~at_rest)[0]]
        raise RuntimeError("scene not at rest after the step cap: " +
                           ", ".join(f"seed {s}: {n} steps, KE {e:.3e} J" for s, n, e in bad))
    return Scenes(seeds, r["state"], r["steps"], r["ke"], at_rest, r["stats"])


def object_origin(state: np.ndarray, com: np.ndarray) -> np.ndarray:
    """frame_origin (rigid.hpp:47-49): canonical-frame origin x - R com."""
    return state[0:3] - _rot(state[3:7]) @ com


def transfer_q(q_base: np.ndarray, state: np.ndarray, com: np.ndarray) -> np.ndarray:
    """Hand config in the scene: base pose composed with the object's pose
    (canonical -> scene: p -> R p + origin; orientation theta (x) q), joints
    unchanged."""
    q = np.array(q_base, np.float64, copy=True)
    R = _rot(state[3:7])
    q[0:3] = R @ q_base[0:3] + object_origin(state, com)
    qq = _quat_mul(state[3:7], q_base[3:7])
    q[3:7] = qq / np.linalg.norm(qq)
    return q


def transfer_grasps(ctx: api.Context, hand: api.Hand, obj: ObjectDesc, q_base: np.ndarray, scenes: Scenes,
                    table_clearance: float = 0.0, allow_unsettled: bool = False):
    """All (grasp, scene) pairs: (q [G, S, 7+J], accepted [G, S], min hand z [G, S]).
    Grasps into a scene that never came to rest are rejected unless
    ``allow_unsettled``."""
    G, S = q_base.shape[0], scenes.state.shape[0]
    qs = np.stack([[transfer_q(q_base[g], scenes.state[s], obj.com) for s in range(S)] for g in range(G)])
    pts = api.forward(ctx, hand, qs.reshape(G * S, -1))      # GPU forward kinematics
    zmin = pts[:, :, 2].min(axis=1).reshape(G, S)
    ok = zmin >= -table_clearance
    if not allow_unsettled:
        ok &= np.asarray(scenes.at_rest, bool)[None, :]
    return qs, ok, zmin


def _fmt(v):
    """9 significant digits; non-finite values are rejected (NaN / Infinity are
    not JSON)."""
    if isinstance(v, dict):
        return {k: _fmt(v[k]) for k in v}
    if isinstance(v, (list, tuple, np.ndarray)):
        return [_fmt(x) for x in np.asarray(v).tolist()]
    if isinstance(v, (float, np.floating)):
        if not np.isfinite(v):
            raise ValueError(f"export: non-finite value {v}")
        return float(f"{float(v):.9g}")
    if isinstance(v, (int, np.integer)):
        return int(v)
    return v


def export_jsonl(records: list, out_dir: str, config: dict | None = None, limits: dict | None = None) -> dict:
    """records: dicts with hand, object, q [7+J], losses{}, metrics{}, scene{}.
    Writes <out_dir>/<hand>__<object>.jsonl per pair and manifest.json.
    ``limits`` {hand: (lower [J], upper [J])}: every exported record must have
    its joints within the hand's limits, else ValueError;
    non-finite values are rejected."""
    for r in records:
        if limits and r["hand"] in limits:
            lo, hi = (np.asarray(x, np.float64) for x in limits[r["hand"]])
            j = np.asarray(r["q"], np.float64)[7:]
            if j.shape != lo.shape or np.any(j < lo) or np.any(j > hi):
                raise ValueError(f"export: {r['hand']} record outside its joint limits")
    os.makedirs(out_dir, exist_ok=True)
    groups: dict = {}
    for r in records:
        groups.setdefault((r["hand"], r["object"]), []).append(r)
    files = {}
    for (h, o), rs in sorted(groups.items()):
        name = f"{h}__{o}.jsonl"
        with open(os.path.join(out_dir, name), "w", encoding="utf-8") as fh:
            for r in rs:
                q = np.asarray(r["q"], np.float64)
                line = {"hand": h, "object": o, "base_position": _fmt(q[0:3]), "base_quaternion": _fmt(q[3:7]),
                        "joint_angles": _fmt(q[7:]), "losses": _fmt(r.get("losses", {})),
                        "metrics": _fmt(r.get("metrics", {})), "scene": _fmt(r.get("scene", {}))}
                fh.write(json.dumps(line, separators=(",", ":")) + "\n")
        files[name] = len(rs)
    cfg = json.dumps(_fmt(config or {}), sort_keys=True)
    manifest = {"count": sum(files.values()), "files": files,
                "config_hash": hashlib.sha256(cfg.encode()).hexdigest()}
    with open(os.path.join(out_dir, "manifest.json"), "w", encoding="utf-8") as fh:
        json.dump(manifest, fh, indent=1, sort_keys=True)
    return manifest


def import_jsonl(path: str) -> list:
    with open(path, encoding="utf-8") as fh:
        return [json.loads(line) for line in fh]
