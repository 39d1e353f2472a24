"""Author the 4-finger (Allegro-style, 16 DOF) and 5-finger (Shadow-style,
22 DOF) hands for BASELINE configs 2-3 in the reference's own description
format (HandModel::load_xml subset, hand.hpp:55-60: <robot><link><mesh/>
</link><joint type="revolute"><parent/><child/><origin xyz rpy/><axis/>
<limit/></joint></robot>, OBJ link meshes). The reference has only barrett3
and pincher2 (assets.cpp:235-300); these files let the UNMODIFIED reference
loader build the same hands the GPU uses.

Conventions follow assets.cpp: palm centred at its origin with +z the
approach axis, finger link boxes spanning z in [0, L] from their joint, box
winding as make_box (assets.cpp:28-41). Flexion axes are chosen so positive
angles curl fingers over the palm toward the opposing digit.

Usage: python tools/make_hands.py  (writes assets/hands/<name>/)
"""
from __future__ import annotations

import math
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "assets", "hands")

# make_box face list (assets.cpp:33-38), 0-based
_BOX_FACES = [(0, 2, 1), (0, 3, 2), (4, 5, 6), (4, 6, 7), (0, 1, 5), (0, 5, 4),
              (2, 3, 7), (2, 7, 6), (1, 2, 6), (1, 6, 5), (3, 0, 4), (3, 4, 7)]


def box_obj(sx: float, sy: float, sz: float, z0: float) -> str:
    hx, hy = 0.5 * sx, 0.5 * sy
    zl, zh = z0, z0 + sz
    v = [(-hx, -hy, zl), (hx, -hy, zl), (hx, hy, zl), (-hx, hy, zl),
         (-hx, -hy, zh), (hx, -hy, zh), (hx, hy, zh), (-hx, hy, zh)]
    lines = [f"v {x:.9g} {y:.9g} {z:.9g}" for (x, y, z) in v]
    lines += [f"f {a + 1} {b + 1} {c + 1}" for (a, b, c) in _BOX_FACES]
    return "\n".join(lines) + "\n"


class Spec:
    def __init__(self, name: str):
        self.name = name
        self.links: list[tuple[str, str]] = []   # (name, obj text)
        self.joints: list[dict] = []

    def link(self, name: str, sx: float, sy: float, sz: float, z0: float) -> None:
        self.links.append((name, box_obj(sx, sy, sz, z0)))

    def joint(self, name, parent, child, xyz, rpy, axis, lower, upper) -> None:
        self.joints.append(dict(name=name, parent=parent, child=child, xyz=xyz, rpy=rpy, axis=axis,
                                lower=lower, upper=upper))

    def write(self, root: str) -> str:
        d = os.path.join(root, self.name)
        os.makedirs(d, exist_ok=True)
        for n, obj in self.links:
            with open(os.path.join(d, n + ".obj"), "w") as f:
                f.write(obj)
        out = [f'<robot name="{self.name}">']
        for n, _ in self.links:
            out.append(f'  <link name="{n}"><mesh filename="{n}.obj"/></link>')
        for j in self.joints:
            out.append(f'  <joint name="{j["name"]}" type="revolute">')
            out.append(f'    <parent link="{j["parent"]}"/>')
            out.append(f'    <child link="{j["child"]}"/>')
            out.append('    <origin xyz="%.9g %.9g %.9g" rpy="%.9g %.9g %.9g"/>' % (*j["xyz"], *j["rpy"]))
            out.append('    <axis xyz="%.9g %.9g %.9g"/>' % tuple(j["axis"]))
            out.append('    <limit lower="%.9g" upper="%.9g"/>' % (j["lower"], j["upper"]))
            out.append("  </joint>")
        out.append("</robot>")
        path = os.path.join(d, self.name + ".xml")
        with open(path, "w") as f:
            f.write("\n".join(out) + "\n")
        return path


def finger(s: Spec, fid: str, base_xyz, flex_axis, seg, width, spread_axis, limits, palm_top):
    """Chain palm -> base (abduction) -> proximal -> middle -> distal."""
    names = [f"{fid}_base", f"{fid}_prox", f"{fid}_mid", f"{fid}_dist"]
    lens = seg
    for n, L in zip(names, lens):
        s.link(n, width, width, L, 0.0)
    (a0, a1), (p0, p1), (m0, m1), (d0, d1) = limits
    s.joint(f"{fid}_abd", "palm", names[0], (base_xyz[0], base_xyz[1], palm_top), (0, 0, 0), spread_axis, a0, a1)
    s.joint(f"{fid}_mcp", names[0], names[1], (0, 0, lens[0]), (0, 0, 0), flex_axis, p0, p1)
    s.joint(f"{fid}_pip", names[1], names[2], (0, 0, lens[1]), (0, 0, 0), flex_axis, m0, m1)
    s.joint(f"{fid}_dip", names[2], names[3], (0, 0, lens[2]), (0, 0, 0), flex_axis, d0, d1)


def allegro16() -> Spec:
    s = Spec("allegro16")
    s.link("palm", 0.095, 0.10, 0.025, -0.0125)
    top = 0.0125
    seg = (0.0164, 0.054, 0.0384, 0.0427)
    lim = ((-0.47, 0.47), (-0.196, 1.61), (-0.174, 1.709), (-0.227, 1.618))
    for fid, x in (("index", -0.030), ("middle", 0.0), ("ring", 0.030)):
        finger(s, fid, (x, 0.035), (1, 0, 0), seg, 0.0196, (0, 1, 0), lim, top)
    # thumb: opposes the fingers from -y, flexes toward +y
    tseg = (0.0176, 0.0514, 0.054, 0.0423)
    tlim = ((0.263, 1.396), (-0.105, 1.163), (-0.189, 1.644), (-0.162, 1.719))
    finger(s, "thumb", (0.0, -0.035), (-1, 0, 0), tseg, 0.0196, (0, 0, 1), tlim, top)
    return s


def shadow22() -> Spec:
    s = Spec("shadow22")
    s.link("palm", 0.09, 0.10, 0.025, -0.0125)
    top = 0.0125
    seg = (0.010, 0.045, 0.025, 0.026)
    lim = ((-0.349, 0.349), (-0.262, 1.571), (0.0, 1.571), (0.0, 1.571))
    for fid, x in (("ff", -0.033), ("mf", -0.011), ("rf", 0.011)):
        finger(s, fid, (x, 0.035), (1, 0, 0), seg, 0.018, (0, 1, 0), lim, top)
    # little finger: extra metacarpal joint (LFJ5) in the palm
    s.link("lf_meta", 0.018, 0.018, 0.012, 0.0)
    s.joint("lf_j5", "palm", "lf_meta", (0.033, 0.030, top), (0, 0, 0), (0, 1, 0.3), 0.0, 0.785)
    names = ["lf_base", "lf_prox", "lf_mid", "lf_dist"]
    for n, L in zip(names, seg):
        s.link(n, 0.018, 0.018, L, 0.0)
    s.joint("lf_abd", "lf_meta", names[0], (0, 0.005, 0.012), (0, 0, 0), (0, 1, 0), *lim[0])
    s.joint("lf_mcp", names[0], names[1], (0, 0, seg[0]), (0, 0, 0), (1, 0, 0), *lim[1])
    s.joint("lf_pip", names[1], names[2], (0, 0, seg[1]), (0, 0, 0), (1, 0, 0), *lim[2])
    s.joint("lf_dip", names[2], names[3], (0, 0, seg[2]), (0, 0, 0), (1, 0, 0), *lim[3])
    # thumb: 5 joints (THJ5 rotation, THJ4 abduction, THJ3, THJ2, THJ1)
    th = ["th_base", "th_hub", "th_prox", "th_mid", "th_dist"]
    thl = (0.012, 0.010, 0.038, 0.030, 0.032)
    for n, L in zip(th, thl):
        s.link(n, 0.020, 0.020, L, 0.0)
    s.joint("th_j5", "palm", th[0], (-0.030, -0.030, top), (0, 0, math.pi / 4), (0, 0, 1), -1.047, 1.047)
    s.joint("th_j4", th[0], th[1], (0, 0, thl[0]), (0, 0, 0), (0, 1, 0), 0.0, 1.222)
    s.joint("th_j3", th[1], th[2], (0, 0, thl[1]), (0, 0, 0), (-1, 0, 0), -0.209, 0.209)
    s.joint("th_j2", th[2], th[3], (0, 0, thl[2]), (0, 0, 0), (-1, 0, 0), -0.698, 0.698)
    s.joint("th_j1", th[3], th[4], (0, 0, thl[3]), (0, 0, 0), (-1, 0, 0), -0.262, 1.571)
    return s


def main() -> None:
    for spec in (allegro16(), shadow22()):
        p = spec.write(OUT)
        print(p, len(spec.links), "links", len(spec.joints), "joints")


if __name__ == "__main__":
    main()
