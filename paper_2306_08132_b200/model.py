"""Hand and object descriptors consumed by the C-ABI (include/dgx.h).

* ``HandDesc`` — the data of a reference ``dg::HandModel`` (hand.hpp:53-102):
  revolute tree, BFS topological order, per-joint axis / origin (R, t) /
  limits, and the link-frame surface samples in ``forward()`` order
  (link-index major, hand.hpp:143-151) with ``sample_link``. Samples are NOT
  regenerated here: they come from the reference's area-weighted sampler
  (hand.cpp:42-68, libstdc++ mt19937_64), exported once into ``assets/hands``
  by ``tools/export_assets.py``.
* ``ObjectDesc`` — an SDF backend (analytic sphere / box, dense FP32 trilinear
  grid; see csrc/dgx_geom.h; or the reference's triangle-mesh MeshSdf,
  csrc/dgx_mesh.h) plus ``InertialData`` (rigid.hpp:8-13): mass, COM, body
  inertia and its inverse. Inertia is analytic for primitives, a voxel
  integral for grids and ``inertia_from_mesh`` (rigid.cpp:24-94, evaluated by
  the C-ABI's dgx_mesh_inertia) for meshes.
"""
from __future__ import annotations

import os
from dataclasses import dataclass, field

import numpy as np

ASSET_DIR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "assets")


@dataclass
class HandDesc:
    name: str
    topo: np.ndarray              # [L] int32, parent before child
    link_parent_joint: np.ndarray  # [L] int32, -1 for the base link
    joint_parent: np.ndarray      # [J] int32
    joint_child: np.ndarray       # [J] int32
    axis: np.ndarray              # [J,3]
    origin_R: np.ndarray          # [J,9] row-major
    origin_t: np.ndarray          # [J,3]
    lower: np.ndarray             # [J]
    upper: np.ndarray             # [J]
    samples: np.ndarray           # [N,3] link frame, forward() order
    sample_link: np.ndarray       # [N] int32
    sample_area: np.ndarray | None = None  # [N] m^2, HandModel::sample_areas (hand.hpp:77)

    @property
    def num_links(self) -> int:
        return int(self.topo.shape[0])

    @property
    def num_joints(self) -> int:
        return int(self.joint_parent.shape[0])

    @property
    def num_samples(self) -> int:
        return int(self.samples.shape[0])

    @property
    def q_dim(self) -> int:
        return 7 + self.num_joints

    @property
    def grad_dim(self) -> int:
        return 6 + self.num_joints

    def mid_range(self) -> np.ndarray:
        """hand.cpp:212-216."""
        return 0.5 * (self.lower + self.upper)

    @classmethod
    def from_dict(cls, name: str, d: dict) -> "HandDesc":
        return cls(
            name=name,
            topo=np.ascontiguousarray(d["topo"], np.int32),
            link_parent_joint=np.ascontiguousarray(d["link_parent_joint"], np.int32),
            joint_parent=np.ascontiguousarray(d["joint_parent"], np.int32),
            joint_child=np.ascontiguousarray(d["joint_child"], np.int32),
            axis=np.ascontiguousarray(d["axis"], np.float64).reshape(-1, 3),
            origin_R=np.ascontiguousarray(d["origin_R"], np.float64).reshape(-1, 9),
            origin_t=np.ascontiguousarray(d["origin_t"], np.float64).reshape(-1, 3),
            lower=np.ascontiguousarray(d["lower"], np.float64),
            upper=np.ascontiguousarray(d["upper"], np.float64),
            samples=np.ascontiguousarray(d["samples"], np.float64).reshape(-1, 3),
            sample_link=np.ascontiguousarray(d["sample_link"], np.int32),
            sample_area=np.ascontiguousarray(d["sample_area"], np.float64) if "sample_area" in d else None,
        )

    def to_dict(self) -> dict:
        d = {k: getattr(self, k) for k in ("topo", "link_parent_joint", "joint_parent", "joint_child", "axis",
                                            "origin_R", "origin_t", "lower", "upper", "samples", "sample_link")}
        if self.sample_area is not None:
            d["sample_area"] = self.sample_area
        return d

    def save(self, path: str) -> None:
        np.savez_compressed(path, name=np.array(self.name), **self.to_dict())

    @classmethod
    def load(cls, path: str) -> "HandDesc":
        z = np.load(path)
        return cls.from_dict(str(z["name"]), {k: z[k] for k in z.files if k != "name"})

    @classmethod
    def asset(cls, name: str) -> "HandDesc":
        """A hand exported from the reference into assets/hands/<name>.npz."""
        return cls.load(os.path.join(ASSET_DIR, "hands", f"{name}.npz"))


@dataclass
class ObjectDesc:
    kind: str                       # "sphere" | "box" | "grid" | "mesh"
    mass: float
    com: np.ndarray
    inertia_body: np.ndarray        # [3,3]
    inertia_body_inv: np.ndarray    # [3,3]
    center: np.ndarray = field(default_factory=lambda: np.zeros(3))
    radius: float = 0.0
    half_extents: np.ndarray = field(default_factory=lambda: np.zeros(3))
    dims: tuple = (0, 0, 0)         # grid nx, ny, nz (x fastest)
    origin: np.ndarray = field(default_factory=lambda: np.zeros(3))
    spacing: float = 0.0
    inv_spacing: float = 0.0
    values: np.ndarray | None = None  # [nz, ny, nx] float32
    name: str = ""
    vertices: np.ndarray | None = None        # mesh [V,3]
    faces: np.ndarray | None = None           # mesh [F,3] int32, outward winding
    vertex_normals: np.ndarray | None = None  # mesh [V,3] unit, or None: area-weighted (mesh.cpp:60-70)
    alpha_phong: float = 0.75                 # MeshSdf alpha (sdf.hpp:24, losses.hpp:42)

    def bounding_radius(self) -> float:
        if self.kind == "mesh":  # TriMesh::bounding_radius(com) (mesh.cpp:97-101)
            return float(np.sqrt(np.max(np.sum((self.vertices - self.com[None, :]) ** 2, axis=1))))
        if self.kind == "sphere":
            return float(self.radius)
        if self.kind == "box":
            return float(np.linalg.norm(self.half_extents))
        inside = np.argwhere(self.values <= 0.0)
        if inside.size == 0:
            return 0.0
        pts = self.origin[None, :] + inside[:, ::-1] * self.spacing
        return float(np.max(np.linalg.norm(pts - self.com[None, :], axis=1)))


def _inv3(I: np.ndarray) -> np.ndarray:
    return np.linalg.inv(I)


def sphere(radius: float, center=(0.0, 0.0, 0.0), density: float = 1000.0) -> ObjectDesc:
    """Solid sphere: m = rho 4/3 pi R^3, I = 2/5 m R^2."""
    c = np.asarray(center, np.float64)
    m = density * 4.0 / 3.0 * np.pi * radius ** 3
    I = np.eye(3) * (0.4 * m * radius * radius)
    return ObjectDesc("sphere", m, c.copy(), I, _inv3(I), center=c, radius=float(radius),
                      name=f"sphere_r{radius:g}")


def box(size, center=(0.0, 0.0, 0.0), density: float = 1000.0) -> ObjectDesc:
    s = np.asarray(size, np.float64)
    c = np.asarray(center, np.float64)
    m = density * float(np.prod(s))
    I = np.diag([m / 12.0 * (s[1] ** 2 + s[2] ** 2), m / 12.0 * (s[0] ** 2 + s[2] ** 2),
                 m / 12.0 * (s[0] ** 2 + s[1] ** 2)])
    return ObjectDesc("box", m, c.copy(), I, _inv3(I), center=c, half_extents=0.5 * s, name="box")


# ---- analytic SDFs used to bake grids (host, float64 → float32 nodes) -------

def sdf_box(p: np.ndarray, half: np.ndarray) -> np.ndarray:
    q = np.abs(p) - half
    outside = np.linalg.norm(np.maximum(q, 0.0), axis=-1)
    inside = np.minimum(np.max(q, axis=-1), 0.0)
    return outside + inside


def sdf_cylinder(p: np.ndarray, radius: float, half_height: float) -> np.ndarray:
    d = np.stack([np.linalg.norm(p[..., :2], axis=-1) - radius, np.abs(p[..., 2]) - half_height], axis=-1)
    return np.minimum(np.max(d, axis=-1), 0.0) + np.linalg.norm(np.maximum(d, 0.0), axis=-1)


def sdf_blob(p: np.ndarray, radius: float, amplitude: float, seed: int) -> np.ndarray:
    """Smooth star-shaped procedural body (make_blob-like lobes, assets.cpp:138-164):
    r(d) = R (1 + A f(d)/6), f = sum of 4 random quadratic lobes; the field is the
    radial distance |p| - r(p/|p|) scaled by a Lipschitz bound (not exact
    Euclidean distance, but a smooth SDF-like field with the right zero set)."""
    rng = np.random.Generator(np.random.Philox(seed))
    u = rng.uniform(-1.0, 1.0, size=(4, 3))
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    ab = rng.uniform(-1.0, 1.0, size=(4, 2))
    n = np.linalg.norm(p, axis=-1)
    d = p / np.maximum(n, 1e-12)[..., None]
    c = d @ u.T
    f = np.sum(ab[:, 0] * c * c + ab[:, 1] * c, axis=-1)
    rr = radius * (1.0 + amplitude * f / 6.0)
    return (n - rr) / (1.0 + amplitude)


def grid_object(sdf_fn, lo, hi, res: int, density: float = 1000.0, name: str = "grid",
                inertial: ObjectDesc | None = None) -> ObjectDesc:
    """Bake ``sdf_fn`` on a res^3 node grid spanning [lo, hi] (cubic cells).

    Inertia: taken from ``inertial`` (the analytic primitive the grid samples)
    when given, else a voxel integral over nodes with phi <= 0."""
    lo = np.asarray(lo, np.float64)
    hi = np.asarray(hi, np.float64)
    h = float(np.max(hi - lo) / (res - 1))
    xs = lo[0] + h * np.arange(res)
    ys = lo[1] + h * np.arange(res)
    zs = lo[2] + h * np.arange(res)
    Z, Y, X = np.meshgrid(zs, ys, xs, indexing="ij")
    P = np.stack([X, Y, Z], axis=-1)
    vals = np.ascontiguousarray(sdf_fn(P), np.float32)
    if inertial is not None:
        mass, com, I = inertial.mass, inertial.com.copy(), inertial.inertia_body.copy()
    else:
        inside = vals <= 0.0
        pts = P[inside]
        dv = h ** 3
        mass = density * dv * pts.shape[0]
        com = pts.mean(axis=0)
        r = pts - com
        I = density * dv * (np.eye(3) * np.sum(r * r) - r.T @ r)
    return ObjectDesc("grid", float(mass), np.asarray(com, np.float64), I, _inv3(I), dims=(res, res, res),
                      origin=lo.copy(), spacing=h, inv_spacing=1.0 / h, values=vals, name=name)


def box_grid(size=(0.04, 0.04, 0.04), res: int = 64, margin: float = 0.03, density: float = 1000.0):
    """Config 2: 40 mm box SDF sampled on res^3 over bounds + 30 mm."""
    s = np.asarray(size, np.float64)
    ref = box(s, density=density)
    half = 0.5 * s
    return grid_object(lambda P: sdf_box(P, half), -half - margin, half + margin, res, density,
                       f"box{res}", inertial=ref)


def cylinder_grid(radius=0.0175, height=0.07, res: int = 64, margin: float = 0.03, density: float = 1000.0):
    """Config 2: cylinder r 17.5 mm, h 70 mm (assets.cpp:316) on res^3 over bounds + 30 mm."""
    m = density * np.pi * radius ** 2 * height
    Ixx = m * (3 * radius ** 2 + height ** 2) / 12.0
    I = np.diag([Ixx, Ixx, 0.5 * m * radius ** 2])
    ref = ObjectDesc("grid", m, np.zeros(3), I, _inv3(I))
    half = np.array([radius, radius, 0.5 * height])
    ext = float(np.max(half)) + margin
    return grid_object(lambda P: sdf_cylinder(P, radius, 0.5 * height), -np.full(3, ext), np.full(3, ext), res,
                       density, f"cyl{res}", inertial=ref)


def blob_grid(seed: int, radius=0.021, amplitude=0.5, res: int = 128, margin: float = 0.03,
              density: float = 1000.0):
    """Config 3/4: procedural blob baked on res^3 (voxel inertia)."""
    ext = radius * (1.0 + amplitude) + margin
    return grid_object(lambda P: sdf_blob(P, radius, amplitude, seed), -np.full(3, ext), np.full(3, ext), res,
                       density, f"blob{seed}_{res}")


# ---------------------------------------------------------------------------
# triangle meshes (dg::TriMesh, mesh.hpp:15-45)
# ---------------------------------------------------------------------------
def mesh_object(vertices, faces, density: float = 1000.0, alpha_phong: float = 0.75, vertex_normals=None,
                name: str = "mesh") -> ObjectDesc:
    """dg::GraspObject(TriMesh, density, alpha_phong) (losses.hpp:42-43): the
    mesh SDF plus inertia_from_mesh (rigid.cpp:24-94) through dgx_mesh_inertia,
    which also validates the mesh as TriMesh::finalize (mesh.cpp:12-71)."""
    import ctypes as C

    from . import capi
    V = np.ascontiguousarray(vertices, np.float64).reshape(-1, 3)
    F = np.ascontiguousarray(faces, np.int32).reshape(-1, 3)
    mass, com, I, Iinv = C.c_double(), np.zeros(3), np.zeros(9), np.zeros(9)
    L = capi.load()
    capi.check(L.dgx_mesh_inertia(V.shape[0], capi.ptr(V), F.shape[0], capi.ptr(F), float(density), C.byref(mass),
                                  com.ctypes.data_as(capi._dp), I.ctypes.data_as(capi._dp),
                                  Iinv.ctypes.data_as(capi._dp)))
    vn = None if vertex_normals is None else np.ascontiguousarray(vertex_normals, np.float64).reshape(-1, 3)
    return ObjectDesc("mesh", float(mass.value), com, I.reshape(3, 3), Iinv.reshape(3, 3), name=name, vertices=V,
                      faces=F, vertex_normals=vn, alpha_phong=float(alpha_phong))


def icosphere_mesh(radius: float = 0.025, subdivisions: int = 3) -> tuple[np.ndarray, np.ndarray]:
    """Geodesic sphere: the regular icosahedron split 4:1 per level, vertices
    pushed to the sphere (20 * 4^s faces; s = 3 -> 1280 faces, the size of
    SURVEY config 1's mesh cross-check)."""
    g = (1.0 + 5.0 ** 0.5) / 2.0
    V = [np.array(v, np.float64) for v in
         [(-1, g, 0), (1, g, 0), (-1, -g, 0), (1, -g, 0), (0, -1, g), (0, 1, g), (0, -1, -g), (0, 1, -g),
          (g, 0, -1), (g, 0, 1), (-g, 0, -1), (-g, 0, 1)]]
    F = [(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11), (1, 5, 9), (5, 11, 4), (11, 10, 2),
         (10, 7, 6), (7, 1, 8), (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9), (4, 9, 5), (2, 4, 11),
         (6, 2, 10), (8, 6, 7), (9, 8, 1)]
    for _ in range(subdivisions):
        mids: dict = {}

        def mid(a, b):
            k = (a, b) if a < b else (b, a)
            if k not in mids:
                V.append(0.5 * (V[a] + V[b]))
                mids[k] = len(V) - 1
            return mids[k]

        nxt = []
        for a, b, c in F:
            ab, bc, ca = mid(a, b), mid(b, c), mid(c, a)
            nxt += [(a, ab, ca), (b, bc, ab), (c, ca, bc), (ab, bc, ca)]
        F = nxt
    P = np.array(V)
    n = np.sqrt(P[:, 0] * P[:, 0] + P[:, 1] * P[:, 1] + P[:, 2] * P[:, 2])
    P = radius * (P / n[:, None])
    return P, np.array(F, np.int32)


def box_mesh(size=(0.04, 0.04, 0.04)) -> tuple[np.ndarray, np.ndarray]:
    """Axis-aligned box centred at the origin, 12 outward-wound triangles."""
    h = 0.5 * np.asarray(size, np.float64)
    V = np.array([[sx * h[0], sy * h[1], sz * h[2]] for sz in (-1, 1) for sy in (-1, 1) for sx in (-1, 1)])
    # vertex id = x + 2y + 4z (bits)
    quads = [(0, 2, 3, 1), (4, 5, 7, 6), (0, 1, 5, 4), (2, 6, 7, 3), (0, 4, 6, 2), (1, 3, 7, 5)]
    F = []
    for a, b, c, d in quads:
        F += [(a, b, c), (a, c, d)]
    return V, np.array(F, np.int32)


def load_obj(path: str) -> tuple[np.ndarray, np.ndarray]:
    """ASCII OBJ v/f records as dg::load_obj (mesh.cpp:112-151): vertex index
    before the first '/', negative indices relative, polygons fan-triangulated,
    other records ignored."""
    V, F = [], []
    with open(path) as fh:
        for ln, line in enumerate(fh, 1):
            tok = line.split()
            if not tok or tok[0].startswith("#"):
                continue
            if tok[0] == "v":
                try:
                    V.append([float(t) for t in tok[1:4]])
                except ValueError:
                    raise RuntimeError(f"{path}:{ln}: malformed vertex") from None
                if len(V[-1]) != 3:
                    raise RuntimeError(f"{path}:{ln}: malformed vertex")
            elif tok[0] == "f":
                idx = []
                for t in tok[1:]:
                    try:
                        i = int(t.split("/")[0])
                    except ValueError:
                        raise RuntimeError(f"{path}:{ln}: malformed face index '{t}'") from None
                    if i < 0:
                        i = len(V) + i + 1
                    if i <= 0 or i > len(V):
                        raise RuntimeError(f"{path}:{ln}: face index out of range")
                    idx.append(i - 1)
                if len(idx) < 3:
                    raise RuntimeError(f"{path}:{ln}: face with fewer than 3 vertices")
                F += [(idx[0], idx[k], idx[k + 1]) for k in range(1, len(idx) - 1)]
    if not F:
        raise RuntimeError(f"{path}: no faces found")
    return np.array(V, np.float64), np.array(F, np.int32)
