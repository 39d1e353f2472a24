"""oracle/ref.py — TEST INFRASTRUCTURE ONLY: ctypes access to the compiled
reference (oracle/_ref/libdgref*.so, built by oracle/Makefile from the
unmodified /root/reference/proj sources plus oracle/ref_shim.cpp).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this
module; it is the parity checker, never the product path.

Two builds:
  * ``libdgref.so``    — the reference exactly, glibc libm ("reference").
  * ``libdgref_sm.so`` — the same objects with sin/cos/sincos/atan2 bound to
    the deterministic shared math the kernels use (parity mode P).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(_HERE, "_ref")
_libs: dict[str, C.CDLL] = {}

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_fp = C.POINTER(C.c_float)


class Params(C.Structure):
    """ref_shim.cpp:Params — SimParams + StabilityProtocol::standard + LossWeights."""

    _fields_ = [
        ("dt", C.c_double), ("mu", C.c_double), ("gs_iters", C.c_int), ("steps", C.c_int),
        ("dilation_radius", C.c_double), ("alpha_leak", C.c_double), ("speed", C.c_double),
        ("w_stable", C.c_double), ("w_qrange", C.c_double), ("w_qlimit", C.c_double),
    ]


class OptCfg(C.Structure):
    _fields_ = [
        ("iters", C.c_int), ("k_begin", C.c_int), ("k_end", C.c_int), ("pad", C.c_int),
        ("r0", C.c_double), ("lr", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double),
        ("eps", C.c_double),
    ]


def default_params(**kw) -> Params:
    """Reference defaults: sim.hpp:33-40, losses.hpp:21-35."""
    p = Params(dt=0.001, mu=1.0, gs_iters=8, steps=1, dilation_radius=0.0, alpha_leak=0.1,
               speed=0.5, w_stable=1.0, w_qrange=0.01, w_qlimit=1.0)
    for k, v in kw.items():
        setattr(p, k, v)
    return p


def available(variant: str = "sm") -> bool:
    name = "libdgref_sm.so" if variant == "sm" else "libdgref.so"
    return os.path.exists(os.path.join(REF_DIR, name))


def lib(variant: str = "sm") -> C.CDLL:
    if variant in _libs:
        return _libs[variant]
    name = "libdgref_sm.so" if variant == "sm" else "libdgref.so"
    path = os.path.join(REF_DIR, name)
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} missing: run `make -C oracle` (needs /root/reference)")
    L = C.CDLL(path, mode=C.RTLD_LOCAL)
    vp = C.c_void_p
    L.dgr_last_error.restype = C.c_char_p
    for fn in ("dgr_hand_barrett3", "dgr_hand_pincher2"):
        getattr(L, fn).restype = vp
        getattr(L, fn).argtypes = [C.c_int, C.c_uint64]
    L.dgr_hand_load_xml.restype = vp
    L.dgr_hand_load_xml.argtypes = [C.c_char_p, C.c_int, C.c_uint64]
    L.dgr_hand_free.argtypes = [vp]
    L.dgr_hand_dims.argtypes = [vp, _ip]
    L.dgr_hand_export.argtypes = [vp, _ip, _ip, _ip, _ip, _dp, _dp, _dp, _dp, _dp, _dp, _ip]
    L.dgr_hand_forward.argtypes = [vp, _dp, _dp]
    L.dgr_hand_sample_areas.argtypes = [vp, _dp]
    L.dgr_object_mesh.restype = vp
    L.dgr_object_mesh.argtypes = [_dp, C.c_int, _ip, C.c_int, C.c_double, C.c_double]
    L.dgr_object_icosphere.restype = vp
    L.dgr_object_icosphere.argtypes = [C.c_double, C.c_int, C.c_double, C.c_double]
    L.dgr_object_box_mesh.restype = vp
    L.dgr_object_box_mesh.argtypes = [C.c_double] * 5
    L.dgr_object_cylinder_mesh.restype = vp
    L.dgr_object_cylinder_mesh.argtypes = [C.c_double, C.c_double, C.c_int, C.c_double, C.c_double]
    L.dgr_object_blob_mesh.restype = vp
    L.dgr_object_blob_mesh.argtypes = [C.c_double, C.c_int, C.c_double, C.c_uint64, C.c_double, C.c_double]
    L.dgr_object_free.argtypes = [vp]
    L.dgr_object_mesh_dims.argtypes = [vp, _ip]
    L.dgr_object_mesh_export.argtypes = [vp, _dp, _ip, _dp]
    L.dgr_object_bvh.argtypes = [vp, _dp, _ip, _ip, C.c_int]
    L.dgr_object_query_within.argtypes = [vp, _dp, C.c_double, _dp]
    L.dgr_drop.argtypes = [vp, _dp, C.c_double, C.c_double, C.c_int, _dp, C.c_int, C.c_int, C.c_double, C.c_int,
                           _dp, _ip, _dp, _dp, _dp, C.c_int, C.c_int]
    L.dgr_set_protocol.argtypes = [C.c_int, _dp]
    L.dgr_debug_step_adjoint.argtypes = [vp, vp, _dp, C.c_int, C.POINTER(Params), _dp]
    L.dgr_object_use_sphere.argtypes = [vp, C.c_double, C.c_double, C.c_double, C.c_double]
    L.dgr_object_use_box.argtypes = [vp, _dp, _dp]
    L.dgr_object_use_grid.argtypes = [vp, _ip, _dp, C.c_double, C.c_double, _fp]
    L.dgr_object_set_inertial.argtypes = [vp, C.c_double, _dp, _dp, _dp]
    L.dgr_object_get_inertial.argtypes = [vp, _dp, _dp, _dp, _dp]
    L.dgr_object_query.argtypes = [vp, _dp, C.c_double, _dp]
    L.dgr_loss_gradient.argtypes = [vp, vp, _dp, C.POINTER(Params), _dp, _dp, _dp, _dp]
    L.dgr_evaluate_losses.argtypes = [vp, vp, _dp, C.POINTER(Params), _dp]
    L.dgr_apply_gradient_step.argtypes = [vp, _dp, _dp, C.c_double, _dp]
    L.dgr_sim_record.argtypes = [vp, vp, _dp, C.c_int, C.POINTER(Params), _dp, _dp, _dp, _dp, C.c_int, _ip]
    L.dgr_sim_forward.argtypes = [vp, vp, _dp, C.c_int, C.POINTER(Params), C.c_int, _dp, _dp, _dp,
                                  C.c_int, _ip]
    L.dgr_optimize.argtypes = [vp, vp, C.c_int, _dp, _dp, _dp, C.POINTER(Params), C.POINTER(OptCfg),
                               C.c_int, _dp, _dp, _ip]
    _libs[variant] = L
    return L


def _d(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _i(a: np.ndarray):
    return a.ctypes.data_as(_ip)


class RefError(RuntimeError):
    pass


def _check(L, rc: int):
    if rc != 0:
        raise RefError(L.dgr_last_error().decode())


@dataclass
class RefHand:
    """A reference HandModel plus its exported descriptor (hand.hpp:53-102)."""

    L: C.CDLL
    ptr: int
    num_links: int = 0
    num_joints: int = 0
    num_samples: int = 0
    desc: dict = field(default_factory=dict)

    @classmethod
    def _wrap(cls, L, ptr):
        if not ptr:
            raise RefError(L.dgr_last_error().decode())
        dims = np.zeros(3, np.int32)
        L.dgr_hand_dims(ptr, _i(dims))
        h = cls(L, ptr, int(dims[0]), int(dims[1]), int(dims[2]))
        Lk, J, N = h.num_links, h.num_joints, h.num_samples
        d = dict(
            topo=np.zeros(Lk, np.int32), link_parent_joint=np.zeros(Lk, np.int32),
            joint_parent=np.zeros(J, np.int32), joint_child=np.zeros(J, np.int32),
            axis=np.zeros((J, 3)), origin_R=np.zeros((J, 9)), origin_t=np.zeros((J, 3)),
            lower=np.zeros(J), upper=np.zeros(J), samples=np.zeros((N, 3)),
            sample_link=np.zeros(N, np.int32),
        )
        L.dgr_hand_export(ptr, _i(d["topo"]), _i(d["link_parent_joint"]), _i(d["joint_parent"]),
                          _i(d["joint_child"]), _d(d["axis"]), _d(d["origin_R"]), _d(d["origin_t"]),
                          _d(d["lower"]), _d(d["upper"]), _d(d["samples"]), _i(d["sample_link"]))
        d["sample_area"] = np.zeros(N)
        L.dgr_hand_sample_areas(ptr, _d(d["sample_area"]))
        h.desc = d
        return h

    @classmethod
    def barrett3(cls, budget=2000, seed=12345, variant="sm"):
        L = lib(variant)
        return cls._wrap(L, L.dgr_hand_barrett3(budget, seed))

    @classmethod
    def pincher2(cls, budget=2000, seed=12345, variant="sm"):
        L = lib(variant)
        return cls._wrap(L, L.dgr_hand_pincher2(budget, seed))

    @classmethod
    def load_xml(cls, path, budget=2000, seed=12345, variant="sm"):
        L = lib(variant)
        return cls._wrap(L, L.dgr_hand_load_xml(str(path).encode(), budget, seed))

    def __del__(self):
        try:
            if self.ptr:
                self.L.dgr_hand_free(self.ptr)
                self.ptr = 0
        except Exception:
            pass

    def forward(self, q) -> np.ndarray:
        q = np.ascontiguousarray(q, np.float64)
        out = np.zeros((self.num_samples, 3))
        _check(self.L, self.L.dgr_hand_forward(self.ptr, _d(q), _d(out)))
        return out


class RefObject:
    """dg::GraspObject with the AnySdf backend selected (ref_shim.cpp)."""

    def __init__(self, L, ptr):
        if not ptr:
            raise RefError(L.dgr_last_error().decode())
        self.L, self.ptr = L, ptr

    def __del__(self):
        try:
            if self.ptr:
                self.L.dgr_object_free(self.ptr)
                self.ptr = 0
        except Exception:
            pass

    @classmethod
    def icosphere(cls, radius, subdiv, density=1000.0, alpha=0.75, variant="sm"):
        L = lib(variant)
        return cls(L, L.dgr_object_icosphere(radius, subdiv, density, alpha))

    @classmethod
    def box_mesh(cls, sx, sy, sz, density=1000.0, alpha=0.75, variant="sm"):
        L = lib(variant)
        return cls(L, L.dgr_object_box_mesh(sx, sy, sz, density, alpha))

    @classmethod
    def cylinder_mesh(cls, radius, height, segments, density=1000.0, alpha=0.75, variant="sm"):
        L = lib(variant)
        return cls(L, L.dgr_object_cylinder_mesh(radius, height, segments, density, alpha))

    @classmethod
    def blob_mesh(cls, radius, subdiv, amplitude, seed, density=1000.0, alpha=0.75, variant="sm"):
        L = lib(variant)
        return cls(L, L.dgr_object_blob_mesh(radius, subdiv, amplitude, seed, density, alpha))

    @classmethod
    def mesh(cls, V, F, density=1000.0, alpha=0.75, variant="sm"):
        L = lib(variant)
        V = np.ascontiguousarray(V, np.float64)
        F = np.ascontiguousarray(F, np.int32)
        return cls(L, L.dgr_object_mesh(_d(V), V.shape[0], _i(F), F.shape[0], density, alpha))

    def mesh_export(self):
        """(vertices [V,3], faces [F,3] int32, vertex_normals [V,3]) of the object's TriMesh."""
        dims = np.zeros(2, np.int32)
        self.L.dgr_object_mesh_dims(self.ptr, _i(dims))
        V, F, VN = np.zeros((dims[0], 3)), np.zeros((dims[1], 3), np.int32), np.zeros((dims[0], 3))
        self.L.dgr_object_mesh_export(self.ptr, _d(V), _i(F), _d(VN))
        return V, F, VN

    def bvh(self):
        """The reference Bvh: boxes [n,6] (lo, hi), links [n,4] (left, right, first, count), face_order."""
        dims = np.zeros(2, np.int32)
        self.L.dgr_object_mesh_dims(self.ptr, _i(dims))
        cap = 2 * int(dims[1]) + 1
        boxes, links, fo = np.zeros((cap, 6)), np.zeros((cap, 4), np.int32), np.zeros(int(dims[1]), np.int32)
        n = self.L.dgr_object_bvh(self.ptr, _d(boxes), _i(links), _i(fo), cap)
        return boxes[:n], links[:n], fo

    def query_within(self, r, radius=0.0):
        r = np.ascontiguousarray(r, np.float64)
        out = np.zeros(8)
        _check(self.L, self.L.dgr_object_query_within(self.ptr, _d(r), radius, _d(out)))
        return out

    @classmethod
    def from_desc(cls, desc, variant="sm"):
        """Non-mesh backend from a paper_2306_08132_b200 ObjectDesc, with its inertia."""
        L = lib(variant)
        o = cls(L, L.dgr_object_icosphere(0.02, 1, 1000.0, 0.75))  # placeholder mesh
        kind = desc.kind
        if kind == "sphere":
            c = desc.center
            L.dgr_object_use_sphere(o.ptr, c[0], c[1], c[2], desc.radius)
        elif kind == "box":
            c = np.ascontiguousarray(desc.center, np.float64)
            h = np.ascontiguousarray(desc.half_extents, np.float64)
            L.dgr_object_use_box(o.ptr, _d(c), _d(h))
        elif kind == "mesh":  # the UNMODIFIED reference MeshSdf over the same TriMesh
            if desc.vertex_normals is not None:
                raise ValueError("explicit vertex normals are not plumbed into the oracle")
            o = cls.mesh(desc.vertices, desc.faces, 1000.0, desc.alpha_phong, variant)
        elif kind == "grid":
            dims = np.ascontiguousarray(desc.dims, np.int32)
            org = np.ascontiguousarray(desc.origin, np.float64)
            vals = np.ascontiguousarray(desc.values, np.float32)
            L.dgr_object_use_grid(o.ptr, _i(dims), _d(org), desc.spacing, desc.inv_spacing,
                                  vals.ctypes.data_as(_fp))
        else:
            raise ValueError(kind)
        o.set_inertial(desc.mass, desc.com, desc.inertia_body, desc.inertia_body_inv)
        return o

    def set_inertial(self, mass, com, I, Iinv):
        com = np.ascontiguousarray(com, np.float64)
        I = np.ascontiguousarray(I, np.float64).reshape(9)
        Iinv = np.ascontiguousarray(Iinv, np.float64).reshape(9)
        self.L.dgr_object_set_inertial(self.ptr, mass, _d(com), _d(I), _d(Iinv))

    def inertial(self):
        m = C.c_double()
        com, I, Iinv = np.zeros(3), np.zeros(9), np.zeros(9)
        self.L.dgr_object_get_inertial(self.ptr, C.byref(m), _d(com), _d(I), _d(Iinv))
        return m.value, com, I.reshape(3, 3), Iinv.reshape(3, 3)

    def query(self, r, radius=0.0):
        r = np.ascontiguousarray(r, np.float64)
        out = np.zeros(8)
        _check(self.L, self.L.dgr_object_query(self.ptr, _d(r), radius, _d(out)))
        return out


class protocol:
    """Context manager: every oracle call inside uses StabilityProtocol with
    these velocities [M,3] (and params.steps) instead of standard(speed)."""

    def __init__(self, velocities, variant="sm"):
        self.v = np.ascontiguousarray(np.asarray(velocities, np.float64).reshape(-1, 3))
        self.L = lib(variant)

    def __enter__(self):
        self.L.dgr_set_protocol(self.v.shape[0], _d(self.v))
        return self

    def __exit__(self, *exc):
        self.L.dgr_set_protocol(0, None)
        return False


def loss_gradient(obj: RefObject, hand: RefHand, q, params: Params):
    """losses.cpp:20-66 → (losses[3], d_stable, d_qrange, d_qlimit)."""
    L = hand.L
    q = np.ascontiguousarray(q, np.float64)
    D = 6 + hand.num_joints
    losses, ds, dr, dl = np.zeros(3), np.zeros(D), np.zeros(D), np.zeros(D)
    _check(L, L.dgr_loss_gradient(obj.ptr, hand.ptr, _d(q), C.byref(params), _d(losses), _d(ds), _d(dr),
                                  _d(dl)))
    return losses, ds, dr, dl


def evaluate_losses(obj, hand, q, params):
    L = hand.L
    q = np.ascontiguousarray(q, np.float64)
    out = np.zeros(3)
    _check(L, L.dgr_evaluate_losses(obj.ptr, hand.ptr, _d(q), C.byref(params), _d(out)))
    return out


def apply_gradient_step(hand, q, g, lr):
    L = hand.L
    q = np.ascontiguousarray(q, np.float64)
    g = np.ascontiguousarray(g, np.float64)
    out = np.zeros_like(q)
    _check(L, L.dgr_apply_gradient_step(hand.ptr, _d(q), _d(g), lr, _d(out)))
    return out


def sim_record(obj, hand, q, m, params, points_grad=False, rho_cap=0):
    """One recorded perturbation sim: (residual, grad(6+J), grad_points|None, rho_log)."""
    L = hand.L
    q = np.ascontiguousarray(q, np.float64)
    res = C.c_double()
    g = np.zeros(6 + hand.num_joints)
    gp = np.zeros((hand.num_samples, 3)) if points_grad else None
    cap = rho_cap or hand.num_samples * params.gs_iters * params.steps
    log = np.zeros(cap)
    n = C.c_int()
    _check(L, L.dgr_sim_record(obj.ptr, hand.ptr, _d(q), m, C.byref(params), C.byref(res), _d(g),
                               _d(gp) if gp is not None else None, _d(log), cap, C.byref(n)))
    return res.value, g, gp, log[: min(n.value, cap)]


def sim_forward(obj, hand, q, m, params, measure_residual=True, rho_cap=0):
    """Forward-only double sim with SolveStats: (residual, stats[5], rho_log)."""
    L = hand.L
    q = np.ascontiguousarray(q, np.float64)
    res = C.c_double()
    st = np.zeros(5)
    cap = rho_cap or hand.num_samples * params.gs_iters * params.steps
    log = np.zeros(cap)
    n = C.c_int()
    _check(L, L.dgr_sim_forward(obj.ptr, hand.ptr, _d(q), m, C.byref(params), int(measure_residual),
                                C.byref(res), _d(st), _d(log), cap, C.byref(n)))
    return res.value, st, log[: min(n.value, cap)]


def optimize(obj, hand, q, params, iters, k_begin=0, k_end=None, r0=0.02, lr=1e-3, beta1=0.9,
             beta2=0.999, eps=1e-8, adam_m=None, adam_v=None, threads=None, record=False):
    """SURVEY App. C driver on std::threads. Returns dict(q, m, v, status[, losses, grads])."""
    L = hand.L
    q = np.array(q, np.float64, copy=True, order="C")
    B = q.shape[0]
    D = 6 + hand.num_joints
    m = np.zeros((B, D)) if adam_m is None else np.array(adam_m, np.float64, copy=True, order="C")
    v = np.zeros((B, D)) if adam_v is None else np.array(adam_v, np.float64, copy=True, order="C")
    k_end = iters if k_end is None else k_end
    steps = k_end - k_begin
    cfg = OptCfg(iters=iters, k_begin=k_begin, k_end=k_end, pad=0, r0=r0, lr=lr, beta1=beta1, beta2=beta2,
                 eps=eps)
    tl = np.zeros((B, steps, 3)) if record else None
    tg = np.zeros((B, steps, D)) if record else None
    status = np.zeros(B, np.int32)
    L.dgr_optimize(obj.ptr, hand.ptr, B, _d(q), _d(m), _d(v), C.byref(params), C.byref(cfg),
                   threads or os.cpu_count() or 1, _d(tl) if record else None, _d(tg) if record else None,
                   _i(status))
    out = dict(q=q, m=m, v=v, status=status)
    if record:
        out.update(losses=tl, grads=tg)
    return out


def drop(obj: RefObject, state, dt=1e-3, mu=1.0, gs=8, gravity=(0.0, 0.0, -9.81), max_steps=5000, min_steps=1,
         ke_tol=1e-6, measure=False, record_every=0, settle=100):
    """step_on_table (sim.cpp:14-94) iterated from one RigidState row [13] with
    dgx_drop_batch's stopping rule -> (state [13], steps, ke, stats [4], traj)."""
    L = obj.L
    st = np.ascontiguousarray(state, np.float64)
    g = np.ascontiguousarray(gravity, np.float64)
    out, ke, stats = np.zeros(13), C.c_double(), np.zeros(4)
    steps = np.zeros(1, np.int32)
    rows = max_steps // record_every if record_every > 0 else 0
    traj = np.zeros((max(rows, 1), 13))
    _check(L, L.dgr_drop(obj.ptr, _d(st), dt, mu, gs, _d(g), max_steps, min_steps, ke_tol, int(measure), _d(out),
                         _i(steps), C.byref(ke), _d(stats), _d(traj) if rows else None, record_every, settle))
    return out, int(steps[0]), ke.value, stats, (traj[:rows] if rows else None)
