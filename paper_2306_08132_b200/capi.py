"""ctypes binding of include/dgx.h (libdgx_cuda.so, built in-tree).

There is no CPU fallback: if the shared library is missing or no sm_100
device is present, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DGX_LIBRARY") or os.path.join(PKG_DIR, "libdgx_cuda.so")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)
_fp = C.POINTER(C.c_float)

DGX_DEVICE_PTRS = 1
DGX_ASYNC = 2
DGX_SDF_SPHERE, DGX_SDF_BOX, DGX_SDF_GRID, DGX_SDF_MESH = 1, 2, 4, 8

STATUS_NAMES = {
    0: "ok",
    1: "loss evaluation produced a non-finite value",
    2: "tape: non-finite adjoint",
    3: "active-correction log overflow",
    4: "contact slot overflow",
    5: "adjoint replay mismatch",
}


class HandDescC(C.Structure):
    _fields_ = [
        ("num_links", C.c_int32), ("num_joints", C.c_int32), ("num_samples", C.c_int32),
        ("topo", _ip), ("link_parent_joint", _ip), ("joint_parent", _ip), ("joint_child", _ip),
        ("axis", _dp), ("origin_R", _dp), ("origin_t", _dp), ("lower", _dp), ("upper", _dp),
        ("samples", _dp), ("sample_link", _ip),
    ]


class ObjectDescC(C.Structure):
    _fields_ = [
        ("kind", C.c_int32), ("center", C.c_double * 3), ("radius", C.c_double),
        ("half_extents", C.c_double * 3), ("dims", C.c_int32 * 3), ("origin", C.c_double * 3),
        ("spacing", C.c_double), ("inv_spacing", C.c_double), ("values", _fp), ("mass", C.c_double),
        ("com", C.c_double * 3), ("inertia_body_inv", C.c_double * 9),
        ("num_vertices", C.c_int32), ("num_faces", C.c_int32), ("vertices", _dp), ("faces", _ip),
        ("vertex_normals", _dp), ("alpha_phong", C.c_double), ("inertia_body", C.c_double * 9),
    ]


class DropParamsC(C.Structure):
    _fields_ = [
        ("dt", C.c_double), ("mu", C.c_double), ("gs_iters", C.c_int32), ("measure_residual", C.c_int32),
        ("gravity", C.c_double * 3), ("max_steps", C.c_int32), ("min_steps", C.c_int32), ("ke_tol", C.c_double),
        ("record_every", C.c_int32), ("settle_steps", C.c_int32),
    ]


class ParamsC(C.Structure):
    _fields_ = [
        ("dt", C.c_double), ("mu", C.c_double), ("gs_iters", C.c_int32), ("steps", C.c_int32),
        ("dilation_radius", C.c_double), ("alpha_leak", C.c_double), ("num_velocities", C.c_int32),
        ("pad", C.c_int32), ("velocities", (C.c_double * 3) * 8), ("w_stable", C.c_double),
        ("w_qrange", C.c_double), ("w_qlimit", C.c_double),
        # ABI 2
        ("velocity_list", C.c_void_p), ("w_force_closure", C.c_double), ("w_penetration", C.c_double),
        ("contact_threshold", C.c_double), ("torque_scale", C.c_double),
    ]


class OptC(C.Structure):
    _fields_ = [
        ("iters", C.c_int32), ("k_begin", C.c_int32), ("k_end", C.c_int32), ("record", C.c_int32),
        ("r0", C.c_double), ("lr", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double),
        ("eps", C.c_double),
    ]


EXPORTS = [
    "dgx_last_error", "dgx_abi_version", "dgx_ctx_create", "dgx_ctx_destroy", "dgx_ctx_set_stream",
    "dgx_ctx_set_correction_capacity", "dgx_ctx_launch_count", "dgx_ctx_set_kernel_timing", "dgx_ctx_set_adjoint",
    "dgx_ctx_kernel_times", "dgx_hand_upload", "dgx_hand_free",
    "dgx_object_upload", "dgx_object_free", "dgx_forward_batch", "dgx_loss_gradient_batch",
    "dgx_evaluate_losses_batch", "dgx_apply_gradient_step_batch", "dgx_optimize_batch", "dgx_debug_sims",
    "dgx_fp64_peak", "dgx_optimize_multi", "dgx_sdf_query_batch", "dgx_mesh_inertia",
    "dgx_mesh_bvh", "dgx_drop_batch", "dgx_contacts_batch", "dgx_grasp_energy_batch",
    "dgx_apply_gradient_step_joints",
]

_lib: C.CDLL | None = None


class DgxError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[dgx {code}] {msg}")
        self.code = code


def load() -> C.CDLL:
    """Load libdgx_cuda.so (raises if it was not built: no fallback path)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(LIB_PATH)
    vp = C.c_void_p
    L.dgx_last_error.restype = C.c_char_p
    L.dgx_abi_version.restype = C.c_int
    L.dgx_ctx_create.argtypes = [C.c_int, C.POINTER(vp)]
    L.dgx_ctx_destroy.argtypes = [vp]
    L.dgx_ctx_set_stream.argtypes = [vp, vp]
    L.dgx_ctx_set_correction_capacity.argtypes = [vp, C.c_int32]
    L.dgx_ctx_launch_count.argtypes = [vp]
    L.dgx_ctx_launch_count.restype = C.c_int64
    L.dgx_ctx_set_kernel_timing.argtypes = [vp, C.c_int]
    L.dgx_ctx_set_adjoint.argtypes = [vp, C.c_int]
    L.dgx_ctx_kernel_times.argtypes = [vp, C.POINTER(C.c_double), C.POINTER(C.c_int64)]
    L.dgx_hand_upload.argtypes = [vp, C.POINTER(HandDescC), C.POINTER(vp)]
    L.dgx_hand_free.argtypes = [vp]
    L.dgx_object_upload.argtypes = [vp, C.POINTER(ObjectDescC), C.POINTER(vp)]
    L.dgx_object_free.argtypes = [vp]
    L.dgx_forward_batch.argtypes = [vp, vp, C.c_int32, vp, vp, C.c_uint32]
    L.dgx_loss_gradient_batch.argtypes = [vp, vp, vp, C.c_int32, vp, C.POINTER(ParamsC), vp, vp, vp, C.c_uint32]
    L.dgx_evaluate_losses_batch.argtypes = [vp, vp, vp, C.c_int32, vp, C.POINTER(ParamsC), vp, vp, vp, C.c_uint32]
    L.dgx_apply_gradient_step_batch.argtypes = [vp, vp, C.c_int32, vp, vp, C.c_double, vp, C.c_uint32]
    L.dgx_optimize_batch.argtypes = [vp, vp, vp, C.c_int32, vp, vp, vp, C.POINTER(ParamsC), C.POINTER(OptC), vp,
                                     vp, C.c_uint32]
    L.dgx_debug_sims.argtypes = [vp, vp, vp, C.c_int32, vp, C.POINTER(ParamsC), vp, vp, vp, vp, C.c_uint32]
    L.dgx_grasp_energy_batch.argtypes = [vp, vp, vp, C.c_int32, vp, C.POINTER(ParamsC), vp, vp, C.c_uint32]
    L.dgx_fp64_peak.argtypes = [C.c_int, _dp, _dp]
    L.dgx_optimize_multi.argtypes = [vp, vp, C.c_int32, vp, vp, vp, vp, vp, C.POINTER(ParamsC), C.POINTER(OptC), vp,
                                     vp, C.c_uint32]
    L.dgx_sdf_query_batch.argtypes = [vp, vp, C.c_int32, vp, C.c_double, C.c_int32, vp, C.c_uint32]
    L.dgx_mesh_inertia.argtypes = [C.c_int32, vp, C.c_int32, vp, C.c_double, _dp, _dp, _dp, _dp]
    L.dgx_mesh_bvh.argtypes = [C.c_int32, vp, C.c_int32, vp, C.c_int32, vp, vp, vp, _ip]
    L.dgx_contacts_batch.argtypes = [vp, vp, vp, C.c_int32, vp, vp, C.c_int32, _dp, C.c_int32, vp, vp, vp, vp, vp,
                                     C.c_uint32]
    L.dgx_drop_batch.argtypes = [vp, vp, C.c_int32, vp, C.POINTER(DropParamsC), vp, vp, vp, vp, vp, C.c_uint32]
    _lib = L
    return L


def check(rc: int) -> None:
    if rc != 0:
        raise DgxError(rc, load().dgx_last_error().decode())


def ptr(a) -> int | None:
    """Address of a C-contiguous numpy array or torch tensor (None passes NULL)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        assert a.flags["C_CONTIGUOUS"], "array must be C-contiguous"
        return a.ctypes.data
    return a.data_ptr()  # torch.Tensor


def hand_desc_c(h) -> tuple[HandDescC, list]:
    keep = [np.ascontiguousarray(getattr(h, k)) for k in ("topo", "link_parent_joint", "joint_parent",
                                                          "joint_child", "axis", "origin_R", "origin_t",
                                                          "lower", "upper", "samples", "sample_link")]
    (topo, lpj, jp, jc, axis, oR, ot, lo, up, smp, sl) = keep
    d = HandDescC(h.num_links, h.num_joints, h.num_samples,
                  topo.ctypes.data_as(_ip), lpj.ctypes.data_as(_ip), jp.ctypes.data_as(_ip),
                  jc.ctypes.data_as(_ip), axis.ctypes.data_as(_dp), oR.ctypes.data_as(_dp),
                  ot.ctypes.data_as(_dp), lo.ctypes.data_as(_dp), up.ctypes.data_as(_dp),
                  smp.ctypes.data_as(_dp), sl.ctypes.data_as(_ip))
    return d, keep


def object_desc_c(o) -> tuple[ObjectDescC, list]:
    d = ObjectDescC()
    keep = []
    d.kind = {"sphere": DGX_SDF_SPHERE, "box": DGX_SDF_BOX, "grid": DGX_SDF_GRID, "mesh": DGX_SDF_MESH}[o.kind]
    d.center[:] = [float(v) for v in o.center]
    d.radius = float(o.radius)
    d.half_extents[:] = [float(v) for v in o.half_extents]
    if o.kind == "grid":
        vals = np.ascontiguousarray(o.values, np.float32)
        keep.append(vals)
        d.dims[:] = [int(v) for v in o.dims]
        d.origin[:] = [float(v) for v in o.origin]
        d.spacing = float(o.spacing)
        d.inv_spacing = float(o.inv_spacing)
        d.values = vals.ctypes.data_as(_fp)
    if o.kind == "mesh":
        V = np.ascontiguousarray(o.vertices, np.float64)
        F = np.ascontiguousarray(o.faces, np.int32)
        keep += [V, F]
        d.num_vertices, d.num_faces = V.shape[0], F.shape[0]
        d.vertices = V.ctypes.data_as(_dp)
        d.faces = F.ctypes.data_as(_ip)
        if o.vertex_normals is not None:
            VN = np.ascontiguousarray(o.vertex_normals, np.float64)
            keep.append(VN)
            d.vertex_normals = VN.ctypes.data_as(_dp)
        d.alpha_phong = float(o.alpha_phong)
    d.mass = float(o.mass)
    d.com[:] = [float(v) for v in o.com]
    d.inertia_body_inv[:] = [float(v) for v in np.asarray(o.inertia_body_inv, np.float64).reshape(9)]
    d.inertia_body[:] = [float(v) for v in np.asarray(o.inertia_body, np.float64).reshape(9)]
    return d, keep
