"""Python mirror of the reference's diffgrasp API for the hot path, over the
C-ABI (include/dgx.h). Names and argument meaning follow
/root/reference/proj/include/diffgrasp:

  SimParams / LeakPolicy       sim.hpp:22-40
  StabilityProtocol.standard   losses.hpp:21-27
  LossWeights                  losses.hpp:31-35
  loss_gradient                losses.hpp:126-127   (batched: q is [B, 7+J])
  evaluate_losses              losses.hpp:119-121   (+ SolveStats per perturbation)
  apply_gradient_step          losses.hpp:136
  HandModel.forward            hand.hpp:86

Errors raise like the reference: invalid arguments -> ValueError
(std::invalid_argument), per-candidate numeric failures are returned in
``status`` and raised by ``check_status`` as RuntimeError with the
reference's message. All compute runs in libdgx_cuda.so; there is no CPU
path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import capi
from .model import HandDesc, ObjectDesc


@dataclass
class SimParams:
    dt: float = 0.001
    mu: float = 1.0
    gs_iters: int = 8
    dilation_radius: float = 0.0
    alpha_leak: float = 0.1  # LeakPolicy::alpha_leak


@dataclass
class StabilityProtocol:
    velocities: list = field(default_factory=list)
    steps: int = 1

    @staticmethod
    def standard(speed: float = 0.5, steps: int = 1) -> "StabilityProtocol":
        s = speed
        return StabilityProtocol([(s, 0, 0), (-s, 0, 0), (0, s, 0), (0, -s, 0), (0, 0, s), (0, 0, -s), (0, 0, 0)],
                                 steps)

    @property
    def m(self) -> int:
        return len(self.velocities)


@dataclass
class LossWeights:
    stable: float = 1.0
    qrange: float = 0.01
    qlimit: float = 1.0
    # grasp-energy terms (north_star (3); no reference counterpart, off by
    # default): see grasp_energy()
    force_closure: float = 0.0
    penetration: float = 0.0
    contact_threshold: float = 0.005
    torque_scale: float = 0.05


@dataclass
class OptConfig:
    """SURVEY App. C driver: linear dilation r0 -> 0, Adam, tangent-space step."""
    iterations: int = 200
    dilation_start_radius: float = 0.02
    learning_rate: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8


def params_c(params: SimParams, protocol: StabilityProtocol, weights: LossWeights | None = None) -> capi.ParamsC:
    if params.dilation_radius < 0.0:
        raise ValueError("dilation radius must be >= 0")
    if protocol.m < 1:
        raise ValueError("protocol must have >= 1 velocities")
    w = weights or LossWeights()
    p = capi.ParamsC()
    p.dt, p.mu, p.gs_iters, p.steps = params.dt, params.mu, params.gs_iters, protocol.steps
    p.dilation_radius, p.alpha_leak = params.dilation_radius, params.alpha_leak
    p.num_velocities = protocol.m
    vl = np.ascontiguousarray(np.asarray(protocol.velocities, np.float64).reshape(protocol.m, 3))
    for m in range(min(protocol.m, 8)):
        for c in range(3):
            p.velocities[m][c] = float(vl[m, c])
    if protocol.m > 8:  # any M: the list itself (kept alive with the struct)
        p._velocity_list = vl
        p.velocity_list = vl.ctypes.data
    p.w_stable, p.w_qrange, p.w_qlimit = w.stable, w.qrange, w.qlimit
    p.w_force_closure, p.w_penetration = w.force_closure, w.penetration
    p.contact_threshold, p.torque_scale = w.contact_threshold, w.torque_scale
    return p


class Context:
    """One CUDA device + stream (dgx_ctx)."""

    def __init__(self, device: int = 0, correction_capacity: int | None = None):
        self.L = capi.load()
        h = C.c_void_p()
        capi.check(self.L.dgx_ctx_create(device, C.byref(h)))
        self.h = h
        self.device = device
        if correction_capacity:
            capi.check(self.L.dgx_ctx_set_correction_capacity(self.h, correction_capacity))

    def set_stream(self, stream_ptr: int | None) -> None:
        """Launch on an external cudaStream_t; None/0 selects the context's own
        stream (the legacy default stream cannot be selected)."""
        capi.check(self.L.dgx_ctx_set_stream(self.h, stream_ptr or None))

    @property
    def launches(self) -> int:
        return int(self.L.dgx_ctx_launch_count(self.h))

    def set_kernel_timing(self, enable: bool) -> None:
        """Bracket every grasp-search launch with CUDA events on its stream
        (resets the record)."""
        capi.check(self.L.dgx_ctx_set_kernel_timing(self.h, int(enable)))

    def set_adjoint(self, variant: str) -> None:
        """Split-execution adjoint kernel: "auto" (default), "cta" or "lane"
        (include/dgx.h dgx_ctx_set_adjoint)."""
        v = {"auto": 0, "cta": 1, "lane": 2}[variant]
        capi.check(self.L.dgx_ctx_set_adjoint(self.h, v))

    def kernel_times(self) -> dict:
        """{kind: (total ms, launches)} for kinds fused / forward / adjoint since
        set_kernel_timing(True); synchronizes on the recorded events."""
        ms = (C.c_double * 3)()
        n = (C.c_int64 * 3)()
        capi.check(self.L.dgx_ctx_kernel_times(self.h, ms, n))
        return {k: (ms[i], n[i]) for i, k in enumerate(("fused", "forward", "adjoint"))}

    def close(self) -> None:
        if getattr(self, "h", None):
            self.L.dgx_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Hand:
    """A HandDesc resident on the device (dgx_hand)."""

    def __init__(self, ctx: Context, desc: HandDesc):
        self.ctx, self.desc = ctx, desc
        d, keep = capi.hand_desc_c(desc)
        h = C.c_void_p()
        capi.check(ctx.L.dgx_hand_upload(ctx.h, C.byref(d), C.byref(h)))
        self.h = h
        self.J, self.N = desc.num_joints, desc.num_samples

    def __del__(self):
        try:
            if self.h:
                self.ctx.L.dgx_hand_free(self.h)
                self.h = None
        except Exception:
            pass


class GraspObject:
    """An ObjectDesc resident on the device (dgx_object)."""

    def __init__(self, ctx: Context, desc: ObjectDesc):
        self.ctx, self.desc = ctx, desc
        d, keep = capi.object_desc_c(desc)
        h = C.c_void_p()
        capi.check(ctx.L.dgx_object_upload(ctx.h, C.byref(d), C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            if self.h:
                self.ctx.L.dgx_object_free(self.h)
                self.h = None
        except Exception:
            pass


def _flags(*arrays) -> int:
    dev = [not isinstance(a, np.ndarray) for a in arrays if a is not None]
    if any(dev) and not all(dev):
        raise ValueError("mix of host (numpy) and device (torch) arrays")
    return capi.DGX_DEVICE_PTRS if dev and dev[0] else 0


def _f64(a, shape):
    a = np.ascontiguousarray(a, np.float64)
    if a.shape != shape:
        a = a.reshape(shape)
    return a


def _check_arr(a, shape, kind: str, name: str) -> None:
    """Validate a caller-supplied array before its pointer crosses the C ABI
    (the ABI trusts sizes): exact shape, dtype ("f64" / "i32") and C order,
    numpy or torch alike."""
    if a is None:
        return
    if isinstance(a, np.ndarray):
        ok_dt = a.dtype == (np.float64 if kind == "f64" else np.int32)
        contig = a.flags["C_CONTIGUOUS"]
    elif hasattr(a, "data_ptr"):
        import torch
        ok_dt = a.dtype == (torch.float64 if kind == "f64" else torch.int32)
        contig = a.is_contiguous()
    else:
        raise ValueError(f"{name}: expected a numpy array or torch tensor")
    if tuple(a.shape) != tuple(shape):
        raise ValueError(f"{name}: shape {tuple(a.shape)} != {tuple(shape)}")
    if not ok_dt:
        raise ValueError(f"{name}: dtype {a.dtype} != {'float64' if kind == 'f64' else 'int32'}")
    if not contig:
        raise ValueError(f"{name}: must be C-contiguous")


def check_status(status) -> None:
    st = np.asarray(status)
    bad = np.nonzero(st)[0]
    if bad.size:
        code = int(st[bad[0]])
        raise RuntimeError(f"candidate {int(bad[0])}: {capi.STATUS_NAMES.get(code, code)}")


def forward(ctx: Context, hand: Hand, q) -> np.ndarray:
    q = _f64(q, (-1, 7 + hand.J))
    out = np.zeros((q.shape[0], hand.N, 3))
    capi.check(ctx.L.dgx_forward_batch(ctx.h, hand.h, q.shape[0], capi.ptr(q), capi.ptr(out), 0))
    return out


def loss_gradient(ctx: Context, obj: GraspObject, hand: Hand, q, protocol: StabilityProtocol, params: SimParams):
    """Batched dg::loss_gradient → (losses [B,3], grads [B,3,6+J], status [B])."""
    q = _f64(q, (-1, 7 + hand.J))
    B = q.shape[0]
    losses = np.zeros((B, 3))
    grads = np.zeros((B, 3, 6 + hand.J))
    status = np.zeros(B, np.int32)
    p = params_c(params, protocol)
    capi.check(ctx.L.dgx_loss_gradient_batch(ctx.h, hand.h, obj.h, B, capi.ptr(q), C.byref(p), capi.ptr(losses),
                                             capi.ptr(grads), capi.ptr(status), 0))
    return losses, grads, status


def evaluate_losses(ctx: Context, obj: GraspObject, hand: Hand, q, protocol: StabilityProtocol, params: SimParams):
    """Batched dg::evaluate_losses → (losses [B,3], stats [B,M,5], status [B])."""
    q = _f64(q, (-1, 7 + hand.J))
    B = q.shape[0]
    losses = np.zeros((B, 3))
    stats = np.zeros((B, protocol.m, 5))
    status = np.zeros(B, np.int32)
    p = params_c(params, protocol)
    capi.check(ctx.L.dgx_evaluate_losses_batch(ctx.h, hand.h, obj.h, B, capi.ptr(q), C.byref(p), capi.ptr(losses),
                                               capi.ptr(stats), capi.ptr(status), 0))
    return losses, stats, status


def grasp_energy(ctx: Context, obj: GraspObject, hand: Hand, q, contact_threshold: float = 0.005,
                 torque_scale: float = 0.05):
    """north_star (3) grasp-energy terms (dgx_grasp_energy_batch; no reference
    counterpart, parity-unpinned) at the object's canonical pose:
    E_fc = |sum_C n|^2 + |sum_C (p - com) x n|^2 / torque_scale^2 over contacts
    C = {|rho| <= contact_threshold}, E_pen = sum max(0, -rho); gradients with
    contact set and normals frozen. -> (energy [B,2], grads [B,2,6+J])."""
    q = _f64(q, (-1, 7 + hand.J))
    B = q.shape[0]
    e = np.zeros((B, 2))
    g = np.zeros((B, 2, 6 + hand.J))
    p = params_c(SimParams(), StabilityProtocol.standard(),
                 LossWeights(contact_threshold=contact_threshold, torque_scale=torque_scale))
    capi.check(ctx.L.dgx_grasp_energy_batch(ctx.h, hand.h, obj.h, B, capi.ptr(q), C.byref(p), capi.ptr(e),
                                            capi.ptr(g), 0))
    return e, g


def sdf_query(ctx: Context, obj: GraspObject, points, radius: float = 0.0, within: bool = False) -> np.ndarray:
    """[n, 8] = rho - radius, unit gradient, smoothed point, sign at object-frame
    points: MeshSdf::dilated (sdf.cpp:62-67), or dilated_within with the
    solver's 5 mm cull (sdf.cpp:69-81) when ``within`` (culled: rho = +inf,
    sign 0). Any backend; only meshes cull."""
    p = _f64(points, (-1, 3))
    out = np.zeros((p.shape[0], 8))
    capi.check(ctx.L.dgx_sdf_query_batch(ctx.h, obj.h, p.shape[0], capi.ptr(p), float(radius), int(bool(within)),
                                         capi.ptr(out), 0))
    return out


@dataclass
class DropParams:
    """step_on_table's SimParams (sim.hpp:33-40) with gravity on, plus the
    scene driver's stopping rule."""
    dt: float = 1e-3
    mu: float = 1.0
    gs_iters: int = 8
    gravity: tuple = (0.0, 0.0, -9.81)
    max_steps: int = 5000
    min_steps: int = 1
    ke_tol: float = 1e-6
    settle_steps: int = 100
    measure_residual: bool = False

    def c(self, record_every: int = 0) -> capi.DropParamsC:
        p = capi.DropParamsC()
        p.dt, p.mu, p.gs_iters = float(self.dt), float(self.mu), int(self.gs_iters)
        p.measure_residual = int(bool(self.measure_residual))
        p.gravity[:] = [float(v) for v in self.gravity]
        p.max_steps, p.min_steps, p.ke_tol = int(self.max_steps), int(self.min_steps), float(self.ke_tol)
        p.record_every = int(record_every)
        p.settle_steps = int(self.settle_steps)
        return p


def drop(ctx: Context, obj: GraspObject, states, params: DropParams = DropParams(), record_every: int = 0,
         flags: int | None = None):
    """Batched scene drop of a mesh object: every RigidState row [13] (x, theta
    w,x,y,z, xdot, thetadot) advanced by step_on_table (sim.cpp:14-94) until at
    rest on the table z = 0 (settle_steps consecutive contact steps with kinetic
    energy < ke_tol). Returns dict(state, steps, ke, stats[, traj])."""
    dev = not isinstance(states, np.ndarray)
    B = states.shape[0]
    rows = params.max_steps // record_every if record_every > 0 else 0
    if dev:
        import torch
        mk = lambda *shape, dt=torch.float64: torch.zeros(*shape, dtype=dt, device=states.device)  # noqa: E731
        out, steps, ke, stats = mk(B, 13), mk(B, dt=torch.int32), mk(B), mk(B, 4)
        traj = mk(B, rows, 13) if rows else None
        fl = capi.DGX_DEVICE_PTRS if flags is None else flags
    else:
        states = _f64(states, (-1, 13))
        out, steps, ke, stats = np.zeros((B, 13)), np.zeros(B, np.int32), np.zeros(B), np.zeros((B, 4))
        traj = np.zeros((B, rows, 13)) if rows else None
        fl = 0 if flags is None else flags
    p = params.c(record_every)
    capi.check(ctx.L.dgx_drop_batch(ctx.h, obj.h, B, capi.ptr(states), C.byref(p), capi.ptr(out), capi.ptr(steps),
                                    capi.ptr(ke), capi.ptr(stats), capi.ptr(traj), fl))
    res = dict(state=out, steps=steps, ke=ke, stats=stats)
    if rows:
        res["traj"] = traj
    return res


def mesh_bvh(vertices, faces):
    """Host-only: the BVH dgx_object_upload builds for a mesh (Bvh::build,
    bvh.cpp:148-163) as (boxes [n,6], links [n,4] left/right/first/count,
    leaf-order face ids)."""
    import ctypes as C
    V = np.ascontiguousarray(vertices, np.float64).reshape(-1, 3)
    F = np.ascontiguousarray(faces, np.int32).reshape(-1, 3)
    cap = 2 * F.shape[0] + 1
    boxes, links, fo = np.zeros((cap, 6)), np.zeros((cap, 4), np.int32), np.zeros(F.shape[0], np.int32)
    n = C.c_int32()
    L = capi.load()
    capi.check(L.dgx_mesh_bvh(V.shape[0], capi.ptr(V), F.shape[0], capi.ptr(F), cap, capi.ptr(boxes),
                              capi.ptr(links), capi.ptr(fo), C.byref(n)))
    return boxes[:n.value], links[:n.value], fo


def apply_gradient_step(ctx: Context, hand: Hand, q, g, lr: float) -> np.ndarray:
    q = _f64(q, (-1, 7 + hand.J))
    g = _f64(g, (q.shape[0], 6 + hand.J))
    out = np.zeros_like(q)
    capi.check(ctx.L.dgx_apply_gradient_step_batch(ctx.h, hand.h, q.shape[0], capi.ptr(q), capi.ptr(g), lr,
                                                   capi.ptr(out), 0))
    return out


def debug_sims(ctx: Context, obj: GraspObject, hand: Hand, q, protocol: StabilityProtocol, params: SimParams,
               point_grads: bool = False):
    """Per-perturbation residuals [B,M], gradients [B,M,6+J] (and d/dp [B,M,N,3])."""
    q = _f64(q, (-1, 7 + hand.J))
    B, M = q.shape[0], protocol.m
    res = np.zeros((B, M))
    g = np.zeros((B, M, 6 + hand.J))
    gp = np.zeros((B, M, hand.N, 3)) if point_grads else None
    status = np.zeros(B, np.int32)
    p = params_c(params, protocol)
    capi.check(ctx.L.dgx_debug_sims(ctx.h, hand.h, obj.h, B, capi.ptr(q), C.byref(p), capi.ptr(res), capi.ptr(g),
                                    capi.ptr(gp), capi.ptr(status), 0))
    return res, g, gp, status


def optimize(ctx: Context, obj: GraspObject, hand: Hand, q, protocol: StabilityProtocol, params: SimParams,
             weights: LossWeights, opt: OptConfig, k_begin: int = 0, k_end: int | None = None, adam_m=None,
             adam_v=None, record: bool = False, flags: int | None = None, status=None):
    """Fused synthesis loop (dgx_optimize_batch). numpy arrays: copied in/out
    (host path, synchronous); torch CUDA tensors: updated in place on device."""
    k_end = opt.iterations if k_end is None else k_end
    D = 6 + hand.J
    host = isinstance(q, np.ndarray) or not hasattr(q, "data_ptr")
    if host:
        q = np.array(q, np.float64, copy=True, order="C").reshape(-1, 7 + hand.J)
        B = q.shape[0]
        adam_m = np.zeros((B, D)) if adam_m is None else np.array(adam_m, np.float64, copy=True, order="C")
        adam_v = np.zeros((B, D)) if adam_v is None else np.array(adam_v, np.float64, copy=True, order="C")
        status = np.zeros(B, np.int32)
        traj = np.zeros((B, k_end - k_begin, 3 + D)) if record else None
    else:
        import torch
        B = q.shape[0]
        dev = q.device
        adam_m = torch.zeros((B, D), dtype=torch.float64, device=dev) if adam_m is None else adam_m
        adam_v = torch.zeros((B, D), dtype=torch.float64, device=dev) if adam_v is None else adam_v
        status = torch.zeros(B, dtype=torch.int32, device=dev) if status is None else status
        traj = torch.zeros((B, k_end - k_begin, 3 + D), dtype=torch.float64, device=dev) if record else None
    if not 0 <= k_begin <= k_end <= opt.iterations:
        raise ValueError("need 0 <= k_begin <= k_end <= iterations")
    for a, shp, kd, nm in ((q, (B, 7 + hand.J), "f64", "q"), (adam_m, (B, D), "f64", "adam_m"),
                           (adam_v, (B, D), "f64", "adam_v"), (status, (B,), "i32", "status"),
                           (traj, (B, k_end - k_begin, 3 + D), "f64", "traj")):
        _check_arr(a, shp, kd, nm)
    p = params_c(params, protocol, weights)
    o = capi.OptC(opt.iterations, k_begin, k_end, int(record), opt.dilation_start_radius, opt.learning_rate,
                  opt.beta1, opt.beta2, opt.eps)
    fl = _flags(q, adam_m, adam_v, status, traj) if flags is None else flags
    capi.check(ctx.L.dgx_optimize_batch(ctx.h, hand.h, obj.h, B, capi.ptr(q), capi.ptr(adam_m), capi.ptr(adam_v),
                                        C.byref(p), C.byref(o), capi.ptr(traj), capi.ptr(status), fl))
    return dict(q=q, m=adam_m, v=adam_v, status=status, traj=traj)


def optimize_multi(ctx: Context, objs: list, hand: Hand, q, counts, protocol: StabilityProtocol,
                   params: SimParams, weights: LossWeights, opt: OptConfig, k_begin: int = 0,
                   k_end: int | None = None, adam_m=None, adam_v=None, record: bool = False, flags: int | None = None,
                   status=None, traj=None, inplace: bool = False):
    """Multi-object fused synthesis (dgx_optimize_multi): candidates object-major,
    counts[i] for objs[i]; objects run concurrently on side streams.
    Host arrays are copied unless inplace=True: then q / adam_m / adam_v (and
    status / traj when given) must be C-contiguous (e.g. pinned) arrays of the
    right dtype and are updated in place."""
    k_end = opt.iterations if k_end is None else k_end
    D = 6 + hand.J
    counts = np.ascontiguousarray(counts, np.int32)
    host = isinstance(q, np.ndarray) or not hasattr(q, "data_ptr")
    if host and inplace:
        for a, dt in ((q, np.float64), (adam_m, np.float64), (adam_v, np.float64)):
            if not (isinstance(a, np.ndarray) and a.dtype == dt and a.flags["C_CONTIGUOUS"]):
                raise ValueError("inplace: q, adam_m, adam_v must be C-contiguous float64 numpy arrays")
        B = q.shape[0]
        status = np.zeros(B, np.int32) if status is None else status
        if record and traj is None:
            traj = np.zeros((B, k_end - k_begin, 3 + D))
        if not record:
            traj = None
    elif host:
        q = np.array(q, np.float64, copy=True, order="C").reshape(-1, 7 + hand.J)
        B = q.shape[0]
        adam_m = np.zeros((B, D)) if adam_m is None else np.array(adam_m, np.float64, copy=True, order="C")
        adam_v = np.zeros((B, D)) if adam_v is None else np.array(adam_v, np.float64, copy=True, order="C")
        status = np.zeros(B, np.int32) if status is None else status
        traj = np.zeros((B, k_end - k_begin, 3 + D)) if record else None
    else:
        import torch
        B = q.shape[0]
        dev = q.device
        adam_m = torch.zeros((B, D), dtype=torch.float64, device=dev) if adam_m is None else adam_m
        adam_v = torch.zeros((B, D), dtype=torch.float64, device=dev) if adam_v is None else adam_v
        status = torch.zeros(B, dtype=torch.int32, device=dev) if status is None else status
        traj = torch.zeros((B, k_end - k_begin, 3 + D), dtype=torch.float64, device=dev) if record else None
    if counts.ndim != 1 or counts.shape[0] != len(objs):
        raise ValueError("counts must hold one entry per object")
    if np.any(counts < 0) or int(counts.sum()) != B:
        raise ValueError("counts must be >= 0 and sum to the number of candidates")
    if not 0 <= k_begin <= k_end <= opt.iterations:
        raise ValueError("need 0 <= k_begin <= k_end <= iterations")
    for a, shp, kd, nm in ((q, (B, 7 + hand.J), "f64", "q"), (adam_m, (B, D), "f64", "adam_m"),
                           (adam_v, (B, D), "f64", "adam_v"), (status, (B,), "i32", "status"),
                           (traj, (B, k_end - k_begin, 3 + D), "f64", "traj")):
        _check_arr(a, shp, kd, nm)
    handles = (C.c_void_p * len(objs))(*[o.h.value for o in objs])
    p = params_c(params, protocol, weights)
    o = capi.OptC(opt.iterations, k_begin, k_end, int(record), opt.dilation_start_radius, opt.learning_rate,
                  opt.beta1, opt.beta2, opt.eps)
    fl = _flags(q, adam_m, adam_v, status, traj) if flags is None else flags
    capi.check(ctx.L.dgx_optimize_multi(ctx.h, hand.h, len(objs), handles, capi.ptr(counts), capi.ptr(q),
                                        capi.ptr(adam_m), capi.ptr(adam_v), C.byref(p), C.byref(o), capi.ptr(traj),
                                        capi.ptr(status), fl))
    return dict(q=q, m=adam_m, v=adam_v, status=status, traj=traj)
