"""The lane adjoint (csrc/dgx_lane_adj.cuh: one thread per (candidate, sim),
the reverse sweep walked serially in the tape's order) against the compiled
reference and against the CTA adjoint, forced through dgx_ctx_set_adjoint on
batches above the SM count (the split path) for every SDF backend it serves.

Bars: losses and per-sim residuals BIT-EXACT (the forward kernel is shared);
gradients within GRAD_RTOL of the reference tape (sim.hpp:105-125,
tape.cpp:27-114) and within LANE_VS_CTA_RTOL of the CTA adjoint (the same
closed forms, summed in a different order); rows of identical configurations
bit-identical wherever they sit in the batch.
"""
import numpy as np
import pytest

from test_gpu_configs import Setup
from test_gpu_parity import GRAD_RTOL, relerr

pytestmark = pytest.mark.gpu
LANE_VS_CTA_RTOL = 1e-11
TILE = 21  # 8 distinct rows x 21 = 168 candidates > 148 SMs: split execution


def _object(name):
    from paper_2306_08132_b200 import model
    return {"sphere": lambda: model.sphere(0.025), "box": lambda: model.box((0.04, 0.06, 0.05)),
            "boxgrid64": lambda: model.box_grid(res=64), "cylinder64": lambda: model.cylinder_grid(res=64),
            "blob128": lambda: model.blob_grid(seed=3, res=128)}[name]()


def _run(ctx, variant, fn):
    ctx.set_adjoint(variant)
    ctx.set_kernel_timing(True)
    try:
        out = fn()
        kt = ctx.kernel_times()
    finally:
        ctx.set_kernel_timing(False)
        ctx.set_adjoint("auto")
    assert kt["adjoint"][1] >= 1 and kt["fused"][1] == 0, kt  # the split path ran
    return out


CASES = [("barrett3", "sphere", 0.01), ("barrett3", "box", 0.0), ("allegro16", "boxgrid64", 0.02),
         ("allegro16", "cylinder64", 0.015), ("shadow22_dense", "blob128", 0.02)]


@pytest.mark.parametrize("hand_name,obj_name,radius", CASES)
def test_lane_adjoint_loss_gradient(ctx, oracle, hand_name, obj_name, radius):
    from paper_2306_08132_b200 import api
    s = Setup(ctx, oracle, hand_name, _object(obj_name), B=8, seed=91)
    q = np.tile(s.q, (TILE, 1))
    proto, params = api.StabilityProtocol.standard(), api.SimParams(dilation_radius=radius)
    lg = lambda: api.loss_gradient(ctx, s.obj, s.hand, q, proto, params)  # noqa: E731
    ll, gl, stl = _run(ctx, "lane", lg)
    lc, gc, stc = _run(ctx, "cta", lg)
    assert not np.any(stl) and not np.any(stc)
    assert np.array_equal(ll, lc)
    assert relerr(gl, gc) < LANE_VS_CTA_RTOL, relerr(gl, gc)
    for t in range(1, TILE):  # position in the batch does not matter
        assert np.array_equal(gl[8 * t:8 * t + 8], gl[:8])
    p = oracle.default_params(dilation_radius=radius)
    for b in range(8):
        rl, ds, dr, dl = oracle.loss_gradient(s.ro, s.rh, s.q[b], p)
        assert np.array_equal(ll[b], rl), (b, ll[b], rl)
        assert relerr(gl[b, 0], ds) < GRAD_RTOL, (b, relerr(gl[b, 0], ds))
        assert relerr(gl[b, 1], dr) < GRAD_RTOL
        assert np.array_equal(gl[b, 2], dl)


def test_lane_adjoint_per_sim_and_point_gradients(ctx, oracle):
    """dgx_debug_sims through the lane adjoint: per-perturbation residuals,
    gradients (sim_grads) and d residual / d p (point_grads) vs the tape."""
    from paper_2306_08132_b200 import api
    s = Setup(ctx, oracle, "allegro16", _object("boxgrid64"), B=8, seed=92)
    q = np.tile(s.q, (TILE, 1))
    proto, params = api.StabilityProtocol.standard(), api.SimParams(dilation_radius=0.02)
    res, g, gp, st = _run(ctx, "lane", lambda: api.debug_sims(ctx, s.obj, s.hand, q, proto, params, point_grads=True))
    assert not np.any(st)
    p = oracle.default_params(dilation_radius=0.02)
    for b in range(3):
        for m in range(7):
            rres, rg, rgp, _ = oracle.sim_record(s.ro, s.rh, s.q[b], m, p, points_grad=True)
            assert res[b, m] == rres and res[b + 8, m] == rres
            assert relerr(g[b, m], rg) < GRAD_RTOL, (b, m)
            assert relerr(gp[b, m], rgp) < GRAD_RTOL, (b, m)


@pytest.mark.parametrize("hand_name,obj_name", [("allegro16", "boxgrid64"), ("barrett3", "sphere")])
def test_lane_adjoint_optimizer_teacher_forced(ctx, oracle, hand_name, obj_name):
    """Two optimizer iterates (Adam state carried on the device) through the
    lane adjoint; each iterate's rows vs the reference optimizer step from the
    same state (losses bit-exact, gradients / q / Adam m within GRAD_RTOL)."""
    from paper_2306_08132_b200 import api
    s = Setup(ctx, oracle, hand_name, _object(obj_name), B=8, seed=93)
    q = np.tile(s.q, (TILE, 1))
    m = v = None
    for k in (0, 1):
        out = _run(ctx, "lane", lambda: api.optimize(
            ctx, s.obj, s.hand, q, api.StabilityProtocol.standard(), api.SimParams(), api.LossWeights(),
            api.OptConfig(iterations=500), k_begin=k, k_end=k + 1, adam_m=m, adam_v=v, record=True))
        assert not np.any(out["status"])
        r = oracle.optimize(s.ro, s.rh, q[:8], oracle.default_params(), iters=500, k_begin=k, k_end=k + 1,
                            adam_m=None if m is None else m[:8], adam_v=None if v is None else v[:8], record=True)
        assert np.array_equal(out["traj"][:8, :, :3], r["losses"])
        assert relerr(out["traj"][:8, :, 3:], r["grads"]) < GRAD_RTOL
        assert relerr(out["q"][:8], r["q"]) < GRAD_RTOL
        assert relerr(out["m"][:8], r["m"]) < GRAD_RTOL
        q, m, v = out["q"], out["m"], out["v"]


def test_lane_adjoint_correction_log_overflow_is_per_candidate():
    """A correction-log capacity of 70 through the lane adjoint: candidates that
    overflow report status 3, the others equal a default-capacity run
    bit-for-bit (the same lane path); statuses equal the CTA adjoint's."""
    from paper_2306_08132_b200 import api, init, model
    small, big = api.Context(0, correction_capacity=70), api.Context(0)
    hd = model.HandDesc.asset("allegro16")
    od = model.box_grid(res=32)
    q = init.approach_init(od, hd, 400, seed=9)
    proto, params = api.StabilityProtocol.standard(), api.SimParams(dilation_radius=0.01)
    res = {}
    for name, c in (("small", small), ("big", big)):
        hand, obj = api.Hand(c, hd), api.GraspObject(c, od)
        for variant in ("lane", "cta"):
            res[name, variant] = _run(c, variant, lambda: api.loss_gradient(c, obj, hand, q, proto, params))
    ls, gs, ss = res["small", "lane"]
    lb, gb, sb = res["big", "lane"]
    assert not np.any(sb)
    assert set(np.unique(ss).tolist()) <= {0, 3} and 0 < np.count_nonzero(ss == 3) < 400
    assert np.array_equal(ss, res["small", "cta"][2])
    ok = ss == 0
    assert np.array_equal(ls[ok], lb[ok]) and np.array_equal(gs[ok], gb[ok])


@pytest.mark.parametrize("gs", [1, 3])
def test_lane_adjoint_odd_sweep_count(ctx, oracle, gs):
    """gs * N even or odd: the reverse walk's last window may reach below
    position 0 (barrett3, N = 1999: gs = 1 / 3 give an even top position);
    sims without further corrections must not read the log there."""
    from paper_2306_08132_b200 import api
    s = Setup(ctx, oracle, "barrett3", _object("boxgrid64"), B=8, seed=94)
    q = np.tile(s.q, (TILE, 1))
    proto = api.StabilityProtocol.standard()
    params = api.SimParams(dilation_radius=0.015, gs_iters=gs)
    ll, gl, stl = _run(ctx, "lane", lambda: api.loss_gradient(ctx, s.obj, s.hand, q, proto, params))
    lc, gc, stc = _run(ctx, "cta", lambda: api.loss_gradient(ctx, s.obj, s.hand, q, proto, params))
    assert not np.any(stl) and np.array_equal(ll, lc)
    assert relerr(gl, gc) < LANE_VS_CTA_RTOL
    p = oracle.default_params(dilation_radius=0.015, gs_iters=gs)
    for b in range(4):
        rl, ds, dr, dl = oracle.loss_gradient(s.ro, s.rh, s.q[b], p)
        assert np.array_equal(ll[b], rl)
        assert relerr(gl[b, 0], ds) < GRAD_RTOL


@pytest.mark.parametrize("nvel", [1, 9, 48])
def test_lane_adjoint_protocol_sizes(ctx, oracle, nvel):
    """Any number of perturbation velocities through the lane adjoint (M = 1:
    32 candidates per warp; M = 9: velocities beyond KSim's inline 8 come from
    the device copy; M = 48: the epilogue's per-sim link sums need fewer
    candidates per CTA), vs the CTA adjoint."""
    from paper_2306_08132_b200 import api
    s = Setup(ctx, oracle, "allegro16", _object("boxgrid64"), B=8, seed=95)
    q = np.tile(s.q, (TILE, 1))
    base = api.StabilityProtocol.standard().velocities
    vel = [tuple(v) for v in base] + [(0.3, 0.3, 0.0), (0.0, 0.2, -0.4)]
    rng = np.random.default_rng(7)
    vel += [tuple(0.5 * d / np.linalg.norm(d)) for d in rng.normal(size=(48, 3))]
    proto = api.StabilityProtocol(vel[:nvel])
    params = api.SimParams(dilation_radius=0.015)
    ll, gl, stl = _run(ctx, "lane", lambda: api.loss_gradient(ctx, s.obj, s.hand, q, proto, params))
    lc, gc, stc = _run(ctx, "cta", lambda: api.loss_gradient(ctx, s.obj, s.hand, q, proto, params))
    assert not np.any(stl) and np.array_equal(ll, lc)
    assert relerr(gl, gc) < LANE_VS_CTA_RTOL
    for t in range(1, TILE):
        assert np.array_equal(gl[8 * t:8 * t + 8], gl[:8])


def test_lane_adjoint_nonfinite_rows_and_energy(ctx, oracle):
    """A NaN base position (free flight, gradient 0) and a NaN joint (status 1)
    in a lane-adjoint batch leave the other rows bit-identical; an optimizer
    iterate with the grasp-energy terms on agrees with the CTA adjoint."""
    from paper_2306_08132_b200 import api
    s = Setup(ctx, oracle, "allegro16", _object("boxgrid64"), B=8, seed=96)
    q = np.tile(s.q, (TILE, 1))
    proto, params = api.StabilityProtocol.standard(), api.SimParams(dilation_radius=0.01)
    bad = q.copy()
    bad[0, 0] = np.nan
    bad[1, 9] = np.nan
    lb, gb, sb = _run(ctx, "lane", lambda: api.loss_gradient(ctx, s.obj, s.hand, bad, proto, params))
    lo, go, so = _run(ctx, "lane", lambda: api.loss_gradient(ctx, s.obj, s.hand, q, proto, params))
    assert sb[0] == 0 and sb[1] == 1 and not np.any(sb[2:]) and not np.any(so)
    assert np.array_equal(lb[2:], lo[2:]) and np.array_equal(gb[2:], go[2:])
    assert np.array_equal(gb[0, 0], np.zeros_like(gb[0, 0]))
    w = api.LossWeights(force_closure=0.3, penetration=2.0, contact_threshold=0.004)
    opt = api.OptConfig(iterations=500)
    ol = _run(ctx, "lane", lambda: api.optimize(ctx, s.obj, s.hand, q, proto, api.SimParams(), w, opt,
                                                 k_begin=2, k_end=3, record=True))
    oc = _run(ctx, "cta", lambda: api.optimize(ctx, s.obj, s.hand, q, proto, api.SimParams(), w, opt,
                                                k_begin=2, k_end=3, record=True))
    assert not np.any(ol["status"]) and np.array_equal(ol["traj"][:, :, :3], oc["traj"][:, :, :3])
    assert relerr(ol["traj"][:, :, 3:], oc["traj"][:, :, 3:]) < LANE_VS_CTA_RTOL
    assert relerr(ol["q"], oc["q"]) < LANE_VS_CTA_RTOL


def test_lane_adjoint_chunks_equal_one_launch(ctx, monkeypatch):
    """A batch split over several lane-adjoint scratch chunks (a small scratch
    budget) gives the same rows bit-for-bit as one launch: per-task math does
    not depend on the chunk."""
    from paper_2306_08132_b200 import api, init, model
    hd = model.HandDesc.asset("allegro16")
    od = model.box_grid(res=64)
    hand, obj = api.Hand(ctx, hd), api.GraspObject(ctx, od)
    q = init.approach_init(od, hd, 2400, seed=21)
    proto, params = api.StabilityProtocol.standard(), api.SimParams(dilation_radius=0.015)
    one = _run(ctx, "lane", lambda: api.loss_gradient(ctx, obj, hand, q, proto, params))
    monkeypatch.setenv("DGX_SPLIT_SCRATCH_MB", "1")  # -> chunks of 4 waves of the forward grid
    ctx.set_kernel_timing(True)
    ctx.set_adjoint("lane")
    try:
        many = api.loss_gradient(ctx, obj, hand, q, proto, params)
        kt = ctx.kernel_times()
    finally:
        ctx.set_kernel_timing(False)
        ctx.set_adjoint("auto")
        monkeypatch.delenv("DGX_SPLIT_SCRATCH_MB")
    assert kt["adjoint"][1] >= 2, kt  # several chunks
    for a, b in zip(one, many):
        assert np.array_equal(a, b)
