"""GPU: StabilityProtocol beyond the standard 7 velocities (losses.hpp:16-27
takes any std::vector<Vec3>): M = 1, 3, 9, 12 perturbation sims per candidate
(a CTA has min(M, 7) warps; warp w runs sims w, w + 7, ...; M > 8 passes the
velocity list through dgx_params.velocity_list), checked against the
reference with the same velocity list (oracle.protocol). Residuals, losses
and SolveStats bit-exact; gradients within GRAD_RTOL. Fused (B <= #SMs) and
split (B > #SMs) execution."""
import numpy as np
import pytest

from test_gpu_parity import GRAD_RTOL, Case, relerr

pytestmark = pytest.mark.gpu

S = 0.5
STD = [(S, 0, 0), (-S, 0, 0), (0, S, 0), (0, -S, 0), (0, 0, S), (0, 0, -S), (0, 0, 0)]
PROTOS = {1: [(0.0, 0.0, -0.4)], 3: STD[4:7],
          9: STD + [(0.3, 0.3, 0.0), (0.0, 0.2, -0.4)],
          12: STD + [(0.3, 0.3, 0.0), (0.0, 0.2, -0.4), (-0.25, 0.1, 0.2), (0.1, -0.3, 0.3), (0.05, 0.05, 0.6)]}


@pytest.mark.parametrize("M", sorted(PROTOS))
@pytest.mark.parametrize("hand_name,obj_name,B", [("barrett3", "sphere25", 2), ("allegro16", "boxgrid64", 160)])
def test_protocol_velocities(ctx, oracle, M, hand_name, obj_name, B):
    from paper_2306_08132_b200 import api
    c = Case(ctx, oracle, hand_name, obj_name, B=B, seed=13 + M)
    vel = PROTOS[M]
    proto = api.StabilityProtocol(vel)
    params = api.SimParams(dilation_radius=0.015)
    p = oracle.default_params(dilation_radius=0.015)
    losses, grads, st = api.loss_gradient(ctx, c.obj, c.hand, c.q, proto, params)
    el, stats, st2 = api.evaluate_losses(ctx, c.obj, c.hand, c.q, proto, params)
    assert stats.shape == (B, M, 5)
    rows = [0, 1] if B == 2 else [0, 77, 159]
    res, g, _, st3 = api.debug_sims(ctx, c.obj, c.hand, c.q[rows], proto, params)
    assert not np.any(st) and not np.any(st2) and not np.any(st3)
    active = 0
    with oracle.protocol(vel):
        for i, b in enumerate(rows):
            rl, ds, dr, dl = oracle.loss_gradient(c.ro, c.rh, c.q[b], p)
            assert np.array_equal(losses[b], rl), (b, losses[b], rl)
            assert relerr(grads[b, 0], ds) < GRAD_RTOL
            assert np.array_equal(el[b], oracle.evaluate_losses(c.ro, c.rh, c.q[b], p))
            for m in range(M):
                rres, rg, _, log = oracle.sim_record(c.ro, c.rh, c.q[b], m, p)
                active += int(np.sum(log < 0))
                assert res[i, m] == rres, (b, m)
                assert relerr(g[i, m], rg) < GRAD_RTOL, (b, m)
                _, rst, _ = oracle.sim_forward(c.ro, c.rh, c.q[b], m, p)
                assert np.array_equal(stats[b, m], rst), (b, m)
    assert active > 0


def test_protocol_optimizer_m9(ctx, oracle):
    """One teacher-forced optimizer step with M = 9 (split execution)."""
    from paper_2306_08132_b200 import api
    c = Case(ctx, oracle, "allegro16", "boxgrid64", B=160, seed=5, pull=0.3)
    vel = PROTOS[9]
    out = api.optimize(ctx, c.obj, c.hand, c.q, api.StabilityProtocol(vel), api.SimParams(), api.LossWeights(),
                       api.OptConfig(iterations=10), k_begin=2, k_end=3, record=True)
    rows = [0, 80, 159]
    with oracle.protocol(vel):
        r = oracle.optimize(c.ro, c.rh, c.q[rows], oracle.default_params(), iters=10, k_begin=2, k_end=3,
                            record=True)
    assert not np.any(out["status"]) and not np.any(r["status"])
    assert np.array_equal(out["traj"][rows, :, :3], r["losses"])
    assert relerr(out["traj"][rows, :, 3:], r["grads"]) < GRAD_RTOL
    assert relerr(out["q"][rows], r["q"]) < GRAD_RTOL


@pytest.mark.parametrize("T", [2, 3])
@pytest.mark.parametrize("hand_name,obj_name,B", [("barrett3", "sphere25", 2), ("allegro16", "boxgrid64", 160),
                                                  ("barrett3", "ico25", 2), ("pincher2", "box40", 2)])
def test_protocol_steps(ctx, oracle, T, hand_name, obj_name, B):
    """StabilityProtocol::steps = T > 1 (losses.hpp:54-55): T predict + solve
    steps per perturbation sim, the reverse through every step's solve, its
    friction's and finalize's dependence on the previous state, and predict
    (quat_exp of the carried angular velocity). Residuals / losses / stats
    bit-exact, gradients within GRAD_RTOL of the reference tape."""
    from paper_2306_08132_b200 import api
    c = Case(ctx, oracle, hand_name, obj_name, B=B, seed=29 + T)
    proto = api.StabilityProtocol.standard(steps=T)
    params = api.SimParams(dilation_radius=0.015)
    p = oracle.default_params(dilation_radius=0.015, steps=T)
    losses, grads, st = api.loss_gradient(ctx, c.obj, c.hand, c.q, proto, params)
    el, stats, st2 = api.evaluate_losses(ctx, c.obj, c.hand, c.q, proto, params)
    rows = [0, 1] if B == 2 else [0, 99, 159]
    res, g, _, st3 = api.debug_sims(ctx, c.obj, c.hand, c.q[rows], proto, params)
    assert not np.any(st) and not np.any(st2) and not np.any(st3)
    active = 0
    for i, b in enumerate(rows):
        rl, ds, dr, dl = oracle.loss_gradient(c.ro, c.rh, c.q[b], p)
        assert np.array_equal(losses[b], rl), (b, losses[b], rl)
        assert relerr(grads[b, 0], ds) < GRAD_RTOL, (b, relerr(grads[b, 0], ds))
        assert np.array_equal(el[b], oracle.evaluate_losses(c.ro, c.rh, c.q[b], p))
        for m in range(7):
            rres, rg, _, log = oracle.sim_record(c.ro, c.rh, c.q[b], m, p)
            active += int(np.sum(log < 0))
            assert res[i, m] == rres, (b, m)
            assert relerr(g[i, m], rg) < GRAD_RTOL, (b, m, relerr(g[i, m], rg))
            _, rst, _ = oracle.sim_forward(c.ro, c.rh, c.q[b], m, p)
            assert np.array_equal(stats[b, m], rst), (b, m, stats[b, m], rst)
    assert active > 0


def test_protocol_steps_optimizer(ctx, oracle):
    """Teacher-forced optimizer steps with T = 2."""
    from paper_2306_08132_b200 import api
    c = Case(ctx, oracle, "allegro16", "boxgrid64", B=3, seed=8, pull=0.3)
    q, m, v = c.q, None, None
    for k in range(2):
        g = api.optimize(ctx, c.obj, c.hand, q, api.StabilityProtocol.standard(steps=2), api.SimParams(),
                         api.LossWeights(), api.OptConfig(iterations=6), k_begin=k, k_end=k + 1, adam_m=m, adam_v=v,
                         record=True)
        r = oracle.optimize(c.ro, c.rh, q, oracle.default_params(steps=2), iters=6, k_begin=k, k_end=k + 1, adam_m=m,
                            adam_v=v, record=True)
        assert not np.any(g["status"]) and not np.any(r["status"])
        assert np.array_equal(g["traj"][:, :, :3], r["losses"])
        assert relerr(g["traj"][:, :, 3:], r["grads"]) < GRAD_RTOL
        assert relerr(g["q"], r["q"]) < GRAD_RTOL
        q, m, v = r["q"], r["m"], r["v"]
