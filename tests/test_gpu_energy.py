"""GPU: the grasp-energy terms of north_star (3) — force closure and
penetration (dgx_grasp_energy_batch). The reference objective has neither
(losses.hpp:47-93), so they are PARITY-UNPINNED: checked here against an
independent float64 numpy restatement of the definition in include/dgx.h on
the same contact sets:
  * energies: numpy sums over the reference's own FK points (oracle
    HandModel::forward) and SDF queries (oracle MeshSdf::dilated contract);
  * gradients: numpy dE/dp (contact set and normals frozen) pushed through a
    central-difference Jacobian of the reference FK in the [pos | tangent |
    joints] layout (tangent = quat_exp(t) (x) q0, hand.cpp:250-253).
Off by default: with zero weights the optimizer is bit-identical to no
energy; with weights the optimizer's weighted gradient is exactly the sum."""
import numpy as np
import pytest

from test_gpu_parity import Case, relerr

pytestmark = pytest.mark.gpu
THR, ELL = 0.004, 0.05


def qexp(v):
    a = np.linalg.norm(v)
    if a < 1e-300:
        return np.array([1.0, 0.0, 0.0, 0.0])
    return np.concatenate([[np.cos(a / 2)], np.sin(a / 2) * v / a])


def qmul(a, b):
    return np.array([a[0] * b[0] - a[1] * b[1] - a[2] * b[2] - a[3] * b[3],
                     a[0] * b[1] + a[1] * b[0] + a[2] * b[3] - a[3] * b[2],
                     a[0] * b[2] - a[1] * b[3] + a[2] * b[0] + a[3] * b[1],
                     a[0] * b[3] + a[1] * b[2] - a[2] * b[1] + a[3] * b[0]])


def perturb(q, d, h):
    out = q.copy()
    if d < 3:
        out[d] += h
    elif d < 6:
        e = np.zeros(3)
        e[d - 3] = h
        qq = qmul(qexp(e), q[3:7])
        out[3:7] = qq / np.linalg.norm(qq)
    else:
        out[7 + d - 6] += h
    return out


def numpy_energy(rh, ro, com, q, thr=THR, ell=ELL):
    P = rh.forward(q)
    Q = np.array([ro.query(p, 0.0) for p in P])
    rho, n = Q[:, 0], Q[:, 1:4]
    C = np.abs(rho) <= thr
    f = n[C].sum(axis=0)
    tau = np.cross(P[C] - com, n[C]).sum(axis=0)
    e_fc = f @ f + tau @ tau / ell ** 2
    pen = rho < 0
    e_pen = -rho[pen].sum()
    gfc = np.zeros_like(P)
    gfc[C] = 2.0 * np.cross(n[C], tau) / ell ** 2
    gpen = np.zeros_like(P)
    gpen[pen] = -n[pen]
    D = 6 + rh.num_joints
    h = 1e-6
    g = np.zeros((2, D))
    for d in range(D):
        Jd = (rh.forward(perturb(q, d, h)) - rh.forward(perturb(q, d, -h))) / (2 * h)
        g[0, d] = np.sum(gfc * Jd)
        g[1, d] = np.sum(gpen * Jd)
    return np.array([e_fc, e_pen]), g, int(C.sum()), int(pen.sum())


@pytest.mark.parametrize("hand_name,obj_name", [("barrett3", "sphere25"), ("allegro16", "boxgrid64"),
                                                ("barrett3", "cylgrid32")])
def test_energy_matches_numpy(ctx, oracle, hand_name, obj_name):
    from paper_2306_08132_b200 import api
    c = Case(ctx, oracle, hand_name, obj_name, B=4, seed=7, pull=0.5)
    e, g = api.grasp_energy(ctx, c.obj, c.hand, c.q, THR, ELL)
    n_con = n_pen = 0
    for b in range(4):
        er, gr, nc, npn = numpy_energy(c.rh, c.ro, c.od.com, c.q[b])
        n_con += nc
        n_pen += npn
        assert np.allclose(e[b], er, rtol=1e-12, atol=1e-15), (b, e[b], er)
        for t in range(2):
            if np.any(gr[t]):
                assert relerr(g[b, t], gr[t]) < 1e-6, (b, t, relerr(g[b, t], gr[t]))
            else:
                assert not np.any(g[b, t])
    assert n_con > 0 and n_pen > 0  # the cases exercise both terms


def test_energy_free_hand_is_zero(ctx, oracle):
    from paper_2306_08132_b200 import api
    c = Case(ctx, oracle, "barrett3", "sphere25", B=2)
    far = c.q.copy()
    far[:, :3] = [0.0, 0.0, -0.5]
    e, g = api.grasp_energy(ctx, c.obj, c.hand, far)
    assert not np.any(e) and not np.any(g)


@pytest.mark.parametrize("B", [4, 200])
def test_optimizer_energy_weights(ctx, oracle, B):
    """Zero weights: bit-identical to the default objective. Nonzero weights:
    the optimizer's recorded weighted gradient equals the default one plus
    w_fc dE_fc + w_pen dE_pen (fused path at B = 4, split path at B = 200),
    every iterate (energy recomputed at each iterate's q)."""
    from paper_2306_08132_b200 import api
    c = Case(ctx, oracle, "allegro16", "boxgrid64", B=B, seed=9, pull=0.5)
    proto, params, opt = api.StabilityProtocol.standard(), api.SimParams(), api.OptConfig(iterations=20)
    base = api.optimize(ctx, c.obj, c.hand, c.q, proto, params, api.LossWeights(), opt, k_begin=3, k_end=4,
                        record=True)
    zero = api.optimize(ctx, c.obj, c.hand, c.q, proto, params,
                        api.LossWeights(force_closure=0.0, penetration=0.0, contact_threshold=THR), opt, k_begin=3,
                        k_end=4, record=True)
    for k in ("q", "m", "v", "traj", "status"):
        assert np.array_equal(base[k], zero[k]), k
    w = api.LossWeights(force_closure=0.3, penetration=2.0, contact_threshold=THR, torque_scale=ELL)
    on = api.optimize(ctx, c.obj, c.hand, c.q, proto, params, w, opt, k_begin=3, k_end=4, record=True)
    _, g = api.grasp_energy(ctx, c.obj, c.hand, c.q, THR, ELL)
    assert not np.any(on["status"])
    want = base["traj"][:, 0, 3:] + (0.3 * g[:, 0] + 2.0 * g[:, 1])
    assert np.array_equal(on["traj"][:, 0, :3], base["traj"][:, 0, :3])
    assert np.allclose(on["traj"][:, 0, 3:], want, rtol=1e-13, atol=0)
    assert np.any(g[:, 1])
    # two iterates in one call: the second iterate's energy is taken at the updated q
    two = api.optimize(ctx, c.obj, c.hand, c.q, proto, params, w, opt, k_begin=3, k_end=5, record=True)
    _, g1 = api.grasp_energy(ctx, c.obj, c.hand, on["q"], THR, ELL)
    base1 = api.optimize(ctx, c.obj, c.hand, on["q"], proto, params, api.LossWeights(), opt, k_begin=4, k_end=5,
                         adam_m=on["m"], adam_v=on["v"], record=True)
    assert np.allclose(two["traj"][:, 1, 3:], base1["traj"][:, 0, 3:] + (0.3 * g1[:, 0] + 2.0 * g1[:, 1]),
                       rtol=1e-13, atol=0)
