"""GPU parity: the CUDA path through the C-ABI vs the compiled reference.

Bars:
  * forward values — FK points, per-perturbation residuals, losses,
    evaluate_losses, SolveStats (contact culling / indexing) — BIT-EXACT
    against the parity-mode oracle (libdgref_sm: the reference with the
    kernels' deterministic sin/cos/atan2);
  * gradients (per perturbation, per point, total) within rel GRAD_RTOL = 1e-8
    of the reference tape. The tape sums adjoints in node order, the kernel in
    closed form, so results differ by rounding amplified along correction
    chains: typically ~1e-13, and over the 43k-sim random fuzz
    (profiles/r01/parity_fuzz.jsonl) the worst case was 3.2e-9 at |grad| ~
    1e17-1e22. The bar is set above that distribution (not tuned to the chosen
    inputs) and is still 4 orders inside north_star's rel 1e-4;
  * one optimizer step from the oracle's iterate (teacher forcing): losses
    bit-exact, q_{k+1} within GRAD_RTOL (north_star: FP32-level rel 1e-4);
  * against the UNMODIFIED reference (glibc libm): losses within rel 1e-6.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GRAD_RTOL = 1e-8  # see the module docstring: fuzz worst case 3.2e-9


def relerr(a, b):
    a, b = np.asarray(a), np.asarray(b)
    den = np.max(np.abs(b))
    return 0.0 if den == 0 and np.max(np.abs(a)) == 0 else float(np.max(np.abs(a - b)) / max(den, 1e-300))


def ref_hand(oracle, name, variant="sm"):
    if name == "barrett3":
        return oracle.RefHand.barrett3(variant=variant)
    if name == "pincher2":
        return oracle.RefHand.pincher2(variant=variant)
    return oracle.RefHand.load_xml(os.path.join(ROOT, "assets", "hands", name, name + ".xml"), 2000, 12345,
                                   variant=variant)


def make_obj(name):
    from paper_2306_08132_b200 import model
    return {"sphere25": lambda: model.sphere(0.025), "box40": lambda: model.box((0.04, 0.04, 0.04)),
            "boxgrid64": lambda: model.box_grid(res=64), "cylgrid32": lambda: model.cylinder_grid(res=32),
            # triangle meshes: the oracle runs the UNMODIFIED reference MeshSdf
            "ico25": lambda: model.mesh_object(*model.icosphere_mesh(0.025, 3)),
            "boxmesh40": lambda: model.mesh_object(*model.box_mesh((0.04, 0.04, 0.04)))}[name]()


class Case:
    def __init__(self, ctx, oracle, hand_name, obj_name, B=3, seed=0, pull=0.45, variant="sm"):
        from paper_2306_08132_b200 import api, init, model
        self.rh = ref_hand(oracle, hand_name, variant)
        self.hd = model.HandDesc.from_dict(hand_name, self.rh.desc)
        self.od = make_obj(obj_name)
        self.ro = oracle.RefObject.from_desc(self.od, variant=variant)
        self.hand, self.obj = api.Hand(ctx, self.hd), api.GraspObject(ctx, self.od)
        q = init.approach_init(self.od, self.hd, B, seed=seed)
        q[:, :3] -= pull * (q[:, :3] - self.od.com)
        self.q = q


COMBOS = [("barrett3", "sphere25"), ("pincher2", "box40"), ("allegro16", "boxgrid64"), ("barrett3", "cylgrid32"),
          ("barrett3", "ico25"), ("pincher2", "boxmesh40")]


@pytest.mark.parametrize("hand_name,obj_name", COMBOS)
def test_forward_points_bit_exact(ctx, oracle, hand_name, obj_name):
    from paper_2306_08132_b200 import api
    c = Case(ctx, oracle, hand_name, obj_name, B=5, seed=11)
    pts = api.forward(ctx, c.hand, c.q)
    for b in range(c.q.shape[0]):
        assert np.array_equal(pts[b], c.rh.forward(c.q[b]))


@pytest.mark.parametrize("radius", [0.0, 0.01, 0.02])
@pytest.mark.parametrize("hand_name,obj_name", COMBOS)
def test_per_perturbation_sims(ctx, oracle, hand_name, obj_name, radius):
    """Residual of every perturbation sim bit-exact (=> identical activation /
    correction sequence); per-sim and per-point gradients vs the tape."""
    from paper_2306_08132_b200 import api
    c = Case(ctx, oracle, hand_name, obj_name, B=2, seed=3)
    proto, params = api.StabilityProtocol.standard(), api.SimParams(dilation_radius=radius)
    res, g, gp, st = api.debug_sims(ctx, c.obj, c.hand, c.q, proto, params, point_grads=True)
    assert not np.any(st)
    p = oracle.default_params(dilation_radius=radius)
    n_active = 0
    for b in range(c.q.shape[0]):
        for m in range(7):
            rres, rg, rgp, log = oracle.sim_record(c.ro, c.rh, c.q[b], m, p, points_grad=True)
            n_active += int(np.sum(log < 0))
            assert res[b, m] == rres, (b, m)
            assert relerr(g[b, m], rg) < GRAD_RTOL, (b, m, relerr(g[b, m], rg))
            assert relerr(gp[b, m], rgp) < GRAD_RTOL, (b, m)
    if radius > 0:
        assert n_active > 0  # the case actually exercises contacts


@pytest.mark.parametrize("hand_name,obj_name", COMBOS)
def test_loss_gradient_and_evaluate(ctx, oracle, hand_name, obj_name):
    from paper_2306_08132_b200 import api
    c = Case(ctx, oracle, hand_name, obj_name, B=4, seed=5)
    proto = api.StabilityProtocol.standard()
    for radius in (0.0, 0.015):
        params = api.SimParams(dilation_radius=radius)
        p = oracle.default_params(dilation_radius=radius)
        losses, grads, st = api.loss_gradient(ctx, c.obj, c.hand, c.q, proto, params)
        el, stats, st2 = api.evaluate_losses(ctx, c.obj, c.hand, c.q, proto, params)
        assert not np.any(st) and not np.any(st2)
        for b in range(c.q.shape[0]):
            rl, ds, dr, dl = oracle.loss_gradient(c.ro, c.rh, c.q[b], p)
            assert np.array_equal(losses[b], rl)
            assert relerr(grads[b, 0], ds) < GRAD_RTOL
            assert relerr(grads[b, 1], dr) < GRAD_RTOL
            assert np.array_equal(grads[b, 2], dl)
            assert np.array_equal(el[b], oracle.evaluate_losses(c.ro, c.rh, c.q[b], p))
            for m in range(7):
                _, rst, _ = oracle.sim_forward(c.ro, c.rh, c.q[b], m, p)
                assert np.array_equal(stats[b, m], rst), (b, m, stats[b, m], rst)


def test_golden_fixtures(ctx, oracle):
    """Committed reference outputs (tests/golden) reproduced by the CUDA path."""
    import glob
    from paper_2306_08132_b200 import api
    for path in sorted(glob.glob(os.path.join(ROOT, "tests", "golden", "*.npz"))):
        z = np.load(path)
        hand_name, obj_name = os.path.basename(path)[:-4].split("_")
        c = Case(ctx, oracle, hand_name, obj_name, B=1)
        q = z["q"]
        params = api.SimParams(dilation_radius=float(z["radius"]))
        proto = api.StabilityProtocol.standard()
        losses, grads, st = api.loss_gradient(ctx, c.obj, c.hand, q, proto, params)
        assert np.array_equal(losses, z["sm_losses"]), path
        assert relerr(grads[:, 0], z["sm_d_stable"]) < GRAD_RTOL
        assert np.all(np.abs(losses[:, 0] - z["glibc_losses"][:, 0]) <= 1e-6 * np.abs(z["glibc_losses"][:, 0]))
        el, stats, _ = api.evaluate_losses(ctx, c.obj, c.hand, q, proto, params)
        assert np.array_equal(el, z["sm_eval"]) and np.array_equal(stats, z["sm_stats"])
        res, g, _, _ = api.debug_sims(ctx, c.obj, c.hand, q, proto, params)
        assert np.array_equal(res, z["sm_sim_res"])
        assert relerr(g, z["sm_sim_grads"]) < GRAD_RTOL
        # teacher-forced optimizer step k=3 -> 4 of a 10-iteration schedule
        out = api.optimize(ctx, c.obj, c.hand, z["sm_opt_q3"], proto, api.SimParams(), api.LossWeights(),
                           api.OptConfig(iterations=10), k_begin=3, k_end=4, adam_m=z["sm_opt_m3"],
                           adam_v=z["sm_opt_v3"], record=True)
        assert not np.any(out["status"])
        assert np.array_equal(out["traj"][:, :, :3], z["sm_opt_traj_losses"])
        assert relerr(out["traj"][:, :, 3:], z["sm_opt_traj_grads"]) < GRAD_RTOL
        assert relerr(out["q"], z["sm_opt_q4"]) < GRAD_RTOL
        assert relerr(out["m"], z["sm_opt_m4"]) < GRAD_RTOL
        assert relerr(out["v"], z["sm_opt_v4"]) < 1e-8


@pytest.mark.parametrize("hand_name,obj_name", [("barrett3", "sphere25"), ("allegro16", "boxgrid64")])
def test_teacher_forced_optimizer(ctx, oracle, hand_name, obj_name):
    """Every step of a short run, each started from the oracle's own iterate."""
    from paper_2306_08132_b200 import api
    c = Case(ctx, oracle, hand_name, obj_name, B=2, seed=9, pull=0.3)
    K = 6
    proto, w = api.StabilityProtocol.standard(), api.LossWeights()
    q, m, v = c.q, None, None
    for k in range(K):
        r = oracle.optimize(c.ro, c.rh, q, oracle.default_params(), iters=K, k_begin=k, k_end=k + 1, adam_m=m,
                            adam_v=v, record=True)
        g = api.optimize(ctx, c.obj, c.hand, q, proto, api.SimParams(), w, api.OptConfig(iterations=K), k_begin=k,
                         k_end=k + 1, adam_m=m, adam_v=v, record=True)
        assert not np.any(g["status"]) and not np.any(r["status"])
        assert np.array_equal(g["traj"][:, :, :3], r["losses"]), k
        assert relerr(g["traj"][:, :, 3:], r["grads"]) < GRAD_RTOL
        assert relerr(g["q"], r["q"]) < GRAD_RTOL, k
        q, m, v = r["q"], r["m"], r["v"]


def test_against_unmodified_reference(ctx, oracle):
    """GPU vs the glibc build (the reference exactly): same objective to rounding."""
    from paper_2306_08132_b200 import api
    c = Case(ctx, oracle, "allegro16", "boxgrid64", B=4, seed=21, variant="glibc")
    params, proto = api.SimParams(dilation_radius=0.02), api.StabilityProtocol.standard()
    losses, grads, st = api.loss_gradient(ctx, c.obj, c.hand, c.q, proto, params)
    for b in range(4):
        rl, ds, dr, dl = oracle.loss_gradient(c.ro, c.rh, c.q[b], oracle.default_params(dilation_radius=0.02))
        assert abs(losses[b, 0] - rl[0]) <= 1e-6 * abs(rl[0])
        assert relerr(grads[b, 0], ds) < 1e-4  # north_star tolerance; differs only at rounding-decided contacts


def test_edge_cases(ctx, oracle):
    from paper_2306_08132_b200 import api
    c = Case(ctx, oracle, "barrett3", "sphere25", B=3, seed=1)
    proto = api.StabilityProtocol.standard()
    # no contact: free flight 6s/7, gradient exactly zero
    far = c.q.copy()
    far[:, :3] = [0.0, 0.0, -0.5]
    losses, grads, st = api.loss_gradient(ctx, c.obj, c.hand, far, proto, api.SimParams(dilation_radius=0.01))
    assert np.allclose(losses[:, 0], 3 / 7, rtol=1e-15, atol=0)
    assert not np.any(grads[:, 0])
    # joints outside / exactly at the limits (tie rule +-1)
    q = c.q.copy()
    q[0, 7] = c.hd.upper[0] + 0.1
    q[1, 7] = c.hd.upper[0]
    q[2, 7 + 5] = c.hd.lower[5] - 0.05
    losses, grads, st = api.loss_gradient(ctx, c.obj, c.hand, q, proto, api.SimParams())
    for b in range(3):
        rl, ds, dr, dl = oracle.loss_gradient(c.ro, c.rh, q[b], oracle.default_params())
        assert np.array_equal(losses[b], rl) and np.array_equal(grads[b, 2], dl)
    # leak 0, mu 0, gs_iters 1: still exact
    for sp in (api.SimParams(dilation_radius=0.01, alpha_leak=0.0), api.SimParams(dilation_radius=0.01, mu=0.0),
               api.SimParams(dilation_radius=0.01, gs_iters=1)):
        losses, grads, st = api.loss_gradient(ctx, c.obj, c.hand, c.q, proto, sp)
        rp = oracle.default_params(dilation_radius=0.01, alpha_leak=sp.alpha_leak, mu=sp.mu, gs_iters=sp.gs_iters)
        for b in range(3):
            rl, ds, dr, dl = oracle.loss_gradient(c.ro, c.rh, c.q[b], rp)
            assert np.array_equal(losses[b], rl)
            assert relerr(grads[b, 0], ds) < GRAD_RTOL
    # empty batch is a no-op; B=1 works
    l0, g0, s0 = api.loss_gradient(ctx, c.obj, c.hand, c.q[:0], proto, api.SimParams())
    assert l0.shape == (0, 3)
    l1, g1, s1 = api.loss_gradient(ctx, c.obj, c.hand, c.q[:1], proto, api.SimParams(dilation_radius=0.01))
    l3, g3, s3 = api.loss_gradient(ctx, c.obj, c.hand, c.q, proto, api.SimParams(dilation_radius=0.01))
    assert np.array_equal(l1[0], l3[0]) and np.array_equal(g1[0], g3[0])


def test_invalid_arguments(ctx, oracle):
    from paper_2306_08132_b200 import api, capi
    c = Case(ctx, oracle, "barrett3", "sphere25", B=1)
    with pytest.raises(ValueError):
        api.loss_gradient(ctx, c.obj, c.hand, c.q, api.StabilityProtocol.standard(),
                          api.SimParams(dilation_radius=-0.1))
    with pytest.raises(capi.DgxError) as e:
        api.loss_gradient(ctx, c.obj, c.hand, c.q, api.StabilityProtocol.standard(steps=0), api.SimParams())
    assert e.value.code == 100
    # NaN configuration: like the reference, every SDF gate sees NaN (inactive),
    # the sim is untouched, the loss is the free-flight constant, gradient 0
    bad = c.q.copy()
    bad[0, 0] = np.nan
    losses, grads, st = api.loss_gradient(ctx, c.obj, c.hand, bad, api.StabilityProtocol.standard(),
                                          api.SimParams(dilation_radius=0.01))
    rl, ds, dr, dl = oracle.loss_gradient(c.ro, c.rh, bad[0], oracle.default_params(dilation_radius=0.01))
    assert np.array_equal(losses[0], rl) and np.array_equal(grads[0, 0], ds)


def test_nonfinite_adjoint_matches_reference(ctx, oracle):
    """Error behaviour: at an iterate (tests/golden/errors, from
    tools/make_nonfinite_fixture.py) where the reference's tape throws
    "non-finite adjoint" (tape.cpp:35-38) on a procedural blob mesh, the GPU
    reports DGX_E_NONFINITE_GRAD for that candidate; the forward-only objective
    still matches bit-exactly."""
    from paper_2306_08132_b200 import api, capi, model
    z = np.load(os.path.join(ROOT, "tests", "golden", "errors", "nonfinite_adjoint_blob.npz"))
    rad, sub, amp, seed = z["blob"]
    ro_mesh = oracle.RefObject.blob_mesh(float(rad), int(sub), float(amp), int(seed))
    od = model.mesh_object(*ro_mesh.mesh_export()[:2])
    ro = oracle.RefObject.from_desc(od)
    rh = oracle.RefHand.barrett3()
    hd = model.HandDesc.from_dict("barrett3", rh.desc)
    hand, obj = api.Hand(ctx, hd), api.GraspObject(ctx, od)
    r = float(z["radius"])
    with pytest.raises(oracle.RefError, match="non-finite adjoint"):
        oracle.loss_gradient(ro, rh, z["q"], oracle.default_params(dilation_radius=r))
    losses, grads, st = api.loss_gradient(ctx, obj, hand, z["q"][None, :], api.StabilityProtocol.standard(),
                                          api.SimParams(dilation_radius=r))
    assert capi.STATUS_NAMES[int(st[0])] == "tape: non-finite adjoint"
    # the forward-only objective is unaffected and bit-exact
    el, _, st2 = api.evaluate_losses(ctx, obj, hand, z["q"][None, :], api.StabilityProtocol.standard(),
                                     api.SimParams(dilation_radius=r))
    assert not np.any(st2)
    assert np.array_equal(el[0], oracle.evaluate_losses(ro, rh, z["q"], oracle.default_params(dilation_radius=r)))


def test_nonfinite_configuration_grid(ctx, oracle):
    """Non-finite inputs on the FP32 grid backend. The cell index of a NaN point
    is clamped like an outside point, so the NaN reaches rho instead of an
    address (this used to be an illegal memory access).
    * A NaN base position leaves every gate inactive: free flight, gradient 0,
      bit-exact with the reference.
    * A NaN joint angle: the reference returns non-finite losses (its zero-depth
      axpy multiplies NaN coefficients by 0); the GPU flags the candidate
      non-finite (status 1). The values of a non-finite candidate are not
      compared.
    * In a 200-candidate batch (split execution) the other rows are unaffected."""
    from paper_2306_08132_b200 import api
    c = Case(ctx, oracle, "allegro16", "boxgrid64", B=200)
    params = api.SimParams(dilation_radius=0.01)
    proto = api.StabilityProtocol.standard()
    bad = c.q.copy()
    bad[0, 0] = np.nan
    bad[1, 9] = np.nan
    losses, grads, st = api.loss_gradient(ctx, c.obj, c.hand, bad, proto, params)
    l_ok, g_ok, s_ok = api.loss_gradient(ctx, c.obj, c.hand, c.q, proto, params)
    assert np.array_equal(losses[2:], l_ok[2:]) and np.array_equal(grads[2:], g_ok[2:])
    assert np.array_equal(st[2:], s_ok[2:])
    rl, ds, dr, dl = oracle.loss_gradient(c.ro, c.rh, bad[0], oracle.default_params(dilation_radius=0.01))
    assert st[0] == 0 and np.array_equal(losses[0], rl) and np.array_equal(grads[0, 0], ds)
    rl1, _, _, _ = oracle.loss_gradient(c.ro, c.rh, bad[1], oracle.default_params(dilation_radius=0.01))
    assert not np.all(np.isfinite(rl1)) and st[1] == 1
    # forward-only evaluation: no crash, the NaN candidate is flagged, the others are unaffected
    el, est, es = api.evaluate_losses(ctx, c.obj, c.hand, bad, proto, params)
    el_ok, _, es_ok = api.evaluate_losses(ctx, c.obj, c.hand, c.q, proto, params)
    assert es[1] != 0 and np.array_equal(el[2:], el_ok[2:]) and np.array_equal(es[2:], es_ok[2:])
