"""GPU: size-independent properties at full BASELINE sizes, and the
distribution-level parity of full untethered runs (north_star: "distributions
of final grasp contact count and penetration must agree over full runs")."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def setup(ctx, hand="allegro16", obj="box", B=1024, seed=17):
    from paper_2306_08132_b200 import api, init, model
    hd = model.HandDesc.asset(hand)
    od = model.box_grid(res=64) if obj == "box" else model.cylinder_grid(res=64)
    q = init.approach_init(od, hd, B, seed=seed)
    return hd, od, api.Hand(ctx, hd), api.GraspObject(ctx, od), q


def test_full_batch_deterministic_and_shard_independent(ctx):
    """Config 2 size (1024 candidates): identical results across runs, and any
    contiguous shard computed alone equals the same rows of the full batch
    (the multi-GPU partition cannot change results)."""
    from paper_2306_08132_b200 import api
    hd, od, hand, obj, q = setup(ctx)
    proto, params = api.StabilityProtocol.standard(), api.SimParams(dilation_radius=0.02)
    l1, g1, s1 = api.loss_gradient(ctx, obj, hand, q, proto, params)
    l2, g2, s2 = api.loss_gradient(ctx, obj, hand, q, proto, params)
    assert not np.any(s1)
    assert np.array_equal(l1, l2) and np.array_equal(g1, g2)
    for lo, hi in ((0, 256), (256, 512), (700, 1024)):
        ls, gs, ss = api.loss_gradient(ctx, obj, hand, q[lo:hi], proto, params)
        assert np.array_equal(ls, l1[lo:hi]) and np.array_equal(gs, g1[lo:hi])
    # a multi-iteration fused run equals the same iterations one launch at a time
    opt = api.OptConfig(iterations=500)
    w = api.LossWeights()
    a = api.optimize(ctx, obj, hand, q[:64], proto, api.SimParams(), w, opt, k_begin=0, k_end=4)
    b = dict(q=q[:64], m=None, v=None)
    for k in range(4):
        b = api.optimize(ctx, obj, hand, b["q"], proto, api.SimParams(), w, opt, k_begin=k, k_end=k + 1,
                         adam_m=b["m"], adam_v=b["v"])
    assert np.array_equal(a["q"], b["q"]) and np.array_equal(a["m"], b["m"])


def test_full_run_finite_and_stats(ctx):
    from paper_2306_08132_b200 import api
    hd, od, hand, obj, q = setup(ctx, obj="cyl", B=256)
    out = api.optimize(ctx, obj, hand, q, api.StabilityProtocol.standard(), api.SimParams(), api.LossWeights(),
                       api.OptConfig(iterations=40), record=True)
    assert not np.any(out["status"])
    assert np.all(np.isfinite(out["traj"]))
    assert np.allclose(np.linalg.norm(out["q"][:, 3:7], axis=1), 1.0, atol=1e-12)
    el, stats, st = api.evaluate_losses(ctx, obj, hand, out["q"], api.StabilityProtocol.standard(), api.SimParams())
    assert not np.any(st) and np.all(el[:, 0] >= 0)
    assert np.all(stats[:, :, 1] >= stats[:, :, 0])  # corrections >= distinct contacts


def test_distribution_parity_full_runs(ctx, oracle):
    """Untethered runs diverge at rounding-decided contacts, so
    full runs are compared at the distribution level: final stability loss,
    contact count and penetration (evaluate at dilation 0) — two-sample KS."""
    from scipy.stats import ks_2samp
    from paper_2306_08132_b200 import api
    hd, od, hand, obj, q = setup(ctx, B=32, seed=99)
    q[:, :3] -= 0.3 * (q[:, :3] - od.com)
    K = 30
    proto, w = api.StabilityProtocol.standard(), api.LossWeights()
    g = api.optimize(ctx, obj, hand, q, proto, api.SimParams(), w, api.OptConfig(iterations=K))
    rh = oracle.RefHand.load_xml(os.path.join(ROOT, "assets", "hands", "allegro16", "allegro16.xml"), 2000, 12345,
                                 variant="sm")
    ro = oracle.RefObject.from_desc(od, variant="sm")
    r = oracle.optimize(ro, rh, q, oracle.default_params(), iters=K)
    assert not np.any(g["status"]) and not np.any(r["status"])
    el, stats, _ = api.evaluate_losses(ctx, obj, hand, g["q"], proto, api.SimParams())
    rl, rstats = [], []
    for b in range(q.shape[0]):
        rl.append(oracle.evaluate_losses(ro, rh, r["q"][b], oracle.default_params()))
        rstats.append([oracle.sim_forward(ro, rh, r["q"][b], m, oracle.default_params())[1] for m in range(7)])
    rl, rstats = np.array(rl), np.array(rstats)
    contacts_g, contacts_r = stats[:, :, 0].sum(1), rstats[:, :, 0].sum(1)
    pen_g, pen_r = stats[:, :, 3].max(1), rstats[:, :, 3].max(1)
    for a, b in ((el[:, 0], rl[:, 0]), (contacts_g, contacts_r), (pen_g, pen_r)):
        assert ks_2samp(a, b).pvalue > 0.01, (a, b)
    # (individual trajectories are NOT compared: the first rounding-decided
    # re-activation after a 1-ulp difference in q sends each run its own way;
    # per-step agreement is covered by test_teacher_forced_optimizer)


def test_multi_object_launch_matches_per_object(ctx):
    """dgx_optimize_multi (objects on concurrent side streams) == one optimize per object, bitwise."""
    from paper_2306_08132_b200 import api, init, model
    hd = model.HandDesc.asset("allegro16")
    ods = [model.box_grid(res=64), model.cylinder_grid(res=32), model.sphere(0.03)]
    hand = api.Hand(ctx, hd)
    objs = [api.GraspObject(ctx, o) for o in ods]
    counts = [40, 0, 25]
    qs = [init.approach_init(o, hd, n, seed=5 + i) for i, (o, n) in enumerate(zip(ods, counts))]
    q = np.concatenate(qs, axis=0)
    proto, w, opt = api.StabilityProtocol.standard(), api.LossWeights(), api.OptConfig(iterations=50)
    multi = api.optimize_multi(ctx, objs, hand, q, counts, proto, api.SimParams(), w, opt, k_begin=0, k_end=3,
                               record=True)
    assert not np.any(multi["status"])
    off = 0
    for o, n, qi in zip(objs, counts, qs):
        if n == 0:
            continue
        one = api.optimize(ctx, o, hand, qi, proto, api.SimParams(), w, opt, k_begin=0, k_end=3, record=True)
        assert np.array_equal(one["q"], multi["q"][off:off + n])
        assert np.array_equal(one["m"], multi["m"][off:off + n])
        assert np.array_equal(one["traj"], multi["traj"][off:off + n])
        off += n


def test_optimize_multi_inplace_host_path(ctx):
    """The pinned / in-place host path of optimize_multi (bench e2e) equals the
    copying host path and the device path."""
    import torch
    from paper_2306_08132_b200 import api, init, model
    hd = model.HandDesc.asset("barrett3")
    od = model.sphere(0.025)
    hand, obj = api.Hand(ctx, hd), api.GraspObject(ctx, od)
    q0 = init.approach_init(od, hd, 12, seed=9)
    proto, params, w, opt = api.StabilityProtocol.standard(), api.SimParams(), api.LossWeights(), api.OptConfig(50)
    counts = np.array([12], np.int32)
    a = api.optimize_multi(ctx, [obj], hand, q0, counts, proto, params, w, opt, k_begin=0, k_end=3, record=True)
    pin = lambda x: torch.tensor(x).pin_memory().numpy()  # noqa: E731
    q, m, v = pin(q0), pin(np.zeros((12, 6 + hd.num_joints))), pin(np.zeros((12, 6 + hd.num_joints)))
    b = api.optimize_multi(ctx, [obj], hand, q, counts, proto, params, w, opt, k_begin=0, k_end=3, adam_m=m,
                           adam_v=v, record=True, inplace=True)
    assert b["q"] is q and np.array_equal(q, a["q"]) and np.array_equal(m, a["m"]) and np.array_equal(v, a["v"])
    assert np.array_equal(b["traj"], a["traj"]) and not np.any(b["status"])
    with pytest.raises(ValueError):
        api.optimize_multi(ctx, [obj], hand, q0.astype(np.float32), counts, proto, params, w, opt, k_begin=0,
                           k_end=1, adam_m=m, adam_v=v, inplace=True)


def test_optimize_multi_mixed_backends(ctx):
    """One dgx_optimize_multi call over a mesh, a grid and an analytic object
    (each on its own side stream with its own scratch, including the mesh
    caches) equals separate single-object runs bit-for-bit."""
    from paper_2306_08132_b200 import api, init, model
    hd = model.HandDesc.asset("barrett3")
    hand = api.Hand(ctx, hd)
    ods = [model.mesh_object(*model.icosphere_mesh(0.025, 2)), model.box_grid(res=32), model.sphere(0.025)]
    objs = [api.GraspObject(ctx, o) for o in ods]
    qs = [init.approach_init(o, hd, 5, seed=31 + i) for i, o in enumerate(ods)]
    proto, params, w, opt = api.StabilityProtocol.standard(), api.SimParams(), api.LossWeights(), api.OptConfig(50)
    multi = api.optimize_multi(ctx, objs, hand, np.concatenate(qs), np.array([5, 5, 5], np.int32), proto, params, w,
                               opt, k_begin=0, k_end=3)
    assert not np.any(multi["status"])
    for i, (o, q) in enumerate(zip(objs, qs)):
        one = api.optimize(ctx, o, hand, q, proto, params, w, opt, k_begin=0, k_end=3)
        assert np.array_equal(multi["q"][5 * i:5 * i + 5], one["q"]), i
        assert np.array_equal(multi["m"][5 * i:5 * i + 5], one["m"]), i


def test_split_execution_equals_fused(tmp_path):
    """Split execution (forward kernel at 2 CTAs/SM, then the adjoint kernel,
    handing over through per-(candidate, sim) logs) computes exactly what the
    fused kernel does: eval, loss_gradient and multi-iterate optimize outputs
    are bit-identical for grid and analytic objects. Both also equal the
    static candidate stride (DGX_STATIC_SCHED=1): which CTA claims a candidate
    does not change its results."""
    import subprocess
    import sys
    outs = {}
    for tag, extra in (("split", {}), ("fused", {"DGX_FUSED": "1"}), ("split_static", {"DGX_STATIC_SCHED": "1"}),
                       ("fused_static", {"DGX_FUSED": "1", "DGX_STATIC_SCHED": "1"})):
        p = tmp_path / f"{tag}.npz"
        env = dict(os.environ, **extra)
        subprocess.run([sys.executable, os.path.join(ROOT, "tools", "split_vs_fused.py"), str(p)], env=env,
                       check=True, timeout=600)
        outs[tag] = np.load(p)
    a, b = outs["split"], outs["fused"]
    assert set(a.files) == set(b.files)
    for k in a.files:
        if k.endswith("_kernel_counts"):  # [fused, forward, adjoint] launches of the 6-iterate optimize
            assert a[k].tolist() == [0, 6, 6] and b[k].tolist() == [1, 0, 0], (k, a[k], b[k])
            continue
        assert np.array_equal(a[k], b[k], equal_nan=True), k
    for dyn, sta in (("split", "split_static"), ("fused", "fused_static")):
        for k in outs[dyn].files:
            assert np.array_equal(outs[dyn][k], outs[sta][k], equal_nan=True), (dyn, k)
    assert np.any(a["grid_grad_s"] != 0) and np.any(a["grid_grad_s"] == 0)  # the NaN row failed alone


def test_split_chunks_equal_single_rows(ctx, monkeypatch):
    """More candidates than one split chunk (the scratch budget lowered so a
    chunk is 4 x the resident CTAs = 1184): every chunk's rows equal the same
    candidates run alone."""
    from paper_2306_08132_b200 import api
    hd, od, hand, obj, q = setup(ctx, B=1300, seed=23)
    proto, params = api.StabilityProtocol.standard(), api.SimParams(dilation_radius=0.015)
    monkeypatch.setenv("DGX_SPLIT_SCRATCH_MB", "1")
    l1, g1, s1 = api.loss_gradient(ctx, obj, hand, q, proto, params)
    monkeypatch.delenv("DGX_SPLIT_SCRATCH_MB")
    assert not np.any(s1)
    for lo, hi in ((0, 40), (1180, 1240), (1250, 1300)):
        ls, gs, ss = api.loss_gradient(ctx, obj, hand, q[lo:hi], proto, params)
        assert np.array_equal(ls, l1[lo:hi]) and np.array_equal(gs, g1[lo:hi])


def test_execution_choice_and_kernel_timing(ctx):
    """dgx_ctx_set_kernel_timing / dgx_ctx_kernel_times count every launch by
    kind, and the host picks the execution DESIGN.md §3 states: split forward /
    adjoint kernels above #SMs candidates for grids, fused at or below it and
    for mesh objects."""
    from paper_2306_08132_b200 import api, init, model
    hd = model.HandDesc.asset("allegro16")
    od = model.box_grid(res=32)
    hand, obj = api.Hand(ctx, hd), api.GraspObject(ctx, od)
    proto, params = api.StabilityProtocol.standard(), api.SimParams(dilation_radius=0.01)
    for B, kind in ((64, "fused"), (400, "split")):
        q = init.approach_init(od, hd, B, seed=3)
        n0 = ctx.launches
        ctx.set_kernel_timing(True)
        _, _, st = api.loss_gradient(ctx, obj, hand, q, proto, params)
        kt = ctx.kernel_times()
        ctx.set_kernel_timing(False)
        assert not np.any(st)
        launched = ctx.launches - n0
        if kind == "fused":
            assert kt["fused"][1] == launched == 1 and kt["forward"][1] == kt["adjoint"][1] == 0
        else:
            assert kt["fused"][1] == 0 and kt["forward"][1] == kt["adjoint"][1] >= 1
            assert kt["forward"][1] + kt["adjoint"][1] == launched
        assert all(ms >= 0.0 for ms, _ in kt.values()) and sum(ms for ms, _ in kt.values()) > 0.0
    mo = api.GraspObject(ctx, model.mesh_object(*model.icosphere_mesh(0.025, 2)))
    q = init.approach_init(od, hd, 200, seed=4)
    ctx.set_kernel_timing(True)
    api.evaluate_losses(ctx, mo, hand, q, proto, params)
    kt = ctx.kernel_times()
    ctx.set_kernel_timing(False)
    assert kt["fused"][1] == 1 and kt["forward"][1] == 0


@pytest.mark.parametrize("B", [100, 400])
def test_correction_log_overflow_is_per_candidate(B):
    """A small correction-log capacity (70, about the median sim): candidates whose sims need more active
    corrections report status 3 (log overflow) without touching other
    candidates, in the fused (B <= #SMs) and the split execution alike; the
    candidates that fit are bit-identical to a run with the default capacity."""
    from paper_2306_08132_b200 import api, init, model
    small, big = api.Context(0, correction_capacity=70), api.Context(0)  # ~p50 of the sims
    hd = model.HandDesc.asset("allegro16")
    od = model.box_grid(res=32)
    q = init.approach_init(od, hd, B, seed=9)
    proto, params = api.StabilityProtocol.standard(), api.SimParams(dilation_radius=0.01)
    res = {}
    for name, c in (("small", small), ("big", big)):
        hand, obj = api.Hand(c, hd), api.GraspObject(c, od)
        res[name] = api.loss_gradient(c, obj, hand, q, proto, params)
    ls, gs, ss = res["small"]
    lb, gb, sb = res["big"]
    assert not np.any(sb)
    assert set(np.unique(ss).tolist()) <= {0, 3}
    assert 0 < np.count_nonzero(ss == 3) < B  # both kinds present
    ok = ss == 0
    assert np.array_equal(ls[ok], lb[ok]) and np.array_equal(gs[ok], gb[ok])


@pytest.mark.parametrize("hand_name,grid", [("allegro16", "box64"), ("shadow22_dense", "blob128")])
def test_grid_block_bounds_keep_decisions(monkeypatch, hand_name, grid):
    """The forward pre-filter's block lower bounds (GridSdf::bmin, DESIGN.md
    3.10) only skip cell lookups of points they prove inactive: the same grid
    uploaded without them (DGX_GRID_BLOCK=0) gives bit-identical losses,
    gradients, statuses and SolveStats through the split path."""
    from paper_2306_08132_b200 import api, init, model
    c = api.Context(0)
    hd = model.HandDesc.asset(hand_name)
    od = model.box_grid(res=64) if grid == "box64" else model.blob_grid(seed=3, res=128)
    hand = api.Hand(c, hd)
    with_b = api.GraspObject(c, od)
    monkeypatch.setenv("DGX_GRID_BLOCK", "0")
    without = api.GraspObject(c, od)
    monkeypatch.delenv("DGX_GRID_BLOCK")
    q = init.approach_init(od, hd, 200, seed=12)
    q[:, :3] -= 0.3 * (q[:, :3] - od.com)
    proto = api.StabilityProtocol.standard()
    for radius in (0.0, 0.015):
        params = api.SimParams(dilation_radius=radius)
        a = api.loss_gradient(c, with_b, hand, q, proto, params)
        b = api.loss_gradient(c, without, hand, q, proto, params)
        for x, y in zip(a, b):
            assert np.array_equal(x, y, equal_nan=True)
        ea = api.evaluate_losses(c, with_b, hand, q, proto, params)
        eb = api.evaluate_losses(c, without, hand, q, proto, params)
        for x, y in zip(ea, eb):
            assert np.array_equal(x, y, equal_nan=True)
