"""GPU parity at the BASELINE configs the round-1 suite did not pin (VERDICT r1
"Next round" #1), each through the C-ABI vs the compiled reference
(libdgref_sm: the reference's own solver and tape, parity mode P):

  * config 3: shadow22_dense (J=22, N=4093) on the 128^3 procedural blob grid,
    including a batch larger than the SM count (the bench's execution path);
  * config 4: barrett3 on 64^3 blob grids (three of the 64 objects);
  * config 5: a 256^3 grid (the sweep's largest resolution);
  * config 2's second object: allegro16 on cylinder_grid(64);
  * the benchmarked path itself: full-size optimize batches (config 2: 1024
    candidates over two objects via dgx_optimize_multi; config 3: 4096
    candidates), sampled rows compared with the reference's optimizer step
    from the same iterate (teacher forcing).

Bars: residuals / losses / SolveStats BIT-EXACT (identical contact culling and
correction order); gradients within GRAD_RTOL (tests/test_gpu_parity.py: the
closed-form adjoint associates sums differently from the tape).
Reference: sim.hpp:138-210, losses.cpp:20-66, losses.cpp:92-102.
"""
import os

import numpy as np
import pytest

from test_gpu_parity import GRAD_RTOL, relerr

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def ref_hand(oracle, name):
    if name == "barrett3":
        return oracle.RefHand.barrett3()
    base, budget = {"allegro16": ("allegro16", 2000), "shadow22": ("shadow22", 2000),
                    "shadow22_dense": ("shadow22", 4096)}[name]
    return oracle.RefHand.load_xml(os.path.join(ROOT, "assets", "hands", base, base + ".xml"), budget, 12345)


class Setup:
    def __init__(self, ctx, oracle, hand_name, od, B, seed, pull=0.4, jitter=0.1):
        from paper_2306_08132_b200 import api, init, model
        self.rh = ref_hand(oracle, hand_name)
        self.hd = model.HandDesc.from_dict(hand_name, self.rh.desc)
        assert np.array_equal(self.hd.samples, model.HandDesc.asset(hand_name).samples)  # committed asset
        self.od = od
        self.ro = oracle.RefObject.from_desc(od)
        self.hand, self.obj = api.Hand(ctx, self.hd), api.GraspObject(ctx, od)
        q = init.approach_init(od, self.hd, B, seed=seed)
        rng = np.random.default_rng(seed)
        q[:, :3] -= rng.uniform(pull * 0.5, pull, size=(B, 1)) * (q[:, :3] - od.com)
        q[:, 7:] += rng.normal(scale=jitter, size=(B, self.hd.num_joints))
        self.q = q


def check_loss_gradient(ctx, oracle, s, rows, radius):
    from paper_2306_08132_b200 import api
    proto, params = api.StabilityProtocol.standard(), api.SimParams(dilation_radius=radius)
    p = oracle.default_params(dilation_radius=radius)
    losses, grads, st = api.loss_gradient(ctx, s.obj, s.hand, s.q, proto, params)
    el, stats, st2 = api.evaluate_losses(ctx, s.obj, s.hand, s.q, proto, params)
    assert not np.any(st) and not np.any(st2)
    n_contacts = 0
    for b in rows:
        rl, ds, dr, dl = oracle.loss_gradient(s.ro, s.rh, s.q[b], p)
        assert np.array_equal(losses[b], rl), (b, losses[b], rl)
        assert relerr(grads[b, 0], ds) < GRAD_RTOL, (b, relerr(grads[b, 0], ds))
        assert relerr(grads[b, 1], dr) < GRAD_RTOL
        assert np.array_equal(grads[b, 2], dl)
        assert np.array_equal(el[b], oracle.evaluate_losses(s.ro, s.rh, s.q[b], p))
        for m in range(7):
            _, rst, _ = oracle.sim_forward(s.ro, s.rh, s.q[b], m, p)
            assert np.array_equal(stats[b, m], rst), (b, m, stats[b, m], rst)
            n_contacts += int(rst[0])
    return n_contacts


def check_sims(ctx, oracle, s, rows, radius):
    """Per-perturbation residuals bit-exact (=> the same activation and
    correction sequence) and per-sim gradients vs the reference tape."""
    from paper_2306_08132_b200 import api
    proto, params = api.StabilityProtocol.standard(), api.SimParams(dilation_radius=radius)
    res, g, _, st = api.debug_sims(ctx, s.obj, s.hand, s.q[rows], proto, params)
    assert not np.any(st)
    p = oracle.default_params(dilation_radius=radius)
    active = 0
    for i, b in enumerate(rows):
        for m in range(7):
            rres, rg, _, log = oracle.sim_record(s.ro, s.rh, s.q[b], m, p)
            active += int(np.sum(log < 0))
            assert res[i, m] == rres, (b, m)
            assert relerr(g[i, m], rg) < GRAD_RTOL, (b, m, relerr(g[i, m], rg))
    return active


@pytest.fixture(scope="module")
def blob128():
    from paper_2306_08132_b200 import model
    return model.blob_grid(seed=3, res=128)


def test_config3_dense_hand_blob128(ctx, oracle, blob128):
    """Config 3: N=4093 (forward shared memory > 96 KB) on the 128^3 blob."""
    s = Setup(ctx, oracle, "shadow22_dense", blob128, B=3, seed=41)
    assert s.hd.num_samples == 4093 and s.od.dims == (128, 128, 128)
    assert check_sims(ctx, oracle, s, [0, 1, 2], 0.015) > 0
    check_loss_gradient(ctx, oracle, s, [0, 1, 2], 0.0)
    assert check_loss_gradient(ctx, oracle, s, [0, 1, 2], 0.02) > 0


def test_config3_large_batch_rows(ctx, oracle, blob128):
    """Config 3 at more candidates than SMs (the bench's execution path:
    persistent CTAs claiming candidates): sampled rows vs the reference."""
    from paper_2306_08132_b200 import api
    s = Setup(ctx, oracle, "shadow22_dense", blob128, B=320, seed=43)
    n = check_loss_gradient(ctx, oracle, s, [0, 157, 319], 0.02)
    assert n > 0
    # the rows do not depend on the batch they run in
    l1, g1, _ = api.loss_gradient(ctx, s.obj, s.hand, s.q[[0, 157, 319]], api.StabilityProtocol.standard(),
                                  api.SimParams(dilation_radius=0.02))
    lb, gb, _ = api.loss_gradient(ctx, s.obj, s.hand, s.q, api.StabilityProtocol.standard(),
                                  api.SimParams(dilation_radius=0.02))
    assert np.array_equal(l1, lb[[0, 157, 319]]) and np.array_equal(g1, gb[[0, 157, 319]])


@pytest.mark.parametrize("seed", [0, 21, 63])
def test_config4_barrett3_blob64(ctx, oracle, seed):
    from paper_2306_08132_b200 import model
    s = Setup(ctx, oracle, "barrett3", model.blob_grid(seed=seed, res=64), B=3, seed=50 + seed)
    assert check_sims(ctx, oracle, s, [0, 1], 0.02) > 0
    check_loss_gradient(ctx, oracle, s, [0, 1, 2], 0.01)


def test_config5_grid256(ctx, oracle):
    """The sweep's largest resolution: 256^3 (64 MB of FP32 nodes, 512 MB of
    corner-packed cells)."""
    from paper_2306_08132_b200 import model
    s = Setup(ctx, oracle, "allegro16", model.blob_grid(seed=11, res=256), B=3, seed=61)
    assert check_sims(ctx, oracle, s, [0, 1], 0.02) > 0
    check_loss_gradient(ctx, oracle, s, [0, 1, 2], 0.0)


def test_config2_cylinder_grid64(ctx, oracle):
    from paper_2306_08132_b200 import model
    s = Setup(ctx, oracle, "allegro16", model.cylinder_grid(res=64), B=3, seed=71)
    assert check_sims(ctx, oracle, s, [0, 1, 2], 0.02) > 0
    check_loss_gradient(ctx, oracle, s, [0, 1, 2], 0.015)


def _teacher_forced_rows(oracle, ro, rh, q, m, v, k, rows, gpu_out):
    r = oracle.optimize(ro, rh, q[rows], oracle.default_params(), iters=500, k_begin=k, k_end=k + 1,
                        adam_m=None if m is None else m[rows], adam_v=None if v is None else v[rows], record=True)
    assert not np.any(r["status"]) and not np.any(gpu_out["status"][rows])
    traj = gpu_out["traj"][rows]
    assert np.array_equal(traj[:, :, :3], r["losses"])
    assert relerr(traj[:, :, 3:], r["grads"]) < GRAD_RTOL
    assert relerr(gpu_out["q"][rows], r["q"]) < GRAD_RTOL
    assert relerr(gpu_out["m"][rows], r["m"]) < GRAD_RTOL


def test_bench_config2_split_path_rows(ctx, oracle):
    """The config-2 bench step exactly as bench.py runs it: allegro16, box64 +
    cylinder64, 1024 candidates through dgx_optimize_multi (split forward /
    adjoint kernels, both objects concurrently), iterates 0 and 1; 24 sampled
    rows vs the reference optimizer from the same iterate."""
    from paper_2306_08132_b200 import api, init, model
    rh = ref_hand(oracle, "allegro16")
    hd = model.HandDesc.from_dict("allegro16", rh.desc)
    ods = [model.box_grid(res=64), model.cylinder_grid(res=64)]
    ros = [oracle.RefObject.from_desc(o) for o in ods]
    hand, objs = api.Hand(ctx, hd), [api.GraspObject(ctx, o) for o in ods]
    qs = [init.approach_init(o, hd, 512, seed=17 + i) for i, o in enumerate(ods)]
    q = np.concatenate(qs)
    counts = np.array([512, 512], np.int32)
    proto, opt = api.StabilityProtocol.standard(), api.OptConfig(iterations=500)
    ctx.set_kernel_timing(True)
    m = v = None
    for k in (0, 1):
        out = api.optimize_multi(ctx, objs, hand, q, counts, proto, api.SimParams(), api.LossWeights(), opt,
                                 k_begin=k, k_end=k + 1, adam_m=m, adam_v=v, record=True)
        kt = ctx.kernel_times()
        assert kt["forward"][1] >= 2 and kt["adjoint"][1] >= 2, kt  # the split path ran
        rows = np.random.default_rng(k).choice(512, size=12, replace=False)
        for i in range(2):
            sl = slice(512 * i, 512 * (i + 1))
            sub = {key: out[key][sl] for key in ("q", "m", "v", "status", "traj")}
            _teacher_forced_rows(oracle, ros[i], rh, q[sl], None if m is None else m[sl],
                                 None if v is None else v[sl], k, rows, sub)
        q, m, v = out["q"], out["m"], out["v"]
    ctx.set_kernel_timing(False)


def test_bench_config3_rows(ctx, oracle, blob128):
    """The config-3 bench step as bench.py runs it: 4096 candidates of
    shadow22_dense on the 128^3 blob, iterate 0; 8 sampled rows vs the
    reference optimizer step."""
    from paper_2306_08132_b200 import api, init
    rh = ref_hand(oracle, "shadow22_dense")
    from paper_2306_08132_b200 import model
    hd = model.HandDesc.from_dict("shadow22_dense", rh.desc)
    ro = oracle.RefObject.from_desc(blob128)
    hand, obj = api.Hand(ctx, hd), api.GraspObject(ctx, blob128)
    q = init.approach_init(blob128, hd, 4096, seed=3)
    out = api.optimize(ctx, obj, hand, q, api.StabilityProtocol.standard(), api.SimParams(), api.LossWeights(),
                       api.OptConfig(iterations=500), k_begin=0, k_end=1, record=True)
    rows = np.array([0, 1, 777, 2048, 3001, 4000, 4094, 4095])
    _teacher_forced_rows(oracle, ro, rh, q, None, None, 0, rows, out)
