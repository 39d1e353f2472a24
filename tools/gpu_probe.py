"""First-contact parity probe: GPU (libdgx_cuda.so) vs the compiled reference
(oracle/_ref/libdgref_sm.so, parity mode P). Prints a compact report."""
import sys, time, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import ref
from paper_2306_08132_b200 import api, model

def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))

rh = ref.RefHand.barrett3(variant="sm")
hd = model.HandDesc.from_dict("barrett3", rh.desc)
sph = model.sphere(0.025)
ro = ref.RefObject.from_desc(sph, variant="sm")
ctx = api.Context(0)
hand = api.Hand(ctx, hd)
obj = api.GraspObject(ctx, sph)
rng = np.random.default_rng(0)
mid = hd.mid_range()
qs = []
for k in range(6):
    pos = np.array([0.0, 0.0, -0.040]) + rng.normal(0, 0.003, 3)
    ax = rng.normal(size=3); ax /= np.linalg.norm(ax); ang = rng.uniform(0, 0.3)
    quat = np.concatenate([[np.cos(ang / 2)], np.sin(ang / 2) * ax])
    qs.append(np.concatenate([pos, quat, mid + rng.normal(0, 0.1, hd.num_joints)]))
qs = np.array(qs)
# FK
pts = api.forward(ctx, hand, qs)
fk_bits = all(np.array_equal(pts[b], rh.forward(qs[b])) for b in range(len(qs)))
print("FK bit-exact:", fk_bits, flush=True)
for radius in (0.0, 0.01):
    params = api.SimParams(dilation_radius=radius)
    proto = api.StabilityProtocol.standard()
    rp = ref.default_params(dilation_radius=radius)
    res, g, gp, st = api.debug_sims(ctx, obj, hand, qs, proto, params, point_grads=True)
    print(f"radius {radius}: status", st, flush=True)
    worst_g = worst_gp = 0.0; res_bits = True
    for b in range(len(qs)):
        for m in range(7):
            rres, rg, rgp, log = ref.sim_record(ro, rh, qs[b], m, rp, points_grad=True)
            res_bits &= (rres == res[b, m])
            if rres != res[b, m]:
                print(f"  b{b} m{m} residual mismatch gpu {res[b,m]!r} ref {rres!r} nact_ref={(log<0).sum()}")
            worst_g = max(worst_g, rel(g[b, m], rg))
            worst_gp = max(worst_gp, rel(gp[b, m], rgp))
    print(f"  per-sim residual bit-exact: {res_bits}; max rel err sim grad {worst_g:.3e}, point grad {worst_gp:.3e}", flush=True)
    losses, grads, st = api.loss_gradient(ctx, obj, hand, qs, proto, params)
    lbits = True; wg = 0.0
    for b in range(len(qs)):
        rl, ds, dr, dl = ref.loss_gradient(ro, rh, qs[b], rp)
        lbits &= np.array_equal(rl, losses[b])
        wg = max(wg, rel(grads[b, 0], ds), rel(grads[b, 1], dr) if np.any(dr) else 0.0)
        if not np.array_equal(grads[b, 2], dl): print("  qlimit grad mismatch", grads[b, 2], dl)
    print(f"  loss_gradient: losses bit-exact {lbits}; max rel grad err {wg:.3e}", flush=True)
    el, stats, st = api.evaluate_losses(ctx, obj, hand, qs, proto, params)
    ebits = True; sbits = True
    for b in range(len(qs)):
        re_ = ref.evaluate_losses(ro, rh, qs[b], rp)
        ebits &= np.array_equal(re_, el[b])
        for m in range(7):
            r_, rst, _ = ref.sim_forward(ro, rh, qs[b], m, rp)
            if not np.array_equal(rst, stats[b, m]):
                sbits = False
                print("  stats mismatch", b, m, rst, stats[b, m])
    print(f"  evaluate_losses bit-exact {ebits}; stats exact {sbits}", flush=True)
# optimizer, teacher-forced steps
params = api.SimParams()
proto = api.StabilityProtocol.standard()
w = api.LossWeights(); opt = api.OptConfig(iterations=20)
out = api.optimize(ctx, obj, hand, qs, proto, params, w, opt, k_begin=0, k_end=5, record=True)
rout = ref.optimize(ro, rh, qs, ref.default_params(), iters=20, k_begin=0, k_end=5, record=True)
print("opt status", out["status"], rout["status"])
print("opt q rel err", rel(out["q"], rout["q"]), " traj loss rel", rel(out["traj"][:, :, :3], rout["losses"]),
      " traj grad rel", rel(out["traj"][:, :, 3:], rout["grads"]))
# timing
B = 1024
qb = np.repeat(qs, B // len(qs) + 1, axis=0)[:B]
for it in range(2):
    t = time.time(); out = api.optimize(ctx, obj, hand, qb, proto, params, w, api.OptConfig(iterations=10)); dt = time.time() - t
    print(f"optimize B={B} x 10 iters: {dt:.3f}s -> {B*10/dt:.1f} cand-iter/s; status nonzero {np.count_nonzero(out['status'])}", flush=True)
