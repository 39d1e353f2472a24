"""Dump results of the public API for a fixed workload to an .npz (used by
tests/test_gpu_props.py to compare split execution against DGX_FUSED=1)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_08132_b200 import api, init, model  # noqa: E402


def main(out_path: str) -> None:
    ctx = api.Context(0)
    res = {}
    hd = model.HandDesc.asset("allegro16")
    proto = api.StabilityProtocol.standard()
    for name, od in (("grid", model.box_grid(res=64)), ("sphere", model.sphere(0.03)),
                     ("box", model.box((0.04, 0.04, 0.04)))):
        hand, obj = api.Hand(ctx, hd), api.GraspObject(ctx, od)
        # more candidates than SMs (148): the default run takes the split path
        q = init.approach_init(od, hd, 200, seed=5)
        q[7, 8] = np.nan  # a non-finite joint: per-candidate status, same in both executions
        q[11, 7:] = hd.upper + 0.01  # every joint past its upper limit (qlimit tie rules)
        prm = api.SimParams(dilation_radius=0.01)
        l, st, s = api.evaluate_losses(ctx, obj, hand, q, proto, prm)
        res[f"{name}_eval_l"], res[f"{name}_eval_stats"], res[f"{name}_eval_s"] = l, st, s
        l, g, s = api.loss_gradient(ctx, obj, hand, q, proto, prm)
        res[f"{name}_grad_l"], res[f"{name}_grad_g"], res[f"{name}_grad_s"] = l, g, s
        ctx.set_kernel_timing(True)
        o = api.optimize(ctx, obj, hand, q, proto, api.SimParams(), api.LossWeights(), api.OptConfig(iterations=50),
                         k_begin=0, k_end=6, record=True)
        res[f"{name}_kernel_counts"] = np.array([n for _, n in ctx.kernel_times().values()])
        ctx.set_kernel_timing(False)
        for k in ("q", "m", "v", "status", "traj"):
            res[f"{name}_opt_{k}"] = o[k]
    np.savez(out_path, **res)


if __name__ == "__main__":
    main(sys.argv[1])
