"""Small grasp-search workloads for compute-sanitizer (memcheck / racecheck):

  split  160 candidates (> #SMs): split forward + CTA adjoint (and, with
         DGX_ADJ_TASK=1, the warp-task adjoint), then the lane adjoint, allegro16 on the 64^3 box grid,
         loss_gradient + a 2-iterate optimize; plus the global-points forward
         (shadow22_dense, N = 4093) at 150 candidates
  fused  16 candidates: fused kernel (sphere, grid, mesh), a T = 2 protocol,
         M = 9 velocities, the grasp-energy kernel
usage: python tools/sanitize_run.py split|fused
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_08132_b200 import api, init, model  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "fused"
ctx = api.Context(0)
proto, w = api.StabilityProtocol.standard(), api.LossWeights()


def run(hand_name, od, B, protocol=proto, weights=w, k=2):
    hd = model.HandDesc.asset(hand_name)
    hand, obj = api.Hand(ctx, hd), api.GraspObject(ctx, od)
    q = init.approach_init(od, hd, B, seed=5)
    q[:, :3] -= 0.4 * (q[:, :3] - od.com)
    l, g, s = api.loss_gradient(ctx, obj, hand, q, protocol, api.SimParams(dilation_radius=0.015))
    e, st, s2 = api.evaluate_losses(ctx, obj, hand, q, protocol, api.SimParams(dilation_radius=0.015))
    out = api.optimize(ctx, obj, hand, q, protocol, api.SimParams(), weights, api.OptConfig(iterations=10),
                       k_begin=0, k_end=k)
    print(hand_name, od.name, B, "status", int(np.count_nonzero(s)), int(np.count_nonzero(s2)),
          int(np.count_nonzero(out["status"])), flush=True)


if which == "split":
    run("allegro16", model.box_grid(res=64), 160)
    run("shadow22_dense", model.blob_grid(seed=3, res=64), 150, k=1)
    ctx.set_adjoint("lane")  # the lane adjoint (dgx_lane_adj.cuh) on the same workloads
    run("allegro16", model.box_grid(res=64), 160)
    run("shadow22_dense", model.blob_grid(seed=3, res=64), 150, k=1)
    run("barrett3", model.sphere(0.025), 150, k=1)
    ctx.set_adjoint("auto")
else:
    run("barrett3", model.sphere(0.025), 16)
    run("allegro16", model.box_grid(res=32), 16)
    run("barrett3", model.mesh_object(*model.icosphere_mesh(0.025, 2)), 8, k=1)
    run("barrett3", model.sphere(0.025), 8, protocol=api.StabilityProtocol.standard(steps=2), k=1)
    vel = [tuple(v) for v in proto.velocities] + [(0.3, 0.3, 0.0), (0.0, 0.2, -0.4)]
    run("barrett3", model.box_grid(res=32), 8, protocol=api.StabilityProtocol(vel), k=1)
    run("allegro16", model.box_grid(res=32), 8, weights=api.LossWeights(force_closure=0.5, penetration=1.0), k=1)
print("sanitize run ok")
