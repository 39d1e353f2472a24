"""A/B probe: config 3's 4096 candidates as one launch sequence vs two halves
on two side streams (dgx_optimize_multi with the object listed twice)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_08132_b200 import api, init, model  # noqa: E402

ctx = api.Context(0)
hd = model.HandDesc.asset("shadow22_dense")
od = model.blob_grid(seed=3, res=128)
hand, obj = api.Hand(ctx, hd), api.GraspObject(ctx, od)
B = 4096
D = 6 + hd.num_joints
dev = torch.device("cuda", 0)
q0 = torch.tensor(init.approach_init(od, hd, B, seed=3), device=dev)
args = (api.StabilityProtocol.standard(), api.SimParams(), api.LossWeights(), api.OptConfig(iterations=500))
for mode in sys.argv[1:] or ["single", "halves"]:
    q = q0.clone()
    m = torch.zeros(B, D, dtype=torch.float64, device=dev)
    v = torch.zeros_like(m)
    s = torch.zeros(B, dtype=torch.int32, device=dev)
    ts = []
    for k in range(8):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if mode == "single":
            api.optimize(ctx, obj, hand, q, *args, k_begin=k, k_end=k + 1, adam_m=m, adam_v=v, status=s)
        else:
            api.optimize_multi(ctx, [obj, obj], hand, q, np.array([B // 2, B // 2], np.int32), *args, k_begin=k,
                               k_end=k + 1, adam_m=m, adam_v=v, status=s)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print(mode, "ms per step", [round(1e3 * t, 2) for t in ts[3:]], flush=True)
