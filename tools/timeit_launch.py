"""Time fused launches (single object) for a few batch sizes: python tools/timeit_launch.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_08132_b200 import api, capi, init, model  # noqa: E402

dev = torch.device("cuda", 0)
ctx = api.Context(0)
st = torch.cuda.Stream(dev)
torch.cuda.set_stream(st)
ctx.set_stream(st.cuda_stream)
hd = model.HandDesc.asset("allegro16")
od = model.box_grid(res=64)
hand, obj = api.Hand(ctx, hd), api.GraspObject(ctx, od)
D = 6 + hd.num_joints
for B in (148, 296, 512, 1024):
    q = torch.tensor(init.approach_init(od, hd, B, seed=17), device=dev)
    m = torch.zeros(B, D, dtype=torch.float64, device=dev)
    v = torch.zeros_like(m)
    s = torch.zeros(B, dtype=torch.int32, device=dev)
    args = (ctx, obj, hand, q, api.StabilityProtocol.standard(), api.SimParams(), api.LossWeights(),
            api.OptConfig(iterations=500))
    api.optimize(*args, k_begin=0, k_end=1, adam_m=m, adam_v=v, status=s, flags=3)
    torch.cuda.synchronize()
    ts = []
    for k in range(1, 4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        api.optimize(*args, k_begin=k, k_end=k + 1, adam_m=m, adam_v=v, status=s, flags=3)
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"B={B}: {np.mean(ts):.2f} ms per iteration -> {B / np.mean(ts) * 1e3:.0f} cand-iter/s", flush=True)
