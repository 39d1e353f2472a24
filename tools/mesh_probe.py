"""Time the fused kernel on triangle-mesh objects (config 1's icosphere mesh
cross-check and a blob mesh): candidate-iterations/s over a short optimize
window, CUDA events on the launching stream.

usage: python tools/mesh_probe.py [B] [iters]
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2306_08132_b200 import api, capi, init, model  # noqa: E402


def run(hand_name, od, B, iters, label):
    dev = torch.device("cuda", 0)
    ctx = api.Context(0)
    hd = model.HandDesc.asset(hand_name)
    hand, obj = api.Hand(ctx, hd), api.GraspObject(ctx, od)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    q0 = init.approach_init(od, hd, B, seed=1)
    D = 6 + hd.num_joints
    q = torch.tensor(q0, device=dev)
    m = torch.zeros(B, D, dtype=torch.float64, device=dev)
    v = torch.zeros_like(m)
    st = torch.zeros(B, dtype=torch.int32, device=dev)
    proto, params, w = api.StabilityProtocol.standard(), api.SimParams(), api.LossWeights()
    opt = api.OptConfig(iterations=500)
    flags = capi.DGX_DEVICE_PTRS | capi.DGX_ASYNC
    api.optimize_multi(ctx, [obj], hand, q, np.array([B], np.int32), proto, params, w, opt, k_begin=0, k_end=1,
                       adam_m=m, adam_v=v, flags=flags, status=st)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    api.optimize_multi(ctx, [obj], hand, q, np.array([B], np.int32), proto, params, w, opt, k_begin=1,
                       k_end=1 + iters, adam_m=m, adam_v=v, flags=flags, status=st)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    ctx.set_stream(None)
    return dict(label=label, hand=hand_name, B=B, iters=iters, ms=ms, cand_iter_per_s=B * iters / (ms * 1e-3),
                failed=int(torch.count_nonzero(st)))


def main():
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    ico = model.mesh_object(*model.icosphere_mesh(0.025, 3))
    print(json.dumps(run("barrett3", ico, B, iters, "icosphere3 mesh (1280 faces)")), flush=True)
    print(json.dumps(run("allegro16", ico, B, iters, "icosphere3 mesh (1280 faces)")), flush=True)
    sph = model.sphere(0.025)
    print(json.dumps(run("barrett3", sph, B, iters, "analytic sphere")), flush=True)


if __name__ == "__main__":
    main()
