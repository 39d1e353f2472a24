"""Occupancy probe: forward-only (evaluate_losses) and optimizer-step timings of
the grid instance under different register budgets / staging lengths.

python tools/occ_probe.py            # runs the env variants in subprocesses
python tools/occ_probe.py --child    # one measurement under the current env
"""
import json
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def child():
    import numpy as np
    import torch
    from paper_2306_08132_b200 import api, init, model

    dev = torch.device("cuda", 0)
    ctx = api.Context(0)
    hd = model.HandDesc.asset("allegro16")
    od = model.box_grid(res=64)
    hand, obj = api.Hand(ctx, hd), api.GraspObject(ctx, od)
    B = int(os.environ.get("PROBE_B", "1024"))
    D = 6 + hd.num_joints
    qh = init.approach_init(od, hd, B, seed=17)
    out = {}
    prm = api.SimParams(dilation_radius=0.01)
    proto = api.StabilityProtocol.standard()
    api.evaluate_losses(ctx, obj, hand, qh, proto, prm)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        api.evaluate_losses(ctx, obj, hand, qh, proto, prm)
        ts.append(time.perf_counter() - t0)
    out["eval_ms"] = 1e3 * float(np.median(ts))
    st = torch.cuda.Stream(dev)
    torch.cuda.set_stream(st)
    ctx.set_stream(st.cuda_stream)
    q = torch.tensor(qh, device=dev)
    m = torch.zeros(B, D, dtype=torch.float64, device=dev)
    v = torch.zeros_like(m)
    s = torch.zeros(B, dtype=torch.int32, device=dev)
    args = (ctx, obj, hand, q, proto, api.SimParams(), api.LossWeights(), api.OptConfig(iterations=500))
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
    out["opt_ms"] = float(np.mean(ts))
    out["bad_status"] = int((s != 0).sum().item())
    out["opt_cand_iter_s"] = B / out["opt_ms"] * 1e3
    print(json.dumps(out))


def main():
    variants = [
        {},
        {"DGX_SEGMAX": "1"},
        {"DGX_SEGMAX": "1", "DGX_OCC3": "1"},
        {"DGX_SEGMAX": "2", "DGX_OCC3": "1"},
    ]
    for v in variants:
        env = dict(os.environ, **v)
        r = subprocess.run([sys.executable, __file__, "--child"], env=env, capture_output=True, text=True, timeout=600)
        line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-800:]
        print(json.dumps(v), line, flush=True)


if __name__ == "__main__":
    child() if "--child" in sys.argv else main()
