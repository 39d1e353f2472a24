"""Per-region cycle breakdown of the fused kernel (profiling build).

  DGX_LIBRARY=exp/libdgx_prof.so python tools/region_profile.py
(build: nvcc ... -DDGX_PROFILE_REGIONS -shared csrc/*.cu -o exp/libdgx_prof.so)
Cycles are summed over warps (lane 0), so shares are of total warp-time.
"""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2306_08132_b200 import api, capi, init, model  # noqa: E402

NAMES = {0: "forward sweeps (incl. corrections)", 1: "  apply_correction", 2: "friction fwd",
         4: "friction adjoint", 5: "adjoint runs (process_run)", 6: "  pass 1a (classify+coef)",
         7: "  pass 1b (compose)", 8: "  pass 2 (scan)", 9: "  pass 3 (emit)", 10: "  flush",
         11: "correction adjoints", 12: "run_sim total", 13: "scheduler: claim / spin",
         14: "scheduler: finalize (losses, FK adjoint, Adam)", 15: "scheduler: FK / load next"}
COUNTS = {16: "forward chunk iterations", 17: "forward candidate lanes", 18: "adjoint blocks", 19: "runs",
          20: "forward corrections tried", 21: "frictions applied", 22: "sims",
          23: "mesh nearest queries (lane 0)", 24: "mesh nearest node pops (lane 0)",
          25: "mesh ray casts (lane 0)", 26: "mesh ray node pops (lane 0)", 27: "mesh exact queries (lane 0)",
          28: "mesh certified queries (lane 0)", 29: "mesh cycles: certified argmin (lane 0)",
          30: "mesh cycles: re-certification (lane 0)", 31: "mesh cycles: phong + ray-cast sign (lane 0)",
          32: "sims entering the adjoint (touched)", 33: "  of which fold-eligible (>= 2 final cycles)",
          34: "  final-run cycles Kc (sum)", 35: "adjoint emitted positions (point-sweeps)",
          36: "  corrections in adjoint sims"}


def main():
    hand_name = sys.argv[1] if len(sys.argv) > 1 else "allegro16"
    B = int(sys.argv[2]) if len(sys.argv) > 2 else 512
    obj_name = sys.argv[3] if len(sys.argv) > 3 else "boxgrid64"
    K0 = int(sys.argv[4]) if len(sys.argv) > 4 else 2  # profiled iterate
    L = capi.load()
    L.dgx_prof_read.argtypes = [C.POINTER(C.c_ulonglong), C.c_int, C.c_int]
    ctx = api.Context(0)
    hd = model.HandDesc.asset(hand_name)
    od = {"boxgrid64": lambda: model.box_grid(res=64),
          "ico3": lambda: model.mesh_object(*model.icosphere_mesh(0.025, 3)),
          "blob128": lambda: model.blob_grid(seed=3, res=128),
          "sphere": lambda: model.sphere(0.025)}[obj_name]()
    hand, obj = api.Hand(ctx, hd), api.GraspObject(ctx, od)
    q = init.approach_init(od, hd, B, seed=3 if obj_name == "blob128" else 17)
    proto, w = api.StabilityProtocol.standard(), api.LossWeights()
    opt = api.OptConfig(iterations=500)
    buf = (C.c_ulonglong * 48)()
    out = api.optimize(ctx, obj, hand, q, proto, api.SimParams(), w, opt, k_begin=0, k_end=K0)
    L.dgx_prof_read(buf, 48, 1)
    out = api.optimize(ctx, obj, hand, out["q"], proto, api.SimParams(), w, opt, k_begin=K0, k_end=K0 + 1,
                       adam_m=out["m"], adam_v=out["v"])
    L.dgx_prof_read(buf, 48, 1)
    v = np.array(list(buf), dtype=np.float64)
    ci = B * 1
    tot = v[12]
    print(f"{hand_name} x {obj_name} B={B}: per candidate-iteration (7 sims), cycles summed over warps")
    for k, n in NAMES.items():
        print(f"  {n:38s} {v[k] / ci:12.0f} cyc  {100 * v[k] / tot:5.1f}%")
    for k, n in COUNTS.items():
        if v[k]:
            print(f"  {n:38s} {v[k] / ci:12.1f} per cand-iter")


if __name__ == "__main__":
    main()
