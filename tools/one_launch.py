"""One warm-up + one timed fused launch (for ncu duration comparisons)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_08132_b200 import api, init, model  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 148
dev = torch.device("cuda", 0)
ctx = api.Context(0)
hd = model.HandDesc.asset(sys.argv[2] if len(sys.argv) > 2 else "allegro16")
OBJ = sys.argv[3] if len(sys.argv) > 3 else "boxgrid64"
od = {"boxgrid64": lambda: model.box_grid(res=64),
      "blob128": lambda: model.blob_grid(seed=3, res=128),  # config 3 (bench.py headline)
      "ico3": lambda: model.mesh_object(*model.icosphere_mesh(0.025, 3))}[OBJ]()
hand, obj = api.Hand(ctx, hd), api.GraspObject(ctx, od)
D = 6 + hd.num_joints
q = torch.tensor(init.approach_init(od, hd, B, seed=3 if OBJ == "blob128" else 17), device=dev)
m = torch.zeros(B, D, dtype=torch.float64, device=dev)
v = torch.zeros_like(m)
s = torch.zeros(B, dtype=torch.int32, device=dev)
args = (ctx, obj, hand, q, api.StabilityProtocol.standard(), api.SimParams(), api.LossWeights(),
        api.OptConfig(iterations=500))
for k in range(3):
    api.optimize(*args, k_begin=k, k_end=k + 1, adam_m=m, adam_v=v, status=s, flags=1)
torch.cuda.synchronize()
print("ok")
