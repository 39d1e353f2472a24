import sys, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2306_08132_b200 import api, init, model
ctx = api.Context(0)
hd = model.HandDesc.asset("allegro16"); od = model.cylinder_grid(res=64)
hand, obj = api.Hand(ctx, hd), api.GraspObject(ctx, od)
q = init.approach_init(od, hd, 256, seed=17)
proto, w = api.StabilityProtocol.standard(), api.LossWeights()
st = None; m = v = None
for k in range(40):
    out = api.optimize(ctx, obj, hand, q, proto, api.SimParams(), w, api.OptConfig(iterations=40), k_begin=k, k_end=k+1, adam_m=m, adam_v=v)
    bad = np.nonzero(out["status"])[0]
    if bad.size:
        print("iter", k, "bad", bad[:10], out["status"][bad[:10]])
        b = bad[0]
        res, g, gp, st2 = api.debug_sims(ctx, obj, hand, q[b:b+1], proto, api.SimParams(dilation_radius=0.02*(1-k/39)))
        print(" debug status", st2, res)
        break
    q, m, v = out["q"], out["m"], out["v"]
print("done")
