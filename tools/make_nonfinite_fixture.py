"""Find an iterate where the reference's tape raises "non-finite adjoint"
(tape.cpp:35-38) along a GPU synthesis run on a procedural blob mesh, and save
it as tests/golden/errors/nonfinite_adjoint_blob.npz (q, dilation radius). The test
(tests/test_gpu_parity.py::test_nonfinite_adjoint_matches_reference) checks that
the GPU reports DGX_E_NONFINITE_GRAD for that candidate exactly where the
reference throws. Run on a GPU box (needs oracle/_ref)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import ref  # noqa: E402
from paper_2306_08132_b200 import api, init, model  # noqa: E402


def main():
    hd = model.HandDesc.asset("barrett3")
    ctx = api.Context(0)
    hand = api.Hand(ctx, hd)
    od = model.mesh_object(*ref.RefObject.blob_mesh(0.021, 3, 0.5, 7, variant="sm").mesh_export()[:2])
    obj = api.GraspObject(ctx, od)
    q = init.approach_init(od, hd, 20, seed=5)[[6]].copy()
    m = np.zeros((1, 6 + hd.num_joints))
    v = np.zeros_like(m)
    proto, params, w = api.StabilityProtocol.standard(), api.SimParams(), api.LossWeights()
    opt = api.OptConfig(iterations=200)
    for k in range(200):
        qk = q.copy()
        out = api.optimize(ctx, obj, hand, q, proto, params, w, opt, k_begin=k, k_end=k + 1, adam_m=m, adam_v=v)
        if np.any(np.asarray(out["status"])):
            r = opt.dilation_start_radius * (1.0 - k / (opt.iterations - 1.0))
            np.savez(os.path.join(ROOT, "tests", "golden", "errors", "nonfinite_adjoint_blob.npz"), q=qk[0], radius=r,
                     blob=np.array([0.021, 3, 0.5, 7]))
            print("saved k", k, "radius", r)
            return
        q, m, v = out["q"], out["m"], out["v"]
    print("no failure found")


if __name__ == "__main__":
    main()
