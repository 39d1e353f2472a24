"""Parity at scale (run on a GPU box): random approach-sampled configurations
per (hand, object, dilation) combination; every perturbation residual of the
GPU (dgx_debug_sims) compared BIT-EXACTLY with the reference's recorded sim
(oracle libdgref_sm, std::threads through ctypes), and the per-sim gradients
within rel 1e-9. Prints one JSON summary line per combination.

usage: python tools/parity_fuzz.py [candidates_per_combo]
"""
import json
import os
import sys
import time
import zlib
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import ref  # noqa: E402
from paper_2306_08132_b200 import api, init, model  # noqa: E402


def ref_hand(name):
    if name == "barrett3":
        return ref.RefHand.barrett3()
    if name == "pincher2":
        return ref.RefHand.pincher2()
    return ref.RefHand.load_xml(os.path.join(ROOT, "assets", "hands", name, name + ".xml"), 2000, 12345)


OBJECTS = {
    "sphere25": lambda: model.sphere(0.025),
    "box40": lambda: model.box((0.04, 0.04, 0.04)),
    "boxgrid64": lambda: model.box_grid(res=64),
    "cylgrid64": lambda: model.cylinder_grid(res=64),
    "blobgrid64": lambda: model.blob_grid(seed=3, res=64),
    "ico25mesh": lambda: model.mesh_object(*model.icosphere_mesh(0.025, 3)),
}
COMBOS = [("barrett3", "sphere25"), ("allegro16", "boxgrid64"), ("allegro16", "cylgrid64"),
          ("shadow22", "blobgrid64"), ("pincher2", "box40"), ("barrett3", "ico25mesh")]


def main():
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    ctx = api.Context(0)
    threads = os.cpu_count() or 8
    for hname, oname in COMBOS:
        t0 = time.time()
        rh = ref_hand(hname)
        hd = model.HandDesc.from_dict(hname, rh.desc)
        od = OBJECTS[oname]()
        ro = ref.RefObject.from_desc(od)
        hand, obj = api.Hand(ctx, hd), api.GraspObject(ctx, od)
        rng = np.random.default_rng(zlib.crc32(f"{hname}/{oname}".encode()))
        q = init.approach_init(od, hd, B, seed=int(rng.integers(1 << 30)))
        pull = rng.uniform(0.2, 0.6, size=(B, 1))  # pull toward the object: contacts of varied depth
        q[:, :3] -= pull * (q[:, :3] - od.com)
        q[:, 7:] += rng.normal(scale=0.15, size=(B, hd.num_joints))
        stats = dict(residuals=0, mismatched=0, max_grad_rel=0.0, active_calls=0, grad_rel_gt_1e_12=0,
                     grad_rel_gt_1e_10=0, grad_rel_gt_1e_9=0, worst=None)
        for radius in (0.0, 0.01):
            res, g, _, st = api.debug_sims(ctx, obj, hand, q, api.StabilityProtocol.standard(),
                                           api.SimParams(dilation_radius=radius))
            p = ref.default_params(dilation_radius=radius)
            jobs = [(b, m) for b in range(B) for m in range(7) if not st[b]]

            def run(job):
                b, m = job
                rres, rg, _, log = ref.sim_record(ro, rh, q[b], m, p)
                return job, rres, rg, int(np.sum(log < 0))

            with ThreadPoolExecutor(threads) as ex:
                for (b, m), rres, rg, nact in ex.map(run, jobs):
                    stats["residuals"] += 1
                    stats["active_calls"] += nact
                    if res[b, m] != rres:
                        stats["mismatched"] += 1
                    den = max(np.max(np.abs(rg)), 1e-300)
                    if np.max(np.abs(rg)) > 0:
                        e = float(np.max(np.abs(g[b, m] - rg)) / den)
                        stats["grad_rel_gt_1e_12"] += e > 1e-12
                        stats["grad_rel_gt_1e_10"] += e > 1e-10
                        stats["grad_rel_gt_1e_9"] += e > 1e-9
                        if e > stats["max_grad_rel"]:
                            stats["max_grad_rel"] = e
                            stats["worst"] = dict(candidate=b, sim=m, radius=radius, grad_norm=float(den),
                                                  residual=float(rres))
            stats.setdefault("failed_status", 0)
            stats["failed_status"] += int(np.count_nonzero(st))
        stats.update(hand=hname, object=oname, candidates=B, wall_s=round(time.time() - t0, 1))
        print(json.dumps(stats), flush=True)


if __name__ == "__main__":
    main()
