"""Generate tests/golden/*.npz from the compiled reference (oracle/_ref).

Each fixture holds seeded inputs and the reference's outputs for them, from
BOTH oracle builds: "sm" (parity mode P: shared deterministic sin/cos/atan2)
and "glibc" (the unmodified reference). Committed so GPU parity tests have
fixed expectations that do not depend on rebuilding the oracle; tests also
re-derive them from the oracle when it is present (pinning it).

  python tools/make_golden.py
"""
import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import ref  # noqa: E402
from paper_2306_08132_b200 import init, model  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def hand_for(name, variant):
    if name == "barrett3":
        return ref.RefHand.barrett3(variant=variant)
    if name == "pincher2":
        return ref.RefHand.pincher2(variant=variant)
    return ref.RefHand.load_xml(os.path.join(ROOT, "assets", "hands", name, name + ".xml"), 2000, 12345,
                                variant=variant)


def object_for(name):
    return {"sphere25": lambda: model.sphere(0.025), "box40": lambda: model.box((0.04, 0.04, 0.04)),
            "boxgrid64": lambda: model.box_grid(res=64), "cylgrid32": lambda: model.cylinder_grid(res=32)}[name]()


CASES = [
    # (fixture, hand, object, B, seed, radius)
    ("barrett3_sphere25", "barrett3", "sphere25", 4, 1, 0.01),
    ("pincher2_box40", "pincher2", "box40", 3, 2, 0.02),
    ("allegro16_boxgrid64", "allegro16", "boxgrid64", 3, 3, 0.02),
    ("barrett3_cylgrid32", "barrett3", "cylgrid32", 3, 4, 0.0),
]


def grid_hash(o):
    return hashlib.sha256(np.ascontiguousarray(o.values).tobytes()).hexdigest() if o.kind == "grid" else ""


def make(fixture, hand_name, obj_name, B, seed, radius):
    o = object_for(obj_name)
    hd = model.HandDesc.from_dict(hand_name, hand_for(hand_name, "glibc").desc)
    q = init.approach_init(o, hd, B, seed=seed)
    # pull the palm in so the dilated contact set is non-trivial
    q[:, :3] -= 0.45 * (q[:, :3] - o.com)
    out = dict(q=q, radius=np.array(radius), grid_sha256=np.array(grid_hash(o)))
    for variant in ("sm", "glibc"):
        rh = hand_for(hand_name, variant)
        ro = ref.RefObject.from_desc(o, variant=variant)
        p = ref.default_params(dilation_radius=radius)
        L, DS, DR, DL, EV, ST, RES, SG = [], [], [], [], [], [], [], []
        for b in range(B):
            l, ds, dr, dl = ref.loss_gradient(ro, rh, q[b], p)
            L.append(l); DS.append(ds); DR.append(dr); DL.append(dl)
            EV.append(ref.evaluate_losses(ro, rh, q[b], p))
            st, res, sg = [], [], []
            for m in range(7):
                r_, s_, _ = ref.sim_forward(ro, rh, q[b], m, p)
                st.append(s_)
                rr, g, _, _ = ref.sim_record(ro, rh, q[b], m, p)
                res.append(rr); sg.append(g)
            ST.append(st); RES.append(res); SG.append(sg)
        # one teacher-forced optimizer step from iterate k=3 of a 10-iteration schedule
        o3 = ref.optimize(ro, rh, q, ref.default_params(), iters=10, k_begin=0, k_end=3)
        o4 = ref.optimize(ro, rh, o3["q"], ref.default_params(), iters=10, k_begin=3, k_end=4,
                          adam_m=o3["m"], adam_v=o3["v"], record=True)
        out.update({
            f"{variant}_losses": np.array(L), f"{variant}_d_stable": np.array(DS),
            f"{variant}_d_qrange": np.array(DR), f"{variant}_d_qlimit": np.array(DL),
            f"{variant}_eval": np.array(EV), f"{variant}_stats": np.array(ST),
            f"{variant}_sim_res": np.array(RES), f"{variant}_sim_grads": np.array(SG),
            f"{variant}_opt_q3": o3["q"], f"{variant}_opt_m3": o3["m"], f"{variant}_opt_v3": o3["v"],
            f"{variant}_opt_q4": o4["q"], f"{variant}_opt_m4": o4["m"], f"{variant}_opt_v4": o4["v"],
            f"{variant}_opt_traj_losses": o4["losses"], f"{variant}_opt_traj_grads": o4["grads"],
        })
    np.savez_compressed(os.path.join(OUT, fixture + ".npz"), **out)
    print(fixture, "losses", out["sm_losses"][:, 0])


def main():
    os.makedirs(OUT, exist_ok=True)
    for c in CASES:
        make(*c)


if __name__ == "__main__":
    main()
