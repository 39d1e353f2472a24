"""Export hand descriptors from the UNMODIFIED reference (oracle/_ref/libdgref.so,
glibc build) into assets/hands/<name>.npz. The samples come from the
reference's own area-weighted sampler (hand.cpp:42-68, libstdc++ mt19937_64,
seed 12345 + link index), so they are never regenerated elsewhere.

  barrett3      make_three_finger_hand(2000)          (assets.cpp:304)
  pincher2      make_two_finger_hand(2000)            (assets.cpp:308)
  allegro16     HandModel::load_xml(allegro16.xml, 2000)
  shadow22      HandModel::load_xml(shadow22.xml, 2000)
  shadow22_dense HandModel::load_xml(shadow22.xml, 4096)  (config 3)
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import ref  # noqa: E402
from paper_2306_08132_b200.model import HandDesc  # noqa: E402

HANDS = os.path.join(ROOT, "assets", "hands")


def load(name, variant="glibc"):
    if name == "barrett3":
        return ref.RefHand.barrett3(2000, 12345, variant=variant)
    if name == "pincher2":
        return ref.RefHand.pincher2(2000, 12345, variant=variant)
    base, budget = {"allegro16": ("allegro16", 2000), "shadow22": ("shadow22", 2000),
                    "shadow22_dense": ("shadow22", 4096)}[name]
    return ref.RefHand.load_xml(os.path.join(HANDS, base, base + ".xml"), budget, 12345, variant=variant)


def main():
    for name in ("barrett3", "pincher2", "allegro16", "shadow22", "shadow22_dense"):
        h = load(name)
        HandDesc.from_dict(name, h.desc).save(os.path.join(HANDS, name + ".npz"))
        print(name, "L", h.num_links, "J", h.num_joints, "N", h.num_samples)


if __name__ == "__main__":
    main()
