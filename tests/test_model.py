"""CPU: descriptors, grids, inertia and the approach-sampling initializer."""
import os

import numpy as np
import pytest

from paper_2306_08132_b200 import init, model

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("name,L,J,N", [("barrett3", 10, 9, 1999), ("pincher2", 5, 4, 1999),
                                        ("allegro16", 17, 16, 2001), ("shadow22", 23, 22, 2001),
                                        ("shadow22_dense", 23, 22, 4093)])
def test_hand_assets(name, L, J, N):
    h = model.HandDesc.asset(name)
    assert (h.num_links, h.num_joints, h.num_samples) == (L, J, N)
    assert h.topo[0] == int(np.nonzero(h.link_parent_joint < 0)[0][0])
    assert np.all(np.diff(h.sample_link) >= 0)          # forward() order: link-index major
    assert np.all(h.lower < h.upper)
    assert np.allclose(np.linalg.norm(h.axis, axis=1), 1.0)


def test_hand_assets_match_reference(oracle):
    for name in ("barrett3", "allegro16"):
        h = model.HandDesc.asset(name)
        rh = (oracle.RefHand.barrett3(variant="glibc") if name == "barrett3" else
              oracle.RefHand.load_xml(os.path.join(ROOT, "assets", "hands", name, name + ".xml"), 2000, 12345,
                                      variant="glibc"))
        for k, v in rh.desc.items():
            assert np.array_equal(getattr(h, k).reshape(v.shape), v), k


def test_analytic_inertia():
    s = model.sphere(0.025)
    assert abs(s.mass - 1000 * 4 / 3 * np.pi * 0.025 ** 3) < 1e-15
    assert np.allclose(s.inertia_body @ s.inertia_body_inv, np.eye(3))
    b = model.box((0.04, 0.02, 0.01))
    assert np.isclose(b.inertia_body[0, 0], b.mass / 12 * (0.02 ** 2 + 0.01 ** 2))


def test_box_grid_matches_analytic():
    g = model.box_grid(res=64)
    assert g.dims == (64, 64, 64) and g.values.dtype == np.float32
    half = np.array([0.02, 0.02, 0.02])
    rng = np.random.default_rng(0)
    p = rng.uniform(-0.045, 0.045, size=(500, 3))
    err = np.abs(init._grid_phi(g, p) - model.sdf_box(p, half))
    assert np.max(err) < 2 * g.spacing   # trilinear error bounded by the cell size


@pytest.mark.parametrize("obj", ["sphere", "box", "grid"])
def test_approach_init_properties(obj):
    """determinism, approach axis anti-parallel to the normal, coverage."""
    o = {"sphere": model.sphere(0.025), "box": model.box((0.04, 0.04, 0.04)),
         "grid": model.cylinder_grid(res=32)}[obj]
    h = model.HandDesc.asset("barrett3")
    q1 = init.approach_init(o, h, 100, seed=5)
    q2 = init.approach_init(o, h, 100, seed=5)
    assert np.array_equal(q1, q2)
    assert np.allclose(np.linalg.norm(q1[:, 3:7], axis=1), 1.0)
    assert np.allclose(q1[:, 7:], h.mid_range())
    # palm +z axis points back toward the object along -n
    for b in range(0, 100, 7):
        w, x, y, z = q1[b, 3:7]
        zaxis = np.array([2 * (x * z + w * y), 2 * (y * z - w * x), 1 - 2 * (x * x + y * y)])
        to_obj = o.com - q1[b, :3]
        assert np.dot(zaxis, to_obj) > 0
    if obj == "sphere":
        for b in range(100):
            w, x, y, z = q1[b, 3:7]
            zaxis = np.array([2 * (x * z + w * y), 2 * (y * z - w * x), 1 - 2 * (x * x + y * y)])
            n = q1[b, :3] / np.linalg.norm(q1[b, :3])
            assert abs(np.dot(zaxis, n) + 1.0) < 1e-6
        octants = {tuple(np.sign(q1[b, :3]).astype(int)) for b in range(100)}
        assert len(octants) == 8
    # shards compose: candidates [50, 100) drawn independently equal the tail of the batch
    q3 = init.approach_init(o, h, 50, seed=5, first=50)
    assert np.array_equal(q3, q1[50:])
