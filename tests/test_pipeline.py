"""Scene pipeline host logic (no GPU): scene sampling, grasp transfer
composition, JSONL export."""
import json

import numpy as np


def test_scene_states_deterministic_and_unit():
    from paper_2306_08132_b200 import model, pipeline
    od = model.mesh_object(*model.icosphere_mesh(0.025, 2))
    a = pipeline.scene_states(od, [3, 4, 5])
    b = pipeline.scene_states(od, [3, 4, 5])
    assert np.array_equal(a, b)
    assert np.allclose(np.linalg.norm(a[:, 3:7], axis=1), 1.0, atol=1e-15)
    assert np.allclose(a[:, 2], 2.0 * od.bounding_radius())
    assert not np.array_equal(a[0], a[1])
    assert np.all(a[:, 7:] == 0.0)


def test_transfer_composition():
    """Identity scene -> grasp unchanged; the hand's pose relative to the
    object is invariant under transfer."""
    from paper_2306_08132_b200 import model, pipeline
    od = model.mesh_object(*model.box_mesh((0.04, 0.05, 0.03)))
    rng = np.random.default_rng(0)
    q = np.concatenate([rng.normal(size=3) * 0.05, [0.9, 0.1, -0.3, 0.2], rng.normal(size=4)])
    q[3:7] /= np.linalg.norm(q[3:7])
    ident = np.zeros(13)
    ident[0:3] = od.com
    ident[3] = 1.0
    assert np.allclose(pipeline.transfer_q(q, ident, od.com), q, atol=1e-15)
    s = np.zeros(13)
    s[0:3] = [0.3, -0.2, 0.015]
    s[3:7] = rng.normal(size=4)
    s[3:7] /= np.linalg.norm(s[3:7])
    qt = pipeline.transfer_q(q, s, od.com)
    R = pipeline._rot(s[3:7])
    assert np.allclose(R.T @ (qt[0:3] - pipeline.object_origin(s, od.com)), q[0:3], atol=1e-12)
    # relative orientation: conj(theta) (x) q_t == q_base
    conj = s[3:7] * np.array([1, -1, -1, -1])
    assert np.allclose(pipeline._quat_mul(conj, qt[3:7]), q[3:7], atol=1e-12)
    assert np.array_equal(qt[7:], q[7:])


def test_export_roundtrip(tmp_path):
    from paper_2306_08132_b200 import pipeline
    recs = []
    for k in range(5):
        q = np.linspace(0, 1, 16) + k
        recs.append({"hand": "barrett3" if k < 3 else "pincher2", "object": "box", "q": q,
                     "losses": {"stable": 0.1 * k, "qrange": 1.0, "qlimit": 0.0},
                     "metrics": {"contact_area_cm2": 3.25}, "scene": {"seed": k}})
    man = pipeline.export_jsonl(recs, str(tmp_path), config={"lr": 1e-3})
    assert man["count"] == 5 and sum(man["files"].values()) == 5
    lines = pipeline.import_jsonl(str(tmp_path / "barrett3__box.jsonl"))
    assert len(lines) == 3
    assert lines[1]["base_quaternion"] == [float(f"{v:.9g}") for v in recs[1]["q"][3:7]]
    assert list(lines[0].keys()) == ["hand", "object", "base_position", "base_quaternion", "joint_angles", "losses",
                                     "metrics", "scene"]
    man2 = pipeline.export_jsonl(recs, str(tmp_path / "again"), config={"lr": 1e-3})
    assert man2 == man
    assert (tmp_path / "barrett3__box.jsonl").read_bytes() == (tmp_path / "again" / "barrett3__box.jsonl").read_bytes()
    empty = pipeline.export_jsonl([], str(tmp_path / "empty"))
    assert empty["count"] == 0 and empty["files"] == {}
    json.loads((tmp_path / "manifest.json").read_text())


def test_export_rejects_nonfinite_and_limits(tmp_path):
    """Exported records are valid JSON (no NaN / Infinity) and, given the
    hand's limits, within them."""
    import pytest
    from paper_2306_08132_b200 import pipeline
    q = np.concatenate([[0, 0, 0, 1, 0, 0, 0], np.full(9, 0.5)])
    ok = {"hand": "barrett3", "object": "box", "q": q, "losses": {"stable": 0.1}}
    lim = {"barrett3": (np.zeros(9), np.ones(9))}
    pipeline.export_jsonl([ok], str(tmp_path / "a"), limits=lim)
    with pytest.raises(ValueError, match="non-finite"):
        pipeline.export_jsonl([dict(ok, losses={"stable": float("nan")})], str(tmp_path / "b"))
    bad = dict(ok, q=np.concatenate([q[:7], np.full(9, 1.5)]))
    with pytest.raises(ValueError, match="joint limits"):
        pipeline.export_jsonl([bad], str(tmp_path / "c"), limits=lim)
