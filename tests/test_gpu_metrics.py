"""GPU contact generation (dgx_contacts_batch).

Oracle: the reference's own FK (HandModel::forward) and SDF query (the real
MeshSdf::dilated for meshes, the shared backends otherwise) evaluated per
sample on the CPU; a contact is |rho| <= t. Contact index lists, counts and
the recorded (rho, smoothed point, gradient) are bit-exact; the contact area
(a sum in a different order) within 1e-12 relative.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("obj_name", ["ico25", "sphere25", "boxgrid64"])
def test_contacts_vs_reference(ctx, oracle, obj_name):
    from paper_2306_08132_b200 import api, init, metrics, model
    od = {"ico25": lambda: model.mesh_object(*model.icosphere_mesh(0.025, 3)),
          "sphere25": lambda: model.sphere(0.025), "boxgrid64": lambda: model.box_grid(res=64)}[obj_name]()
    hd = model.HandDesc.asset("barrett3")
    rh = oracle.RefHand.barrett3()
    ro = oracle.RefObject.from_desc(od)
    hand, obj = api.Hand(ctx, hd), api.GraspObject(ctx, od)
    q = init.approach_init(od, hd, 6, seed=4)
    q[:, :3] -= 0.5 * (q[:, :3] - od.com)  # pull in so there are contacts
    thr_mm = (1.0, 2.0, 5.0, 9.0)
    con = metrics.contacts(ctx, hand, obj, q, thr_mm)
    assert np.all(np.diff(con.count, axis=1) >= 0) and np.all(np.diff(con.area, axis=1) >= 0)
    assert np.sum(con.n) > 0
    for b in range(q.shape[0]):
        pts = rh.forward(q[b])
        qs = np.array([ro.query(p, 0.0) for p in pts])
        rho = np.abs(qs[:, 0])
        for t, tm in enumerate(thr_mm):
            sel = rho <= tm * 1e-3
            assert con.count[b, t] == int(np.sum(sel)), (b, t)
            want = float(np.sum(hd.sample_area[sel]))
            assert abs(con.area[b, t] - want) <= 1e-12 * max(want, 1e-30), (b, t)
        idx = np.flatnonzero(rho <= thr_mm[-1] * 1e-3)
        assert con.n[b] == idx.size
        assert np.array_equal(con.index[b, : idx.size], idx)
        assert np.array_equal(con.rec[b, : idx.size, 0], qs[idx, 0])
        assert np.array_equal(con.rec[b, : idx.size, 1:4], qs[idx, 4:7])
        assert np.array_equal(con.rec[b, : idx.size, 4:7], qs[idx, 1:4])


def test_flush_plate_and_metrics(ctx):
    """100 samples of a 10 cm^2 plate flush on a cube face
    are all contacts at 5 mm and give CA = 10 cm^2; a plate 2 cm away has none."""
    from paper_2306_08132_b200 import api, metrics, model
    g = (np.arange(10) - 4.5) * 1e-3
    samples = np.array([[x, y, 0.0] for x in g for y in g])
    hd = model.HandDesc(name="plate", topo=np.array([0], np.int32), link_parent_joint=np.array([-1], np.int32),
                        joint_parent=np.zeros(0, np.int32), joint_child=np.zeros(0, np.int32),
                        axis=np.zeros((0, 3)), origin_R=np.zeros((0, 9)), origin_t=np.zeros((0, 3)),
                        lower=np.zeros(0), upper=np.zeros(0), samples=samples,
                        sample_link=np.zeros(100, np.int32), sample_area=np.full(100, 0.1e-4))
    hand = api.Hand(ctx, hd)
    obj = api.GraspObject(ctx, model.box((0.04, 0.04, 0.04)))
    q = np.array([[0.0, 0.0, 0.02, 1.0, 0.0, 0.0, 0.0], [0.0, 0.0, 0.04, 1.0, 0.0, 0.0, 0.0]])
    con = metrics.contacts(ctx, hand, obj, q, (5.0,))
    assert con.count[0, 0] == 100 and abs(con.area[0, 0] * 1e4 - 10.0) < 1e-9
    assert con.count[1, 0] == 0 and con.area[1, 0] == 0.0
    rep = metrics.evaluate(ctx, hand, obj, q, (5.0,))
    # a single flat contact patch: no force closure
    assert rep[0][0]["epsilon"] == 0.0 and rep[1][0]["contacts"] == 0
