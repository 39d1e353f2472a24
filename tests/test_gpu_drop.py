"""GPU scene drop (csrc/dgx_drop.cu) vs the reference's step_on_table.

Bar: BIT-EXACT against the reference's own step_on_table (sim.cpp:14-94) and
kinetic_energy (sim.cpp:8-12), iterated on the CPU with the same stopping rule
(oracle/ref_shim.cpp dgr_drop, parity mode P). Checked over the whole
trajectory (every 25th state), the final state, step count, final kinetic
energy and the shared SolveStats, for icosphere / box / cylinder / blob meshes
dropped from random orientations. Plus SPEC.md:541-545 properties.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def objects(oracle):
    from paper_2306_08132_b200 import model
    out = {}
    for name, ro in {"ico3": oracle.RefObject.icosphere(0.025, 3), "box": oracle.RefObject.box_mesh(0.04, 0.05, 0.03),
                     "cyl32": oracle.RefObject.cylinder_mesh(0.0175, 0.07, 32),
                     "blob2": oracle.RefObject.blob_mesh(0.021, 2, 0.5, 3)}.items():
        V, F, _ = ro.mesh_export()
        out[name] = (ro, model.mesh_object(V, F))
    return out


@pytest.mark.parametrize("mu", [1.0, 0.0])
def test_drop_bit_exact(ctx, oracle, mu):
    from paper_2306_08132_b200 import api, pipeline
    params = api.DropParams(mu=mu, max_steps=1500, ke_tol=1e-6, measure_residual=True)
    for name, (ro, od) in objects(oracle).items():
        obj = api.GraspObject(ctx, od)
        s0 = pipeline.scene_states(od, np.arange(6) + 40)
        s0[1, 7:10] = [0.05, -0.02, 0.0]     # thrown
        s0[2, 10:13] = [3.0, -1.0, 2.0]      # spinning
        r = api.drop(ctx, obj, s0, params, record_every=25)
        for b in range(s0.shape[0]):
            st, steps, ke, stats, traj = oracle.drop(ro, s0[b], mu=mu, max_steps=1500, ke_tol=1e-6, measure=True,
                                                     record_every=25)
            assert r["steps"][b] == steps, (name, b, r["steps"][b], steps)
            assert np.array_equal(r["state"][b], st), (name, b, r["state"][b] - st)
            assert r["ke"][b] == ke, (name, b)
            assert np.array_equal(r["stats"][b], stats), (name, b, r["stats"][b], stats)
            assert np.array_equal(r["traj"][b, : steps // 25], traj[: steps // 25]), (name, b)


def test_drop_rest_properties(ctx, oracle):
    """sphere rests at COM height = radius within 2 mm; a box
    rests on a face (within 1 degree); same seed -> identical scene."""
    from paper_2306_08132_b200 import api, model, pipeline
    sph = api.GraspObject(ctx, model.mesh_object(*model.icosphere_mesh(0.025, 3)))
    sc = pipeline.generate_scenes(ctx, sph, np.arange(8))
    # the reference's step_on_table keeps a faceted sphere rocking on its
    # vertices (KE ~1e-6..5e-5 J after 5 s, bit-identical on the CPU), so only
    # the rest height is asserted for it
    assert np.all(np.abs(sc.state[:, 2] - 0.025) < 2e-3), sc.state[:, 2]
    box = api.GraspObject(ctx, model.mesh_object(*model.box_mesh((0.04, 0.05, 0.03))))
    sb = pipeline.generate_scenes(ctx, box, np.arange(8))
    assert np.all(sb.at_rest)
    for q in sb.state[:, 3:7]:
        R = pipeline._rot(q)
        # some body axis is (anti)parallel to world z within 1 degree
        assert np.max(np.abs(R[2, :])) > np.cos(np.radians(1.0)), R
    sb2 = pipeline.generate_scenes(ctx, box, np.arange(8))
    assert np.array_equal(sb.state, sb2.state) and np.array_equal(sb.steps, sb2.steps)
    # rest poses are stable: 1 s more simulation moves the COM < 1 mm
    again = api.drop(ctx, box, sb.state, api.DropParams(max_steps=1000, min_steps=1000))
    assert np.all(np.linalg.norm(again["state"][:, 0:3] - sb.state[:, 0:3], axis=1) < 1e-3)


def test_drop_free_fall_and_errors(ctx):
    """No contact: the predicted state stands (free flight exact); grids /
    analytic objects are rejected (the table contacts are mesh vertices)."""
    from paper_2306_08132_b200 import api, capi, model
    obj = api.GraspObject(ctx, model.mesh_object(*model.icosphere_mesh(0.02, 2)))
    s0 = np.zeros((1, 13))
    s0[0, 2] = 10.0
    s0[0, 3] = 1.0
    r = api.drop(ctx, obj, s0, api.DropParams(max_steps=100))
    assert r["steps"][0] == 100 and r["stats"][0, 1] == 0
    v = 0.0
    z = 10.0
    for _ in range(100):  # symplectic Euler of predict (sim.hpp:74-83)
        v = v + (-9.81 * 1e-3)
        z = z + 1e-3 * v
    assert r["state"][0, 2] == z and r["state"][0, 9] == v
    sph = api.GraspObject(ctx, model.sphere(0.02))
    with pytest.raises(capi.DgxError):
        api.drop(ctx, sph, s0)


def test_transfer_grasps(ctx):
    """Transfer keeps the hand-object relative pose (to 1e-9) and
    rejects a grasp whose hand dips below the table."""
    from paper_2306_08132_b200 import api, init, model, pipeline
    hd = model.HandDesc.asset("barrett3")
    od = model.mesh_object(*model.box_mesh((0.04, 0.05, 0.03)))
    ctx_h = api.Hand(ctx, hd)
    gobj = api.GraspObject(ctx, od)
    sc = pipeline.generate_scenes(ctx, gobj, np.arange(4))
    qb = init.approach_init(od, hd, 6, seed=2)
    qs, ok, zmin = pipeline.transfer_grasps(ctx, ctx_h, od, qb, sc)
    for g in range(qb.shape[0]):
        for s in range(4):
            R = pipeline._rot(sc.state[s, 3:7])
            # relative pose: hand base in the object's frame is unchanged
            rel_new = R.T @ (qs[g, s, 0:3] - pipeline.object_origin(sc.state[s], od.com))
            assert np.allclose(rel_new, qb[g, 0:3], atol=1e-9)
    pts = api.forward(ctx, ctx_h, qs.reshape(-1, qs.shape[-1]))
    assert np.array_equal(ok.reshape(-1), pts[:, :, 2].min(axis=1) >= 0.0)
    assert not np.all(ok) or np.all(zmin >= 0)
