"""Mesh backend, host side (no GPU): the BVH the C-ABI builds for a mesh object,
inertia_from_mesh, TriMesh validation and the mesh generators / OBJ loader,
each against the compiled reference (oracle/_ref).

  * BVH (bvh.cpp:66-103): node boxes, child links and leaf face SETS identical
    to the reference's Bvh::nodes() (so traversal order and pruning match);
  * inertia_from_mesh (rigid.cpp:24-94): mass / COM / inertia / inverse
    bit-identical;
  * TriMesh::finalize errors (mesh.cpp:12-71): same messages;
  * model.icosphere_mesh == assets.cpp make_icosphere bit-for-bit.
"""
import numpy as np
import pytest


def ref_meshes(oracle):
    return {
        "ico3": oracle.RefObject.icosphere(0.025, 3),
        "ico1": oracle.RefObject.icosphere(0.03, 1),
        "box": oracle.RefObject.box_mesh(0.04, 0.05, 0.03),
        "cyl32": oracle.RefObject.cylinder_mesh(0.0175, 0.07, 32),
        "blob3": oracle.RefObject.blob_mesh(0.021, 3, 0.5, 7),
    }


def test_bvh_matches_reference(oracle):
    from paper_2306_08132_b200 import api
    for name, ro in ref_meshes(oracle).items():
        V, F, _ = ro.mesh_export()
        b1, l1, fo1 = ro.bvh()
        b2, l2, fo2 = api.mesh_bvh(V, F)
        assert b1.shape == b2.shape, name
        assert np.array_equal(b1, b2), name
        assert np.array_equal(l1[:, :2], l2[:, :2]), name          # children
        leaf = l1[:, 0] < 0
        assert np.array_equal(l1[leaf, 2:], l2[leaf, 2:]), name     # leaf ranges
        for i in np.flatnonzero(leaf):
            a, n = l1[i, 2], l1[i, 3]
            assert sorted(fo1[a:a + n]) == sorted(fo2[a:a + n]), (name, i)


def test_inertia_from_mesh_bit_exact(oracle):
    from paper_2306_08132_b200 import model
    for name, ro in ref_meshes(oracle).items():
        V, F, _ = ro.mesh_export()
        od = model.mesh_object(V, F, 1000.0)
        m, com, I, Iinv = ro.inertial()
        assert od.mass == m and np.array_equal(od.com, com), name
        assert np.array_equal(od.inertia_body, I) and np.array_equal(od.inertia_body_inv, Iinv), name


def test_icosphere_generator_matches_reference(oracle):
    from paper_2306_08132_b200 import model
    for r, s in ((0.025, 3), (0.04, 2), (0.01, 0)):
        V, F = model.icosphere_mesh(r, s)
        V2, F2, _ = oracle.RefObject.icosphere(r, s).mesh_export()
        assert np.array_equal(F, F2) and np.array_equal(V, V2)


def _ref_error(oracle, V, F):
    with pytest.raises(oracle.RefError) as ei:
        oracle.RefObject.mesh(V, F)
    return str(ei.value)


def _our_error(V, F):
    from paper_2306_08132_b200 import capi, model
    with pytest.raises(capi.DgxError) as ei:
        model.mesh_object(V, F)
    return str(ei.value)


@pytest.mark.parametrize("defect", ["hole", "flip", "degenerate", "range", "repeat", "inverted"])
def test_mesh_validation_messages(oracle, defect):
    from paper_2306_08132_b200 import model
    V, F = model.icosphere_mesh(0.02, 1)
    F = F.copy()
    V = V.copy()
    if defect == "hole":
        F = F[1:]
    elif defect == "flip":
        F[3] = F[3][::-1]
    elif defect == "degenerate":
        V[F[5][1]] = V[F[5][0]]
    elif defect == "range":
        F[2, 1] = V.shape[0] + 3
    elif defect == "repeat":
        F[4, 2] = F[4, 0]
    elif defect == "inverted":
        F = F[:, ::-1].copy()
    ours, theirs = _our_error(V, F), _ref_error(oracle, V, F)
    assert theirs in ours, (ours, theirs)


def test_load_obj(tmp_path):
    from paper_2306_08132_b200 import model
    p = tmp_path / "quad.obj"
    p.write_text("# cube as quads\nv -1 -1 -1\nv 1 -1 -1\nv -1 1 -1\nv 1 1 -1\n"
                 "v -1 -1 1\nv 1 -1 1\nv -1 1 1\nv 1 1 1\nvn 0 0 1\n"
                 "f 1 3 4 2\nf 5/1 6/1 8/1 7/1\nf 1//1 2//1 6//1 5//1\nf -6 -2 -1 -5\nf 1 5 7 3\nf 2 4 8 6\n")
    V, F = model.load_obj(str(p))
    assert V.shape == (8, 3) and F.shape == (12, 3)
    assert F[:2].tolist() == [[0, 2, 3], [0, 3, 1]]
    assert F[6:8].tolist() == [[2, 6, 7], [2, 7, 3]]  # negative indices are relative
    od = model.mesh_object(V, F, density=1.0)
    assert abs(od.mass - 8.0) < 1e-12
    with pytest.raises(RuntimeError, match="fewer than 3"):
        bad = tmp_path / "bad.obj"
        bad.write_text("v 0 0 0\nv 1 0 0\nf 1 2\n")
        model.load_obj(str(bad))


def test_box_mesh_volume():
    from paper_2306_08132_b200 import model
    od = model.mesh_object(*model.box_mesh((0.04, 0.05, 0.03)), density=1000.0)
    assert abs(od.mass - 0.06) < 1e-15
    assert np.allclose(od.com, 0.0, atol=1e-18)
