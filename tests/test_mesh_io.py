"""Mesh file formats either side of the solve: Gmsh MSH 2.2
and the native "HXSM0001" binary, host C++ in csrc/setup_mesh_io.cpp behind
hxb_read_mesh_file / hxb_write_mesh_file.

Cases follow the reference's tests/test_io.cpp (native round trip exact, msh
round trip keeps topology and tags, sparse node ids and foreign element
types, garbage rejected) and add cross-implementation checks: files written
by the unmodified reference (oracle/_ref) read back identically by the
product and vice versa, byte-identical files from both writers.
"""
import os

import numpy as np
import pytest

import paper_1506_05996_b200 as hx
from oracle import ref_available, ref_read_mesh, ref_write_mesh

needs_ref = pytest.mark.skipif(not ref_available(), reason="oracle/_ref/libhexsem_ref.so not built")


def _faces(m):
    return sorted(zip(m.bf_elem.tolist(), m.bf_face.tolist(), m.bf_tag.tolist()))


def _same(a, b, exact=True):
    assert a.num_vertices == b.num_vertices and a.num_elements == b.num_elements
    if exact:
        assert np.array_equal(a.xyz, b.xyz)
    else:
        np.testing.assert_allclose(a.xyz, b.xyz, rtol=1e-15, atol=0)
    assert np.array_equal(a.conn, b.conn)
    assert _faces(a) == _faces(b)


def _mixed(k=2, family="distorted_domain"):
    m = hx.generate_cube_mesh(k, family)
    m.bf_tag = np.where(m.bf_face == 0, 1, m.bf_tag).astype(np.uint8)  # -x faces Neumann
    return m


def test_native_round_trip_exact(tmp_path):
    m = hx.generate_cube_mesh(3, "distorted_elements")
    p = str(tmp_path / "roundtrip.hxm")
    hx.write_native(m, p)
    assert os.path.getsize(p) == 32 + 24 * m.num_vertices + 32 * m.num_elements + 12 * m.bf_elem.size
    _same(m, hx.read_native(p))
    _same(m, hx.read_mesh_file(p))  # anything but .msh dispatches to native


def test_msh_round_trip_topology_and_tags(tmp_path):
    m = _mixed()
    p = str(tmp_path / "roundtrip.msh")
    hx.write_msh(m, p)
    back = hx.read_mesh_file(p)
    _same(m, back)  # %.17g round-trips doubles exactly
    a, b = hx.HostSetup(m, 2, precond="none"), hx.HostSetup(back, 2, precond="none")
    assert a.N == b.N
    assert np.array_equal(a.maps(sub=False)["dirichlet_mask"], b.maps(sub=False)["dirichlet_mask"])


SPARSE = (
    "$MeshFormat\n2.2 0 8\n$EndMeshFormat\n"
    "$PhysicalNames\n1\n2 1 \"wall\"\n$EndPhysicalNames\n"
    "$Nodes\n12\n"
    "100 0 0 0\n101 1 0 0\n102 1 1 0\n103 0 1 0\n"
    "104 0 0 1\n105 1 0 1\n106 1 1 1\n107 0 1 1\n"
    "200 0 0 2.0e0\n201 1 0 2\n202 1 1 2\n203 0 1 2\n"
    "$EndNodes\n"
    "$Elements\n6\n"
    "1 15 2 0 0 100\n"
    "2 1 2 0 0 100 101\n"
    "3 5 2 0 0 100 101 102 103 104 105 106 107\n"
    "4 5 2 0 0 104 105 106 107 200 201 202 203\n"
    "5 3 2 1 1 100 101 102 103\n"
    "6 3 2 2 2 203 202 201 200\n"
    "$EndElements\n"
)


def test_msh_sparse_ids_and_foreign_types(tmp_path):
    p = tmp_path / "sparse.msh"
    p.write_text(SPARSE)
    m = hx.read_msh(str(p))
    assert m.num_vertices == 12 and m.num_elements == 2
    assert _faces(m) == [(0, 4, 0), (1, 5, 1)]  # bottom Dirichlet (tag 1), top Neumann (tag 2)
    hs = hx.HostSetup(m, 2, precond="none")
    assert hs.N == 5 * 3 * 3  # the two hexes share a conforming face


def test_crlf_and_blank_tolerance(tmp_path):
    p = tmp_path / "crlf.msh"
    p.write_bytes(SPARSE.replace("\n", "\r\n").encode())
    m = hx.read_msh(str(p))
    assert m.num_elements == 2 and len(_faces(m)) == 2


@pytest.mark.parametrize("text,code", [
    ("$MeshFormat\n4.1 0 8\n$EndMeshFormat\n", hx.HxbError),
    ("$MeshFormat\n2.2 0 8\n$EndMeshFormat\n$Nodes\n1\n1 0 0 0\n$EndNodes\n", hx.HxbError),  # no hexahedra
    ("$Nodes\n8\n" + "".join(f"{i} {i & 1} {(i >> 1) & 1} {i >> 2}\n" for i in range(8)) + "$EndNodes\n"
     "$Elements\n1\n1 5 2 0 0 0 1 3 2 4 5 7 99\n$EndElements\n", hx.HxbError),  # unknown node id
    ("$Nodes\n3\n1 0 0\n", hx.HxbError),  # malformed / truncated
])
def test_msh_rejects_garbage(tmp_path, text, code):
    p = tmp_path / "bad.msh"
    p.write_text(text)
    with pytest.raises(code) as ei:
        hx.read_msh(str(p))
    assert ei.value.code == 6  # HXB_EIO


def test_missing_and_corrupt_files(tmp_path):
    for fn in (hx.read_msh, hx.read_native, hx.read_mesh_file):
        with pytest.raises(hx.HxbError):
            fn(str(tmp_path / "does_not_exist.msh"))
    m = hx.generate_cube_mesh(2)
    p = str(tmp_path / "m.hxm")
    hx.write_native(m, p)
    raw = open(p, "rb").read()
    open(p, "wb").write(raw[:-5])
    with pytest.raises(hx.HxbError, match="truncated"):
        hx.read_native(p)
    open(p, "wb").write(b"HXSM0002" + raw[8:])
    with pytest.raises(hx.HxbError, match="not a hexsem native mesh"):
        hx.read_native(p)


def test_unmatched_quad_and_inverted_element(tmp_path):
    p = tmp_path / "q.msh"
    p.write_text(SPARSE.replace("5 3 2 1 1 100 101 102 103", "5 3 2 1 1 100 101 105 104")
                 .replace("6 3 2 2 2 203 202 201 200", "6 3 2 2 2 100 102 105 107"))
    with pytest.raises(hx.HxbError, match="does not match"):
        hx.read_msh(str(p))
    m = hx.generate_cube_mesh(1)
    m.conn = m.conn[:, [1, 0, 2, 3, 5, 4, 6, 7]].copy()  # mirrored: negative Jacobian
    q = str(tmp_path / "inv.hxm")
    hx.write_native(m, q)
    with pytest.raises(hx.HxbError) as ei:
        hx.read_native(q)
    assert ei.value.code == 2  # HXB_EMESH, check_jacobians (geometry.cpp:153-161)


def test_problem_config_mesh_file(tmp_path):
    """make_mesh reads config.mesh_file first (problem.cpp:16-17); write_mesh
    (module.cpp:102-105) writes make_mesh(config)."""
    p = str(tmp_path / "gen.msh")
    hx.write_mesh(p, k=2, family="distorted_elements", refine=1)
    gen = hx.make_mesh(hx.ProblemConfig(k=2, family="distorted_elements", refine=1))
    _same(gen, hx.make_mesh(hx.ProblemConfig(mesh_file=p)))
    info = hx.mesh_info(mesh_file=p, order=3)
    assert info["num_elements"] == 64


@needs_ref
@pytest.mark.parametrize("fmt,ext", [("msh", "msh"), ("native", "hxm")])
def test_cross_implementation(tmp_path, fmt, ext):
    """Reference writer -> product reader and product writer -> reference
    reader give the same mesh; both writers emit byte-identical files."""
    m = _mixed(3, "distorted_elements")
    pr, pp = str(tmp_path / f"ref.{ext}"), str(tmp_path / f"prod.{ext}")
    ref_write_mesh(m.as_dict(), pr, fmt)
    hx.write_mesh_file(m, pp, fmt)
    assert open(pr, "rb").read() == open(pp, "rb").read()
    _same(m, hx.read_mesh_file(pr, fmt))
    r = ref_read_mesh(pp, fmt)
    _same(m, hx.HexMesh(r["xyz"], r["conn"], r["bf_elem"], r["bf_face"], r["bf_tag"]))


@needs_ref
def test_reader_parity_on_handwritten_file(tmp_path):
    p = tmp_path / "sparse.msh"
    p.write_text(SPARSE)
    r = ref_read_mesh(str(p), "msh")
    _same(hx.HexMesh(r["xyz"], r["conn"], r["bf_elem"], r["bf_face"], r["bf_tag"]), hx.read_msh(str(p)))


@pytest.mark.gpu
def test_solve_from_mesh_file_matches_generator(tmp_path):
    """test_io.cpp "solving from a mesh file matches the generator": the device
    solve on a re-read mesh gives the same iterations and residual history."""
    p = str(tmp_path / "gen.msh")
    hx.write_mesh(p, k=2, family="distorted_elements")
    a = hx.solve_poisson(k=2, family="distorted_elements", order=2)
    b = hx.solve_poisson(mesh_file=p, order=2)
    assert a["report"]["iterations"] == b["report"]["iterations"]
    assert a["report"]["N"] == b["report"]["N"]
    assert a["report"]["residual_history"] == b["report"]["residual_history"]
