"""The C-ABI library (include/hexsem_b200.h) loads on a CPU-only host,
exports every declared symbol, and maps reference exceptions to error codes
(SURVEY §8b). No compute call needs a GPU here."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_1506_05996_b200 as hx

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "hexsem_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hxb_[a-z0-9_]+)\s*\(", src)))


def test_every_declared_symbol_is_exported():
    names = _declared()
    assert len(names) >= 30
    L = C.CDLL(hx.hexsem.LIB_PATH)
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    # and the Python mirror binds every one of them
    assert set(names) <= set(hx.hexsem.SIGNATURES), set(names) - set(hx.hexsem.SIGNATURES)


def test_library_is_sm100a_only():
    """The kernels are compiled for sm_100a and nothing else (no PTX/JIT fallback)."""
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", hx.hexsem.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    archs = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert archs == {"100a"}, archs
    ptx = subprocess.run(["cuobjdump", "--list-ptx", hx.hexsem.LIB_PATH], capture_output=True, text=True)
    assert "ptx" not in ptx.stdout.lower().replace("list-ptx", "")


def test_error_codes():
    L = hx.lib()
    t = np.zeros(2)
    assert L.hxb_gll(0, t.ctypes.data, t.ctypes.data, t.ctypes.data) == 1  # HXB_EINVAL: order >= 1 (gll.cpp:34)
    assert b"order" in L.hxb_last_error()
    with pytest.raises(hx.HxbError) as ei:
        hx.generate_cube_mesh(0)
    assert ei.value.code == 1
    # non-conforming mesh: three elements on one face (mesh.cpp:402-403)
    m = hx.generate_box_mesh(2, 1, 1)
    conn = np.vstack([m.conn, m.conn[:1]])
    bad = hx.HexMesh(m.xyz, conn, m.bf_elem, m.bf_face, m.bf_tag)
    with pytest.raises(hx.HxbError) as ei:
        hx.HostSetup(bad, 2)
    assert ei.value.code == 2
    # inverted element (geometry.cpp:70-72)
    m = hx.generate_box_mesh(1, 1, 1)
    xyz = m.xyz.copy()
    xyz[:, 0] *= -1
    with pytest.raises(hx.HxbError) as ei:
        hx.HostSetup(hx.HexMesh(xyz, m.conn, m.bf_elem, m.bf_face, m.bf_tag), 2)
    assert ei.value.code == 2


def test_counter_models_match_reference():
    assert hx.residual_flops_model(32768, 3) == 138412032
    assert hx.residual_words_model(1, 1) == 86
    assert hx.fine_ops_model(1, 1) == 6 * 256 + 15 * 64
    # cfg2 algorithmic Ax bytes
    assert hx.residual_words_model(52 ** 3, 7) * 8 == 5833544704


def test_gll_and_pencil_tables_match_oracle():
    from oracle import oracle_available, oracle_gll, oracle_pencil

    if not oracle_available():
        pytest.skip("oracle not built")
    for n in range(1, 11):
        t, w, D = hx.gll(n)
        to, wo, Do, _ = oracle_gll(n)
        assert np.array_equal(t, to) and np.array_equal(w, wo) and np.array_equal(D, Do)
        P, Po = hx.pencil(n), oracle_pencil(n)
        assert np.array_equal(P["K"], Po["K"]) and np.array_equal(P["M"], Po["M"])
        R = P["V_inv"] @ np.diag(P["lambda"]) @ P["V"]
        Ro = Po["V_inv"] @ np.diag(Po["lambda"]) @ Po["V"]
        assert np.max(np.abs(R - Ro)) <= 1e-12 * np.max(np.abs(Ro))


def test_plan_create_fails_loudly_without_gpu():
    """No CPU fallback: without an sm_100 device the plan refuses (HXB_ECUDA)."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    mesh = hx.generate_cube_mesh(2)
    with pytest.raises(hx.HxbError) as ei:
        hx.Plan(mesh, 2)
    assert ei.value.code == 4


def test_plan_rejects_empty_mesh():
    """An empty mesh is an argument error (HXB_EINVAL), raised before any
    device work, like the reference readers' "no hexahedra" (mesh_io.cpp:118)."""
    import numpy as np

    empty = hx.HexMesh(np.zeros((0, 3)), np.zeros((0, 8), dtype=np.int32), np.zeros(0, dtype=np.int32),
                       np.zeros(0, dtype=np.int32), np.zeros(0, dtype=np.uint8))
    with pytest.raises(hx.HxbError) as ei:
        hx.Plan(empty, 3)
    assert ei.value.code == 1 and "no hexahedra" in str(ei.value)


def test_pencil_bitwise_vs_reference():
    """build_pencil (fine.cpp:15-80): the product's pencil (K, M, V, V^-1,
    lambda) equals the compiled reference's bit for bit for every order, so
    the bitwise-reference FDM (compat.cu) can reproduce solve_subdomain."""
    from oracle import ref_available, ref_pencil

    if not ref_available():
        pytest.skip("reference not built")
    for n in range(1, 11):
        P, R = hx.pencil(n), ref_pencil(n)
        for key in ("K", "M", "V", "V_inv", "lambda"):
            assert np.array_equal(P[key], R[key]), (n, key)
