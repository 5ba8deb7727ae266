"""Host-side setup of the B200 plan (no GPU): the product's O(N) numbering,
Dirichlet mask, sub_l2g, lumped mass, coarse matrix and AMG aggregation must
equal the reference's (oracle) bit for bit (SURVEY §8a "build_index_maps",
north star: "global numbering and gather lists bit-exact").

The product computes the numbering with a closed-form entity ranking
(csrc/setup_numbering.cpp) instead of the reference's 48-byte-key sort
(mesh.cpp:287-453), so this is an independent check, not a tautology.
"""
import numpy as np
import pytest

import paper_1506_05996_b200 as hx
from oracle import OracleSystem, RefConfig, oracle_available

pytestmark = pytest.mark.skipif(not oracle_available(), reason="oracle/_ref/libhexsem_oracle.so not built")

FAMILIES = ["uniform", "distorted_domain", "distorted_elements"]


def _pair(k, order, family="uniform", refine=0, precond="two_scale", coarse_solve="automatic", boundary="dirichlet",
          kappa_e=None, c_e=None):
    ref = OracleSystem(RefConfig(k=k, order=order, family=family, refine=refine, precond=precond,
                                 coarse_solve=coarse_solve, boundary=boundary))
    mesh = hx.generate_cube_mesh(k, family, boundary)
    for _ in range(refine):
        mesh = hx.refine_uniform(mesh)
    hs = hx.HostSetup(mesh, order, kappa_e, c_e, precond=precond, coarse_solve=coarse_solve)
    return ref, hs, mesh


@pytest.mark.parametrize("family", FAMILIES)
@pytest.mark.parametrize("k", [1, 2, 3])
@pytest.mark.parametrize("refine", [0, 1])
def test_numbering_bit_exact(family, k, refine):
    """3 families x k in {1,2,3} x refine in {0,1} x n = 1..6 (108 cases)."""
    for order in range(1, 7):
        ref, hs, mesh = _pair(k, order, family, refine, precond="fine_only")
        assert hs.N == ref.N
        a, b = hs.maps(), ref.maps()
        for key in ("l2g", "g2l_offsets", "g2l_elem", "g2l_local", "sub_l2g", "dirichlet_mask"):
            assert np.array_equal(a[key], b[key]), (key, family, k, refine, order)


def test_mesh_generators_bit_exact():
    for family in FAMILIES:
        ref = OracleSystem(RefConfig(k=4, order=1, family=family, refine=1, precond="none"))
        m = hx.refine_uniform(hx.generate_cube_mesh(4, family))
        r = ref.mesh()
        assert np.array_equal(m.xyz, r["xyz"]) and np.array_equal(m.conn, r["conn"])
        assert np.array_equal(m.bf_elem, r["bf_elem"]) and np.array_equal(m.bf_face, r["bf_face"])
    box = hx.generate_box_mesh(2, 3, 5, (1.0, 2.0, 3.0))
    assert box.num_elements == 30 and box.num_vertices == 3 * 4 * 6


def test_distorted_elements_rejects_large_k():
    """generate_cube_mesh(k>=9, distorted_elements) throws 'inverted element' (SURVEY §8d caveat)."""
    with pytest.raises(hx.HxbError) as ei:
        hx.generate_cube_mesh(9, "distorted_elements")
    assert ei.value.code == 2  # HXB_EMESH


def test_neumann_and_mixed_masks():
    ref, hs, mesh = _pair(3, 3, boundary="neumann", precond="none")
    assert np.array_equal(hs.maps()["dirichlet_mask"], ref.maps()["dirichlet_mask"])
    assert hs.maps()["dirichlet_mask"].sum() == 0


@pytest.mark.parametrize("case", [dict(k=8, order=3, coarse_solve="amg"), dict(k=4, order=2, coarse_solve="amg"),
                                  dict(k=6, order=4, coarse_solve="amg", family="distorted_elements"),
                                  dict(k=22, order=1, coarse_solve="amg"),
                                  dict(k=20, order=1, coarse_solve="amg", family="distorted_domain")])
def test_amg_hierarchy_bit_exact(case):
    """Aggregates and Galerkin matrices (amg.cpp:53-186) reproduced exactly.
    The k >= 20 cases have 0.5M+ coarse triplets, so the threaded replica of
    the reference's std::sort (setup_parallel.hpp) is what orders the
    duplicate sums there."""
    ref, hs, _ = _pair(**case)
    assert hs.coarse_amg and ref.coarse_amg and hs.amg_levels == ref.amg_levels
    for lvl in range(hs.amg_levels):
        a, b = hs.amg_level(lvl), ref.amg_level(lvl)
        for key in ("ptr", "col", "val", "aggregate"):
            assert np.array_equal(a[key], b[key]), (lvl, key)


def test_lumped_mass_bit_exact():
    for fam in FAMILIES:
        ref, hs, _ = _pair(3, 5, fam, precond="none")
        assert np.array_equal(hs.lumped_mass(), ref.lumped_mass())


def test_per_element_coefficients():
    """Per-element kappa/c (operator.hpp:49-55) enter the coarse matrix exactly."""
    mesh = hx.generate_cube_mesh(4, "distorted_elements")
    ne = mesh.num_elements
    cent = mesh.xyz[mesh.conn].mean(axis=1)
    kap = 1 + 0.5 * np.sin(2 * np.pi * cent[:, 0]) * np.cos(2 * np.pi * cent[:, 1])
    c = 0.1 + cent[:, 2]
    hs = hx.HostSetup(mesh, 3, kap, c, coarse_solve="amg")
    ref = OracleSystem(RefConfig(order=3, coarse_solve="amg"), mesh=mesh.as_dict(), order=3, kappa_e=kap, c_e=c)
    for lvl in range(hs.amg_levels):
        a, b = hs.amg_level(lvl), ref.amg_level(lvl)
        assert np.array_equal(a["val"], b["val"]) and np.array_equal(a["aggregate"], b["aggregate"])
    assert ne == 64


@pytest.mark.parametrize("k,family", [(8, "uniform"), (6, "distorted_elements"), (12, "distorted_domain"), (20, "uniform")])
def test_sparse_direct_coarse_factor(k, family):
    """Nested dissection + supernodal Cholesky of the coupled coarse block
    (setup_nd.cpp), the replacement of the dense coarse inverse behind the
    reference's SimplicialLLT path (coarse.cpp:112-127): a solve with the
    factor reproduces b to rounding, and the factor stays O(n^{4/3})."""
    hs = hx.HostSetup(hx.generate_cube_mesh(k, family), 2, coarse_solve="direct")
    r = hs.coarse_direct_check()
    m = (k - 1) ** 3
    assert r["rel_residual"] <= 1e-12, r
    assert r["factor_entries"] <= 40 * m ** (4 / 3), r
    assert r["levels"] >= 2


@pytest.mark.slow
def test_numbering_bit_exact_cfg2():
    """cfg2 (52^3 hexes, N=7: 72M local entries, 140M subdomain slots): the
    closed-form numbering equals the compiled reference's build_index_maps
    (mesh.cpp:287-453) entry for entry: l2g, the g2l CSR, sub_l2g and the
    Dirichlet mask. Run with HXB_RUN_SLOW=1 (about a minute and 10 GB)."""
    from oracle import RefSystem, ref_available

    if not ref_available():
        pytest.skip("compiled reference not built")
    ref = RefSystem(RefConfig(k=52, order=7, precond="fine_only"))
    b = ref.maps()
    ref.close()
    hs = hx.HostSetup(hx.generate_cube_mesh(52), 7, precond="fine_only")
    a = hs.maps()
    assert hs.N == 48627125
    for key in ("l2g", "g2l_offsets", "g2l_elem", "g2l_local", "sub_l2g", "dirichlet_mask"):
        assert np.array_equal(a[key], b[key]), key
