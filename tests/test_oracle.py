"""Pin the CPU oracle (oracle/hexsem_oracle.cpp restatement) before trusting it.

(a) Known answers from the reference's own tests and recorded runs
    (SURVEY §8c): node counts (test_mesh.cpp:64-110), counter models
    (test_operator.cpp:151-181, test_fine.cpp:150-162), PCG iteration ladders
    (proj/test_output.txt:28-30) and the cfg1 residual endpoints
    (BASELINE.md §2).
(b) The compiled reference (oracle/_ref/libhexsem_ref.so, unmodified
    /root/reference sources + Eigen-API shim) on identical inputs: integer
    maps bit-exact, Ax bit-exact, P / PCG within rounding.
No GPU needed.
"""
import numpy as np
import pytest

from oracle import (OracleSystem, RefConfig, RefSystem, oracle_available, oracle_gll, oracle_pencil, ref_available,
                    ref_gll, ref_pencil, splitmix_vector)

pytestmark = pytest.mark.skipif(not oracle_available(), reason="oracle/_ref/libhexsem_oracle.so not built")
needs_ref = pytest.mark.skipif(not ref_available(), reason="compiled reference (oracle/_ref) not built")


def orc(**kw):
    return OracleSystem(RefConfig(**kw))


# --- (a) known answers -------------------------------------------------------
@pytest.mark.parametrize("k", [1, 2, 4])
@pytest.mark.parametrize("n", [1, 2, 3, 4, 5])
def test_structured_node_count(k, n):
    """(k n + 1)^3 global nodes (test_mesh.cpp:64-74)."""
    assert orc(k=k, order=n, precond="none").N == (k * n + 1) ** 3


def test_k32_n3_node_count():
    """test_mesh.cpp:76-81: k=32, n=3 -> 97^3 = 912,673."""
    assert orc(k=32, order=3, precond="none").N == 912673


def test_copies_and_single_element():
    s = orc(k=1, order=2, precond="none")
    m = s.maps(sub=False)
    assert s.N == 27 and np.all(np.diff(m["g2l_offsets"]) == 1)  # test_mesh.cpp:83-89
    s = orc(k=2, order=2, precond="none")
    m = s.maps(sub=False)
    copies = np.diff(m["g2l_offsets"])
    assert copies.max() == 8 and copies.sum() == s.NE * 27  # test_mesh.cpp:91-110
    # centre vertex (0.5,0.5,0.5) is mesh vertex 13 -> global id 13 (vertices ranked first)
    assert copies[13] == 8


def test_dirichlet_shell():
    """Dirichlet shell of a 2^3, n=2 cube: 5^3 - 3^3 = 98 nodes (test_mesh.cpp:243-256)."""
    m = orc(k=2, order=2, precond="none").maps(sub=False)
    assert int(m["dirichlet_mask"].sum()) == 98


def test_sub_l2g_structure():
    """sub_l2g: interior slots mirror l2g, edges/corners are sentinel (mesh.cpp:385-451)."""
    n = 3
    s = orc(k=2, order=n, precond="none")
    m = s.maps()
    p, np1 = n + 3, n + 1
    sub = m["sub_l2g"].reshape(s.NE, p, p, p)
    l2g = m["l2g"].reshape(s.NE, np1, np1, np1)
    assert np.array_equal(sub[:, 1:-1, 1:-1, 1:-1], l2g)
    for a, b in [(0, 0), (0, -1), (-1, 0), (-1, -1)]:
        assert np.all(sub[:, a, b, :] == -1) and np.all(sub[:, :, a, b] == -1) and np.all(sub[:, a, :, b] == -1)
    # element 0 touches the x+ neighbour (element 1): its x=n+1 face slots are filled
    assert np.all(sub[0, 1:-1, 1:-1, -1] >= 0) and np.all(sub[0, 1:-1, 1:-1, 0] == -1)


def test_counter_models():
    """O_R(32768,3)=138,412,032 and B_R(1,1)=86 words (test_operator.cpp:151-181); O_P(1,1) (test_fine.cpp:161)."""
    from oracle.ctypes_oracle import _ORC_SO, _load

    L = _load(_ORC_SO, "orc_")
    assert L.orc_flops_model(32768, 3) == 138412032
    assert L.orc_words_model(1, 1, 0) == 86
    assert L.orc_fine_ops_model(1, 1) == 6 * 256 + 15 * 64
    assert L.orc_fine_words_model(1, 1) == 3 * 64 + 4 * 16


def test_gll_tables():
    for n in range(1, 11):
        t, w, D, B = oracle_gll(n)
        assert t[0] == -1 and t[-1] == 1 and np.all(np.diff(t) > 0)
        assert abs(w.sum() - 2) < 1e-14
        # D differentiates polynomials of degree <= n exactly: sum_i u(t_i) D[i][j] = u'(t_j)
        for deg in range(n + 1):
            assert np.allclose((t ** deg) @ D, deg * t ** max(deg - 1, 0) if deg else 0, atol=1e-10 * n * n)
        assert np.allclose(B.sum(axis=0), 1.0)  # partition of unity of the 8 hats


def test_pencil_reconstruction():
    """V^-1 diag(lambda) V == M^-1 K (test_fine.cpp:66-84), lambda > 0 ascending (:58-65)."""
    for n in range(1, 11):
        P = oracle_pencil(n)
        lam = P["lambda"]
        assert np.all(lam > 0) and np.all(np.diff(lam) >= 0)
        L = np.diag(1 / P["M"]) @ P["K"]
        R = P["V_inv"] @ np.diag(lam) @ P["V"]
        assert np.max(np.abs(L - R)) <= 1e-10 * np.max(np.abs(L))


@pytest.mark.parametrize("precond,tol,iters", [("two_scale", 1e-6, 22), ("two_scale", 1e-8, 29), ("none", 1e-6, 97),
                                               ("none", 1e-8, 118)])
def test_cfg1_iterations(precond, tol, iters):
    """cfg1 8^3, N=4, s=1 (BASELINE.md §2 reference runs)."""
    s = orc(k=8, order=4, precond=precond)
    res = s.pcg(s.load_ones(), tol=tol, max_iterations=500)
    assert res["status"] == "converged" and res["iterations"] == iters
    assert res["residual_history"][0] == pytest.approx(0.006666808217133652, rel=1e-15)
    if precond == "two_scale" and tol == 1e-8:
        assert res["residual_history"][-1] == pytest.approx(5.3053096645428634e-11, rel=1e-9)


@pytest.mark.parametrize("family,expect", [("uniform", [18, 21]), ("distorted_domain", [21, 24])])
def test_table1_ladder(family, expect):
    """Two-scale ladder k=8 -> 16 (refine 0,1), n=3, tol 1e-6 (test_output.txt:28: Mesh1 18,21,22; Mesh2 21,24,26)."""
    its = []
    for refine in range(2):
        s = orc(k=8, order=3, refine=refine, family=family)
        its.append(s.pcg(s.load_ones(), tol=1e-6)["iterations"])
    assert its == expect


def test_fine_only_growth():
    """Fine-only growth ratio Mesh1 8^3 -> 16^3 = 1.76 (test_output.txt:30: 21 -> 37)."""
    its = []
    for refine in range(2):
        s = orc(k=8, order=3, refine=refine, precond="fine_only")
        its.append(s.pcg(s.load_ones(), tol=1e-6)["iterations"])
    assert its == [21, 37]


def test_operator_properties():
    """Symmetry on random pairs and Dirichlet identity rows (test_operator.cpp:68-89)."""
    s = orc(k=3, order=4, family="distorted_elements", c=0.3)
    m = s.maps(sub=False)["dirichlet_mask"].astype(bool)
    x, y = splitmix_vector(s.N, 1), splitmix_vector(s.N, 2)
    x[m] = 0
    y[m] = 0
    ax, ay = s.apply_A(x), s.apply_A(y)
    assert abs(x @ ay - y @ ax) <= 1e-12 * abs(x @ ay)
    assert x @ ax > 0
    u = splitmix_vector(s.N, 3)
    assert np.array_equal(s.apply_A(u)[m], u[m])


# --- (b) the compiled reference ---------------------------------------------
CASES = [
    dict(k=8, order=4),
    dict(k=4, order=3, coarse_solve="amg"),
    dict(k=8, order=3, coarse_solve="amg"),
    dict(k=3, order=5, family="distorted_elements", c=0.7, kappa=2.5),
    dict(k=2, order=2, refine=1, family="distorted_domain"),
    dict(k=4, order=1),
    dict(k=2, order=7, precond="fine_only"),
    dict(k=3, order=2, boundary="neumann", c=1.0),
]


@needs_ref
@pytest.mark.parametrize("kw", CASES, ids=lambda kw: "-".join(f"{k}{v}" for k, v in kw.items()))
def test_oracle_matches_reference(kw):
    a, b = RefSystem(RefConfig(**kw)), orc(**kw)
    assert (a.N, a.NE, a.NV, a.coarse_amg, a.amg_levels) == (b.N, b.NE, b.NV, b.coarse_amg, b.amg_levels)
    ma, mb = a.maps(), b.maps()
    for key in ma:
        assert np.array_equal(ma[key], mb[key]), key
    assert np.array_equal(a.lumped_mass(), b.lumped_mass())
    u = splitmix_vector(a.N, 12345)
    assert np.array_equal(a.apply_A(u), b.apply_A(u))
    pa, pb = a.apply_P(u), b.apply_P(u)
    assert np.max(np.abs(pa - pb)) <= 1e-14 * np.max(np.abs(pa))
    if a.coarse_amg:
        for lvl in range(a.amg_levels):
            la, lb = a.amg_level(lvl), b.amg_level(lvl)
            for key in ("ptr", "col", "aggregate"):
                assert np.array_equal(la[key], lb[key])
            assert np.array_equal(la["val"], lb["val"])
    rhs = a.load_ones()
    # the all-Neumann c=1 case ends in a steep residual drop (9 orders in two
    # iterations) that amplifies 1e-15 differences in P to 1e-8 of r_0 at
    # 1e-8 (SURVEY §8c parity study); it is compared before the drop
    tol = 1e-4 if kw.get("boundary") == "neumann" else 1e-8
    ra, rb = a.pcg(rhs, tol=tol), b.pcg(rhs, tol=tol)
    assert ra["iterations"] == rb["iterations"] and ra["status"] == rb["status"]
    dr = np.max(np.abs(ra["residual_history"] - rb["residual_history"])) / ra["residual_history"][0]
    assert dr <= 1e-10
    assert np.linalg.norm(ra["u"] - rb["u"]) <= 1e-10 * np.linalg.norm(ra["u"])


@needs_ref
def test_gll_and_pencil_match_reference():
    for n in range(1, 11):
        ta, wa, Da, Ba = ref_gll(n)
        tb, wb, Db, Bb = oracle_gll(n)
        assert np.array_equal(ta, tb) and np.array_equal(wa, wb) and np.array_equal(Da, Db) and np.array_equal(Ba, Bb)
        Pa, Pb = ref_pencil(n), oracle_pencil(n)
        assert np.array_equal(Pa["K"], Pb["K"]) and np.array_equal(Pa["M"], Pb["M"])
        assert np.max(np.abs(Pa["lambda"] - Pb["lambda"])) <= 1e-13 * Pa["lambda"].max()
        # eigenvector signs may differ; the operator they represent may not
        Ra = Pa["V_inv"] @ np.diag(Pa["lambda"]) @ Pa["V"]
        Rb = Pb["V_inv"] @ np.diag(Pb["lambda"]) @ Pb["V"]
        assert np.max(np.abs(Ra - Rb)) <= 1e-12 * np.max(np.abs(Ra))


@needs_ref
def test_restrict_prolong_match_reference():
    kw = dict(k=4, order=4, family="distorted_elements")
    a, b = RefSystem(RefConfig(**kw)), orc(**kw)
    r = splitmix_vector(a.N, 9)
    assert np.array_equal(a.restrict(r), b.restrict(r))
    Z = splitmix_vector(a.NV, 10)
    assert np.array_equal(a.prolongate(Z), b.prolongate(Z))
    assert np.array_equal(a.element_h(), b.element_h())


# --- on-the-fly operator variant (operator.cpp:174-253) ------------------------
@pytest.mark.parametrize("family", ["distorted_domain", "distorted_elements"])
def test_oracle_otf_agrees_with_stored(family):
    """test_operator.cpp:103-121: stored and on-the-fly agree to 1e-12."""
    kw = dict(k=2, order=3, family=family, kappa=2.5, c=0.7, precond="none")
    a, b = orc(**kw), orc(variant="on_the_fly", **kw)
    u = splitmix_vector(a.N, 42)
    ra, rb = a.apply_A(u), b.apply_A(u)
    assert np.linalg.norm(ra - rb) <= 1e-12 * np.linalg.norm(ra)


@needs_ref
@pytest.mark.parametrize("order", [1, 3, 6])
def test_oracle_otf_matches_reference(order):
    """The restated on-the-fly geometry is the reference's, bit for bit."""
    kw = dict(k=3, order=order, family="distorted_elements", kappa=1.5, c=0.3, precond="none",
              variant="on_the_fly")
    u = splitmix_vector(orc(**kw).N, 3)
    assert np.array_equal(orc(**kw).apply_A(u), RefSystem(RefConfig(**kw)).apply_A(u))
