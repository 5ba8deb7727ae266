"""Bitwise parity: plans built with ``bitwise_reference=True`` (compat.cu,
hxb_options.bitwise_reference) equal the reference (oracle/_ref, the
unmodified sources compiled by oracle/Makefile) BIT FOR BIT: Ax, the fine,
coarse and two-scale preconditioners, and the whole PCG run (status,
iterations, every residual, every z.r and the solution vector).

This is the proof behind the tolerance-based parity of the fast path
(test_gpu_parity.py): the fast kernels differ from these only by FMA
contraction and summation order, and the compatible mode shows that every
other arithmetic step (numbering, geometry, pencil, coarse matrix, AMG
hierarchy, envelope Cholesky, operator/preconditioner/Krylov recurrences) is
the reference's own, including on the problems whose rounding floor exceeds
1e-10 of r0 (tiny high-order meshes, distorted geometry)."""
import json
import os

import numpy as np
import pytest

import paper_1506_05996_b200 as hx
from oracle import RefConfig, RefSystem, ref_available, splitmix_vector

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not ref_available(), reason="oracle/_ref (compiled reference) not built")]
HERE = os.path.dirname(os.path.abspath(__file__))


def _pair(k=8, order=4, family="uniform", precond="two_scale", coarse_solve="automatic", kappa=1.0, c=0.0,
          boundary="dirichlet", variant="stored", refine=0):
    ref = RefSystem(RefConfig(k=k, order=order, family=family, refine=refine, precond=precond,
                              coarse_solve=coarse_solve, kappa=kappa, c=c, boundary=boundary, variant=variant))
    mesh = hx.generate_cube_mesh(k, family, boundary)
    for _ in range(refine):
        mesh = hx.refine_uniform(mesh)
    ne = mesh.num_elements
    plan = hx.Plan(mesh, order, np.full(ne, kappa), np.full(ne, c), precond=precond, coarse_solve=coarse_solve,
                   variant=variant, bitwise_reference=True)
    return ref, plan


def assert_bitwise(a, b, what=""):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape, (what, a.shape, b.shape)
    if not np.array_equal(a, b):
        bad = np.flatnonzero(a != b)
        raise AssertionError(f"{what}: {bad.size} of {a.size} entries differ; first at {bad[0]}: "
                             f"{a.flat[bad[0]]!r} vs {b.flat[bad[0]]!r}, max |d| {np.max(np.abs(a - b)):.3e}")


def assert_pcg_bitwise(ours, theirs, what=""):
    assert ours["status"] == theirs["status"], (what, ours["status"], theirs["status"])
    assert ours["iterations"] == theirs["iterations"], (what, ours["iterations"], theirs["iterations"])
    assert_bitwise(ours["residual_history"], theirs["residual_history"], what + " residual_history")
    assert_bitwise(ours["zr_history"], theirs["zr_history"], what + " zr_history")
    assert_bitwise(ours["u"], theirs["u"], what + " u")


@pytest.mark.parametrize("order", list(range(1, 11)))
def test_ax_bitwise_all_orders(order):
    """SemOperator::apply, stored variant, distorted elements, kappa and c != 0."""
    k = 3 if order <= 6 else 2
    ref, plan = _pair(k=k, order=order, family="distorted_elements", kappa=2.5, c=0.7, precond="none")
    u = splitmix_vector(plan.N, 12345)
    assert_bitwise(plan.apply_A(u), ref.apply_A(u), f"Ax n={order}")


@pytest.mark.parametrize("order", [1, 3, 5, 8])
def test_ax_on_the_fly_bitwise(order):
    """otf_element_kernel (operator.cpp:174-253): geometry per node from the corners."""
    ref, plan = _pair(k=3, order=order, family="distorted_domain", kappa=1.7, c=0.3, precond="none",
                      variant="on_the_fly")
    u = splitmix_vector(plan.N, 99)
    assert_bitwise(plan.apply_A(u), ref.apply_A(u), f"OTF Ax n={order}")


@pytest.mark.parametrize("k,order,coarse", [(8, 4, "automatic"), (12, 3, "amg"), (4, 6, "direct"),
                                            (6, 5, "amg")])
def test_preconditioner_bitwise(k, order, coarse):
    """FinePreconditioner::apply, CoarsePreconditioner::apply (envelope LLT or
    the AMG K-cycles) and TwoScalePreconditioner::apply on an unmasked r."""
    ref, plan = _pair(k=k, order=order, family="distorted_elements" if k <= 8 else "uniform", coarse_solve=coarse)
    assert plan.coarse_amg == (coarse == "amg")
    r = splitmix_vector(plan.N, 5)
    assert_bitwise(plan.apply_fine(r), ref.apply_fine(r), "fine")
    assert_bitwise(plan.apply_coarse(r), ref.apply_coarse(r), "coarse")
    assert_bitwise(plan.apply_P(r), ref.apply_P(r), "two-scale P")


PCG_CASES = [
    # cfg1 = BASELINE configs[0] (8^3, N=4), every preconditioner mode
    dict(k=8, order=4, precond="two_scale"),
    dict(k=8, order=4, precond="fine_only"),
    dict(k=8, order=4, precond="coarse_only"),
    dict(k=8, order=4, precond="none"),
    # k = 4..8 meshes across orders and families
    dict(k=4, order=7, family="distorted_domain"),
    dict(k=5, order=5, family="distorted_elements", kappa=2.0, c=0.5),
    dict(k=6, order=4, family="uniform", boundary="neumann", c=1.0),
    dict(k=7, order=3, family="distorted_elements"),
    # the AMG coarse path (K-cycles, envelope LLT on the coarsest level)
    dict(k=12, order=3, coarse_solve="amg"),
    dict(k=8, order=5, family="distorted_domain", coarse_solve="amg"),
    # the ill-conditioned tiny high-order meshes (rounding floor up to 2.7e-8 r0)
    dict(k=2, order=8),
    dict(k=2, order=9),
    dict(k=2, order=10),
    # on-the-fly operator variant
    dict(k=6, order=5, family="distorted_elements", variant="on_the_fly"),
    dict(k=6, order=5, family="uniform", variant="on_the_fly"),
    # the distributed-PCG problems of test_gpu_parity.py
    dict(k=6, order=3, family="distorted_elements"),
    dict(k=8, order=5, family="distorted_domain"),
]
# the order sweep of test_gpu_parity.py::test_order_sweep_pcg (cfg4 shape, small)
SWEEP_K = {1: 8, 2: 6, 3: 5, 4: 4, 5: 3, 6: 3, 7: 3, 8: 2, 9: 2, 10: 2}
PCG_CASES += [dict(k=SWEEP_K[n], order=n) for n in range(1, 8)]


@pytest.mark.parametrize("case", PCG_CASES, ids=lambda c: "-".join(f"{k}{v}" for k, v in c.items()))
def test_pcg_bitwise(case):
    """pcg (krylov.cpp:20-71) with the two-scale Schwarz preconditioner: every
    recorded residual and z.r, the iteration count and u equal the reference's."""
    ref, plan = _pair(**case)
    b = ref.load_ones()
    ours, theirs = plan.pcg(b, tol=1e-8), ref.pcg(b, tol=1e-8)
    assert_pcg_bitwise(ours, theirs, str(case))
    # and the Poisson load assembled by the plan (b = None) is the reference's
    assert_bitwise(plan.load_ones(), b, "load")


def _cfg3_mesh(k=4, refine=1):
    mesh = hx.generate_cube_mesh(k, "distorted_elements")
    for _ in range(refine):
        mesh = hx.refine_uniform(mesh)
    mesh.bf_tag = np.where(mesh.bf_face <= 1, 0, 1).astype(np.uint8)
    cent = mesh.xyz[mesh.conn].mean(axis=1)
    kappa = 1 + 0.5 * np.sin(2 * np.pi * cent[:, 0]) * np.cos(2 * np.pi * cent[:, 1])
    c = 0.1 + cent[:, 2]
    return mesh, kappa, c


@pytest.mark.parametrize("coarse_solve", ["automatic", "amg"])
def test_cfg3_bitwise(coarse_solve):
    """cfg3 proxy (BASELINE configs[2]): refined distorted mesh, kappa(x), c(x),
    x-faces Dirichlet and the rest Neumann, N=5."""
    mesh, kappa, c = _cfg3_mesh()
    order = 5
    ref = RefSystem(RefConfig(order=order, coarse_solve=coarse_solve), mesh=mesh.as_dict(), order=order,
                    kappa_e=kappa, c_e=c)
    with hx.Plan(mesh, order, kappa, c, coarse_solve=coarse_solve, bitwise_reference=True) as plan:
        u = splitmix_vector(plan.N, 4)
        assert_bitwise(plan.apply_A(u), ref.apply_A(u), "Ax")
        assert_bitwise(plan.apply_P(u), ref.apply_P(u), "P")
        b = ref.load_ones()
        assert_pcg_bitwise(plan.pcg(b, tol=1e-8), ref.pcg(b, tol=1e-8), f"cfg3 {coarse_solve}")


def test_cfg2_bitwise_against_golden():
    """cfg2 (52^3, N=7, 48.6M DOF, AMG coarse path): the bitwise-reference plan
    reproduces the reference's committed run (tests/golden/cfg2_pcg.json) bit
    for bit: all 47 residuals, all 46 z.r values, the solution digest."""
    gold = json.load(open(os.path.join(HERE, "golden", "cfg2_pcg.json")))
    mesh = hx.generate_cube_mesh(52)
    with hx.Plan(mesh, 7, bitwise_reference=True) as plan:
        u = hx.synthetic_vector(plan.N, 12345)
        r = plan.apply_A(u)
        if "ax_digest_seed12345" in gold:
            d = gold["ax_digest_seed12345"]
            s = d["stride"]
            assert_bitwise(r[::s][:len(d["sample"])], np.array(d["sample"]), "cfg2 Ax sample")
        # (numpy's norm itself rounds differently on different host CPUs: 1e-14)
        assert abs(np.linalg.norm(r) - gold["ax_norm_seed12345"]) <= 1e-14 * gold["ax_norm_seed12345"]
        res = plan.pcg(None, tol=1e-8, max_iterations=500)
    assert res["iterations"] == gold["iterations"]
    assert_bitwise(res["residual_history"], np.array(gold["residual_history"]), "cfg2 residual_history")
    assert_bitwise(res["zr_history"], np.array(gold["zr_history"]), "cfg2 zr_history")
    d = gold["u_digest"]
    assert_bitwise(res["u"][::d["stride"]][:len(d["sample"])], np.array(d["sample"]), "cfg2 u sample")
    nb = res["u"].size
    blk = np.array([np.linalg.norm(res["u"][b * nb // 64:(b + 1) * nb // 64]) for b in range(64)])
    assert np.max(np.abs(blk - np.array(d["block_norms"])) / np.array(d["block_norms"])) <= 1e-14
    assert abs(np.linalg.norm(res["u"]) - gold["u_norm2"]) <= 1e-14 * gold["u_norm2"]
