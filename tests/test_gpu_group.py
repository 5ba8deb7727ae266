"""Multi-GPU plans inside the library (hxb_options.n_gpus / devices, SURVEY
§8e): the mesh is cut into element slabs, one per listed device, and
hxb_solve / hxb_apply_A / hxb_apply_P run the distributed protocol with one
host thread per GPU. Here every slab lives on device 0 (this box has one
B200), so the messages travel as device-to-device copies; with distinct
devices the same code calls NCCL. The single-plan result is the reference
point: Ax is bitwise equal (the interface sums continue across ranks in the
reference's (e, l) order), the PCG differs only in the dot products'
cross-rank reduction order."""
import numpy as np
import pytest

import paper_1506_05996_b200 as hx
from helpers import rel
from oracle import splitmix_vector

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("R,k,order,family", [(2, 6, 7, "uniform"), (3, 6, 4, "distorted_elements"),
                                              (4, 8, 3, "distorted_domain"), (2, 5, 3, "uniform"),
                                              (3, 5, 2, "uniform")])
def test_group_ax_bitwise_equals_single_plan(R, k, order, family):
    mesh = hx.generate_cube_mesh(k, family)
    single = hx.Plan(mesh, order, precond="none")
    group = hx.Plan(mesh, order, precond="none", devices=[0] * R)
    assert group.N == single.N and group.NE == single.NE
    u = splitmix_vector(single.N, 77)
    assert np.array_equal(group.apply_A(u), single.apply_A(u))


@pytest.mark.parametrize("R,k,order,family,coarse", [(2, 6, 4, "uniform", "automatic"),
                                                     (3, 6, 3, "distorted_elements", "automatic"),
                                                     (2, 8, 5, "distorted_domain", "amg"),
                                                     (4, 10, 3, "uniform", "amg")])
def test_group_pcg_matches_single_plan(R, k, order, family, coarse):
    mesh = hx.generate_cube_mesh(k, family)
    single = hx.Plan(mesh, order, coarse_solve=coarse)
    group = hx.Plan(mesh, order, coarse_solve=coarse, devices=[0] * R)
    r = splitmix_vector(single.N, 3)
    assert rel(group.apply_P(r), single.apply_P(r)) <= 1e-13
    one = single.pcg(None, tol=1e-8)
    many = group.pcg(None, tol=1e-8)
    assert many["status"] == one["status"] == "converged"
    assert abs(many["iterations"] - one["iterations"]) <= 1
    ra, rb = many["residual_history"], one["residual_history"]
    m = min(len(ra), len(rb))
    dr = float(np.max(np.abs(ra[:m] - rb[:m])) / rb[0])
    # only the dots' cross-rank reduction order differs from the single plan:
    # judged against this problem's own rounding floor (helpers.reference_noise)
    from helpers import reference_noise
    from oracle import RefConfig, RefSystem

    cfg = RefConfig(k=k, order=order, family=family, coarse_solve=coarse)
    ref = RefSystem(cfg)
    b = ref.load_ones()
    tol = max(1e-10, 2 * reference_noise(ref.pcg(b, tol=1e-8), b, cfg))
    print(f"R={R} k={k} n={order}: iterations {many['iterations']} vs {one['iterations']}, max|dr|/r0 {dr:.2e} "
          f"(tol {tol:.2e})")
    assert dr <= tol, dr
    assert len(many["zr_history"]) == many["iterations"]
    assert rel(many["u"], one["u"]) <= 1e-9


def test_group_precond_none_and_reuse():
    """precond none on a group plan (z = r, precond.cpp:30-33); the plan is
    reusable across solves and right-hand sides."""
    mesh = hx.generate_cube_mesh(5)
    single = hx.Plan(mesh, 3, precond="none")
    group = hx.Plan(mesh, 3, precond="none", devices=[0, 0])
    r = splitmix_vector(single.N, 9)
    assert np.array_equal(group.apply_P(r), r)
    assert np.array_equal(group.apply_A(r), single.apply_A(r))
    for seed in (1, 2):
        b = splitmix_vector(single.N, seed) * single.load_ones()
        one, many = single.pcg(b, tol=1e-8), group.pcg(b, tol=1e-8)
        assert many["iterations"] == one["iterations"]
        assert rel(many["u"], one["u"]) <= 1e-9


def test_group_rejects_device_entry_points():
    mesh = hx.generate_cube_mesh(4)
    group = hx.Plan(mesh, 3, devices=[0, 0])
    with pytest.raises(hx.HxbError):
        group.apply_fine(np.zeros(group.N))
    with pytest.raises(hx.HxbError):
        hx.Plan(mesh, 3, devices=[0, 0], bitwise_reference=True)
