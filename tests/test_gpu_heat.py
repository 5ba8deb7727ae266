"""Backward-Euler heat driver (solve_heat, problem.cpp:145-255)
on the device plan, against the reference's own solve_heat (oracle/_ref) and
the reference acceptance criteria 8a-8c (acceptance_main.cpp:305-363,
test_output.txt:36-38)."""
import numpy as np
import pytest

import paper_1506_05996_b200 as hx
from helpers import rel
from oracle import RefConfig, ref_solve_heat

pytestmark = pytest.mark.gpu

BAR = dict(bar=(4, 4, 16), bar_size=(0.5, 0.5, 2.0), order=2, boundary="neumann", kappa=1e-2)


def _ours(tol, **heat):
    return hx.solve_heat(**{**BAR, "tol": tol, **heat})


@pytest.mark.parametrize("coarse", ["automatic"])
def test_heat_matches_reference(coarse):
    heat = dict(dt=0.04, steps=10, source_radius=0.4, has_source=True)
    ours = _ours(1e-12, **heat)
    theirs = ref_solve_heat(RefConfig(**BAR), heat, tol=1e-12)
    assert ours["all_converged"] and theirs["all_converged"]
    assert len(ours["steps"]) == len(theirs["steps"]) == 10
    for a, b in zip(ours["steps"], theirs["steps"]):
        assert abs(a["iterations"] - b["iterations"]) <= 1, (a, b)
        assert a["source_integral"] == pytest.approx(b["source_integral"], rel=1e-12)
        assert a["mean_temperature"] == pytest.approx(b["mean_temperature"], rel=1e-10)
        assert a["l2_norm"] == pytest.approx(b["l2_norm"], rel=1e-10)
    assert rel(ours["final_field"], theirs["final_field"]) <= 1e-10


def test_heat_constant_preserved():
    """Acceptance 8a: no source, u0 = 5, Neumann walls: u stays 5 (< 1e-10)."""
    out = _ours(1e-6, dt=0.04, steps=10, has_source=False, initial_value=5.0)
    assert out["all_converged"]
    assert np.max(np.abs(out["final_field"] - 5.0)) < 1e-10


def test_heat_mean_balance():
    """Acceptance 8b: mean temperature grows by dt * source integral / volume (< 1e-8)."""
    out = _ours(1e-12, dt=0.04, steps=10, has_source=True, source_radius=0.4)
    volume = 0.5 * 0.5 * 2.0
    prev, worst = 0.0, 0.0
    for s in out["steps"]:
        worst = max(worst, abs(s["mean_temperature"] - (prev + 0.04 * s["source_integral"] / volume)))
        prev = s["mean_temperature"]
    assert out["all_converged"] and worst < 1e-8, worst


def test_heat_70_step_run():
    """Acceptance 8c: 8x8x64 bar, n=2, 70 steps (kappa=1e-2, dt=0.04, Q=1000,
    rho=7000, cp=0.8): all converge, at most 25 iterations (test_output.txt:38)."""
    kw = dict(bar=(8, 8, 64), bar_size=(1.0, 1.0, 8.0), order=2, boundary="neumann", kappa=1e-2)
    out = hx.solve_heat(**kw, dt=0.04, steps=70, Q=1000.0, rho=7000.0, cp=0.8)
    its = [s["iterations"] for s in out["steps"]]
    print(f"heat 70 steps: max {max(its)} iterations, {out['solve_seconds']:.2f} s on the device")
    assert out["all_converged"] and len(its) == 70 and max(its) <= 25


def test_mms_convergence():
    """Acceptance 7 (acceptance_main.cpp:284-302): 4^3 cube, tol 1e-12, orders
    2..6; errors as recorded in test_output.txt:35 (2.94e-4 ... 6.57e-11)."""
    rep = hx.mms_convergence(2, 6, k=4, tol=1e-12, max_iterations=2000)
    errs = [r["error"] for r in rep["rows"]]
    for got, want in zip(errs, [2.94e-4, 8.03e-6, 1.66e-7, 3.41e-9, 6.57e-11]):
        assert got == pytest.approx(want, rel=0.005), (got, want)
    assert all(errs[i] * 10 <= errs[i - 1] for i in (1, 2, 3)) and errs[4] <= 1e-8
