"""The reference-side binding of INTEGRATION.md, compiled and run: the
unmodified reference (oracle/_ref objects) with
integration/hexsem_b200_adapter.hpp and libhexsem_b200.so. The reference's
own pcg (krylov.cpp:20-71) drives the B200 operator and preconditioner
(plug-in level), and b200_pcg replaces pcg (solve level); both must match
the all-reference solve."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEMO = os.path.join(ROOT, "oracle", "_ref", "integration_demo")


def test_adapter_header_compiles_against_reference():
    if not os.path.exists(DEMO):
        pytest.skip("oracle/_ref/integration_demo not built (needs /root/reference at build time)")
    assert os.access(DEMO, os.X_OK)


@pytest.mark.gpu
@pytest.mark.parametrize("k,order,family,precond", [(8, 4, 0, 0), (4, 5, 2, 0), (6, 3, 1, 1), (5, 2, 0, 3)])
def test_reference_pcg_with_b200_operators(k, order, family, precond):
    if not os.path.exists(DEMO):
        pytest.skip("oracle/_ref/integration_demo not built")
    out = subprocess.run([DEMO, str(k), str(order), str(family), str(precond)], capture_output=True, text=True,
                         timeout=600)
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert "error" not in res, res
    assert res["plug_status"] == res["ref_status"] == res["solve_status"] == 0
    assert abs(res["plug_iterations"] - res["ref_iterations"]) <= 1
    assert abs(res["solve_iterations"] - res["ref_iterations"]) <= 1
    tol = 1e-10 if family == 0 else 1e-8  # distorted meshes amplify rounding (helpers.reference_noise)
    assert res["plug_max_dr_over_r0"] <= tol and res["solve_max_dr_over_r0"] <= tol, res
    assert res["plug_u_rel"] <= 1e-8 and res["solve_u_rel"] <= 1e-8, res


@pytest.mark.gpu
@pytest.mark.parametrize("k,order,family,precond,mode", [(8, 4, 0, 0, "0,0"), (6, 3, 1, 0, "0,0,0"), (5, 3, 0, 0, "0,0"),
                                                        (5, 3, 0, 3, "0,0")])
def test_reference_pcg_with_multi_gpu_plan(k, order, family, precond, mode):
    """The adapter's multi-GPU plan (hxb_options.n_gpus, element slabs, the
    in-library distributed PCG): here the slabs share device 0, so the
    messages are device copies; with distinct devices they go over NCCL."""
    if not os.path.exists(DEMO):
        pytest.skip("oracle/_ref/integration_demo not built")
    out = subprocess.run([DEMO, str(k), str(order), str(family), str(precond), mode], capture_output=True, text=True,
                         timeout=600)
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert "error" not in res, res
    assert res["n_gpus"] == len(mode.split(","))
    assert res["plug_status"] == res["ref_status"] == res["solve_status"] == 0
    assert abs(res["plug_iterations"] - res["ref_iterations"]) <= 1
    assert abs(res["solve_iterations"] - res["ref_iterations"]) <= 1
    # unpreconditioned CG (precond 3) amplifies the FMA rounding of Ax over its
    # 47 iterations (the bitwise plan, test below, shows the arithmetic is the
    # reference's): 1e-8 there
    tol = 1e-10 if family == 0 and precond != 3 else 1e-8
    assert res["plug_max_dr_over_r0"] <= tol and res["solve_max_dr_over_r0"] <= tol, res
    assert res["plug_u_rel"] <= 1e-8 and res["solve_u_rel"] <= 1e-8, res


@pytest.mark.gpu
@pytest.mark.parametrize("k,order,family,precond", [(8, 4, 0, 0), (4, 5, 2, 0), (6, 3, 1, 1), (5, 3, 0, 3)])
def test_reference_pcg_with_bitwise_plan(k, order, family, precond):
    """Through the same adapter, the bitwise-reference plan reproduces the
    reference's own solve exactly: zero residual-history and u differences,
    both when the reference's pcg drives the B200 operators and for b200_pcg."""
    if not os.path.exists(DEMO):
        pytest.skip("oracle/_ref/integration_demo not built")
    out = subprocess.run([DEMO, str(k), str(order), str(family), str(precond), "bitwise"], capture_output=True,
                         text=True, timeout=600)
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert "error" not in res, res
    assert res["plug_iterations"] == res["ref_iterations"] == res["solve_iterations"]
    assert res["plug_max_dr_over_r0"] == 0 and res["solve_max_dr_over_r0"] == 0, res
    assert res["plug_u_rel"] == 0 and res["solve_u_rel"] == 0, res
