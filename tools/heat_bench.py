"""solve_heat (problem.cpp:145-255) 70-step run on the device plan: bar 8x8x64,
N=2 and N=7, backward Euler dt=0.04, moving source. Prints one JSON line per case."""
import json, sys, time
sys.path.insert(0, ".")
import paper_1506_05996_b200 as hx

for order in (2, 7):
    kw = dict(bar=(8, 8, 64), bar_size=(1.0, 1.0, 8.0), order=order, boundary="neumann", kappa=1e-2, tol=1e-8)
    t = time.time()
    out = hx.solve_heat(**kw)
    wall = time.time() - t
    its = [s["iterations"] for s in out["steps"]]
    print(json.dumps({"order": order, "N": out["N"], "steps": len(its), "all_converged": out["all_converged"],
                      "iterations_max": max(its), "iterations_total": sum(its),
                      "device_solve_s": out["solve_seconds"], "wall_s_incl_setup": wall}))
