"""cfg4 (BASELINE.json configs[3]): polynomial-order sweep N=1..10 at ~20M DOF.
Ax-only throughput vs the HBM roofline for every order, and the two-scale PCG
solve to 1e-8 for the orders whose host setup is quick. Run on the GPU box:
    python tools/order_sweep.py > gpurun_out/order_sweep.json
"""
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_1506_05996_b200 as hx
from oracle import splitmix_vector

PEAK = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if __import__("os").path.exists("MEASURED_PEAKS.json") else 6650.0
orders = [int(x) for x in sys.argv[1:]] or list(range(1, 11))
rows = []
for n in orders:
    k = round((20e6 ** (1 / 3) - 1) / n)  # SURVEY §8d cfg4 sizes
    t0 = time.time()
    mesh = hx.generate_cube_mesh(k)
    plan = hx.Plan(mesh, n, precond="none")
    setup = time.time() - t0
    u = torch.from_numpy(splitmix_vector(plan.N, 12345)).cuda()
    r = torch.empty_like(u)
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(3):
        plan.apply_A_device(u.data_ptr(), r.data_ptr(), s)
    plan.kernel_timing(True, 200)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    reps = 20
    for _ in range(reps):
        plan.apply_A_device(u.data_ptr(), r.data_ptr(), s)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    em, ec = plan.kernel_time("ax_elem")
    np1 = n + 1
    bytes_ax = 8 * plan.NE * (10 * np1 ** 3 + np1 ** 2 + 2)
    row = {"order": n, "k": k, "N": plan.N, "NE": plan.NE, "setup_s": round(setup, 2), "ax_ms": ms,
           "ax_gdofs": plan.N / ms / 1e6, "ax_elem_ms": em / max(1, ec),
           "elem_frac_of_hbm": bytes_ax / (em / max(1, ec) * 1e-3) / 1e9 / PEAK,
           "whole_ax_frac_of_hbm": bytes_ax / (ms * 1e-3) / 1e9 / PEAK}
    plan.close()
    del u, r
    torch.cuda.empty_cache()
    if n >= 3:  # two-scale PCG to 1e-8 (host AMG setup grows quickly at low order)
        t0 = time.time()
        with hx.Plan(mesh, n) as p2:
            row["pcg_setup_s"] = round(time.time() - t0, 2)
            res = p2.pcg(None, tol=1e-8, max_iterations=500, want_u=False)
            res = p2.pcg(None, tol=1e-8, max_iterations=500, want_u=False)
            row.update({"pcg_iterations": res["iterations"], "pcg_solve_s": res["solve_seconds"],
                        "pcg_ms_per_iteration": 1e3 * res["solve_seconds"] / max(1, res["iterations"])})
    rows.append(row)
    print(json.dumps(row), flush=True)
