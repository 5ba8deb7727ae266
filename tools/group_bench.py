"""In-library multi-GPU plan (hxb_options.n_gpus) on the devices given, cfg2
by default: the distributed PCG's time and iteration count next to the single
plan's. With every slab on one device this measures the protocol's overhead
(device-copy transport), not scaling.
    python tools/group_bench.py 52 7 0,0"""
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_1506_05996_b200 as hx  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 52
n = int(sys.argv[2]) if len(sys.argv) > 2 else 7
devices = [int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "0,0").split(",")]
mesh = hx.generate_cube_mesh(k)
one = hx.Plan(mesh, n)
one.pcg(None, tol=1e-8)
r1 = one.pcg(None, tol=1e-8)
one.close()
t = time.time()
grp = hx.Plan(mesh, n, devices=devices)
setup = time.time() - t
grp.pcg(None, tol=1e-8)
t = time.time()
rg = grp.pcg(None, tol=1e-8)
wall = time.time() - t
m = min(len(r1["residual_history"]), len(rg["residual_history"]))
dr = float(np.max(np.abs(r1["residual_history"][:m] - rg["residual_history"][:m])) / r1["residual_history"][0])
print(json.dumps({"k": k, "order": n, "devices": devices, "N": grp.N, "setup_s": setup,
                  "single": {"iterations": r1["iterations"], "solve_s": r1["solve_seconds"]},
                  "group": {"iterations": rg["iterations"], "solve_s": rg["solve_seconds"], "wall_s": wall},
                  "max_dr_over_r0_vs_single": dr,
                  "u_rel_vs_single": float(np.linalg.norm(rg["u"] - r1["u"]) / np.linalg.norm(r1["u"]))}))
