"""cfg3 (BASELINE configs[2]) at scale on one B200: distorted_elements 8^3
refined R times (R=3: 64^3 hexes), N=5, per-element kappa(x), c(x) at the
centroid, x-faces Dirichlet / others Neumann. Ax throughput and two-scale PCG
to 1e-8 with b = lumped-mass load. The reference CPU timing on the 8^3 proxy
(oracle/_ref) is printed alongside when available locally.
    python tools/cfg3_bench.py [R] > gpurun_out/cfg3.json"""
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_1506_05996_b200 as hx
from oracle import splitmix_vector

R = int(sys.argv[1]) if len(sys.argv) > 1 else 3
order = 5
mesh = hx.generate_cube_mesh(8, "distorted_elements")
for _ in range(R):
    mesh = hx.refine_uniform(mesh)
mesh.bf_tag = np.where(mesh.bf_face <= 1, 0, 1).astype(np.uint8)
cent = mesh.xyz[mesh.conn].mean(axis=1)
kappa = 1 + 0.5 * np.sin(2 * np.pi * cent[:, 0]) * np.cos(2 * np.pi * cent[:, 1])
c = 0.1 + cent[:, 2]
out = {"workload": f"cfg3: distorted_elements 8^3 refined {R}x ({mesh.num_elements} hexes), N={order}, "
                   "kappa=1+0.5 sin2pi x cos2pi y, c=0.1+z per element, x-faces Dirichlet, others Neumann"}
t = time.time()
plan = hx.Plan(mesh, order, kappa, c)
out["setup_s"] = time.time() - t
out["N"] = plan.N
u = torch.from_numpy(splitmix_vector(plan.N, 12345)).cuda()
r = torch.empty_like(u)
s = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    plan.apply_A_device(u.data_ptr(), r.data_ptr(), s)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
for _ in range(20):
    plan.apply_A_device(u.data_ptr(), r.data_ptr(), s)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
out["ax_ms"] = ms
out["ax_gdofs"] = plan.N / ms / 1e6
b = plan.load_ones()
plan.pcg(b, tol=1e-8, want_u=False)
res = plan.pcg(b, tol=1e-8, want_u=False)
out.update({"pcg_iterations": res["iterations"], "pcg_status": res["status"], "pcg_solve_s": res["solve_seconds"],
            "pcg_ms_per_iteration": res["solve_seconds"] * 1e3 / max(1, res["iterations"]),
            "coarse": "amg" if plan.coarse_amg else "direct"})
print(json.dumps(out))
