"""cfg5 (BASELINE configs[4]) shape on ONE B200: 104^3 hexes at N=7 (387M DOF).
Plan setup, Ax throughput and the two-scale PCG to 1e-8. Guarded by the host
memory a cfg2 plan needs (scaled by the element ratio) against the box's RAM.
    python tools/cfg5_single.py > gpurun_out/cfg5.json"""
import json
import os
import resource
import sys
import time

sys.path.insert(0, ".")
import torch

import paper_1506_05996_b200 as hx
from oracle import splitmix_vector

k = int(sys.argv[1]) if len(sys.argv) > 1 else 104
out = {"k": k, "order": 7}
p2 = hx.Plan(hx.generate_cube_mesh(52), 7)
rss2 = resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6  # GB
p2.close()
del p2
mem_total = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES") / 1e9
est = rss2 * (k / 52) ** 3
out.update({"cfg2_peak_rss_gb": rss2, "est_peak_rss_gb": est, "host_ram_gb": mem_total})
if est > 0.75 * mem_total:
    out["skipped"] = "estimated host memory too large"
    print(json.dumps(out))
    raise SystemExit(0)
t = time.time()
mesh = hx.generate_cube_mesh(k)
plan = hx.Plan(mesh, 7)
out["setup_s"] = time.time() - t
out["N"] = plan.N
out["NE"] = plan.NE
out["device_gb"] = plan.device_bytes / 1e9 if hasattr(plan, "device_bytes") else None
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
bytes_ax = 8 * plan.NE * (10 * 512 + 64 + 2)
out["ax_whole_frac_of_hbm"] = bytes_ax / (ms * 1e-3) / 1e9 / 6451.8
del u, r
res = plan.pcg_device(None, tol=1e-8, want_u=False)
out["pcg_iterations"] = res["iterations"]
out["pcg_status"] = res["status"]
out["pcg_solve_s"] = res["solve_seconds"]
out["pcg_ms_per_iteration"] = res["solve_seconds"] * 1e3 / max(1, res["iterations"])
out["peak_rss_gb"] = resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6
out["gpu_mem_peak_gb"] = torch.cuda.max_memory_allocated() / 1e9
print(json.dumps(out))
