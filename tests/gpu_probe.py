"""Scratch probe run on the GPU box: correctness + timing summary (not a test)."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1506_05996_b200 as hx
from oracle import RefConfig, RefSystem, splitmix_vector

out = {}
k = int(sys.argv[1]) if len(sys.argv) > 1 else 52
n = int(sys.argv[2]) if len(sys.argv) > 2 else 7
t0 = time.time()
mesh = hx.generate_cube_mesh(k)
plan = hx.Plan(mesh, n)
out["setup_s"] = time.time() - t0
out["N"] = plan.N
out["amg"] = [plan.amg_rows, plan.amg_nnz]
u = splitmix_vector(plan.N, 12345)
r = plan.apply_A(u)
out["ax_checksum"] = float(r.sum())
out["profile_ms"] = plan.profile(10)
ms, ms_elem = plan.bench_apply_A(20)
words = hx.residual_words_model(plan.NE, n)
out["ax_ms"] = ms
out["ax_elem_ms"] = ms_elem
out["ax_gdofs"] = plan.N / (ms * 1e-3) / 1e9
out["ax_frac"] = words * 8 / (ms * 1e-3) / 6547.5e9
t0 = time.time()
res = plan.pcg(None, tol=1e-8, max_iterations=200, want_u=True)
out["pcg_wall_s"] = time.time() - t0
out["pcg"] = {k2: v for k2, v in res.items() if k2 not in ("u", "residual_history", "zr_history")}
out["r0"] = float(res["residual_history"][0])
out["rlast"] = float(res["residual_history"][-1])
out["unorm"] = float(np.linalg.norm(res["u"]))
print(json.dumps(out, indent=1))
