"""Per-kernel live times inside a cfg2 PCG solve (plan kernel timing, CUDA events)."""
import json, sys
sys.path.insert(0, ".")
import paper_1506_05996_b200 as hx
import os
p = hx.Plan(hx.generate_cube_mesh(int(sys.argv[1]) if len(sys.argv) > 1 else 52), 7,
            split_combine=os.environ.get("SPLIT", "1") == "1")
p.pcg_device(None, tol=1e-8, want_u=False)
p.kernel_timing(True, 4000)
r = p.pcg_device(None, tol=1e-8, want_u=False)
out = {"split": os.environ.get("SPLIT", "1"), "cluster": os.environ.get("CLUSTER", "0"), "iterations": r["iterations"], "solve_ms": r["solve_seconds"] * 1e3}
for k in ("ax_elem", "ax_gather", "fdm", "combine", "coarse", "combine_fine"):
    ms, n = p.kernel_time(k)
    out[k] = {"total_ms": round(ms, 3), "n": n, "avg_ms": round(ms / max(n, 1), 4)}
p.kernel_timing(False)
print(json.dumps(out))
