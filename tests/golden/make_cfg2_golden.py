"""Generate the cfg2 golden fixture (52^3 hexes, N=7, two-scale PCG to 1e-8)
with the compiled reference (oracle/_ref). Run in the build container:
    python tests/golden/make_cfg2_golden.py
Writes tests/golden/cfg2_pcg.json (residual/zr histories, ||u||, Ax checksum,
and, for the solution-vector and Ax-vector checks, a strided sample of 4096
entries plus 64 contiguous block 2-norms of u and of r = A u)."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import RefConfig, RefSystem, splitmix_vector  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 52
n = int(sys.argv[2]) if len(sys.argv) > 2 else 7
t0 = time.time()
ref = RefSystem(RefConfig(k=k, order=n, precond="two_scale", concurrent_precond=True,
                          fine_threads=max(1, (os.cpu_count() or 2) - 1)))
setup_s = time.time() - t0
u = splitmix_vector(ref.N, 12345)
t0 = time.time()
r = ref.apply_A(u)
ax_s = time.time() - t0
b = ref.load_ones()
res = ref.pcg(b, tol=1e-8, max_iterations=500)
out = {
    "config": {"k": k, "order": n, "family": "uniform", "precond": "two_scale", "tol": 1e-8, "kappa": 1.0, "c": 0.0},
    "N": ref.N, "NE": ref.NE, "coarse_amg": bool(ref.coarse_amg),
    "ax_checksum_seed12345": float(r.sum()), "ax_norm_seed12345": float(np.linalg.norm(r)),
    "iterations": res["iterations"], "status": res["status"],
    "residual_history": [float(x) for x in res["residual_history"]],
    "zr_history": [float(x) for x in res["zr_history"]],
    "u_norm2": float(np.linalg.norm(res["u"])), "u_sum": float(res["u"].sum()),
    "u_max": float(res["u"].max()),
    "timing": {"setup_s": setup_s, "ax_s": ax_s, "solve_s": res["solve_seconds"]},
    "generator": "oracle/_ref (unmodified reference + Eigen shim), tests/golden/make_cfg2_golden.py",
}
def vector_digest(x):
    """4096 strided entries (index g = q * (N // 4096)) and the 2-norms of 64
    contiguous blocks [b*N//64, (b+1)*N//64)."""
    n = x.size
    stride = max(1, n // 4096)
    idx = np.arange(0, min(n, 4096 * stride), stride)[:4096]
    blocks = [float(np.linalg.norm(x[b * n // 64:(b + 1) * n // 64])) for b in range(64)]
    return {"stride": int(stride), "sample": [float(v) for v in x[idx]], "block_norms": blocks}


out["u_digest"] = vector_digest(res["u"])
out["ax_digest_seed12345"] = vector_digest(r)
name = "cfg2_pcg.json" if (k, n) == (52, 7) else f"pcg_k{k}_n{n}.json"
with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), name), "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps({kk: v for kk, v in out.items() if kk not in ("residual_history", "zr_history")}))
