#!/bin/bash
# A/B: component profile + PCG at cfg2 for each library build given (HXB_LIB)
mkdir -p gpurun_out
for L in "$@"; do
  HXB_LIB=$L timeout 300 python - <<'PY' >> gpurun_out/ab.log 2>&1
import os, sys, json
sys.path.insert(0, ".")
import paper_1506_05996_b200 as hx
p = hx.Plan(hx.generate_cube_mesh(52), 7)
prof = p.profile(10)
for _ in range(2):
    r = p.pcg(None, tol=1e-8, want_u=False)
print(os.environ["HXB_LIB"], json.dumps({k: round(v, 4) for k, v in prof.items() if k in ("fdm", "combine", "precond", "ax_elem")}),
      "pcg", r["iterations"], round(r["solve_seconds"], 4))
PY
done
