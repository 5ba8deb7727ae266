#!/bin/bash
# quick GPU iteration: parity tests (minus cfg2 golden), component profile at cfg2, ncu of chosen kernels
# usage: tools/gpu_profile.sh "kernel_regex" [tag]
rx=${1:-"fdm_kernel|combine_prolong|restrict_warp"}; tag=${2:-it}
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not golden" > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_quick.log
timeout 300 python - > gpurun_out/profile.log 2>&1 <<'PY'
import sys, json
sys.path.insert(0, ".")
import paper_1506_05996_b200 as hx
p = hx.Plan(hx.generate_cube_mesh(52), 7)
print(json.dumps({k: round(v, 4) for k, v in p.profile(10).items()}))
for _ in range(2):
    r = p.pcg(None, tol=1e-8, want_u=False)
print("pcg", r["iterations"], r["solve_seconds"], r["residual_history"][-1])
PY
[ -n "$rx" ] && bash tools/ncu_kernels.sh $tag "$rx"
exit 0
