"""Profiling driver for the nested-dissection direct coarse solve (cfg4 n=10:
27^3 elements, 21,952 coarse unknowns): a few preconditioner applications."""
import sys

sys.path.insert(0, ".")
import paper_1506_05996_b200 as hx

k = int(sys.argv[1]) if len(sys.argv) > 1 else 27
n = int(sys.argv[2]) if len(sys.argv) > 2 else 10
plan = hx.Plan(hx.generate_cube_mesh(k), n, precond="coarse_only")
r = hx.synthetic_vector(plan.N, 3)
for _ in range(3):
    plan.apply_P(r)
