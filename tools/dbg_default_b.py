import sys; sys.path.insert(0,'.')
import numpy as np
import paper_1506_05996_b200 as hx
a = hx.solve_poisson(k=2, family="distorted_elements", order=2)
print("a iterations", a["report"]["iterations"], a["report"]["residual_history"][:3], a["report"].get("diagnostic"))
m = hx.generate_cube_mesh(2, "distorted_elements")
p = hx.Plan(m, 2)
print("N", p.N, "load_ones sum", p.load_ones().sum())
r = p.pcg(None, 1e-6, 500); print("pcg None iterations", r["iterations"], r["residual_history"][:3])
r = p.pcg(p.load_ones(), 1e-6, 500); print("pcg b iterations", r["iterations"], r["residual_history"][:3])
p2 = hx.Plan(m, 2, coarse_solve="amg")
r = p2.pcg(None, 1e-6, 500); print("amg pcg None iterations", r["iterations"])
for k in (3,4):
    p = hx.Plan(hx.generate_cube_mesh(k), 2); r = p.pcg(None, 1e-6, 500); print(k, "pcg None iterations", r["iterations"])
