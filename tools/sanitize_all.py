"""Workload for compute-sanitizer (memcheck / racecheck / synccheck) over the
whole solver path on small meshes: the Ax tile and low-order kernels (stored
and on-the-fly), the FDM, the restriction pass, the AMG and nested-dissection
coarse solves, the combine, the PCG vector kernels, the bitwise-reference
mode and a 2-slab multi-GPU plan. Run on the GPU box:
    compute-sanitizer --tool memcheck python tools/sanitize_all.py"""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_1506_05996_b200 as hx  # noqa: E402

cases = [
    dict(k=5, order=7),                                   # tile Ax, FDM, direct coarse (dense inverse, m < 1500)
    dict(k=16, order=3),                                  # direct coarse through the nested-dissection factor
    dict(k=12, order=3, coarse_solve="amg"),              # AMG K-cycles
    dict(k=6, order=2, variant="on_the_fly"),             # low-order kernel, on-the-fly geometry
    dict(k=4, order=5, family="distorted_elements", bitwise_reference=True),
    dict(k=12, order=7),                                  # TMA-staged combine over many full tiles, gather order
    dict(k=9, order=2, coarse_solve="amg"),               # 256-node combine tiles
    dict(k=10, order=4, coarse_sms=16),                   # coarse solve on a green-context SM partition
]
for c in cases:
    c = dict(c)
    fam = c.pop("family", "uniform")
    mesh = hx.generate_cube_mesh(c.pop("k"), fam)
    order = c.pop("order")
    with hx.Plan(mesh, order, **c) as p:
        u = hx.synthetic_vector(p.N, 3)
        p.apply_A(u)
        p.apply_P(u)
        res = p.pcg(None, tol=1e-8)
        print(f"{fam} n={order} {c}: N={p.N} iterations={res['iterations']}", flush=True)
with hx.Plan(hx.generate_cube_mesh(6), 3, devices=[0, 0]) as g:
    res = g.pcg(None, tol=1e-8)
    print(f"2-slab plan: iterations={res['iterations']}", flush=True)
print("done")
