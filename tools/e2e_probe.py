"""Time hxb_apply_A with pinned host buffers at cfg2 (transfer-schedule A/B)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1506_05996_b200 as hx
from oracle import splitmix_vector
import os
p = hx.Plan(hx.generate_cube_mesh(52), 7, precond=os.environ.get("PRECOND", "two_scale"))
u = torch.from_numpy(splitmix_vector(p.N, 12345)).pin_memory()
r = torch.empty(p.N, dtype=torch.float64).pin_memory()
for _ in range(3):
    p.apply_A_host_ptr(u.data_ptr(), r.data_ptr())
t = time.perf_counter()
for _ in range(10):
    p.apply_A_host_ptr(u.data_ptr(), r.data_ptr())
dt = (time.perf_counter() - t) / 10
print(f"apply_A host {dt*1e3:.2f} ms  {p.N/dt/1e9:.2f} GDOF/s  checksum {float(r.sum()):.12e}")
