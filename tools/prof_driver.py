"""Profiling driver (run under ncu on the GPU box): one plan, a few Ax and
P applications and a short PCG. Not a bench — numbers printed here are
never reported."""
import sys

sys.path.insert(0, ".")
import paper_1506_05996_b200 as hx
splitmix_vector = hx.synthetic_vector

k = int(sys.argv[1]) if len(sys.argv) > 1 else 30
n = int(sys.argv[2]) if len(sys.argv) > 2 else 7
variant = sys.argv[3] if len(sys.argv) > 3 else "stored"
plan = hx.Plan(hx.generate_cube_mesh(k), n, variant=variant)
u = splitmix_vector(plan.N, 12345)
import torch  # noqa: E402  (device buffers: full-mesh Ax launches, not the host API's 8 chunks)

du = torch.from_numpy(u).cuda()
dr = torch.empty_like(du)
for _ in range(4):
    plan.apply_A_device(du.data_ptr(), dr.data_ptr(), torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
plan.apply_P(u)
plan.pcg(None, tol=1e-8, max_iterations=3, want_u=False)
