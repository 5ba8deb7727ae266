"""A/B Ax timing for library builds (HXB_LIB) at cfg4 sizes: python tools/ab_ax.py n [n ...]"""
import json, os, sys
sys.path.insert(0, ".")
import torch
import paper_1506_05996_b200 as hx
from oracle import splitmix_vector

PEAK = 6451.8
for n in [int(x) for x in sys.argv[1:]]:
    k = round((20e6 ** (1 / 3) - 1) / n)
    plan = hx.Plan(hx.generate_cube_mesh(k), n, precond="none")
    u = torch.from_numpy(splitmix_vector(plan.N, 12345)).cuda()
    r = torch.empty_like(u)
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(3):
        plan.apply_A_device(u.data_ptr(), r.data_ptr(), s)
    plan.kernel_timing(True, 200)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(20):
        plan.apply_A_device(u.data_ptr(), r.data_ptr(), s)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    em, en = plan.kernel_time("ax_elem")
    np1 = n + 1
    b = 8 * plan.NE * (10 * np1 ** 3 + np1 ** 2 + 2)
    print(json.dumps({"lib": os.environ.get("HXB_LIB", "default"), "order": n, "ax_ms": round(ms, 4),
                      "gdofs": round(plan.N / ms / 1e6, 2), "elem_ms": round(em / en, 4),
                      "elem_frac": round(b / (em / en * 1e-3) / 1e9 / PEAK, 3), "sum": float(r.sum())}), flush=True)
    plan.close()
