"""GPU diagnostic (not a test): Ax on the B200 vs the compiled reference
elementwise, over a ladder of mesh sizes; prints mismatch statistics."""
import sys, time, json
import numpy as np
sys.path.insert(0, ".")
import paper_1506_05996_b200 as hx
from oracle import RefSystem, RefConfig, splitmix_vector

cases = [(8, 7), (16, 7), (24, 7), (32, 3), (40, 4), (52, 7)]
if len(sys.argv) > 1:
    cases = [tuple(int(x) for x in c.split(",")) for c in sys.argv[1:]]
for k, n in cases:
    t = time.time()
    ref = RefSystem(RefConfig(k=k, order=n, precond="none"))
    plan = hx.Plan(hx.generate_cube_mesh(k), n, precond="none")
    u = splitmix_vector(ref.N, 12345)
    a = plan.apply_A(u)
    b = ref.apply_A(u)
    d = np.abs(a - b)
    bad = np.nonzero(d > 1e-12 * np.abs(b).max())[0]
    out = {"k": k, "n": n, "N": ref.N, "max_abs": float(d.max()), "rel_norm": float(np.linalg.norm(a - b) / np.linalg.norm(b)),
           "nbad": int(bad.size), "first_bad": bad[:20].tolist(), "sum_ours": float(a.sum()), "sum_ref": float(b.sum()),
           "repeat_equal": all(bool(np.array_equal(a, plan.apply_A(u))) for _ in range(5)), "s": time.time() - t}
    if bad.size:
        m = ref.maps(sub=False)
        off = m["g2l_offsets"]
        els = sorted(set(int(m["g2l_elem"][off[g]]) for g in bad[:2000]))
        out["bad_elems_first"] = els[:40]
        out["n_bad_elems"] = len(els)
    print(json.dumps(out), flush=True)
    plan.close()
    ref.close()
