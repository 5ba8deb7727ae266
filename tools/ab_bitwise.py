"""Print digests of apply_coarse / PCG outputs of the loaded build (HXB_LIB) for bitwise A/B."""
import hashlib
import json
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_1506_05996_b200 as hx
from oracle import splitmix_vector

out = {}
for k, n in [(24, 4), (52, 7)]:
    p = hx.Plan(hx.generate_cube_mesh(k), n, coarse_solve="amg")
    r = splitmix_vector(p.N, 3)
    h = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]
    out[f"zc_{k}"] = h(p.apply_coarse(r))
    res = p.pcg(None, tol=1e-8)
    out[f"rh_{k}"] = h(np.asarray(res["residual_history"]))
    out[f"u_{k}"] = h(res["u"])
    out[f"it_{k}"] = res["iterations"]
    p.close()
print(json.dumps(out))
