"""A/B timing of one library build (HXB_LIB) and plan options on cfg2:
per-component device times (hxb_profile) and the live kernel times inside a
PCG solve. usage: HXB_LIB=... python tools/ab_run.py [k] [order] [opt=val ...]"""
import json
import os
import sys

sys.path.insert(0, ".")
import paper_1506_05996_b200 as hx  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 52
n = int(sys.argv[2]) if len(sys.argv) > 2 else 7
opts = {}
for a in sys.argv[3:]:
    key, val = a.split("=")
    opts[key] = int(val) if key in ("coarse_sms",) else val.lower() in ("1", "true", "yes")
p = hx.Plan(hx.generate_cube_mesh(k), n, **opts)
prof = p.profile(5)
p.pcg_device(None, tol=1e-8, want_u=False)
p.kernel_timing(True, 4000)
r = p.pcg_device(None, tol=1e-8, want_u=False)
live = {}
for tag in ("ax_elem", "ax_gather", "fdm", "combine", "coarse", "combine_fine"):
    ms, cnt = p.kernel_time(tag)
    live[tag] = ms / max(1, cnt)
print(json.dumps({"lib": os.environ.get("HXB_LIB", "default"), "opts": opts, "k": k, "n": n,
                  "coarse_sms": getattr(p, "coarse_sms", None),
                  "iterations": r["iterations"], "solve_ms": r["solve_seconds"] * 1e3,
                  "ms_per_it": r["solve_seconds"] * 1e3 / r["iterations"], "live": live,
                  "profile": {kk: round(v, 4) for kk, v in prof.items() if v}}))
