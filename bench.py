"""bench.py — B200 matrix-free SEM PCG (hexsem solver path) benchmark.

Workload (BASELINE.json configs[1], "cfg2"): 52^3 uniform hexes, N=7
(48,627,125 DOF), Poisson (kappa=1, c=0, s=1), all-Dirichlet, two-scale
Schwarz PCG to 1e-8.

A "step" is one Ax = SemOperator::apply (operator.cpp:255-287) over the full
mesh: the element contraction kernel plus the deterministic CSR gather. The
headline `value` is Ax GDOF/s = N / (ms per step) with u already in HBM;
`e2e` is the same metric through the reference-facing C-ABI call
`hxb_apply_A` on pinned HOST buffers (H2D of u and D2H of r inside the timed
region). The PCG solve to 1e-8 (the metric's second half) is measured in the
same run and reported under "pcg" (device-timed, plus the host-API e2e).

`roofline` is for the Ax step (ax_elem_kernel + ax_gather_kernel): the
reference's own byte model B_R = 8*NE*(10 np^3 + np^2 + 2) (operator.cpp:31-37,
SURVEY §8d) divided by the device-timed step, against MEASURED_PEAKS.json
hbm_gbs; the element kernel's own share (live CUDA-event time, ncu DRAM bytes)
is a sub-field. `pcg.roofline` does the same for a whole PCG iteration
(Ax + FDM + restriction/prolongation + vector passes).

`cpu_baseline` and `--impl reference` run the unmodified reference
(oracle/_ref/libhexsem_ref.so, compiled from /root/reference sources by
oracle/Makefile) on this box's host cores at the SAME cfg2 workload: its Ax
(single-threaded by design) and its two-scale PCG to 1e-8 in its fastest mode
(fine_threads = cores-1, coarse solve concurrent), measured, not extrapolated.

Multi-GPU (torchrun, N>1): the cfg2 mesh is split into N element slabs
(strong scaling, `"scaling": "strong"`); `--replicas` runs N independent cfg2
replicas instead (weak scaling).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Ax GDOF/s (FP64) and PCG solve time to 1e-8 at N=7, ~50M DOF, 1/2/4/8 B200"
SAMPLE_K = 26  # bounded CPU sample: 26^3 hexes at N=7 (6.1M DOF, 1/8 of cfg2)


def _env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def _ncu_traffic(kernel: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel` from
    the committed `ncu --set full` capture summary (profiles/ncu_traffic.json,
    written by tools/ncu_table.py); None when absent."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        return json.load(open(path))["kernels"][kernel]["dram_bytes_per_launch"]
    except (OSError, KeyError, ValueError):
        return None


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,utilization.gpu,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.idx = device_index
        self.proc = None
        self.f = None

    def start(self):
        try:
            self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.3)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.flush()
        rows = []
        with open(self.f.name) as fh:
            for line in fh:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 10:
                    rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "samples": 0}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None

        load = [r for r in rows if (num(r[4]) or 0) >= 50] or rows
        sm = [num(r[1]) for r in load if num(r[1]) is not None]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in load:
            for name, v in zip(names, r[6:10]):
                if v.strip().lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": num(rows[0][2]),
                "reasons": sorted(reasons), "samples": len(rows), "samples_under_load": len(load),
                "power_w_max": max((num(r[3]) or 0) for r in rows)}


def workload_config(k: int, order: int, N: int, NE: int) -> dict:
    """The one `config` both arms print (same keys, same values)."""
    return {"workload": f"cfg2: {k}^3 uniform hexes, N={order}, Poisson kappa=1 c=0, all-Dirichlet; "
                        "step = one Ax (SemOperator::apply); PCG to 1e-8 under pcg",
            "k": k, "order": order, "N": N, "NE": NE,
            "l2": "inputs larger than L2 (5.83 GB per Ax vs 126 MB L2); no flush"}


# ---------------------------------------------------------------------------
def cpu_reference(k: int, order: int, steps: int, warmup: int, pcg: bool):
    """The unmodified reference (oracle/_ref) on this host at the given
    workload: SemOperator::apply timed `steps` times after `warmup`, and one
    two-scale pcg to 1e-8 (krylov.cpp:20-71) in the reference's fastest mode
    (fine_threads = cores-1 plus the concurrent coarse solve, precond.cpp:38-45),
    timed by the reference itself (PcgResult wall clock)."""
    from oracle import RefConfig, RefSystem, ref_available, splitmix_vector, OracleSystem

    kind = "reference" if ref_available() else "port"
    cls = RefSystem if kind == "reference" else OracleSystem
    cores = os.cpu_count() or 1
    t0 = time.time()
    sys_ = cls(RefConfig(k=k, order=order, precond="two_scale", concurrent_precond=True,
                         fine_threads=max(1, cores - 1)))
    setup_s = time.time() - t0
    u = splitmix_vector(sys_.N, 12345)
    for _ in range(warmup):
        sys_.apply_A(u)
    times = []
    for _ in range(steps):
        t = time.perf_counter()
        sys_.apply_A(u)
        times.append(time.perf_counter() - t)
    out = {"kind": kind, "N": sys_.N, "mean_s": sum(times) / len(times), "best_s": min(times),
           "setup_s": setup_s, "steps": steps, "warmup": warmup, "cores": cores}
    if pcg:
        b = sys_.load_ones()
        t = time.perf_counter()
        res = sys_.pcg(b, tol=1e-8, max_iterations=500)
        out["pcg"] = {"iterations": res["iterations"], "status": res["status"], "solve_s": res["solve_seconds"],
                      "wall_s": time.perf_counter() - t, "threads": cores,
                      "mode": f"two_scale, fine_threads={max(1, cores - 1)}, concurrent coarse (reference fastest)",
                      "r_final_over_r0": float(res["residual_history"][-1] / res["residual_history"][0])}
    sys_.close()
    return out


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    r = cpu_reference(args.k, args.order, args.steps, args.warmup, not args.no_pcg)
    gdofs = r["N"] / r["mean_s"] / 1e9
    NE = args.k ** 3
    line = {
        "impl": "reference", "metric": METRIC, "value": gdofs, "unit": "GDOF/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["mean_s"] * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (generated mesh, splitmix64 u, s=1 load)",
        "config": workload_config(args.k, args.order, r["N"], NE),
        "parallelism": f"host CPU: Ax single-threaded by design (operator.cpp:255-287); PCG {r['cores']} threads",
        "cpu_baseline": {"value": gdofs, "unit": "GDOF/s", "cores": 1, "kind": r["kind"],
                         "sample": f"reference SemOperator::apply on the full cfg2 mesh ({r['N']} DOF), mean of "
                                   f"{args.steps} after {args.warmup} warm-up (host has {r['cores']} cores)"},
        "e2e": {"value": gdofs, "unit": "GDOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "pcg": r.get("pcg"), "setup_s": r["setup_s"],
    }
    print(json.dumps(line), flush=True)
    return 0


def pcg_roofline(N: int, NE: int, order: int, ms_per_iteration: float, peak: float) -> dict:
    """Algorithmic bytes of one two-scale PCG iteration over
    its device time: Ax (B_R, operator.cpp:31-37), the fine solves (B_P,
    fine.cpp:88-92), the coarse restriction (r, 1/m_N and the local masses,
    coarse.cpp:138-162) and prolongation + combine (local masses, 1/m_N, r,
    the mask and z, coarse.cpp:164-186 + precond.cpp:56-66), and the vector
    passes of krylov.cpp:53-66 (u, r updates with p, f; p = z + beta p: 9 N
    words)."""
    np1, p = order + 1, order + 3
    nl = NE * np1 ** 3
    parts = {"ax": 8 * NE * (10 * np1 ** 3 + np1 ** 2 + 2),
             "fine": 8 * NE * (3 * p ** 3 + 4 * p ** 2),
             "restrict": 8 * (2 * N + nl),
             "prolong_combine": 8 * (4 * N + nl) + N,
             "vectors": 8 * 9 * N}
    total = sum(parts.values())
    gbs = total / (ms_per_iteration * 1e-3) / 1e9
    return {"bound": "hbm", "bytes_per_iteration": total, "parts": parts, "achieved": gbs, "peak": peak,
            "unit": "GB/s", "frac": gbs / peak}


# ---------------------------------------------------------------------------
def run_ours(args, rank, world, local_rank):
    import numpy as np
    import torch

    import paper_1506_05996_b200 as hx

    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device (the B200 path has no CPU fallback)")
    local_rank = local_rank % torch.cuda.device_count()  # --backend gloo tests: ranks may share a GPU
    torch.cuda.set_device(local_rank)
    dist = None
    host_staging = args.backend == "gloo"
    if world > 1:
        import torch.distributed as dist

        if host_staging:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if dist is None:
            return x
        t = torch.tensor([x], device="cpu" if host_staging else "cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    k, order = args.k, args.order
    t0 = time.time()
    mesh = hx.generate_cube_mesh(k)
    distributed = world > 1 and not args.replicas
    if distributed:
        # element-slab partition of the one cfg2 mesh over the ranks (strong scaling)
        plan = hx.Plan(mesh, order, device=local_rank, rank=rank, nranks=world)
        from paper_1506_05996_b200.dist import DistOperator

        dop = DistOperator(plan, torch, dist, host_staging)
    else:
        plan = hx.Plan(mesh, order, device=local_rank)
    setup_s = time.time() - t0
    N, NE = plan.N, plan.NE  # NE: elements this rank owns
    np1 = order + 1
    bytes_ax = 8 * NE * (10 * np1 ** 3 + np1 ** 2 + 2)  # B_R, operator.cpp:31-37 (this rank's share)
    bytes_fdm = 8 * NE * (3 * (order + 3) ** 3 + 4 * (order + 3) ** 2)  # B_P, fine.cpp:88-92

    # u: splitmix64 seed 12345 (oracles.cpp:126-139), the vector the reference is fed
    u_host = hx.synthetic_vector(N, 12345)
    d_u = torch.from_numpy(u_host).to("cuda")
    d_r = torch.empty(N, dtype=torch.float64, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream

    def ax_step():
        if distributed:
            dop.apply(d_u.data_ptr(), d_r.data_ptr(), stream)
        else:
            plan.apply_A_device(d_u.data_ptr(), d_r.data_ptr(), stream)

    # ---- device-resident Ax: W warm-up, K timed --------------------------
    for _ in range(args.warmup):
        ax_step()
    sampler = ClockSampler(local_rank)
    sampler.start()
    plan.kernel_timing(True, max_launches=4 * args.steps + 16)
    launches0 = plan.launch_count()
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(args.steps):
        ax_step()
    ev1.record()
    barrier()
    ms_total = ev0.elapsed_time(ev1)
    launches = plan.launch_count() - launches0
    elem_ms, elem_n = plan.kernel_time("ax_elem")
    gath_ms, gath_n = plan.kernel_time("ax_gather")
    plan.kernel_timing(False)
    ms_step = max_over_ranks(ms_total / args.steps)
    # strong scaling: the ranks share one mesh of N DOF; replicas: N each
    value = (N if distributed else world * N) / (ms_step * 1e-3) / 1e9
    r_dev = d_r.cpu().numpy()
    if distributed:
        return finish_distributed(args, rank, world, plan, value, ms_step, launches, elem_ms, elem_n, gath_ms,
                                  gath_n, ms_total, bytes_ax, N, NE, setup_s, sampler, dist, torch, max_over_ranks)

    # ---- e2e through the C-ABI with pinned host buffers -------------------
    h_u = torch.from_numpy(u_host).pin_memory()
    h_r = torch.empty(N, dtype=torch.float64).pin_memory()
    for _ in range(min(args.warmup, 3)):
        plan.apply_A_host_ptr(h_u.data_ptr(), h_r.data_ptr())
    barrier()
    e2e_steps = max(3, min(args.steps, 20))
    t = time.perf_counter()
    for _ in range(e2e_steps):
        plan.apply_A_host_ptr(h_u.data_ptr(), h_r.data_ptr())
    e2e_s = max_over_ranks((time.perf_counter() - t) / e2e_steps)
    e2e_parity = float(np.max(np.abs(h_r.numpy() - r_dev)))

    # ---- FDM (fine Schwarz) kernel timing from the same plan ---------------
    fdm = None
    try:
        prof = plan.profile(5)
        fdm = {"ms": prof["fdm"], "algorithmic_bytes": bytes_fdm,
               "gbs": bytes_fdm / (prof["fdm"] * 1e-3) / 1e9 if prof["fdm"] > 0 else None,
               "components_ms": prof}
    except Exception as exc:  # noqa: BLE001
        fdm = {"error": str(exc)}

    # ---- PCG solve to 1e-8 (device-resident) + e2e (host b in, host u out) --
    pcg = None
    if not args.no_pcg:
        res = plan.pcg_device(None, tol=1e-8, max_iterations=500, want_u=False)  # warm-up solve
        barrier()
        l0 = plan.launch_count()
        res = plan.pcg_device(None, tol=1e-8, max_iterations=500, want_u=False)
        pcg_launches = plan.launch_count() - l0
        solve_s = max_over_ranks(res["solve_seconds"])
        # host b in and host u out through pinned buffers (the contract's e2e leg)
        b_pin = torch.empty(N, dtype=torch.float64).pin_memory().numpy()
        u_pin = torch.empty(N, dtype=torch.float64).pin_memory().numpy()
        b_pin[:] = plan.load_ones()
        t = time.perf_counter()
        res_e2e = plan.pcg(b_pin, tol=1e-8, max_iterations=500, u_out=u_pin)
        e2e_solve = max_over_ranks(time.perf_counter() - t)
        pcg = {"tol": 1e-8, "iterations": res["iterations"], "status": res["status"],
               "solve_s": solve_s, "ms_per_iteration": solve_s * 1e3 / max(1, res["iterations"]),
               "gpu_launches": pcg_launches,
               "e2e_solve_s": e2e_solve, "e2e_h2d_bytes": 8 * N, "e2e_d2h_bytes": 8 * N,
               "r0": float(res["residual_history"][0]), "r_final": float(res["residual_history"][-1]),
               "u_norm2": float(np.linalg.norm(res_e2e["u"]))}
        gold_path = os.path.join(ROOT, "tests", "golden", "cfg2_pcg.json")
        exact_path = os.path.join(ROOT, "tests", "golden", "cfg2_oracle_exactdot.json")
        if (k, order) == (52, 7) and os.path.exists(gold_path):
            gold = json.load(open(gold_path))
            rh = np.asarray(res["residual_history"])
            gh = np.asarray(gold["residual_history"])
            m = min(len(rh), len(gh))
            ex = None
            if os.path.exists(exact_path):
                eh = np.asarray(json.load(open(exact_path))["1"]["residual_history"])
                me = min(len(rh), len(eh))
                ex = {"max_abs_dr_over_rk_vs_exact_dot_oracle": float(np.max(np.abs(rh[:me] - eh[:me]) / eh[:me])),
                      "reference_own_dot_rounding_floor": float(np.max(np.abs(eh[:min(len(eh), len(gh))] -
                                                                             gh[:min(len(eh), len(gh))]) /
                                                                      gh[:min(len(eh), len(gh))]))}
            pcg["parity_vs_reference"] = {
                "ref_iterations": gold["iterations"],
                "exact_dot": ex,
                "max_abs_dr_over_r0": float(np.max(np.abs(rh[:m] - gh[:m])) / gh[0]),
                "max_abs_dr_over_rk": float(np.max(np.abs(rh[:m] - gh[:m]) / gh[:m])),
                "u_norm2_rel_diff": abs(pcg["u_norm2"] - gold["u_norm2"]) / gold["u_norm2"],
                "ref_cpu_solve_s_build_host": gold["timing"]["solve_s"],
            }
    # ---- operator variant on_the_fly (operator.cpp:174-253): same Ax, geometry from corners
    otf = None
    if not args.no_otf:
        try:
            plan_o = hx.Plan(mesh, order, device=local_rank, precond="none", variant="on_the_fly")
            d_r2 = torch.empty_like(d_r)
            for _ in range(args.warmup):
                plan_o.apply_A_device(d_u.data_ptr(), d_r2.data_ptr(), stream)
            plan_o.kernel_timing(True, max_launches=4 * args.steps + 16)
            barrier()
            ev0.record()
            for _ in range(args.steps):
                plan_o.apply_A_device(d_u.data_ptr(), d_r2.data_ptr(), stream)
            ev1.record()
            barrier()
            ms_o = ev0.elapsed_time(ev1) / args.steps
            oe_ms, oe_n = plan_o.kernel_time("ax_elem")
            plan_o.kernel_timing(False)
            d_r_t = torch.from_numpy(r_dev).to("cuda")
            otf = {"ms_per_step": ms_o, "gdofs": N / (ms_o * 1e-3) / 1e9,
                   "elem_kernel_ms": oe_ms / max(1, oe_n),
                   "words_model_bytes": 8 * NE * (3 * np1 ** 3 + np1 ** 2 + 2),
                   "rel_l2_vs_stored": float(torch.linalg.norm(d_r2 - d_r_t) / torch.linalg.norm(d_r_t)),
                   "device_bytes_saved": 8 * NE * 6 * ((np1 ** 3 + 1) & ~1)}
            plan_o.close()
        except Exception as exc:  # noqa: BLE001
            otf = {"error": str(exc)}
    clocks = sampler.stop()

    # ---- CPU baseline (rank 0, N=1 only): the reference at the same cfg2 workload
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            r = cpu_reference(k, order, 3, 1, not (args.no_pcg or args.no_cpu_pcg))
            cpu = {"value": r["N"] / r["mean_s"] / 1e9, "unit": "GDOF/s", "cores": 1, "kind": r["kind"],
                   "sample": f"reference SemOperator::apply on the full cfg2 mesh ({r['N']} DOF), mean of 3 after "
                             f"1 warm-up, single-threaded by design; host has {r['cores']} cores",
                   "pcg": r.get("pcg"), "setup_s": r["setup_s"]}
        except Exception as exc:  # noqa: BLE001
            cpu = {"value": None, "unit": "GDOF/s", "cores": 1, "kind": "reference", "sample": f"failed: {exc}"}

    peak, peak_src = _peaks()
    elem_avg_ms = elem_ms / max(1, elem_n)
    gath_avg_ms = gath_ms / max(1, gath_n)
    achieved = bytes_ax / (ms_step * 1e-3) / 1e9  # whole Ax step: B_R / device-timed step
    t_elem, t_gath = _ncu_traffic("ax_elem_kernel"), _ncu_traffic("ax_gather_kernel")
    if pcg is not None:
        pcg["roofline"] = pcg_roofline(N, NE, order, pcg["ms_per_iteration"], peak)
    line = {
        "metric": METRIC, "value": value, "unit": "GDOF/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak" if args.replicas else "strong",  # N>1 default: one mesh split in element slabs
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (generated 52^3 mesh, splitmix64 u, s=1 load)",
        "config": workload_config(k, order, N, NE),
        "parallelism": "single GPU" if world == 1 else f"{world} independent replicas (weak)",
        "e2e": {"value": N * world / e2e_s / 1e9, "unit": "GDOF/s", "h2d_bytes_per_step": 8 * N,
                "d2h_bytes_per_step": 8 * N, "api": "hxb_apply_A (host pointers, pinned)",
                "ms_per_step": e2e_s * 1e3, "max_abs_diff_vs_device_path": e2e_parity},
        "gpu_launches": launches,
        "roofline": {"kernel": "Ax step = ax_elem_kernel + ax_gather_kernel", "bound": "hbm",
                     "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": (t_elem + t_gath) if (t_elem and t_gath) else None,
                     "peak_source": peak_src, "algorithmic_bytes_per_launch": bytes_ax,
                     "algorithmic_bytes_model": "B_R = 8*NE*(10 np^3 + np^2 + 2) (operator.cpp:31-37)",
                     "avg_step_ms": ms_step,
                     "elem_kernel": {"avg_launch_ms": elem_avg_ms, "launches_timed": elem_n,
                                     "share_of_step": elem_ms / ms_total if ms_total else None,
                                     "ncu_dram_bytes": t_elem,
                                     "dram_frac": (t_elem / (elem_avg_ms * 1e-3) / 1e9 / peak)
                                     if (t_elem and elem_n) else None},
                     "gather_kernel": {"avg_launch_ms": gath_avg_ms, "ncu_dram_bytes": t_gath}},
        "fdm": fdm,
        "pcg": pcg,
        "ax_on_the_fly": otf,
        "clocks": clocks,
        "setup_s": setup_s,
        "cpu_baseline": cpu,
    }
    plan.close()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


def finish_distributed(args, rank, world, plan, value, ms_step, launches, elem_ms, elem_n, gath_ms, gath_n,
                       ms_total, bytes_ax, N, NE, setup_s, sampler, dist, torch, max_over_ranks):
    """JSON line of the element-slab distributed Ax (strong scaling of cfg2)."""
    clocks = sampler.stop()
    peak, peak_src = _peaks()
    elem_avg_ms = elem_ms / max(1, elem_n)
    achieved = bytes_ax / (elem_avg_ms * 1e-3) / 1e9 if elem_n else None
    info = plan.dist_info()
    pcg = None
    if not args.no_pcg:  # distributed two-scale PCG to 1e-8 (paper_1506_05996_b200/dist.py)
        from paper_1506_05996_b200.dist import RankCtx, TorchComm, dist_pcg

        ctx = RankCtx(plan, torch)
        comm = TorchComm(dist, torch, host_staging=args.backend == "gloo")
        ctx.b.copy_(torch.from_numpy(plan.load_ones()).cuda())
        dist_pcg([ctx], comm, tol=1e-8)  # warm-up
        dist.barrier()
        torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record()
        res = dist_pcg([ctx], comm, tol=1e-8)
        t1.record()
        torch.cuda.synchronize()
        solve_s = max_over_ranks(t0.elapsed_time(t1) / 1e3)
        pcg = {"tol": 1e-8, "iterations": res["iterations"], "status": res["status"], "solve_s": solve_s,
               "r0": res["residual_history"][0], "r_final": res["residual_history"][-1],
               "orchestration": "Python loop over staged C-ABI calls, NCCL p2p + all-reduce (torch.distributed)"}
    line = {
        "metric": METRIC, "value": value, "unit": "GDOF/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (generated mesh, splitmix64 u)",
        "config": {"workload": f"cfg2 Ax distributed: {args.k}^3 hexes N={args.order} split in {world} element slabs",
                   "k": args.k, "order": args.order, "N": N, "NE_per_rank": NE,
                   "parallelism": f"element-slab partition x{world}, {args.backend} neighbour exchange (2 messages per Ax)",
                   "interface_doubles_rank0": info["n_up"],
                   "l2": "inputs larger than L2; no flush"},
        "e2e": None, "gpu_launches": launches,
        "roofline": {"kernel": "ax_elem_kernel", "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak if achieved else None, "traffic": _ncu_traffic("ax_elem_kernel"), "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": bytes_ax, "avg_launch_ms": elem_avg_ms,
                     "share_of_step": elem_ms / ms_total if ms_total else None},
        "pcg": pcg,
        "clocks": clocks, "setup_s": setup_s, "cpu_baseline": None,
    }
    plan.close()
    if rank == 0:
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--k", type=int, default=52)
    ap.add_argument("--order", type=int, default=7)
    ap.add_argument("--no-pcg", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cpu-pcg", action="store_true", help="cpu_baseline: Ax only (skip the reference cfg2 PCG)")
    ap.add_argument("--no-otf", action="store_true", help="skip the on-the-fly operator variant measurement")
    ap.add_argument("--replicas", action="store_true", help="N>1: independent cfg2 replicas instead of a partition")
    ap.add_argument("--backend", choices=["nccl", "gloo"], default="nccl",
                    help="gloo: host-staged messages, lets several ranks share one GPU (tests)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    rank = _env_int("RANK", 0)
    world = _env_int("WORLD_SIZE", 1)
    local_rank = _env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        return run_reference(args, rank, world)
    return run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    sys.exit(main())
