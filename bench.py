"""Benchmark: time to precision of the truncated-Newton EOT solver (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N = 1 (the metric's configuration, BASELINE configs[1]): D2 -- n = 4096 (64x64
pixel grid), squared-L2 cost, smooth-random marginals (seeds 0 / 1), MDOT
annealing gamma 2^5 -> 2^16 until ||r(P)-r||_1 + ||c(P)-c||_1 <= 1e-6.  One
step = one complete ``mdot`` solve (all stages, final plan, rounding, primal
cost); the metric is seconds per solve (lower is better).

  value     device-resident: C already in HBM (a CUDA tensor problem); CUDA
            events bracket each solve on the solver stream; L2 is flushed
            (512 MB write) between steps, and the 134 MB cost is itself > L2.
  e2e       the same solve through the public API with a HOST (page-locked)
            problem: the 134 MB cost H2D, the solve, and the 134 MB rounded
            plan D2H all inside the timed region (bytes counted by the package).
  parity    the timed configuration against the reference's own trajectory
            (tests/golden/traj_D2_grid64_l2sq_s0.npz, produced by the reference):
            stages, CG iterations, u / v inf-norm-relative differences.
  roofline  the persistent CG/Newton kernel (k_coop), the dominant kernel,
            against the bytes each launch has to stream: per HVP two passes
            over the plan entries inside the rows' nonzero 64-column segments
            (ring mode, HBM / L2) or over the compressed nonzeros (value +
            column index, modes 2 / 3: shared memory / L2) -- what the kernel
            actually reads, not the dense 16 n^2; peak = measured HBM copy
            bandwidth.  ``traffic`` = ncu DRAM bytes per launch.
  cpu_baseline  complete solves of the reference's CPU path (the bit-exact
            oracle port of otnewton.mdot, oracle/) on the host cores: OpenBLAS
            and the oracle's 256-row slabs on all threads.

N > 1 (``--gpus N`` re-executes itself under torch.distributed.run when not
already launched that way): the headline is the ROW-SHARDED on-the-fly solve
D4 (BASELINE configs[3]): n = 65536 3-D points, L2^2 cost recomputed in every
pass, gamma 2^5 -> 2^10 (``--sharded d5``: D5, n = 2^20, BASELINE configs[4]), rank g owning rows [g n/N, (g+1) n/N) with one NCCL
allreduce per column-direction product; strong scaling (same n at every N);
value = max over ranks of the solve time.  ``extras.d4_1gpu`` is the same solve
on rank 0's GPU alone (the scaling reference), ``extras.d2_replicas`` the D2
solve on every rank independently.

--impl reference: the reference's CPU path (the oracle port) timed on full
solves of the same workload on the host cores (rank 0 only).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sec to ||r(P)-r||_1+||c(P)-c||_1<=1e-6 (n=4096)"
METRIC_D4 = "sec to solve n={n} on-the-fly 3-D OT (gamma 2^5->2^10), row-sharded"
D2 = dict(spec="grid:64:l2sq:0", gamma_i=2.0 ** 5, gamma_f=2.0 ** 16, p=1.5, q_init=2.0)
D2_GOLDEN = os.path.join(ROOT, "tests", "golden", "traj_D2_grid64_l2sq_s0.npz")
D4_GAMMA = (2.0 ** 5, 2.0 ** 10)
L2_FLUSH_BYTES = 512 << 20

CONFIG_D2 = {
    "workload": "D2 n=4096 grid64 L2^2 smooth-random seeds 0/1 gamma 2^5->2^16 to 1e-6",
    "n": 4096, "gamma_i": D2["gamma_i"], "gamma_f": D2["gamma_f"], "p": 1.5, "q_init": 2.0,
    "parallelism": "single",
    "l2": "flushed between steps (512 MB write); C and P are 134 MB > L2",
}


def config_d4(n, world):
    tag = "D5" if n >= 2 ** 20 else "D4"
    return {"workload": f"{tag} n={n} 3-D uniform points on-the-fly L2^2 gamma 2^5->2^10",
            "n": n, "gamma_i": D4_GAMMA[0], "gamma_f": D4_GAMMA[1],
            "parallelism": f"rows{world}",
            "l2": "no n x n array exists: every pass recomputes the cost from the points"}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------------------
# clocks during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi in a subprocess (no GIL contention with the solver's host
    loop) sampling SM clocks and throttle reasons every 200 ms."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        clk, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            try:
                clk.append(float(parts[0]))
                mx = float(parts[1])
            except (ValueError, IndexError):
                continue
            for name, val in zip(names, parts[3:7]):
                if val.lower() == "active":
                    reasons.add(name)
        if not clk:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": ["nvidia-smi unavailable"]}
        return {"sm_mhz": float(statistics.median(clk)), "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(clk)}


# ---------------------------------------------------------------------------
# roofline of the persistent solver from its launch records
# ---------------------------------------------------------------------------
# bytes per compressed nonzero per pass: the value (8) and its column / row
# index (2, u16) -- the CSR for P w, the CSC for P^T x
SPARSE_BYTES_PER_NNZ = 10
MODE_NAMES = {0: "ring (streamed spans)", 2: "compressed rows, shared memory",
              3: "compressed rows, global memory (L2)"}


def kcoop_roofline(coop, peak_gbs, n):
    """Per-mode and total roofline of k_coop from TELEMETRY.coop records
    (ms, hvps, dv, n, mode, nnz, span, cg)."""
    per_mode = {}
    tot_bytes = tot_ms = 0.0
    for (ms, hvps, dv, _n, mode, nnz, span, cg) in coop:
        if mode == 0:
            # each HVP streams the spans twice (P^T x, then P w); d_v once more
            b = 8.0 * span * (2 * hvps + dv)
        else:
            # compression reads the spans once; then every pass walks the
            # compressed nonzeros (value + index)
            b = 8.0 * span + SPARSE_BYTES_PER_NNZ * nnz * (2 * hvps + dv)
        m = per_mode.setdefault(mode, {"launches": 0, "hvps": 0, "cg_iters": 0, "ms": 0.0,
                                       "bytes": 0.0, "nnz_mean": 0.0})
        m["launches"] += 1
        m["hvps"] += hvps
        m["cg_iters"] += cg
        m["ms"] += ms
        m["bytes"] += b
        m["nnz_mean"] += nnz
        tot_bytes += b
        tot_ms += ms
    for mode, m in per_mode.items():
        m["nnz_mean"] /= max(m["launches"], 1)
        m["gbps"] = m["bytes"] / (m["ms"] * 1e-3) / 1e9 if m["ms"] > 0 else 0.0
        m["frac_of_hbm_peak"] = m["gbps"] / peak_gbs
        m["us_per_hvp"] = m["ms"] * 1e3 / max(m["hvps"], 1)
        m["path"] = MODE_NAMES.get(mode, str(mode))
    achieved = tot_bytes / (tot_ms * 1e-3) / 1e9 if tot_ms > 0 else 0.0
    return achieved, tot_bytes, tot_ms, {str(k): v for k, v in sorted(per_mode.items())}


def kcoop_traffic():
    """ncu DRAM bytes per k_coop launch of one D2 solve (profiles/, tools/kcoop_dram.py)."""
    path = os.path.join(ROOT, "profiles", "kcoop_traffic.json")
    if not os.path.exists(path):
        return None
    with open(path) as fh:
        return json.load(fh).get("dram_bytes_per_launch")


# ---------------------------------------------------------------------------
# our arm, N = 1: D2
# ---------------------------------------------------------------------------
def parity_block(sol, prob):
    """The timed configuration against the reference's own trajectory."""
    z = np.load(D2_GOLDEN, allow_pickle=False)
    meta = json.loads(str(z["meta"]))
    st = sol.final_state
    u, v = st.u, st.v
    du = float(np.abs(u - z["u"]).max() / np.abs(z["u"]).max())
    dv = float(np.abs(v - z["v"]).max() / np.abs(z["v"]).max())
    st.set_targets(prob.r, prob.c)
    ss = meta["self_spread"]
    return {"stages": len(sol.iterations), "stages_ref": len(meta["stages"]),
            "cg_iters": sum(i.stats.cg_iters for i in sol.iterations),
            "cg_iters_ref": meta["totals"]["cg"],
            "cg_iters_ref_deterministic": ss["cg_total"],
            "newton_steps": sum(i.stats.newton_steps for i in sol.iterations),
            "newton_steps_ref": meta["totals"]["newton"],
            "du_rel": du, "dv_rel": dv, "ref_self_spread_du": ss["du"],
            "ref_self_spread_dv": ss["dv"],
            "primal_rel": abs(sol.primal_cost - meta["primal"]) / abs(meta["primal"]),
            "true_marginal_err": st.grad_norm_l1(), "target": 1e-6}


def run_d2(args, dev):
    import torch

    import paper_2504_02067_b200 as ot
    from paper_2504_02067_b200._device import TELEMETRY

    host_prob = ot.workload(D2["spec"])
    n = host_prob.n
    pinned_C = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
    pinned_C.numpy()[:] = host_prob.C                    # e2e H2D source: page-locked
    host_prob = ot.Problem(C=pinned_C.numpy(), r=host_prob.r, c=host_prob.c, label=host_prob.label)
    dprob = ot.Problem(C=torch.from_numpy(host_prob.C).to(dev), r=host_prob.r, c=host_prob.c,
                       label=host_prob.label)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def solve(prob):
        return ot.mdot(prob, D2["gamma_i"], D2["gamma_f"], p=D2["p"], q_init=D2["q_init"])

    for _ in range(args.warmup):
        solve(dprob)
    torch.cuda.synchronize()

    # ---- device-resident timed region --------------------------------------
    TELEMETRY.reset()
    TELEMETRY.time_coop = True
    step_ms = []
    with ClockSampler(dev.index) as clocks:
        torch.cuda.synchronize()
        for _ in range(args.steps):
            flush.fill_(1.0)                             # evict L2 between steps (untimed)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            sol = solve(dprob)
            e1.record(stream)
            e1.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            del sol                                      # a held result pins a 134 MB plan
        torch.cuda.synchronize()
    TELEMETRY.time_coop = False
    launches = TELEMETRY.launches
    coop = list(TELEMETRY.coop)
    calls = dict(TELEMETRY.calls)

    # ---- e2e through the public API with host buffers ------------------------
    _warm = solve(host_prob)                             # warm the page-locked result buffer
    del _warm
    TELEMETRY.reset()
    e2e_ms = []
    for _ in range(args.steps):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sol_h = solve(host_prob)                         # H2D of C inside, D2H of P inside
        torch.cuda.synchronize()
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
        if len(e2e_ms) < args.steps:
            del sol_h
    h2d = TELEMETRY.h2d / args.steps
    d2h = TELEMETRY.d2h / args.steps

    # ---- parity of the timed configuration (after the timed regions) -------
    sol = solve(dprob)
    parity = parity_block(sol, host_prob)
    st = sol_h.final_state
    st.set_targets(host_prob.r, host_prob.c)
    parity["true_marginal_err_e2e"] = st.grad_norm_l1()

    peaks, peak_src = load_peaks()
    hbm = float(peaks["hbm_gbs"])
    achieved, alg_bytes, coop_ms, modes = kcoop_roofline(coop, hbm, n)
    ms = statistics.mean(step_ms)
    out = {
        "metric": METRIC,
        "value": ms / 1e3,
        "unit": "s",
        "n_gpus": 1,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": False,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded 64x64 grid cost + smooth-random marginals, reference generators)",
        "config": dict(CONFIG_D2),
        "e2e": {"value": statistics.mean(e2e_ms) / 1e3, "unit": "s",
                "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
        "gpu_launches": launches,
        "gpu_launches_per_step": launches / max(args.steps, 1),
        "parity": parity,
        "roofline": {
            "bound": "hbm", "kernel": "k_coop (persistent CG/Newton)",
            "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
            "peak_source": peak_src,
            "traffic": kcoop_traffic(),
            "basis": "bytes each launch must stream: ring mode 8 B x span entries per pass "
                     "(2 passes per HVP + 1 for d_v); compressed modes 8 B x span once + "
                     f"{SPARSE_BYTES_PER_NNZ} B x nnz per pass (value + u16 index, from shared "
                     "memory / L2); traffic = ncu dram__bytes per launch (profiles/)",
            "alg_bytes_per_launch": alg_bytes / max(len(coop), 1),
            "launches": len(coop), "kernel_ms_total": coop_ms,
            "kernel_share_of_step": coop_ms / sum(step_ms),
            "per_mode": modes,
        },
        "clocks": clocks.summary(),
        "per_step_ms": step_ms,
        "e2e_per_step_ms": e2e_ms,
        "calls_per_step": {k: v / args.steps for k, v in calls.items()},
    }
    return out


# ---------------------------------------------------------------------------
# extras (N = 1): the other configurations, one timed solve each
# ---------------------------------------------------------------------------
# FP64-pipe instructions per plan entry of the on-the-fly passes at d = 3 (ncu
# smsp__inst_executed_pipe_fp64 x 32 / entries, n = 65536, separable exponent:
# 21.2 for the product pass; 32 with the exact-cost exponent, OTN_PC_EXACT=1)
PAIR_FP64_INSTR_PER_ENTRY = 21


def fused_px(dev, peak, reps=200):
    """BASELINE's "fused P.x GB/s": steady-state time of one HVP (P^T x, the
    column combine, P w) repeated inside one persistent launch on the D2 plan
    of the first stage (dense) and of the last (~450 K nonzeros).  The dense
    figure is effective bandwidth over 16 n^2 bytes; P (134 MB) is about the
    L2 size, so part of the stream is served from L2."""
    import torch

    import paper_2504_02067_b200 as ot
    from paper_2504_02067_b200._device import vptr
    p = ot.workload(D2["spec"])
    dp = ot.Problem(C=torch.from_numpy(p.C).to(dev), r=p.r, c=p.c)
    res = {}
    for key, gf in (("dense_gamma_2^5", 2.0 ** 5), ("sparse_gamma_2^16", 2.0 ** 16)):
        st = ot.mdot(dp, 2.0 ** 5, gf).final_state
        s = ot.DiscountedSystem.from_state(st)
        k = s._ctx
        x = torch.randn(k.ld, dtype=torch.float64, device=dev)
        out = k.vec()

        def go(reps_):
            k.call("otn_probe", vptr(s._P), vptr(s._mask), vptr(s._cP), vptr(s._rP), vptr(x),
                   vptr(out), 5, reps_)
        go(reps)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        go(reps)
        e1.record()
        e1.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / reps
        dense = 16.0 * p.n * p.n
        res[key] = {"hvp_us": us, "effective_gbps_dense_bytes": dense / (us * 1e-6) / 1e9,
                    "effective_frac_of_hbm_peak": dense / (us * 1e-6) / 1e9 / peak}
    res["peak_gbps"] = peak
    return res


def d4_solve(dev, n, comm=None):
    """One timed D4 solve (cost object built outside the timed region);
    returns (seconds, record)."""
    import torch

    import paper_2504_02067_b200 as ot
    from paper_2504_02067_b200._device import TELEMETRY
    from paper_2504_02067_b200.pointcloud import Comm, PointCloudCost
    comm = comm or Comm()
    pc = ot.points_problem(n, 3, 0)
    cost = PointCloudCost(pc, dev, comm=comm)
    TELEMETRY.reset()
    before = dict(comm.stats)
    torch.cuda.synchronize()
    comm.barrier()
    t0 = time.perf_counter()
    sol = ot.mdot(pc, D4_GAMMA[0], D4_GAMMA[1], cost=cost)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    collectives = {k: v - before.get(k, 0) for k, v in comm.stats.items()}
    passes = TELEMETRY.calls.get("otn_pc_pass", 0)
    launches = TELEMETRY.launches
    st = sol.final_state
    st.set_targets(pc.r, pc.c)
    err = st.grad_norm_l1()
    entries = float(n) * n * passes / comm.world        # per rank: n x n/world per pass
    peak_entries = 148 * 64 * 1.965e9 / PAIR_FP64_INSTR_PER_ENTRY
    rec = {"n": n, "dim": 3, "gamma": list(D4_GAMMA), "gpus": comm.world,
           "sharding": f"rows over {comm.world} ranks" if comm.world > 1 else "none",
           "stages": len(sol.iterations), "cg": sum(i.stats.cg_iters for i in sol.iterations),
           "passes_per_rank": passes, "launches_per_rank": launches,
           "true_marginal_err": err, "primal": sol.primal_cost,
           "collectives": collectives,
           "entries_per_s_per_gpu": entries / dt,
           "fp64_pipe_frac_est": entries / dt / peak_entries,
           "fp64_basis": f"{PAIR_FP64_INSTR_PER_ENTRY} FP64 instr/entry (SASS), "
                         "64 FP64 instr/clk/SM x 148 SMs x 1.965 GHz"}
    return dt, rec


def d3_from_points(dev, gi, gf, host_C):
    """D3 end to end from its 8-bit point sets: the host -> device copy of X, Y
    (float64), the cost built on the tensor cores (problems.pixel_cost_device,
    bit-identical to the host's), the solve, the plan back to the host."""
    import torch

    import paper_2504_02067_b200 as ot
    from paper_2504_02067_b200 import problems
    X, Y = problems.pixel_points(4096, 784, 0)
    r = np.full(4096, 1.0 / 4096)
    Xp, Yp = torch.from_numpy(X).pin_memory(), torch.from_numpy(Y).pin_memory()
    Ph = torch.empty((4096, 4096), dtype=torch.float64).pin_memory()

    def once():
        Xd, Yd = Xp.to(dev, non_blocking=True), Yp.to(dev, non_blocking=True)
        t0 = time.perf_counter()
        C = problems.pixel_cost_device(Xd, Yd, dev)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        sol = ot.mdot(ot.Problem(C=C, r=r, c=r.copy()), gi, gf)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        if torch.is_tensor(sol.P):
            Ph.copy_(sol.P)
        else:
            Ph.numpy()[...] = sol.P
        return C, t1 - t0, t2 - t1
    C, _, _ = once()
    same = bool(np.array_equal(C.cpu().numpy(), host_C))
    del C
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _, t_cost, t_solve = once()
    torch.cuda.synchronize()
    return {"from_points_e2e_s": time.perf_counter() - t0, "cost_build_s": t_cost,
            "from_points_solve_s": t_solve, "cost_bitwise_equal_host": same,
            "from_points_h2d_bytes": 2 * X.nbytes, "from_points_d2h_bytes": Ph.numel() * 8,
            "cost_build": "otn_pixel_cost: u8 x u8 -> s32 tcgen05.mma kind::i8 (exact), "
                          "then /max; host numpy builds the same C in ~0.2 s"}


def run_extras(args, dev):
    import torch

    import paper_2504_02067_b200 as ot
    extras = {}
    peaks, _ = load_peaks()
    try:
        for key, spec, gi, gf in (("d1_fixed", "pts:1024:2:0", 2.0 ** 10, 2.0 ** 10),
                                  ("d3", "pix:4096:784:0", 2.0 ** 5, 2.0 ** 16)):
            p = ot.workload(spec)
            dp = ot.Problem(C=torch.from_numpy(p.C).to(dev), r=p.r, c=p.c)
            ot.mdot(dp, gi, gf)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            sol = ot.mdot(dp, gi, gf)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            st = sol.final_state
            st.set_targets(p.r, p.c)
            extras[key] = {"spec": spec, "gamma": [gi, gf], "s": dt,
                           "stages": len(sol.iterations),
                           "cg": sum(i.stats.cg_iters for i in sol.iterations),
                           "true_marginal_err": st.grad_norm_l1()}
            if key == "d3":
                extras[key].update(d3_from_points(dev, gi, gf, p.C))
        # the median over seeds 0..4 (L2^2) and the L1 cost
        seeds = []
        for spec in [f"grid:64:l2sq:{s}" for s in range(5)] + ["grid:64:l1:0"]:
            p = ot.workload(spec)
            dp = ot.Problem(C=torch.from_numpy(p.C).to(dev), r=p.r, c=p.c)
            ot.mdot(dp, D2["gamma_i"], D2["gamma_f"])
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            sol = ot.mdot(dp, D2["gamma_i"], D2["gamma_f"])
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            st = sol.final_state
            st.set_targets(p.r, p.c)
            seeds.append({"spec": spec, "s": dt, "stages": len(sol.iterations),
                          "cg": sum(i.stats.cg_iters for i in sol.iterations),
                          "true_marginal_err": st.grad_norm_l1()})
        l2 = sorted(x["s"] for x in seeds if "l2sq" in x["spec"])
        extras["d2_seeds"] = {"runs": seeds, "l2sq_median_s": l2[len(l2) // 2]}
        extras["fused_px"] = fused_px(dev, float(peaks["hbm_gbs"]))
        if args.d4_n:
            d4_solve(dev, args.d4_n)                      # warm-up (context, modules)
            dt, rec = d4_solve(dev, args.d4_n)
            rec["s"] = dt
            extras["d4_1gpu"] = rec
    except Exception as exc:                              # extras never break the headline
        extras["error"] = f"{type(exc).__name__}: {exc}"
    return extras


# ---------------------------------------------------------------------------
# our arm, N > 1: D4 row-sharded (headline), D2 replicas (extras)
# ---------------------------------------------------------------------------
def run_sharded(args, rank, world, dev):
    import torch

    import paper_2504_02067_b200 as ot
    from paper_2504_02067_b200._device import TELEMETRY
    from paper_2504_02067_b200.pointcloud import Comm, PointCloudCost
    comm = Comm()
    n = 2 ** 20 if args.sharded == "d5" else (args.d4_n or 65536)
    out_extras = {}
    # the 1-GPU reference solve of the same n on rank 0 (strong-scaling basis;
    # D5 on one GPU takes ~7 min: profiles/r02_d5_solve.json instead)
    if rank == 0 and not args.no_extras and n <= 2 ** 17:
        dt1, rec1 = d4_solve(dev, n, comm=Comm.local())
        rec1["s"] = dt1
        out_extras["d4_1gpu"] = rec1
    comm.barrier()
    for _ in range(min(args.warmup, 1)):                  # a D4 solve is seconds: one warm-up
        d4_solve(dev, n, comm)
    times, rec, launches = [], None, 0
    with ClockSampler(dev.index) as clocks:
        for _ in range(args.steps):
            dt, rec = d4_solve(dev, n, comm)
            times.append(max_over_ranks(dt, world))
            launches += rec["launches_per_rank"]
    TELEMETRY.reset()
    # e2e: the same public call with the points built on the host inside the
    # timed region (H2D of the row shard + all column points; D2H of the result)
    comm.barrier()
    t0 = time.perf_counter()
    pc = ot.points_problem(n, 3, 0)
    sol = ot.mdot(pc, D4_GAMMA[0], D4_GAMMA[1], cost=PointCloudCost(pc, dev, comm=comm))
    _ = sol.primal_cost
    torch.cuda.synchronize()
    e2e = max_over_ranks(time.perf_counter() - t0, world)
    h2d, d2h = TELEMETRY.h2d, TELEMETRY.d2h
    if not args.no_extras:
        out_extras["d2_replicas"] = d2_replicas(dev, rank, world)
    val = statistics.mean(times)
    return {
        "metric": METRIC_D4.format(n=n), "value": val, "unit": "s", "n_gpus": world,
        "steps": args.steps, "warmup": min(args.warmup, 1), "ms_per_step": val * 1e3,
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded U[0,1)^3 point clouds, uniform marginals)",
        "config": config_d4(n, world),
        "e2e": {"value": e2e, "unit": "s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h)},
        "gpu_launches": launches,
        "gpu_launches_per_step": launches / max(args.steps, 1),
        "solve": rec, "per_step_s": times, "clocks": clocks.summary(),
        "collectives": {"backend": _BACKEND, "ranks": world,
                        "per_solve": rec.get("collectives")},
        "extras": out_extras,
    }


def d2_replicas(dev, rank, world):
    """D2 on every rank independently (each its own seed)."""
    import torch

    import paper_2504_02067_b200 as ot
    p = ot.workload(f"grid:64:l2sq:{rank}")
    dp = ot.Problem(C=torch.from_numpy(p.C).to(dev), r=p.r, c=p.c)
    ot.mdot(dp, D2["gamma_i"], D2["gamma_f"])
    torch.cuda.synchronize()
    barrier(world)
    t0 = time.perf_counter()
    ot.mdot(dp, D2["gamma_i"], D2["gamma_f"])
    torch.cuda.synchronize()
    dt = max_over_ranks(time.perf_counter() - t0, world)
    return {"s_per_solve_max_over_ranks": dt, "solves_per_s_total": world / dt}


# ---------------------------------------------------------------------------
# reference arm / CPU baseline: the oracle port, complete solves
# ---------------------------------------------------------------------------
def oracle_full_solves(max_solves, budget_s):
    """Complete solves of the D2 workload by the oracle port of otnewton.mdot
    (bit-identical to the reference), BLAS threads and the oracle's row slabs on
    all host cores.  Runs solves until `max_solves` or until `budget_s` of
    solving has elapsed (at least one).  Returns (seconds per solve, count,
    cores, details)."""
    cores = os.cpu_count() or 1
    from oracle import otn_oracle as orc
    from paper_2504_02067_b200 import problems
    orc.set_threads(cores)
    d1 = problems.workload("pts:1024:2:0")
    t0 = time.perf_counter()
    orc.mdot(d1.C, d1.r, d1.c, 2.0 ** 10, 2.0 ** 10)      # warm-up: BLAS / page-in (untimed)
    warm_s = time.perf_counter() - t0
    prob = problems.workload(D2["spec"])
    times, run = [], None
    while len(times) < max(1, max_solves):
        t0 = time.perf_counter()
        run = orc.mdot(prob.C, prob.r, prob.c, D2["gamma_i"], D2["gamma_f"], p=D2["p"],
                       q_init=D2["q_init"])
        times.append(time.perf_counter() - t0)
        if sum(times) >= budget_s:
            break
    st = run.state
    st.r, st.c = prob.r, prob.c
    detail = {"stages": len(run.stages), "cg_iters": sum(pr.cg_iters for *_, pr in run.stages),
              "true_marginal_err": st.gnorm(), "per_solve_s": times,
              "warmup_s_d1": warm_s}
    return statistics.mean(times), len(times), cores, detail


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(budget_s):
    os.environ.setdefault("OPENBLAS_NUM_THREADS", str(os.cpu_count()))
    v, k, cores, detail = oracle_full_solves(1, budget_s)
    return {"value": v, "unit": "s", "cores": cores, "kind": "port",
            "sample": f"{k} complete D2 solve(s) of the oracle port of otnewton.mdot "
                      "(bit-identical to the reference: tests/test_oracle_pin.py), OpenBLAS "
                      f"and the 256-row slabs on {cores} threads; {cpu_model()}",
            "detail": detail}


def run_reference(args, world):
    os.environ.setdefault("OPENBLAS_NUM_THREADS", str(os.cpu_count()))
    if world > 1:
        return {"impl": "reference", "unavailable":
                "the N>1 workload is D4 (n=65536): the reference stores 4 dense n x n float64 "
                "arrays (137 GB) and cannot run it (SURVEY 8(c))"}
    v, k, cores, detail = oracle_full_solves(args.steps, args.ref_budget)
    cb = {"value": v, "unit": "s", "cores": cores, "kind": "port",
          "sample": f"{k} complete D2 solve(s) timed (oracle port of otnewton.mdot, "
                    "bit-identical to the reference), OpenBLAS and 256-row slabs on "
                    f"{cores} threads; {cpu_model()}",
          "detail": detail}
    return {
        "metric": METRIC, "value": v, "unit": "s", "n_gpus": world, "steps": k,
        "warmup": 1, "ms_per_step": v * 1e3, "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded 64x64 grid cost + smooth-random marginals, reference generators)",
        "config": dict(CONFIG_D2), "impl": "reference",
        "steps_requested": args.steps, "warmup_note": "one untimed n=1024 solve",
        "cpu_baseline": cb,
        "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


# ---------------------------------------------------------------------------
# distributed plumbing
# ---------------------------------------------------------------------------
_PG = None


# BENCH_DIST_BACKEND=gloo + BENCH_DEVICE=0: every rank on cuda:0 with host-staged
# allreduces -- only for the process-group test of this script on a one-GPU
# box (tests/test_gpu_bench_sharded.py); a real run is one rank per GPU on NCCL.
_BACKEND = os.environ.get("BENCH_DIST_BACKEND", "nccl")


def local_device():
    return int(os.environ.get("BENCH_DEVICE", os.environ.get("LOCAL_RANK", 0)))


def init_dist(args):
    global _PG
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1 and args.impl != "reference":
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_device())
        dist.init_process_group(_BACKEND)
        _PG = dist
    return rank, world


def barrier(world):
    if world > 1 and _PG is not None:
        _PG.barrier()


def max_over_ranks(x, world):
    if world > 1 and _PG is not None:
        import torch
        t = torch.tensor([x], dtype=torch.float64,
                         device="cuda" if _BACKEND == "nccl" else "cpu")
        _PG.all_reduce(t, op=_PG.ReduceOp.MAX)
        return float(t.item())
    return x


def relaunch_under_torchrun(args):
    """`python bench.py --gpus N` (N > 1) without torchrun: re-execute this
    script with one rank per GPU (NCCL over NVLink), rendezvous on 127.0.0.1."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--cpu-budget", type=float, default=30.0,
                    help="seconds of oracle solving for cpu_baseline (at least one solve)")
    ap.add_argument("--ref-budget", type=float, default=150.0,
                    help="--impl reference: stop after this many seconds of solves")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--d4-n", type=int, default=65536)
    ap.add_argument("--sharded", choices=["d4", "d5"], default="d4",
                    help="N > 1 workload: D4 (n = 65536, --d4-n) or D5 (n = 2^20)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 0)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_under_torchrun(args))
    rank, world = init_dist(args)
    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args, world)))
        return
    import torch
    dev = torch.device("cuda", local_device())
    torch.cuda.set_device(dev)
    if world == 1:
        out = run_d2(args, dev)
        if not args.no_extras:
            out["extras"] = run_extras(args, dev)
        if not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline(args.cpu_budget)
    else:
        out = run_sharded(args, rank, world, dev)
    if rank == 0:
        print(json.dumps(out))
    if world > 1 and _PG is not None:
        _PG.destroy_process_group()


if __name__ == "__main__":
    main()
