#!/usr/bin/env python3
"""Benchmark of the B200 SEM Jacobi-PCG hot path (arxiv 2503.02134) -- driver contract.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--policy mixed]

Workload (BASELINE.json configs[1], the metric's configuration): 16x16x16 undeformed
hex elements on [0,1]^3, p = 7 (2,097,152 local DOF), Dirichlet faces, uniform[-1,1]
RHS from seed 0, Jacobi-PCG to rtol 1e-8, mixed policy (fp32 vectors/Ax, fp64 GS,
dots and Jacobi).  One step = one complete nb_cg solve (all SURVEY.md §8(a) per-iteration
rows a5..a12; setup a1..a4 is done once before timing, like Nekbone's solve time).
value = local DOF x iterations / solve time, summed over ranks / max-over-ranks time.

Multi-GPU (--mode replicas, default): the single-GPU solve is replicated (independent problems
per rank, no data-path collective) -> "scaling": "weak".  --mode slab: ONE box of 16x16x(16 N)
elements split into N z-slabs, one per rank/GPU (configs[1] per GPU, weak scaling), solved by
the multi-rank megakernel that reads the neighbour slabs' interface layers over NVLink peer
memory (CUDA IPC) and reduces the dot products across ranks in-kernel;
with one GPU, --mode slab --slabs K runs K slabs of one box in one launch (the emulation the
multi-rank path is tested with).  DESIGN.md §7.
--impl reference times the oracle (plain C, one core) on bounded samples of the same
workload (the tier's reference arm).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOAD = {"workload": "configs[1]: box 16x16x16 undeformed, p=7, uniform RHS seed 0, Jacobi-PCG rtol 1e-8",
            "nel": [16, 16, 16], "p": 7, "deform": 0.0, "rtol": 1e-8, "rhs": "uniform seed 0"}
METRIC = "DOF·iter/s and time-to-1e-8 residual (fp64 vs mixed); Ax/dssum HBM GB/s"
UNIT = "DOF·iter/s"
POLICIES = {"fp64": 0, "fp32": 1, "mixed": 2}
# Algorithmic bytes per local DOF moved by each kernel, by policy: every
# vector, g and dinv entry once at its policy precision; c and the mask are analytic.
#   K1 (k_ax, CG):  z, p_old, x, 6 g  ->  p, x, w
#   K2 (k_upd):     w, r, dinv        ->  r, z      (gather re-reads are not algorithmic)
SV = {0: 8, 1: 4, 2: 4}          # vector entry
SJ = {0: 8, 1: 4, 2: 8}          # dinv entry
K1_BYTES = {p: 3 * SV[p] + 6 * SV[p] + 3 * SV[p] for p in SV}
K2_BYTES = {p: 2 * SV[p] + SJ[p] + 2 * SV[p] for p in SV}
AX_BYTES = {p: 2 * SV[p] + 6 * SV[p] for p in SV}     # standalone local Ax: u + 6 g -> w


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, torch copy burst)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class Clocks:
    """nvidia-smi sampler (clocks + throttle reasons), started before the timed region and
    filtered to the samples whose timestamps fall inside it."""
    Q = ("timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.t0 = self.t1 = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "10"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.5)   # let the sampler come up before the timed region
        except Exception:
            self.proc = None
        self.t0 = time.time()

    def mark_end(self):
        self.t1 = time.time()

    def stop(self):
        if not self.proc:
            return None
        if self.t1 is None:
            self.t1 = time.time()
        time.sleep(0.05)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        import datetime
        rows = []
        for r in out.strip().splitlines():
            f = [x.strip() for x in r.split(",")]
            if len(f) < 7:
                continue
            try:
                ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
            except ValueError:
                continue
            rows.append((ts, f[1:]))
        inside = [f for ts, f in rows if self.t0 - 0.01 <= ts <= self.t1 + 0.01] or [f for _, f in rows[-3:]]
        if not inside:
            return None
        sm = [float(f[0]) for f in inside if f[0].replace(".", "").isdigit()]
        mx = [float(f[1]) for f in inside if f[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for f in inside for i in range(4) if "Active" in f[2 + i] and "Not" not in f[2 + i]})
        loaded = [s for s in sm if mx and s > 0.3 * max(mx)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(inside),
                "samples_total": len(rows)}


def dist_init(n_gpus):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        import torch
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    return rank, world, local


def barrier_sync(world):
    import torch
    torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()


def _reduce(v, world, op, device):
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=op)
    return float(t.item())


def max_over_ranks(v, world, device="cuda"):
    import torch.distributed as dist
    return _reduce(v, world, dist.ReduceOp.MAX if world > 1 else None, device)


def sum_over_ranks(v, world, device="cuda"):
    import torch.distributed as dist
    return _reduce(v, world, dist.ReduceOp.SUM if world > 1 else None, device)


def aggregate(dof_iters_local, t_local, world, device="cuda"):
    """Whole-job throughput: DOF*iterations summed over ranks / the slowest rank's time."""
    t_max = max_over_ranks(t_local, world, device)
    return sum_over_ranks(float(dof_iters_local), world, device) / t_max, t_max


# ---------------------------------------------------------------------------- CPU oracle legs
def oracle_sample(iters: int, policy: str = "mixed"):
    """Time the oracle (as it stands, one core) on `iters` CG iterations of configs[1]."""
    import oracle
    nel, p = WORKLOAD["nel"], WORKLOAD["p"]
    t0 = time.perf_counter()
    m = oracle.Mesh(*nel, p, deform=0.0, seed=0)
    b = m.rhs(oracle.RHS_UNIFORM, seed=0)
    t_setup = time.perf_counter() - t0
    t0 = time.perf_counter()
    _, _, rep = m.cg(b, {"fp64": oracle.FP64, "fp32": oracle.FP32, "mixed": oracle.MIXED}[policy],
                     max_iter=iters, rtol=0.0)
    dt = time.perf_counter() - t0
    return m.n_local * rep.iterations / dt, dt, t_setup, rep.iterations, m.n_local


def run_oracle_timing(args):
    """--oracle-timing: SURVEY.md §8(d) "Oracle timing" on this box's host (one core, the plain C
    oracle as it stands): per config setup, one Ax, one dssum and the CG rate; full solves for
    configs[0..1]; configs[2..3] from 5 iterations, extrapolated to the GPU's iteration count
    measured in the same run (labelled as such).  Prints one JSON document."""
    import platform

    import oracle
    import paper_2503_02134_b200 as nb
    cases = [("configs[0]", (2, 2, 2), 7, 0.0, 0, 0.0, ["fp64"], True, 100),
             ("configs[1]", (16, 16, 16), 7, 0.0, 0, 1e-8, ["fp64", "fp32", "mixed"], True, 4000),
             ("configs[2]", (32, 32, 32), 9, 0.1, 0, 1e-8, ["mixed", "fp64"], False, 8000),
             ("configs[3]", (64, 32, 32), 11, 0.0, 1, 1e-10, ["fp64", "mixed"], False, 8000)]
    opol = {"fp64": oracle.FP64, "fp32": oracle.FP32, "mixed": oracle.MIXED}
    model = ""
    try:
        txt = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        model = next((ln.split(":", 1)[1].strip() for ln in txt.splitlines() if ln.startswith("Model name")), "")
    except Exception:
        pass
    out = {"host": {"cpu_model": model or platform.processor(), "nproc": os.cpu_count(), "threads_used": 1,
                    "oracle_cflags": " ".join(oracle.CFLAGS)}, "cases": []}
    for name, nel, p, d, kind, rtol, pols, full, max_iter in cases:
        if args.oracle_max_dof and nel[0] * nel[1] * nel[2] * (p + 1) ** 3 > args.oracle_max_dof:
            continue
        t0 = time.perf_counter()
        m = oracle.Mesh(*nel, p, deform=d, seed=0)
        rec = {"config": name, "nel": nel, "p": p, "deform": d, "n_local": m.n_local,
               "setup_s": time.perf_counter() - t0}
        b = m.rhs(oracle.RHS_UNIFORM if kind == 0 else oracle.RHS_MANUFACTURED, noise=1e-3, seed=0)
        for pol in pols:
            t0 = time.perf_counter()
            m.ax(b, opol[pol])
            rec[f"ax_s_{pol}"] = time.perf_counter() - t0
            t0 = time.perf_counter()
            m.dssum(b, opol[pol])
            rec[f"dssum_s_{pol}"] = time.perf_counter() - t0
            if full:
                t0 = time.perf_counter()
                _, _, r = m.cg(b, opol[pol], max_iter=max_iter, rtol=rtol)
                dt = time.perf_counter() - t0
                rec[f"solve_{pol}"] = {"iterations": r.iterations, "status": r.status, "seconds": dt,
                                       "dof_iter_per_s": m.n_local * r.iterations / dt}
            else:
                g = nb.Mesh(*nel, p, deform=d, seed=0)
                gb = g.rhs(POLICIES[pol], nb.NB_RHS_UNIFORM if kind == 0 else nb.NB_RHS_MANUFACTURED, noise=1e-3, seed=0)
                _, gr = g.cg(gb, POLICIES[pol], max_iter=max_iter, rtol=rtol)
                g.close()
                t0 = time.perf_counter()
                m.cg(b, opol[pol], max_iter=5, rtol=0.0)
                dt = (time.perf_counter() - t0) / 5
                rec[f"solve_{pol}"] = {"seconds_per_iteration": dt, "dof_iter_per_s": m.n_local / dt,
                                       "gpu_iterations": gr.iterations, "gpu_solve_ms": gr.solve_ms,
                                       "extrapolated_seconds_to_rtol": dt * gr.iterations,
                                       "note": "extrapolated: 5 oracle iterations x the GPU's iteration count"}
            print(json.dumps({"progress": name, "policy": pol}), file=sys.stderr, flush=True)
        out["cases"].append(rec)
        del m
    print(json.dumps(out, indent=1), flush=True)
    return 0


def run_reference(args):
    rank, world, _ = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), 0
    if rank != 0:
        return 0
    iters = args.ref_iters
    for _ in range(args.warmup):
        oracle_sample(max(1, iters // 4), args.policy)
    vals, times = [], []
    for _ in range(args.steps):
        v, dt, _, it, nl = oracle_sample(iters, args.policy)
        vals.append(v)
        times.append(dt)
    total = sum(times)
    value = nl * iters * args.steps / total
    sample = (f"{iters} CG iterations ({args.policy}, rtol=0) of configs[1] per step, mesh setup excluded; "
              f"oracle plain C -O2 single-threaded")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32+f64 (mixed)",
            "data": "synthetic", "config": dict(WORKLOAD, policy=args.policy),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------- GPU arm
def time_launches(fn, n, stream):
    """Device time (ms) of one fn() launch, median over n.  Each launch is bracketed by CUDA
    events queued behind a short GPU sleep, so the host work of the ctypes call (argument checks,
    pointer queries) is absorbed by the sleep and the events time the kernel alone."""
    import statistics

    import torch
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(2_000_000)        # ~1 ms of GPU work ahead of the events
        a.record(stream)
        fn()
        b.record(stream)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def run_ours(args):
    import torch
    import paper_2503_02134_b200 as nb

    rank, world, local = dist_init(args.gpus)
    dev = local if world > 1 else 0
    torch.cuda.set_device(dev)
    pol = POLICIES[args.policy]
    nel, p = list(WORKLOAD["nel"]), WORKLOAD["p"]
    slab = args.mode == "slab"
    group = []
    if slab:
        args.quick = True        # the per-policy table / companion run on rank 0 alone
        if world > 1:
            nel[2] = WORKLOAD["nel"][2] * world          # configs[1] per GPU, stacked along z
            mesh = nb.Mesh(*nel, p, deform=0.0, seed=0, device=dev, slab=nb.slab_bounds(nel[2], world, rank))
            nb.peer_attach_dist(mesh, pol)
        else:
            K = args.slabs
            group = [nb.Mesh(*nel, p, deform=0.0, seed=0, device=dev, slab=nb.slab_bounds(nel[2], K, r))
                     for r in range(K)]
            mesh = group[0]
    else:
        mesh = nb.Mesh(*nel, p, deform=0.0, seed=0, device=dev)
    NL = sum(m.n_local for m in group) if group else mesh.n_local
    info = mesh.info
    b = mesh.rhs(pol, nb.NB_RHS_UNIFORM, seed=0)
    x = mesh.empty(pol)
    gb = [m.rhs(pol, nb.NB_RHS_UNIFORM, seed=0) for m in group]
    gx = [m.empty(pol) for m in group]
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{dev}")
    max_iter = 4000
    st = torch.cuda.current_stream()

    def solve():
        if group:
            reps, _ = nb.nb_cg_group([m.h for m in group], gb, gx, pol, max_iter, WORKLOAD["rtol"], history=False)
            return reps[0]
        rep, _ = nb.nb_cg(mesh.h, b, x, pol, max_iter, WORKLOAD["rtol"], history=False)
        return rep

    for _ in range(max(3, args.warmup)):
        solve()
    clocks = Clocks(dev)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    iters, launches, statuses, lib_ms = [], 0, set(), []
    barrier_sync(world)
    clocks.start()
    for s in range(args.steps):
        flush.zero_()                          # L2 flush between steps (outside the events)
        ev[s][0].record(st)
        rep = solve()
        ev[s][1].record(st)
        iters.append(rep.iterations)
        statuses.add(rep.status)
        launches += rep.kernel_launches
        lib_ms.append(rep.solve_ms)
    barrier_sync(world)
    clocks.mark_end()
    ck = clocks.stop()
    step_ms = [a.elapsed_time(b2) for a, b2 in ev]
    t_local = sum(step_ms) / 1e3
    value, t_max = aggregate(NL * sum(iters), t_local, world)

    # per-phase device time of the same solve: the megakernel's block 0 stamps %globaltimer after
    # every grid barrier (nb_cg_report k_ax_ms / k_upd_ms)
    kt = [solve() for _ in range(max(1, min(args.steps, 3)))]
    it_k = sum(r.iterations for r in kt)
    k1_ms = sum(r.k_ax_ms for r in kt) / it_k
    k2_ms = sum(r.k_upd_ms for r in kt) / it_k
    peak, peak_src = load_peaks()
    vs = SV[pol]
    k1_bytes = K1_BYTES[pol] * NL
    k2_bytes = K2_BYTES[pol] * NL
    # standalone operator pieces (the metric's "Ax/dssum HBM GB/s"): local Ax and the CSR dssum
    u = mesh.rhs(pol, nb.NB_RHS_UNIFORM, seed=5)
    wv = mesh.empty(pol)
    ax_ms = time_launches(lambda: nb.nb_ax(mesh.h, pol, u, wv, nb.NB_AX_LOCAL), 50, st)
    gs_ms = time_launches(lambda: nb.nb_dssum(mesh.h, pol, nb.NB_GS_CONSISTENT, wv), 50, st)
    gs_bytes = info.n_shared_copies * (2 * vs + 4) + (info.n_shared_global + 1) * 4
    # DRAM traffic of the solve kernel from the committed ncu capture (profiles/), per iteration
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            traffic = json.load(f).get(f"{args.policy}_configs1_dram_bytes_per_iteration")
    except Exception:
        pass

    # e2e: the public host-buffer call, pinned host b/x, copies inside the timed region
    e2e = None
    if not group:
        bh = b.cpu().pin_memory()
        xh = torch.empty_like(bh).pin_memory()
        e2e_t, e2e_it = 0.0, 0
        barrier_sync(world)
        for s in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rep, _ = nb.nb_cg_host(mesh.h, bh, xh, pol, max_iter, WORKLOAD["rtol"])
            e2e_t += time.perf_counter() - t0
            e2e_it += rep.iterations
        e2e_t = max_over_ranks(e2e_t, world)
        e2e_val = sum_over_ranks(float(NL * e2e_it), world) / e2e_t
        e2e = {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": NL * SV[pol], "d2h_bytes_per_step": NL * SV[pol]}

    # time-to-1e-8 for every policy (reported next to the headline; not the timed region)
    ttr = {}
    if rank == 0 and not args.quick:
        for name, pp in POLICIES.items():
            bb = mesh.rhs(pp, nb.NB_RHS_UNIFORM, seed=0)
            xx = mesh.empty(pp)
            reps = []
            for _ in range(3):
                flush.zero_()
                r, _ = nb.nb_cg(mesh.h, bb, xx, pp, max_iter, WORKLOAD["rtol"], history=False)
                reps.append(r)
            rk, _ = nb.nb_cg(mesh.h, bb, xx, pp, max_iter, WORKLOAD["rtol"], history=False)
            n_it = rk.iterations
            tmed = statistics.median(r.solve_ms for r in reps)
            ttr[name] = {"iterations": reps[-1].iterations, "status": reps[-1].status, "time_ms": tmed,
                         "dof_iter_per_s": NL * reps[-1].iterations / (tmed * 1e-3),
                         "k1_us": 1e3 * rk.k_ax_ms / n_it, "k2_us": 1e3 * rk.k_upd_ms / n_it,
                         "k1_alg_GBps": K1_BYTES[pp] * NL / (rk.k_ax_ms * 1e-3 / n_it) / 1e9,
                         "k2_alg_GBps": K2_BYTES[pp] * NL / (rk.k_upd_ms * 1e-3 / n_it) / 1e9}
        ttr["speedup_fp64_over_mixed_time"] = ttr["fp64"]["time_ms"] / ttr["mixed"]["time_ms"]

    # HBM-bound companion point: configs[1]'s working set (~100 MB mixed) fits in the 126 MB L2,
    # so its phase GB/s are not an HBM measurement.  configs[2] (32^3, p=9, deformed, 32.8M DOF,
    # ~1.6 GB per mixed iteration) is: fixed 100 iterations, phase times from the same stamps.
    large = None
    if rank == 0 and not args.quick and not args.no_large:
        lm = nb.Mesh(32, 32, 32, 9, deform=0.1, seed=0, device=dev)
        lnl = lm.n_local
        large = {"workload": "configs[2]: box 32x32x32 deformed 0.1, p=9, uniform RHS seed 0, 100 fixed iterations"}
        for name, pp in (("mixed", POLICIES["mixed"]), ("fp64", POLICIES["fp64"])):
            lb = lm.rhs(pp, nb.NB_RHS_UNIFORM, seed=0)
            lx = lm.empty(pp)
            nb.nb_cg(lm.h, lb, lx, pp, 100, 0.0, history=False)
            flush.zero_()
            r, _ = nb.nb_cg(lm.h, lb, lx, pp, 100, 0.0, history=False)
            a_us, b_us = 1e3 * r.k_ax_ms / r.iterations, 1e3 * r.k_upd_ms / r.iterations
            large[name] = {"us_per_iteration": 1e3 * r.solve_ms / r.iterations,
                           "dof_iter_per_s": lnl * r.iterations / (r.solve_ms * 1e-3),
                           "phaseA_us": a_us, "phaseA_GBps": K1_BYTES[pp] * lnl / (a_us * 1e-6) / 1e9,
                           "phaseA_frac": K1_BYTES[pp] * lnl / (a_us * 1e-6) / 1e9 / load_peaks()[0],
                           "phaseB_us": b_us, "phaseB_GBps": K2_BYTES[pp] * lnl / (b_us * 1e-6) / 1e9,
                           "phaseB_frac": K2_BYTES[pp] * lnl / (b_us * 1e-6) / 1e9 / load_peaks()[0]}
            del lb, lx
        lm.close()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        v, dt, _, it, _ = oracle_sample(args.cpu_iters, args.policy)
        cpu = {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"{it} CG iterations ({args.policy}, rtol=0) of configs[1], setup excluded, "
                         f"{dt:.1f} s on one host core"}

    if rank == 0:
        ms_per_step = 1e3 * t_max / args.steps
        k1_ach = k1_bytes / (k1_ms * 1e-3) / 1e9
        k2_ach = k2_bytes / (k2_ms * 1e-3) / 1e9
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": max(3, args.warmup), "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": {0: "f64", 1: "f32", 2: "f32+f64 (mixed)"}[pol],
                "data": "synthetic",
                "config": dict(WORKLOAD, policy=args.policy, iterations=iters[0], status=sorted(statuses),
                               n_local=NL, l2="256 MiB write between steps (outside the step events)",
                               parallelism=(f"z-slabs over {world} GPUs (NVLink peer memory)" if slab and world > 1
                                            else f"{len(group)} z-slabs in one launch on one GPU" if group
                                            else "replicas" if world > 1 else "single GPU"),
                               **({"nel": nel} if slab else {})),
                "time_to_rtol_ms": ms_per_step,
                "step_ms": {"events_around_call": step_ms, "library_device_ms": lib_ms},
                "roofline": {"bound": "hbm",
                             "kernel": "k_cg_mega phase A (Jacobi p-update + deferred x update + local Ax + mask + pap), "
                                       "per CG iteration",
                             "achieved": k1_ach, "peak": peak, "unit": "GB/s", "frac": k1_ach / peak,
                             "traffic": traffic, "traffic_note": "ncu dram read+write of the whole megakernel "
                                                                 "(both phases) per iteration, profiles/",
                             "alg_bytes_per_iteration": k1_bytes + k2_bytes, "peak_source": peak_src,
                             "alg_bytes_per_launch": k1_bytes, "avg_launch_us": 1e3 * k1_ms,
                             "share_of_iteration": k1_ms / (k1_ms + k2_ms)},
                "kernels": {
                    "phaseA_ax": {"avg_us": 1e3 * k1_ms, "alg_bytes": k1_bytes, "GBps": k1_ach, "frac": k1_ach / peak},
                    "phaseB_gather_update": {"avg_us": 1e3 * k2_ms, "alg_bytes": k2_bytes, "GBps": k2_ach,
                                             "frac": k2_ach / peak},
                    "ax_local": {"avg_us": 1e3 * ax_ms, "alg_bytes": AX_BYTES[pol] * NL,
                                 "GBps": AX_BYTES[pol] * NL / (ax_ms * 1e-3) / 1e9,
                                 "frac": AX_BYTES[pol] * NL / (ax_ms * 1e-3) / 1e9 / peak},
                    "dssum_csr": {"note": "standalone nb_dssum (CSR segments; setup/API kernel, not on the solve "
                                          "path: the solve gathers in phase B)",
                                  "avg_us": 1e3 * gs_ms, "alg_bytes": gs_bytes,
                                  "GBps": gs_bytes / (gs_ms * 1e-3) / 1e9,
                                  "frac": gs_bytes / (gs_ms * 1e-3) / 1e9 / peak}},
                "e2e": e2e,
                "gpu_launches": launches, "clocks": ck, "cpu_baseline": cpu, "policies": ttr,
                "hbm_bound_companion": large}
        print(json.dumps(line), flush=True)
    for m in group or [mesh]:
        m.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--policy", default="mixed", choices=list(POLICIES))
    ap.add_argument("--cpu-iters", type=int, default=60)
    ap.add_argument("--ref-iters", type=int, default=20)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--quick", action="store_true", help="skip the per-policy table and the large companion")
    ap.add_argument("--no-large", action="store_true", help="skip the HBM-bound configs[2] companion point")
    ap.add_argument("--mode", default="replicas", choices=["replicas", "slab"],
                    help="N>1: independent replicas, or one box split in z-slabs over the GPUs")
    ap.add_argument("--slabs", type=int, default=2, help="--mode slab on one GPU: slabs in the launch")
    ap.add_argument("--oracle-timing", action="store_true",
                    help="instead of the bench line: time the CPU oracle per config (SURVEY §8(d))")
    ap.add_argument("--oracle-max-dof", type=float, default=0, help="--oracle-timing: skip larger configs")
    args = ap.parse_args()
    if args.oracle_timing:
        return run_oracle_timing(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
