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
ROOF_ITERS = 200                                       # fixed iterations of the configs[2] roofline launch


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


def survey_bytes(pol, info):
    """SURVEY.md §8(d) algorithmic bytes per local DOF and CG iteration of the fused iteration
    K1 + K2 + K3 (every vector, g and dinv entry at its policy precision, c as a vector, int32 CSR
    indices for the shared copies), evaluated with the mesh's own shared fractions."""
    sv, sj = SV[pol], SJ[pol]
    NL = info.n_local
    f_sh, f_g = info.n_shared_copies / NL, info.n_shared_global / NL
    k1 = 2 * sv + sj + 6 * sv + 2 * sv          # K1: r, dinv, p_old, 6 g -> p, w          (88 / 48 / 44)
    k2 = f_sh * (2 * sv + 4) + f_g * 4 + f_g * sv   # K2: dssum (copies + int32 idx + offsets) + shared pap
    k3 = 6 * sv + sj + sv                       # K3: x, p, r, w, dinv, c -> x, r          (64 / 36 / 32)
    return k1 + k2 + k3


def impl_bytes(pol):
    """Bytes per local DOF and iteration this implementation moves: phase A
    z, p_old, x, 6 g -> p, x, w; phase B w, r, dinv -> r, z; c and the mask are analytic."""
    return K1_BYTES[pol] + K2_BYTES[pol]


def roofline_point(nb, args, flush, dev, cfg_name="configs[2]"):
    """The HBM-bound roofline measurement: the CG megakernel on configs[2] (32^3 deformed, p = 9,
    32.8M local DOF, ~2.4 GB/iteration of mixed traffic: 19x the 126 MB L2), `ROOF_ITERS` fixed
    iterations in one launch, timed with CUDA events on the launching stream; per-phase time from
    the kernel's own %globaltimer stamps.  DRAM traffic of the same launch from the committed ncu
    capture (profiles/r2_ncu_roofline.json, tools/ncu_roofline.sh)."""
    import torch
    st = torch.cuda.current_stream()
    m = nb.Mesh(32, 32, 32, 9, deform=0.1, seed=0, device=dev)
    info, NL = m.info, m.n_local
    peak, peak_src = load_peaks()
    traffic = {}
    try:
        with open(os.path.join(ROOT, "profiles", "r2_ncu_roofline.json")) as f:
            traffic = json.load(f)
    except Exception:
        pass
    out = {"workload": "configs[2]: box 32x32x32 deformed 0.1, p=9, uniform RHS seed 0, "
                       f"{ROOF_ITERS} fixed CG iterations in one k_cg_mega launch", "n_local": NL,
           "l2": "working set 19x the L2 (mixed); 256 MiB flush before each launch", "policies": {}}
    for name in args.roof_policies:
        pol = POLICIES[name]
        b = m.rhs(pol, nb.NB_RHS_UNIFORM, seed=0)
        x = m.empty(pol)
        nb.nb_cg(m.h, b, x, pol, ROOF_ITERS, 0.0, history=False)      # warm-up (and the ncu target)
        if args.roofline_only:
            break
        best = None
        for _ in range(3):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            rep, _ = nb.nb_cg(m.h, b, x, pol, ROOF_ITERS, 0.0, history=False)
            e1.record(st)
            e1.synchronize()
            ms = e0.elapsed_time(e1)
            if best is None or ms < best[0]:
                best = (ms, rep)
        ms, rep = best
        it = rep.iterations
        sb, ib = survey_bytes(pol, info), impl_bytes(pol)
        a_us, b_us = 1e3 * rep.k_ax_ms / it, 1e3 * rep.k_upd_ms / it
        tr = traffic.get(f"configs2_{name}")
        rec = {"launch_ms": ms, "iterations": it, "dof_iter_per_s": NL * it / (ms * 1e-3),
               "survey_bytes_per_dof_iter": sb, "impl_bytes_per_dof_iter": ib,
               "achieved_GBps": sb * NL * it / (ms * 1e-3) / 1e9,
               "achieved_impl_GBps": ib * NL * it / (ms * 1e-3) / 1e9,
               "phaseA_us": a_us, "phaseB_us": b_us,
               "phaseA_GBps": K1_BYTES[pol] * NL / (a_us * 1e-6) / 1e9,
               "phaseB_GBps": K2_BYTES[pol] * NL / (b_us * 1e-6) / 1e9}
        rec["phaseA_frac"] = rec["phaseA_GBps"] / peak
        rec["phaseB_frac"] = rec["phaseB_GBps"] / peak
        if tr:
            rec["ncu_dram_bytes_per_iteration"] = tr.get("dram_bytes_per_iteration")
            rec["ncu_dram_bytes_per_launch"] = tr.get("dram_bytes_per_iteration", 0) * it
            rec["ncu_dram_GBps_at_this_launch_time"] = rec["ncu_dram_bytes_per_launch"] / (ms * 1e-3) / 1e9
            for ph in ("A", "B"):
                if tr.get(f"phase{ph}_dram_bytes_per_iteration"):
                    rec[f"ncu_phase{ph}_dram_bytes_per_iteration"] = tr[f"phase{ph}_dram_bytes_per_iteration"]
                    us = a_us if ph == "A" else b_us
                    rec[f"ncu_phase{ph}_dram_frac"] = tr[f"phase{ph}_dram_bytes_per_iteration"] / (us * 1e-6) / 1e9 / peak
            rec["ncu_source"] = tr.get("source")
        # standalone operators at this HBM-bound size (the metric's "Ax/dssum HBM GB/s")
        u = m.rhs(pol, nb.NB_RHS_UNIFORM, seed=5)
        w = m.empty(pol)
        ax_ms = time_launches(lambda: nb.nb_ax(m.h, pol, u, w, nb.NB_AX_LOCAL), 10, st)
        gs_ms = time_launches(lambda: nb.nb_dssum(m.h, pol, nb.NB_GS_CONSISTENT, w), 10, st)
        gs_bytes = info.n_shared_copies * (2 * SV[pol] + 4) + (info.n_shared_global + 1) * 4
        rec["nb_ax_local"] = {"us": 1e3 * ax_ms, "alg_bytes": AX_BYTES[pol] * NL,
                              "GBps": AX_BYTES[pol] * NL / (ax_ms * 1e-3) / 1e9,
                              "frac": AX_BYTES[pol] * NL / (ax_ms * 1e-3) / 1e9 / peak}
        rec["nb_dssum"] = {"us": 1e3 * gs_ms, "alg_bytes": gs_bytes, "GBps": gs_bytes / (gs_ms * 1e-3) / 1e9,
                           "frac": gs_bytes / (gs_ms * 1e-3) / 1e9 / peak}
        out["policies"][name] = rec
        del b, x, u, w
    m.close()
    torch.cuda.empty_cache()
    return out, peak, peak_src


def spawn(args):
    """--gpus N without a torchrun environment: relaunch this script under torch.distributed.run
    with N local ranks (127.0.0.1 rendezvous) and pass its output through."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def run_dry(args):
    """--dry-run: the multi-rank plumbing only (CPU, gloo): every rank joins, rank 0 prints the
    line's shape with n_gpus = world size.  Used by the CPU tests of --gpus N spawning."""
    import torch.distributed as dist
    rank, world = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1:
        dist.init_process_group("gloo")
        dist.barrier()
    mode = args.mode or ("slab" if world > 1 else "single")
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "mode": mode,
                          "parallelism": parallelism(mode, world, 0)}), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def parallelism(mode, world, nslab_local):
    if mode == "slab" and world > 1:
        return f"z-slabs over {world} GPUs (NVLink peer memory, in-kernel exchange)"
    if nslab_local:
        return f"{nslab_local} z-slabs in one launch on one GPU"
    if world > 1:
        return f"replicas over {world} GPUs"
    return "single GPU"


def ae_mae(h_m, h_d):
    """PAPER.md:489-497 (Sec. 5.1.1): AE_i = |r_m,i - r_d,i| of the residual histories of the mixed
    and the double-precision solve, MAE = mean over the common iterations."""
    import numpy as np
    n = min(len(h_m), len(h_d))
    ae = np.abs(np.asarray(h_m[1:n]) - np.asarray(h_d[1:n]))
    return {"iterations_compared": int(n - 1), "MAE": float(ae.mean()) if ae.size else 0.0,
            "AE_max": float(ae.max()) if ae.size else 0.0, "AE_final": float(ae[-1]) if ae.size else 0.0,
            "AE_at": {str(k): float(ae[k - 1]) for k in (1, 10, 100, 300) if k <= ae.size}}


def run_ours(args):
    import torch
    import paper_2503_02134_b200 as nb

    rank, world, local = dist_init(args.gpus)
    dev = local if world > 1 else 0
    torch.cuda.set_device(dev)
    pol = POLICIES[args.policy]
    nel, p = list(WORKLOAD["nel"]), WORKLOAD["p"]
    mode = args.mode or ("slab" if world > 1 else "single")
    group = []
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{dev}")
    if args.roofline_only:
        roofline_point(nb, args, flush, dev)
        return 0
    if mode == "slab":
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
    b = mesh.rhs(pol, nb.NB_RHS_UNIFORM, seed=0)
    x = mesh.empty(pol)
    gb = [m.rhs(pol, nb.NB_RHS_UNIFORM, seed=0) for m in group]
    gx = [m.empty(pol) for m in group]
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
    # per-phase device time of the timed solve (block 0's %globaltimer stamps after each barrier)
    kt = solve()
    k1_us, k2_us = 1e3 * kt.k_ax_ms / kt.iterations, 1e3 * kt.k_upd_ms / kt.iterations

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

    # time-to-1e-8 for every policy on the headline workload, and AE/MAE
    ttr = {}
    companions = rank == 0 and world == 1 and not group and not args.quick
    if companions:
        hists = {}
        for name, pp in POLICIES.items():
            bb = mesh.rhs(pp, nb.NB_RHS_UNIFORM, seed=0)
            xx = mesh.empty(pp)
            reps = []
            for _ in range(3):
                flush.zero_()
                r, hh = nb.nb_cg(mesh.h, bb, xx, pp, max_iter, WORKLOAD["rtol"], history=True)
                reps.append(r)
            hists[name] = hh
            tmed = statistics.median(r.solve_ms for r in reps)
            rk = reps[-1]
            ttr[name] = {"iterations": rk.iterations, "status": rk.status, "time_ms": tmed,
                         "dof_iter_per_s": NL * rk.iterations / (tmed * 1e-3),
                         "phaseA_us": 1e3 * rk.k_ax_ms / rk.iterations, "phaseB_us": 1e3 * rk.k_upd_ms / rk.iterations}
        ttr["speedup_fp64_over_mixed_time"] = ttr["fp64"]["time_ms"] / ttr["mixed"]["time_ms"]
        ttr["accuracy_AE_MAE_mixed_vs_fp64"] = ae_mae(hists["mixed"], hists["fp64"])
        ttr["accuracy_AE_MAE_fp32_vs_fp64"] = ae_mae(hists["fp32"], hists["fp64"])
        # NEXT-4: the same workload with the two-level Schwarz preconditioner
        # (Nekbone's multigrid-preconditioned CG) -- time to 1e-8 per policy
        sw = {}
        for name, pp in POLICIES.items():
            bb = mesh.rhs(pp, nb.NB_RHS_UNIFORM, seed=0)
            xx = mesh.empty(pp)
            nb.nb_cg(mesh.h, bb, xx, pp, max_iter, WORKLOAD["rtol"], history=False, precond=nb.NB_PC_SCHWARZ)
            reps = []
            for _ in range(3):
                flush.zero_()
                r, _ = nb.nb_cg(mesh.h, bb, xx, pp, max_iter, WORKLOAD["rtol"], history=False,
                                precond=nb.NB_PC_SCHWARZ)
                reps.append(r)
            tmed = statistics.median(r.solve_ms for r in reps)
            rk = reps[-1]
            it = max(rk.iterations, 1)
            sw[name] = {"iterations": rk.iterations, "status": rk.status, "time_ms": tmed,
                        "speedup_vs_jacobi": ttr[name]["time_ms"] / tmed,
                        "phaseA_us": 1e3 * rk.k_ax_ms / it, "phaseB_us": 1e3 * rk.k_upd_ms / it,
                        "solveM_us": 1e3 * rk.k_gs_ms / it}
        sw["speedup_fp64_over_mixed_time"] = sw["fp64"]["time_ms"] / sw["mixed"]["time_ms"]
        ttr["schwarz_pcg"] = sw

    # the HBM roofline point (configs[2]); configs[1] above is L2-resident
    roof, peak, peak_src = None, None, None
    if companions and not args.no_large:
        roof, peak, peak_src = roofline_point(nb, args, flush, dev)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        v, dt, _, it, _ = oracle_sample(args.cpu_iters, args.policy)
        cpu = {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"{it} CG iterations ({args.policy}, rtol=0) of configs[1], setup excluded, "
                         f"{dt:.1f} s on one host core"}

    if rank == 0:
        ms_per_step = 1e3 * t_max / args.steps
        roofline = None
        if roof:
            r = roof["policies"][args.policy if args.policy in roof["policies"] else "mixed"]
            roofline = {"bound": "hbm", "kernel": "k_cg_mega (the whole CG solve: phase A p-update + x + local Ax "
                                                   "+ pap, phase B gather-scatter + r/z update + dots)",
                        "workload": roof["workload"], "policy": args.policy,
                        "achieved": r["achieved_GBps"], "peak": peak, "unit": "GB/s",
                        "frac": r["achieved_GBps"] / peak,
                        "traffic": r.get("ncu_dram_bytes_per_launch"),
                        "achieved_note": "SURVEY.md §8(d) fused-iteration bytes per DOF "
                                         f"({r['survey_bytes_per_dof_iter']:.1f} B at this mesh's shared fractions) x "
                                         f"n_local x iterations / launch time (CUDA events on the launching stream)",
                        "achieved_impl_bytes": r["achieved_impl_GBps"], "frac_impl_bytes": r["achieved_impl_GBps"] / peak,
                        "ncu_dram_GBps": r.get("ncu_dram_GBps_at_this_launch_time"),
                        "ncu_dram_frac": (r["ncu_dram_GBps_at_this_launch_time"] / peak
                                          if r.get("ncu_dram_GBps_at_this_launch_time") else None),
                        "alg_bytes_per_launch": r["survey_bytes_per_dof_iter"] * roof["n_local"] * r["iterations"],
                        "avg_launch_us": 1e3 * r["launch_ms"], "peak_source": peak_src,
                        "ncu_source": r.get("ncu_source")}
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": max(3, args.warmup), "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": {0: "f64", 1: "f32", 2: "f32+f64 (mixed)"}[pol],
                "data": "synthetic",
                "config": dict(WORKLOAD, policy=args.policy, iterations=iters[0], status=sorted(statuses),
                               n_local=NL, l2="256 MiB write between steps (outside the step events); "
                                              "configs[1]'s working set (~100 MB mixed) is L2-resident: "
                                              "throughput and time only, the HBM roofline is taken on configs[2]",
                               parallelism=parallelism(mode, world, len(group)), mode=mode,
                               **({"nel": nel} if mode == "slab" else {})),
                "time_to_rtol_ms": ms_per_step,
                "step_ms": {"events_around_call": step_ms, "library_device_ms": lib_ms},
                "phases_us": {"A": k1_us, "B": k2_us},
                "roofline": roofline, "hbm_roofline_point": roof,
                "e2e": e2e, "gpu_launches": launches, "clocks": ck, "cpu_baseline": cpu, "policies": ttr}
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
    ap.add_argument("--quick", action="store_true", help="skip the per-policy table and the roofline point")
    ap.add_argument("--no-large", action="store_true", help="skip the HBM-bound configs[2] roofline point")
    ap.add_argument("--roofline-only", action="store_true",
                    help="one configs[2] megakernel launch per --roof-policies entry (the ncu target), nothing else")
    ap.add_argument("--roof-policies", nargs="+", default=["mixed", "fp64"], choices=list(POLICIES))
    ap.add_argument("--mode", default=None, choices=["single", "replicas", "slab"],
                    help="N>1 default: slab (one box split in z-slabs over the GPUs); replicas: independent solves")
    ap.add_argument("--slabs", type=int, default=2, help="--mode slab on one GPU: slabs in the launch")
    ap.add_argument("--dry-run", action="store_true", help="multi-rank plumbing only (gloo, no GPU work)")
    ap.add_argument("--oracle-timing", action="store_true",
                    help="instead of the bench line: time the CPU oracle per config (SURVEY §8(d))")
    ap.add_argument("--oracle-max-dof", type=float, default=0, help="--oracle-timing: skip larger configs")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn(args)
    if args.dry_run:
        return run_dry(args)
    if args.oracle_timing:
        return run_oracle_timing(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
