#!/usr/bin/env python
"""Benchmark: all-at-once space-time MLK solve on B200.

Metric (BASELINE.json): space-time unknowns/s to a 1e-8 relative residual.
A "step" is one complete multilevel_solve (outer FGMRES to tol, inner
recursion, coarsest solves, true-residual check) of the workload.

Default workload ("c5_c"): the BASELINE config-5 shape -- 2-D heat equation,
255x255 interior grid, n_t = 4096 (2.66e8 unknowns, 2.13 GB per vector),
theta = 1/2, 5-level MLK, nu = 2, FGMRES(30), tol 1e-8 -- at the paper's
Courant number C = 0.16 (the literal T = 1 gives C = 48, where the reference
MLK stagnates; SURVEY.md sections 0.3 and 8(d)).  Seeded synthetic u0
(sin(pi x) sin(pi y) + 0.1 N(0,1)).  Every vector is larger than L2, so no
L2 flush is needed between steps.

  value  device-resident: u0 and the hierarchy already on the GPU, CUDA
         events around K solves, max over ranks.
  e2e    through the public API with host buffers: pinned u0 -> FineSystem
         -> build_hierarchy -> multilevel_solve -> x into pinned host memory.
  --gpus N > 1 (torchrun): every rank solves its own seeded instance
         (independent problems, no data-path collective): weak scaling.
  --impl reference: the CPU oracle (numpy/scipy restatement of pintmk,
         bitwise equal to the reference) on the host cores, rank 0 only.
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "space-time unknowns/s to 1e-8 rel. residual"
UNIT = "unknowns/s"
CPU_SAMPLE = "mid_2d"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--case", default="c5_c")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--e2e-warmup", type=int, default=2,
                    help="untimed end-to-end steps first (allocator / pinned-buffer steady state)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-profile", action="store_true")
    ap.add_argument("--no-extra", action="store_true",
                    help="skip the extra workload lines (other BASELINE shapes)")
    ap.add_argument("--no-full-shape-cpu", action="store_true",
                    help="reference arm: skip the one-iteration CPU run on the full shape")
    return ap.parse_args()


def dist_info():
    from paper_2401_00228_b200.dist import rank_info

    return rank_info()


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "samples": len(sm), "reasons": sorted(reasons)}


def cpu_sample_solve():
    """One CPU-oracle solve of the bounded sample; returns (unknowns/s, seconds, info)."""
    from oracle import pintmk_oracle as O
    from tests.cases import BASELINE, oracle_hierarchy

    case = BASELINE[CPU_SAMPLE]
    h = oracle_hierarchy(case)
    t0 = time.perf_counter()
    x, info = O.solve(h)
    dt = time.perf_counter() - t0
    return case.N / dt, dt, info, case


def cpu_desc(case, info):
    return (f"CPU oracle (numpy/scipy restatement of pintmk, bitwise equal to the reference) "
            f"full solve of the {case.nx}x{case.nx} x {case.n_t}-step companion of the workload "
            f"(same theta, levels, nu, Courant number; {info['iterations']} iterations, "
            f"{case.N} unknowns); scipy sparse/SuperLU single-threaded, BLAS-1 dots on "
            f"OpenBLAS default threads")


def cpu_full_shape_iteration(name: str):
    """One outer FGMRES iteration of the CPU oracle on the workload's own
    inputs (full shape; the reference's wall_time, solver.py:463-467, for one
    iteration).  Returns (seconds for the iteration, setup seconds)."""
    from oracle import pintmk_oracle as O
    from tests.cases import BASELINE, oracle_hierarchy

    case = BASELINE[name].scaled(max_outer=1, restart=None)
    t0 = time.perf_counter()
    h = oracle_hierarchy(case)
    t1 = time.perf_counter()
    O.fgmres(h, 0, h.rhs.ravel(), None, 1)
    t2 = time.perf_counter()
    del h
    gc.collect()
    return t2 - t1, t1 - t0


def run_reference(args):
    rank, world, _ = dist_info()
    if rank != 0:
        return
    vals = []
    for _ in range(max(args.warmup, 0)):
        cpu_sample_solve()
    for _ in range(args.steps):
        v, dt, info, case = cpu_sample_solve()
        vals.append(v)
    value = statistics.mean(vals)
    cores = os.cpu_count()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": max(args.warmup, 0),
        "ms_per_step": 1000.0 * case.N / value, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.case, "sample": CPU_SAMPLE},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": cpu_desc(case, info)},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if not args.no_full_shape_cpu:
        from tests.cases import BASELINE

        it_s, setup_s = cpu_full_shape_iteration(args.case)
        full = BASELINE[args.case]
        iters = FULL_SHAPE_ITERS.get(args.case)
        line["cpu_full_shape_s_per_iter"] = round(it_s, 2)
        line["cpu_full_shape"] = {
            "workload": args.case, "unknowns": full.N, "setup_s": round(setup_s, 2),
            "s_per_iteration": round(it_s, 2),
            "what": "one outer FGMRES iteration (preconditioner recursion, matvec, MGS) of the "
                    "CPU oracle on the workload's own 255^2 x 4096 inputs, timed on this host",
            "extrapolated_solve_s": round(it_s * iters, 1) if iters else None,
            "extrapolated_unknowns_per_s": round(full.N / (it_s * iters), 1) if iters else None,
            "extrapolation": (f"EXTRAPOLATED, not measured: x {iters} iterations (the live "
                              f"reference's count on this workload, tests/golden/); later "
                              f"iterations cost more (MGS grows with j), so this flatters "
                              f"the CPU") if iters else None,
        }
    print(json.dumps(line), flush=True)


# outer iterations of the live reference on the full-shape workloads
# (tests/golden/make_c5c_reference.py fingerprint)
FULL_SHAPE_ITERS = {"c5_c": 19}


def run_ours(args):
    import numpy as np
    import torch

    from paper_2401_00228_b200 import _lib, multilevel_solve
    from tests.cases import BASELINE, gpu_hierarchy

    from paper_2401_00228_b200 import dist as pdist

    rank, world, local = dist_info()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        pdist.init("nccl")
    # replicas: every rank solves its own seeded instance (no data-path collective)
    from tests.cases import MID

    base = {**MID, **BASELINE}[args.case]
    case = base.scaled(seed=pdist.instance_seed(base.seed, rank))
    u0 = torch.from_numpy(case.u0_vector()).cuda()
    hier = gpu_hierarchy(case, u0=u0)

    for _ in range(max(args.warmup, 0)):
        x, rep = multilevel_solve(hier)
        del x
    gc.collect()
    torch.cuda.synchronize()
    pdist.barrier()
    torch.cuda.synchronize()

    sampler = ClockSampler(local)
    sampler.start()
    profile = not args.no_profile
    n0 = _lib.launch_count()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    iters, trues = [], []
    ev0.record()
    for _ in range(args.steps):
        x, rep = multilevel_solve(hier)
        iters.append(rep.outer_iterations)
        trues.append(rep.metadata["true_relative_residual"])
        del x
    ev1.record()
    torch.cuda.synchronize()
    launches = _lib.launch_count() - n0
    clocks = sampler.stop()
    ms = pdist.max_over_ranks(ev0.elapsed_time(ev1), device="cuda")
    pdist.barrier()
    # per-kernel table / roofline: the same K steps again with CUDA events
    # around every launch (kept out of the timed region above: the events
    # add launch-side overhead)
    kernels, prof_ms = {}, None
    if profile:
        torch.cuda.synchronize()
        _lib.profile_begin(True)
        p0 = torch.cuda.Event(enable_timing=True)
        p1 = torch.cuda.Event(enable_timing=True)
        p0.record()
        for _ in range(args.steps):
            x, rep = multilevel_solve(hier)
            del x
        p1.record()
        torch.cuda.synchronize()
        kernels = _lib.profile_end()
        prof_ms = p0.elapsed_time(p1)
    ms_per_step = ms / args.steps
    value = case.N * args.steps * world / (ms / 1000.0)

    # ----- plain space-time matvec (K-MV, BASELINE's second metric): 16 B per
    # unknown (read v, write out; the k-1 slice comes from shared memory)
    mv = matvec_roofline(hier, case, args.steps) if rank == 0 else None

    # ----- e2e: public API, host buffers, H2D + setup + solve + D2H per step
    pin_u0 = torch.from_numpy(case.u0_vector()).pin_memory()
    pin_x = torch.empty(case.N, dtype=torch.float64).pin_memory()
    del hier  # its device memory returns to the caching allocator (a serving
    # process keeps its pool: every e2e step still allocates, builds and frees
    # its own hierarchy and buffers through the public API)
    gc.collect()
    torch.cuda.synchronize()
    e2e_t = []
    n_e2e = max(args.e2e_steps, 0)
    n_e2e_warm = max(args.e2e_warmup, 0) if n_e2e else 0
    for i_e2e in range(n_e2e_warm + n_e2e):
        torch.cuda.synchronize()
        pdist.barrier()
        t0 = time.perf_counter()
        h2 = gpu_hierarchy(case, u0=pin_u0)
        xh, rep2 = multilevel_solve(h2, out=pin_x)
        torch.cuda.synchronize()
        if i_e2e >= n_e2e_warm:
            e2e_t.append(time.perf_counter() - t0)
        del h2, xh
        gc.collect()  # the previous hierarchy's native teardown (cudaFree
        # synchronises) happens here, not inside the next timed step
    # per-step mean (total time / steps, like the device-timed value), max over ranks
    e2e_s = (pdist.max_over_ranks(sum(e2e_t) / len(e2e_t), device="cuda") if e2e_t
             else float("nan"))

    # ----- roofline of the dominant memory-bound kernel
    peak, peak_kind = peaks()
    roof = None
    table = {}
    for name, k in kernels.items():
        gbs = k["bytes"] / (k["ms"] / 1000.0) / 1e9 if k["ms"] > 0 else 0.0
        table[name] = {"launches": k["launches"], "ms": round(k["ms"], 3),
                       "share": round(k["ms"] / prof_ms, 4) if prof_ms else None,
                       "GB/s": round(gbs, 1),
                       "TFLOP/s": round(k["flops"] / (k["ms"] / 1000.0) / 1e12, 2)
                       if k["ms"] > 0 and k["flops"] else None}
    mem = {n: k for n, k in kernels.items() if n not in ("coarse_gemm", "fgmres_small", "coarse_chain")}
    if mem:
        dom = max(mem, key=lambda n: mem[n]["ms"])
        k = mem[dom]
        achieved = k["bytes"] / (k["ms"] / 1000.0) / 1e9
        traffic = None
        tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tpath):
            try:
                traffic = json.load(open(tpath)).get(dom)
            except Exception:
                traffic = None
        roof = {"kernel": dom, "bound": "hbm", "achieved": round(achieved, 1),
                "peak": peak, "unit": "GB/s", "frac": round(achieved / peak, 4),
                "traffic": traffic, "bytes_per_launch": k["bytes"] / k["launches"],
                "peak_source": peak_kind,
                # DRAM rate implied by the ncu per-launch traffic and this run's mean
                # launch time; frac can exceed 1 because the peak is a copy (50/50
                # read/write) figure while the Gram/dot passes are read-dominated
                # (read-only streams sustain ~7.0 TB/s), and inner-level vectors
                # (<= 266 MB) are partly served from the 126 MB L2 (traffic < alg. bytes)
                "dram_achieved": (round(traffic / (k["ms"] / k["launches"] / 1000.0) / 1e9, 1)
                                  if traffic else None),
                "timing": "CUDA events around every launch on its stream, over a second "
                          "pass of the same K steps right after the timed region"}

    extra = None
    if rank == 0 and world == 1 and not args.no_extra:
        extra = extra_workloads()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, dt, info, c = cpu_sample_solve()
        cpu = {"value": v, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
               "sample": cpu_desc(c, info) + f"; {dt:.1f} s"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded u0 = sin(pi x) sin(pi y) + 0.1 N(0,1); no dataset)",
            "config": {"workload": case.name, "grid": f"{case.nx}x{case.ny}", "n_t": case.n_t,
                       "theta": case.theta, "levels": case.n_levels, "nu": case.nu,
                       "schedule": case.schedule_arg(), "courant": case.courant,
                       "coarsest_n_cgs": case.n_cgs, "restart": case.restart, "tol": case.tol,
                       "unknowns": case.N, "per_rank_instances": 1,
                       "l2": "inputs larger than L2 (2.13 GB vectors), no flush needed"},
            "iterations": iters[-1] if iters else None,
            "true_relative_residual": max(trues) if trues else None,
            "e2e": None if not e2e_t else {"value": case.N * world / e2e_s, "unit": UNIT,
                    "h2d_bytes_per_step": 8 * case.m, "d2h_bytes_per_step": 8 * case.N,
                    "seconds_per_step": e2e_s,
                    "step_seconds": [round(t, 4) for t in e2e_t],
                    "warmup_steps": n_e2e_warm,
                    "includes": "H2D of u0 from pinned memory, hierarchy setup, solve, "
                                "D2H of x into pinned memory"},
            "roofline": roof,
            "roofline_matvec": mv,
            "cpu_baseline": cpu,
            "extra_workloads": extra,
            "gpu_launches": launches,
            "clocks": clocks,
            "kernels": table,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def matvec_roofline(hier, case, steps: int):
    """K-MV alone on the fine level (pmk_stmv, the reference's
    BlockBidiagonalSystem.matvec): CUDA events on the launch stream around
    `reps` launches; achieved = 16 B x unknowns / mean launch time."""
    import torch

    from paper_2401_00228_b200 import _lib

    peak, peak_kind = peaks()
    fine = hier.fine
    v = torch.randn(case.N, dtype=torch.float64, device="cuda")
    out = torch.empty_like(v)
    reps = max(steps, 5)
    fine.matvec_into(v, out)  # warm-up
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fine.matvec_into(v, out)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / reps / 1000.0
    achieved = 16.0 * case.N / t / 1e9
    del v, out
    return {"kernel": "march_tma<MV> (pmk_stmv)", "bound": "hbm", "achieved": round(achieved, 1),
            "peak": peak, "unit": "GB/s", "frac": round(achieved / peak, 4),
            "bytes_per_launch": 16.0 * case.N, "ms_per_launch": round(t * 1000.0, 4),
            "launches": reps, "peak_source": peak_kind,
            "timing": "CUDA events on the launch stream around back-to-back launches "
                      "(2.13 GB in, 2.13 GB out: larger than L2)"}


# Other BASELINE shapes, device-resident, CUDA events: the "_c" companions
# to 1e-8 (c1_c-c3_c), c4's companion (TS x TS nu = 4, theta = 1; the
# reference needs > 200 iterations there) and literal c5 (C = 48, stagnant)
# at a fixed budget, and c5_c_dec: BASELINE config 5's literal solver
# structure (n_cgs = 256, one independent solve per coarse slice, FGMRES(30))
# at the paper's Courant number, to 1e-8.
EXTRA = [("c1_c", None), ("c2_c", None), ("c3_c", None), ("c4", 10), ("c4_c", 40),
         ("c5", 30), ("c5_c_dec", None), ("ttts_255", None), ("c1", 12), ("pcr_dec_mid", None),
         ("line_mid", None), ("line_dec_mid", None), ("c4_fw", 10), ("c4_fw_c", 40)]


def extra_workloads():
    import torch

    from paper_2401_00228_b200 import multilevel_solve
    from tests.cases import BASELINE, MID, gpu_hierarchy

    out = {}
    for name, budget in EXTRA:
        base = {**MID, **BASELINE}[name]
        case = base if budget is None else base.scaled(max_outer=budget)
        try:
            u0 = torch.from_numpy(case.u0_vector()).cuda()
            h = gpu_hierarchy(case, u0=u0)
            reps = 1 if case.N > 1e8 else 3
            x, rep = multilevel_solve(h)  # warm-up (graph capture, tables)
            del x
            torch.cuda.synchronize()
            times = []
            for _ in range(reps):  # one event pair per solve; the median is reported
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
                x, rep = multilevel_solve(h)
                e1.record()
                torch.cuda.synchronize()
                times.append(e0.elapsed_time(e1))
                del x
            ms = statistics.median(times)
            out[name] = {
                "unknowns": case.N, "grid": f"{case.nx}x{case.ny}", "n_t": case.n_t,
                "theta": case.theta, "levels": case.n_levels, "schedule": case.schedule_arg(),
                "nu": case.nu, "courant": case.courant, "T": case.T,
                "coarsest_n_cgs": case.n_cgs, "restart": case.restart,
                "coarsest_kind": getattr(h.levels[-1].system.diag_factorization,
                                         "kind_detail", None),
                "budget": budget, "ms_per_solve": round(ms, 3),
                "iterations": rep.outer_iterations,
                "converged": bool(rep.converged),
                "true_relative_residual": rep.metadata["true_relative_residual"],
                "restart_cycles": rep.metadata.get("restart_cycles"),
                ("unknowns_per_s" if budget is None else "unknown_iterations_per_s"):
                    (case.N / (ms / 1000.0) if budget is None
                     else case.N * rep.outer_iterations / (ms / 1000.0)),
            }
            del h
        except Exception as exc:  # reported, never silently dropped
            out[name] = {"error": f"{type(exc).__name__}: {exc}"}
        torch.cuda.synchronize()
        gc.collect()
        torch.cuda.empty_cache()
    return out


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
