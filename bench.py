"""bench.py -- CIRR stage throughput on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl cirr|reference] [--config 4]

Workload (config.workload): BASELINE.json config 4 -- the dense non-Hermitian
GEP at n = 4096, two ellipses (0.3 x 0.15 at +-0.5), N = 64 quadrature points
each (128 complex128 4096^2 pencils), L = 32, M = 8, tol 1e-10, max_refine 8
-- the config the north-star's ">= 60 % of FP64 tensor peak" target is quoted
on.  A step = one full ``solve_multi`` of one GEP (K1..K7 + the reference's
refinement loop).  N > 1: weak scaling, rank r solves its own seeded GEP
(seed = r), no data-path collective.

Metric: GEP/s (whole job).  `value` has A, B resident in HBM before the timed
region; `e2e` runs the public ``solve_multi`` on pinned host A, B (H2D of the
inputs and D2H of eigenpairs inside the timed region).  The pencils (34 GB)
exceed L2 (126 MB), so no L2 flush is needed between steps.

`--impl reference` times the CPU oracle (oracle/cirr.py, the restated
reference path with LAPACK dense LU) on the host cores: a bounded sample of the
same GEP (6 of the 128 pencils: assembly + LU + every solve pass; one
Rayleigh-Ritz round), extrapolated to one GEP.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP64_DMMA_PEAK_TFLOPS = 37.1  # tools/fp64_peak.cu on this pool's B200 (profiles/fp64_peak_r01.jsonl)
METRIC = "CIRR GEP solves per second (config 4: n=4096 dense non-Hermitian, 2 ellipses x 64 nodes, L=32, M=8)"
UNIT = "GEP/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="cirr", choices=["cirr", "reference"])
    ap.add_argument("--config", type=int, default=4, choices=[4])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-variants", action="store_true", help="skip the labelled (non-reference) variants")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ---------------------------------------------------------------------------
# clocks sampled during the timed region


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        return False

    def summary(self):
        sm, smax, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax = max(smax, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU baseline (oracle) -- bounded sample of one GEP


def cpu_sample(wl, refine_cols=None, passes=None, sample_pencils=6, threads_label=None):
    """Time the oracle's per-pencil work (assembly, LAPACK LU, every solve pass)
    on `sample_pencils` pencils and one Rayleigh-Ritz round; extrapolate to
    one GEP.  Returns (seconds_per_gep, description)."""
    import scipy.linalg as sla

    from oracle.cirr import OracleConfig, Pencil, quadrature, rank_truncate_svd, rayleigh_ritz

    cores = os.cpu_count() or 1
    p = Pencil(wl.a, wl.b, wl.hermitian)
    n = p.n
    nodes_per = wl.n_q
    total_pencils = nodes_per * len(wl.contours)
    passes = passes or 8
    refine_cols = refine_cols or 118
    rng = np.random.default_rng(0)
    t0 = time.perf_counter()
    for j in range(sample_pencils):
        z = complex(quadrature(wl.contours[0], wl.n_q)[0][j])
        m = z * p.b - p.a
        lu = sla.lu_factor(m, check_finite=False)
        bv = p.b @ rng.standard_normal((n, wl.source_cols)).astype(complex)
        sla.lu_solve(lu, bv, check_finite=False)
        for _ in range(passes - 1):
            sla.lu_solve(lu, rng.standard_normal((n, refine_cols)) + 0j, check_finite=False)
    t_pencils = time.perf_counter() - t0
    t1 = time.perf_counter()
    s = rng.standard_normal((n, wl.source_cols * wl.n_moments)) + 1j * rng.standard_normal(
        (n, wl.source_cols * wl.n_moments))
    q = rank_truncate_svd(s, 1e-12)
    rayleigh_ritz(p, q, "general" if not wl.hermitian else "hermitian")
    t_rr = time.perf_counter() - t1
    per_gep = t_pencils / sample_pencils * total_pencils + t_rr * passes * len(wl.contours)
    desc = (f"oracle (scipy LAPACK, BLAS threads={threads_label or os.environ.get('OPENBLAS_NUM_THREADS', 'default')}) on "
            f"{sample_pencils}/{total_pencils} pencils (assemble+zgetrf+{passes} solve passes, L={wl.source_cols} "
            f"then K={refine_cols}) + 1 RR round (SVD n x {wl.source_cols * wl.n_moments}, A Q, B Q, eig), "
            f"extrapolated x{total_pencils / sample_pencils:.0f} pencils and x{passes * len(wl.contours)} RR rounds; "
            f"sample wall {t_pencils + t_rr:.1f} s")
    del cores, OracleConfig
    return per_gep, desc, t_pencils + t_rr


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def lu_traffic():
    """DRAM bytes of the LU stage per step, measured by ncu on this code
    (profiles/r01_lu_traffic_v14.json: dram__bytes_read + dram__bytes_write over
    every LU kernel of one solve_multi); null when the profile is absent."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r01_lu_traffic_v14.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return {"traffic": d["lu_dram_bytes"], "traffic_unit": "bytes per step (all LU kernels)",
                "traffic_over_algorithmic_min": d["traffic_over_min"], "traffic_source": os.path.relpath(path)}
    except (OSError, KeyError, ValueError):
        return {"traffic": None}


def build_workload(seed):
    from paper_2511_01927_b200 import workloads as W
    return W.config4(seed=seed)


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    wl = build_workload(0)
    cores = os.cpu_count() or 1
    times = []
    desc = ""
    for _ in range(max(args.warmup, 0) and 1):  # one untimed warm-up sample (page-in, BLAS init)
        cpu_sample(wl, sample_pencils=1)
    for _ in range(args.steps):
        per_gep, desc, _ = cpu_sample(wl)
        times.append(per_gep)
    per = statistics.median(times)
    value = 1.0 / per
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": per * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "c128 (f64)", "data": "synthetic (seeded config 4)",
        "config": {"workload": "BASELINE config 4: n=4096 dense non-Hermitian GEP, 2 ellipses, N=64, L=32, M=8",
                   "parallelism": "cpu"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": desc,
                         "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm


def run_cirr(args):
    import torch

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2511_01927_b200 import DevicePencil, SolverConfig, _lib, solve_multi
    from paper_2511_01927_b200 import solvers as S

    wl = build_workload(rank)
    cfg = SolverConfig(n_q=wl.n_q, source_cols=wl.source_cols, n_moments=wl.n_moments, tol=1e-10)
    dp = DevicePencil(wl.a, wl.b, hermitian=False)
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        import torch.distributed as dist
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        solve_multi(dp, wl.contours, cfg, seed=0)
    torch.cuda.synchronize()

    timer = S.StageTimer()
    S.set_stage_timer(timer)
    l0 = _lib.call("cirr_launch_count")
    stream = torch.cuda.current_stream()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    results = []
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        e0.record(stream)
        for _ in range(args.steps):
            results.append(solve_multi(dp, wl.contours, cfg, seed=0))
        e1.record(stream)
        torch.cuda.synchronize()
    barrier()
    S.set_stage_timer(None)
    launches = _lib.call("cirr_launch_count") - l0
    ms = e0.elapsed_time(e1)
    ms_max = max_over_ranks(ms)
    stages = timer.totals()
    work = dict(timer.work)
    per_step = ms_max / args.steps
    value = world * args.steps / (ms_max / 1e3)

    last = results[-1]
    pairs = sum(len(r.eigenvalues) for r in last.results if r is not None)
    counts = [len(r.eigenvalues) if r is not None else 0 for r in last.results]
    iters = [r.stats.iterations if r is not None else 0 for r in last.results]
    solves = last.stats.n_linear_solves

    lu_ms = stages.get("lu", 0.0)
    lu_tflops = work.get("lu_flops", 0.0) / (lu_ms / 1e3) / 1e12 if lu_ms else 0.0
    stage_ms = sum(stages.get(k, 0.0) for k in ("assemble", "lu", "solve", "moments"))
    stage_flops = work.get("lu_flops", 0.0) + work.get("solve_flops_exec", 0.0) + work.get("moment_flops", 0.0)
    stage_tflops = stage_flops / (stage_ms / 1e3) / 1e12 if stage_ms else 0.0

    # e2e: public API on pinned host buffers (H2D of A, B + D2H of eigenpairs inside the region)
    class HostPencil:
        pass

    hp = HostPencil()
    hp.a = torch.from_numpy(wl.a).pin_memory()
    hp.b = torch.from_numpy(wl.b).pin_memory()
    hp.hermitian = False
    e2e_times = []
    h2d = 2 * wl.a.nbytes
    d2h = 0
    for _ in range(max(args.e2e_steps, 1)):
        barrier()
        torch.cuda.synchronize()
        t = time.perf_counter()
        m = solve_multi(hp, wl.contours, cfg, seed=0)
        torch.cuda.synchronize()
        e2e_times.append(time.perf_counter() - t)
        d2h = sum(r.eigenvectors.nbytes + r.eigenvalues.nbytes + r.residuals.nbytes
                  for r in m.results if r is not None)
    e2e_s = max_over_ranks(statistics.median(e2e_times))
    e2e_value = world / e2e_s

    # labelled variants (NOT the path of record): SURVEY.md finding 9
    # (conjugate-pair halving) and finding 8 (early exit), same workload and tol
    variants = {}
    if not args.no_variants:
        import dataclasses

        labels = {
            "conjugate_pairs": "factor the N/2 upper-half nodes of each real-axis-symmetric contour, mirror the "
                               "rest by conjugation",
            "early_exit": "stop refining a contour once its converged set is unchanged across two passes",
            "conjugate_pairs+early_exit": "both of the above",
        }
        for name, label in labels.items():
            vcfg = dataclasses.replace(cfg, conjugate_pairs="conjugate_pairs" in name, early_exit="early_exit" in name)
            solve_multi(dp, wl.contours, vcfg, seed=0)
            vt = S.StageTimer()
            S.set_stage_timer(vt)
            barrier()
            torch.cuda.synchronize()
            v0 = torch.cuda.Event(enable_timing=True)
            v1 = torch.cuda.Event(enable_timing=True)
            v0.record(stream)
            for _ in range(args.steps):
                vm = solve_multi(dp, wl.contours, vcfg, seed=0)
            v1.record(stream)
            torch.cuda.synchronize()
            S.set_stage_timer(None)
            vms = max_over_ranks(v0.elapsed_time(v1))
            vcounts = [len(r.eigenvalues) if r is not None else 0 for r in vm.results]
            diff = 0.0
            for rv, rr in zip(vm.results, last.results):
                if rv is not None and rr is not None and len(rv.eigenvalues) == len(rr.eigenvalues):
                    for lam in rr.eigenvalues:
                        diff = max(diff, float(np.min(np.abs(rv.eigenvalues - lam)) / abs(lam)))
            vwork = dict(vt.work)
            variants[name] = {
                "label": "variant, not the reference's algorithm: " + label,
                "value": world * args.steps / (vms / 1e3), "unit": UNIT, "ms_per_step": vms / args.steps,
                "eigenpairs": vcounts, "iterations": [r.stats.iterations if r is not None else 0 for r in vm.results],
                "n_factorizations": vm.stats.n_factorizations, "n_linear_solves": vm.stats.n_linear_solves,
                "executed_flops_per_step": (vwork.get("lu_flops", 0.0) + vwork.get("solve_flops_exec", 0.0)
                                            + vwork.get("moment_flops", 0.0)) / args.steps,
                "max_rel_eig_diff_vs_record": diff}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        passes = max(iters) if iters else 8
        ref_cols = max(counts) if counts else 118
        per_gep, desc, wall = cpu_sample(wl, refine_cols=ref_cols, passes=passes)
        cpu = {"value": 1.0 / per_gep, "unit": UNIT, "cores": os.cpu_count() or 1, "kind": "port",
               "sample": desc, "cpu_model": cpu_model()}
        # the same sample with the BLAS pinned to one thread as well
        try:
            from threadpoolctl import threadpool_limits
            with threadpool_limits(limits=1):
                per1, desc1, _ = cpu_sample(wl, refine_cols=ref_cols, passes=passes, sample_pencils=1,
                                             threads_label="1 (threadpoolctl)")
            cpu["single_thread"] = {"value": 1.0 / per1, "unit": UNIT, "cores": 1, "sample": desc1}
        except ImportError:
            pass

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "c128 (f64 DMMA)", "data": "synthetic (seeded BASELINE config 4)",
            "config": {"workload": "BASELINE config 4: n=4096 dense non-Hermitian GEP, 2 ellipses (0.3x0.15 at "
                                   "+-0.5), N=64, L=32, M=8, tol=1e-10, max_refine=8",
                       "pencils": wl.n_q * len(wl.contours), "n": wl.n, "parallelism": f"replicas x{world}",
                       "l2_flush": "not needed: 34 GB of pencils per step >> 126 MB L2"},
            "roofline": {"bound": "tensor", "kernel": "batched zgetrf (K2: panel + DMMA trailing GEMM)",
                         "achieved": lu_tflops, "peak": FP64_DMMA_PEAK_TFLOPS, "unit": "TFLOP/s",
                         "frac": lu_tflops / FP64_DMMA_PEAK_TFLOPS,
                         "peak_source": "measured DMMA.8x8x4 FP64 peak (tools/fp64_peak.cu; "
                                        "MEASURED_PEAKS.json has no FP64 entry)",
                         "algorithmic": "8 n^3 / 3 per pencil x 128 pencils per step",
                         **lu_traffic()},
            "lu_plus_moment_stage": {"tflops": stage_tflops, "frac_of_fp64_peak": stage_tflops / FP64_DMMA_PEAK_TFLOPS,
                                     "flops_per_step": stage_flops / args.steps,
                                     "ms_per_step": stage_ms / args.steps},
            "stage_ms_per_step": {k: v / args.steps for k, v in sorted(stages.items())},
            "time_per_gep_s": per_step / 1e3,
            "eigenpairs_per_s": pairs * world / (per_step / 1e3),
            # shifted solves = pencils x passes; RHS columns = sum of n_linear_solves
            "shifted_solves_per_s": (last.stats.n_factorizations * max(iters or [1])) * world / (per_step / 1e3),
            "rhs_columns_per_s": solves * world / (per_step / 1e3),
            "eigenpairs": counts, "iterations": iters,
            "n_factorizations": last.stats.n_factorizations, "n_linear_solves": solves,
            "executed_flops_per_step": stage_flops / args.steps,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "seconds_per_step": e2e_s},
            "gpu_launches": launches,
            "clocks": clocks.summary(),
        }
        if variants:
            line["variants"] = variants
        if cpu is not None:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_cirr(args)


if __name__ == "__main__":
    main()
