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
reference path with LAPACK dense LU, all host threads) on ONE FULL config-4
GEP (its whole solve_multi: 128 LUs, every refinement pass, every
Rayleigh-Ritz round), so its `value` is measured, not extrapolated; it also
reports the bounded-sample estimate beside it.  `steps` there is the number of
full GEPs timed (1): a GEP takes minutes on the host.  Both arms print the same
`config` dict.

`per_config` (GPU arm, N=1): BASELINE configs 2 (one solve_multi_batch of the
256 GEPs), 1, 3 and 5 (one solve_multi each), each device-timed and end to end,
with the LU TF/s (band flops for the banded pencils) and the in-contour counts
checked against the oracle fixtures.
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
# complex128 in and out; the k = 512 updates of the dense LU and of the blocked solves as exact int8 digit
# products (Ozaki splitting, 55 bits per operand) on tcgen05, every other GEMM in FP64 on DMMA
DTYPE = "c128 (int8 slice products on tcgen05 for the k=512 LU/solve updates, f64 DMMA elsewhere)"


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
    ap.add_argument("--no-per-config", action="store_true", help="skip the config 2 / config 5 block")
    ap.add_argument("--shard", default="geps", choices=["geps", "nodes"],
                    help="N > 1: 'geps' (default) = one GEP per rank, weak scaling, no data-path collective; "
                         "'nodes' = ONE GEP split by quadrature node over the ranks, one NCCL all-reduce of the "
                         "moment blocks per pass (dist.solve_multi_node_sharded), strong scaling")
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
    (profiles/r02_v7_lu_traffic.json, TAG=_v7 tools/ncu_r02.sh: dram__bytes_read +
    dram__bytes_write over every LU kernel of one solve_multi); null when the
    profile is absent."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r02_v7_lu_traffic.json")
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


def bench_config(wl) -> dict:
    """The `config` dict both arms print (identical, so the driver can pair them)."""
    return {"workload": "BASELINE config 4: n=4096 dense non-Hermitian GEP, 2 ellipses (0.3x0.15 at +-0.5), "
                        "N=64, L=32, M=8, tol=1e-10, max_refine=8",
            "pencils": wl.n_q * len(wl.contours), "n": wl.n, "n_q": wl.n_q, "source_cols": wl.source_cols,
            "n_moments": wl.n_moments, "tol": 1e-10, "seed": 0, "parallelism": "replicas (one GEP per rank)",
            "l2_flush": "not needed: 34 GB of pencils per step >> 126 MB L2"}


def run_reference(args):
    """The reference's CPU path (the restated oracle: reference solve_multi plus
    the SURVEY 8(c) deltas, LAPACK dense LU) on one full config-4 GEP, all host
    threads; the bounded-sample estimate is reported beside it."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle.cirr import OracleConfig, Pencil
    from oracle.cirr import solve_multi as oracle_solve_multi

    wl = build_workload(0)
    cores = os.cpu_count() or 1
    if args.warmup > 0:  # untimed: page-in, BLAS thread pool start-up
        cpu_sample(wl, sample_pencils=1, passes=1)
    ocfg = OracleConfig(n_q=wl.n_q, source_cols=wl.source_cols, n_moments=wl.n_moments, tol=1e-10)
    t0 = time.perf_counter()
    m = oracle_solve_multi(Pencil(wl.a, wl.b, False), wl.contours, ocfg, seed=0)
    full = time.perf_counter() - t0
    counts = [0 if r is None else len(r.eigenvalues) for r in m.results]
    iters = [0 if r is None else r.iterations for r in m.results]
    est, desc, wall = cpu_sample(wl, refine_cols=max(counts), passes=max(iters))
    value = 1.0 / full
    sample = (f"one full config-4 GEP: oracle solve_multi (scipy LAPACK zgetrf/zgetrs, BLAS threads="
              f"{os.environ.get('OPENBLAS_NUM_THREADS', 'default')}), 128 pencils, {max(iters)} passes, "
              f"{sum(counts)} eigenpairs, wall {full:.1f} s")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": world,
        "steps": 1, "steps_requested": args.steps, "warmup": args.warmup, "ms_per_step": full * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128 (f64)",
        "data": "synthetic (seeded BASELINE config 4)", "config": bench_config(wl),
        "eigenpairs": counts, "iterations": iters,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample,
                         "cpu_model": cpu_model(),
                         "sampled_estimate": {"value": 1.0 / est, "unit": UNIT, "sample": desc}},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm


class HostPencil:
    """What a reference caller passes: host numpy A, B (dense) and the flag."""

    def __init__(self, a, b, hermitian):
        self.a, self.b, self.hermitian = a, b, hermitian


def _timed(fn, reps=1):
    """CUDA-event time (ms, median over reps) of fn() on torch's current stream
    (the stream libcirr launches on), plus the stage timer totals of the last rep."""
    import torch

    from paper_2511_01927_b200 import solvers as S

    times, out, timer = [], None, None
    for _ in range(reps):
        timer = S.StageTimer()
        S.set_stage_timer(timer)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = fn()
        e1.record()
        torch.cuda.synchronize()
        S.set_stage_timer(None)
        times.append(e0.elapsed_time(e1))
    return statistics.median(times), out, timer


def _wall(fn, reps=1):
    import torch

    times, out = [], None
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t)
    return statistics.median(times), out


def _lu_line(timer):
    lu_ms = timer.totals().get("lu", 0.0)
    fl = timer.work.get("lu_flops", 0.0)
    tf = fl / (lu_ms / 1e3) / 1e12 if lu_ms else 0.0
    return {"lu_ms": lu_ms, "lu_flops": fl, "lu_tflops": tf, "lu_frac_of_fp64_peak": tf / FP64_DMMA_PEAK_TFLOPS}


INT8_PEAK_TOPS = 4570.0   # measured: tools/i8_peak.cu, back-to-back tcgen05.mma kind::i8 (M128 N128 K32), 148 SMs


def int8_kernel_roofline():
    """The int8 (Ozaki) trailing update timed alone at the LU's largest step
    (m = 3584, k = 512, 16 pencils; the step processes 128 in chunks): CUDA
    events over the split kernels + ozaki_gemm_kernel on the launching stream.
    int8 operations: 36 slice products x 2 x m x 2n x 2k = 288 mnk."""
    import torch
    from paper_2511_01927_b200 import _lib

    m, W, batch, reps = 3584, 512, 16, 5
    n = m + W
    g = torch.Generator(device="cuda").manual_seed(0)
    P = torch.randn((batch, n, n), dtype=torch.complex128, device="cuda", generator=g)
    st = torch.cuda.current_stream().cuda_stream
    base = P.data_ptr()
    off = lambda r, c: base + 16 * (r * n + c)

    def run():
        _lib.call("cirr_ozaki_zgemm_sub", off(W, 0), n, n * n, off(0, W), n, n * n, off(W, W), n, n * n, m, m, W,
                  batch, st)

    for _ in range(2):
        run()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    ops = 288.0 * m * m * W * batch
    del P
    torch.cuda.empty_cache()
    return {"kernel": "ozaki_gemm_kernel + splits (tcgen05.mma kind::i8, one k = 512 trailing update, m = 3584, "
                      "16 pencils, timed alone)",
            "bound": "tensor", "achieved": ops / (ms / 1e3) / 1e12, "peak": INT8_PEAK_TOPS, "unit": "TOP/s (int8)",
            "frac": ops / (ms / 1e3) / 1e12 / INT8_PEAK_TOPS,
            "peak_source": "measured tcgen05.mma kind::i8 issue rate, burst (tools/i8_peak.cu; MEASURED_PEAKS.json "
                           "has bf16 only: 2 x its 1633.6 bf16 TF/s burst = 3267)",
            "fp64_equivalent_tflops": 8.0 * m * m * W * batch / (ms / 1e3) / 1e12, "ms": ms}



def per_config_block():
    """BASELINE configs 1, 2, 3 and 5 on the driver's clock.
    Contours and the oracle's in-contour counts come from the committed oracle
    fixtures (tests/golden/oracle_config{1,2,3,5}.npz, the checker)."""
    import torch

    from paper_2511_01927_b200 import Contour, DevicePencil, SolverConfig, solve_multi, solve_multi_batch
    from paper_2511_01927_b200 import workloads as W

    gold = os.path.join(ROOT, "tests", "golden")
    out = {}

    # config 2: 256 independent n=256 GEPs, one solve_multi_batch
    fix = np.load(os.path.join(gold, "oracle_config2.npz"))
    ng = int(fix["n_gep"])
    mats = [W.config2_matrices(s) for s in range(ng)]
    cons = [[Contour.from_json_dict(d) for d in json.loads(str(fix[f"s{s}_contours"]))] for s in range(ng)]
    want = [[len(fix[f"s{s}_c{i}_eigs"]) for i in range(len(cons[s]))] for s in range(ng)]
    cfg = SolverConfig(n_q=16, source_cols=8, n_moments=4)
    dps = [DevicePencil(a, b, hermitian=True) for a, b in mats]
    solve_multi_batch(dps, cons, cfg)  # warm-up
    ms, res, timer = _timed(lambda: solve_multi_batch(dps, cons, cfg), reps=3)
    got = [[0 if x is None else len(x.eigenvalues) for x in m.results] for m in res]
    hps = [HostPencil(a, b, True) for a, b in mats]
    e2e_s, _ = _wall(lambda: solve_multi_batch(hps, cons, cfg), reps=3)
    pairs = sum(map(sum, got))
    out["config2"] = {
        "workload": "BASELINE config 2: 256 independent n=256 2-D FD GEPs, 2 circles each, N=16, L=8, M=4 "
                    "(one solve_multi_batch call = one step)",
        "ms_per_step": ms, "time_per_gep_ms": ms / ng, "gep_per_s": ng / (ms / 1e3),
        "eigenpairs_per_s": pairs / (ms / 1e3), "pencils": 16 * 2 * ng,
        "e2e": {"value": ng / e2e_s, "unit": "GEP/s", "seconds_per_step": e2e_s,
                "h2d_bytes_per_step": int(sum(a.nbytes + b.nbytes for a, b in mats))},
        **_lu_line(timer), "stage_ms_per_step": {k: round(v, 3) for k, v in sorted(timer.totals().items())},
        "counts_equal_oracle": got == want, "eigenpairs": pairs}
    del dps, res, hps, mats
    torch.cuda.empty_cache()

    # configs 1, 3, 5: one solve_multi each (config 5: 128 pencils of n=8000 in one wave)
    single = {
        1: ("BASELINE config 1: n=512 1-D FD GEP (tridiagonal), 2 circles, N=32, L=16, M=4", W.config1_matrices, (32, 16, 4)),
        3: ("BASELINE config 3: n=2304 2-D FD GEP, 3 circles, N=32, L=32, M=4", W.config3_matrices, (32, 32, 4)),
        5: ("BASELINE config 5: n=8000 3-D FD GEP, 4 circles, N=32, L=64, M=4", W.config5_matrices, (32, 64, 4)),
    }
    for cno, (label, mk, (nq, L, M)) in single.items():
        fix = np.load(os.path.join(gold, f"oracle_config{cno}.npz"))
        cons = [Contour.from_json_dict(d) for d in json.loads(str(fix["contours"]))]
        want = [len(fix[f"c{i}_eigs"]) for i in range(len(cons))]
        a, b = mk()
        cfg = SolverConfig(n_q=nq, source_cols=L, n_moments=M)
        dp = DevicePencil(a, b, hermitian=True)
        solve_multi(dp, cons, cfg, seed=0)  # warm-up
        ms, m, timer = _timed(lambda: solve_multi(dp, cons, cfg, seed=0), reps=3)
        got = [0 if r is None else len(r.eigenvalues) for r in m.results]
        worst = 0.0
        for i, r in enumerate(m.results):
            ref = fix[f"c{i}_eigs"]
            if r is not None and len(r.eigenvalues) == len(ref):
                worst = max(worst, float(np.max(np.abs(r.eigenvalues - ref) / np.abs(ref))))
        del dp
        torch.cuda.empty_cache()
        e2e_s, _ = _wall(lambda: solve_multi(HostPencil(a, b, True), cons, cfg, seed=0), reps=3)
        out[f"config{cno}"] = {
            "workload": label + " (one solve_multi = one step)",
            "ms_per_step": ms, "gep_per_s": 1e3 / ms, "eigenpairs_per_s": sum(got) / (ms / 1e3),
            "pencils": nq * len(cons), "n": int(a.shape[0]),
            "e2e": {"value": 1.0 / e2e_s, "unit": "GEP/s", "seconds_per_step": e2e_s,
                    "h2d_bytes_per_step": int(a.nbytes + b.nbytes)},
            **_lu_line(timer), "stage_ms_per_step": {k: round(v, 3) for k, v in sorted(timer.totals().items())},
            "counts_equal_oracle": got == want, "eigenpairs": got, "max_rel_eig_diff_vs_oracle": worst,
            "iterations": [0 if r is None else r.stats.iterations for r in m.results]}
    torch.cuda.empty_cache()
    return out


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

    node_split = args.shard == "nodes" and world > 1
    if node_split:   # one GEP (rank 0's matrices on every rank) split by node; the other ranks' work is its share
        from paper_2511_01927_b200.dist import solve_multi_node_sharded
        wl = build_workload(0)
        dp = DevicePencil(wl.a, wl.b, hermitian=False)
        solve_multi = lambda p, cs, c, seed=0: solve_multi_node_sharded(p, cs, c, "cirr", seed)  # noqa: E731
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
    value = (1 if node_split else world) * args.steps / (ms_max / 1e3)

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

    # e2e: the public solve_multi on the plain (pageable) numpy A, B a reference
    # caller holds -- H2D of A, B and D2H of the eigenpairs inside the region
    hp = HostPencil(wl.a, wl.b, False)
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
    e2e_value = (1 if node_split else world) / e2e_s

    # labelled variants (NOT the path of record): SURVEY.md finding 9
    # (conjugate-pair halving) and finding 8 (early exit), same workload and tol
    variants = {}
    if not args.no_variants and not node_split:
        import dataclasses

        labels = {
            "conjugate_pairs": "factor the N/2 upper-half nodes of each real-axis-symmetric contour, mirror the "
                               "rest by conjugation",
            "early_exit": "stop refining a contour once its converged set is unchanged across two passes",
            "conjugate_pairs+early_exit": "both of the above",
        }
        labels["fp64_dmma"] = ("every GEMM in FP64 on DMMA (cirr_set_lu_gemm(0)): the reference's own arithmetic "
                               "type on the tensor cores, the path of record before the int8 slices")
        for name, label in labels.items():
            vcfg = dataclasses.replace(cfg, conjugate_pairs="conjugate_pairs" in name, early_exit="early_exit" in name)
            _lib.call("cirr_set_lu_gemm", 0 if name == "fp64_dmma" else 1)
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
            if name == "fp64_dmma":
                variants[name + "_stage_ms"] = {k: v / args.steps for k, v in sorted(vt.totals().items())}
            _lib.call("cirr_set_lu_gemm", 1)
            variants[name] = {
                "label": ("variant (same algorithm, FP64 arithmetic): " if name == "fp64_dmma" else
                          "variant, not the reference's algorithm: ") + label,
                "value": world * args.steps / (vms / 1e3), "unit": UNIT, "ms_per_step": vms / args.steps,
                "eigenpairs": vcounts, "iterations": [r.stats.iterations if r is not None else 0 for r in vm.results],
                "n_factorizations": vm.stats.n_factorizations, "n_linear_solves": vm.stats.n_linear_solves,
                "executed_flops_per_step": (vwork.get("lu_flops", 0.0) + vwork.get("solve_flops_exec", 0.0)
                                            + vwork.get("moment_flops", 0.0)) / args.steps,
                "max_rel_eig_diff_vs_record": diff}

    # per-config block before the CPU samples: the host BLAS threads those
    # leave behind slow the host-side work of config 2's batch (94 vs 74 ms)
    per_cfg = None
    if rank == 0 and world == 1 and not args.no_per_config:
        del dp
        torch.cuda.empty_cache()
        per_cfg = per_config_block()

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

    int8_roof = None
    if rank == 0:
        try:
            int8_roof = int8_kernel_roofline()
        except Exception as exc:  # the measurement is evidence, not the product: report why it is missing
            int8_roof = {"error": repr(exc)}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": per_step, "higher_is_better": True,
            "scaling": "strong" if node_split else "weak",
            "vs_baseline": None, "dtype": DTYPE, "data": "synthetic (seeded BASELINE config 4)",
            "config": dict(bench_config(wl), **({"parallelism": "one GEP split by quadrature node over the ranks, one "
                                                                       "all-reduce of the moment blocks per pass"}
                                                      if node_split else {})),
            "roofline": {"bound": "tensor", "kernel": "batched zgetrf (K2: panel + trailing updates; the k = 512 "
                                                      "updates on int8 tensor cores, the rest on FP64 DMMA)",
                         "achieved": lu_tflops, "peak": FP64_DMMA_PEAK_TFLOPS, "unit": "TFLOP/s",
                         "frac": lu_tflops / FP64_DMMA_PEAK_TFLOPS,
                         "peak_source": "measured DMMA.8x8x4 FP64 peak (tools/fp64_peak.cu; "
                                        "MEASURED_PEAKS.json has no FP64 entry)",
                         "algorithmic": "8 n^3 / 3 per pencil x 128 pencils per step (FP64-equivalent flops)",
                         "note": "frac exceeds 1 because 82 % of the LU's flops (the k = 512 trailing updates) run as "
                                 "exact int8 slice products on tcgen05 (4.57 POPS measured) instead of FP64 DMMA "
                                 "(37.1 TF/s): see int8_kernel for that kernel against its own peak, and "
                                 "variants.fp64_dmma for the all-FP64 path",
                         "int8_kernel": int8_roof,
                         **lu_traffic()},
            "lu_plus_moment_stage": {"tflops": stage_tflops, "frac_of_fp64_peak": stage_tflops / FP64_DMMA_PEAK_TFLOPS,
                                     "flops_per_step": stage_flops / args.steps,
                                     "ms_per_step": stage_ms / args.steps},
            "stage_ms_per_step": {k: v / args.steps for k, v in sorted(stages.items())},
            "time_per_gep_s": per_step / 1e3,
            "eigenpairs_per_s": pairs * (1 if node_split else world) / (per_step / 1e3),
            # shifted solves = pencils x passes; RHS columns = sum of n_linear_solves
            "shifted_solves_per_s": (last.stats.n_factorizations * max(iters or [1])) * world / (per_step / 1e3),
            "rhs_columns_per_s": solves * world / (per_step / 1e3),
            "eigenpairs": counts, "iterations": iters,
            # the reference's residual metric (solvers.py:140-147) of the returned pairs, computed in FP64
            "max_residual": max([float(r.residuals.max()) for r in last.results if r is not None] or [None]),
            "n_factorizations": last.stats.n_factorizations, "n_linear_solves": solves,
            "executed_flops_per_step": stage_flops / args.steps,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "seconds_per_step": e2e_s},
            "gpu_launches": launches,
            "clocks": clocks.summary(),
        }
        if variants:
            line["variants"] = variants
        if per_cfg:
            line["per_config"] = per_cfg
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
