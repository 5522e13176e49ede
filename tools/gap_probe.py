"""Where does the un-staged time of a config-4 step go?  Per step: wall time, sum of the stage
timers, cudaMalloc/cudaFree counts of torch's caching allocator, free HBM."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import bench
from paper_2511_01927_b200 import DevicePencil, SolverConfig, solve_multi
from paper_2511_01927_b200 import solvers as S

wl = bench.build_workload(0)
cfg = SolverConfig(n_q=wl.n_q, source_cols=wl.source_cols, n_moments=wl.n_moments, tol=1e-10)
dp = DevicePencil(wl.a, wl.b, hermitian=False)
host = len(sys.argv) > 1 and sys.argv[1] == "host"
hp = bench.HostPencil(wl.a, wl.b, False)
for step in range(5):
    st0 = torch.cuda.memory_stats()
    timer = S.StageTimer(); S.set_stage_timer(timer)
    torch.cuda.synchronize(); t = time.perf_counter()
    solve_multi(hp if host else dp, wl.contours, cfg, seed=0)
    torch.cuda.synchronize(); wall = time.perf_counter() - t
    S.set_stage_timer(None)
    tot = timer.totals()
    st1 = torch.cuda.memory_stats()
    top = sum(v for k, v in tot.items() if "." not in k)
    free, total = torch.cuda.mem_get_info()
    print(f"step {step}: wall {wall*1e3:.0f} ms, stages {top:.0f} ms, cudaMalloc +{st1['num_device_alloc']-st0['num_device_alloc']}, "
          f"cudaFree +{st1['num_device_free']-st0['num_device_free']}, retries +{st1['num_alloc_retries']-st0['num_alloc_retries']}, "
          f"reserved {torch.cuda.memory_reserved()/2**30:.1f} GiB, driver free {free/2**30:.1f} GiB", flush=True)

# host-side time of each C-ABI entry (they are asynchronous: anything above a few ms blocks the host)
from paper_2511_01927_b200 import _lib
import collections
orig = _lib.call
acc = collections.defaultdict(lambda: [0, 0.0, 0.0])
def timed(name, *a):
    t0 = time.perf_counter(); r = orig(name, *a); dt = time.perf_counter() - t0
    e = acc[name]; e[0] += 1; e[1] += dt; e[2] = max(e[2], dt)
    return r
_lib.call = timed
S._lib.call = timed
for step in range(3):
    acc.clear()
    torch.cuda.synchronize(); t = time.perf_counter()
    solve_multi(dp, wl.contours, cfg, seed=0)
    torch.cuda.synchronize(); wall = time.perf_counter() - t
    top = sorted(acc.items(), key=lambda kv: -kv[1][1])[:4]
    print(f"probe step {step}: wall {wall*1e3:.0f} ms; host time in entries: " +
          ", ".join(f"{k} n={v[0]} sum={v[1]*1e3:.0f} ms max={v[2]*1e3:.0f} ms" for k, v in top), flush=True)
