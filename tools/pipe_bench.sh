# config-4 step time: batched vs pipelined with several cooperative caps
make -s >/dev/null
cat > /tmp/pb.py << 'PY'
import sys, time; sys.path.insert(0, ".")
import torch
from paper_2511_01927_b200 import DevicePencil, SolverConfig, solve_multi
from paper_2511_01927_b200 import solvers as S
from paper_2511_01927_b200 import workloads as W
wl = W.config4()
dp = DevicePencil(wl.a, wl.b, hermitian=False)
cfg = SolverConfig(n_q=64, source_cols=32, n_moments=8)
for mode in sys.argv[1:]:
    if mode == "batched":
        S._PIPELINE = False
    else:
        S._PIPELINE = True; S._COOP_CAP = int(mode)
    solve_multi(dp, wl.contours, cfg)
    torch.cuda.synchronize()
    ts = []
    for _ in range(2):
        t = time.perf_counter(); m = solve_multi(dp, wl.contours, cfg); torch.cuda.synchronize(); ts.append(time.perf_counter() - t)
    print(mode, [len(r.eigenvalues) for r in m.results], " ".join(f"{x*1e3:.0f}" for x in ts), "ms", flush=True)
PY
python /tmp/pb.py batched 0 64 32 16 8 > gpurun_out/pipe_bench.log 2>&1
