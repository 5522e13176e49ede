for cfg in "0 0 64" "1 0 64" "1 146 16" "1 144 16" "1 140 8"; do
  set -- $cfg
  echo "PIPELINE=$1 GEMM_CAP=$2 COOP_CAP=$3"
  CIRR_PIPELINE=$1 CIRR_GEMM_CAP=$2 CIRR_COOP_CAP=$3 timeout 300 python bench.py --steps 2 --warmup 2 --e2e-steps 1 --no-variants --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['eigenpairs'])"
done
