set -u
for cfg in "1e-3 1" "1e-2 1"; do
  set -- $cfg
  export DABD_GPU_PCG_ETA=$1 DABD_GPU_PCG_ETA_FACTOR=$2
  t=$(timeout 900 python -m pytest tests/test_gpu_scale_parity.py tests/test_gpu_solver.py tests/test_gpu_acceptance.py tests/test_gpu_audit.py -q -p no:cacheprovider 2>&1 | tail -1)
  b=$(timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); r=d['roofline']; print(round(d['value'],2), d['newton_iters_per_step'], d['pcg_iters_per_step'])")
  echo "eta=$1 factor=$2 | tests: $t | bench: $b"
done
