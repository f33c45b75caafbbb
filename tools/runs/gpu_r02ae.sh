set -u
mkdir -p gpurun_out
for cfg in "2 1e-4 2" "1 1e-4 2" "2 1e-3 2" "2 1e-4 1" "2 1e-3 1" "2 1e-2 2"; do
  set -- $cfg
  b=$(DABD_GPU_PCG_WARM=$1 DABD_GPU_PCG_ETA=$2 DABD_GPU_PCG_ETA_FACTOR=$3 timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); r=d['roofline']; print(round(d['value'],2), d['newton_iters_per_step'], d['pcg_iters_per_step'], round(r['avg_launch_us'],1))")
  echo "warm=$1 eta=$2 factor=$3: $b"
done
