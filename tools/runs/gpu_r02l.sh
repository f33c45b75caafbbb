set -u
mkdir -p gpurun_out
O=gpurun_out/r02l
for cfg in "0 10" "1e-4 10" "1e-3 10" "1e-4 100" "1e-2 10"; do
  set -- $cfg
  DABD_GPU_PCG_ETA=$1 DABD_GPU_PCG_ETA_FACTOR=$2 timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > ${O}_bench_eta$1_f$2.json 2>&1
  python - "$1 $2" ${O}_bench_eta$1_f$2.json <<'PY'
import json, sys
d = json.load(open(sys.argv[2])); r = d["roofline"]
print(sys.argv[1], round(d["value"], 2), "steps/s", d["newton_iters_per_step"], "newton", d["pcg_iters_per_step"], "pcg", round(r["avg_launch_us"], 1), "us/launch")
PY
done
timeout 1500 python -m pytest tests -m gpu -k "not pour_10k" -q -p no:cacheprovider --durations=15 > ${O}_pytest_gpu.log 2>&1; echo "pytest exit=$?"
