# A/B of PCG knobs on one box: ABAB order, bench (20 steps) per run.
# usage: bash tools/pcg_ab.sh TAG "ENV_A" "ENV_B"
TAG=$1; A=$2; B=$3
mkdir -p gpurun_out
for rep in 1 2; do
  for v in A B; do
    if [ $v = A ]; then E=$A; else E=$B; fi
    env $E timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_${v}${rep}.json 2>/dev/null
    python - "$v" "$E" gpurun_out/${TAG}_${v}${rep}.json <<'PY'
import json, sys
d = json.load(open(sys.argv[3])); r = d["roofline"]
print(sys.argv[1], sys.argv[2], round(d["value"], 2), "steps/s", round(r["avg_launch_us"], 1), "us/launch",
      round(r["avg_launch_us"] / r["iterations_per_launch"], 3), "us/iter", d["pcg_iters_per_step"])
PY
  done
done
