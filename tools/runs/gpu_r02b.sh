# PCG experiments: per-CTA phase timelines and the rows-per-CTA knob
set -u
mkdir -p gpurun_out
O=gpurun_out/r02b
python tools/pcg_phases.py pile-1k 0:0 0:15 5:0 15:0 > ${O}_phases.txt 2>&1; echo "phases exit=$?"
for mr in 32 64 128; do
  DABD_GPU_PCG_MIN_ROWS=$mr timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > ${O}_bench_mr$mr.json 2>&1; echo "bench $mr exit=$?"
  DABD_GPU_PCG_MIN_ROWS=$mr python tools/pcg_phases.py pile-1k 0:0 > ${O}_phases_mr$mr.txt 2>&1
done
