set -u
mkdir -p gpurun_out
O=gpurun_out/r02ai
for i in 1 2; do timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); r=d['roofline']; print(round(d['value'],2), d['newton_iters_per_step'], d['pcg_iters_per_step'], round(r['avg_launch_us'],1))"; done
python tools/pcg_phases.py pile-1k 0:0 > ${O}_phases.txt 2>&1; tail -12 ${O}_phases.txt
timeout 900 python -m pytest tests/test_gpu_solver.py tests/test_gpu_admm.py tests/test_gpu_scale_parity.py -q -p no:cacheprovider 2>&1 | tail -1
