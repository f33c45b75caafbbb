set -u
mkdir -p gpurun_out
O=gpurun_out/r02u
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > ${O}_bench.json 2>&1; python -c "import json; d=json.load(open('${O}_bench.json')); r=d['roofline']; print(round(d['value'],2), d['newton_iters_per_step'], d['pcg_iters_per_step'], round(r['avg_launch_us'],1))"
python tools/pcg_phases.py pile-1k 0:0 > ${O}_phases.txt 2>&1; head -9 ${O}_phases.txt
timeout 900 python -m pytest tests/test_gpu_scale_parity.py::test_pile_1k_bench_settings tests/test_gpu_solver.py tests/test_gpu_admm.py -q -p no:cacheprovider 2>&1 | tail -2
