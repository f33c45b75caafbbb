set -u
mkdir -p gpurun_out
O=gpurun_out/r02as
for pr in 0 1 0 1; do echo "pairs=$pr"; DABD_GPU_PCG_PAIRS=$pr timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>${O}_bench_p$pr.err | python -c "import json,sys; d=json.load(sys.stdin); r=d['roofline']; print(round(d['value'],2), d['newton_iters_per_step'], d['pcg_iters_per_step'], round(r['avg_launch_us'],1))"; done
DABD_GPU_PCG_PAIRS=1 timeout 900 python -m pytest tests/test_gpu_solver.py tests/test_gpu_admm.py tests/test_gpu_scale_parity.py tests/test_gpu_edge.py -q -x -p no:cacheprovider > ${O}_pytest_pairs.log 2>&1; echo "pytest pairs exit=$?"; tail -15 ${O}_pytest_pairs.log
