set -u
mkdir -p gpurun_out
O=gpurun_out/r02f
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > ${O}_bench.json 2>&1; echo "bench exit=$?"
python tools/pcg_phases.py pile-1k 0:0 0:15 > ${O}_phases.txt 2>&1; echo "phases exit=$?"
timeout 900 python -m pytest tests/test_gpu_solver.py tests/test_gpu_admm.py tests/test_gpu_scale_parity.py -k "not pour_10k and not sweep" -q -p no:cacheprovider --durations=5 > ${O}_pytest.log 2>&1; echo "pytest exit=$?"
