set -u
mkdir -p gpurun_out
O=gpurun_out/r02e
./tools/exchange_probe > ${O}_exchange_probe.jsonl 2>&1; echo "probe exit=$?"
for sp in 0 2; do
  DABD_GPU_PCG_SPREAD=$sp timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > ${O}_bench_sp$sp.json 2>&1; echo "bench sp$sp exit=$?"
  DABD_GPU_PCG_SPREAD=$sp python tools/pcg_phases.py pile-1k 0:0 0:15 > ${O}_phases_sp$sp.txt 2>&1
done
timeout 300 python tools/admm_ab.py cubes-64 2 0 8 > ${O}_admm_ab_cubes.jsonl 2>&1; echo "ab cubes exit=$?"
timeout 300 python tools/admm_ab.py funnel-analog 2 0 12 > ${O}_admm_ab_funnel.jsonl 2>&1; echo "ab funnel exit=$?"
timeout 600 python tools/admm_ab.py pour-10k 8 30 3 > ${O}_admm_ab_pour.jsonl 2>&1; echo "ab pour exit=$?"
timeout 900 python -m pytest tests/test_gpu_admm.py tests/test_dist.py tests/test_gpu_acceptance.py tests/test_gpu_scale_parity.py -k "not pour_10k" -q -p no:cacheprovider --durations=10 > ${O}_pytest.log 2>&1; echo "pytest exit=$?"
