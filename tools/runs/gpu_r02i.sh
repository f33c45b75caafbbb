set -u
mkdir -p gpurun_out
O=gpurun_out/r02i
./tools/exchange_probe > ${O}_exchange_probe.jsonl 2>&1; echo "probe exit=$?"
timeout 300 python tools/admm_ab.py cubes-64 2 0 8 > ${O}_admm_ab_cubes.jsonl 2>&1; echo "ab cubes exit=$?"
timeout 300 python tools/admm_ab.py funnel-analog 2 0 12 > ${O}_admm_ab_funnel.jsonl 2>&1; echo "ab funnel exit=$?"
timeout 600 python tools/admm_ab.py pour-10k 8 30 3 > ${O}_admm_ab_pour.jsonl 2>&1; echo "ab pour exit=$?"
timeout 900 python -m pytest tests/test_gpu_admm.py tests/test_dist.py tests/test_gpu_acceptance.py tests/test_balance.py tests/test_gpu_scale_parity.py tests/test_cpp_adapter.py -k "not pour_10k" -q -p no:cacheprovider --durations=5 > ${O}_pytest.log 2>&1; echo "pytest exit=$?"
DABD_GPU_ADMM_PROFILE=1 timeout 900 python tools/scale_probe.py pour-10k:8:5 sweep-100k:8:3 > ${O}_scale_probe.jsonl 2> ${O}_scale_profile.txt; echo "scale exit=$?"
timeout 900 python tools/scale_probe.py pour-10k:8:5 sweep-100k:8:3 > ${O}_scale_probe_noprof.jsonl 2>&1; echo "scale2 exit=$?"
