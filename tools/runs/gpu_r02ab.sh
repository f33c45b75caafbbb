set -u
mkdir -p gpurun_out
O=gpurun_out/r02ab
timeout 900 python -m pytest tests/test_dist.py -x -q -p no:cacheprovider --durations=20 > ${O}_dist.log 2>&1; echo "dist exit=$?"; tail -30 ${O}_dist.log
timeout 600 python -m pytest tests/test_gpu_admm.py tests/test_gpu_scale_parity.py -q -p no:cacheprovider 2>&1 | tail -2
