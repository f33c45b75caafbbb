set -u
mkdir -p gpurun_out
O=gpurun_out/r02t
timeout 600 python -m pytest tests/test_gpu_sim3d.py -q -p no:cacheprovider > ${O}_sim3d.log 2>&1; echo "sim3d exit=$?"; grep -E "^E  |passed|failed" ${O}_sim3d.log | head -12
timeout 1700 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > ${O}_pytest_gpu.log 2>&1; echo "pytest exit=$?"; tail -16 ${O}_pytest_gpu.log
