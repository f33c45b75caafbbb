set -u
mkdir -p gpurun_out
O=gpurun_out/r02r
timeout 600 python -m pytest tests/test_gpu_sim3d.py -q -p no:cacheprovider > ${O}_sim3d.log 2>&1; echo "sim3d exit=$?"; tail -15 ${O}_sim3d.log
timeout 1700 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=20 > ${O}_pytest_gpu.log 2>&1; echo "pytest exit=$?"; tail -30 ${O}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > ${O}_smoke.log 2>&1; echo "smoke exit=$?"; tail -2 ${O}_smoke.log
