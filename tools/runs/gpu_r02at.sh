set -u
mkdir -p gpurun_out
O=gpurun_out/r02at
for pr in 0 1; do DABD_GPU_PCG_PAIRS=$pr timeout 300 python tools/pcg_phases.py pile-1k 0:0 > ${O}_phases_p$pr.txt 2>&1; echo "pairs=$pr"; head -24 ${O}_phases_p$pr.txt | tail -22; done
DABD_GPU_PCG_PAIRS=1 timeout 900 python -m pytest tests/test_gpu_solver.py tests/test_gpu_admm.py tests/test_gpu_scale_parity.py tests/test_gpu_edge.py -q -p no:cacheprovider > ${O}_pytest_pairs.log 2>&1; echo "pytest pairs exit=$?"; grep -E "FAILED|passed|failed|^E  " ${O}_pytest_pairs.log | head -30
