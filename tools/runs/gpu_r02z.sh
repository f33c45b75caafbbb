set -u
timeout 600 python -m pytest tests/test_gpu_sim3d.py -q -p no:cacheprovider > gpurun_out/r02z_sim3d.log 2>&1; echo "sim3d exit=$?"; tail -1 gpurun_out/r02z_sim3d.log
bash tools/profile_r02z.sh r02z
