set -u
mkdir -p gpurun_out
O=gpurun_out/r02m2
CUDA_LAUNCH_BLOCKING=1 timeout 900 python tools/crit3_probe.py 300 > ${O}_crit3.txt 2>&1; echo "crit3 exit=$?"
tail -3 ${O}_crit3.txt
