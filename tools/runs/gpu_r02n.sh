set -u
mkdir -p gpurun_out
O=gpurun_out/r02n
export CUDA_LAUNCH_BLOCKING=1
timeout 300 python tools/crit3_probe.py 300 density-sweep-10000 > ${O}_a.txt 2>&1; echo "a: $(tail -1 ${O}_a.txt)"
DABD_GPU_PCG_ETA=0 timeout 300 python tools/crit3_probe.py 300 density-sweep-10000 > ${O}_b.txt 2>&1; echo "b eta0: $(tail -1 ${O}_b.txt)"
DABD_GPU_ADMM_HOST=1 timeout 300 python tools/crit3_probe.py 300 density-sweep-10000 > ${O}_c.txt 2>&1; echo "c host: $(tail -1 ${O}_c.txt)"
CRIT3_AUDIT=0 timeout 300 python tools/crit3_probe.py 300 density-sweep-10000 > ${O}_d.txt 2>&1; echo "d noaudit: $(tail -1 ${O}_d.txt)"
