set -u
mkdir -p gpurun_out
O=gpurun_out/r02o
timeout 300 python tools/crit3_probe.py 300 > ${O}_a1.txt 2>&1; echo "a1: $(tail -1 ${O}_a1.txt)"
timeout 300 python tools/crit3_probe.py 300 > ${O}_a2.txt 2>&1; echo "a2: $(tail -1 ${O}_a2.txt)"
DABD_GPU_PCG_ETA=0 timeout 300 python tools/crit3_probe.py 300 > ${O}_b.txt 2>&1; echo "b eta0: $(tail -1 ${O}_b.txt)"
DABD_GPU_ADMM_HOST=1 timeout 300 python tools/crit3_probe.py 300 > ${O}_c.txt 2>&1; echo "c host: $(tail -1 ${O}_c.txt)"
