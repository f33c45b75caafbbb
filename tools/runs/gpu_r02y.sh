set -u
mkdir -p gpurun_out
O=gpurun_out/r02y
for cfg in "1 1" "0 1" "1 0"; do
  set -- $cfg
  DABD_GPU_PCG_WARM=$1 DABD_GPU_PCG_ETA=$( [ $2 = 1 ] && echo 1e-4 || echo 0 ) timeout 600 python tools/kpcg_probe.py 30 1 > ${O}_kpcg_w$1_i$2.log 2>&1; echo "warm=$1 inexact=$2: $(tail -1 ${O}_kpcg_w$1_i$2.log)"
done
timeout 900 python -m pytest tests/test_gpu_scale_parity.py tests/test_gpu_solver.py -q -p no:cacheprovider 2>&1 | tail -2
timeout 900 python tools/scale_probe.py sweep-100k:8:5 pour-10k:0:5 > ${O}_scale.jsonl 2>&1; cat ${O}_scale.jsonl
