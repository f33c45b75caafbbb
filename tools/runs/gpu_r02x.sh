set -u
mkdir -p gpurun_out
O=gpurun_out/r02x
for g in 1 0; do
  DABD_GPU_PCG_GRID=$g timeout 600 python tools/kpcg_probe.py 30 1 > ${O}_kpcg_g$g.log 2>&1; echo "grid=$g: $(tail -1 ${O}_kpcg_g$g.log)"
done
timeout 900 python tools/scale_probe.py sweep-100k:8:5 > ${O}_scale.jsonl 2>&1; cat ${O}_scale.jsonl
timeout 900 python -m pytest tests/test_gpu_scale_parity.py tests/test_gpu_solver.py -q -p no:cacheprovider 2>&1 | tail -2
