set -u
mkdir -p gpurun_out
O=gpurun_out/r02g
for rf in 1 0; do
  DABD_GPU_PCG_REMOTE_FIRST=$rf timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > ${O}_bench_rf$rf.json 2>&1; echo "bench rf$rf exit=$?"
  DABD_GPU_PCG_REMOTE_FIRST=$rf python tools/pcg_phases.py pile-1k 0:0 0:15 > ${O}_phases_rf$rf.txt 2>&1
done
timeout 600 python -m pytest tests/test_gpu_solver.py tests/test_gpu_admm.py tests/test_gpu_scale_parity.py -k "not pour_10k and not sweep" -q -p no:cacheprovider > ${O}_pytest.log 2>&1; echo "pytest exit=$?"
timeout 900 python tools/scale_probe.py pour-10k:8:5 sweep-100k:8:3 > ${O}_scale_probe.jsonl 2>&1; echo "scale exit=$?"
