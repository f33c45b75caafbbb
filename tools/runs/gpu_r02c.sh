# PCG send spreading / fold experiments
set -u
mkdir -p gpurun_out
O=gpurun_out/r02c
for cfg in "0 0" "1 0" "1 1" "0 1"; do
  set -- $cfg
  export DABD_GPU_PCG_SPREAD=$1 DABD_GPU_PCG_FOLD_ALL=$2
  timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > ${O}_bench_s$1f$2.json 2>&1; echo "bench $cfg exit=$?"
  python tools/pcg_phases.py pile-1k 0:0 0:15 > ${O}_phases_s$1f$2.txt 2>&1
done
export DABD_GPU_PCG_SPREAD=1 DABD_GPU_PCG_FOLD_ALL=1
timeout 900 python -m pytest tests/test_gpu_solver.py tests/test_gpu_admm.py -x -q -p no:cacheprovider --durations=10 > ${O}_pytest.log 2>&1; echo "pytest exit=$?"
