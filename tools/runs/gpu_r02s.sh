set -u
mkdir -p gpurun_out
O=gpurun_out/r02s
timeout 600 python -m pytest tests/test_gpu_sim3d.py -q -p no:cacheprovider > ${O}_sim3d.log 2>&1; echo "sim3d exit=$?"; grep -E "^E|passed|failed" ${O}_sim3d.log | head -12
for cfg in "1e-4 10" "1e-5 10" "1e-6 10" "1e-4 30" "1e-3 30"; do
  set -- $cfg
  export DABD_GPU_PCG_ETA=$1 DABD_GPU_PCG_ETA_FACTOR=$2
  r=$(timeout 600 python -m pytest tests/test_gpu_admm.py::test_drop_grid_four_workers_default_solver tests/test_gpu_scale_parity.py::test_pile_1k_bench_settings tests/test_gpu_solver.py::test_bench_settings_match_oracle_on_a_pile tests/test_gpu_acceptance.py -q -p no:cacheprovider 2>&1 | tail -1)
  b=$(timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['value'],2), d['newton_iters_per_step'], d['pcg_iters_per_step'])")
  echo "eta=$1 f=$2 | tests: $r | bench: $b"
done
