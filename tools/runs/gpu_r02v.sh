set -u
mkdir -p gpurun_out
O=gpurun_out/r02v
for f in 1 2 3 5; do
  export DABD_GPU_PCG_ETA_FACTOR=$f
  b=$(timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); r=d['roofline']; print(round(d['value'],2), d['newton_iters_per_step'], d['pcg_iters_per_step'], round(r['avg_launch_us'],1))")
  t=$(timeout 600 python -m pytest tests/test_gpu_scale_parity.py::test_pile_1k_bench_settings tests/test_gpu_solver.py::test_bench_settings_match_oracle_on_a_pile tests/test_gpu_acceptance.py -q -p no:cacheprovider 2>&1 | tail -1)
  echo "factor=$f bench: $b | tests: $t"
done
