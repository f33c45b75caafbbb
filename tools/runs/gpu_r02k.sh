set -u
mkdir -p gpurun_out
O=gpurun_out/r02k
for eta in 0 1e-6 1e-4; do
  DABD_GPU_PCG_ETA=$eta timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > ${O}_bench_eta$eta.json 2>&1; echo "bench $eta exit=$?"
  DABD_GPU_PCG_ETA=$eta timeout 900 python -m pytest tests/test_gpu_scale_parity.py::test_pile_1k_bench_settings tests/test_gpu_solver.py tests/test_gpu_admm.py::test_drop_grid_four_workers_default_solver tests/test_gpu_acceptance.py -q -p no:cacheprovider > ${O}_pytest_eta$eta.log 2>&1; echo "pytest $eta exit=$?"
done
