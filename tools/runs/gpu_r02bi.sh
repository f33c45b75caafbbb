# A/B on one box: A = IF(step) node around the CCD + line search (DABD_GPU_STEP_IF=1), B = flat fused
# Newton body (default); then the GPU suite and smoke on B
set -u
mkdir -p gpurun_out
for v in A B A B; do
  if [ $v = A ]; then export DABD_GPU_STEP_IF=1; else unset DABD_GPU_STEP_IF; fi
  timeout 600 python bench.py --steps 20 --no-cpu-baseline > gpurun_out/r02bi_$v.json 2>gpurun_out/r02bi_$v.err
  python -c "import json; d=json.load(open('gpurun_out/r02bi_$v.json')); print('$v', round(d['value'],2), 'e2e', round(d['e2e']['value'],2), d['newton_iters_per_step'], d['pcg_iters_per_step'], d['gpu_launches'])"
done
unset DABD_GPU_STEP_IF
timeout 1700 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02bi_pytest_gpu.log 2>&1; echo "pytest exit=$?"; tail -3 gpurun_out/r02bi_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02bi_smoke.log 2>&1; echo "smoke exit=$?"; tail -1 gpurun_out/r02bi_smoke.log
