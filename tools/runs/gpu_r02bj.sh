# A/B on one box: A = flat Newton body (HEAD default), B = + the first line-search trial outside the
# WHILE(ls) node (DABD_GPU_LS_FIRST_FLAT=1); then the GPU suite and smoke on B
set -u
mkdir -p gpurun_out
for v in A B A B; do
  if [ $v = B ]; then export DABD_GPU_LS_FIRST_FLAT=1; else unset DABD_GPU_LS_FIRST_FLAT; fi
  timeout 600 python bench.py --steps 20 --no-cpu-baseline > gpurun_out/r02bj_$v.json 2>gpurun_out/r02bj_$v.err
  python -c "import json; d=json.load(open('gpurun_out/r02bj_$v.json')); print('$v', round(d['value'],2), 'e2e', round(d['e2e']['value'],2), d['newton_iters_per_step'], d['pcg_iters_per_step'], d['gpu_launches'])"
done
export DABD_GPU_LS_FIRST_FLAT=1
timeout 1700 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02bj_pytest_gpu.log 2>&1; echo "pytest exit=$?"; tail -3 gpurun_out/r02bj_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02bj_smoke.log 2>&1; echo "smoke exit=$?"; tail -1 gpurun_out/r02bj_smoke.log
