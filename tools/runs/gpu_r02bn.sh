# A/B on one box: A = k_ccd beside k_ccd_prep (HEAD default), B = both in one launch of disjoint block
# ranges (DABD_GPU_CCD_MERGED=1); then the GPU suite and smoke on B
set -u
mkdir -p gpurun_out
for v in A B A B; do
  if [ $v = B ]; then export DABD_GPU_CCD_MERGED=1; else unset DABD_GPU_CCD_MERGED; fi
  timeout 600 python bench.py --steps 20 --no-cpu-baseline > gpurun_out/r02bn_$v.json 2>gpurun_out/r02bn_$v.err
  python -c "import json; d=json.load(open('gpurun_out/r02bn_$v.json')); print('$v', round(d['value'],2), 'e2e', round(d['e2e']['value'],2), d['newton_iters_per_step'], d['pcg_iters_per_step'], d['gpu_launches'])"
done
export DABD_GPU_CCD_MERGED=1
timeout 1700 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02bn_pytest_gpu.log 2>&1; echo "pytest exit=$?"; tail -3 gpurun_out/r02bn_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02bn_smoke.log 2>&1; echo "smoke exit=$?"; tail -1 gpurun_out/r02bn_smoke.log
