# A/B on one box: A = HEAD, B = k_assemble prefetches each active contact's blocks into L1;
# then the GPU suite on B
set -u
mkdir -p gpurun_out
L=paper_2605_15875_b200
for v in A B A B; do
  cp $L/libdabd_gpu_$v.so $L/libdabd_gpu.so
  timeout 600 python bench.py --steps 20 --no-cpu-baseline > gpurun_out/r02bf_$v.json 2>gpurun_out/r02bf_$v.err
  python -c "import json; d=json.load(open('gpurun_out/r02bf_$v.json')); print('$v', round(d['value'],2), 'e2e', round(d['e2e']['value'],2), d['newton_iters_per_step'], d['pcg_iters_per_step'], d['gpu_launches'])"
done
rm -f $L/libdabd_gpu_A.so $L/libdabd_gpu_B.so
timeout 1700 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02bf_pytest_gpu.log 2>&1; echo "pytest exit=$?"; tail -3 gpurun_out/r02bf_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02bf_smoke.log 2>&1; echo "smoke exit=$?"; tail -1 gpurun_out/r02bf_smoke.log
