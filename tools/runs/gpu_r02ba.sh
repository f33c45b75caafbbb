# A/B on one box: A = r02ax code, B = + load hoists in k_assemble / k_ccd
set -u
mkdir -p gpurun_out
L=paper_2605_15875_b200
for v in A B A B; do
  cp $L/libdabd_gpu_$v.so $L/libdabd_gpu.so
  timeout 600 python bench.py --steps 20 --no-cpu-baseline > gpurun_out/r02ba_$v.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/r02ba_$v.json')); print('$v', round(d['value'],2), 'e2e', round(d['e2e']['value'],2))"
done
