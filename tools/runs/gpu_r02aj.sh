set -u
mkdir -p gpurun_out
O=gpurun_out/r02aj
timeout 1700 python -m pytest tests -m gpu -q -p no:cacheprovider > ${O}_pytest_gpu.log 2>&1; echo "pytest exit=$?"; tail -3 ${O}_pytest_gpu.log
for i in 1 2; do timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); r=d['roofline']; print(round(d['value'],2), d['newton_iters_per_step'], d['pcg_iters_per_step'], round(r['avg_launch_us'],1), d['gpu_launches'])"; done
timeout 900 python bench.py > ${O}_bench.json 2> ${O}_bench.err; python -c "import json; d=json.load(open('${O}_bench.json')); print('default bench', round(d['value'],2), 'e2e', round(d['e2e']['value'],2), d['gpu_launches'])"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
