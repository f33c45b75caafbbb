set -u
mkdir -p gpurun_out
O=gpurun_out/r02ad
timeout 1700 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > ${O}_pytest_gpu.log 2>&1; echo "pytest exit=$?"; tail -15 ${O}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > ${O}_smoke.log 2>&1; echo "smoke exit=$?"; tail -1 ${O}_smoke.log
timeout 900 python bench.py > ${O}_bench.json 2> ${O}_bench.err; echo "bench exit=$?"; python -c "import json; d=json.load(open('${O}_bench.json')); r=d['roofline']; print(round(d['value'],2), 'e2e', round(d['e2e']['value'],2), d['newton_iters_per_step'], d['pcg_iters_per_step'], round(r['avg_launch_us'],1), d['gpu_launches'], d['cpu_baseline']['value'])"
