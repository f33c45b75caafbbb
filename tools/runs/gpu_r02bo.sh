set -u
mkdir -p gpurun_out
O=gpurun_out/r02bo
timeout 1700 python -m pytest tests -m gpu -q -p no:cacheprovider > ${O}_pytest_gpu.log 2>&1; echo "pytest exit=$?"; tail -3 ${O}_pytest_gpu.log
timeout 900 python bench.py > ${O}_bench.json 2> ${O}_bench.err; python -c "import json; d=json.load(open('${O}_bench.json')); print('default bench', round(d['value'],2), 'e2e', round(d['e2e']['value'],2), d['gpu_launches'], d['clocks'])"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > ${O}_smoke.log 2>&1; echo "smoke exit=$?"; tail -1 ${O}_smoke.log
