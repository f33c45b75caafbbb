# fused CCD without body boxes: GPU suite, bench x2, ncu of one trial-energy launch
set -u
mkdir -p gpurun_out
O=gpurun_out/r02bc
timeout 900 python bench.py > ${O}_bench.json 2> ${O}_bench.err; python -c "import json; d=json.load(open('${O}_bench.json')); print('default bench', round(d['value'],2), 'e2e', round(d['e2e']['value'],2), d['gpu_launches'], d['clocks'])"
timeout 1700 python -m pytest tests -m gpu -q -p no:cacheprovider > ${O}_pytest_gpu.log 2>&1; echo "pytest exit=$?"; tail -3 ${O}_pytest_gpu.log
timeout 900 python bench.py > ${O}_bench2.json 2> ${O}_bench2.err; python -c "import json; d=json.load(open('${O}_bench2.json')); print('default bench', round(d['value'],2), 'e2e', round(d['e2e']['value'],2), d['gpu_launches'], d['clocks'])"
DABD_GPU_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_energy -s 60 -c 1 \
    -o ${O}_k_energy python bench.py --steps 1 --warmup 3 --no-cpu-baseline > ${O}_ncu_energy.log 2>&1
echo "ncu energy exit=$?"
python tools/ncu_summary.py ${O}_k_energy.ncu-rep > ${O}_k_energy_ncu_full.txt 2>/dev/null
