set -u
mkdir -p gpurun_out
O=gpurun_out/r02d
./tools/exchange_probe > ${O}_exchange_probe.jsonl 2>&1; echo "probe exit=$?"
python tools/pcg_phases.py pile-1k 0:0 > ${O}_phases.txt 2>&1; echo "phases exit=$?"
timeout 1700 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=40 > ${O}_pytest_gpu.log 2>&1; echo "pytest exit=$?"
