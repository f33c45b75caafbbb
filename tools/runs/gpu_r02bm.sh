# final sanity: default bench line and the reference arm on the committed tree
set -u
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r02bm_bench.json 2> gpurun_out/r02bm_bench.err; echo "bench exit=$?"
python -c "import json; d=json.load(open('gpurun_out/r02bm_bench.json')); print(round(d['value'],2), round(d['e2e']['value'],2), d['roofline']['traffic'], d['roofline']['traffic_source'], round(d['roofline']['frac'],4), d['clocks'])"
timeout 900 python bench.py --impl reference > gpurun_out/r02bm_bench_ref.json 2> gpurun_out/r02bm_bench_ref.err; echo "ref exit=$?"; tail -c 300 gpurun_out/r02bm_bench_ref.json
