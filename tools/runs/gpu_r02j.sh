set -u
mkdir -p gpurun_out
O=gpurun_out/r02j
timeout 300 python tools/admm_ab.py blocked-merge 2 0 3 > ${O}_admm_ab_blocked.jsonl 2>&1; echo "ab blocked exit=$?"
timeout 300 python tools/admm_ab.py drop-grid-4 4 0 8 > ${O}_admm_ab_dg4.jsonl 2>&1; echo "ab dg4 exit=$?"
timeout 900 python -m pytest tests/test_dist.py tests/test_gpu_admm.py tests/test_gpu_acceptance.py -q -p no:cacheprovider > ${O}_pytest.log 2>&1; echo "pytest exit=$?"
timeout 600 python tools/make_pour_fixture.py start > ${O}_pour_start.log 2>&1; echo "pour start exit=$?"
timeout 900 python bench.py --mode strong --steps 5 --warmup 3 > ${O}_bench_strong.json 2> ${O}_bench_strong.err; echo "strong exit=$?"
