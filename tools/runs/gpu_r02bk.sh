# Final measurement bundle on the final code (flat fused Newton body, first trial outside WHILE(ls)), plus GPU suite and smoke
set -u
bash tools/profile_r02z.sh r02bk
OUT=gpurun_out
timeout 1700 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/r02bk_pytest_gpu.log 2>&1; echo "pytest exit=$?"; tail -3 $OUT/r02bk_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/r02bk_smoke.log 2>&1; echo "smoke exit=$?"; tail -1 $OUT/r02bk_smoke.log
timeout 900 python bench.py > $OUT/r02bk_bench2.json 2> $OUT/r02bk_bench2.err; echo "bench2 exit=$?"
