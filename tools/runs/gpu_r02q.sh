set -u
mkdir -p gpurun_out
O=gpurun_out/r02q
timeout 600 python -m pytest tests/test_gpu_sim3d.py -x -q -p no:cacheprovider > ${O}_sim3d.log 2>&1; echo "sim3d exit=$?"
tail -30 ${O}_sim3d.log
timeout 1500 compute-sanitizer --tool memcheck --print-limit 3 --show-backtrace device python tools/crit3_probe.py 300 > ${O}_memcheck.txt 2>&1; echo "memcheck exit=$?"
grep -m3 -A10 "Invalid" ${O}_memcheck.txt | head -40; tail -14 ${O}_memcheck.txt
