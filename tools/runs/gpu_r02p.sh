set -u
mkdir -p gpurun_out
O=gpurun_out/r02p
timeout 2400 compute-sanitizer --tool memcheck --print-limit 3 --show-backtrace device python tools/crit3_probe.py 300 > ${O}_memcheck.txt 2>&1; echo "memcheck exit=$?"
grep -m5 -A25 "Invalid\|=========.*Error" ${O}_memcheck.txt | head -80
tail -5 ${O}_memcheck.txt
