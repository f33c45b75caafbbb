#!/bin/bash
# Round-2 measurement bundle (one B200, under gpurun):
#   FP64 peak, bench line, launch lists (bench command in graph mode, eager
#   window), ncu --set full of the cluster PCG with source, kernel breakdown.
set -u
OUT=gpurun_out
TAG=${1:-r02}
mkdir -p $OUT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu && ./tools/fp64_peak > $OUT/${TAG}_fp64_peak.json
echo "fp64 exit=$?"
timeout 600 python bench.py > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err
echo "bench exit=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file $OUT/${TAG}_launches_benchcmd.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    > $OUT/${TAG}_launches_benchcmd.log 2>&1
echo "launch list (bench cmd) exit=$?"
DABD_GPU_NO_GRAPH=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/${TAG}_launches.csv python tools/launch_window.py 2 > $OUT/${TAG}_launches_window.log 2>&1
echo "launch window exit=$?"
python tools/launch_list.py $OUT/${TAG}_launches.csv > $OUT/${TAG}_launch_summary.txt 2>&1
for ks in ${KERNELS:-k_pcg_cluster:100}; do
    k=${ks%%:*}; s=${ks##*:}
    DABD_GPU_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${k}" -s $s -c 1 \
        -o $OUT/${TAG}_${k} python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
        > $OUT/${TAG}_${k}_ncu.log 2>&1
    echo "ncu $k exit=$?"
    python tools/ncu_summary.py $OUT/${TAG}_${k}.ncu-rep > $OUT/${TAG}_${k}_ncu_full.txt 2>/dev/null
done
