#!/bin/bash
# Round-2 final measurement bundle (one B200, under gpurun): bench line,
# launch lists (graph-mode bench command; eager window with warm caches),
# ncu --set full of the cluster PCG with source, PCG phases, strong-mode and
# scale probes.
set -u
OUT=gpurun_out
TAG=${1:-r02z}
mkdir -p $OUT
timeout 900 python bench.py > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err; echo "bench exit=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/${TAG}_bench_ref.json 2> $OUT/${TAG}_bench_ref.err; echo "ref exit=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file $OUT/${TAG}_launches_benchcmd.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    > $OUT/${TAG}_launches_benchcmd.log 2>&1; echo "launch list (bench cmd) exit=$?"
DABD_GPU_NO_GRAPH=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
    --cache-control none --csv --log-file $OUT/${TAG}_launches_warm.csv python tools/launch_window.py 2 \
    > $OUT/${TAG}_launches_window.log 2>&1; echo "launch window exit=$?"
python tools/launch_list.py $OUT/${TAG}_launches_warm.csv > $OUT/${TAG}_launch_summary_warm.txt 2>&1
DABD_GPU_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pcg_cluster -s 100 -c 1 \
    -o $OUT/${TAG}_k_pcg_cluster python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $OUT/${TAG}_ncu.log 2>&1
echo "ncu exit=$?"
python tools/ncu_summary.py $OUT/${TAG}_k_pcg_cluster.ncu-rep > $OUT/${TAG}_k_pcg_cluster_ncu_full.txt 2>/dev/null
python tools/pcg_phases.py pile-1k 0:0 0:15 > $OUT/${TAG}_pcg_phases.txt 2>&1
timeout 900 python bench.py --mode strong --steps 5 --warmup 3 > $OUT/${TAG}_bench_strong.json 2>&1; echo "strong exit=$?"
timeout 900 python tools/scale_probe.py pour-10k:8:20 sweep-100k:8:5 > $OUT/${TAG}_scale_probe.jsonl 2>&1; echo "scale exit=$?"
