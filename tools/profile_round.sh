#!/bin/bash
# Round profiling bundle (run under gpurun on ONE B200):
#   1. launch list of the bench command (cold-cache, serialised: shares only)
#   2. ncu --set full of the top kernels (one launch each, from the settled pile)
#   3. per-kernel eager breakdown next to the graph step time
# ncu cannot profile kernel nodes of a graph with conditional nodes, so the
# profiled runs use DABD_GPU_NO_GRAPH=1: the same kernels with the same
# arguments, launched eagerly from the host-driven Newton loop.
# Outputs land in gpurun_out/; summaries are copied into profiles/ by hand.
set -u
OUT=gpurun_out
mkdir -p $OUT
TAG=${1:-r01}
export DABD_GPU_NO_GRAPH=1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/${TAG}_launches.csv python tools/launch_window.py 2 \
    > $OUT/${TAG}_launches_bench.log 2>&1
echo "launch list exit=$?"
# kernel:skip (launches of that kernel before the captured one: ~40 settle frames)
for ks in ${KERNELS:-k_pcg_cluster:500 k_assemble:500 k_contact_select:500 k_body_terms:500 k_energy:500}; do
    k=${ks%%:*}; s=${ks##*:}
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:"${k}" -s $s -c 1 \
        -o $OUT/${TAG}_${k} python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
        > $OUT/${TAG}_${k}_ncu.log 2>&1
    echo "ncu $k exit=$?"
    python tools/ncu_summary.py $OUT/${TAG}_${k}.ncu-rep > $OUT/${TAG}_${k}_ncu_full.txt 2>/dev/null
done
python tools/launch_list.py $OUT/${TAG}_launches.csv > $OUT/${TAG}_launch_summary.txt 2>&1
unset DABD_GPU_NO_GRAPH
timeout 600 python tools/kernel_breakdown.py pile-1k 40 3 > $OUT/${TAG}_breakdown.json 2> $OUT/${TAG}_breakdown.err
echo "breakdown exit=$?"
