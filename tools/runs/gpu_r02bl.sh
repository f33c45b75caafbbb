# cost of an IF node inside the WHILE body (graph_gap_probe modes while / if0 / if1)
set -u
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gap tools/graph_gap_probe.cu || exit 1
for r in 1 2 3; do for m in while if0 if1; do timeout 20 /tmp/gap 148 0 $m; done; done | tee gpurun_out/r02bl_graph_if_probe.jsonl
