# tools/graph_gap_probe.cu on the GPU box, one process per configuration
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gap tools/graph_gap_probe.cu || exit 1
for b in 16 148; do for p in 0 1; do for m in top while; do timeout 20 /tmp/gap $b $p $m || echo "{\"blocks\": $b, \"pdl\": $p, \"mode\": \"$m\", \"failed\": $?}"; done; done; done
