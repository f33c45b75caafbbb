# Final round-2 measurement bundle on the committed code, plus ncu of the changed trial-energy kernel
set -u
bash tools/profile_r02z.sh r02bb
OUT=gpurun_out
DABD_GPU_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_energy -s 300 -c 1 \
    -o $OUT/r02bb_k_energy python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $OUT/r02bb_ncu_energy.log 2>&1
echo "ncu energy exit=$?"
python tools/ncu_summary.py $OUT/r02bb_k_energy.ncu-rep > $OUT/r02bb_k_energy_ncu_full.txt 2>/dev/null
