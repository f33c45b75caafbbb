set -u
mkdir -p gpurun_out
O=gpurun_out/r02aa
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_pcg_grid -s 20 -c 1 \
   -o ${O}_k_pcg_grid python tools/kpcg_probe.py 30 1 > ${O}_ncu.log 2>&1; echo "ncu exit=$?"
python tools/ncu_summary.py ${O}_k_pcg_grid.ncu-rep > ${O}_k_pcg_grid_ncu_full.txt 2>/dev/null; head -36 ${O}_k_pcg_grid_ncu_full.txt
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
   --log-file ${O}_launches.csv python tools/kpcg_probe.py 30 1 > ${O}_list.log 2>&1
python tools/launch_list.py ${O}_launches.csv > ${O}_launch_summary.txt 2>&1; head -8 ${O}_launch_summary.txt
