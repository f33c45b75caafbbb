set -u
mkdir -p gpurun_out
O=gpurun_out/r02w
timeout 900 python -m pytest tests/test_dist.py tests/test_gpu_admm.py -q -p no:cacheprovider > ${O}_pytest.log 2>&1; echo "pytest exit=$?"; tail -2 ${O}_pytest.log
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
   --log-file ${O}_kpcg_launches.csv python tools/kpcg_probe.py 30 1 > ${O}_kpcg_list.log 2>&1; echo "list exit=$?"
python tools/launch_list.py ${O}_kpcg_launches.csv > ${O}_kpcg_launch_summary.txt 2>&1; head -12 ${O}_kpcg_launch_summary.txt
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"k_pcg\b|k_pcg\(" -c 1 \
   -o ${O}_k_pcg python tools/kpcg_probe.py 30 1 > ${O}_kpcg_ncu.log 2>&1; echo "ncu exit=$?"
python tools/ncu_summary.py ${O}_k_pcg.ncu-rep > ${O}_k_pcg_ncu_full.txt 2>/dev/null; head -40 ${O}_k_pcg_ncu_full.txt
