mkdir -p gpurun_out
DABD_GPU_NO_GRAPH=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
    --cache-control none --csv --log-file gpurun_out/r02ap_pour_launches.csv python tools/launch_window_pour.py 1 \
    > gpurun_out/r02ap_pour_window.log 2>&1; echo "exit=$?"
python tools/launch_list.py gpurun_out/r02ap_pour_launches.csv > gpurun_out/r02ap_pour_launch_summary.txt 2>&1
head -30 gpurun_out/r02ap_pour_launch_summary.txt; tail -2 gpurun_out/r02ap_pour_window.log
