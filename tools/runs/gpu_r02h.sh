bash tools/pcg_ab.sh r02h_rcp "DABD_GPU_PCG_FAST_RCP=1" "DABD_GPU_PCG_FAST_RCP=0" > gpurun_out/r02h_ab_rcp.txt 2>&1
bash tools/pcg_ab.sh r02h_rf "DABD_GPU_PCG_REMOTE_FIRST=1" "DABD_GPU_PCG_REMOTE_FIRST=0" > gpurun_out/r02h_ab_rf.txt 2>&1
