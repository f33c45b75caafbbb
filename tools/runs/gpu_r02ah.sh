set -u
mkdir -p gpurun_out
O=gpurun_out/r02ah
for k in k_contact_select k_body_terms k_assemble k_energy; do
  DABD_GPU_NO_GRAPH=1 timeout 900 ncu --profile-from-start off --set full --clock-control none --cache-control none --import-source on \
     -k regex:"^${k}" -s 30 -c 1 -o ${O}_${k} python tools/launch_window.py 1 > ${O}_${k}_ncu.log 2>&1; echo "ncu $k exit=$?"
  python tools/ncu_summary.py ${O}_${k}.ncu-rep > ${O}_${k}_ncu_full.txt 2>/dev/null
  grep -E "gpu__time_duration|fp64|warps_active|sm__throughput" ${O}_${k}_ncu_full.txt
done
