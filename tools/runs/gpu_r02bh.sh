# N>1 functional check on the final code: 2 ranks sharing one GPU (device ADMM loop over IPC-mapped
# peer slots), the strong mode at N=2, and the reference arm at N=2 (rank 0 only)
set -u
mkdir -p gpurun_out
O=gpurun_out/r02bh
DABD_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 > ${O}_bench_n2_shared.json 2> ${O}_bench_n2_shared.err; echo "n2 exit=$?"; tail -c 400 ${O}_bench_n2_shared.json
DABD_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --mode strong --steps 2 --warmup 3 > ${O}_bench_strong_n2_shared.json 2> ${O}_bench_strong_n2_shared.err; echo "strong n2 exit=$?"; tail -c 400 ${O}_bench_strong_n2_shared.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --impl reference --gpus 2 --steps 2 --warmup 3 > ${O}_bench_ref_n2.json 2> ${O}_bench_ref_n2.err; echo "ref n2 exit=$?"; tail -c 300 ${O}_bench_ref_n2.json
