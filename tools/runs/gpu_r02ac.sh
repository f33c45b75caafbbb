set -u
mkdir -p gpurun_out
O=gpurun_out/r02ac
timeout 900 python -m pytest tests/test_dist.py -x -q -p no:cacheprovider > ${O}_dist.log 2>&1; echo "dist exit=$?"; tail -3 ${O}_dist.log
# 2 ranks sharing the GPU, weak mode bench (functional: per-iteration sync and exchange timing)
DABD_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 > ${O}_bench_n2_shared.json 2> ${O}_bench_n2_shared.err; echo "n2 exit=$?"; tail -c 600 ${O}_bench_n2_shared.json
DABD_GPU_FANIN=0 DABD_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 3 --warmup 3 > ${O}_bench_n2_shared_host.json 2> ${O}_bench_n2_shared_host.err; echo "n2 host exit=$?"; tail -c 600 ${O}_bench_n2_shared_host.json
