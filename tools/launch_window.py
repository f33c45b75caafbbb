"""Launch-list window for `ncu --profile-from-start off`: loads bench.py's
start state (the oracle-settled pile-1k) and runs 3 warm-up frames
unprofiled, then profiles exactly `frames` frames between
cudaProfilerStart/Stop (eager launches, DABD_GPU_NO_GRAPH=1: ncu cannot
replay kernel nodes inside conditional graph nodes; the kernels and their
arguments are the graph's).

ncu --profile-from-start off --metrics gpu__time_duration.sum --csv \
    --log-file gpurun_out/launches.csv python tools/launch_window.py 2
"""
import os
import sys

os.environ.setdefault("DABD_GPU_NO_GRAPH", "1")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_2605_15875_b200 import api
    from paper_2605_15875_b200.scene import make_scenario

    frames = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    from bench import start_state

    sd = make_scenario("pile-1k")
    ctx = api.Context(api.Scene(sd))
    ctx.set_state(*start_state(sd, 1))
    ctx.run_frames(3)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    st = ctx.run_frames(frames)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print(st)


if __name__ == "__main__":
    main()
