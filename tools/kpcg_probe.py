"""Undivided pour-10k (one partition of 10,000 rows: the grid-cooperative k_pcg,
not the cluster kernel): settle, then run `frames` eager frames inside a
cudaProfilerStart/Stop window for ncu.

ncu --profile-from-start off --set full -k regex:k_pcg -c 1 python tools/kpcg_probe.py 30 1
"""
import os
import sys
import time

os.environ.setdefault("DABD_GPU_NO_GRAPH", "1")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_2605_15875_b200 import api
    from paper_2605_15875_b200.scene import make_scenario

    settle = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    frames = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    sd = make_scenario("pour-10k")
    ctx = api.Context(api.Scene(sd))
    ctx.run_frames(settle)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    t = time.perf_counter()
    st = ctx.run_frames(frames)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    torch.cuda.profiler.stop()
    print({"frames": frames, "s_per_frame": dt / frames, "pcg_iterations": [s["pcg_iterations"] for s in st],
           "newton": [s["newton_iterations"] for s in st]})


if __name__ == "__main__":
    main()
