"""Launch-list window of the multi-partition frame: pour-10k on 8 partitions
from the contact-rich fixture start (tests/golden/pour-10k_w8.npz), default
solver settings, one unprofiled frame then `frames` profiled frames (eager
launches, DABD_GPU_NO_GRAPH=1, as tools/launch_window.py).

ncu --profile-from-start off --metrics gpu__time_duration.sum --csv \
    --log-file gpurun_out/pour_launches.csv python tools/launch_window_pour.py 1
"""
import os
import sys

os.environ.setdefault("DABD_GPU_NO_GRAPH", "1")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    from paper_2605_15875_b200 import api
    from paper_2605_15875_b200.scene import make_scenario

    frames = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    z = np.load(os.path.join(ROOT, "tests", "golden", "pour-10k_w8.npz"))
    sd = make_scenario("pour-10k")
    ctx = api.Context(api.Scene(sd), num_workers=8)
    ctx.set_state(z["q0"], z["qd0"])
    ctx.run_frames(1)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    st = ctx.run_frames(frames)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print(st)


if __name__ == "__main__":
    main()
