"""Repro probe for the pour-10k 8-partition frames of
tests/test_gpu_scale_parity.py::test_pour_10k_eight_partitions.

python tools/probe_pour.py [settle] [frames] [tight] [eager]

The settled state is cached in tools/_cache/pour_settled_<settle>.npz (a probe
artefact) so sanitizer runs can skip the settle.
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2605_15875_b200 import api  # noqa: E402
from paper_2605_15875_b200.scene import make_scenario  # noqa: E402


def main():
    settle = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    frames = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    tight = len(sys.argv) > 3 and sys.argv[3] == "1"
    solver = dict(pcg_rel_tol=1e-12, pcg_max_iters=20000) if tight else {}
    eager = len(sys.argv) > 4 and sys.argv[4] == "1"
    sd = make_scenario("pour-10k")
    cache = os.path.join(ROOT, "tools", "_cache", f"pour_settled_{settle}.npz")
    if os.path.exists(cache):
        z = np.load(cache)
        q, qd = z["q"], z["qd"]
    else:
        ctx = api.Context(api.Scene(sd))
        t = time.time()
        ctx.run_frames(settle)
        q, qd = ctx.state()
        os.makedirs(os.path.dirname(cache), exist_ok=True)
        np.savez(cache, q=q, qd=qd)
        print(f"settled {settle} frames in {time.time() - t:.1f}s", flush=True)
    if eager:
        os.environ["DABD_GPU_NO_GRAPH"] = "1"
    c8 = api.Context(api.Scene(sd), num_workers=8, **solver)
    c8.set_state(q, qd)
    for f in range(frames):
        t = time.time()
        st = c8.run_frames(1)[0]
        print(f, f"{time.time() - t:.2f}s", st, flush=True)


if __name__ == "__main__":
    main()
