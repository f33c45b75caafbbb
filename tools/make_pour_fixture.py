"""C3 parity fixture (tests/test_gpu_scale_parity.py::test_pour_10k_eight_partitions):
the CPU oracle pours pour-10k for 30 single-domain frames (sim.cpp:186-249),
runs 2 consensus-ADMM frames on 8 partitions (runtime.cpp:110-694, one
oracle thread per worker) to reach an 8-partition state, and records the
next 8-partition frame: state, ADMM trace, counts, attempts and final rho.
The GPU test starts from the recorded state and compares its frame with the
recorded one, so the oracle's minutes-long frames run here, once, not on the
GPU box.

python tools/make_pour_fixture.py   (tens of minutes on 8 cores)
writes tests/golden/pour-10k_w8.npz
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def main():
    import oracle as O
    from paper_2605_15875_b200.scene import make_scenario

    settle, split = 30, 2
    sd = make_scenario("pour-10k")
    o = O.Scene(sd)
    t = time.time()
    r = o.run(settle, workers=0)
    print(f"settled {settle} frames in {time.time() - t:.0f}s, admm {list(r['admm'])}", flush=True)
    o = O.Scene(sd)
    o.set_state(r["q"][-1], r["qdot"][-1])
    t = time.time()
    r = o.run(split, workers=8)
    print(f"{split} 8-partition frames in {time.time() - t:.0f}s, admm {list(r['admm'])}", flush=True)
    q0, qd0 = r["q"][-1].copy(), r["qdot"][-1].copy()
    o = O.Scene(sd)
    o.set_state(q0, qd0)
    t = time.time()
    ref = o.run(1, workers=8)
    print(f"recorded frame in {time.time() - t:.0f}s, admm {list(ref['admm'])}, "
          f"attempts {list(ref['attempts'])}, trace rows {len(ref['trace'])}", flush=True)
    out = os.path.join(ROOT, "tests", "golden", "pour-10k_w8.npz")
    np.savez_compressed(out, q0=q0, qd0=qd0, q1=ref["q"][-1], qd1=ref["qdot"][-1], trace=ref["trace"],
                        rho=ref["rho"], admm=ref["admm"], attempts=ref["attempts"],
                        newton=ref["newton"], settle=settle, split=split, seed=sd.seed)
    print(out, os.path.getsize(out), "bytes")


if __name__ == "__main__":
    main()
