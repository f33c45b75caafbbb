"""C3 parity fixture (tests/test_gpu_scale_parity.py::test_pour_10k_eight_partitions),
in two steps:

  python tools/make_pour_fixture.py start   (on a GPU box, ~10 s)
      the B200 path pours pour-10k for 30 single-domain frames (sim.cpp:186-249)
      and runs 2 consensus-ADMM frames on 8 partitions (runtime.cpp:110-694) to
      reach a contact-rich 8-partition state: gpurun_out/pour-10k_w8_start.npz
  python tools/make_pour_fixture.py record START.npz   (CPU, tens of minutes)
      the CPU oracle runs the next 8-partition frame from that state (one
      oracle thread per worker) and records state, ADMM trace, counts,
      attempts and final rho: tests/golden/pour-10k_w8.npz

The GPU test starts from the recorded start state and compares its frame
with the oracle's, so the oracle's minutes-long frame runs once, here, not
on the GPU box. (Pouring the start state with the oracle itself takes hours
single-threaded; the start state only has to be contact-rich and the same
for both sides.)
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


SETTLE, SPLIT = 30, 2


def start():
    from paper_2605_15875_b200 import api
    from paper_2605_15875_b200.scene import make_scenario

    sd = make_scenario("pour-10k")
    ctx = api.Context(api.Scene(sd))
    ctx.run_frames(SETTLE)
    q, qd = ctx.state()
    c8 = api.Context(api.Scene(sd), num_workers=8)
    c8.set_state(q, qd)
    st = c8.run_frames(SPLIT)
    q, qd = c8.state()
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    out = os.path.join(ROOT, "gpurun_out", "pour-10k_w8_start.npz")
    np.savez_compressed(out, q0=q, qd0=qd)
    print(out, [s["admm_iterations"] for s in st])


def record(start_npz):
    import oracle as O
    from paper_2605_15875_b200.scene import make_scenario

    sd = make_scenario("pour-10k")
    z = np.load(start_npz)
    q0, qd0 = z["q0"], z["qd0"]
    o = O.Scene(sd)
    o.set_state(q0, qd0)
    t = time.time()
    ref = o.run(1, workers=8)
    print(f"recorded frame in {time.time() - t:.0f}s, admm {list(ref['admm'])}, "
          f"attempts {list(ref['attempts'])}, trace rows {len(ref['trace'])}", flush=True)
    out = os.path.join(ROOT, "tests", "golden", "pour-10k_w8.npz")
    np.savez_compressed(out, q0=q0, qd0=qd0, q1=ref["q"][-1], qd1=ref["qdot"][-1], trace=ref["trace"],
                        rho=ref["rho"], admm=ref["admm"], attempts=ref["attempts"],
                        newton=ref["newton"], settle=SETTLE, split=SPLIT, seed=sd.seed)
    print(out, os.path.getsize(out), "bytes")


if __name__ == "__main__":
    if sys.argv[1] == "start":
        start()
    else:
        record(sys.argv[2])
