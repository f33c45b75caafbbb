"""Bench start state: the CPU oracle's own 40-frame drop of the pile-1k
lattice (run_reference semantics, sim.cpp:186-249), i.e. the reference
algorithm's contact-rich pile. bench.py starts BOTH arms (the B200 path and
the CPU reference arm) from this state, so the timed frames are the same
frames; for N > 1 the pile is tiled into the N slabs of pile_slabs(N).

python tools/make_bench_fixture.py   (~75 s on one core)
writes tests/golden/pile-1k_settled40.npz
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def main():
    import oracle as O
    from paper_2605_15875_b200.scene import make_scenario

    frames = 40
    sd = make_scenario("pile-1k")
    r = O.Scene(sd).run(frames, workers=0)
    out = os.path.join(ROOT, "tests", "golden", "pile-1k_settled40.npz")
    np.savez_compressed(out, q=r["q"][-1], qdot=r["qdot"][-1], frames=frames, seed=sd.seed,
                        admm=r["admm"])
    print(out, r["q"][-1].shape)


if __name__ == "__main__":
    main()
