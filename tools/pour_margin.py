"""Margins of test_pour_10k_eight_partitions (tests/test_gpu_scale_parity.py),
repeated to see the run-to-run spread on the device."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_2605_15875_b200 import api
from paper_2605_15875_b200.scene import make_scenario

TIGHT = dict(pcg_rel_tol=1e-12, pcg_max_iters=20000, inexact=(0.0, 10.0))  # tests/test_gpu_scale_parity.py

z = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "pour-10k_w8.npz"))
sd = make_scenario("pour-10k")
norm = sd.params.h * sd.params.scene_scale
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    ctx = api.Context(api.Scene(sd), num_workers=8, **TIGHT)
    ctx.set_state(z["q0"], z["qd0"])
    st = ctx.run_frames(1)[0]
    qg, _ = ctx.state()
    tr_g, tr_o = ctx.take_trace(), z["trace"]
    errs = [np.abs(tr_g[:, c] - tr_o[:, c]).max() / norm for c in (3, 4, 5)] if tr_g.shape == tr_o.shape else None
    print(rep, st["admm_iterations"], z["admm"][0], "rel errs col3-5 / (h l):", errs,
          "q err / l:", np.abs(qg - z["q1"]).max() / sd.params.scene_scale, flush=True)
