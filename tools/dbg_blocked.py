import os, sys, json
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/oracle"); sys.path.insert(0, "/root/repo/tests")
from paper_2605_15875_b200 import api
from paper_2605_15875_b200.scene import make_scenario
import oracle as O
sd = make_scenario("blocked-merge")
gpu = api.run_distributed(sd, 2, 3, pcg_rel_tol=1e-12, pcg_max_iters=20000)
print("env fused-off" if os.environ.get("DABD_GPU_NO_FUSED_PCG") else "fused", "h", list(gpu.h), [s["attempts"] for s in gpu.stats], [s["admm_iterations"] for s in gpu.stats], [s["newton_iterations"] for s in gpu.stats])
if not os.environ.get("DABD_GPU_NO_FUSED_PCG"):
    ref = O.Scene(sd).run(3, workers=2)
    print("oracle h", list(ref["h"]), list(ref["attempts"]), list(ref["admm"]))
