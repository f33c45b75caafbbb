"""Does an audit between frames change the run? (diagnostic)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2605_15875_b200 import api  # noqa: E402
from paper_2605_15875_b200.scene import make_scenario  # noqa: E402

sd = make_scenario("density-sweep-10")
a = api.Context(api.Scene(sd), num_workers=2)
b = api.Context(api.Scene(sd), num_workers=2)
for f in range(100):
    sa = a.run_frames(1)[0]
    try:
        sb = b.run_frames(1)[0]
    except Exception as e:  # noqa: BLE001
        print("audited run failed at frame", f, e)
        break
    b.audit()
    qa, qb = a.state()[0], b.state()[0]
    d = float(np.abs(qa - qb).max())
    if d > 0 or sa["admm_iterations"] != sb["admm_iterations"]:
        print("frame", f, "diff", d, sa["admm_iterations"], sb["admm_iterations"])
        if f > 5 and d > 1e-3:
            break
print("done")
