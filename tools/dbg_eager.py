import os, sys
os.environ["DABD_GPU_NO_GRAPH"] = "1"
sys.path.insert(0, "/root/repo")
from paper_2605_15875_b200 import api
from paper_2605_15875_b200.scene import make_scenario
sd = make_scenario("pile-1k")
ctx = api.Context(api.Scene(sd))
for f in range(45):
    try:
        st = ctx.run_frames(1)[0]
    except Exception as e:
        print("frame", f, "error", e); break
    if f % 5 == 0: print(f, st)
