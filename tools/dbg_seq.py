"""Cross-context state check: drop-grid-2 (2 workers) alone vs after other
contexts in the same process (diagnostic)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_15875_b200 import api  # noqa: E402
from paper_2605_15875_b200.scene import make_scenario  # noqa: E402


def run(name, workers, frames):
    ctx = api.Context(api.Scene(make_scenario(name)), num_workers=workers)
    for f in range(frames):
        try:
            ctx.run_frames(1)
        except Exception as e:  # noqa: BLE001
            return f"{name}: frame {f}: {e}"
    q, _ = ctx.state()
    return f"{name}: ok, q checksum {float(abs(q).sum()):.17g}"


order = sys.argv[1:]
for spec in order:
    n, w, f = spec.split(":")
    print(run(n, int(w), int(f)), flush=True)
