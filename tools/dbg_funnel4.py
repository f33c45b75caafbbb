"""Funnel frame 4 (first frame with split bodies): GPU vs oracle shared sets,
masks and states (diagnostic)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
from paper_2605_15875_b200 import api  # noqa: E402
from paper_2605_15875_b200.scene import make_scenario  # noqa: E402

sd = make_scenario("funnel-analog")
T = dict(pcg_rel_tol=1e-12, pcg_max_iters=20000)
for nf in (4, 5):
    ref = O.Scene(sd).run(nf, workers=2)
    gpu = api.run_distributed(sd, 2, nf, **T)
    print("frames", nf, "shared gpu", np.nonzero(~np.isnan(gpu.rho))[0], "ref", np.nonzero(~np.isnan(ref["rho"]))[0])
    print("  rho gpu", gpu.rho[~np.isnan(gpu.rho)], "ref", ref["rho"][~np.isnan(ref["rho"])])
    d = np.abs(gpu.q[-1] - ref["q"][-1]).max(axis=1)
    print("  max |dq| per body (top 5):", np.argsort(-d)[:5], np.sort(d)[::-1][:5])
# masks at the start of frame 4 from both implementations' frame-3 state
ref3 = O.Scene(sd).run(4, workers=2)
q3, qd3 = ref3["q"][-1], ref3["qdot"][-1]
o = O.Scene(sd)
vmax = o.max_vertex_speed(qd3)[~np.asarray(o.is_static, bool)].max()
w = max(2.0 * vmax * sd.params.h, sd.w_min)
planes = [[p.point[0], p.point[1], p.normal[0], p.normal[1]] for p in sd.planes]
mo = o.holder_masks(q3, planes, w)
ctx = api.Context(api.Scene(sd), num_workers=2)
mg = ctx.holder_masks(q3, planes, w)
print("w", w, "masks equal", np.array_equal(mo, mg), "shared(mask==3):", np.nonzero(mo == 3)[0])

# per-partition objective at the start of frame 4 (k = 1: z = q_tilde, u = 0, rho0)
p = sd.params
f = np.zeros((o.n, 6))
for b in range(o.n):
    if not o.is_static[b]:
        f[b, 0] = o.mass[b] * p.gravity[0]
        f[b, 1] = o.mass[b] * p.gravity[1]
qt = o.predicted_position(q3, qd3, f, p.h)
for part in (0, 1):
    local = [b for b in range(o.n) if mo[b] & (1 << part)]
    kappa = [1.0 / bin(int(mo[b])).count("1") for b in local]
    anchors = [(b, qt[b], np.zeros(6), float(sd.adapt.beta * o.mass[b])) for b in local
               if not o.is_static[b] and bin(int(mo[b])).count("1") >= 2]
    ro = o.objective(q3, local, kappa, qt[local], p.as_array(), anchors=anchors, holder_mask=mo, mode=2)
    rg = ctx.objective(q3, local, kappa, qt[local], p, anchors=anchors, holder_mask=mg, mode=2)
    print("part", part, "value", ro["value"], rg["value"], "active", ro["active"], rg["active"],
          "cand", ro["candidates"], rg["candidates"],
          "grad", np.abs(ro["grad"] - rg["grad"]).max(), "hess", np.abs(ro["hess"] - rg["hess"]).max())
    qa = o.newton_solve(q3, local, kappa, qt[local], p.as_array(), 32, p.theta * p.h * p.scene_scale,
                        anchors=anchors, holder_mask=mo)
    qb = ctx.newton_solve(q3, local, kappa, qt[local], p, 32, p.theta * p.h * p.scene_scale,
                          anchors=anchors, holder_mask=mg)
    print("   newton", qa[1], qb[1], "max |dq| shared 4,5:", np.abs(qa[0][[4, 5]] - qb[0][[4, 5]]).max())

print("--- per-iteration (partition 0)")
part = 0
local = [b for b in range(o.n) if mo[b] & (1 << part)]
kappa = [1.0 / bin(int(mo[b])).count("1") for b in local]
anchors = [(b, qt[b], np.zeros(6), float(sd.adapt.beta * o.mass[b])) for b in local
           if not o.is_static[b] and bin(int(mo[b])).count("1") >= 2]
tol = p.theta * p.h * p.scene_scale
for it in (1, 2, 3, 4):
    qa = o.newton_solve(q3, local, kappa, qt[local], p.as_array(), it, tol, anchors=anchors, holder_mask=mo)
    qb = ctx.newton_solve(q3, local, kappa, qt[local], p, it, tol, anchors=anchors, holder_mask=mg)
    dd = np.abs(qa[0] - qb[0]).max(axis=1)
    print(it, "max diff", dd.max(), "worst bodies", np.argsort(-dd)[:3], qa[1]["final_update_inf"], qb[1]["final_update_inf"])
    if it == 1:
        q1o, q1g = qa[0], qb[0]
# CCD of the first step
dqo = q1o - q3
print("oracle ccd toi q3->q3+dq(oracle)", o.ccd_toi(q3, q3 + 1.0 * dqo, subset=local))
print("gpu    ccd toi q3->q3+dq(oracle)", ctx.ccd_toi(q3, q3 + 1.0 * dqo, subset=local))

print("--- objective at q1 (after iteration 1)")
ro = o.objective(q1o, local, kappa, qt[local], p.as_array(), anchors=anchors, holder_mask=mo, mode=2)
rg = ctx.objective(q1o, local, kappa, qt[local], p, anchors=anchors, holder_mask=mg, mode=2)
print("value", ro["value"], rg["value"], "active", ro["active"], rg["active"], "cand", ro["candidates"], rg["candidates"],
      "grad", np.abs(ro["grad"] - rg["grad"]).max(), "hess", np.abs(ro["hess"] - rg["hess"]).max())
H, g = ro["hess"], ro["grad"]
nd = H.shape[0]
A = H + 1e-8 * np.trace(H) / nd * np.eye(nd)
dq_exact = np.linalg.solve(A, -g)
Hg, gg = rg["hess"], rg["grad"]
dq_g = np.linalg.solve(Hg + 1e-8 * np.trace(Hg) / nd * np.eye(nd), -gg)
print("dense-solve dq diff (oracle H vs gpu H):", np.abs(dq_exact - dq_g).max(), " |dq|", np.abs(dq_exact).max())
