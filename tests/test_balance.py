"""PD load balancer of the interface planes (proj/src/balance.cpp:8-83).

CPU: the reference's own known answers (proj/tests/test_balance.cpp:10-109)
through the library's C ABI and through the oracle restatement, and the two
bitwise equal on random time sequences. GPU: a balanced consensus-ADMM run
moves the planes exactly as the oracle balancer fed the run's per-partition
costs, and stays penetration-free.
"""

import numpy as np
import pytest

import balance as OB
from paper_2605_15875_b200 import api
from paper_2605_15875_b200 import _lib as L
from paper_2605_15875_b200.scene import make_scenario

IMPLS = [pytest.param(api, id="c_abi"), pytest.param(OB, id="oracle")]


def _mk(impl, n, **kw):
    return impl.Balancer(n, **kw)


@pytest.mark.parametrize("impl", IMPLS)
def test_imbalance_metric(impl):  # test_balance.cpp:10-17
    assert impl.imbalance_metric(2.5, 2.5) == pytest.approx(0.0)
    assert impl.imbalance_metric(3.0, 1.0) == pytest.approx(0.5)
    assert impl.imbalance_metric(1.0, 3.0) == pytest.approx(-0.5)
    for a in (0.5, 1.0, 2.0, 7.5):
        assert impl.imbalance_metric(a, 2.0) == pytest.approx(-impl.imbalance_metric(2.0, a))
    with pytest.raises(Exception, match="must be > 0"):
        impl.imbalance_metric(0.0, 1.0)


@pytest.mark.parametrize("impl", IMPLS)
def test_pd_update_and_factor(impl):  # test_balance.cpp:19-39
    assert impl.pd_update(0.0, 0.0, 1.0, 1.0, 10.0) == pytest.approx(0.0)
    assert impl.pd_update(0.5, 0.5, 1.0, 0.0, 10.0) == pytest.approx(0.5)
    assert impl.pd_update(0.3, 0.1, 0.0, 2.0, 10.0) == pytest.approx(0.4)
    assert impl.pd_update(0.9, 0.0, 1.0, 0.0, 0.25) == pytest.approx(0.25)
    assert impl.balance_factor([2.0, 2.0, 2.0]) == pytest.approx(1.0)
    assert impl.balance_factor([1.0, 1.0, 1.0, 3.0]) == pytest.approx(0.5)
    assert impl.balance_factor([7.0]) == pytest.approx(1.0)


@pytest.mark.parametrize("impl", IMPLS)
def test_balanced_fixed_point_and_sign(impl):  # test_balance.cpp:41-65
    b = _mk(impl, 2, kp=0.4, kd=0.2)
    planes = np.array([[0.7, 0.0, -1.0, 0.0]]) if impl is api else [[0.7, 0.0, -1.0, 0.0]]
    for _ in range(10):
        dp = b.update([1.0, 1.0], planes, 0.2)
        assert dp[0] == pytest.approx(0.0)
        assert planes[0][0] == pytest.approx(0.7)
    b = _mk(impl, 2, kp=0.4, kd=0.0)
    planes = np.array([[3.0, 0.0, -1.0, 0.0]]) if impl is api else [[3.0, 0.0, -1.0, 0.0]]
    dp = b.update([3.0, 1.0], planes, 0.2)
    assert dp[0] > 0.0 and planes[0][0] < 3.0  # a slower worker 0 sheds area


@pytest.mark.parametrize("impl", IMPLS)
def test_area_proportional_workload_converges(impl):  # test_balance.cpp:67-94
    extent, w = 4.0, 0.2
    b = _mk(impl, 2, kp=0.1 * extent, kd=0.05 * extent)
    planes = np.array([[1.0, 0.0, -1.0, 0.0]]) if impl is api else [[1.0, 0.0, -1.0, 0.0]]
    settled = -1
    for frame in range(80):
        p = planes[0][0]
        b.update([p, extent - p], planes, w)
        p = planes[0][0]
        t_abs = abs(OB.imbalance_metric(p, extent - p))
        if settled < 0 and t_abs < 0.05:
            settled = frame
        if settled >= 0:
            assert t_abs < 0.05
            assert OB.balance_factor([p, extent - p]) >= 0.9
    assert 0 <= settled < 50


@pytest.mark.parametrize("impl", IMPLS)
def test_neighbour_clearance(impl):  # test_balance.cpp:96-109
    b = _mk(impl, 3, kp=100.0, kd=0.0, dp_max=100.0)
    rows = [[-0.5, 0.0, -1.0, 0.0], [0.5, 0.0, -1.0, 0.0]]
    planes = np.array(rows) if impl is api else [list(r) for r in rows]
    b.update([10.0, 1.0, 1.0], planes, 0.3)
    assert planes[1][0] - planes[0][0] >= 0.3 - 1e-12


def test_c_abi_matches_oracle_bitwise():
    rng = np.random.default_rng(5)
    for n in (2, 3, 5):
        kw = dict(kp=float(rng.uniform(0.05, 2.0)), kd=float(rng.uniform(0.0, 1.0)),
                  smoothing=float(rng.uniform(0.1, 0.9)), dp_max=float(rng.choice([0.0, 0.05])))
        a, o = api.Balancer(n, **kw), OB.Balancer(n, **kw)
        rows = [[-1.0 + 1.7 * k + 0.01 * k * k, 0.2 * k, -1.0, 0.0] for k in range(n - 1)]
        pa, po = np.array(rows), [list(r) for r in rows]
        for _ in range(40):
            t = list(rng.uniform(0.1, 5.0, size=n))
            w = float(rng.uniform(0.1, 0.5))
            da, do = a.update(t, pa, w), o.update(t, po, w)
            assert list(da) == do
            assert pa.tolist() == po
    with pytest.raises(L.DabdGpuError, match="interface count"):
        api.Balancer(3).update([1.0, 1.0, 1.0], np.zeros((1, 4)), 0.2)


@pytest.mark.gpu
def test_balanced_admm_run_moves_planes_like_the_oracle_balancer():
    """cubes-64 (2 partitions, plane through the x=0.35 column) with the
    balancer on. Frame f+1 partitions with the planes the balancer derives
    from frame f's per-partition costs and frame f's overlap width w
    (runtime.cpp:537-560): the device planes equal the oracle Balancer fed
    the same costs and w, bitwise, every frame; the run stays
    penetration-free and the plane moves."""
    import oracle as O

    sd = make_scenario("cubes-64")
    sd.balance = {"enabled": True, "kp": 0.2, "kd": 0.05, "smoothing": 0.5, "dp_max": 0.0}
    ctx = api.Context(api.Scene(sd), num_workers=2)
    o = O.Scene(sd)
    ob = OB.Balancer(2, kp=0.2, kd=0.05, smoothing=0.5, dp_max=0.0)
    planes = [[0.35, 0.0, -1.0, 0.0]]
    assert ctx.planes().tolist() == planes
    prev = None
    for f in range(12):
        _, qd = ctx.state()
        v = float(o.max_vertex_speed(qd)[~np.asarray(o.is_static, dtype=bool)].max())
        if prev is not None:
            ob.update(prev[0], planes, prev[1])
        st = ctx.run_frames(1)[0]
        assert ctx.planes().tolist() == planes, f"frame {f}"
        costs = ctx.partition_costs()
        assert (costs > 0).all()
        prev = (costs.tolist(), max(2.0 * v * st["h"], sd.w_min))
        inter, _, dmin = ctx.audit(cutoff=1.0)
        assert not inter and dmin > 0.0
    assert planes != [[0.35, 0.0, -1.0, 0.0]]
