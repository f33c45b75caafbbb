"""Test-only CPU restatement of the reference's PD load balancer
(proj/src/balance.cpp:8-83, proj/include/dabd/balance.hpp:9-56).

Pure-Python scalar arithmetic in the reference's evaluation order (IEEE
double, no FMA), used by tests/ as the checker of the library's balancer.
Planes are [px, py, nx, ny] lists.
"""


class BalanceError(RuntimeError):
    pass


def imbalance_metric(tau_i, tau_j):
    """balance.cpp:8-13."""
    if not (tau_i > 0.0) or not (tau_j > 0.0):
        raise BalanceError("imbalance_metric: compute times must be > 0")
    eta = tau_i / tau_j
    return (eta - 1.0) / (eta + 1.0)


def pd_update(t, t_prev, kp, kd, dp_max):
    """balance.cpp:15-19."""
    dp = kp * t + kd * (t - t_prev)
    if dp_max > 0.0:
        return min(max(dp, -dp_max), dp_max)
    return dp


def shift_boundary(plane, dp):
    """balance.cpp:21-25: p' = p + dp n."""
    px, py, nx, ny = plane
    return [px + dp * nx, py + dp * ny, nx, ny]


def balance_factor(times):
    """balance.cpp:27-36."""
    if not times:
        return 1.0
    s, peak = 0.0, 0.0
    for t in times:
        if not (t > 0.0):
            raise BalanceError("balance_factor: compute times must be > 0")
        s += t
        peak = max(peak, t)
    return s / len(times) / peak


class Balancer:
    """balance.cpp:38-81."""

    def __init__(self, num_workers, kp=0.0, kd=0.0, smoothing=0.5, dp_max=0.0):
        self.kp, self.kd, self.smoothing, self.dp_max = kp, kd, smoothing, dp_max
        self.smoothed = [0.0] * num_workers
        self.t_prev = [0.0] * max(0, num_workers - 1)
        self.primed = False

    def update(self, times, planes, w):
        if len(times) != len(self.smoothed):
            raise BalanceError("Balancer: worker count mismatch")
        if len(planes) != len(self.t_prev):
            raise BalanceError("Balancer: interface count mismatch")
        for i in range(len(self.smoothed)):
            self.smoothed[i] = (self.smoothing * times[i] + (1.0 - self.smoothing) * self.smoothed[i]
                                if self.primed else times[i])
        self.primed = True
        dp_max = self.dp_max if self.dp_max > 0.0 else w / 2.0
        applied = [0.0] * len(planes)

        def gap(a, b):  # (a.point - b.point) . b.normal
            return (a[0] - b[0]) * b[2] + (a[1] - b[1]) * b[3]

        for k in range(len(planes)):
            t = imbalance_metric(self.smoothed[k], self.smoothed[k + 1])
            dp = pd_update(t, self.t_prev[k], self.kp, self.kd, dp_max)
            self.t_prev[k] = t
            if k > 0:
                s = gap(planes[k - 1], planes[k])
                if s < 0.0:
                    dp = max(dp, s + w)
                if s > 0.0:
                    dp = min(dp, s - w)
            if k + 1 < len(planes):
                s = gap(planes[k + 1], planes[k])
                if s < 0.0:
                    dp = max(dp, s + w)
                if s > 0.0:
                    dp = min(dp, s - w)
            planes[k] = shift_boundary(planes[k], dp)
            applied[k] = dp
        return applied
