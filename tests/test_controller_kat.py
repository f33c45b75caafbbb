"""The reference's controller known answers on the product's host code:
check_stopping (consensus.cpp:54-64) and TimestepController
(consensus.hpp:60-87) as the multi-partition frame runs them, through the
C ABI (dabd_gpu_check_stopping / dabd_gpu_timestep_apply; no device needed),
and bit-for-bit equal to the oracle's restatement on random inputs.
"""

import numpy as np
import pytest

import oracle as O
from paper_2605_15875_b200 import api
from paper_2605_15875_b200._lib import DabdGpuError


def test_stopping_rule_known_answers():  # test_consensus.cpp:131-161
    h, l, th = 0.01, 2.0, 1e-3
    assert api.check_stopping(0, 0, 0, [1.0, 1.0], h, l, th)
    assert not api.check_stopping(0, 0, 0, [1.0, 0.7], h, l, th)
    at = th * h * l
    assert not api.check_stopping(0, at, 0, [1.0], h, l, th)  # strict boundary
    assert api.check_stopping(0, np.nextafter(at, 0.0), 0, [1.0], h, l, th)
    assert api.check_stopping(0, 0, 0, [], h, l, th)


def test_stopping_rule_equals_oracle():
    rng = np.random.default_rng(39)
    h, l, th = 0.01, 2.0, 1e-3
    at = th * h * l
    for _ in range(500):
        dq, r, s = rng.uniform(0, 2 * at, 3)
        tois = rng.choice([1.0, 0.9, np.nextafter(1.0, 0.0)], size=rng.integers(0, 4), p=[0.8, 0.1, 0.1])
        assert api.check_stopping(dq, r, s, tois, h, l, th) == O.check_stopping(dq, r, s, tois, h, l, th)


def test_timestep_controller_known_answers():  # test_consensus.cpp:246-261
    assert list(api.timestep_apply(0.02, 4, [0, 0, 1, 1, 1])) == pytest.approx([0.01, 0.005, 0.01, 0.02, 0.02])
    with pytest.raises(DabdGpuError):
        api.timestep_apply(0.02, 4, [0, 0, 0, 0, 0])


def test_timestep_controller_equals_oracle():
    rng = np.random.default_rng(7)
    for _ in range(50):
        ev, run = [], 0
        for _ in range(int(rng.integers(1, 16))):
            e = 1 if run == 3 else int(rng.integers(0, 2))  # at most max_halvings failures in a row
            run = run + 1 if e == 0 else 0
            ev.append(e)
        assert np.array_equal(api.timestep_apply(0.02, 3, ev), O.timestep_apply(0.02, 3, ev))
