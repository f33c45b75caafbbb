"""The C++ adapter (include/dabd_gpu.hpp): the reference's C++ scene / step /
parameter API (proj/include/dabd/{params,scene,sim}.hpp) over the C ABI.

CPU: the adapter compiles and links against libdabd_gpu.so; its built-in
scenarios build the same body table as scene.py (bitwise); its snapshot and
metrics files have the reference's layout (sim.cpp:34-137) and read back in
Python. GPU: a C++ host program stepping run_reference / run_distributed
writes the trajectory the Python path computes (bitwise) and the oracle's
within tolerance.
"""

import csv
import os
import subprocess

import numpy as np
import pytest

from paper_2605_15875_b200 import api
from paper_2605_15875_b200 import build as B
from paper_2605_15875_b200.scene import make_scenario


@pytest.fixture(scope="module")
def adapter():
    return B.build_adapter()


def _run(adapter, *args):
    r = subprocess.run([adapter, *map(str, args)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    return r.stdout


@pytest.mark.parametrize("name", ["funnel-analog", "drop-grid-2", "density-sweep-10", "pile-1k",
                                  "pour-10k"])
def test_cpp_scenarios_match_python(adapter, name):
    """make_scenario in C++ (scene.cpp:345-557 arithmetic) == scene.py, bitwise."""
    lines = _run(adapter, "scene", name).split("\n")
    n = int(lines[0])
    vals = np.array([[float.fromhex(t) for t in ln.split()] for ln in lines[1:1 + n]])
    sc = api.Scene(make_scenario(name))
    assert n == sc.n
    assert np.array_equal(vals[:, :6], sc.q0)
    assert np.array_equal(vals[:, 6], sc.mass)


def test_cpp_snapshot_and_metrics_files(adapter, tmp_path):
    out = _run(adapter, "io", tmp_path)
    assert "io ok" in out
    frame, ids, q, qd = api.read_snapshot(api.frame_path(str(tmp_path), 1))
    assert frame == 1 and list(ids) == [1, 2]
    assert q[0, 0] == 0.3 and qd[1, 5] == -6.0
    # byte layout: 16-byte header + 104 bytes per dynamic body (sim.cpp:34-51)
    assert os.path.getsize(api.frame_path(str(tmp_path), 0)) == 16 + 2 * 104
    # Python writer produces the identical bytes
    init = np.array([[0, 0, 1, 0, 0, 1], [0.1, 0.2, 1, 1e-3, -1e-3, 1], [-1.5, 2.25, 0.5, 0, 0, 2]])
    vel = np.array([[0] * 6, [1, 2, 3, 4, 5, 6], [-1, -2, -3, -4, -5, -6]], dtype=float)
    api.write_snapshot(str(tmp_path / "py.bin"), 0, [True, False, False], init, vel)
    assert (tmp_path / "py.bin").read_bytes() == open(api.frame_path(str(tmp_path), 0), "rb").read()
    tr = api.load_trajectory(str(tmp_path), np.tile([7.0, 7, 1, 0, 0, 1], (3, 1)))
    assert tr.q.shape == (2, 3, 6) and tr.q[0, 0, 0] == 7.0 and tr.q[1, 1, 0] == 0.3
    with open(tmp_path / "metrics.csv") as f:
        rows = list(csv.reader(f))
    assert rows[0] == ["frame", "attempt", "k", "committed", "r_inf", "s_inf", "min_toi",
                       "active_contacts", "candidate_pairs", "mse", "dq_inf_w0", "dq_inf_w1",
                       "newton_w0", "newton_w1", "t_compute_w0", "t_compute_w1", "t_sync_w0",
                       "t_sync_w1"]
    assert rows[1][:4] == ["0", "0", "2", "1"] and float(rows[1][4]) == 1.5e-7 and rows[1][9] == ""
    (tmp_path / "bad.bin").write_bytes(np.array([0, 1], dtype="<u8").tobytes() + b"\0" * 20)
    with pytest.raises(Exception, match="truncated"):
        api.read_snapshot(str(tmp_path / "bad.bin"))


@pytest.mark.gpu
def test_cpp_run_reference_matches_python_and_oracle(adapter, tmp_path):
    import oracle as O

    sd = make_scenario("funnel-analog")
    out = _run(adapter, "reference", "funnel-analog", 3, tmp_path)
    assert '"frames": 3' in out
    sc = api.Scene(sd)
    cpp = api.load_trajectory(str(tmp_path), sc.q0)
    py = api.run_reference(sd, 3)
    assert np.array_equal(cpp.q, py.q)
    assert np.array_equal(cpp.q_dot[:, ~sc.is_static], py.q_dot[:, ~sc.is_static])
    ref = O.Scene(sd).run(3, workers=0)
    assert np.abs(cpp.q - np.asarray(ref["q"])).max() < 1e-5 * sd.params.scene_scale


@pytest.mark.gpu
def test_cpp_run_distributed_matches_python(adapter, tmp_path):
    out = _run(adapter, "distributed", "drop-grid-2", 3, 2, tmp_path)
    assert '"intersection_violations": 0' in out
    sd = make_scenario("drop-grid-2")
    sc = api.Scene(sd)
    cpp = api.load_trajectory(str(tmp_path), sc.q0)
    py = api.run_distributed(sd, 2, 3)
    assert np.array_equal(cpp.q, py.q)
    with open(tmp_path / "metrics.csv") as f:
        rows = list(csv.DictReader(f))
    assert len(rows) == len(py.trace)
    assert [int(r["k"]) for r in rows] == [int(t[2]) for t in py.trace]
    assert sum(int(r["committed"]) for r in rows) == 3
    assert np.allclose([float(r["r_inf"]) for r in rows], py.trace[:, 4], rtol=0, atol=0)
