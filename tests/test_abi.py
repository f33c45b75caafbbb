"""CPU-side checks of the C-ABI boundary: the library loads and exports every
symbol include/dabd_gpu.h declares; argument validation needs no device."""

import ctypes as C
import os
import re

import pytest

from paper_2605_15875_b200 import _lib as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    text = open(os.path.join(ROOT, "include", "dabd_gpu.h")).read()
    return sorted(set(re.findall(r"DABD_GPU_API\s+[\w\s\*]+?\b(dabd_gpu_\w+)\s*\(", text)))


def test_header_symbols_match_binding_list():
    assert _header_symbols() == sorted(L.EXPORTS)


def test_library_exports_every_symbol():
    lib = L.load()
    for name in _header_symbols():
        assert hasattr(lib, name), name
    assert lib.dabd_gpu_version().decode() == "0.1.0"


def test_null_arguments_are_invalid():
    lib = L.load()
    assert lib.dabd_gpu_scene_create(0, None, None, None, None, None, None, None, None) == 3
    assert b"null" in lib.dabd_gpu_last_error()
    assert lib.dabd_gpu_ctx_create(None, 0, 0, 0, 1, None) == 3


def test_scene_build_matches_oracle_bitwise():
    """Host-side body construction (body.cpp:96-118) is bit-identical to the oracle."""
    import numpy as np

    import oracle as O
    from paper_2605_15875_b200 import api
    from paper_2605_15875_b200.scene import make_scenario

    for name in ("funnel-analog", "drop-grid-4", "heterogeneous", "blocked-merge", "pile-1k"):
        sd = make_scenario(name)
        g = api.Scene(sd)
        o = O.Scene(sd)
        assert np.array_equal(g.rest, o.rest)
        assert np.array_equal(g.q0, o.q0)
        assert np.array_equal(g.mass, o.mass)
        assert np.array_equal(g.mass_matrix, o.mass_matrix)


def test_invalid_scene_rejected():
    from paper_2605_15875_b200 import api
    from paper_2605_15875_b200.scene import BodySpec, SceneData

    sd = SceneData()
    sd.bodies.append(BodySpec(loops=[[(0.5, 0.5), (-0.5, 0.5), (-0.5, -0.5), (0.5, -0.5)][::-1][::-1][::-1]]))
    with pytest.raises(L.DabdGpuError) as e:
        api.Scene(sd)
    assert e.value.status == 3


def test_header_is_plain_c99_and_links(tmp_path):
    """include/dabd_gpu.h is a C header (no C++ in the signatures): a C99
    translation unit calling through it compiles with -pedantic and links
    against libdabd_gpu.so."""
    import subprocess

    from paper_2605_15875_b200 import build as B

    lib = B.build()
    src = tmp_path / "abi.c"
    src.write_text('#include "dabd_gpu.h"\n'
                   "int main(void) {\n"
                   "    dabd_gpu_scene* s = 0;\n"
                   "    int n = 0, nv = 0;\n"
                   "    if (dabd_gpu_scene_counts(s, &n, &nv) != DABD_GPU_ERR_INVALID) return 1;\n"
                   "    return dabd_gpu_last_error()[0] == 0;\n"
                   "}\n")
    exe = tmp_path / "abi"
    r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Wextra", "-pedantic", "-Werror", "-I",
                        os.path.join(ROOT, "include"), str(src), "-L", os.path.dirname(lib),
                        "-ldabd_gpu", "-Wl,-rpath," + os.path.dirname(lib), "-o", str(exe)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert subprocess.run([str(exe)]).returncode == 0
