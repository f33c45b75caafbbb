"""B200-native distributed ADMM split-and-merge solver for affine body dynamics.

A from-scratch sm_100a implementation of the hot path of arxiv/paper_2605_15875
(`dabd`): per-partition projected Newton with IPC barrier contacts, CCD-filtered
line search and consensus ADMM merge of interface bodies. The compute path is
the in-tree C-ABI library `libdabd_gpu.so` (CUDA kernels + C++ host driver);
this package is its Python-side mirror of the reference interface.
"""

from . import scene  # noqa: F401

__version__ = "0.1.0"


def __getattr__(name):
    # The native API is imported lazily so `import paper_2605_15875_b200` works
    # on a CPU-only build host; every compute call fails loudly without the
    # CUDA library or a device (no CPU fallback).
    if name in ("api", "lib"):
        import importlib

        return importlib.import_module(f".{'api' if name == 'api' else '_lib'}", __name__)
    raise AttributeError(name)
