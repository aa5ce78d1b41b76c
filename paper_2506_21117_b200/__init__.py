"""B200-native (sm_100a) implementation of the CL-Splats local-optimisation step
(arXiv 2506.21117, §3.3 "Local Optimization Kernel" and Supp. L508-541).

The step -- membership of O^t, dynamic tile mask, projection, binning, masked compositing,
masked backward, masked Adam -- is hand-written CUDA in ``csrc/`` behind the C ABI of
``include/cls.h`` (``libcls.so``).  ``step`` is the thin Python front end; ``dist`` shards
views over ranks with one NCCL all-reduce of the active gradient rows per step.

Importing a name from this package loads libcls.so; if it is not built, that raises
(there is no CPU fallback).  ``paper_2506_21117_b200.build`` compiles it.
"""
_LAZY = {"GaussianParams": "step", "LocalOptimizer": "step", "default_limits": "step", "k4": "step",
         "row4": "step", "Rows": "step", "GraphStep": "step"}

__all__ = list(_LAZY)


def __getattr__(name):
    if name in _LAZY:
        import importlib
        mod = importlib.import_module(f"{__name__}.{_LAZY[name]}")
        return getattr(mod, name)
    raise AttributeError(name)
