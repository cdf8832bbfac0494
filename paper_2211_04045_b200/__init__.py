"""B200-native two-way continuous collision handling (arXiv 2211.04045).

The hot path — proximity search (LBVH broad phase + exact FP64 narrow phase),
contact / edge-length linearization, multi-color projected Gauss-Seidel and the
conservative forward step, with Alg. 1's loop and convergence test resident on
the device — is hand-written CUDA for sm_100a in ``csrc/``, exported through
the C-ABI ``include/tw_c.h`` (``libtwoway_b200.so``). ``capi`` binds it from
Python; ``_twoway`` mirrors the reference's pybind11 module; ``scenes`` builds
the fixture battery and the benchmark scenes.
"""
import os

__all__ = ["capi", "scenes", "lib_path"]


def lib_path() -> str:
    return os.path.join(os.path.dirname(os.path.abspath(__file__)), "libtwoway_b200.so")
