"""paper_1803_04782_b200 — B200-native engine for the per-tick hot path of the discrete
social-field pedestrian model (arXiv 1803.04782).

Layout:
  csrc/      hand-written sm_100a CUDA kernels + the C ABI (include/socfield_cuda.h)
  host/      C++ host mirror of the reference's socfield API (include/socfield/*.hpp)
  bindings/  pybind11 module with the reference's Python surface -> socfield/_core
  lib/       built shared libraries (git-ignored; `python -m paper_1803_04782_b200.build`)

Nothing in this package imports the CPU oracle (oracle/); there is no CPU fallback.
"""
import os

PACKAGE_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.path.join(PACKAGE_DIR, "lib")


def library_path(name: str) -> str:
    """Absolute path of a built shared library; raises if the build has not been run."""
    path = os.path.join(LIB_DIR, name)
    if not os.path.exists(path):
        raise FileNotFoundError(
            f"{path} is missing: run `python -m paper_1803_04782_b200.build` (nvcc, sm_100a). "
            "The engine has no CPU fallback.")
    return path
