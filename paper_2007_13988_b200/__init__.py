"""paper_2007_13988_b200 — B200-native accelerated PIFu inference path.

Progressive surface localization + mesh-free first-crossing rendering as
hand-written sm_100a kernels behind a C ABI (include/isocull_b200.h).  This
package holds the CUDA sources (csrc/), the built library
(libisocull_b200.so) and a thin ctypes face (abi.py, api.py) mirroring the
reference's operator API.  Nothing here imports the CPU oracle (oracle/).
"""
from . import abi  # noqa: F401

__all__ = ["abi", "api"]
