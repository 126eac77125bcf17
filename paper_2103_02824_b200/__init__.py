"""B200-native correction-step hot path of the multilevel-correction adaptive FEM
for Kohn-Sham (arXiv 2103.02824): C++ host + hand-written sm_100a CUDA kernels
behind the C-ABI in include/ksb.h. See DESIGN.md."""
from .api import (MAT_AOP, MAT_M, MAT_S, MAT_USER0, POT_COULOMB, POT_GAUSSIAN, Context, DeviceArray,  # noqa: F401
                  Hierarchy, Level, Mesh, SolveStats, dorfler_mark, load_state, save_state)
from ._native import KsbError, LIB_PATH  # noqa: F401
