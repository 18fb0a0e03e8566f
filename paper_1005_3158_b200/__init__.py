"""B200-native explicit element-by-element FE step of the castfem reference
(arXiv 1005.3158): transient heat conduction with phase change.

Public API: paper_1005_3158_b200.castfem (reference-mirrored types and
solve()), paper_1005_3158_b200.configs (BASELINE fixtures). The compute path
is libcastfem_b200.so (sm_100a CUDA + C++ host) behind include/castfem_b200.h.
"""
from . import castfem  # noqa: F401
from .castfem import *  # noqa: F401,F403
