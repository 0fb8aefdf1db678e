"""B200-native hot path of arXiv:1009.4975 (dynamic AMR topology optimization):
matrix-free SIMP elasticity operator with hanging-node elimination inside
Jacobi-PCG, sensitivities and the volume-weighted filter, as a C-ABI CUDA
library (libtomesh.so, include/tomesh.h) with a thin Python binding.
"""
from . import _lib  # noqa: F401
from . import api, amr, shard  # noqa: F401
from .api import HostMesh, Mesh, CgStats, prepare, tomesh_host_build  # noqa: F401
from ._lib import (TO_WARM, TO_FIXED_ITERS, TO_HISTORY, TO_NO_TRUE_RES, TO_PROFILE, TO_PROFILE_LOOP,  # noqa: F401
                   TO_FILTER_SENS, TO_FILTER_DENS, TO_UPLOAD_GENERAL, TO_UPLOAD_LAUNCHED, TO_UPLOAD_NO_CLUSTER,
                   TO_UPLOAD_EP, TO_UPLOAD_NO_EP,
                   TomeshError, TO_PC_JACOBI, TO_PC_IC0,
                   TO_OK, TO_NOT_CONVERGED, TO_EINVAL, TO_ECUDA, TO_ENOMEM, TO_EMESH, TO_ENAN,
                   TO_EBREAKDOWN, TO_ENONPOS_DIAG)
