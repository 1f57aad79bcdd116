"""B200-native Paralpha hot path (arXiv 2103.12571): libpint.so (C ABI, sm_100a kernels) + ctypes binding."""
from .pint import (EXPORTS, Group, PintError, Solver, adaptive_schedule, experiments_enabled,  # noqa: F401
                   load_library, make_problem,
                   nccl_unique_id, tableau)
