"""B200-native Paralpha hot path (arXiv 2103.12571): libpint.so (C ABI, sm_100a kernels) + ctypes binding."""
from .pint import (EXPORTS, Group, PintError, Solver, adaptive_schedule, load_library, make_problem,  # noqa: F401
                   nccl_unique_id, tableau)
