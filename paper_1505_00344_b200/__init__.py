"""B200-native Fireflies hot path (arXiv:1505.00344): RK4 particle swarms + density images.

The product is libfireflies.so (C ABI, include/fireflies.h); this package is its thin binding.
"""
from . import systems, views  # noqa: F401
from .fireflies import (Context, FFError, ff_abi_version, ff_compile_cubin, ff_create, ff_destroy,  # noqa: F401
                        ff_emit_source, ff_group_info, ff_init_group, ff_last_error, ff_project, ff_read_state,
                        ff_set_param, ff_step, ff_sweep_param, ff_sync, ff_write_state)
