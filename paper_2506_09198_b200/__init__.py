"""B200-native state-vector gate engine for the hot path of arXiv 2506.09198.

The product is the C-ABI library ``libqs_b200.so`` (include/qs.h), built from csrc/ for sm_100a;
``qs`` is its thin ctypes binding.  Import fails loudly if the library has not been built.
"""
from .qs import (  # noqa: F401
    QState, QSError, load_library, gates_array, qs_create, qs_create_virtual, qs_create_rank, qs_get_unique_id,
    qs_destroy, qs_init_basis, qs_init_random, qs_apply_1q, qs_apply_ctrl_1q, qs_apply_2q, qs_run_circuit,
    qs_read_amps, qs_write_amps, qs_read_amps_async, qs_write_amps_async, qs_norm2, qs_sync, qs_last_error, qs_info, qs_launch_count, qs_stream,
    qs_set_option, qs_last_plan, qs_jit_stats, qs_plan_route, qs_plan_decompose, qs_plan_passes, qs_plan_tile_jit,
    qs_plan_remap, qs_plan_hoist, LIB_PATH,
)
