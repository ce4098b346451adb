"""B200-native initial guesses for sequences of linear systems (arXiv 2009.10863).

The hot path is hand-written sm_100a CUDA in ``libig.so`` behind the C ABI ``include/ig.h``;
this package is its thin Python binding (``ig``) plus the build script.  There is no CPU
fallback: if ``libig.so`` is missing every call raises.
"""

from .ig import (  # noqa: F401
    IG_EXTRAP_LS,
    IG_EXTRAP_SPARSE,
    IG_PROJ_CLASSIC,
    IG_PROJ_QR,
    IGError,
    InitialGuess,
    comm_from_process_group,
    ig_attach_comm,
    ig_bytes,
    ig_comm_create,
    ig_comm_destroy,
    ig_comm_unique_id,
    ig_copy_history,
    ig_create,
    ig_create_ext,
    ig_storage_bytes,
    ig_destroy,
    ig_form_guess,
    ig_form_guess_host,
    ig_get_stats,
    ig_history_dim,
    ig_next_slot,
    ig_profile,
    ig_profile_read,
    ig_reset,
    ig_set_admit_tol,
    ig_set_schedule,
    ig_set_stream,
    ig_total_launches,
    ig_update,
    ig_update_host,
    ig_weights,
    shard_range,
    ig_set_grid_limit,
    ig_set_watchdog,
    ig_xwin_export,
    ig_xwin_ptr,
    ig_attach_peers,
    peers_from_process_group,
    attach_virtual_ranks,
)
