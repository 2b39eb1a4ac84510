"""paper_2104_05877_b200 -- B200-native randomized LUPP skeleton selection.

The hot path of Dong & Martinsson, arXiv 2104.05877 (sketch X = Gamma A, LUPP on X^T
for the column skeletons J_s, LUPP on C = A(:, J_s) for the row skeletons I_s, the ID
coefficients and the residual), as hand-written sm_100a kernels behind the C ABI in
include/skel.h (libskel.so) with this thin ctypes binding on top.
"""
from .api import (  # noqa: F401
    DistSession, COL_ID, CUR, GAUSSIAN, ID_COEFFS, ROW_ID, SPARSE_SIGN, SkelError, context, fortran, gather_cols,
    gather_cols_shard, id_coeffs, launch_count, rand_lupp, residual, residual_cols, select_cols, select_cols_cpqr, select_cols_deim,
    LuppDist, LuppDistP2P, ipc_alloc, ipc_close, ipc_export, ipc_free, ipc_import, mailbox_bytes, select_rows,
    set_sketch_tuning, sketch, sketch_cols, sketch_dual, sketch_power, stream_select, id_estimate_cols,
    id_estimate_rows, ROW_COEFFS, CUR_CSS,
)
