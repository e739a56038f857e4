"""B200-native (sm_100a) hot path of arXiv 2201.10369: fp32 Winograd / Toom-Cook
convolution with transform matrices built from arbitrary real point sets, scored
against fp64 direct convolution, swept over many candidate point sets.

Boundary: include/wino.h (C ABI, libwino.so).  This package is its thin binding
(``api``), the point-set templates (``points``) and the sweep/layer drivers
(``sweep``, ``layer``).  It never imports ``oracle/``.
"""
from .api import (  # noqa: F401
    WINO_MAXS,
    WINO_SUMS,
    WINO_SWEEP_NOFMA,
    conv2d,
    wino_conv2d_fp32,
    wino_conv2d_workspace_bytes,
    wino_error_sweep,
    wino_error_sweep_workspace_bytes,
    wino_last_launch_count,
    wino_points_to_matrices,
    wino_relu_pool_fp32,
    wino_supported,
    wino_sweep_outputs,
)
