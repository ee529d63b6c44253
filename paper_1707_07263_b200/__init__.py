"""B200-native complex-to-complex FFT path of tilefft (arXiv 1707.07263).

Public API mirrors the reference's plan/execute entry points; see
``tilefft.py`` (Python) and ``include/tilefft/*.hpp`` (C++). The compute runs
in ``libtilefft_b200.so`` (CUDA, sm_100a) behind the C ABI in
``include/tilefft_b200.h``.
"""
from .tilefft import (  # noqa: F401
    ExecConfig, FastBuffer, StageGeometry, apply_interstage_twiddles, exchange_transpose, fft_levelwise,
    ifft_levelwise, make_stage_buffer, stage_row_fft, StagePlan, TwiddleTable, bit_reverse, bit_reverse_permutation,
    build_twiddle_table, exchange_index_map, fft2_tiled, fft_tiled, fft_tiled_device, final_output_index,
    gather_source_index, ifft_tiled, is_power_of_two, kDefaultTwiddleResolution, log2_exact, make_plan,
    scatter_target_index, twiddle_lookup,
)
from . import _capi  # noqa: F401

__version__ = "0.1.0"
