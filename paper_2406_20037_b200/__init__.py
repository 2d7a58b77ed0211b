"""paper_2406_20037_b200 — B200-native hot path of "Explore as a Storm, Exploit
as a Raindrop" (arXiv 2406.20037): measuring candidate kernel schedules for
Ansor-style sampling + Droplet Search, behind the C ABI in include/tuner.h.
"""
from .tuner import (Sample, Tuner, global_launch_count, knob_names, probe_fp32_peak, rank_sum_p, schedule, sketch_name,  # noqa: F401
                    sketch_space, sketch_valid, sketches)
from ._lib import LIB_PATH, TunerError  # noqa: F401

SK_SIMT_GEMM_F32 = 0
SK_SIMT_IGEMM_CONV_F32 = 1
SK_TC_GEMM_BF16 = 2
SK_TC_IGEMM_CONV_BF16 = 3
SK_SIMT_IGEMM_CONV_BF16 = 4
SK_SIMT_DWCONV_F32 = 5
SK_SIMT_DWCONV_BF16 = 6
SK_SIMT_PIPE_GEMM_F32 = 7
SK_SIMT_PIPE_CONV_F32 = 8
SK_SIMT_DIRECT_CONV_F32 = 9
SK_SIMT_DIRECT_CONV_BF16 = 10
SK_TC_HALO_CONV_BF16 = 11
