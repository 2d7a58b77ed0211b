"""ctypes mirror of include/tuner.h (argument marshalling only).

Loads the in-tree ``lib/libdroplet_b200.so`` and fails loudly if it is missing:
there is no Python or CPU fallback for any step of the hot path.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# DB200_LIB: another build of the same library (A/B experiments under tools/ only)
LIB_PATH = os.environ.get("DB200_LIB") or os.path.join(_HERE, "lib", "libdroplet_b200.so")

MAX_KNOBS = 16
MAX_VALUES = 64

OK, EINVAL, EDIM, ERANGE, EOVERFLOW, ESTATE, ECUDA, ENCCL, ENOMEM = range(9)
STATUS_NAMES = ["OK", "EINVAL", "EDIM", "ERANGE", "EOVERFLOW", "ESTATE", "ECUDA", "ENCCL", "ENOMEM"]
OP = {"dense": 0, "batch_matmul": 1, "conv2d": 2, "depthwise_conv2d": 3}
DTYPE = {"f32": 0, "bf16": 1}
S_OK, S_INVALID, S_TIMEOUT, S_WRONG, S_LAUNCH_FAIL = range(5)
SAMPLE_STATUS = ["ok", "invalid", "timeout", "wrong", "launch_fail"]
POLICY = {"plain": 0, "grow": 1, "radius": 2}


class Shape(C.Structure):
    _fields_ = [("dtype", C.c_int32), ("b", C.c_int64), ("m", C.c_int64), ("n", C.c_int64), ("k", C.c_int64),
                ("N", C.c_int64), ("C", C.c_int64), ("H", C.c_int64), ("W", C.c_int64), ("K", C.c_int64),
                ("R", C.c_int64), ("S", C.c_int64), ("stride_h", C.c_int32), ("stride_w", C.c_int32),
                ("pad_h", C.c_int32), ("pad_w", C.c_int32), ("dil_h", C.c_int32), ("dil_w", C.c_int32)]


class KnobSpace(C.Structure):
    _fields_ = [("sketch", C.c_int32), ("nknobs", C.c_int32), ("card", C.POINTER(C.c_int32)),
                ("values", C.POINTER(C.c_int32))]


class Point(C.Structure):
    _fields_ = [("sketch", C.c_int32), ("n", C.c_int32), ("idx", C.c_int32 * MAX_KNOBS)]


class Result(C.Structure):
    _fields_ = [("pt", Point), ("cost_ns", C.c_double), ("max_err", C.c_double), ("status", C.c_int32),
                ("rank", C.c_int32)]


ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64)


class Opts(C.Structure):
    _fields_ = [("warmup", C.c_int32), ("repeats", C.c_int32), ("number", C.c_int32), ("timeout_ms", C.c_double),
                ("seed", C.c_uint64), ("policy", C.c_int32), ("alpha", C.c_double), ("max_batch", C.c_int32),
                ("verify", C.c_int32), ("early_cut", C.c_double), ("cost_table", C.POINTER(C.c_double)), ("cost_table_len", C.c_int64),
                ("cost_samples", C.POINTER(C.c_double)), ("cost_nsamp", C.c_int32),
                ("rank", C.c_int32), ("world", C.c_int32), ("nccl_unique_id", C.c_void_p),
                ("allgather", ALLGATHER_FN), ("allgather_ctx", C.c_void_p), ("x", C.c_void_p), ("w", C.c_void_p),
                ("y", C.c_void_p), ("y_ref", C.c_void_p), ("y_absref", C.c_void_p), ("stream", C.c_void_p),
                ("trial_log", C.c_char_p)]


class DropletReport(C.Structure):
    _fields_ = [("best", Point), ("best_cost", C.c_double), ("trials_used", C.c_int32), ("rounds", C.c_int32),
                ("converged", C.c_int32), ("traj_len", C.c_int32)]


class Buffers(C.Structure):
    _fields_ = [("x", C.c_void_p), ("w", C.c_void_p), ("y", C.c_void_p)]


class Stats(C.Structure):
    _fields_ = [("kernel_launches", C.c_int64), ("candidates", C.c_int64), ("collectives", C.c_int64),
                ("batches", C.c_int64), ("measure_wall_ns", C.c_double), ("early_cut", C.c_int64),
                ("light", C.c_int64), ("precise", C.c_int64), ("calibrations", C.c_int64),
                ("replayed", C.c_int64)]


# name -> (restype, argtypes); every function declared in include/tuner.h
SIGNATURES = {
    "tuner_opts_default": (None, [C.POINTER(Opts)]),
    "tuner_sketches": (C.c_int, [C.c_int32, C.c_int32, C.POINTER(C.c_int32), C.c_int32, C.POINTER(C.c_int32)]),
    "tuner_sketch_space": (C.c_int, [C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "tuner_sketch_valid": (C.c_int, [C.c_int32, C.POINTER(Shape), C.c_int32, C.POINTER(C.c_int32), C.c_int32,
                                     C.POINTER(C.c_int32)]),
    "tuner_sketch_name": (C.c_char_p, [C.c_int32]),
    "tuner_knob_name": (C.c_char_p, [C.c_int32, C.c_int32]),
    "tuner_create": (C.c_int, [C.c_int32, C.POINTER(Shape), C.POINTER(KnobSpace), C.c_int32, C.POINTER(Opts),
                               C.POINTER(C.c_void_p)]),
    "tuner_point_valid": (C.c_int, [C.c_void_p, C.POINTER(Point), C.POINTER(C.c_int32)]),
    "tuner_sample": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(Result), C.POINTER(C.c_int32)]),
    "tuner_measure": (C.c_int, [C.c_void_p, C.POINTER(Point), C.c_int32, C.POINTER(Result)]),
    "tuner_schedule": (C.c_int, [C.POINTER(C.c_void_p), C.c_int32, C.POINTER(C.c_double), C.c_int64, C.c_int32,
                                 C.c_double, C.c_int32, C.c_int32, C.POINTER(C.c_int64)]),
    "tuner_grid": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(Result), C.POINTER(C.c_int32)]),
    "tuner_evolve": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.POINTER(Result), C.POINTER(C.c_int32)]),
    "tuner_droplet": (C.c_int, [C.c_void_p, C.POINTER(Point), C.c_int32, C.POINTER(Point), C.c_int32,
                                C.POINTER(DropletReport)]),
    "tuner_best": (C.c_int, [C.c_void_p, C.POINTER(Result)]),
    "tuner_best_of_sketch": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(Result)]),
    "tuner_timings": (C.c_int, [C.c_void_p, C.POINTER(Point), C.POINTER(C.c_float), C.c_int32, C.POINTER(C.c_int32)]),
    "tuner_history": (C.c_int, [C.c_void_p, C.POINTER(Result), C.c_int64, C.POINTER(C.c_int64)]),
    "kernel_run": (C.c_int, [C.c_void_p, C.POINTER(Point), C.POINTER(Buffers), C.c_void_p]),
    "tuner_reference": (C.c_int, [C.c_void_p, C.POINTER(Buffers), C.c_void_p, C.c_void_p, C.c_void_p]),
    "tuner_get_stats": (C.c_int, [C.c_void_p, C.POINTER(Stats)]),
    "tuner_nccl_unique_id": (C.c_int, [C.c_void_p]),
    "tuner_destroy": (None, [C.c_void_p]),
    "tuner_last_error": (C.c_char_p, []),
    "tuner_global_launch_count": (C.c_int64, []),
    "tuner_rank_sum_p": (C.c_int, [C.POINTER(C.c_float), C.c_int32, C.POINTER(C.c_float), C.c_int32,
                                   C.POINTER(C.c_double)]),
    "tuner_probe_fp32_peak": (C.c_int, [C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
}

_LIB = None


def lib():
    """The loaded library (raises if the CUDA extension was not built)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
        if "DROPLET_NCCL_LIB" not in os.environ:
            try:
                import nvidia.nccl  # the libnccl torch uses
                cand = os.path.join(list(nvidia.nccl.__path__)[0], "lib", "libnccl.so.2")
                if os.path.exists(cand):
                    os.environ["DROPLET_NCCL_LIB"] = cand
            except Exception:
                pass
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _LIB = L
    return _LIB


class TunerError(RuntimeError):
    def __init__(self, status, msg):
        self.status = status
        name = STATUS_NAMES[status] if 0 <= status < len(STATUS_NAMES) else str(status)
        super().__init__(f"{name}: {msg}")


def check(status):
    if status != OK:
        raise TunerError(status, lib().tuner_last_error().decode(errors="replace"))
