"""The C-ABI library loads without a GPU and exports every symbol include/*.h
declares; the catalogue answers; the Python binding mirrors the header."""
import ctypes
import glob
import os
import re

import pytest

from paper_2406_20037_b200 import _lib as L
from paper_2406_20037_b200 import knob_names, sketch_name, sketch_space, sketches

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*([a-z_0-9]+)\s*\(", src, re.M):
            names.add(m.group(1))
    names -= {"if", "int", "typedef"}
    return names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(L.LIB_PATH)
    names = declared_functions()
    assert len(names) >= 19
    missing = [n for n in sorted(names) if not hasattr(lib, n)]
    assert not missing, missing
    assert names <= set(L.SIGNATURES), sorted(names - set(L.SIGNATURES))


def test_struct_sizes_match_c_layout():
    assert ctypes.sizeof(L.Point) == 72
    assert ctypes.sizeof(L.Result) == 96
    assert ctypes.sizeof(L.Shape) == 4 + 4 + 11 * 8 + 6 * 4


def test_catalogue():
    assert sketches("dense", "f32") == [0, 7]
    assert sketches("batch_matmul", "f32") == [0, 7]
    assert sketches("conv2d", "f32") == [1, 8, 9]
    assert sketches("conv2d", "bf16") == [3, 11, 4, 10]
    assert sketches("dense", "bf16") == [2]
    assert sketch_name(0) == "simt_gemm_f32"
    assert knob_names(0) == ["BM", "BN", "BK", "TT", "UNROLL", "VEC", "STAGES", "SPLIT_K"]
    sp = sketch_space(0)
    assert sp[0] == [16, 32, 64, 128] and sp[7] == [1, 2, 3, 4, 6, 8, 12, 16]
    assert knob_names(2) == ["BM", "BN", "BK", "STAGES", "SPLIT_K", "SCHED", "RASTER", "EPI", "EW"]
    assert knob_names(3) == ["BM", "BN", "BK", "STAGES", "SPLIT_K", "TILE_Q", "SCHED", "RASTER", "EPI", "EW"]
    assert sketch_name(8) == "simt_pipe_conv_f32"
    assert knob_names(8) == ["BM", "BN", "BK", "TT", "KW", "VEC", "STAGES", "SPLIT_K", "OCC", "RED"]
    assert sketch_name(10) == "simt_direct_conv_bf16"
    assert knob_names(9) == ["KT", "TP", "PX", "BKC", "EPI"]
    assert sketch_name(11) == "tc_halo_conv_bf16"
    assert knob_names(11) == ["BM", "BN", "STAGES", "EPI", "EW"]
    assert sketch_name(99) is None


def test_measured_mode_rejects_uncompiled_values():
    import torch
    from paper_2406_20037_b200 import Tuner, TunerError
    x = torch.zeros(4)
    with pytest.raises(TunerError, match="EINVAL"):
        Tuner("dense", {"m": 4, "n": 4, "k": 4}, spaces=[(0, [[24], [16], [4], [4], [1], [4], [2], [1]])], x=x, w=x, y=x,
              stream=0)


def test_instantiation_lists_match_their_generator():
    # the explicit-instantiation TUs of the SIMT sketches are exactly what tools/gen_instantiations.py emits
    import subprocess
    import sys
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "gen_instantiations.py"), "--check"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


def test_sketch_valid_error_paths():
    """tuner_sketch_valid: ERANGE for an unknown sketch, EDIM for a wrong value count, EINVAL for a bad
    shape (include/tuner.h); a valid query answers without a device."""
    import pytest as _pt

    from paper_2406_20037_b200 import TunerError, sketch_space, sketch_valid
    shape = {"N": 1, "C": 64, "H": 56, "W": 56, "K": 64, "R": 3, "S": 3, "pad": (1, 1)}
    v = [s[0] for s in sketch_space(1)]
    assert isinstance(sketch_valid("conv2d", shape, 1, v), bool)
    with _pt.raises(TunerError):
        sketch_valid("conv2d", shape, 99, v)          # ERANGE
    with _pt.raises(TunerError):
        sketch_valid("conv2d", shape, 1, v[:-1])      # EDIM
    with _pt.raises(TunerError):
        sketch_valid("conv2d", dict(shape, C=0), 1, v)  # EINVAL
