"""Seeded input tensors (DESIGN.md §4 input recipe).

Values ~ U[-1, 1) float32 (the "tolerance" pass) or integers in {-2..2} (the
"exact" pass: every product and partial sum is an integer < 2^24, so any
summation order gives the bit-identical fp32 result).  Generator: numpy PCG64.
"""
from __future__ import annotations

import numpy as np


def tensors(shapes, seed: int, dist: str = "uniform"):
    """One float32 array per shape, drawn in order from one PCG64(seed) stream."""
    rng = np.random.Generator(np.random.PCG64(seed))
    out = []
    for shp in shapes:
        if dist == "uniform":
            out.append(rng.uniform(-1.0, 1.0, size=shp).astype(np.float32))
        elif dist == "int":
            out.append(rng.integers(-2, 3, size=shp).astype(np.float32))
        elif dist == "ones":
            out.append(np.ones(shp, np.float32))
        else:
            raise ValueError(dist)
    return out


def int_tensors(shapes, seed: int):
    return tensors(shapes, seed, "int")


def layer_tensors(layer: dict, seed: int, dist: str = "uniform"):
    """(X, W) for a workload layer dict (see synth.workloads)."""
    if layer["op"] == "conv2d":
        xs = (layer["N"], layer["H"], layer["W"], layer["C"])
        ws = (layer["K"], layer["R"], layer["S"], layer["C"])
    elif layer["op"] == "depthwise_conv2d":
        xs = (layer["N"], layer["H"], layer["W"], layer["C"])
        ws = (layer["C"], layer["R"], layer["S"])
    else:
        b = layer.get("b", 1)
        xs = (b, layer["m"], layer["k"])
        ws = (b, layer["n"], layer["k"])
    return tensors([xs, ws], seed, dist)
