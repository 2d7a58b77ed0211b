"""Seeded synthetic inputs shared by tests, bench.py and smoke().

This module holds NO arithmetic of the method (no contraction, no search step):
only seeded random tensors and seeded cost tables ("landscapes") laid out
densely per sketch in row-major linear-id order (DESIGN.md R-T1).  Both the
oracle and the CUDA path consume what it produces; neither is imported here.
"""
from .inputs import tensors, int_tensors, layer_tensors  # noqa: F401
from .landscapes import landscape, FAMILIES  # noqa: F401
from .workloads import RESNET18, RESNET50, VGG16, ALEXNET, BERT, CONFIG1, layer_flops  # noqa: F401
from .models import MODELS, model_layers  # noqa: F401
