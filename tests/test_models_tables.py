"""Pins for synth/models.py (the 20-model sweep's layer tables):
each model's multiply-accumulates, summed over its distinct tasks x count, equal
the published torchvision figure (GMACs per 224x224 image, 299x299 for
Inception-v3; torchvision model documentation [external]) within 4 %; squeeze-
excitation, pooling and element-wise work are excluded, hence the tolerance."""
import pytest

from synth.models import MODELS, model_layers
from synth.workloads import layer_flops, out_hw

TORCHVISION_GMACS = {
    "alexnet": 0.71, "vgg11": 7.61, "vgg13": 11.31, "vgg16": 15.47, "vgg19": 19.63, "resnet18": 1.81,
    "resnet34": 3.66, "resnet50": 4.09, "resnet101": 7.80, "resnet152": 11.51, "densenet121": 2.83,
    "densenet169": 3.36, "densenet201": 4.29, "mobilenetv2": 0.30, "mnasnet": 0.31, "squeezenet1.1": 0.35,
    "shufflenetv2": 0.14, "googlenet": 1.50, "inceptionv3": 5.71, "efficientnetb0": 0.39,
}


def test_twenty_models():
    assert len(MODELS) == 20 and set(MODELS) == set(TORCHVISION_GMACS)


@pytest.mark.parametrize("name", list(MODELS))
def test_model_macs_match_torchvision(name):
    layers = model_layers(name)
    gmacs = sum(layer_flops(L) * L["count"] for L in layers) / 2e9
    assert abs(gmacs / TORCHVISION_GMACS[name] - 1) < 0.04, gmacs
    assert len({L["name"] for L in layers}) == len(layers)
    for L in layers:
        if L["op"] != "dense":
            P, Q = out_hw(L)
            assert P >= 1 and Q >= 1


def test_batch_scales_work():
    a = sum(layer_flops(L) * L["count"] for L in model_layers("resnet50", 1))
    b = sum(layer_flops(L) * L["count"] for L in model_layers("resnet50", 16))
    assert b == 16 * a
