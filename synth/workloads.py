"""Layer shapes of the BASELINE.json configs.

The paper's 20-model list is in a lost figure; the models it names in
prose are AlexNet, VGG, ResNet, MobileNet, Inception, GoogleNet, DenseNet,
MnasNet.  Shapes are the standard torchvision architectures.
conv2d layers are NHWC / KRSC / NPQK, groups = 1.
"""
from __future__ import annotations


def conv(name, N, C, K, H, R, stride=1, pad=None, W=None, S=None, dil=1):
    S = R if S is None else S
    W = H if W is None else W
    pad = (R // 2) if pad is None else pad
    return {"op": "conv2d", "name": name, "N": N, "C": C, "K": K, "H": H, "W": W, "R": R, "S": S,
            "stride": (stride, stride), "pad": (pad, pad), "dil": (dil, dil)}


def dense(name, m, n, k):
    return {"op": "dense", "name": name, "b": 1, "m": m, "n": n, "k": k}


def bmm(name, b, m, n, k):
    return {"op": "batch_matmul", "name": name, "b": b, "m": m, "n": n, "k": k}


def out_hw(layer):
    (sh, sw), (ph, pw), (dh, dw) = layer["stride"], layer["pad"], layer["dil"]
    P = (layer["H"] + 2 * ph - dh * (layer["R"] - 1) - 1) // sh + 1
    Q = (layer["W"] + 2 * pw - dw * (layer["S"] - 1) - 1) // sw + 1
    return P, Q


def layer_flops(layer) -> float:
    if layer["op"] == "conv2d":
        P, Q = out_hw(layer)
        return 2.0 * layer["N"] * layer["K"] * P * Q * layer["C"] * layer["R"] * layer["S"]
    if layer["op"] == "depthwise_conv2d":
        P, Q = out_hw(layer)
        return 2.0 * layer["N"] * layer["C"] * P * Q * layer["R"] * layer["S"]
    return 2.0 * layer.get("b", 1) * layer["m"] * layer["n"] * layer["k"]


# config 1: dense 512x512x512 fp32
CONFIG1 = dense("dense512", 512, 512, 512)

# config 2: ResNet-18 (11 distinct conv layers) and ResNet-50 v1.5 (23), batch 1, 224x224
RESNET18 = [
    conv("r18.conv1", 1, 3, 64, 224, 7, 2, 3),
    conv("r18.l1.3x3", 1, 64, 64, 56, 3, 1),
    conv("r18.l2.3x3s2", 1, 64, 128, 56, 3, 2),
    conv("r18.l2.ds", 1, 64, 128, 56, 1, 2, 0),
    conv("r18.l2.3x3", 1, 128, 128, 28, 3, 1),
    conv("r18.l3.3x3s2", 1, 128, 256, 28, 3, 2),
    conv("r18.l3.ds", 1, 128, 256, 28, 1, 2, 0),
    conv("r18.l3.3x3", 1, 256, 256, 14, 3, 1),
    conv("r18.l4.3x3s2", 1, 256, 512, 14, 3, 2),
    conv("r18.l4.ds", 1, 256, 512, 14, 1, 2, 0),
    conv("r18.l4.3x3", 1, 512, 512, 7, 3, 1),
]

RESNET50 = [
    conv("r50.conv1", 1, 3, 64, 224, 7, 2, 3),
    conv("r50.s1.1x1a", 1, 64, 64, 56, 1),
    conv("r50.s1.3x3", 1, 64, 64, 56, 3),
    conv("r50.s1.1x1b", 1, 64, 256, 56, 1),
    conv("r50.s1.1x1c", 1, 256, 64, 56, 1),
    conv("r50.s2.1x1a0", 1, 256, 128, 56, 1),
    conv("r50.s2.3x3s2", 1, 128, 128, 56, 3, 2),
    conv("r50.s2.1x1b", 1, 128, 512, 28, 1),
    conv("r50.s2.ds", 1, 256, 512, 56, 1, 2, 0),
    conv("r50.s2.1x1a", 1, 512, 128, 28, 1),
    conv("r50.s2.3x3", 1, 128, 128, 28, 3),
    conv("r50.s3.1x1a0", 1, 512, 256, 28, 1),
    conv("r50.s3.3x3s2", 1, 256, 256, 28, 3, 2),
    conv("r50.s3.1x1b", 1, 256, 1024, 14, 1),
    conv("r50.s3.ds", 1, 512, 1024, 28, 1, 2, 0),
    conv("r50.s3.1x1a", 1, 1024, 256, 14, 1),
    conv("r50.s3.3x3", 1, 256, 256, 14, 3),
    conv("r50.s4.1x1a0", 1, 1024, 512, 14, 1),
    conv("r50.s4.3x3s2", 1, 512, 512, 14, 3, 2),
    conv("r50.s4.1x1b", 1, 512, 2048, 7, 1),
    conv("r50.s4.ds", 1, 1024, 2048, 14, 1, 2, 0),
    conv("r50.s4.1x1a", 1, 2048, 512, 7, 1),
    conv("r50.s4.3x3", 1, 512, 512, 7, 3),
]

# config 3: VGG-16 (9 distinct) and AlexNet (5), batch 16, bf16
VGG16 = [
    conv("vgg.3-64@224", 16, 3, 64, 224, 3),
    conv("vgg.64-64@224", 16, 64, 64, 224, 3),
    conv("vgg.64-128@112", 16, 64, 128, 112, 3),
    conv("vgg.128-128@112", 16, 128, 128, 112, 3),
    conv("vgg.128-256@56", 16, 128, 256, 56, 3),
    conv("vgg.256-256@56", 16, 256, 256, 56, 3),
    conv("vgg.256-512@28", 16, 256, 512, 28, 3),
    conv("vgg.512-512@28", 16, 512, 512, 28, 3),
    conv("vgg.512-512@14", 16, 512, 512, 14, 3),
]
ALEXNET = [
    conv("alex.conv1", 16, 3, 64, 224, 11, 4, 2),
    conv("alex.conv2", 16, 64, 192, 27, 5, 1, 2),
    conv("alex.conv3", 16, 192, 384, 13, 3),
    conv("alex.conv4", 16, 384, 256, 13, 3),
    conv("alex.conv5", 16, 256, 256, 13, 3),
]


# config 4: BERT-base, seq 512, bf16
def bert(batch=16, seq=512, hidden=768, heads=12, ffn=3072):
    m = batch * seq
    dh = hidden // heads
    return [
        dense("bert.qkv", m, 3 * hidden, hidden),
        dense("bert.attn_out", m, hidden, hidden),
        dense("bert.ffn1", m, ffn, hidden),
        dense("bert.ffn2", m, hidden, ffn),
        bmm("bert.qk", heads * batch, seq, seq, dh),
        bmm("bert.av", heads * batch, seq, dh, seq),
    ]


BERT = bert()
