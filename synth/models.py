"""Layer tables of the paper's 20-model sweep (BASELINE.json configs[4]).

The paper's model list is in a lost figure; the prose names AlexNet, VGG,
ResNet, MobileNet, Inception, GoogleNet, DenseNet(-201) and MnasNet (P:35,
P:93-95).  SURVEY §8(d).1 fixes the 20: AlexNet, VGG-11/13/16/19,
ResNet-18/34/50/101/152, DenseNet-121/169/201, MobileNet-v2, MnasNet,
SqueezeNet-1.1, ShuffleNet-v2, GoogLeNet, Inception-v3, EfficientNet-B0.  The
shapes are the standard (torchvision) architectures.  Each model is a list of
its DISTINCT tuning tasks (conv2d groups = 1, depthwise conv2d, dense), each with
``count`` = how often the shape occurs in one forward pass (the weight of the
multi-layer budget scheduler).  Squeeze-excitation FCs, pooling and
element-wise ops are not tuning tasks here.  Only shapes: no arithmetic of the
method lives in this module.
"""
from __future__ import annotations

from collections import OrderedDict


class _Net:
    def __init__(self, name: str, batch: int):
        self.name, self.batch = name, batch
        self.tasks: "OrderedDict[tuple, dict]" = OrderedDict()

    def _add(self, key, layer):
        if key in self.tasks:
            self.tasks[key]["count"] += 1
        else:
            layer["name"] = f"{self.name}.{len(self.tasks)}"
            layer["count"] = 1
            self.tasks[key] = layer

    def conv(self, C, K, H, R, stride=1, pad=None, W=None, S=None):
        """groups = 1 conv; returns the output spatial size (P, Q)."""
        S = R if S is None else S
        W = H if W is None else W
        if pad is None:
            pad = (R // 2, S // 2)
        elif isinstance(pad, int):
            pad = (pad, pad)
        P = (H + 2 * pad[0] - (R - 1) - 1) // stride + 1
        Q = (W + 2 * pad[1] - (S - 1) - 1) // stride + 1
        key = ("conv2d", C, K, H, W, R, S, stride, pad)
        self._add(key, {"op": "conv2d", "N": self.batch, "C": C, "K": K, "H": H, "W": W, "R": R, "S": S,
                        "stride": (stride, stride), "pad": tuple(pad), "dil": (1, 1)})
        return P, Q

    def dw(self, C, H, R, stride=1):
        """depthwise conv (groups = C = K); returns the output size."""
        pad = R // 2
        P = (H + 2 * pad - (R - 1) - 1) // stride + 1
        key = ("depthwise_conv2d", C, H, R, stride)
        self._add(key, {"op": "depthwise_conv2d", "N": self.batch, "C": C, "K": C, "H": H, "W": H, "R": R,
                        "S": R, "stride": (stride, stride), "pad": (pad, pad), "dil": (1, 1)})
        return P

    def fc(self, k, n):
        self._add(("dense", k, n), {"op": "dense", "b": 1, "m": self.batch, "n": n, "k": k})

    def layers(self):
        return list(self.tasks.values())


def alexnet(batch=1):
    m = _Net("alexnet", batch)
    m.conv(3, 64, 224, 11, 4, 2)
    m.conv(64, 192, 27, 5, 1, 2)
    m.conv(192, 384, 13, 3)
    m.conv(384, 256, 13, 3)
    m.conv(256, 256, 13, 3)
    m.fc(9216, 4096); m.fc(4096, 4096); m.fc(4096, 1000)
    return m.layers()


_VGG = {11: [64, "M", 128, "M", 256, 256, "M", 512, 512, "M", 512, 512, "M"],
        13: [64, 64, "M", 128, 128, "M", 256, 256, "M", 512, 512, "M", 512, 512, "M"],
        16: [64, 64, "M", 128, 128, "M", 256, 256, 256, "M", 512, 512, 512, "M", 512, 512, 512, "M"],
        19: [64, 64, "M", 128, 128, "M", 256, 256, 256, 256, "M", 512, 512, 512, 512, "M",
             512, 512, 512, 512, "M"]}


def vgg(depth, batch=1):
    m = _Net(f"vgg{depth}", batch)
    c, h = 3, 224
    for v in _VGG[depth]:
        if v == "M":
            h //= 2
        else:
            m.conv(c, v, h, 3)
            c = v
    m.fc(25088, 4096); m.fc(4096, 4096); m.fc(4096, 1000)
    return m.layers()


def resnet(depth, batch=1):
    """torchvision ResNet (v1.5: the bottleneck's stride is on the 3x3)."""
    blocks = {18: [2, 2, 2, 2], 34: [3, 4, 6, 3], 50: [3, 4, 6, 3], 101: [3, 4, 23, 3], 152: [3, 8, 36, 3]}[depth]
    bottleneck = depth >= 50
    m = _Net(f"resnet{depth}", batch)
    m.conv(3, 64, 224, 7, 2, 3)
    h, cin = 56, 64
    for stage, nb in enumerate(blocks):
        width = 64 * 2 ** stage
        cout = width * 4 if bottleneck else width
        for b in range(nb):
            s = 2 if (b == 0 and stage > 0) else 1
            ho = h // s
            if bottleneck:
                m.conv(cin, width, h, 1, 1, 0)
                m.conv(width, width, h, 3, s)
                m.conv(width, cout, ho, 1, 1, 0)
            else:
                m.conv(cin, width, h, 3, s)
                m.conv(width, width, ho, 3, 1)
            if b == 0 and (s != 1 or cin != cout):
                m.conv(cin, cout, h, 1, s, 0)
            cin, h = cout, ho
    m.fc(cin, 1000)
    return m.layers()


def densenet(depth, batch=1):
    cfg = {121: (6, 12, 24, 16), 169: (6, 12, 32, 32), 201: (6, 12, 48, 32)}[depth]
    growth, bn = 32, 4
    m = _Net(f"densenet{depth}", batch)
    m.conv(3, 64, 224, 7, 2, 3)
    c, h = 64, 56
    for i, nl in enumerate(cfg):
        for j in range(nl):
            m.conv(c + j * growth, bn * growth, h, 1, 1, 0)
            m.conv(bn * growth, growth, h, 3)
        c += nl * growth
        if i < len(cfg) - 1:
            m.conv(c, c // 2, h, 1, 1, 0)
            c, h = c // 2, h // 2
    m.fc(c, 1000)
    return m.layers()


def _mbconv(m, cin, cout, h, expand, k, stride):
    mid = cin * expand
    if expand != 1:
        m.conv(cin, mid, h, 1, 1, 0)
    ho = m.dw(mid, h, k, stride)
    m.conv(mid, cout, ho, 1, 1, 0)
    return ho


def mobilenet_v2(batch=1):
    m = _Net("mobilenetv2", batch)
    m.conv(3, 32, 224, 3, 2)
    c, h = 32, 112
    for t, co, n, s in [(1, 16, 1, 1), (6, 24, 2, 2), (6, 32, 3, 2), (6, 64, 4, 2), (6, 96, 3, 1),
                        (6, 160, 3, 2), (6, 320, 1, 1)]:
        for i in range(n):
            h = _mbconv(m, c, co, h, t, 3, s if i == 0 else 1)
            c = co
    m.conv(320, 1280, h, 1, 1, 0)
    m.fc(1280, 1000)
    return m.layers()


def mnasnet(batch=1):
    """torchvision mnasnet1_0."""
    m = _Net("mnasnet", batch)
    m.conv(3, 32, 224, 3, 2)
    h = m.dw(32, 112, 3, 1)
    m.conv(32, 16, h, 1, 1, 0)
    c = 16
    for t, k, s, co, n in [(3, 3, 2, 24, 3), (3, 5, 2, 40, 3), (6, 5, 2, 80, 3), (6, 3, 1, 96, 2),
                           (6, 5, 2, 192, 4), (6, 3, 1, 320, 1)]:
        for i in range(n):
            h = _mbconv(m, c, co, h, t, k, s if i == 0 else 1)
            c = co
    m.conv(320, 1280, h, 1, 1, 0)
    m.fc(1280, 1000)
    return m.layers()


def efficientnet_b0(batch=1):
    m = _Net("efficientnetb0", batch)
    m.conv(3, 32, 224, 3, 2)
    c, h = 32, 112
    for t, k, s, co, n in [(1, 3, 1, 16, 1), (6, 3, 2, 24, 2), (6, 5, 2, 40, 2), (6, 3, 2, 80, 3),
                           (6, 5, 1, 112, 3), (6, 5, 2, 192, 4), (6, 3, 1, 320, 1)]:
        for i in range(n):
            h = _mbconv(m, c, co, h, t, k, s if i == 0 else 1)
            c = co
    m.conv(320, 1280, h, 1, 1, 0)
    m.fc(1280, 1000)
    return m.layers()


def squeezenet11(batch=1):
    m = _Net("squeezenet1.1", batch)
    m.conv(3, 64, 224, 3, 2, 0)  # -> 111, maxpool -> 55
    h = 55
    fires = [(64, 16, 64), (128, 16, 64), "M", (128, 32, 128), (256, 32, 128), "M",
             (256, 48, 192), (384, 48, 192), (384, 64, 256), (512, 64, 256)]
    for f in fires:
        if f == "M":
            h = (h - 3) // 2 + 1 + ((h - 3) % 2 > 0)  # ceil-mode 3x3/2 max pool: 55 -> 27 -> 13
            continue
        cin, sq, ex = f
        m.conv(cin, sq, h, 1, 1, 0)
        m.conv(sq, ex, h, 1, 1, 0)
        m.conv(sq, ex, h, 3)
    m.conv(512, 1000, 13, 1, 1, 0)
    return m.layers()


def shufflenet_v2(batch=1):
    """torchvision shufflenet_v2_x1_0."""
    m = _Net("shufflenetv2", batch)
    m.conv(3, 24, 224, 3, 2)
    c, h = 24, 56
    for co, reps in [(116, 4), (232, 8), (464, 4)]:
        mid = co // 2
        for i in range(reps):
            if i == 0:  # down-sampling unit: both branches see the full input
                ho = m.dw(c, h, 3, 2)
                m.conv(c, mid, ho, 1, 1, 0)
                m.conv(c, mid, h, 1, 1, 0)
                m.dw(mid, h, 3, 2)
                m.conv(mid, mid, ho, 1, 1, 0)
                h = ho
            else:
                m.conv(mid, mid, h, 1, 1, 0)
                m.dw(mid, h, 3, 1)
                m.conv(mid, mid, h, 1, 1, 0)
        c = co
    m.conv(464, 1024, 7, 1, 1, 0)
    m.fc(1024, 1000)
    return m.layers()


def googlenet(batch=1):
    """torchvision GoogLeNet (its '5x5' branch is a 3x3)."""
    m = _Net("googlenet", batch)
    m.conv(3, 64, 224, 7, 2, 3)
    m.conv(64, 64, 56, 1, 1, 0)
    m.conv(64, 192, 56, 3)
    h = 28
    mods = [(192, 64, 96, 128, 16, 32, 32), (256, 128, 128, 192, 32, 96, 64), "M",
            (480, 192, 96, 208, 16, 48, 64), (512, 160, 112, 224, 24, 64, 64), (512, 128, 128, 256, 24, 64, 64),
            (512, 112, 144, 288, 32, 64, 64), (528, 256, 160, 320, 32, 128, 128), "M",
            (832, 256, 160, 320, 32, 128, 128), (832, 384, 192, 384, 48, 128, 128)]
    for md in mods:
        if md == "M":
            h //= 2
            continue
        cin, b1, r3, b3, r5, b5, pp = md
        m.conv(cin, b1, h, 1, 1, 0)
        m.conv(cin, r3, h, 1, 1, 0)
        m.conv(r3, b3, h, 3)
        m.conv(cin, r5, h, 1, 1, 0)
        m.conv(r5, b5, h, 3)
        m.conv(cin, pp, h, 1, 1, 0)
    m.fc(1024, 1000)
    return m.layers()


def inception_v3(batch=1):
    """torchvision Inception-v3 (299 x 299 input, no aux head)."""
    m = _Net("inceptionv3", batch)
    m.conv(3, 32, 299, 3, 2, 0)      # 149
    m.conv(32, 32, 149, 3, 1, 0)     # 147
    m.conv(32, 64, 147, 3, 1, 1)     # 147 -> pool 73
    m.conv(64, 80, 73, 1, 1, 0)
    m.conv(80, 192, 73, 3, 1, 0)     # 71 -> pool 35
    h = 35
    for cin, pool in [(192, 32), (256, 64), (288, 64)]:  # InceptionA
        m.conv(cin, 64, h, 1, 1, 0)  # branch1x1
        m.conv(cin, 64, h, 1, 1, 0)  # branch3x3dbl_1
        m.conv(cin, 48, h, 1, 1, 0)
        m.conv(48, 64, h, 5, 1, 2)
        m.conv(64, 96, h, 3)
        m.conv(96, 96, h, 3)
        m.conv(cin, pool, h, 1, 1, 0)
    m.conv(288, 384, 35, 3, 2, 0)    # InceptionB -> 17
    m.conv(288, 64, 35, 1, 1, 0)
    m.conv(64, 96, 35, 3)
    m.conv(96, 96, 35, 3, 2, 0)
    h = 17
    for c7 in (128, 160, 160, 192):  # InceptionC
        m.conv(768, 192, h, 1, 1, 0)            # branch1x1
        m.conv(768, c7, h, 1, 1, 0)             # branch7x7_1
        m.conv(c7, c7, h, 1, 1, (0, 3), S=7)    # 1x7
        m.conv(c7, 192, h, 7, 1, (3, 0), S=1)   # 7x1
        m.conv(768, c7, h, 1, 1, 0)             # branch7x7dbl_1
        m.conv(c7, c7, h, 7, 1, (3, 0), S=1)    # 7x1
        m.conv(c7, c7, h, 1, 1, (0, 3), S=7)    # 1x7
        m.conv(c7, c7, h, 7, 1, (3, 0), S=1)    # 7x1
        m.conv(c7, 192, h, 1, 1, (0, 3), S=7)   # 1x7
        m.conv(768, 192, h, 1, 1, 0)            # branch_pool
    m.conv(768, 192, 17, 1, 1, 0)   # InceptionD -> 8
    m.conv(192, 320, 17, 3, 2, 0)
    m.conv(768, 192, 17, 1, 1, 0)
    m.conv(192, 192, 17, 1, 1, (0, 3), S=7)
    m.conv(192, 192, 17, 7, 1, (3, 0), S=1)
    m.conv(192, 192, 17, 3, 2, 0)
    h = 8
    for cin in (1280, 2048):         # InceptionE
        m.conv(cin, 320, h, 1, 1, 0)
        m.conv(cin, 384, h, 1, 1, 0)
        m.conv(384, 384, h, 1, 1, (0, 1), S=3)
        m.conv(384, 384, h, 3, 1, (1, 0), S=1)
        m.conv(cin, 448, h, 1, 1, 0)
        m.conv(448, 384, h, 3)
        m.conv(384, 384, h, 1, 1, (0, 1), S=3)
        m.conv(384, 384, h, 3, 1, (1, 0), S=1)
        m.conv(cin, 192, h, 1, 1, 0)
    m.fc(2048, 1000)
    return m.layers()


MODELS = OrderedDict([
    ("alexnet", alexnet), ("vgg11", lambda b=1: vgg(11, b)), ("vgg13", lambda b=1: vgg(13, b)),
    ("vgg16", lambda b=1: vgg(16, b)), ("vgg19", lambda b=1: vgg(19, b)),
    ("resnet18", lambda b=1: resnet(18, b)), ("resnet34", lambda b=1: resnet(34, b)),
    ("resnet50", lambda b=1: resnet(50, b)), ("resnet101", lambda b=1: resnet(101, b)),
    ("resnet152", lambda b=1: resnet(152, b)),
    ("densenet121", lambda b=1: densenet(121, b)), ("densenet169", lambda b=1: densenet(169, b)),
    ("densenet201", lambda b=1: densenet(201, b)),
    ("mobilenetv2", mobilenet_v2), ("mnasnet", mnasnet), ("squeezenet1.1", squeezenet11),
    ("shufflenetv2", shufflenet_v2), ("googlenet", googlenet), ("inceptionv3", inception_v3),
    ("efficientnetb0", efficientnet_b0),
])


def model_layers(name: str, batch: int = 1):
    """The distinct tuning tasks of one of the 20 models (each with its ``count``)."""
    return MODELS[name](batch)
