"""BASELINE.json configurations restated as layer lists.

Each layer is (name, batch, ConvGeometry).  Synthetic inputs for a layer come
from ``tensors.synthetic_layer(geom, batch, seed)`` with
``seed = 1000 * config_idx + layer_idx`` (config_idx is 1-based as in
BASELINE.md).  No dataset items are involved: BASELINE names only shapes.
"""

from .geometry import ConvGeometry

__all__ = ["CONFIGS", "NETWORKS", "network_geometries", "layer_seed", "config_layers",
           "all_layers"]


def _c3(c_i, c_o, hw, k=3, s=1, p=1):
    return ConvGeometry(c_i, c_o, hw, hw, k, k, stride_h=s, stride_w=s, pad_h=p, pad_w=p)


_RESNET_SWEEP = [(64, 56), (128, 28), (256, 14), (512, 7)]
_VGG16 = [(3, 64, 224), (64, 64, 224), (64, 128, 112), (128, 128, 112),
          (128, 256, 56), (256, 256, 56), (256, 256, 56), (256, 512, 28),
          (512, 512, 28), (512, 512, 28), (512, 512, 14), (512, 512, 14),
          (512, 512, 14)]

CONFIGS = {
    1: {
        "title": "single layer 64->64 @56 3x3 s1 p1, N=1",
        "layers": [("conv64@56_n1", 1, _c3(64, 64, 56))],
    },
    2: {
        "title": "ResNet-style 3x3 s1 p1 sweep, N in {1, 32}",
        "layers": [(f"conv{c}@{hw}_n{n}", n, _c3(c, c, hw))
                   for n in (1, 32) for c, hw in _RESNET_SWEEP],
    },
    3: {
        "title": "large-kernel / strided layers, N=8",
        "layers": [
            ("conv7x7s2p3_3to64@224_n8", 8, _c3(3, 64, 224, k=7, s=2, p=3)),
            ("conv11x11s4_3to96@227_n8", 8, _c3(3, 96, 227, k=11, s=4, p=0)),
            ("conv5x5p2_96to256@27_n8", 8, _c3(96, 256, 27, k=5, s=1, p=2)),
            ("conv1x1_256to64@56_n8", 8, _c3(256, 64, 56, k=1, s=1, p=0)),
        ],
    },
    4: {
        "title": "VGG-16 conv layers, N=64",
        "layers": [(f"vgg{i + 1:02d}_{ci}to{co}@{hw}_n64", 64, _c3(ci, co, hw))
                   for i, (ci, co, hw) in enumerate(_VGG16)],
    },
    5: {
        "title": "multi-GPU scaling: N=256 batch-sharded, 512@7 N=8 c_o-sharded",
        "layers": [
            ("conv1x1_64to256@56_n256", 256, _c3(64, 256, 56, k=1, s=1, p=0)),
            ("conv128@28_n256", 256, _c3(128, 128, 28)),
            ("conv256@14_n256", 256, _c3(256, 256, 14)),
            ("conv512@7_n8_coshard", 8, _c3(512, 512, 7)),
        ],
    },
}


def layer_seed(config_idx, layer_idx):
    return 1000 * config_idx + layer_idx


def config_layers(config_idx):
    return CONFIGS[config_idx]["layers"]


def all_layers():
    for ci, cfg in CONFIGS.items():
        for li, (name, n, g) in enumerate(cfg["layers"]):
            yield ci, li, name, n, g


# The reference's three network presets (``layers.py:28``, ``builtin_network``
# over ``presets/{alexnet,vgg16,yolov3}.cfg``) as layer tables: (name, c_i, c_o,
# h, w, k_h, k_w, s_h, s_w, p_h, p_w).  Spatial sizes account for the
# interleaved pooling layers; AlexNet is the single-tower (ungrouped) variant
# at 224x224, YOLOv3 the compact ("tiny") detector at 416x416 whose conv12
# consumes the 256 + 128 channel route concatenation.
NETWORKS = {
    "alexnet": [
        ("conv1", 3, 64, 224, 224, 11, 11, 4, 4, 2, 2),
        ("conv2", 64, 192, 27, 27, 5, 5, 1, 1, 2, 2),
        ("conv3", 192, 384, 13, 13, 3, 3, 1, 1, 1, 1),
        ("conv4", 384, 256, 13, 13, 3, 3, 1, 1, 1, 1),
        ("conv5", 256, 256, 13, 13, 3, 3, 1, 1, 1, 1),
    ],
    "vgg16": [(nm, ci, co, hw, hw, 3, 3, 1, 1, 1, 1) for nm, (ci, co, hw) in zip(
        ["conv1_1", "conv1_2", "conv2_1", "conv2_2", "conv3_1", "conv3_2", "conv3_3",
         "conv4_1", "conv4_2", "conv4_3", "conv5_1", "conv5_2", "conv5_3"], _VGG16)],
    "yolov3": [
        ("conv1", 3, 16, 416, 416, 3, 3, 1, 1, 1, 1),
        ("conv2", 16, 32, 208, 208, 3, 3, 1, 1, 1, 1),
        ("conv3", 32, 64, 104, 104, 3, 3, 1, 1, 1, 1),
        ("conv4", 64, 128, 52, 52, 3, 3, 1, 1, 1, 1),
        ("conv5", 128, 256, 26, 26, 3, 3, 1, 1, 1, 1),
        ("conv6", 256, 512, 13, 13, 3, 3, 1, 1, 1, 1),
        ("conv7", 512, 1024, 13, 13, 3, 3, 1, 1, 1, 1),
        ("conv8", 1024, 256, 13, 13, 1, 1, 1, 1, 0, 0),
        ("conv9", 256, 512, 13, 13, 3, 3, 1, 1, 1, 1),
        ("conv10", 512, 255, 13, 13, 1, 1, 1, 1, 0, 0),
        ("conv11", 256, 128, 13, 13, 1, 1, 1, 1, 0, 0),
        ("conv12", 384, 256, 26, 26, 3, 3, 1, 1, 1, 1),
        ("conv13", 256, 255, 26, 26, 1, 1, 1, 1, 0, 0),
    ],
}


def network_geometries(name):
    """[(layer name, ConvGeometry)] of a preset network."""
    return [(row[0], ConvGeometry(*row[1:])) for row in NETWORKS[name]]
