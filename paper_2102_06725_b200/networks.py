"""Network builders.

``lenet`` and ``mlp`` are the reference's (src/networks.py:13-55).  The
ResNets are the paper's benchmark models written with the
reference's layers: every convolution carries a bias (src/parametric.py:52),
BN parameters are F32, and the residual add / global average pooling use the
``Add2`` / ``GlobalAveragePooling`` extensions.  oracle/nnl_oracle.py builds
the same graphs in the same parameter-creation order, so a registry seed
gives identical initial weights on both sides.
"""

from __future__ import annotations

from . import functions as F
from . import parametric as PF
from .graph import Variable
from .parameters import ParameterScope, parameter_scope

__all__ = ["lenet", "mlp", "resnet18_cifar", "resnet50", "RESNET50_STAGES", "RESNET18_STAGES"]


def _where(params, layer):
    return {"name": layer} if params is None else {"params": params[layer]}


def lenet(x: Variable, n_classes: int = 10, params: ParameterScope | None = None) -> Variable:
    h = PF.convolution(x, 16, (5, 5), **_where(params, "conv1"))
    h = F.max_pooling(h, (2, 2))
    h = F.relu(h, inplace=False)
    h = PF.convolution(h, 16, (5, 5), **_where(params, "conv2"))
    h = F.max_pooling(h, (2, 2))
    h = F.relu(h, inplace=False)
    h = PF.affine(h, 50, **_where(params, "affine3"))
    h = F.relu(h, inplace=False)
    return PF.affine(h, n_classes, **_where(params, "affine4"))


def mlp(x: Variable, n_classes: int, hidden: tuple[int, ...] = (32,),
        params: ParameterScope | None = None) -> Variable:
    h = x
    for i, width in enumerate(hidden):
        h = PF.affine(h, width, **_where(params, f"fc{i + 1}"))
        h = F.relu(h, inplace=False)
    return PF.affine(h, n_classes, **_where(params, "out"))


def _conv_bn(x, maps, k, stride, pad, name, relu, train=True):
    h = PF.convolution(x, maps, (k, k), stride=(stride, stride), pad=(pad, pad),
                       name=f"{name}")
    h = PF.batch_normalization(h, batch_stat=train, name=f"{name}_bn")
    return F.relu(h) if relu else h


def _bottleneck(x: Variable, width: int, stride: int, project: bool,
                train: bool = True) -> Variable:
    """ResNet v1.5 bottleneck: the stride sits on the 3x3 convolution."""
    out = width * 4
    h = _conv_bn(x, width, 1, 1, 0, "conv1", True, train)
    h = _conv_bn(h, width, 3, stride, 1, "conv2", True, train)
    h = _conv_bn(h, out, 1, 1, 0, "conv3", False, train)
    s = _conv_bn(x, out, 1, stride, 0, "shortcut", False, train) if project else x
    return F.relu(F.add2(h, s))


def _basic(x: Variable, width: int, stride: int, project: bool, train: bool = True) -> Variable:
    h = _conv_bn(x, width, 3, stride, 1, "conv1", True, train)
    h = _conv_bn(h, width, 3, 1, 1, "conv2", False, train)
    s = _conv_bn(x, width, 1, stride, 0, "shortcut", False, train) if project else x
    return F.relu(F.add2(h, s))


RESNET50_STAGES = ((64, 3, 1), (128, 4, 2), (256, 6, 2), (512, 3, 2))
RESNET18_STAGES = ((64, 2, 1), (128, 2, 2), (256, 2, 2), (512, 2, 2))


def resnet50(x: Variable, n_classes: int = 1000, train: bool = True) -> Variable:
    """ResNet-50 v1.5 for (B,3,224,224) inputs; ``train=False`` builds the eval
    graph (BN on running statistics) over the same registry parameters."""
    h = _conv_bn(x, 64, 7, 2, 3, "stem", True, train)
    h = F.max_pooling(h, (3, 3), stride=(2, 2), pad=(1, 1))
    in_c = 64
    for si, (width, blocks, stride) in enumerate(RESNET50_STAGES):
        for bi in range(blocks):
            with parameter_scope(f"stage{si + 1}_block{bi + 1}"):
                s = stride if bi == 0 else 1
                h = _bottleneck(h, width, s, project=(bi == 0 and (s != 1 or in_c != width * 4)),
                                train=train)
            in_c = width * 4
    h = F.global_average_pooling(h)
    return PF.affine(h, n_classes, name="fc")


def resnet18_cifar(x: Variable, n_classes: int = 10, train: bool = True) -> Variable:
    """ResNet-18 for (B,3,32,32): 3x3 stem, no max-pool, GAP over 4x4."""
    h = _conv_bn(x, 64, 3, 1, 1, "stem", True, train)
    in_c = 64
    for si, (width, blocks, stride) in enumerate(RESNET18_STAGES):
        for bi in range(blocks):
            with parameter_scope(f"stage{si + 1}_block{bi + 1}"):
                s = stride if bi == 0 else 1
                h = _basic(h, width, s, project=(bi == 0 and (s != 1 or in_c != width)),
                           train=train)
            in_c = width
    h = F.global_average_pooling(h)
    return PF.affine(h, n_classes, name="fc")
