"""B200-native blocked implicit-im2col convolution (arXiv 2110.03901 §5).

Drop-in for the hot path of the reference package ``sasim``
(/root/reference/pkg/src/sasim): the same public names for the convolution
path (``direct_conv``, ``gemm``, ``ConvSpec``, ``Tensor``, the lowering
helpers, the block scheduler and the ``_kernels`` plug-in surface), computed
by hand-written sm_100a CUDA (TMA im2col + tcgen05/TMEM) behind the C ABI in
``include/imconv.h``.  No CPU fallback, no backend switch.
"""

from ._kernels import BACKEND as KERNEL_BACKEND
from .core import CapacityError, ConvSpec, Layout, ShapeError, Tensor, direct_conv, gemm, relayout
from .functional import ALL_METHODS, Method, channel_first_implicit, explicit_im2col, functional_ofmap
from .lowering import (ColumnOrdering, TileDescriptor, column_permutation, decompose_tiles, im2col_explicit,
                       lower_filter, lowered_memory_footprint, tile_overlap)
from .workloads import default_operands, random_spec

__version__ = "0.1.0"

__all__ = [
    "ALL_METHODS", "CapacityError", "ColumnOrdering", "ConvSpec", "KERNEL_BACKEND", "Layout", "Method",
    "ShapeError", "Tensor", "TileDescriptor", "channel_first_implicit", "column_permutation", "decompose_tiles",
    "default_operands", "direct_conv", "explicit_im2col", "functional_ofmap", "gemm", "im2col_explicit",
    "lower_filter", "lowered_memory_footprint", "random_spec", "relayout", "tile_overlap",
]
