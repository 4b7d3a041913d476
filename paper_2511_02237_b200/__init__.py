"""B200-native Opportunistic Expert Activation (arXiv 2511.02237) MoE decode layer.

The reference's router / MoE-layer operator API (proj/include/oea/routing.hpp,
moe_layer.hpp) mirrored over the C ABI in include/oea_cuda.h, whose kernels
are hand-written for sm_100a (paper_2511_02237_b200/csrc). There is no CPU
fallback: without the built library or an sm_100 GPU every compute call raises.
"""
from ._capi import (DomainError, InvalidArgument, OeaError, Context, default_context,  # noqa
                    LIB_PATH, EXPORTED)
from .routing import *  # noqa: F401,F403
from .routing import __all__ as _routing_all
from .moe_layer import *  # noqa: F401,F403
from .moe_layer import __all__ as _layer_all

__all__ = ["DomainError", "InvalidArgument", "OeaError", "Context", "default_context",
           "LIB_PATH"] + list(_routing_all) + list(_layer_all)
