"""B200-native (sm_100a) routed FFN of SPT (arXiv 2312.10365).

The compute path is libspt_ffn.so (C ABI: include/spt_ffn.h); this package is
its thin Python binding plus the data-parallel helper.  Importing the package
does not load the library; the first ABI call does, and fails loudly if the
library has not been built.
"""
from ._lib import (SPT_ACT_GELU, SPT_ACT_RELU, SPT_ACT_SWIGLU, SPT_BF16, SPT_BWD_ACCUMULATE_DW,  # noqa: F401
                   SPT_F32, SPT_GATE_NONE, SPT_GATE_SIGMOID, SPT_ROUTE_LOGITS_IN, SPT_TILE_M, SptError)
from .ffn import (RouteBuffers, RoutedFFN, RoutedLoRAFFN, launch_count, make_desc,  # noqa: F401
                  profile_enable, profile_read, spt_ffn_backward, spt_ffn_balance_loss,
                  spt_ffn_forward, spt_ffn_lora_backward, spt_ffn_lora_forward, spt_ffn_lora_sizes,
                  spt_ffn_route, spt_ffn_sizes, spt_mha_topl, spt_status_string)
