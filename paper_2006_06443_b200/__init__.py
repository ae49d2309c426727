"""B200-native (sm_100a) compressed convolution W ~ L + S (arXiv 2006.06443).

The product is the C-ABI library liblrs_conv.so (include/lrs_conv.h); this
package is its thin Python binding.  It never imports `oracle/`.
"""
from .lrs_conv import (LrsConv, LrsConvBackward, LrsDecomp, LrsTucker2Decomp, LrsError, lrs_conv_create, lrs_conv_destroy,  # noqa: F401
                       lrs_conv_forward, lrs_conv_forward_host, lrs_conv_last_error,
                       load_library, make_desc, sparse_from_slices, EXPORTED, LIB_PATH,
                       LRS_CORE_TUCKER2, LRS_CORE_CP)

__all__ = ["LrsConv", "LrsConvBackward", "LrsDecomp", "LrsTucker2Decomp", "LrsError", "lrs_conv_create", "lrs_conv_forward", "lrs_conv_forward_host",
           "lrs_conv_destroy", "lrs_conv_last_error", "load_library", "make_desc", "sparse_from_slices",
           "LRS_CORE_TUCKER2", "LRS_CORE_CP"]
