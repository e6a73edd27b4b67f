"""B200-native (sm_100a) DCNv4 spatial aggregation (arxiv 2401.06197).

The product is libdcnv4.so (C ABI, include/dcnv4.h); this package is its thin binding.
"""
from .binding import (DCNv4Error, DCNv4Function, Params, backward, dcnv4, forward,  # noqa: F401
                    forward_grouped, launch_info, lib, make_params, om_channels, output_size,
                    workspace_bytes)
from . import msda  # noqa: F401  (multi-scale deformable attention, include/msda.h)
from . import module  # noqa: F401  (module path: fused offset/mask linear, include/dcnv4_module.h)

__all__ = ["DCNv4Error", "DCNv4Function", "Params", "backward", "dcnv4", "forward", "forward_grouped",
           "launch_info", "lib", "make_params", "om_channels", "output_size",
           "workspace_bytes", "msda", "module"]
