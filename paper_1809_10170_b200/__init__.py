"""B200-native (sm_100a) direct convolution in the blocked layout of
arXiv 1809.10170, behind the reference ``dconv`` operator API.

The compute lives in ``libdconv_b200.so`` (hand-written CUDA, C-ABI in
``include/dconv_cuda.h``); this package is the host-side mirror of the
reference interface (``dconv``), the network layer catalog / chain executor
(``nets``) and the multi-GPU sharding logic (``shard``).
"""
from . import _abi  # noqa: F401
from .dconv import (BlockedFeatureMap, BlockedKernel, BlockingParams,  # noqa: F401
                    ConvShape, add_blocked, conv_direct, conv_flops,
                    layer_chain, layout_transform_count, maxpool2x2_blocked,
                    pack_feature_map, pack_kernel, relu_blocked,
                    unpack_feature_map, unpack_kernel)
