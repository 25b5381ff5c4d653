"""B200-native split block Bloom filter (arxiv 2101.01719), drop-in for the
reference core's batched insert/find-by-64-bit-hash path.

The compute path is ``libsbbf_gpu.so`` (hand-written sm_100a CUDA behind the C
ABI in ``include/sbbf_gpu.h``); this package is the Python mirror of the
reference's ``sbbf::SplitBlockFilter`` plus workload generators and the
multi-GPU sharded layer.
"""
from ._lib import SbbfError, launch_count  # noqa: F401
from .filter import (PersistError, SplitBlockFilter, block_index_batch, hash_counter_strings,  # noqa: F401
                     hash_keys, hash_u64_keys, make_mask_batch)

LANE_SEEDS = (0x44974D91, 0x47B6137B, 0xA2B7289D, 0x8824AD5B,
              0x2DF1424B, 0x705495C7, 0x5C6BFB31, 0x9EFC4947)  # filter.hpp:18-21
BLOCK_BYTES = 32  # filter.hpp:14
