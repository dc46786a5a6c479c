"""paper_2008_02002_b200 -- B200-native drop-in for the hot path of the `xfbq` reference
(arXiv 2008.02002): quantize -> bit-plane pack -> XOR/POPC scan with fused top-K -> merge.

Same names as the reference package facade (/root/reference/pkg/src/xfbq/__init__.py:95-160)
for everything on that path, plus the batched `search`.  All compute runs in hand-written
sm_100a kernels behind the C ABI in include/xfbq_b200.h; there is no CPU fallback.
"""
from .bitplane import (PackedMatrix, PackedVector, pack_matrix, quantize_matrix, quantize_queries,
                       quantize_vector, unpack_matrix, words_needed)
from .distance import (batch_distances, decode_inner_product, decode_inner_product_values,
                       distance_upper_bound, packed_distance)
from .errors import (BadMagicError, DimensionMismatchError, IndexFormatError, InvalidInputError, NativeLibraryError,
                     TruncatedIndexError, UnsupportedVersionError, XfbqError)
from .index import Index, QuantParams, build_index, estimate_scale, load_index, save_index
from .sharded import ShardedIndex, shard_bounds
from .search import (DistanceHistogram, SearchRequest, SearchResult, gather_candidates, histogram_kth_distance, k_select,
                     refine, search, search_device, suggest_extra_distance)

__version__ = "0.1.0"
__all__ = [
    "BadMagicError", "IndexFormatError", "TruncatedIndexError", "UnsupportedVersionError", "load_index", "save_index",
    "DimensionMismatchError", "Index", "InvalidInputError", "NativeLibraryError", "PackedMatrix",
    "PackedVector", "QuantParams", "SearchRequest", "SearchResult", "XfbqError", "batch_distances",
    "build_index", "decode_inner_product", "decode_inner_product_values", "distance_upper_bound",
    "estimate_scale", "k_select", "pack_matrix", "quantize_matrix", "quantize_queries",
    "quantize_vector", "search", "search_device", "ShardedIndex", "shard_bounds", "unpack_matrix", "words_needed",
    "DistanceHistogram", "gather_candidates", "histogram_kth_distance", "packed_distance", "refine", "suggest_extra_distance",
]
