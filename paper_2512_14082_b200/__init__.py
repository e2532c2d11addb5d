"""B200-native (sm_100a) UniSparse dynamic sparse attention hot path.

compress -> fused proxy + Top-P/top-k select -> tcgen05 block-sparse attention,
behind the C ABI in include/us_api.h; this package is the Python mirror of the
reference operator API (see api.py). The product path is the CUDA library
paper_2512_14082_b200/_build/libunisparse_b200.so — there is no CPU fallback.
"""
from .api import (  # noqa: F401
    CompressionConfig, Engine, Selection, SparsityReport, UniSparseResult, UnsupportedError,
    InvalidMaskError, CudaError, block_sparse_attention, build_block_mask, compress,
    dense_attention, select_blocks, selection_flops, unisparse_attn, make_params, validate,
    POOL_MEAN, POST_SOFTMAX_BLOCK_CAUSAL, PRE_SOFTMAX_COMPRESSED_CAUSAL, SELECT_TOP_P, SELECT_TOP_K,
    exact_block_mass, output_fidelity, block_recall, mean_row_spearman, planted_recall,
)

__version__ = "0.1.0"
