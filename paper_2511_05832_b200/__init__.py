"""paper_2511_05832_b200 -- B200-native hot path of Hilbert-guided local attention.

arXiv 2511.05832: image tokens are reordered along a Hilbert curve, windows /
slides / neighborhoods are formed on the 1D sequence, and attention runs as a
block-sparse forward/backward that skips empty tiles (P:L7).

Layers:
  csrc/            hand-written CUDA for sm_100a (tcgen05 / TMEM / TMA) behind the
                   C ABI of include/hla.h, built into libhla.so
  api.py           ctypes marshalling with the C ABI's names
  attention.py     HilbertLocalAttention: cached path + mask, preallocated buffers,
                   one call per forward / backward step (the public API)
"""

from ._lib import HlaError  # noqa: F401
from .api import (KINDS, BlockMask, hla_attn_bwd, hla_attn_bwd_workspace, hla_attn_fwd,  # noqa: F401
                  hla_build_block_mask, hla_debug_umma, hla_hilbert_index, hla_hilbert_perm,
                  hla_hilbert_tiled_index, pattern_desc,
                  version)
from .attention import HilbertLocalAttention  # noqa: F401
