"""B200-native DeepSpeed-Ulysses sequence-parallel attention (arXiv 2309.14509).

Public API (drop-in for the reference's DistributedAttention path):

    DistributedAttention(local_attn, sequence_process_group, scatter_idx=2, gather_idx=0)
    seq_all_to_all(input, scatter_idx, gather_idx, group)
    SequenceGroup.from_process_group(pg) / SequenceGroup.local_group(P)
    FlashAttention(mask="causal"|"none"|"blocked"), get_kernel("causal"|"dense"|"blocked")
    UlyssesAttention(d, heads, group) / UlyssesBlock(...)   (layer with projections / block)

All compute runs in libulysses_b200.so (sm_100a); see include/ulysses_b200.h.
"""

from .attention import (  # noqa: F401
    KERNELS,
    DistributedAttention,
    FlashAttention,
    get_kernel,
    seq_all_to_all,
)
from .comm import CommLedger, CommRecord, SequenceGroup, a2a_out_shape, check_ledger  # noqa: F401
from .layer import HybridAttention, RingAttention, UlyssesAttention, UlyssesBlock, make_weights, ring_attention_core  # noqa: F401
from .errors import (  # noqa: F401
    DegenerateRowError,
    DivisibilityError,
    ForwardStateError,
    GroupDesyncError,
    KernelError,
    NativeError,
    ShapeError,
    ShardError,
)

__version__ = "0.1.0"
