"""B200-native LoRS masked-LoRA linear (arXiv 2501.08582).

Drop-in for the reference's hot path (`lors` variant of AdaptedLayer,
/root/reference/pkg/src/lors/adapters.py:359-406): PyTorch host code over a
C-ABI library of hand-written sm_100a kernels (include/lors_b200.h).
"""

from .errors import ArgumentError, CheckpointFormatError, DeviceError, GraphError, NumericError, ShapeError
from .prune import SparseWeight, prune_magnitude, prune_rowwise, prune_two_four, two_four_valid, sparsity
from .adapters import (
    COST_MODELS, FAULT_INJECTION, VARIANTS, AdaptedLayer, AdapterPair, CostCounters, VariantGrads,
    counted_saved, lors_backward, lors_forward, make_layer, mask_matrix, merge, merged_weight, predict_cost,
    sqft_gc_backward, sqft_gc_forward, variant_backward, variant_forward,
)
from .module import LoRSFunction, LoRSGroupFunction, LoRSLinear, LoRSParams, lors_group

__version__ = "0.1.0"
