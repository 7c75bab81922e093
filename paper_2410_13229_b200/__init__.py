"""B200-native Quamba W8A8 Mamba-block path (arXiv 2410.13229), drop-in for the
reference package `ssmq`'s quantized operators.

Compute runs in libqmb.so (hand-written sm_100a CUDA behind a C ABI,
include/qmb.h); torch provides device memory and streams only.  There is no
CPU fallback: without the built library or a GPU, the operators raise.
"""
from .quant import (  # noqa: F401
    DEFAULT_PERCENTILE, SCALE_FLOOR, QTensor, QuantScheme, SchemeKind, compute_scale_absmax,
    compute_scale_percentile, dequantize, nearest_rank, qmax, qmin, quantize,
)
from .hadamard import HadamardPlan, apply_hadamard, dense_matrix, hadamard_quantize, plan_for_dim  # noqa: F401
from .ssm import BlockConfig, SSMParams, init_block_params  # noqa: F401
from .qblock import (  # noqa: F401
    ACT_SITES, MODE_TAGS, Mode, QuantizedBlock, ScaleEntry, block_forward_q, device_block, fused_qconv,
    fused_rmsnorm_quant, qlinear, quantize_block, quantize_weight, quantized_selective_scan,
)
from .model import DeviceModel, ModelConfig, QuantizedLayer, QuantizedModel, device_model, forward_q  # noqa: F401

__version__ = "0.1.0"
