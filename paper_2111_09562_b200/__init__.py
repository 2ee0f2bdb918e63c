"""B200-native COMET activation-compression hot path (arXiv 2111.09562).

Drop-in for the reference's codec / hook / controller API
(/root/reference/pkg/src/actcomp/__init__.py:5-79, hot-path subset): every
codec stage runs as hand-written sm_100a CUDA in libactc.so (include/actc.h).
"""
from .codec import (
    CodecParams,
    CompressedActivation,
    check_decode_status,
    CompressionReport,
    compress,
    compress_batch,
    compress_begin,
    compress_end,
    compress_device,
    decompress,
    decompress_batch,
    decompress_device,
    lorenzo_decode,
    lorenzo_encode,
    prequantize,
    read_compressed,
    write_compressed,
)
from .controller import (
    AdaptiveController,
    CompressionPlan,
    ControllerConfig,
    LayerTrainingStats,
    assess_gradient_tolerance,
    choose_batch_size,
    collect_layer_stats,
    estimate_eb,
    plan_compression,
    predict_sigma,
    update_interval,
)
from .errors import (
    ActcompError,
    DataError,
    DimensionError,
    FormatError,
    LifecycleError,
    MemoryInfeasibleError,
    ParameterError,
    SchemaError,
)
from .errorprop import inject_uniform_error
from .tensor import Tensor, TensorStats, compute_stats, make_tensor

__version__ = "0.1.0"
