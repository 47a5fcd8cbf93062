"""B200-native (sm_100a) drop-in for the lossy-checkpoint compressor of
arXiv 1805.07384 (reference package: lossyckpt).

Public names mirror lossyckpt/__init__.py:3-23 for the compressor and the
checkpoint/restart layer that calls it.
"""

from .compressor import (  # noqa: F401
    CompressedBlock,
    CompressorConfig,
    DistortionStats,
    QuantizerModel,
    bound_from_target_psnr,
    compress,
    decompress,
    error_identity_check,
    estimate_mse_general,
    estimate_psnr_from_bound,
    measured_psnr,
    predict_lorenzo1,
    psnr_from_bin_width,
)
from .errors import (  # noqa: F401
    BreakdownError,
    CheckpointFailedError,
    DimensionMismatchError,
    IntegrityError,
    ParameterError,
    SingularPreconditionerError,
    UndefinedPsnrError,
    UnrecoverableImageError,
)

from . import checkpoint  # noqa: F401
from .checkpoint import (  # noqa: F401
    AsyncCheckpointer,
    CheckpointImage,
    CkptCost,
    RecCost,
    StorageTarget,
    checkpoint_lossy,
    checkpoint_traditional,
    decode_payload,
    recover,
)

__version__ = "0.1.0"
