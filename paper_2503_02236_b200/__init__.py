"""B200-native fused vector-quantization kernels (VQ-LLM, arXiv 2503.02236).

Drop-in for the hot path of the reference package ``vqforge``: the quantized
tensor containers and ``dequantize`` (codec), the planner (``plan_kernel``) and
the fused-kernel executor (``B200Machine.run_fused_kernel``, same contract as
``SimMachine.run_fused_kernel``), backed by hand-written sm_100a CUDA kernels in
``libvqb.so`` behind the C ABI of ``include/vqb.h``. There is no CPU fallback.
"""

from .codec import (Codebook, QuantizedTensor, Sharing, VQConfig, compression_ratio, dequantize,
                    region_layout)
from .errors import (CapacityError, CodeRangeError, ConfigError, ForgeError, KernelError,
                     MappingError, ShapeError)

__version__ = "0.1.0"

__all__ = [
    "Codebook", "QuantizedTensor", "Sharing", "VQConfig", "compression_ratio", "dequantize",
    "region_layout", "ForgeError", "ShapeError", "ConfigError", "CodeRangeError", "CapacityError",
    "MappingError", "KernelError", "__version__",
]
