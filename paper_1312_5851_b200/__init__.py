"""paper_1312_5851_b200 -- B200-native FFT convolution layer (arXiv 1312.5851).

The hot path (fprop / bprop / accGrad of the FFT convolution layer) runs as
hand-written sm_100a CUDA kernels in ``lib/libfftconv_b200.so`` behind the
reference fftconv::ConvWorkspace interface.  See DESIGN.md.
"""
from .errors import (CapacityError, ConfigError, CudaError, FftconvError, NcclError, PlanError,
                     ShapeError, SizeError)
from .layer_config import LayerConfig, is_pow2, next_pow2
from .workspace import (ConvWorkspace, OpCounters, forward_fft, grad_input_fft, grad_weight_fft,
                        workspace_for)

__all__ = [
    "CapacityError", "ConfigError", "CudaError", "FftconvError", "NcclError", "PlanError",
    "ShapeError", "SizeError", "LayerConfig", "is_pow2", "next_pow2", "ConvWorkspace",
    "OpCounters", "forward_fft", "grad_input_fft", "grad_weight_fft", "workspace_for",
]
