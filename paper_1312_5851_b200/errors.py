"""Exception taxonomy of the reference (/root/reference/proj/include/fftconv/errors.hpp:7-41).

The C ABI returns the matching status code (include/fftconv_b200.h); the
host wrappers re-raise the class below so callers can catch exactly what
they caught with the reference.
"""


class FftconvError(RuntimeError):
    """fftconv::error (errors.hpp:7-10)."""


class SizeError(FftconvError):
    """fftconv::size_error (errors.hpp:14-17)."""


class ShapeError(FftconvError):
    """fftconv::shape_error (errors.hpp:20-23)."""


class PlanError(FftconvError):
    """fftconv::plan_error (errors.hpp:26-29)."""


class CapacityError(FftconvError):
    """fftconv::capacity_error (errors.hpp:32-35)."""


class ConfigError(FftconvError):
    """fftconv::config_error (errors.hpp:38-41)."""


class CudaError(FftconvError):
    """CUDA runtime/driver failure inside the B200 library (no reference analogue)."""


class NcclError(FftconvError):
    """Collective failure in the sharded path (no reference analogue)."""


STATUS_TO_ERROR = {
    1: SizeError,
    2: ShapeError,
    3: ConfigError,
    4: CapacityError,
    5: PlanError,
    6: CudaError,
    7: NcclError,
    8: FftconvError,
}


def raise_for_status(code: int, message: str) -> None:
    if code == 0:
        return
    raise STATUS_TO_ERROR.get(code, FftconvError)(message)
