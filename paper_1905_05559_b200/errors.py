"""Error classes mirroring /root/reference/proj/include/curv/errors.hpp."""


class CurvError(Exception):
    """Base class for errors raised by the curvkit B200 library."""


class ShapeError(CurvError, ValueError):
    """curv::ShapeError (errors.hpp:10-13): dimension mismatch."""


class ContractError(CurvError, ValueError):
    """curv::ContractError (errors.hpp:17-20): violated value precondition."""


class CurvRuntimeError(CurvError, RuntimeError):
    """std::runtime_error raised by the reference (e.g. curvature.cpp:81-84)."""


class ConvergenceError(CurvError, RuntimeError):
    """curv::ConvergenceError (errors.hpp:24-30)."""

    def __init__(self, msg, best_residuals=()):
        super().__init__(msg)
        self.best_residuals = list(best_residuals)


class CudaError(CurvError, RuntimeError):
    """A CUDA runtime failure inside the library."""


_BY_CODE = {1: ShapeError, 2: ContractError, 3: CurvRuntimeError, 4: ConvergenceError, 5: CudaError,
            6: MemoryError}


def raise_for(code: int, message: str):
    cls = _BY_CODE.get(code, CurvRuntimeError)
    raise cls(message)
