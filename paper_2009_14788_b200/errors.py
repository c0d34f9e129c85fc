"""Exception taxonomy of the reference (``proj/core/include/radonkit/errors.hpp:9-40``).

ValidationError -> CLI exit code 1, NumericalError family -> exit code 2
(``tools/cli.cpp:718-730``).  ``CudaError`` has no reference equivalent.
"""


class ValidationError(ValueError):
    """Invalid shapes, parameters or geometry (errors.hpp:9-13)."""


class NumericalError(RuntimeError):
    """Numerical failure at runtime (errors.hpp:16-20)."""


class DivergenceError(NumericalError):
    """A solver iterate became non-finite (errors.hpp:22-27)."""

    def __init__(self, what: str, iteration: int | None = None):
        super().__init__(what)
        self.iteration = iteration


class NotPositiveDefiniteError(NumericalError):
    """CG met non-positive curvature p'Ap (errors.hpp:29-34)."""

    def __init__(self, what: str, iteration: int | None = None):
        super().__init__(what)
        self.iteration = iteration


class HalfOverflowError(NumericalError):
    """Checked narrowing to half overflowed (errors.hpp:36-40)."""

    def __init__(self, what: str, index: int | None = None):
        super().__init__(what)
        self.index = index


class CudaError(RuntimeError):
    """CUDA runtime failure inside the library (no reference equivalent)."""
