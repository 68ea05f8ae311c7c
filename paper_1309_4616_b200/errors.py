"""Error hierarchy of the drop-in API.

Class names and attributes match what callers of the reference catch
(reference errors.py:1-52): ``ConvergenceError.residual/.degree`` from a
series that ran out of nodes, ``DomainError.index`` from the combustion term,
``MatrixMarketError.line`` from the reader.  ``_lib.check`` maps the C ABI
status codes onto them.
"""


class ExpStencilError(Exception):
    pass


class ConfigError(ExpStencilError):
    pass


class BoundaryKindError(ExpStencilError):
    pass


class GridMismatchError(ExpStencilError):
    pass


class EvaluationError(ExpStencilError):
    pass


class ConvergenceError(ExpStencilError):
    def __init__(self, message, residual=None, degree=None):
        super().__init__(message)
        self.residual, self.degree = residual, degree


class DomainError(ExpStencilError):
    def __init__(self, message, index=None):
        super().__init__(message)
        self.index = index


class MatrixMarketError(ExpStencilError):
    def __init__(self, message, line=None):
        super().__init__(message if line is None else f"line {line}: {message}")
        self.line = line
