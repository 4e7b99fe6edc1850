"""Exception types of the drop-in surface.

Same names and meaning as the reference ``sumfact`` package so that callers'
``except`` clauses keep working:

* ``InvalidArity``              quadrature.py:16  (rule with too few points)
* ``InvalidDegree``, ``DimensionMismatch``, ``ShapeMismatch``,
  ``Unsupported``               elements.py:29-45
* ``ArityMismatch``, ``UnsupportedCell``, ``ExtentMismatch``
                                forms.py:30-39
* ``UnboundVariable``           interpreter.py:23 (missing input array)
* ``UsageError``                cli.py:54 (bad compile request)

``NativeError`` is new: it carries a non-zero status of the C-ABI
(``include/sfk.h``) together with ``sfk_last_error()``.
"""


class InvalidArity(Exception):
    pass


class InvalidDegree(Exception):
    pass


class DimensionMismatch(Exception):
    pass


class ShapeMismatch(Exception):
    pass


class ValueShapeMismatch(Exception):
    pass


class Unsupported(Exception):
    pass


class ArityMismatch(Exception):
    pass


class UnsupportedCell(Exception):
    pass


class ExtentMismatch(Exception):
    pass


class UnboundVariable(Exception):
    pass


class UsageError(Exception):
    pass


class NativeError(RuntimeError):
    """A C-ABI call returned a non-zero status."""

    def __init__(self, status, message):
        super().__init__("sfk status %d: %s" % (status, message))
        self.status = status
