"""Exception taxonomy shared by the host API and the device error flags.

Mirrors the reference's class tree (``pkg/src/mmkit/errors.py:10-48``) so
that ``except mmkit.DomainError`` style handlers keep working after the
switch.  The C-ABI reports problems as integer status codes plus a
device-side error record; :func:`raise_for_status` and
:func:`raise_for_record` translate both into these classes.

Families:
  * ``InputError``   - caller supplied bad shapes / values (CLI exit 2)
  * ``NumericsError`` - an invariant broke during iteration (CLI exit 3)
"""


class MmkitError(Exception):
    """Root of every error raised by this package."""


class InputError(MmkitError):
    """Caller-side problem: shapes, domains or file contents."""


class ShapeError(InputError):
    """Operands have non-conforming shapes."""


class DomainError(InputError):
    """A value lies outside the mathematical domain of the operation."""


class MatrixFormatError(InputError):
    """A serialized matrix could not be parsed."""


class NumericsError(MmkitError):
    """An iteration produced a state that violates a numerical invariant."""


class NonFiniteError(NumericsError):
    """NaN or +-inf appeared in an objective or intermediate."""


class MonotonicityError(NumericsError):
    """The objective moved against the solver's direction beyond slack.

    Same constructor and message layout as the reference
    (``errors.py:38-48``): ``iteration``, ``previous`` and ``current`` are
    kept as attributes for callers that inspect them.
    """

    def __init__(self, iteration, previous, current, direction):
        self.iteration = iteration
        self.previous = previous
        self.current = current
        msg = ("objective moved against the %s direction at iteration %d: "
               "%r -> %r" % (direction, iteration, previous, current))
        super().__init__(msg)


class DeviceError(MmkitError):
    """The CUDA runtime or the native library reported a failure that is
    not a data problem (launch failure, missing extension, OOM)."""


# ---------------------------------------------------------------------------
# C-ABI status codes (include/mmk.h: enum mmk_status) -> exception classes.
MMK_OK = 0
MMK_E_SHAPE = 1
MMK_E_DOMAIN = 2
MMK_E_NUMERICS = 3
MMK_E_NONFINITE = 4
MMK_E_CUDA = 5

_STATUS_CLASS = {
    MMK_E_SHAPE: ShapeError,
    MMK_E_DOMAIN: DomainError,
    MMK_E_NUMERICS: NumericsError,
    MMK_E_NONFINITE: NonFiniteError,
    MMK_E_CUDA: DeviceError,
}


def raise_for_status(status, message):
    """Raise the exception class mapped to a non-zero C-ABI status."""
    if status == MMK_OK:
        return
    cls = _STATUS_CLASS.get(status, DeviceError)
    raise cls(message)
