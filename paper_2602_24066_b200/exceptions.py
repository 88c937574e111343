"""Error types of the public API.

Same class names and bases as the reference hierarchy
(/root/reference/pkg/src/sigkit/errors.py:4-37) so that ``except`` clauses
written against ``sigkit`` keep working.  The C ABI status codes
(include/sigkit_b200.h) map onto these in ``_lib.check``.
"""


class SigkitError(Exception):
    """Root of every error raised by this package."""


def _kind(name: str, base: type, doc: str) -> type:
    return type(name, (SigkitError, base), {"__doc__": doc, "__module__": __name__})


InvalidLetterError = _kind("InvalidLetterError", ValueError, "Letter outside the alphabet 1..d.")
CapacityError = _kind("CapacityError", OverflowError, "Word code beyond the unsigned 64-bit range.")
CorruptWordError = _kind("CorruptWordError", ValueError, "Integer code inconsistent with the word length.")
WordRangeError = _kind("WordRangeError", ValueError, "Prefix/suffix length outside [0, |w|].")
DomainError = _kind("DomainError", ValueError, "Parameter outside its domain.")
ShapeError = _kind("ShapeError", ValueError, "Array shape inconsistent with the batch layout.")
WindowError = _kind("WindowError", ValueError, "Window indices violate 0 <= l < r <= M.")
UnsupportedWordSetError = _kind(
    "UnsupportedWordSetError", ValueError, "Operation needs a fully truncated word set."
)

__all__ = [
    "SigkitError",
    "InvalidLetterError",
    "CapacityError",
    "CorruptWordError",
    "WordRangeError",
    "DomainError",
    "ShapeError",
    "WindowError",
    "UnsupportedWordSetError",
]
