"""Exception hierarchy of the package.

Mirrors the reference error classes (`pkg/src/contactamg/errors.py:4-25`) so
that code written against the reference catches the same types.  Native
status codes returned by `libcamg.so` are mapped onto these classes in
`_native.py`.
"""


class ContactAmgError(Exception):
    """Root of every error raised here."""


class DimensionError(ContactAmgError):
    """Inconsistent operand shapes."""


class SingularMatrixError(ContactAmgError):
    """Zero pivot, zero diagonal or an all-zero lumped row."""


class AssemblyError(ContactAmgError):
    """Invalid mesh / element data in the problem generator."""


class ConfigError(ContactAmgError):
    """Invalid configuration value."""


class SetupError(ContactAmgError):
    """The hierarchy cannot be built (empty aggregation, lost interface, ...)."""


class NativeError(ContactAmgError):
    """A CUDA / native-library failure that has no reference counterpart."""
