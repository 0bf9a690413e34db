"""Exception taxonomy of the reference (proj/include/skewdx/error.hpp:12-49).

``Error`` > ``InvalidArgument`` / ``DomainViolation(row, value, domain)`` /
``IoError`` / ``FormatError``; messages follow error.hpp:22-24.
"""


class Error(RuntimeError):
    """skewdx::Error"""


class InvalidArgument(Error):
    """A parameter or configuration violates a documented precondition."""


class DomainViolation(Error):
    """A column value falls outside the dimension domain 1..D (error.hpp:20-33)."""

    def __init__(self, row: int, value: int, domain: int):
        super().__init__(f"domain violation at row {row}: value {value} outside 1..{domain}")
        self._row, self._value, self.domain = int(row), int(value), int(domain)

    def row(self) -> int:
        return self._row

    def value(self) -> int:
        return self._value


class IoError(Error):
    pass


class FormatError(Error):
    """Bad magic, unsupported version, or a header that disagrees with the payload."""


class NativeUnavailable(Error):
    """libskx.so or a B200 is not available: there is no CPU fallback."""
