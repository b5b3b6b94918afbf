"""Error classes of the reference API (pkg/src/seele/errors.py:5-30) and the
mapping from C-ABI status codes (include/seele_b200.h) onto them."""


class SeeleError(Exception):
    """Root of every error raised by this package."""


class UserInputError(SeeleError):
    """Caller-side problem (CLI exit code 2 in the reference, cli.py:262-276)."""


class SchemaError(UserInputError):
    """Structurally invalid input file."""


class DataError(UserInputError):
    """Well-formed input carrying unusable values."""


class CorruptionError(UserInputError):
    """A compiled scene container disagrees with its manifest."""


class InvalidArgumentError(UserInputError, ValueError):
    """An API call outside its contract."""


class ContractViolationError(SeeleError):
    """An internal precondition broke (pipeline bug)."""


class DeviceError(SeeleError):
    """A CUDA error reported by the native library, or the library is missing."""


# C-ABI status codes (include/seele_b200.h, enum seele_status).
STATUS_OK = 0
STATUS_INVALID_ARGUMENT = 1
STATUS_DATA = 2
STATUS_CONTRACT = 3
STATUS_CUDA = 4
STATUS_CAPACITY = 5

_STATUS_TO_ERROR = {
    STATUS_INVALID_ARGUMENT: InvalidArgumentError,
    STATUS_DATA: DataError,
    STATUS_CONTRACT: ContractViolationError,
    STATUS_CUDA: DeviceError,
}


def raise_for_status(code: int, message: str) -> None:
    if code == STATUS_OK:
        return
    raise _STATUS_TO_ERROR.get(code, DeviceError)(message or f"native status {code}")
