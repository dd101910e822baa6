"""Exception tree of the reference (`lsrm/errors.py:8-59`), same names, same
CLI exit codes, so callers that catch `lsrm` errors keep working."""


class LsrmError(Exception):
    exit_code = 4


class ConfigurationError(LsrmError):
    exit_code = 3


class VerificationError(LsrmError):
    exit_code = 2


class EmptyAttentionRowError(LsrmError):
    pass


class EmptyContextError(LsrmError):
    pass


class OutOfDomainError(LsrmError):
    pass


class BehindCameraError(LsrmError):
    pass


class ProtocolError(LsrmError):
    pass


class GoldenFormatError(LsrmError):
    def __init__(self, message: str, byte_offset=None):
        if byte_offset is not None:
            message = f"{message} (byte offset {byte_offset})"
        super().__init__(message)
        self.byte_offset = byte_offset


def require(condition: bool, message: str) -> None:
    if not condition:
        raise ConfigurationError(message)


# C-ABI status code -> exception class (include/lsrm_b200.h, enum lsrm_status)
STATUS_CLASSES = {
    1: ConfigurationError,
    2: EmptyContextError,
    3: EmptyAttentionRowError,
    4: ProtocolError,
    5: LsrmError,
    6: OutOfDomainError,
}
