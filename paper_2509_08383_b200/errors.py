"""Python mirror of the drop-in error hierarchy (include/polyargmax/errors.hpp,
interface-compatible with /root/reference/proj/include/polyargmax/errors.hpp:9-87)."""
from __future__ import annotations

from . import _abi


class Error(RuntimeError):
    """Root error (errors.hpp:9)."""


class DegenerateInputError(Error):
    """Variance below eps_var."""


class InvalidParamsError(Error):
    """CutMaxParams invariant violated."""


class RangeError(Error):
    """Plaintext input outside an approximation's domain."""


class DomainError(Error):
    """u in {0,1} or p, q outside (0,1)."""


class NonFiniteError(Error):
    """Non-finite entry in a logit vector; carries the vector (row) index."""

    def __init__(self, msg: str, vector_index: int):
        super().__init__(f"{msg} (vector {vector_index})")
        self.vector_index = vector_index


class FormatError(Error):
    """Malformed logit file; carries the byte offset of the problem (errors.hpp:65)."""

    def __init__(self, msg: str, byte_offset: int):
        super().__init__(f"{msg} (byte offset {byte_offset})")
        self.byte_offset = byte_offset


class SingularityError(Error):
    """Variance below eps_var on the JVP path (errors.hpp:55)."""


class CudaError(Error):
    """CUDA launch or copy failure inside the library."""


_BY_STATUS = {
    _abi.PAM_ERR_INVALID_PARAMS: InvalidParamsError,
    _abi.PAM_ERR_DEGENERATE_INPUT: DegenerateInputError,
    _abi.PAM_ERR_RANGE: RangeError,
    _abi.PAM_ERR_DOMAIN: DomainError,
    _abi.PAM_ERR_CUDA: CudaError,
    _abi.PAM_ERR_BAD_ARGUMENT: InvalidParamsError,
    _abi.PAM_ERR_UNSUPPORTED: InvalidParamsError,
    _abi.PAM_ERR_SINGULAR: SingularityError,
}


def raise_for_status(status: int, row: int = 0, what: str = "") -> None:
    """Raise the errors.hpp-equivalent exception for a pam_status (no-op for OK)."""
    s = int(status) & 0xFF
    if s == _abi.PAM_OK:
        return
    lib = _abi.load()
    msg = lib.pam_status_string(s).decode()
    if what:
        msg = f"{what}: {msg}"
    if s == _abi.PAM_ERR_NON_FINITE:
        raise NonFiniteError(msg, row)
    if s == _abi.PAM_ERR_FORMAT:
        raise FormatError(msg, row)
    if s == _abi.PAM_ERR_CUDA:
        msg += ": " + lib.pam_last_cuda_error().decode()
    cls = _BY_STATUS.get(s, Error)
    if s in (_abi.PAM_ERR_DEGENERATE_INPUT, _abi.PAM_ERR_RANGE, _abi.PAM_ERR_SINGULAR):
        msg += f" (row {row})"
    raise cls(msg)


class TieWarning(UserWarning):
    """TieWarning: the input's top-2 gap is below 1e-9.  Reported,
    never raised as an error: rows carry the PAM_ROW_FLAG_TIE bit in their status."""
