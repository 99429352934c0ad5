"""Exception types of the B200 hot path.

Names and base classes mirror the reference's error module
(`pkg/src/moesim/errors.py:4-29`) so callers that catch the reference's
exceptions keep working.  The C-ABI returns an integer status; `raise_status`
maps it back onto these classes (see `include/vismmoe.h`, `VMM_E*`).
"""
from __future__ import annotations


class ValidationError(ValueError):
    """An input value violates a documented invariant (errors.py:4)."""


class ParseError(ValueError):
    """A serialized artifact could not be parsed (errors.py:8)."""


class TraceError(ValueError):
    """A trace lacks data an operation needs (errors.py:12)."""


class ContractError(RuntimeError):
    """An internal precondition was violated by the caller (errors.py:16)."""


class TrainingError(RuntimeError):
    """Training diverged (errors.py:20)."""


class PlanningError(ValueError):
    """Memory planning found no feasible configuration (errors.py:24)."""


class SimulationError(RuntimeError):
    """The run hit an unrecoverable state, e.g. cache too small (errors.py:28)."""


class DeviceError(RuntimeError):
    """A CUDA call failed or the sm_100a extension is unavailable."""


# status codes shared with include/vismmoe.h
STATUS_OK = 0
_BY_CODE = {
    1: ValidationError,
    2: ContractError,
    3: SimulationError,
    4: TraceError,
    5: PlanningError,
    6: DeviceError,
}


def raise_status(code: int, message: str) -> None:
    if code == STATUS_OK:
        return
    raise _BY_CODE.get(code, DeviceError)(message)
