"""Exception taxonomy of the Harmony B200 runtime.

Mirrors the reference's error tree (`pkg/src/wrapsched/errors.py:4-73`) so a
caller that catches ``ValidationError`` / ``DeadlockError`` around
``generate_task_graph`` / ``simulate`` keeps working when it switches to this
package.  The native extension reports failures as negative status codes
(``include/harmony_b200.h``); :func:`raise_for_status` maps them back here.
"""

from __future__ import annotations


class WrapschedError(Exception):
    """Root of every error raised by the planner or the runtime."""


HarmonyError = WrapschedError


class ValidationError(WrapschedError):
    """Malformed input or a broken invariant."""


class CyclicGraphError(ValidationError):
    """A layer graph has a cycle."""


class InvalidConfigurationError(ValidationError):
    """The four-tuple <u_f, p_f, u_b, p_b> violates a structural rule."""


class UnroutableBranchError(ValidationError):
    """A relay annotation has no consumer downstream in the chain."""


class SchemaError(ValidationError):
    """A JSON document does not match the expected kind/version."""


class InsufficientSamplesError(ValidationError):
    """Too few distinct-microbatch profile samples to fit a model."""


class CapacityViolationError(ValidationError):
    """A task's working set exceeds the per-GPU memory budget alpha."""


class NonUniformModelError(ValidationError):
    """Closed-form analysis needs identical per-layer sizes."""


class NoFeasibleMicrobatchError(WrapschedError):
    """Not even a microbatch of one fits in device memory."""


class ProfileRangeError(WrapschedError):
    """A cost model was evaluated outside its fitted microbatch range."""


class MissingProfileError(WrapschedError):
    """No cost model exists for the requested (layer, pass)."""


class LayerTooLargeError(WrapschedError):
    """One layer alone exceeds the capacity at the requested microbatch."""


class UnpackableError(WrapschedError):
    """No capacity-feasible packing exists."""


class NoFeasibleConfigurationError(WrapschedError):
    """Every candidate of a configuration sweep was infeasible."""


class DeadlockError(WrapschedError):
    """Work items never became runnable (estimator) or an event was never
    signalled (runtime)."""


class DeviceError(WrapschedError):
    """A CUDA / NCCL call failed inside the native runtime."""


# Native status codes -> exception classes (see include/harmony_b200.h).
HM_OK = 0
HM_ERR_VALIDATION = -1
HM_ERR_CAPACITY = -2
HM_ERR_DEADLOCK = -3
HM_ERR_DEVICE = -4
HM_ERR_MISSING_PROFILE = -5
HM_ERR_INTERNAL = -6
HM_ERR_PROFILE_RANGE = -7
HM_ERR_LAYER_TOO_LARGE = -8
HM_ERR_UNPACKABLE = -9

_STATUS = {
    HM_ERR_VALIDATION: ValidationError,
    HM_ERR_CAPACITY: CapacityViolationError,
    HM_ERR_DEADLOCK: DeadlockError,
    HM_ERR_DEVICE: DeviceError,
    HM_ERR_MISSING_PROFILE: MissingProfileError,
    HM_ERR_INTERNAL: WrapschedError,
    HM_ERR_PROFILE_RANGE: ProfileRangeError,
    HM_ERR_LAYER_TOO_LARGE: LayerTooLargeError,
    HM_ERR_UNPACKABLE: UnpackableError,
}


def raise_for_status(code: int, message: str) -> None:
    """Raise the exception class a native status code stands for."""
    if code >= 0:
        return
    raise _STATUS.get(code, WrapschedError)(message or f"native status {code}")
