"""Exception taxonomy of the host-side plugin API.

Mirrors the five exception classes the reference exposes
(reference: pkg/src/agentsched/errors.py:6-30) so that callers catching the
reference's errors keep working when the GPU data path is plugged in.
``DeviceError`` is new: it is raised when the native library reports a CUDA
failure and is never swallowed.
"""

from __future__ import annotations


class ConfigError(ValueError):
    """A configuration value is out of range or inconsistent."""


class ValidationError(ValueError):
    """Input data (a trace, a batch, a duration) violates an invariant."""


class TraceParseError(ValueError):
    """A trace line could not be parsed; carries the 1-based line number."""

    def __init__(self, line_number: int, message: str):
        self.line_number = line_number
        super().__init__(f"line {line_number}: {message}")


class ProtocolError(RuntimeError):
    """A component was driven through an illegal state transition."""


class SimulationError(RuntimeError):
    """The event loop could not make progress (deadlock, leak, oversize)."""


class DeviceError(RuntimeError):
    """The native CUDA library returned a non-zero status."""
