"""Error taxonomy of the drop-in API.

Mirrors the reference hierarchy (reference: pkg/src/gshare_sim/errors.py:4-31)
so callers that catch ``ValidationError`` / ``GShareError`` keep working when
they switch to the CUDA backend.  The C-ABI status codes map onto these:

    GS_OK            -> no error
    GS_ERR_VALIDATION-> ValidationError   (e.g. zero serving rate mid-run)
    GS_ERR_CAPACITY  -> retried on device with larger capacities, then
                        CapacityError (a ValidationError) if still too small
    GS_ERR_INVARIANT -> InvariantError
"""


class GShareError(Exception):
    """Root of every error raised by this package."""


class ValidationError(GShareError):
    """Input violates a documented constraint (raised before or during a run)."""


class ParseError(GShareError):
    """A profile, trace or scenario file could not be parsed."""

    def __init__(self, message: str, line_number: int | None = None):
        self.line_number = line_number
        if line_number is not None:
            message = f"line {line_number}: {message}"
        super().__init__(message)


class ConflictError(GShareError):
    """Duplicate or inconsistent records."""


class MissingConfigurationError(GShareError):
    """Lookup of a profile point / memory spec that does not exist."""


class InvariantError(GShareError):
    """The device reported corrupt scheduler state."""


class CapacityError(ValidationError):
    """A scenario outgrew the largest device capacity the backend will try."""


class BackendUnavailableError(GShareError):
    """The CUDA extension is missing or no GPU is visible.

    There is deliberately no CPU fallback: the product path fails loudly.
    """
