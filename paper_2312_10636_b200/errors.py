"""Exception hierarchy mirroring the reference's (fragserve/errors.py:4-17).

When fragserve is importable the reference classes are used directly, so callers that catch
`fragserve.InfeasibleError` also catch executor failures; otherwise identical stand-ins are
defined here (same names, same bases, same meaning).
"""
from __future__ import annotations

try:  # pragma: no cover - depends on the environment
    from fragserve.errors import FragserveError, InfeasibleError, ProfileParseError, ValidationError
except Exception:  # noqa: BLE001 - the reference is optional at run time
    class FragserveError(Exception):
        pass

    class ProfileParseError(FragserveError, ValueError):
        """Malformed profile/trace/spec input; message names the offending line."""

    class ValidationError(FragserveError, ValueError):
        """Input violates a structural requirement."""

    class InfeasibleError(FragserveError, RuntimeError):
        """No allocation/placement satisfies the constraints."""

GX_EINVAL, GX_EINFEASIBLE, GX_ECUDA, GX_EINTERNAL = -1, -2, -3, -4


def raise_for_status(rc: int, msg: str):
    """Map a libgx status (include/graft_exec.h) onto the reference's error classes."""
    if rc == 0:
        return
    if rc == GX_EINVAL:
        raise ValidationError(msg)
    if rc == GX_EINFEASIBLE:
        raise InfeasibleError(msg)
    raise FragserveError(msg)
