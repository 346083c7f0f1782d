"""Random structured programs (placeholder; see fuzz generator below)."""
from .corpus import c4


def program(seed, minor=10, **kw):
    return c4(seed, minor, target_units=kw.get("units", 300))
