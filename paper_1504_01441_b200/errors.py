"""Exception types of the reference, re-exported by the mirror modules.

`RegistrationError` and `ConfigError` mirror pipeline.py:27-32,
`DegenerateFit` mirrors geometry.py:18.
"""


class RegistrationError(RuntimeError):
    """Too few reliable matches to register the pair."""


class ConfigError(ValueError):
    """Invalid parameter value or malformed configuration."""


class DegenerateFit(ValueError):
    """Raised when a point configuration cannot support a homography fit."""
