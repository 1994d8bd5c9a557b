"""Error types of the host API (mirrors smshare/errors.py:1-9).

`InvalidArgumentError` is raised for out-of-domain arguments, `ConfigError`
for malformed experiment configs; both subclass ValueError like the
reference so callers catching ValueError keep working.
"""


class InvalidArgumentError(ValueError):
    """Arguments outside an operation's domain."""


class ConfigError(ValueError):
    """A malformed or inconsistent experiment configuration."""
