"""Error types, same names and bases as the reference (sp/core.py:29-34)."""


class ConfigError(ValueError):
    """Malformed input: bad file, bad schema, violated structural invariant."""


class InfeasibleError(RuntimeError):
    """Well-formed input with no feasible answer (e.g. the model cannot fit)."""
