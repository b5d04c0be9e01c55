"""Error types of the drop-in API (data.py:31, engine.py:45 of the reference)."""


class InvalidInput(ValueError):
    """An operation's preconditions are violated."""


class EngineError(RuntimeError):
    """A pipeline stage or device call failed; the message names the stage."""


class FormatError(ValueError):
    """Malformed or truncated file payload (serialize.py:28)."""
