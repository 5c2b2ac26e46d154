"""Exception classes of the reference engine (packedhe/engine.py:32-41)."""


class EngineError(ValueError):
    """Malformed engine input: incompatible operands or bad parameters."""


class CapacityError(EngineError):
    """Payload does not fit the slot vector."""


class LayoutError(EngineError):
    """Operand layout does not match what the operation requires."""
