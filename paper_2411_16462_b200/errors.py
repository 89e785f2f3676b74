"""Error classes of the drop-in API.

Names, base classes and message formats follow the reference's error
contract (lioncomm/errors.py:4-52) so callers can catch the same types:
``ConfigError`` for bad configuration or values, ``CapacityError`` raised
before any exchange when a p-bit sum would not fit, ``CollectiveError`` for a
failed/timed-out exchange.  ``DeviceError`` is new: the CUDA library is
missing or a CUDA call failed -- there is no CPU fallback to hide behind.
"""


class LionCommError(Exception):
    pass


class ConfigError(LionCommError):
    pass


class CapacityError(ConfigError):
    pass


class PackFormatError(LionCommError):
    pass


class DeviceError(LionCommError):
    pass


class PackRangeError(LionCommError):
    def __init__(self, index: int, value: int, width: int):
        self.index, self.value, self.width = index, value, width
        super().__init__(f"value {value} at index {index} does not fit "
                         f"{width}-bit storage")


class CollectiveError(LionCommError):
    def __init__(self, message: str, rank=None, generation=None, phase=None):
        self.rank, self.generation, self.phase = rank, generation, phase
        parts = [f"{k}={v}" for k, v in
                 (("rank", rank), ("generation", generation), ("phase", phase))
                 if v is not None]
        super().__init__(f"{message} ({', '.join(parts)})" if parts else message)
