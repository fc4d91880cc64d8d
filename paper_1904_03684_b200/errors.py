"""Error taxonomy of the reference (errors.hpp:12-44), one class per type.

The C ABI reports these as b2m_status codes; ``raise_for_status`` turns a
status back into the exception the reference would throw, with the
reference's message text.
"""


class MinipicError(RuntimeError):
    """Base of the taxonomy (every reference error is a std::runtime_error)."""


class ConfigError(MinipicError):
    """Bad configuration value or inconsistent setup (errors.hpp:15-17)."""


class DomainError(MinipicError):
    """Position outside [0,l) handed to a grid operation (errors.hpp:20-22)."""


class AllocError(MinipicError):
    """Device / batch capacity exceeded (errors.hpp:25-27)."""


class NumericalFault(MinipicError):
    """Mover produced a non-finite value; names the particle (errors.hpp:30-32)."""

    def __init__(self, msg: str, index: int = -1, species: int = -1):
        super().__init__(msg)
        self.index = index
        self.species = species


class CflViolation(MinipicError):
    """A particle crossed more than one slab in one step (errors.hpp:35-37)."""


class EngineFault(MinipicError):
    """Offload failure; the engine / simulation state is invalid (errors.hpp:40-42)."""


class MetricError(MinipicError):
    """Nonsensical benchmark-metric input (errors.hpp:45-47)."""


class CudaError(EngineFault):
    """CUDA runtime failure inside libb2m (surfaced like an engine fault)."""


_BY_STATUS = {1: ConfigError, 2: DomainError, 3: AllocError, 4: NumericalFault,
              5: CflViolation, 6: EngineFault, 7: MetricError, 8: CudaError, 9: ValueError}


def raise_for_status(status: int, msg: str) -> None:
    cls = _BY_STATUS.get(status, MinipicError)
    raise cls(msg)
