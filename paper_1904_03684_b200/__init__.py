"""B200-native semi-implicit particle mover (iPIC3D, arXiv 1904.03684).

Drop-in for the reference minipic mover path: ``pic::move_batch``
(kernels.cpp:52-104) and the ``pic::Engine`` interface (engines.hpp:20-48),
backed by hand-written sm_100a CUDA kernels in ``libb2m.so`` (C ABI:
include/b2m.h).
"""
from .errors import (AllocError, CflViolation, ConfigError, DomainError, EngineFault,
                     MetricError, MinipicError, NumericalFault)
from .mover import (FieldMesh, Grid, MomentMesh, MoverParams, ParticleBatch, deposit_moments,
                    field_phase_stub, move_batch)

__all__ = ["AllocError", "CflViolation", "ConfigError", "DomainError", "EngineFault",
           "MetricError", "MinipicError", "NumericalFault", "FieldMesh", "Grid", "MomentMesh",
           "MoverParams", "ParticleBatch", "deposit_moments", "field_phase_stub", "move_batch"]
