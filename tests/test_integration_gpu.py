"""The unmodified reference Simulation (runtime, exchange, moments, field
stub, timings) driving its mover through the B200 engine plug-in
(integration/minipic_b200_engine.cpp -> libb2m C ABI).

Mirrors the reference's own cross-engine checks: acceptance #3 / 
test_runtime.cpp:198-212 (engines bitwise identical after several cycles),
test_runtime.cpp:214-226 (worker-count multiset), test_runtime.cpp:271-282
(an offload kernel fault surfaces as EngineFault naming the particle)."""
import os

import numpy as np
import pytest

import oracle
from tests._util import assert_within_contract

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not oracle.b200_integration_available(),
                                 reason="integration library not built (needs /root/reference)")]
GRID_T = (8, 8, 8, 6.4, 6.4, 6.4)


def _run(engine, workers, cycles, b2m=False, mode="strict", inject=None):
    os.environ["B2M_ENGINE"] = "1" if b2m else "0"
    os.environ["B2M_MODE"] = mode
    try:
        sim = oracle.RefSimulation(GRID_T, 8, workers=workers, engine=engine, field_passes=10,
                                   lib=oracle.ref_b200(), inject=inject)
        sim.run(cycles)
        return sim, [sim.gather(s) for s in range(4)]
    finally:
        os.environ["B2M_ENGINE"] = "0"


@pytest.mark.parametrize("engine", ["naive", "pinned", "prefetch"])
@pytest.mark.parametrize("workers", [1, 4])
def test_reference_simulation_on_b200_engine_is_bitwise_cpu(gpu, engine, workers):
    _, cpu = _run("cpu", workers, 5)
    sim, b200 = _run(engine, workers, 5, b2m=True, mode="strict")
    for s in range(4):
        for a in range(6):
            np.testing.assert_array_equal(b200[s][a].view(np.uint64), cpu[s][a].view(np.uint64))
    assert sim.mean_mover_s() > 0


def test_reference_simulation_on_b200_fast_mode(gpu):
    _, cpu = _run("cpu", 1, 3)
    _, fast = _run("pinned", 1, 3, b2m=True, mode="fast")
    for s in range(4):
        assert_within_contract(fast[s], cpu[s], GRID_T, tol=1e-11, what=f"species {s}")


def test_reference_simulation_b200_fault_is_engine_fault(gpu):
    os.environ["B2M_ENGINE"] = "1"
    try:
        ref_parts, E, B = oracle.ref_init_gem(GRID_T, 8)
        ref_parts[0][3][5] = np.nan
        with pytest.raises(oracle.OracleError) as ei:
            _run("naive", 1, 1, b2m=True, inject=(ref_parts, E, B))
        assert ei.value.status == 6 and "particle" in ei.value.msg
    finally:
        os.environ["B2M_ENGINE"] = "0"
