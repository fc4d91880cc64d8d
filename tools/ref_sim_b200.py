"""The UNMODIFIED reference Simulation (oracle/_ref/libminipic_b200.so: the
reference sources + the B200 pic::Engine plug-in) at C2: mean mover time per
cycle with its own CPU engine (16 workers) vs the B200 engine (STRICT and
FAST, 1 worker, host batches over PCIe) -- what a reference user gets by
setting B2M_ENGINE=1."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (test/measurement infrastructure)

C2 = (64, 64, 32, 25.6, 12.8, 6.4)
cycles = int(sys.argv[1]) if len(sys.argv) > 1 else 3
out = {}
for label, env, engine, workers in [("cpu_engine_16_workers", {}, "cpu", 16),
                                    ("b200_strict", {"B2M_ENGINE": "1", "B2M_MODE": "strict"},
                                     "pinned", 1),
                                    ("b200_fast", {"B2M_ENGINE": "1", "B2M_MODE": "fast"},
                                     "pinned", 1)]:
    for k in ("B2M_ENGINE", "B2M_MODE"):
        os.environ.pop(k, None)
    os.environ.update(env)
    t0 = time.perf_counter()
    sim = oracle.RefSimulation(C2, 216, workers=workers, engine=engine, field_passes=0,
                               lib=oracle.ref_b200())
    sim.run(cycles)
    out[label] = {"mean_mover_s": sim.mean_mover_s(), "wall_s": time.perf_counter() - t0,
                  "mpa_s": 61046784 / sim.mean_mover_s() / 1e6}
    print(label, json.dumps(out[label]), flush=True)
    del sim
print(json.dumps(out))
