"""Generate tests/golden/golden.json from the UNMODIFIED reference library.

Run in the container that has /root/reference (the reference is compiled from
its own sources by oracle/Makefile into oracle/_ref/libminipic_ref.so):

    python tests/golden/make_golden.py

Everything written here comes out of the reference's own functions
(pic::move_batch, pic::init_gem, pic::wrap_len, pic::grid_cell_of,
pic::implicit_velocity) on fixed, seeded inputs.  Doubles are stored as
hex strings (float.hex) so they round-trip bit-exactly; large arrays are
stored as SHA-256 digests of their little-endian bytes plus a short prefix.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")
PREFIX = 16


def digest(arrs) -> str:
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(a, dtype="<f8").tobytes())
    return h.hexdigest()


def hexs(a):
    return [float(v).hex() for v in np.asarray(a).ravel()]


def mover_case(name, grid, parts, E, B, dt, qoms, pc):
    out = {"grid": list(grid), "dt": dt, "pc": pc, "field_sha": digest([E, B]), "species": []}
    for s, p in enumerate(parts):
        inp = [a.copy() for a in p]
        res = [a.copy() for a in p]
        oracle.ref_move_batch(res, E, B, grid, dt, qoms[s], pc)
        out["species"].append({
            "qom": qoms[s], "count": len(inp[0]), "in_sha": digest(inp), "out_sha": digest(res),
            "out_prefix": [hexs(a[:PREFIX]) for a in res]})
    return out


def main():
    oracle.build()
    g = {}

    # C1: the reference small_cfg (test_runtime.cpp:18-27) GEM state with the
    # gem_like_field fixture (nonzero E, test_offload.cpp:60-71), one mover step
    c1 = (8, 8, 8, 6.4, 6.4, 6.4)
    parts, E0, B0 = oracle.ref_init_gem(c1, 8)
    g["c1_init"] = {"grid": list(c1), "ppc": 8, "seed": 12345,
                    "counts": [len(p[0]) for p in parts],
                    "species_sha": [digest(p) for p in parts], "field_sha": digest([E0, B0])}
    E, B = oracle.port_gem_like_field(c1)
    g["c1_gem_like_field_sha"] = digest([E, B])
    qoms = [-25.0, 1.0, -25.0, 1.0]
    g["c1_move"] = mover_case("c1", c1, parts, E, B, 0.1, qoms, 3)
    # same state, the stock GEM field (E = 0) and pc 1 / 5
    g["c1_move_gemfield_pc5"] = mover_case("c1b", c1, parts, E0, B0, 0.1, qoms, 5)
    g["c1_move_pc1"] = mover_case("c1c", c1, parts, E, B, 0.05, qoms, 1)

    # deposit_moments (kernels.cpp:147-183) of the C1 GEM state, per species,
    # with the pressure tensor: digests of the 10 moment arrays
    _, qpp, _ = oracle.ref_gem_species(c1, 8)
    g["c1_moments"] = {"qpp": hexs(qpp), "species": []}
    for s, p in enumerate(parts):
        m = oracle.ref_deposit_moments(p, c1, float(qpp[s]), True)
        g["c1_moments"]["species"].append({"sha": [digest([a]) for a in m],
                                           "rho_prefix": hexs(m[0][:8])})

    # field_phase_stub (kernels.cpp:185-215) of the C1 gem_like field, 3 passes
    Es, Bs = oracle.ref_field_phase_stub(E, B, c1, 3)
    g["c1_field_stub3"] = {"sha": digest([Es, Bs]), "E_prefix": hexs(Es[:12])}

    # desk preset (sim_config.hpp desk_benchmark_config): 32x32x16 at 64 ppc
    desk = (32, 32, 16, 25.6, 12.8, 6.4)
    parts, E0, B0 = oracle.ref_init_gem(desk, 64)
    g["desk_init"] = {"grid": list(desk), "ppc": 64, "seed": 12345,
                      "counts": [len(p[0]) for p in parts],
                      "species_sha": [digest(p) for p in parts], "field_sha": digest([E0, B0])}
    E = E0.copy()
    Eg, _ = oracle.port_gem_like_field(desk)
    E[:] = Eg
    g["desk_move"] = mover_case("desk", desk, parts, E, B0, 0.1, qoms, 3)

    # SPEC.md KATs (implicit_velocity / one mover step, uniform B=(0,0,1), beta=0.1)
    vbar = oracle.ref_implicit_velocity([1.0, 0.0, 0.0], [0.0, 0.0, 0.0], [0.0, 0.0, 1.0], 0.2, 1.0)
    kat_grid = (4, 4, 4, 4.0, 4.0, 4.0)
    nodes = 5 * 5 * 5
    Eu = np.zeros(3 * nodes)
    Bu = np.tile([0.0, 0.0, 1.0], nodes)
    p = [np.array([1.5]), np.array([1.5]), np.array([1.5]), np.array([1.0]), np.array([0.0]),
         np.array([0.0])]
    oracle.ref_move_batch(p, Eu, Bu, kat_grid, 0.2, 1.0, 3)
    g["kat"] = {"vbar": hexs(vbar), "grid": list(kat_grid), "dt": 0.2, "qom": 1.0, "pc": 3,
                "x0": hexs([1.5, 1.5, 1.5]), "v0": hexs([1.0, 0.0, 0.0]),
                "x1": hexs([p[0][0], p[1][0], p[2][0]]), "v1": hexs([p[3][0], p[4][0], p[5][0]])}

    # wrap_len edge cases (test_core.cpp:18-32 and more)
    l = 6.4
    vs = [0.0, -0.0, 10.0, -0.1, 23.5, -20.0, l - 1e-17, -1e-17, np.nextafter(l, 0.0),
          np.nextafter(0.0, -1.0), l, 2 * l, np.nextafter(2 * l, 0.0), -l, np.nextafter(-l, 0.0),
          np.nextafter(-l, -100.0), 3.3, -3.3, 1e-300, -1e-300, 5e-324, -5e-324, 12.7999999,
          -6.3999999999]
    g["wrap_len"] = [{"v": float(v).hex(), "l": l.hex(), "w": oracle.ref_wrap_len(float(v), l).hex()}
                     for v in vs]
    for L in (10.0, 25.6, 12.8, 0.3):
        for v in (np.nextafter(L, 0.0), -1e-17, np.nextafter(0.0, -1.0), np.nextafter(2 * L, 0.0),
                  np.nextafter(-L, 0.0), -L, L, 1.5 * L, -0.5 * L):
            g["wrap_len"].append({"v": float(v).hex(), "l": float(L).hex(),
                                  "w": oracle.ref_wrap_len(float(v), L).hex()})

    # grid_cell_of known answers (test_core.cpp:54-69)
    cg = (4, 4, 4, 4.0, 4.0, 4.0)
    cells = []
    for pos in ([1.25, 2.5, 3.75], [float(np.nextafter(4.0, 0.0)), 0.0, 0.0], [0.0, 0.0, 0.0],
                [3.999999999, 1.0, 2.0]):
        ijk, f = oracle.ref_grid_cell_of(pos, cg)
        cells.append({"pos": hexs(pos), "ijk": list(ijk), "f": hexs(f)})
    g["grid_cell_of"] = {"grid": list(cg), "cases": cells}

    # NaN fault (test_kernels.cpp:216-230): the reference names index 1
    fg = (4, 4, 4, 4.0, 4.0, 4.0)
    Ef = np.zeros(3 * nodes)
    Bf = np.tile([0.0, 0.0, 1.0], nodes)
    p = [np.array([1.0, 2.0, 3.0]), np.array([1.0, 2.0, 3.0]), np.array([1.0, 2.0, 3.0]),
         np.array([0.1, np.nan, 0.1]), np.zeros(3), np.zeros(3)]
    try:
        oracle.ref_move_batch(p, Ef, Bf, fg, 0.1, 1.0, 2)
        raise SystemExit("reference did not fault")
    except oracle.OracleError as e:
        g["nan_fault"] = {"status": e.status, "message": e.msg,
                          "after": [hexs(a) for a in p]}

    with open(OUT, "w") as f:
        json.dump(g, f, indent=1, sort_keys=True)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
