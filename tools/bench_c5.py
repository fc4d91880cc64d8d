"""Large-configuration mover measurement (or C4 with
--config c4 --ppc 905): 128x128x64 cells,
L = (51.2, 25.6, 12.8), 460 ppc -> ~1.0e9 particles (48 GB of SoA) on ONE B200.

The reference GEM state is generated on the host with the bit-exact
generator in chunks (background species by counter-RNG jump-ahead, the sheet
species whole) and uploaded chunk by chunk, so host memory stays small.
Reports MPA/s of the FAST mover (device-resident, cell-sorted once, CUDA
events), per pc in {3, 4, 5} as C5 asks, and the HBM roofline fraction.
Usage: python tools/bench_c5.py [--steps 5] [--ppc 460]
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1904_03684_b200 import _capi, gem  # noqa: E402
from paper_1904_03684_b200.engine import DeviceStore  # noqa: E402
from paper_1904_03684_b200.mover import Grid, MoverParams  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--ppc", type=int, default=460)
    ap.add_argument("--chunk", type=int, default=1 << 24)
    ap.add_argument("--config", choices=["c5", "c4"], default="c5",
                    help="c4: SURVEY C4's 64x64x32 grid (run with --ppc 905: 255.8M particles)")
    a = ap.parse_args()
    grid = (Grid.make(128, 128, 64, 51.2, 25.6, 12.8) if a.config == "c5"
            else Grid.make(64, 64, 32, 25.6, 12.8, 6.4))
    counts = gem.gem_counts(grid, a.ppc)
    qom, _ = gem.gem_species_params(grid, a.ppc)
    n_total = sum(counts)
    t0 = time.perf_counter()
    st = DeviceStore(grid, counts, "fast")
    st.upload_field(gem.gem_field(grid))
    g = grid.to_c()
    for s in range(4):
        if s < 2:
            for m0 in range(0, counts[s], a.chunk):
                m1 = min(counts[s], m0 + a.chunk)
                arrs = [np.empty(m1 - m0) for _ in range(6)]
                _capi.check(_capi.lib().b2m_gem_fill_species_range(
                    C.byref(g), a.ppc, gem.DEFAULT_SEED, s, m0, m1, _capi.ptr6(arrs), 0))
                _capi.check(_capi.lib().b2m_species_upload_range(st.h, s, _capi.ptr6(arrs), m0,
                                                                 m1 - m0))
            _capi.check(_capi.lib().b2m_species_set_count(st.h, s, counts[s]))
        else:
            b = gem.init_gem_species(grid, a.ppc, species=(s,))[0]
            st.upload(s, b.span())
    st.sync()
    t_init = time.perf_counter() - t0
    for s in range(4):
        st.sort(s)
    st.sync()
    label = ("C5 128x128x64, L=(51.2,25.6,12.8)" if a.config == "c5"
             else "C4 64x64x32, L=(25.6,12.8,6.4)")
    out = {"config": "%s, ppc %d" % (label, a.ppc), "particles": n_total,
           "soa_gb": n_total * 48 / 1e9, "init_s": t_init, "runs": []}
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(
        os.path.abspath(__file__))), "MEASURED_PEAKS.json"))).get("hbm_gbs", 6450.3)
    for pc in (3, 4, 5):
        mps = [MoverParams.make(0.1, float(qom[s]), pc) for s in range(4)]
        st.move_all(mps)  # warm-up (and table build)
        st.sync()
        ms = []
        for _ in range(a.steps):
            st.record(2)
            st.move_all(mps)
            st.record(3)
            st.sync()
            ms.append(st.elapsed_ms(2, 3))
        m = sum(ms) / len(ms)
        out["runs"].append({"pc": pc, "ms_per_step": m, "mpa_s": n_total / (m * 1e-3) / 1e6,
                            "hbm_frac": 96 * n_total / (m * 1e-3) / 1e9 / peak})
        print(json.dumps(out["runs"][-1]), flush=True)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
