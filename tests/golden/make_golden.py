#!/usr/bin/env python3
"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref/liblbmref.so).

Run in the build container (needs /root/reference to build oracle/_ref):

    make -C oracle && python tests/golden/make_golden.py

Every array is produced by the reference's own code path through
oracle/ref_shim.cpp: VelocityModel::d2q37 (model.cpp), make_random_lattice
(lattice.cpp:8-23), halo_exchange / propagate / collide / step on a
LatticeState (kernels.cpp) and the validation oracle (validation.cpp:13-38).
Canonical arrays have shape (37, lx, ly) (dump.hpp:19-21); padded arrays are
Field::data() in Descriptor order (layout.hpp:67-79).
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import pyoracle as po  # noqa: E402


def model():
    m = po.ref_model()
    np.savez_compressed(os.path.join(HERE, "ref_model.npz"), cx=m.cx, cy=m.cy, w=m.w, t0=np.float64(m.t0), eq=m.eq)


def lattice_case(lx, ly, seed, name, steps=10, omega_step=1.0, omega_collide=1.2, vl_csoa=4):
    init = po.ref_random_lattice(lx, ly, seed)
    out = {"init": init, "lx": lx, "ly": ly, "seed": seed, "omega_step": omega_step,
           "omega_collide": omega_collide, "steps": steps, "vl_csoa": vl_csoa}
    # halo_exchange + propagate on the SoA and CSoA layouts (kernels.cpp:197-258)
    for tag, layout, vl in (("aos", po.AOS, 1), ("soa", po.SOA, 1), ("csoa", po.CSOA, vl_csoa),
                            ("caosoa", po.CAOSOA, vl_csoa)):
        s = po.RefSim(layout, lx, ly, vl, workers=2)
        s.load(init)
        s.halo_exchange()
        out[f"padded_{tag}"] = s.raw(0)
        s.propagate()
        out[f"propagate_{tag}"] = s.dump(1)
    # collide on nxt -> prv (kernels.cpp:260-274)
    s = po.RefSim(po.SOA, lx, ly, 1, workers=2)
    s.load(init, which=1)
    s.collide(omega_collide)
    out["collide"] = s.dump(0)
    # the validation oracle's per-site collide (validation.cpp:27-38)
    out["oracle_collide"] = po.ref_oracle_collide(init, omega_collide)
    # full steps (kernels.cpp:276-283)
    s = po.RefSim(po.CSOA, lx, ly, vl_csoa, workers=2)
    s.load(init)
    s.step(omega_step, steps)
    out["step"] = s.dump(0)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)


def main():
    po.build()
    model()
    lattice_case(16, 32, 2024, "ref_random_16x32")
    lattice_case(5, 12, 606, "ref_random_5x12", steps=5, omega_step=1.3, vl_csoa=4)  # strip == halo
    # an LBDUMP01 file written by the reference's save_dump (dump.cpp:44-58)
    po.ref_save_dump(po.ref_random_lattice(5, 12, 606), os.path.join(HERE, "ref_dump_5x12.lbd"))
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
