"""One banded FUSED2 sweep (two steps) on an lx x ly wall lattice, for ncu (-k regex:k_band_sweep)."""
import sys

sys.path.insert(0, ".")
import paper_1804_01918_b200 as lbm  # noqa: E402

lx, ly = (int(a) for a in (sys.argv[1:3] if len(sys.argv) > 2 else (4096, 4096)))
s = lbm.Simulation("banded", lx, ly, 1, device=0, bc="wall", variant="fused2")
s.init_rt_device(12345)
s.step(0.8, 2)
s.sync()
