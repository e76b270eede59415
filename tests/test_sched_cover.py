"""Host-side check of the FUSED2 sweep schedules (tests/cpp/sched_check.cu; no GPU needed): every
(band, column) item of a sweep is swept by exactly one persistent CTA -- the lockstep schedule
(lockstep_plan / LockSched), the band-major ranges (RangeSched) and the overlapped slab plan of the pair
form (pair_slab_plan: face CTAs' face + adjacent bands, main CTAs in lockstep) -- over a grid of
extents, band counts and CTA counts; face CTAs sweep their face items first."""
import os
import shutil
import subprocess

import pytest

from conftest import ROOT

SRC = os.path.join(ROOT, "tests", "cpp", "sched_check.cu")
EXE = os.path.join(ROOT, "tests", "cpp", "_build", "sched_check")


def test_schedules_cover_every_item_once():
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.access(nvcc, os.X_OK):
        pytest.skip("nvcc absent")
    os.makedirs(os.path.dirname(EXE), exist_ok=True)
    subprocess.run([nvcc, "-std=c++17", "-O1", "-arch=sm_100a", "-I", os.path.join(ROOT, "paper_1804_01918_b200", "csrc"),
                    "-I", os.path.join(ROOT, "include"), SRC, "-o", EXE], check=True, capture_output=True, timeout=600)
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout + r.stderr
