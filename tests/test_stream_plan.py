"""Host-side check of the streamed run's schedule (d2q37_debug_stream_plan; no GPU needed).

A pipelined d2q37_run_canonical queues uploads of y-chunks, FUSED2 sweeps of row ranges (each chunk as a
parallelogram of sweeps on the two alternating state buffers), wall / periodic image refreshes and
downloads.  This test replays the operation list on a model of the two buffers -- a version number per
row, and per ghost-row block -- and checks what makes the result equal to load + step + dump
(LatticeState::load, n x lbm::step, LatticeState::dump; lattice.hpp:18-19, kernels.cpp:276-283):

* every sweep s reads rows [lo - 6, hi + 6) (ghost rows included) at version s - 1, all uploaded;
* no compute operation touches buffer-0 rows whose upload it has not waited for (the copy engine may
  still be writing them), and nothing writes rows a download has been queued for;
* image refreshes copy rows that are complete at that version;
* a download reads final rows, is queued only after the host rows it overwrites were uploaded (the call
  may run in place), and the downloads cover every row exactly once;
* the ghost rows are left holding the final state's images (the handle keeps stepping afterwards).
"""
import os

import numpy as np
import pytest

UPLOAD, WAIT, SWEEP, MIRROR, WRAP, DOWNLOAD = range(6)
H = 6  # rows a two-step sweep reaches


class _Env:
    def __init__(self, **kv):
        self.kv = {k: str(v) for k, v in kv.items()}

    def __enter__(self):
        self.old = {k: os.environ.get(k) for k in self.kv}
        os.environ.update(self.kv)

    def __exit__(self, *exc):
        for k, v in self.old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def replay(ops, ly, nsteps, bc):
    S = nsteps // 2
    ver = np.full((2, ly), -1, dtype=np.int64)      # state version of each row of the two buffers
    ghost = np.full((2, 2), -1, dtype=np.int64)     # [buffer][lo / hi]: version the image rows mirror
    influx = np.zeros(ly, dtype=bool)               # buffer 0: uploads queued, not yet waited for
    uploaded = np.zeros(ly, dtype=bool)             # host rows already copied up (and waited for)
    queued = np.zeros((2, ly), dtype=bool)          # rows a queued download still reads
    got = np.zeros(ly, dtype=np.int64)              # downloads per row
    uploads = {}
    seen_compute = False
    for kind, a, b, c in ops:
        if kind == UPLOAD:
            assert not seen_compute, "uploads are queued first"
            assert 0 <= a < b <= ly and not influx[a:b].any(), (a, b)
            influx[a:b] = True
            uploads.setdefault(int(c), []).append((a, b))
            continue
        seen_compute = True
        if kind == WAIT:
            for idx, rows in uploads.items():  # the copy stream is in order: everything up to c is done
                if idx <= c:
                    for a0, b0 in rows:
                        if influx[a0]:
                            influx[a0:b0] = False
                            uploaded[a0:b0] = True
                            ver[0, a0:b0] = 0
        elif kind == SWEEP:
            s, lo, hi = int(c), int(a), int(b)
            assert 1 <= s <= S and 0 <= lo < hi <= ly and lo % 2 == 0, (s, lo, hi)
            src, dst = (s - 1) & 1, s & 1
            r0, r1 = max(0, lo - H), min(ly, hi + H)
            assert (ver[src, r0:r1] == s - 1).all(), f"sweep {s} [{lo},{hi}) reads rows not at version {s - 1}"
            if src == 0:
                assert not influx[r0:r1].any(), f"sweep {s} [{lo},{hi}) reads rows still being uploaded"
            if lo - H < 0:
                assert ghost[src, 0] == s - 1, f"sweep {s} [{lo},{hi}): low images at {ghost[src, 0]}"
            if hi + H > ly:
                assert ghost[src, 1] == s - 1, f"sweep {s} [{lo},{hi}): high images at {ghost[src, 1]}"
            assert not queued[dst, lo:hi].any(), f"sweep {s} [{lo},{hi}) overwrites rows queued for download"
            if dst == 0:
                assert not influx[lo:hi].any(), f"sweep {s} [{lo},{hi}) writes rows still being uploaded"
            ver[dst, lo:hi] = s
        elif kind in (MIRROR, WRAP):
            s, buf = int(c), int(c) & 1
            mask = 3 if kind == WRAP else int(a)
            assert (kind == WRAP) == (bc == "periodic")
            need_lo = (mask & 1) or kind == WRAP  # periodic images: each side copies the other side's rows
            need_hi = (mask & 2) or kind == WRAP
            if need_lo:
                assert (ver[buf, :H] == s).all() and not (buf == 0 and influx[:H].any()), f"images of sweep {s}: rows 0..5"
            if need_hi:
                assert (ver[buf, ly - H:] == s).all() and not (buf == 0 and influx[ly - H:].any()), \
                    f"images of sweep {s}: rows ly-6..ly-1"
            if mask & 1:
                ghost[buf, 0] = s
            if mask & 2:
                ghost[buf, 1] = s
        elif kind == DOWNLOAD:
            assert 0 <= a < b <= ly
            assert (ver[S & 1, a:b] == S).all(), f"download [{a},{b}) of rows that are not final"
            assert uploaded[a:b].all(), f"download [{a},{b}) over host rows not uploaded yet (in-place call)"
            queued[S & 1, a:b] = True
            got[a:b] += 1
        else:
            raise AssertionError(f"unknown operation {kind}")
    assert not influx.any(), "an upload nobody waited for"
    assert (got == 1).all(), "the downloads do not cover every row exactly once"
    assert (ver[S & 1] == S).all()
    assert (ghost[S & 1] == S).all(), "the ghost rows do not hold the final state's images"


CASES = [(16384, 200), (16384, 170), (16384, 400), (16384, 2), (2400, 20), (2400, 100), (1201, 10), (486, 4), (700, 6), (40000, 60), (7, 2), (13, 4)]


@pytest.mark.parametrize("ly,nsteps", CASES)
@pytest.mark.parametrize("bc", ["wall", "periodic"])
def test_default_plan_replays(lbm, ly, nsteps, bc):
    ops = lbm.stream_plan(ly, nsteps, bc)
    if bc == "periodic" and len(ops) == 0:  # too short for the two seam pieces: three verbs
        assert ly < 2 * (8 * (nsteps // 2) + 240) + 480
        return
    assert len(ops) > 0
    replay(ops.tolist(), ly, nsteps, bc)


@pytest.mark.parametrize("rows,first,last,skew", [(480, 240, 120, 8), (240, 120, 240, 8), (124, 36, 12, 8), (24, 8, 8, 8),
                                                  (720, 120, 6, 6), (360, 120, 120, 14), (4440, 4440, 4440, 12)])
@pytest.mark.parametrize("ly,nsteps,bc", [(2400, 40, "wall"), (1203, 100, "wall"), (600, 8, "wall"),
                                          (2400, 20, "periodic"), (5001, 100, "periodic")])
def test_plans_of_other_chunk_heights_replay(lbm, rows, first, last, skew, ly, nsteps, bc):
    with _Env(D2Q37_STREAM_ROWS=rows, D2Q37_STREAM_FIRST=first, D2Q37_STREAM_LAST=last, D2Q37_STREAM_SKEW=skew):
        ops = lbm.stream_plan(ly, nsteps, bc)
        if len(ops):
            replay(ops.tolist(), ly, nsteps, bc)
        else:
            assert bc == "periodic"


@pytest.mark.parametrize("ly,nsteps", [(16384, 170), (16384, 400), (16384, 200), (8192, 170), (16216, 200), (5000, 120)])
@pytest.mark.parametrize("bc", ["wall", "periodic"])
def test_no_narrow_download_between_chunks(lbm, ly, nsteps, bc):
    """A chunk whose final rows are a sliver (its range clipped at row 0 after leaning back 8 rows per
    sweep: 40 rows at 170 steps, 80 at 400 on 16384 rows) hands them to the next chunk's download: a
    first download that narrow measured 0.4-0.9 s per run (DESIGN 3.3).  Only the last download may
    be as narrow as the rows left."""
    ops = lbm.stream_plan(ly, nsteps, bc).tolist()
    downs = [(a, b) for kind, a, b, _ in ops if kind == DOWNLOAD]
    assert downs
    wave = downs[2:] if bc == "periodic" else downs  # the two seam pieces come first (two bands each)
    for a, b in wave[:-1]:
        assert b - a >= 240, (a, b)
    with _Env(D2Q37_STREAM_MIN_DOWNLOAD=1):  # the rule off: the sliver is back (walls, 170 steps)
        if (ly, nsteps, bc) == (16384, 170, "wall"):
            raw = [(a, b) for kind, a, b, _ in lbm.stream_plan(ly, nsteps, bc).tolist() if kind == DOWNLOAD]
            assert min(b - a for a, b in raw[:-1]) == 40
            replay(lbm.stream_plan(ly, nsteps, bc).tolist(), ly, nsteps, bc)


def test_random_plans_replay(lbm):
    """300 seeded random draws of height, step count, boundary mode, chunk heights and skew."""
    rng = np.random.default_rng(20181804)
    ran = 0
    for _ in range(300):
        ly = int(rng.integers(6, 6000))
        nsteps = 2 * int(rng.integers(1, 60))
        bc = "periodic" if rng.random() < 0.4 else "wall"
        env = dict(D2Q37_STREAM_ROWS=int(rng.integers(6, 3000)), D2Q37_STREAM_FIRST=int(rng.integers(6, 800)),
                   D2Q37_STREAM_LAST=int(rng.integers(6, 800)), D2Q37_STREAM_SKEW=int(rng.choice([6, 8, 10, 12, 16])))
        with _Env(**env):
            ops = lbm.stream_plan(ly, nsteps, bc)
            if len(ops):
                try:
                    replay(ops.tolist(), ly, nsteps, bc)
                except AssertionError as e:
                    raise AssertionError(f"ly {ly} nsteps {nsteps} bc {bc} env {env}: {e}") from e
                ran += 1
    assert ran > 150


def test_replay_catches_a_broken_plan(lbm):
    """The model is not vacuous: dropping an image refresh, or a sweep, fails the replay."""
    ops = lbm.stream_plan(2400, 20, "wall").tolist()
    mirrors = [i for i, op in enumerate(ops) if op[0] == MIRROR and op[3] > 0]
    with pytest.raises(AssertionError):
        replay(ops[:mirrors[0]] + ops[mirrors[0] + 1:], 2400, 20, "wall")
    sweeps = [i for i, op in enumerate(ops) if op[0] == SWEEP]
    with pytest.raises(AssertionError):
        replay(ops[:sweeps[5]] + ops[sweeps[5] + 1:], 2400, 20, "wall")


def test_plan_arguments(lbm):
    with pytest.raises(ValueError):
        lbm.stream_plan(2400, 3, "wall")
    with pytest.raises(ValueError):
        lbm.stream_plan(0, 2, "wall")
