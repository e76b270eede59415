"""bench.py's launch contract on CPU: ``--gpus N`` starts N ranks itself (torch.distributed.run on
127.0.0.1) and prints exactly one JSON line with ``n_gpus: N``; a request for more GPUs than the host
has fails loudly instead of printing a 1-GPU line.  ``--stub`` replaces the lattice with a no-op and
the NCCL process group with gloo, so the rank plumbing (launch, barriers, max over ranks, the second
scaling mode, the 1-GPU points) runs here without a GPU."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH = os.path.join(ROOT, "bench.py")


def _run(args, env_extra=None, timeout=240):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR",
                                                            "MASTER_PORT")}
    env.update(env_extra or {})
    return subprocess.run([sys.executable, BENCH] + args, capture_output=True, text=True, timeout=timeout, env=env,
                          cwd=ROOT)


def _json_lines(out):
    return [json.loads(ln) for ln in out.splitlines() if ln.startswith("{")]


@pytest.mark.parametrize("n", [2, 3])
def test_gpus_n_launches_n_ranks(n):
    r = _run(["--stub", "--gpus", str(n), "--steps", "4", "--warmup", "3", "--no-extras", "--no-e2e"])
    assert r.returncode == 0, r.stderr[-3000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    line = lines[0]
    assert line["n_gpus"] == n
    assert line["config"]["parallelism"] == f"y-slab x{n}"
    assert line["config"]["ly_global"] == 16384 * n  # weak: 4096 x 16384 per GPU
    assert line["scaling"] == "weak"
    strong = line["scaling_strong"]
    assert strong["n_gpus"] == n and f"global 4096x{(32768 // n) * n}" in strong["config"]  # 32768 rows split
    assert set(line["efficiency_vs_1gpu_same_run"]) == {"weak", "strong"}
    assert line["stub"]


def test_strong_headline_reports_weak_beside_it():
    r = _run(["--stub", "--gpus", "2", "--scaling", "strong", "--steps", "4", "--warmup", "3", "--no-extras",
              "--no-e2e"])
    assert r.returncode == 0, r.stderr[-3000:]
    line = _json_lines(r.stdout)[0]
    assert line["scaling"] == "strong" and line["config"]["ly_per_gpu"] == 32768 // 2
    assert line["scaling_weak"]["n_gpus"] == 2


def test_more_gpus_than_the_host_has_fails_loudly():
    """No stub: this container has no GPU, so --gpus 4 must exit non-zero without a JSON line."""
    r = _run(["--gpus", "4", "--steps", "4", "--warmup", "3", "--no-extras", "--no-e2e"])
    assert r.returncode != 0
    assert not _json_lines(r.stdout)
    assert "requested" in r.stderr


def test_world_size_mismatch_is_refused():
    r = _run(["--stub", "--gpus", "2", "--steps", "4"], env_extra={"WORLD_SIZE": "1", "RANK": "0"})
    assert r.returncode != 0
    assert not _json_lines(r.stdout)


def test_reference_arm_with_gpus_n_prints_one_line_without_ranks():
    """The reference arm is rank-0 CPU work: with --gpus N and no launcher it still prints one line."""
    pytest.importorskip("numpy")
    from oracle import pyoracle  # noqa: F401  (test-side: the compiled reference must be present)

    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "liblbmref.so")):
        pytest.skip("oracle/_ref not built")
    r = _run(["--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "1"], timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1 and lines[0]["impl"] == "reference" and lines[0]["n_gpus"] == 2
    assert lines[0]["cpu_baseline"]["physical_cores"]
