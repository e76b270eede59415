"""The device bench matrix in the reference's CSV schema v1 (proj/tests/test_bench_matrix.cpp,
acceptance.cpp C7/C8 analogues)."""
import io

import pytest

HEADER = ("schema_version,kernel,layout,vl,workers,lx,ly,iterations,warmup,traffic_model,"
          "flops_per_site,t_iter_s,t_min_s,mlups,gbps,gflops,clock_res_ns,status")


def test_csv_header_matches_reference_schema():
    """acceptance.cpp:240-243 (exact header) and the energy variant (metrics.cpp:100-106)."""
    from paper_1804_01918_b200 import bench_matrix as bm
    out = io.StringIO()
    bm.write_csv_header(out, False)
    assert out.getvalue() == HEADER + "\n"
    out = io.StringIO()
    bm.write_csv_header(out, True)
    assert out.getvalue().endswith(",energy_pkg_j,energy_dram_j,energy_total_j,avg_power_w,status\n")


def test_row_format_and_derived_metrics():
    """6 significant digits; derived columns recompute exactly from the row (acceptance C7)."""
    from paper_1804_01918_b200 import bench_matrix as bm
    import paper_1804_01918_b200 as lbm
    r = bm.BenchReport("step", "caosoa", 32, 1, 1024, 8192, 50, 5, t_iter_s=0.0012345678, t_min_s=0.0012)
    bm.finalize_metrics(r)
    assert r.mlups == lbm.mlups(1024, 8192, r.t_iter_s)
    assert r.gbps == lbm.propagate_gbps(1024, 8192, 37, r.t_iter_s, "nt") * 2
    assert r.gflops == lbm.collide_gflops(1024, 8192, 1522.0, r.t_iter_s)
    out = io.StringIO()
    bm.write_csv_row(out, r, False)
    cols = out.getvalue().strip().split(",")
    assert len(cols) == len(HEADER.split(","))
    assert cols[:11] == ["1", "step", "caosoa", "32", "1", "1024", "8192", "50", "5", "nt", "1522"]
    assert cols[11] == "0.00123457" and cols[-1] == "ok"
    p = bm.BenchReport("propagate", "soa", 1, 1, 8, 16, 1, 0, t_iter_s=1e-3)
    bm.finalize_metrics(p)
    assert p.gflops == 0.0
    out = io.StringIO()
    bm.write_csv_row(out, p, True)  # energy columns requested but no energy: four empty fields
    assert ",,,,ok" in out.getvalue()


@pytest.mark.gpu
def test_bench_matrix_on_device(gpu):
    """Full grid with three kernel rows per cell; a failing cell is recorded and the run continues."""
    from paper_1804_01918_b200 import bench_matrix as bm
    import paper_1804_01918_b200 as lbm
    csv, log = io.StringIO(), io.StringIO()
    reports = bm.run_bench_matrix(8, 16, vls=[8], iterations=2, warmup=1, energy=True, csv=csv, log=log)
    assert len(reports) == 4 * 3
    ok = [r for r in reports if r.status == "ok"]
    bad = [r for r in reports if r.status != "ok"]
    assert {r.layout for r in ok} == {"aos", "soa"} and {r.layout for r in bad} == {"csoa", "caosoa"}
    lines = [ln for ln in csv.getvalue().splitlines() if ln]
    assert len(lines) == len(reports) + 1
    for r in ok:
        assert r.t_iter_s > 0 and r.mlups == lbm.mlups(r.lx, r.ly, r.t_iter_s)
    csv = io.StringIO()
    reports = bm.run_bench_matrix(64, 128, vls=[4], iterations=3, warmup=1, csv=csv, log=io.StringIO())
    assert all(r.status == "ok" for r in reports)
    trend = io.StringIO()
    bm.write_trend_summary(trend, reports)
    assert "propagate csoa/aos bandwidth ratio" in trend.getvalue()
    assert "collide caosoa/soa throughput ratio" in trend.getvalue()
