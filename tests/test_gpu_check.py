"""GPU `check` / `traffic` commands (paper_2501_06480_b200/check.py)."""

import pytest

pytestmark = pytest.mark.gpu

chk = pytest.importorskip("paper_2501_06480_b200.check")


def test_check_suite_small_grid_all_pass():
    res = chk.run_check_suite(42, [1, 8, 49], [16, 32], ["1", "2", "auto"])
    table = chk.render_suite_table(res)
    assert all(r.ok for r in res), table
    ids = {r.case_id for r in res}
    assert "roundtrip_224x224x3_k7" in ids and "fwd_L49_C32_r2" in ids and "bwd_L49_C32_r1" in ids
    assert "invariance_L49_C32" in ids


def test_check_suite_capacity_cases_refuse():
    # a 4 KB arena cannot hold L=49's S block: every case must be an expected CapacityError
    res = chk.run_check_suite(42, [49], [32], ["1"], capacity_bytes=4096)
    caps = [r for r in res if r.case_id.startswith("capacity_")]
    assert caps and all(r.ok for r in caps)


def test_traffic_report_lines():
    out = chk.run_traffic(49, 32, 2, "f16")
    assert "instrumented counts match closed form: yes" in out
    assert "forward moves 12544 B/unit" in out
    assert "forward kernel tc" in out


def test_cli_main_exit_codes(capsys):
    assert chk.main(["check", "--L", "8", "--C", "16", "--r", "1"]) == 0
    assert "cases passed" in capsys.readouterr().out
    assert chk.main(["traffic", "--L", "144", "--C", "32"]) == 0
    assert "B200 f16" in capsys.readouterr().out
