"""bench/report.hpp restated (paper_1012_0365_b200/report.py); cases and golden
strings of proj/tests/test_bench.cpp."""
import csv
import io

import pytest

from paper_1012_0365_b200.report import MC, RPCA, ReportRow, emit_table


def sample_rpca_row():
    return ReportRow(problem=RPCA, m=500, method="ADM", rel_err=5.27e-6, rank_hat=50, e_l0=25009, iters=30,
                     time_s=4.07, matvecs=123456)


def parse_csv(text):
    return [r for r in csv.reader(io.StringIO(text)) if r and not r[0].startswith("speedup=")]


def test_csv_header_matches_fixed_schema():
    text = emit_table([sample_rpca_row()], "csv")
    assert text.startswith("m,method,rel_err,rank_hat,e_l0,iters,time_s,matvecs\n")
    cells = parse_csv(text)
    assert len(cells) == 2
    assert cells[1][0] == "500" and cells[1][1] == "ADM" and cells[1][2] == "5.27e-06" and cells[1][4] == "25009"


def test_rejects_empty_and_mixed():
    with pytest.raises(ValueError):
        emit_table([], "csv")
    mc = sample_rpca_row()
    mc.problem = MC
    with pytest.raises(ValueError):
        emit_table([sample_rpca_row(), mc], "csv")


def test_speedup_line_for_baseline_warm_pair():
    base, warm = sample_rpca_row(), sample_rpca_row()
    warm.method, warm.time_s = "BLWS-ADM", 2.035
    assert "speedup=2.00\n" in emit_table([base, warm], "csv")
    assert "speedup=" not in emit_table([base, base], "csv")


def test_nonconverged_rows_add_flag_column():
    bad = sample_rpca_row()
    bad.converged = False
    text = emit_table([bad], "csv")
    assert text.startswith("m,method,rel_err,rank_hat,e_l0,iters,time_s,matvecs,flag\n")
    assert "nonconverged" in text


def test_markdown_layout():
    text = emit_table([sample_rpca_row()], "markdown")
    assert text.startswith("| m | method |") and "| --- |" in text and "| 500 | ADM |" in text


def test_csv_idempotent_through_parse_reemit():
    mc = ReportRow(problem=MC, m=1000, r=10, s_dr=6, s_m2=0.1194, method="BLWS-SVT", rel_err=1.73e-4, iters=123,
                   time_s=20.02, matvecs=98765)
    text = emit_table([mc], "csv")
    c = parse_csv(text)[1]
    back = ReportRow(problem=MC, m=int(c[0]), r=int(c[1]), s_dr=float(c[2]), s_m2=float(c[3]), method=c[4],
                     time_s=float(c[5]), iters=int(c[6]), rel_err=float(c[7]), matvecs=int(c[8]))
    assert emit_table([back], "csv") == text


def test_csv_escape_quotes():
    row = sample_rpca_row()
    row.method = 'B,L"W'
    assert '"B,L""W"' in emit_table([row], "csv")
