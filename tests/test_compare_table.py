"""Comparison-table formatting and CSV round trip (host logic; reference
harness.py:310-381)."""

from paper_2501_01676_b200.compare import ResultRow, emit_tables, format_table, parse_results_csv


def _rows():
    return [ResultRow("test1 m=4", "old", 8, 4, 8, 5, 14, 0.1, 0.2, 0.3, True),
            ResultRow("test1 m=4", "new", 8, 4, 12, 5, 0, 0.1, 0.2, 0.4, True),
            ResultRow("random n=3 m=4", "old", 27, 4, 12, 93, 228, 1.0, 2.0, 3.0, True),
            ResultRow("random n=3 m=4", "new", 27, 4, 13, 93, 65, 1.0, 2.0, 3.5, False)]


def test_format_table_layout():
    text = format_table(_rows())
    lines = text.splitlines()
    assert lines[0].split() == ["case", "N", "m", "old", "t_old[s]", "new", "t_new[s]"]
    assert "8(5,14)" in lines[1] and "12(5,0)" in lines[1] and "0.50" in lines[1]
    assert "12(93,228)" in lines[2] and "13(93,65)*" in lines[2]
    assert lines[-1] == "(* did not reach the residual tolerance)"


def test_csv_round_trip(tmp_path):
    rows = _rows()
    csv_path, txt_path = emit_tables(rows, tmp_path)
    back = parse_results_csv(csv_path)
    assert [(r.case, r.variant, r.iters, r.pnumF, r.pnumE, r.converged) for r in back] == \
        [(r.case, r.variant, r.iters, r.pnumF, r.pnumE, r.converged) for r in rows]
    assert txt_path.read_text() == format_table(back)
