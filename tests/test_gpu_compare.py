"""Old-vs-new comparison table on the device path (reference harness.py:250-361)
against the golden fixtures of both variants."""

import math

import pytest

from tests.cases import golden, inputs

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,theta_f", [("jump", 1.0 + math.log(4.0)), ("cfg1", 10.0)])
def test_compare_variants_matches_reference(name, theta_f):
    from paper_2501_01676_b200.compare import compare_variants, format_table

    g = golden(name)
    system, part, globs = inputs(name)
    rows = compare_variants(system, part, globs, theta_f, 10.0, name, m=4)
    assert [r.variant for r in rows] == ["old", "new"]
    for r in rows:
        assert r.converged
        assert abs(r.iters - int(g[f"{r.variant}_iterations"])) <= 1
        assert (r.pnumF, r.pnumE) == (int(g[f"{r.variant}_pnumF"]), int(g[f"{r.variant}_pnumE"]))
    text = format_table(rows)
    assert rows[0].cell() in text and rows[1].cell() in text
