"""The reference's units (generator.hpp:183-199, 270-284): unit 0 = the
global unit, unit c + 1 = chunk engine c.

* rhg.unit_stats equals RunStats::unit_edges / unit_comps of the reference (oracle/_ref) and
  its unit_vertices (global vertices, then each chunk's streaming vertices);
* rhg.generate_edges_units is generate()'s stream in unit order: every unit holds exactly the
  reference's edges of that unit (the reference's order inside a unit follows its sweep's
  active-list slots; ours is (u, v) order), and the stats report prints the unit vectors.
"""
import numpy as np
import pytest

import paper_1710_07565_b200 as rhg
from oracle.refbind import ref_available

pytestmark = pytest.mark.gpu

CASES = [(20000, 16.0, 2.6, 5, 4), (50, 6.0, 2.6, 13, 32), (100000, 8.0, 3.0, 2, 7), (1 << 20, 16.0, 3.0, 1, 8)]


@pytest.fixture(scope="module")
def ref():
    if not ref_available():
        pytest.skip("oracle/_ref not built")
    from oracle.refbind import Ref
    return Ref()


def _params(case):
    n, d, g, seed, P = case
    return rhg.ModelParams.from_avg_degree(n, rhg.alpha_from_gamma(g), d, seed, P)


@pytest.mark.parametrize("case", CASES)
def test_unit_stats_equal_reference(ref, oracle, case):
    p = _params(case)
    e, c, v = rhg.unit_stats(p)
    re, rc = ref.generate_units(p.n, p.alpha, p.C, p.seed, p.chunks)
    assert e == [int(x) for x in re] and c == [int(x) for x in rc]
    L = oracle.layout(p.n, p.alpha, p.C, p.seed, p.chunks)
    nG = int(L.counts[:L.first_streaming].sum())
    assert v == [nG] + [int(L.chunk_counts[L.first_streaming:, k].sum()) for k in range(p.chunks)]
    whole = rhg.generate_stats(p)
    assert sum(e) == whole.total.edges and sum(c) == whole.total.comps


@pytest.mark.parametrize("case", CASES[:3])
def test_edges_in_unit_order(ref, case):
    p = _params(case)
    got, offs = rhg.generate_edges_units(p)
    want = ref.generate_edges(p.n, p.alpha, p.C, p.seed, p.chunks)
    re, _ = ref.generate_units(p.n, p.alpha, p.C, p.seed, p.chunks)
    bounds = np.concatenate([[0], np.cumsum(re.astype(np.int64))])
    assert [int(x) for x in offs] == [int(x) for x in bounds]
    for u in range(p.chunks + 1):
        w = want[bounds[u]:bounds[u + 1]]
        w = w[np.lexsort((w[:, 1], w[:, 0]))]
        assert np.array_equal(got[offs[u]:offs[u + 1]], w), u


def test_stats_report_prints_units(ref):
    p = _params(CASES[0])
    rep = rhg.stats_report(p)
    re, rc = ref.generate_units(p.n, p.alpha, p.C, p.seed, p.chunks)
    txt = rep.text()
    assert "unit_edges=" + ",".join(str(int(x)) for x in re) + "\n" in txt
    assert "unit_comps=" + ",".join(str(int(x)) for x in rc) + "\n" in txt
