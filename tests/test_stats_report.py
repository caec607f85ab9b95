"""The CLI `stats` path (proj/tools/rhg.cpp:144-164, stats.hpp:37-208):
per-annulus counters, exact degrees, the power-law MLE and the run report.

* CPU: powerlaw_mle is bit-identical to the reference's (same order, same libm) and fails
  like it below 100 tail samples; the report formats doubles like std::ostream.
* GPU (same points): ChunkStats::{edges,comps,vertices}_by_annulus equal the reference's
  exactly (sweep.hpp:530-539: the node's annulus; generator.hpp:89: the global unit's
  larger annulus), shard arrays sum to the whole, and gamma_hat from the exact degrees
  equals the reference's.
"""
import numpy as np
import pytest

import paper_1710_07565_b200 as rhg
from oracle.refbind import ref_available


@pytest.fixture(scope="module")
def ref():
    if not ref_available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    from oracle.refbind import Ref
    return Ref()


@pytest.mark.parametrize("seed,a", [(1, 2.5), (2, 2.1), (3, 3.5)])
def test_powerlaw_mle_bit_identical(ref, seed, a):
    d = np.random.default_rng(seed).zipf(a, 200000).astype(np.uint32)
    for d_min in (1, 5, 10, 40):
        if (d >= d_min).sum() < 100:
            with pytest.raises(ValueError):
                rhg.powerlaw_mle(d, d_min)
            continue
        assert rhg.powerlaw_mle(d, d_min) == ref.powerlaw_mle(d, d_min)


def test_powerlaw_mle_needs_100_tail_samples():
    d = np.array([50] * 99 + [1] * 1000, np.uint32)
    with pytest.raises(ValueError, match="fewer than 100"):
        rhg.powerlaw_mle(d, 10)
    assert np.isfinite(rhg.powerlaw_mle(np.append(d, 60).astype(np.uint32), 10))


def test_degree_histogram():
    h = rhg.degree_histogram([0, 2, 2, 5])
    assert list(h) == [1, 0, 2, 0, 0, 1]


def test_report_formats_like_ostream():
    rep = rhg.RunReport(n=10, m=3, avg_degree=0.6, expected_avg_degree=123456789.0, gamma_hat=float("nan"),
                        overestimation_ratio=1e-05, r_G=2.0)
    row = rep.csv_row().strip().split(",")
    assert row[:5] == ["10", "3", "0.6", "1.23457e+08", "nan"] and row[6] == "1e-05" and row[9] == "2"
    assert rep.text().startswith("n=10\nm=3\navg_degree=0.6\n")


@pytest.mark.gpu
@pytest.mark.parametrize("n,d,g,seed,P", [(20000, 16.0, 2.6, 5, 4), (200000, 64.0, 2.2, 7, 16),
                                          (100000, 8.0, 3.0, 2, 8), (1 << 20, 16.0, 3.0, 1, 8)])
def test_annulus_counters_same_points(oracle, ref, n, d, g, seed, P):
    p = rhg.ModelParams.from_avg_degree(n, rhg.alpha_from_gamma(g), d, seed, P)
    pts = oracle.points(p.n, p.alpha, p.C, p.seed, p.chunks)
    st = rhg.count_edges_from_points(p, pts, degrees=True)  # the stats path counts per annulus
    e, c, v = ref.generate_annuli(p.n, p.alpha, p.C, p.seed, p.chunks)
    assert st.total.edges_by_annulus == [int(x) for x in e]
    assert st.total.comps_by_annulus == [int(x) for x in c]
    assert st.total.vertices_by_annulus == [int(x) for x in v]
    assert sum(st.total.edges_by_annulus) == st.total.edges and sum(st.total.comps_by_annulus) == st.total.comps


@pytest.mark.gpu
def test_annulus_counters_shards_sum(oracle):
    p = rhg.ModelParams.from_avg_degree(40000, 0.8, 12.0, 11, 14)
    whole = rhg.generate_stats(p, degrees=True).total
    parts = [rhg.generate_stats(p, rhg.GenOptions(rank=r, world=3), degrees=True).total for r in range(3)]
    assert rhg.generate_stats(p).total.edges_by_annulus == []  # counters-only path
    for f in ("edges_by_annulus", "comps_by_annulus", "vertices_by_annulus"):
        assert [sum(x) for x in zip(*[getattr(t, f) for t in parts])] == getattr(whole, f), f


@pytest.mark.gpu
def test_stats_report_gamma_hat_matches_reference(oracle, ref):
    p = rhg.ModelParams.from_avg_degree(200000, rhg.alpha_from_gamma(2.6), 16.0, 3, 8)
    pts = oracle.points(p.n, p.alpha, p.C, p.seed, p.chunks)
    st = rhg.count_edges_from_points(p, pts, degrees=True)
    want = ref.generate_stats(p.n, p.alpha, p.C, p.seed, p.chunks, degrees=True)["degrees"]
    assert np.array_equal(st.degrees, want)
    d_min = 16
    assert rhg.powerlaw_mle(st.degrees, d_min) == ref.powerlaw_mle(want, d_min)
    rep = rhg.stats_report(p)
    assert rep.m == rhg.generate_stats(p).total.edges and np.isfinite(rep.gamma_hat)
    assert "annulus_edges=" in rep.text()
