"""Brute-force oracle and verifier (oracle.hpp:26-111).

* CPU: compare() counts missing / extra / duplicates / boundary-band pairs
  like oracle.hpp:65-104.
* GPU: rhg_naive_edges (all pairs by the direct distance formula) on the
  reference's points equals the reference's naive_edges up to pairs within
  1e-9 R of the threshold (glibc vs CUDA libm), and verify_against_oracle
  (generate on the GPU, diff against the GPU brute force on the generator's
  own vertex stream) passes like the reference's `rhg verify`.
"""
import numpy as np
import pytest

import paper_1710_07565_b200 as rhg
from oracle.refbind import ref_available


def test_compare_counts():
    gen = np.array([[1, 2], [2, 1], [3, 4], [5, 6]], np.uint64)  # (1,2) twice -> one duplicate
    orc = np.array([[1, 2], [3, 4], [7, 8]], np.uint64)
    rep = rhg.compare(gen, orc)
    assert (rep.missing, rep.extra, rep.duplicates, rep.boundary_band) == (1, 1, 1, 0)
    assert not rep.clean()
    assert rhg.compare(orc, orc[::-1]).clean()


def test_compare_boundary_band():
    class P:  # two points exactly at distance R (same angle: d = r2 - r1)
        r = np.array([1.0, 3.0, 0.5])
        theta = np.array([0.0, 0.0, 0.0])
    R = 2.0
    rep = rhg.compare(np.array([[0, 1]], np.uint64), np.zeros((0, 2), np.uint64), P, R)
    assert (rep.extra, rep.boundary_band) == (0, 1) and rep.clean()
    rep = rhg.compare(np.array([[0, 2]], np.uint64), np.zeros((0, 2), np.uint64), P, R)
    assert rep.extra == 1


def test_verify_guard():
    p = rhg.ModelParams.from_avg_degree(100001, 1.0, 8.0, 1, 4)
    with pytest.raises(ValueError, match="100000"):
        rhg.verify_against_oracle(p)


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", [(2000, 1.0, 16.0, 3, 8), (5000, 0.55, 4.0, 11, 2), (20000, 0.8, 16.0, 5, 4)])
def test_gpu_naive_matches_reference_naive(oracle, cfg):
    if not ref_available():
        pytest.skip("oracle/_ref not built")
    from oracle.refbind import Ref
    ref = Ref()
    p = rhg.ModelParams.from_avg_degree(*cfg)
    pts = oracle.points(p.n, p.alpha, p.C, p.seed, p.chunks)
    got = rhg.naive_edges(pts, p.R)
    want = ref.naive_edges(p.n, p.alpha, p.C, p.seed, p.chunks)
    rep = rhg.compare(got, want, pts, p.R)
    assert rep.clean(), rep


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", [(2000, 1.0, 16.0, 3, 8), (10000, 0.75, 16.0, 7, 4), (50000, 0.6, 8.0, 2, 8),
                                 (100000, 1.0, 16.0, 1, 8)])
def test_verify_against_oracle_passes(cfg):
    rep = rhg.verify_against_oracle(rhg.ModelParams.from_avg_degree(*cfg))
    assert rep.clean(), rep
    assert rep.boundary_band <= 2
