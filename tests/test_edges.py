"""Materialised edge stream: generator.hpp:135-215
generate(params, opts, edge sink) and the io.hpp:20-96 file formats.

* CPU: the library's text / binary writers are byte-identical to the
  reference's TextEdgeWriter / BinaryEdgeWriter (compiled from the reference
  headers, oracle/_ref), each side reads the other's binary files, and bad
  magic / truncated pairs fail like read_binary_edges.
* GPU (same points): rhg_edges_from_points on the reference's point set
  returns exactly the reference generate()'s edge multiset (sorted), and the
  text file written from it equals the reference writer's bytes on the
  sorted reference stream.
* GPU (device sampler): the edge list agrees with the run's own counters
  (m, wrapping sum(u+v)), with the same-points path on the device's points,
  and shard lists partition the whole.
"""
import os

import numpy as np
import pytest

import paper_1710_07565_b200 as rhg
from oracle.refbind import ref_available


def canon_sorted(e):
    e = np.asarray(e, np.uint64).reshape(-1, 2)
    lo, hi = np.minimum(e[:, 0], e[:, 1]), np.maximum(e[:, 0], e[:, 1])
    o = np.lexsort((hi, lo))
    return np.stack([lo[o], hi[o]], axis=1)


EDGES = np.array([[0, 1], [0, 2], [7, 9], [123456789, 987654321], [2**40 + 3, 2**41 + 5], [2**63, 2**64 - 1]],
                 np.uint64)


@pytest.fixture(scope="module")
def ref():
    if not ref_available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    from oracle.refbind import Ref
    return Ref()


@pytest.mark.parametrize("binary", [False, True])
@pytest.mark.parametrize("edges", [EDGES, EDGES[:0], EDGES[:1]])
def test_writers_byte_identical_to_reference(tmp_path, ref, edges, binary):
    ours, theirs = tmp_path / "ours", tmp_path / "theirs"
    (rhg.write_edges_binary if binary else rhg.write_edges_text)(ours, edges)
    ref.write_edges(theirs, edges, binary)
    assert ours.read_bytes() == theirs.read_bytes()


def test_binary_round_trip_both_ways(tmp_path, ref):
    a, b = tmp_path / "a.bin", tmp_path / "b.bin"
    rhg.write_edges_binary(a, EDGES)
    ref.write_edges(b, EDGES, True)
    assert np.array_equal(ref.read_edges_binary(a), EDGES)
    assert np.array_equal(rhg.read_edges_binary(b), EDGES)


def test_read_binary_errors(tmp_path):
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"RHGE0002" + b"\0" * 16)
    with pytest.raises(ValueError, match="bad magic"):
        rhg.read_edges_binary(bad)
    tr = tmp_path / "tr.bin"
    tr.write_bytes(b"RHGE0001" + b"\0" * 20)
    with pytest.raises(ValueError, match="truncated pair"):
        rhg.read_edges_binary(tr)
    empty = tmp_path / "empty.bin"
    empty.write_bytes(b"RHGE0001")
    assert rhg.read_edges_binary(empty).shape == (0, 2)


def test_text_format_is_decimal_lines(tmp_path):
    p = tmp_path / "e.txt"
    rhg.write_edges_text(p, EDGES)
    lines = p.read_text().splitlines()
    assert [tuple(map(int, l.split(" "))) for l in lines] == [tuple(int(x) for x in r) for r in EDGES]


# ------------------------------------------------------------------ GPU ---

def _params(n, alpha, d, seed, P):
    return rhg.ModelParams.from_avg_degree(n, alpha, d, seed, P)


@pytest.mark.gpu
@pytest.mark.parametrize("names", [{"grid"}, {"n1", "n2", "more_chunks_than_points"}, {"odd_P", "smoke"}])
def test_same_points_edges_equal_reference_generate(oracle, ref, golden, names):
    rows = [s for s in golden["stats"] if s["name"] in names and s["n"] <= 20000]
    assert rows
    for s in rows:
        p = rhg.ModelParams(s["n"], s["alpha"], float.fromhex(s["C"]), s["seed"], s["P"])
        pts = oracle.points(p.n, p.alpha, p.C, p.seed, p.chunks)
        got, st = rhg.edges_from_points(p, pts)
        want = canon_sorted(ref.generate_edges(p.n, p.alpha, p.C, p.seed, p.chunks))
        assert got.dtype == np.uint64 and got.shape == want.shape, s
        assert np.array_equal(got, want), s
        assert len(got) == st.total.edges == s["edges"]
        assert np.all(got[:, 0] < got[:, 1])


@pytest.mark.gpu
def test_same_points_edges_cfg1_and_text_bytes(oracle, ref, tmp_path):
    """BASELINE configs[0] (n=2^20, d=16, gamma=3, seed=1, P=8): 8.4 M edges."""
    p = _params(1 << 20, 1.0, 16.0, 1, 8)
    pts = oracle.points(p.n, p.alpha, p.C, p.seed, p.chunks)
    got, st = rhg.edges_from_points(p, pts)
    want = canon_sorted(ref.generate_edges(p.n, p.alpha, p.C, p.seed, p.chunks))
    assert np.array_equal(got, want)
    a, b = tmp_path / "ours.txt", tmp_path / "ref.txt"
    rhg.write_edges_text(a, got)
    ref.write_edges(b, want, False)
    assert a.read_bytes() == b.read_bytes()


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", [(20000, 0.8, 16.0, 5, 4), (1 << 18, 0.6, 64.0, 7, 16)])
def test_device_edges_consistent(cfg):
    p = _params(*cfg)
    got, st = rhg.generate_edges(p)
    stats = rhg.generate_stats(p)
    assert len(got) == st.total.edges == stats.total.edges
    assert int(got.sum(dtype=np.uint64)) % 2**64 == stats.total.fingerprint
    assert np.all(got[:, 0] < got[:, 1])
    assert np.all(np.diff(got[:, 0].astype(np.int64)) >= 0)
    again, _ = rhg.edges_from_points(p, rhg.sample_points(p))
    assert np.array_equal(got, again)


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_shard_edges_partition_the_graph(world):
    p = _params(20000, 0.8, 16.0, 5, 6)
    whole, _ = rhg.generate_edges(p)
    parts = [rhg.generate_edges(p, rhg.GenOptions(rank=r, world=world))[0] for r in range(world)]
    assert np.array_equal(canon_sorted(np.concatenate(parts)), whole)


@pytest.mark.gpu
def test_edges_buffer_regrows_when_the_estimate_is_low(monkeypatch):
    p = _params(20000, 0.8, 16.0, 5, 4)
    want, _ = rhg.generate_edges(p)
    monkeypatch.setattr(rhg, "expected_avg_degree", lambda C_, a: 0.0)  # estimate -> 4096 pairs
    got, _ = rhg.generate_edges(p)
    assert np.array_equal(got, want)
