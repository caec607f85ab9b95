"""Parity of the B200 path (through the C ABI) with the reference.

* "same points" mode: the device edge kernels run on the reference's point
  set (the oracle's points are bit-identical to the reference's — pinned in
  test_oracle.py) and must reproduce the reference's golden edges,
  fingerprint AND comps exactly, at every golden config that fits a test.
* device sampler: the integer part (SplitMix seed path + MT19937-64 streams)
  is bit-exact; the full device path equals the reference's edge rule (oracle)
  applied to the device's own points, bit for bit.  (The points themselves are
  bitwise the reference's: test_gpu_sampler.py.)
* shards: partial results of world in {2,3,4,7} engine shards sum to the whole.
"""
import numpy as np
import pytest

import paper_1710_07565_b200 as rhg

pytestmark = pytest.mark.gpu


def params_of(s):
    return rhg.ModelParams(s["n"], s["alpha"], float.fromhex(s["C"]), s["seed"], s["P"])


def triple(st):
    return st.total.edges, st.total.fingerprint, st.total.comps


def rows(golden, names, max_n):
    return [s for s in golden["stats"] if s["name"] in names and s["n"] <= max_n]


@pytest.mark.parametrize("names,max_n", [
    ({"grid"}, 2000),
    ({"n1", "n2", "more_chunks_than_points"}, 100),
    ({"odd_P", "smoke"}, 20000),
    ({"cfg1"}, 1 << 20),
])
def test_same_points_parity_golden(oracle, golden, names, max_n):
    for s in rows(golden, names, max_n):
        p = params_of(s)
        pts = oracle.points(p.n, p.alpha, p.C, p.seed, p.chunks)
        st = rhg.count_edges_from_points(p, pts)
        assert triple(st) == (s["edges"], s["fingerprint"], s["comps"]), s
        assert st.global_vertices == s["global_vertices"]


def test_same_points_parity_cfg2(oracle, golden):
    """configs[1] (n=2^24, d=64, gamma=2.2, seed=7) at P=64 — the bench config."""
    s = rows(golden, {"cfg2"}, 1 << 24)[0]
    p = params_of(s)
    pts = oracle.points(p.n, p.alpha, p.C, p.seed, p.chunks)
    st = rhg.count_edges_from_points(p, pts)
    assert triple(st) == (s["edges"], s["fingerprint"], s["comps"])


@pytest.mark.parametrize("world", [2, 3, 4, 7])
def test_shards_sum_to_whole(oracle, world):
    n, alpha, d, seed, P = 40000, 0.8, 12.0, 11, 14
    p = rhg.ModelParams.from_avg_degree(n, alpha, d, seed, P)
    pts = oracle.points(n, alpha, p.C, seed, P)
    whole = oracle.generate_stats(n, alpha, p.C, seed, P)
    acc = [0, 0, 0]
    for r in range(world):
        st = rhg.count_edges_from_points(p, pts, rhg.GenOptions(rank=r, world=world))
        acc = [acc[0] + st.total.edges, (acc[1] + st.total.fingerprint) % 2**64, acc[2] + st.total.comps]
    assert tuple(acc) == (whole["edges"], whole["fingerprint"], whole["comps"])
    # and the device-sampler path shards identically
    full = rhg.generate_stats(p)
    acc = [0, 0, 0]
    for r in range(world):
        st = rhg.generate_stats(p, rhg.GenOptions(rank=r, world=world))
        acc = [acc[0] + st.total.edges, (acc[1] + st.total.fingerprint) % 2**64, acc[2] + st.total.comps]
    assert tuple(acc) == triple(full)


def _mt_uniforms_expected(oracle, p):
    L = oracle.layout(p.n, p.alpha, p.C, p.seed, p.chunks)
    ua = np.empty(p.n)
    ur = np.empty(p.n)
    for i in range(L.count):
        for c in range(p.chunks):
            cnt, base = int(L.chunk_counts[i, c]), int(L.id_base[i, c])
            if not cnt:
                continue
            for phase, out in ((3, ua), (4, ur)):
                x = oracle.mt_outputs(oracle.derive_seed(p.seed, [phase, i, c]), cnt)
                out[base:base + cnt] = (x >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    return ua, ur


@pytest.mark.parametrize("cfg", [(20000, 16.0, 2.6, 5, 4), (200000, 64.0, 2.2, 7, 64), (3000, 8.0, 3.0, 2, 1)])
def test_sampler_uniform_streams_bit_exact(oracle, cfg):
    n, d, g, seed, P = cfg
    p = rhg.ModelParams.from_avg_degree(n, rhg.alpha_from_gamma(g), d, seed, P)
    ua, ur = rhg.sample_uniforms(p)
    ea, er = _mt_uniforms_expected(oracle, p)
    assert np.array_equal(ua.view(np.uint64), ea.view(np.uint64))
    assert np.array_equal(ur.view(np.uint64), er.view(np.uint64))


@pytest.mark.parametrize("cfg", [(20000, 16.0, 2.6, 5, 4), (1 << 20, 16.0, 3.0, 1, 8)])
def test_device_path_equals_edge_rule_on_its_points(oracle, cfg):
    """The full device path (sampler + engines) equals the reference's edge rule (oracle)
    applied to the device's own points; the points themselves are bitwise the reference's
    (test_gpu_sampler.py), and theta = beta + hw (mod 2pi) exactly."""
    n, d, g, seed, P = cfg
    alpha = rhg.alpha_from_gamma(g)
    p = rhg.ModelParams.from_avg_degree(n, alpha, d, seed, P)
    dev = rhg.sample_points(p)
    th = dev.beta + dev.half_width
    th = np.where(th >= rhg.two_pi, th - rhg.two_pi, th)
    assert np.array_equal(th, dev.theta)
    want = oracle.count_edges_from_points(n, alpha, p.C, seed, P, dev)
    got = rhg.generate_stats(p)
    assert triple(got) == (want["edges"], want["fingerprint"], want["comps"])


def test_degrees_exact(oracle):
    n, alpha, d, seed, P = 50000, 0.75, 16.0, 3, 8
    p = rhg.ModelParams.from_avg_degree(n, alpha, d, seed, P)
    pts = oracle.points(n, alpha, p.C, seed, P)
    want = oracle.generate_stats(n, alpha, p.C, seed, P, degrees=True)
    got = rhg.count_edges_from_points(p, pts, degrees=True)
    assert np.array_equal(got.degrees, want["degrees"])
    got2 = rhg.generate_stats(p, degrees=True)
    assert int(got2.degrees.sum()) == 2 * got2.total.edges


def test_repeatable_and_context_reuse():
    p = rhg.ModelParams.from_avg_degree(300000, 0.8, 16.0, 9, 16)
    a = rhg.generate_stats(p)
    b = rhg.generate_stats(rhg.ModelParams.from_avg_degree(1000, 0.8, 16.0, 9, 2))
    c = rhg.generate_stats(p)
    assert triple(a) == triple(c) and a.total.edges > 0 and b.total.edges > 0
    assert a.kernel_launches > 0 and a.device_ms > 0


@pytest.mark.parametrize("n,alpha,C,seed,P", [(1 << 20, 1.0, 8.0, 3, 8), (1 << 18, 0.6, 10.0, 5, 4),
                                              (1 << 19, 0.8, 4.0, 9, 16)])
def test_same_points_parity_large_R(oracle, n, alpha, C, seed, P):
    """R = 2 ln n + C up to 35: outer-annulus windows fall below the FP64 rounding floor, so
    the slab join runs those groups on the exact predicate and the FP32 pre-filter leaves
    many pairs to the exact recheck — the counters must stay bit-exact."""
    p = rhg.ModelParams(n, alpha, C, seed, P)
    pts = oracle.points(n, alpha, C, seed, P)
    want = oracle.generate_stats(n, alpha, C, seed, P)
    st = rhg.count_edges_from_points(p, pts)
    assert triple(st) == (want["edges"], want["fingerprint"], want["comps"])
    dev = rhg.sample_points(p)
    want2 = oracle.count_edges_from_points(n, alpha, C, seed, P, dev)
    assert triple(rhg.generate_stats(p)) == (want2["edges"], want2["fingerprint"], want2["comps"])


def test_counter_modes_agree(oracle, golden):
    """The counters-only kernels (MODE 0), the degree/per-annulus kernels (MODE 1) and the
    edge-stream kernels (MODE 2) are separate instantiations: all must give the golden counters."""
    for s in rows(golden, {"grid"}, 2000)[::3]:
        p = params_of(s)
        pts = oracle.points(p.n, p.alpha, p.C, p.seed, p.chunks)
        want = (s["edges"], s["fingerprint"], s["comps"])
        assert triple(rhg.count_edges_from_points(p, pts)) == want, s
        assert triple(rhg.count_edges_from_points(p, pts, degrees=True)) == want, s
        _, st = rhg.edges_from_points(p, pts)
        assert triple(st) == want, s
