"""TEST INFRASTRUCTURE ONLY — ctypes bindings to the checkers under oracle/.

* ``Ref``    — oracle/_ref/librhg_ref.so: the UNMODIFIED reference headers
               (/root/reference/proj/include) compiled in place by
               oracle/Makefile, wrapped by oracle/ref_harness.cpp.
* ``Oracle`` — oracle/liboracle.so: the plain-C restatement (rhg_oracle.c).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and the
``--impl reference`` arm) may import this module.  The product package never
does.
"""
from __future__ import annotations

import ctypes as C
import ctypes as C_
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "librhg_ref.so")
ORACLE_SO = os.path.join(HERE, "liboracle.so")

u64 = C.c_uint64
u32 = C.c_uint32
f64 = C.c_double
P_u64 = C.POINTER(C.c_uint64)
P_u32 = C.POINTER(C.c_uint32)
P_f64 = C.POINTER(C.c_double)
P_u8 = C.POINTER(C.c_uint8)


def _p(a, t):
    return a.ctypes.data_as(t) if a is not None else None


@dataclass
class Layout:
    count: int
    lower: np.ndarray
    upper: np.ndarray
    probs: np.ndarray
    cosh_alpha_lower: np.ndarray
    cosh_alpha_upper: np.ndarray
    coth_lower: np.ndarray
    coshR_inv_sinh_lower: np.ndarray
    cell_width: np.ndarray
    counts: np.ndarray
    chunk_counts: np.ndarray  # [count, chunks]
    id_base: np.ndarray  # [count, chunks]
    cells: np.ndarray
    classes: np.ndarray
    R: float
    cosh_R: float
    r_G: float
    first_streaming: int


@dataclass
class Points:
    beta: np.ndarray
    r: np.ndarray
    theta: np.ndarray
    half_width: np.ndarray
    coth_r: np.ndarray
    inv_sinh_r: np.ndarray
    cos_theta: np.ndarray
    sin_theta: np.ndarray
    annulus: np.ndarray


class _Base:
    def _check(self, rc):
        if rc != 0:
            msg = self.lib_last_error().decode()
            if rc == 1:
                raise ValueError(msg)
            raise RuntimeError(msg)


class Ref(_Base):
    """The reference itself (compiled in place)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (make -C oracle)")
        L = C.CDLL(path)
        self.L = L
        L.ref_last_error.restype = C.c_char_p
        self.lib_last_error = L.ref_last_error
        L.ref_radial_const_from_avg_degree.argtypes = [f64, f64, P_f64]
        L.ref_alpha_from_gamma.argtypes = [f64, P_f64]
        L.ref_generate_stats.argtypes = [u64, f64, f64, u64, u32, u32, P_u64, P_f64, P_u32]
        L.ref_generate_units.argtypes = [u64, f64, f64, u64, u32, u32, P_u64, P_u64]
        L.ref_layout.argtypes = [u64, f64, f64, u64, u32, P_u32, P_f64, P_u64, P_u64, P_u64, P_u64, P_u8, P_f64]
        L.ref_points.argtypes = [u64, f64, f64, u64, u32, u32] + [P_f64] * 8 + [P_u32]
        L.ref_generate_edges.argtypes = [u64, f64, f64, u64, u32, u32, P_u64, P_u64]
        L.ref_naive_edges.argtypes = [u64, f64, f64, u64, u32, P_u64, P_u64]
        L.ref_write_edges.argtypes = [C.c_char_p, P_u64, u64, C.c_int]
        L.ref_generate_annuli.argtypes = [u64, f64, f64, u64, u32, u32, P_u64, P_u64, P_u64]
        L.ref_powerlaw_mle.argtypes = [P_u32, u64, u32, P_f64]
        L.ref_read_edges_binary.argtypes = [C.c_char_p, P_u64, P_u64]
        L.ref_derive_seed.argtypes = [u64, P_u64, u32]
        L.ref_derive_seed.restype = u64
        L.ref_mt_outputs.argtypes = [u64, u64, P_u64]
        L.ref_sorted_uniforms.argtypes = [u64, f64, f64, u64, P_u64, u32, P_f64]
        L.ref_binomial.argtypes = [u64, f64, u64]
        L.ref_binomial.restype = u64

    # geometry.hpp:26-39
    def radial_const_from_avg_degree(self, d_bar, alpha):
        out = f64()
        self._check(self.L.ref_radial_const_from_avg_degree(d_bar, alpha, C.byref(out)))
        return out.value

    def alpha_from_gamma(self, gamma):
        out = f64()
        self._check(self.L.ref_alpha_from_gamma(gamma, C.byref(out)))
        return out.value

    def generate_stats(self, n, alpha, Cc, seed, chunks, workers=0, degrees=False):
        out = np.zeros(8, np.uint64)
        outd = np.zeros(4, np.float64)
        deg = np.zeros(n, np.uint32) if degrees else None
        self._check(self.L.ref_generate_stats(n, alpha, Cc, seed, chunks, workers, _p(out, P_u64),
                                              _p(outd, P_f64), _p(deg, P_u32)))
        res = dict(edges=int(out[0]), fingerprint=int(out[1]), comps=int(out[2]), global_vertices=int(out[3]),
                   streaming_vertices=int(out[4]), annuli=int(out[5]), first_streaming=int(out[6]),
                   R=float(outd[0]), r_G=float(outd[1]), seconds=float(outd[2]), cosh_R=float(outd[3]))
        if degrees:
            res["degrees"] = deg
        return res

    def generate_units(self, n, alpha, Cc, seed, chunks, workers=0):
        e = np.zeros(chunks + 1, np.uint64)
        c = np.zeros(chunks + 1, np.uint64)
        self._check(self.L.ref_generate_units(n, alpha, Cc, seed, chunks, workers, _p(e, P_u64), _p(c, P_u64)))
        return e, c

    def layout(self, n, alpha, Cc, seed, chunks) -> Layout:
        cnt = u32()
        self._check(self.L.ref_layout(n, alpha, Cc, seed, chunks, C.byref(cnt), None, None, None, None, None,
                                      None, None))
        k = cnt.value
        dbl = np.zeros(8 * k, np.float64)
        counts = np.zeros(k, np.uint64)
        cc = np.zeros(k * chunks, np.uint64)
        ib = np.zeros(k * chunks, np.uint64)
        cells = np.zeros(k, np.uint64)
        cls = np.zeros(k, np.uint8)
        scal = np.zeros(4, np.float64)
        self._check(self.L.ref_layout(n, alpha, Cc, seed, chunks, C.byref(cnt), _p(dbl, P_f64), _p(counts, P_u64),
                                      _p(cc, P_u64), _p(ib, P_u64), _p(cells, P_u64), _p(cls, P_u8),
                                      _p(scal, P_f64)))
        d = dbl.reshape(8, k)
        return Layout(k, d[0], d[1], d[2], d[3], d[4], d[5], d[6], d[7], counts, cc.reshape(k, chunks),
                      ib.reshape(k, chunks), cells, cls, float(scal[0]), float(scal[1]), float(scal[2]),
                      int(scal[3]))

    def points(self, n, alpha, Cc, seed, chunks, threads=0) -> Points:
        arrs = [np.empty(n, np.float64) for _ in range(8)]
        ann = np.empty(n, np.uint32)
        self._check(self.L.ref_points(n, alpha, Cc, seed, chunks, threads, *[_p(a, P_f64) for a in arrs],
                                      _p(ann, P_u32)))
        return Points(*arrs, ann)

    def generate_edges(self, n, alpha, Cc, seed, chunks, workers=0):
        m = u64()
        self._check(self.L.ref_generate_edges(n, alpha, Cc, seed, chunks, workers, C.byref(m), None))
        buf = np.zeros(2 * m.value, np.uint64)
        self._check(self.L.ref_generate_edges(n, alpha, Cc, seed, chunks, workers, C.byref(m), _p(buf, P_u64)))
        return buf.reshape(-1, 2)

    def generate_annuli(self, n, alpha, Cc, seed, chunks, workers=0):
        K = self.layout(n, alpha, Cc, seed, chunks).count
        e, c, v = (np.zeros(K, np.uint64) for _ in range(3))
        self._check(self.L.ref_generate_annuli(n, alpha, Cc, seed, chunks, workers, _p(e, P_u64), _p(c, P_u64),
                                               _p(v, P_u64)))
        return e, c, v

    def powerlaw_mle(self, degrees, d_min):
        d = np.ascontiguousarray(degrees, np.uint32)
        g = np.zeros(1, np.float64)
        self._check(self.L.ref_powerlaw_mle(_p(d, P_u32), len(d), d_min, _p(g, P_f64)))
        return float(g[0])

    def write_edges(self, path, edges, binary):
        e = np.ascontiguousarray(edges, np.uint64).reshape(-1, 2)
        self._check(self.L.ref_write_edges(str(path).encode(), _p(e, P_u64), len(e), 1 if binary else 0))

    def read_edges_binary(self, path):
        m = u64()
        self._check(self.L.ref_read_edges_binary(str(path).encode(), C.byref(m), None))
        buf = np.zeros(2 * m.value, np.uint64)
        self._check(self.L.ref_read_edges_binary(str(path).encode(), C.byref(m), _p(buf, P_u64)))
        return buf.reshape(-1, 2)

    def naive_edges(self, n, alpha, Cc, seed, chunks):
        m = u64()
        self._check(self.L.ref_naive_edges(n, alpha, Cc, seed, chunks, C.byref(m), None))
        buf = np.zeros(2 * m.value, np.uint64)
        self._check(self.L.ref_naive_edges(n, alpha, Cc, seed, chunks, C.byref(m), _p(buf, P_u64)))
        return buf.reshape(-1, 2)

    def derive_seed(self, root, comps):
        a = np.asarray(comps, np.uint64)
        return int(self.L.ref_derive_seed(root, _p(a, P_u64), len(a)))

    def mt_outputs(self, seed, count):
        out = np.zeros(count, np.uint64)
        self.L.ref_mt_outputs(seed, count, _p(out, P_u64))
        return out

    def sorted_uniforms(self, count, a, b, root, comps):
        cs = np.asarray(comps, np.uint64)
        out = np.zeros(count, np.float64)
        self.L.ref_sorted_uniforms(count, a, b, root, _p(cs, P_u64), len(cs), _p(out, P_f64))
        return out

    def binomial(self, trials, p, seed):
        return int(self.L.ref_binomial(trials, p, seed))


def ref_available() -> bool:
    return os.path.exists(REF_SO)


class OrcStats(C.Structure):
    _fields_ = [("edges", u64), ("fingerprint", u64), ("comps", u64), ("global_vertices", u64),
                ("streaming_vertices", u64), ("global_edges", u64), ("global_comps", u64), ("annuli", u32),
                ("first_streaming", u32), ("R", f64), ("r_G", f64), ("cosh_R", f64), ("seconds", f64)]

    def asdict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class OrcBorder(C.Structure):
    _fields_ = [(k, u64) for k in ("comps", "edges", "band_pairs", "flips_to_edge", "flips_to_nonedge",
                                   "border_pairs", "listed")] + [("max_flip_dmr", f64), ("seconds", f64)]


class Oracle(_Base):
    """The plain-C restatement (oracle/rhg_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (make -C oracle)")
        L = C.CDLL(path)
        self.L = L
        L.orc_last_error.restype = C.c_char_p
        self.lib_last_error = L.orc_last_error
        L.orc_radial_const_from_avg_degree.argtypes = [f64, f64, P_f64]
        L.orc_alpha_from_gamma.argtypes = [f64, P_f64]
        L.orc_derive_seed.argtypes = [u64, P_u64, u32]
        L.orc_derive_seed.restype = u64
        L.orc_mt_outputs.argtypes = [u64, u64, P_u64]
        L.orc_sorted_uniforms.argtypes = [u64, f64, f64, u64, P_u64, u32, P_f64]
        L.orc_binomial.argtypes = [u64, f64, u64]
        L.orc_binomial.restype = u64
        L.orc_layout.argtypes = [u64, f64, f64, u64, u32, P_u32, P_f64, P_u64, P_u64, P_u64, P_u64, P_u8, P_f64]
        L.orc_points.argtypes = [u64, f64, f64, u64, u32, u32] + [P_f64] * 8 + [P_u32]
        L.orc_generate_stats.argtypes = [u64, f64, f64, u64, u32, u32, C.POINTER(OrcStats), P_u32]
        L.orc_count_edges_from_points.argtypes = [u64, f64, f64, u64, u32, u32] + [P_f64] * 7 + [
            C.POINTER(OrcStats), P_u32]
        L.orc_generate_stats_shard.argtypes = [u64, f64, f64, u64, u32, u32, u32, u32, C.POINTER(OrcStats)]
        L.orc_libm_eval.argtypes = [C.c_int, P_f64, P_f64, P_f64, u64, u32]
        L.orc_borderline.argtypes = [u64, f64, f64, u64, u32, u32, u32, u32, f64, u64, C.POINTER(OrcBorder), P_u64,
                                     P_u64, P_f64, P_u8]
        L.orc_libm_eval.restype = None

    def borderline(self, n, alpha, C, seed, P, rank=0, world=1, band=1e-13, cap=10000, threads=0):
        """Threshold-borderline audit of shard (rank, world) (orc_borderline): counts and the
        listed pairs (u, v, d - R, reference decision) with |d - R| < 1e-12 in binary128."""
        out = OrcBorder()
        u, v = np.zeros(cap, np.uint64), np.zeros(cap, np.uint64)
        dmr, dec = np.zeros(cap, np.float64), np.zeros(cap, np.uint8)
        self._check(self.L.orc_borderline(n, alpha, C, seed, P, rank, world, threads, band, cap, C_.byref(out),
                                          _p(u, P_u64), _p(v, P_u64), _p(dmr, P_f64), _p(dec, P_u8)))
        k = out.listed
        rep = {f: getattr(out, f) for f, _ in OrcBorder._fields_}
        rep["pairs"] = [(int(u[i]), int(v[i]), float(dmr[i]), bool(dec[i])) for i in range(k)]
        return rep

    def libm_eval(self, fn: int, x: np.ndarray, y: np.ndarray | None = None, threads: int | None = None):
        """Host glibc exp/log/log1p/acosh/acos/pow/sin/cos (fn 0..7) elementwise."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        yy = None if y is None else np.ascontiguousarray(y, dtype=np.float64)
        out = np.empty_like(x)
        self.L.orc_libm_eval(fn, _p(x, P_f64), _p(yy, P_f64), _p(out, P_f64), x.size,
                             threads or os.cpu_count() or 1)
        return out

    def radial_const_from_avg_degree(self, d_bar, alpha):
        out = f64()
        self._check(self.L.orc_radial_const_from_avg_degree(d_bar, alpha, C.byref(out)))
        return out.value

    def alpha_from_gamma(self, gamma):
        out = f64()
        self._check(self.L.orc_alpha_from_gamma(gamma, C.byref(out)))
        return out.value

    def derive_seed(self, root, comps):
        a = np.asarray(comps, np.uint64)
        return int(self.L.orc_derive_seed(root, _p(a, P_u64), len(a)))

    def mt_outputs(self, seed, count):
        out = np.zeros(count, np.uint64)
        self.L.orc_mt_outputs(seed, count, _p(out, P_u64))
        return out

    def sorted_uniforms(self, count, a, b, root, comps):
        cs = np.asarray(comps, np.uint64)
        out = np.zeros(count, np.float64)
        self.L.orc_sorted_uniforms(count, a, b, root, _p(cs, P_u64), len(cs), _p(out, P_f64))
        return out

    def binomial(self, trials, p, seed):
        return int(self.L.orc_binomial(trials, p, seed))

    def layout(self, n, alpha, Cc, seed, chunks) -> Layout:
        cnt = u32()
        self._check(self.L.orc_layout(n, alpha, Cc, seed, chunks, C.byref(cnt), None, None, None, None, None,
                                      None, None))
        k = cnt.value
        dbl = np.zeros(8 * k, np.float64)
        counts = np.zeros(k, np.uint64)
        cc = np.zeros(k * chunks, np.uint64)
        ib = np.zeros(k * chunks, np.uint64)
        cells = np.zeros(k, np.uint64)
        cls = np.zeros(k, np.uint8)
        scal = np.zeros(4, np.float64)
        self._check(self.L.orc_layout(n, alpha, Cc, seed, chunks, C.byref(cnt), _p(dbl, P_f64), _p(counts, P_u64),
                                      _p(cc, P_u64), _p(ib, P_u64), _p(cells, P_u64), _p(cls, P_u8),
                                      _p(scal, P_f64)))
        d = dbl.reshape(8, k)
        return Layout(k, d[0], d[1], d[2], d[3], d[4], d[5], d[6], d[7], counts, cc.reshape(k, chunks),
                      ib.reshape(k, chunks), cells, cls, float(scal[0]), float(scal[1]), float(scal[2]),
                      int(scal[3]))

    def points(self, n, alpha, Cc, seed, chunks, threads=0) -> Points:
        arrs = [np.empty(n, np.float64) for _ in range(8)]
        ann = np.empty(n, np.uint32)
        self._check(self.L.orc_points(n, alpha, Cc, seed, chunks, threads, *[_p(a, P_f64) for a in arrs],
                                      _p(ann, P_u32)))
        return Points(*arrs, ann)

    def generate_stats(self, n, alpha, Cc, seed, chunks, threads=0, degrees=False):
        st = OrcStats()
        deg = np.zeros(n, np.uint32) if degrees else None
        self._check(self.L.orc_generate_stats(n, alpha, Cc, seed, chunks, threads, C.byref(st), _p(deg, P_u32)))
        res = st.asdict()
        if degrees:
            res["degrees"] = deg
        return res

    def generate_stats_shard(self, n, alpha, Cc, seed, chunks, rank, world, threads=0):
        st = OrcStats()
        self._check(self.L.orc_generate_stats_shard(n, alpha, Cc, seed, chunks, rank, world, threads, C.byref(st)))
        return st.asdict()

    def count_edges_from_points(self, n, alpha, Cc, seed, chunks, pts: Points, threads=0, degrees=False):
        st = OrcStats()
        deg = np.zeros(n, np.uint32) if degrees else None
        arrs = [np.ascontiguousarray(a, np.float64) for a in
                (pts.beta, pts.theta, pts.half_width, pts.coth_r, pts.inv_sinh_r, pts.cos_theta, pts.sin_theta)]
        self._check(self.L.orc_count_edges_from_points(n, alpha, Cc, seed, chunks, threads,
                                                       *[_p(a, P_f64) for a in arrs], C.byref(st), _p(deg, P_u32)))
        res = st.asdict()
        if degrees:
            res["degrees"] = deg
        return res


def oracle_available() -> bool:
    return os.path.exists(ORACLE_SO)
