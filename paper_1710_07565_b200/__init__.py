"""B200-native threshold random hyperbolic graph generator (sm_100a).

Host-side mirror of the reference's stats-only generator interface
(/root/reference/proj/include/rhg/geometry.hpp, generator.hpp): same names,
same argument meaning, same exceptions (ValueError for the reference's
std::invalid_argument, RuntimeError for std::logic_error).  All work runs in
librhg_b200.so (C ABI, include/rhg_b200.h) on the GPU; there is no CPU path.

    >>> import paper_1710_07565_b200 as rhg
    >>> p = rhg.ModelParams.from_avg_degree(1 << 20, rhg.alpha_from_gamma(3.0), 16.0, seed=1, chunks=8)
    >>> st = rhg.generate_stats(p)
    >>> st.total.edges, st.total.fingerprint
"""
from __future__ import annotations

import contextlib
import ctypes as C
import math
import threading
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _native
from ._native import RHG_OK, RhgCudaError, check, lib

__all__ = ["alpha_from_gamma", "gamma_from_alpha", "radial_const_from_avg_degree", "radius_from_size",
           "expected_avg_degree", "ModelParams", "AnnulusLayout", "make_layout", "GenOptions", "ChunkStats", "RunStats", "generate_stats",
           "sample_points", "sample_uniforms", "fp64_peak", "count_edges_from_points", "Points", "RhgCudaError", "two_pi", "libm_eval", "LIBM_FUNCTIONS", "nccl_unique_id", "attach_comm", "shard_extent", "ShardExtent", "audit_predicate", "unit_stats", "generate_edges_units"]

two_pi = 6.283185307179586476925286766559  # geometry.hpp:11


def alpha_from_gamma(gamma: float) -> float:
    """geometry.hpp:35-39 — raises ValueError unless gamma > 2."""
    out = C.c_double()
    check(lib().rhg_alpha_from_gamma(float(gamma), C.byref(out)))
    return out.value


def gamma_from_alpha(alpha: float) -> float:
    """geometry.hpp:41-45."""
    if not alpha > 0.5:
        raise ValueError("gamma_from_alpha: alpha must be > 1/2")
    return 2.0 * alpha + 1.0


def radial_const_from_avg_degree(d_bar: float, alpha: float) -> float:
    """geometry.hpp:26-33 — the C that yields average degree d_bar."""
    out = C.c_double()
    check(lib().rhg_radial_const_from_avg_degree(float(d_bar), float(alpha), C.byref(out)))
    return out.value


def radius_from_size(n: float, C_: float) -> float:
    """geometry.hpp:14-17: R = 2 ln n + C."""
    return 2.0 * math.log(n) + C_


def expected_avg_degree(C_: float, alpha: float) -> float:
    """geometry.hpp:20-23 (leading order)."""
    q = alpha / (alpha - 0.5)
    return 2.0 / math.pi * q * q * math.exp(-C_ / 2.0)


class ModelParams:
    """geometry.hpp:49-73: (n, alpha, C, seed, chunks) pin the graph; R derived."""

    __slots__ = ("n", "alpha", "C", "R", "seed", "chunks")

    def __init__(self, n: int, alpha: float, C_: float, seed: int, chunks: int):
        p = _native.rhg_params(int(n), float(alpha), float(C_), int(seed), int(chunks), 0.0)
        if int(n) < 0 or int(chunks) < 0 or int(chunks) >= 1 << 32:
            raise ValueError("ModelParams: n and chunks must be non-negative integers")
        check(lib().rhg_params_validate(C.byref(p)))
        self.n, self.alpha, self.C, self.R, self.seed, self.chunks = p.n, p.alpha, p.C, p.R, p.seed, p.chunks

    @classmethod
    def from_avg_degree(cls, n: int, alpha: float, d_bar: float, seed: int, chunks: int) -> "ModelParams":
        return cls(n, alpha, radial_const_from_avg_degree(d_bar, alpha), seed, chunks)

    def _c(self) -> _native.rhg_params:
        return _native.rhg_params(self.n, self.alpha, self.C, self.seed, self.chunks, self.R)

    def __repr__(self):
        return (f"ModelParams(n={self.n}, alpha={self.alpha!r}, C={self.C!r}, seed={self.seed}, "
                f"chunks={self.chunks}, R={self.R!r})")


@dataclass
class AnnulusLayout:
    """partition.hpp:22-82 (the graph-defining part): annulus vertex counts, the
    per-(annulus, chunk) counts and first vertex ids, classes (0 clique, 1 global,
    2 streaming), the first streaming annulus."""
    count: int
    first_streaming: int
    counts: np.ndarray        # [count] uint64
    chunk_counts: np.ndarray  # [count, chunks] uint64
    id_base: np.ndarray       # [count, chunks] uint64
    classes: np.ndarray       # [count] uint8


def make_layout(params: ModelParams) -> AnnulusLayout:
    """partition.hpp:233-240: the host layout the generator samples from (no GPU needed)."""
    p = params._c()
    k, fs = C.c_uint32(), C.c_uint32()
    check(lib().rhg_layout(C.byref(p), C.byref(k), C.byref(fs), None, None, None, None))
    n = k.value
    counts = np.zeros(n, np.uint64)
    cc = np.zeros(n * params.chunks, np.uint64)
    ib = np.zeros(n * params.chunks, np.uint64)
    cls = np.zeros(n, np.uint8)
    u64 = C.POINTER(C.c_uint64)
    check(lib().rhg_layout(C.byref(p), C.byref(k), C.byref(fs), counts.ctypes.data_as(u64), cc.ctypes.data_as(u64),
                           ib.ctypes.data_as(u64), cls.ctypes.data_as(C.POINTER(C.c_uint8))))
    return AnnulusLayout(n, fs.value, counts, cc.reshape(n, params.chunks), ib.reshape(n, params.chunks), cls)


@dataclass
class GenOptions:
    """generator.hpp:27-32.  `workers` and `cell_target` are accepted for
    interface parity; neither changes the graph (the reference guarantees the
    same).  `device` picks the GPU; `rank`/`world` select an engine shard
    (chunks [rank*P/world, (rank+1)*P/world)) for multi-GPU runs."""
    workers: int = 0
    cell_target: int = 8
    device: int = 0
    rank: int = 0
    world: int = 1
    # GenOptions.workers mapped to GPUs (generator.hpp:245-268): a tuple of several devices runs
    # the whole graph on all of them from this process (rhg_create_multi; NCCL all-reduce)
    devices: Optional[tuple] = None


@dataclass
class ChunkStats:
    """sweep.hpp:154-177 (max_insertion_bucket is a sweep internal, not produced).
    edges_by_annulus / comps_by_annulus are filled when degrees are tracked (the `stats`
    path) or edges are materialised; the counters-only path leaves them empty."""
    edges: int = 0
    comps: int = 0
    streaming_vertices: int = 0
    fingerprint: int = 0
    edges_by_annulus: list = field(default_factory=list)
    comps_by_annulus: list = field(default_factory=list)
    vertices_by_annulus: list = field(default_factory=list)


@dataclass
class RunStats:
    """generator.hpp:34-46, plus device timing of this call."""
    n: int = 0
    global_vertices: int = 0
    r_G: float = 0.0
    total: ChunkStats = field(default_factory=ChunkStats)
    seconds: float = 0.0
    R: float = 0.0
    annuli: int = 0
    first_streaming: int = 0
    global_edges: int = 0
    global_comps: int = 0
    device_ms: float = 0.0
    sample_ms: float = 0.0
    edges_ms: float = 0.0
    host_ms: float = 0.0
    kernel_launches: int = 0
    device_bytes: int = 0
    h2d_bytes: int = 0
    d2h_bytes: int = 0
    pairs_ms: float = 0.0
    stream_comps: int = 0
    dense_comps: int = 0
    reduced_world: int = 0  # >= 1: counters are the whole graph's (NCCL all-reduce over that many shards)
    degrees: Optional[np.ndarray] = None

    def avg_degree(self) -> float:
        return 2.0 * self.total.edges / self.n if self.n else 0.0

    def overestimation_ratio(self) -> float:
        return self.total.comps / max(self.total.edges, 1)

    @classmethod
    def _from_c(cls, s: _native.rhg_run_stats) -> "RunStats":
        k = int(s.annuli)
        return cls(n=s.n, global_vertices=s.global_vertices, r_G=s.r_G,
                   total=ChunkStats(s.edges, s.comps, s.streaming_vertices, s.fingerprint,
                                    list(s.annulus_edges[:k]) if s.per_annulus else [],
                                    list(s.annulus_comps[:k]) if s.per_annulus else [],
                                    list(s.annulus_vertices[:k])), seconds=s.seconds,
                   R=s.R, annuli=s.annuli, first_streaming=s.first_streaming, global_edges=s.global_edges,
                   global_comps=s.global_comps, device_ms=s.device_ms, sample_ms=s.sample_ms, edges_ms=s.edges_ms,
                   host_ms=s.host_ms, kernel_launches=s.kernel_launches, device_bytes=s.device_bytes,
                   h2d_bytes=s.h2d_bytes, d2h_bytes=s.d2h_bytes, pairs_ms=s.pairs_ms,
                   stream_comps=s.stream_comps, dense_comps=s.dense_comps, reduced_world=s.reduced_world)


class _Context:
    """One rhg_ctx (CUDA streams + device buffers) per device -- or per device tuple for a
    multi-GPU context -- reused across calls.  A context is not re-entrant (rhg_b200.h), so
    every library call holds the context's lock (ctypes releases the GIL during the call)."""

    _lock = threading.Lock()
    _ctx: dict = {}

    @classmethod
    def _key(cls, opts) -> tuple:
        if isinstance(opts, int):
            return (int(opts),)
        if opts.devices:  # a multi-GPU context, even over one device
            return ("multi",) + tuple(int(d) for d in opts.devices)
        return (int(opts.device),)

    @classmethod
    def _entry(cls, key: tuple):
        with cls._lock:
            e = cls._ctx.get(key)
            if e is None:
                h = C.c_void_p()
                if key[0] != "multi":
                    check(lib().rhg_create(key[0], C.byref(h)))
                else:
                    devs = key[1:]
                    arr = (C.c_int * len(devs))(*devs)
                    check(lib().rhg_create_multi(len(devs), arr, C.byref(h)))
                e = (h, threading.Lock())
                cls._ctx[key] = e
            return e

    @classmethod
    def get(cls, opts) -> C.c_void_p:
        return cls._entry(cls._key(opts))[0]

    @classmethod
    @contextlib.contextmanager
    def use(cls, opts):
        h, lk = cls._entry(cls._key(opts))
        with lk:
            yield h

    @classmethod
    def release_all(cls):
        with cls._lock:
            for h, lk in cls._ctx.values():
                with lk:
                    lib().rhg_destroy(h)
            cls._ctx.clear()


def _shard(opts: GenOptions) -> _native.rhg_shard:
    return _native.rhg_shard(int(opts.rank), int(opts.world))


def generate_stats(params: ModelParams, opts: GenOptions = GenOptions(), degrees: bool = False) -> RunStats:
    """generator.hpp:219-291: edge count, wrapping Σ(u+v) fingerprint and
    distance computations of the graph (or of this shard), on the GPU.  With
    degrees=True, RunStats.degrees is the exact u32 per-vertex degree."""
    st = _native.rhg_run_stats()
    deg = np.zeros(params.n, np.uint32) if degrees else None
    with _Context.use(opts) as ctx:
        check(lib().rhg_generate_stats(ctx, C.byref(params._c()), C.byref(_shard(opts)), C.byref(st),
                                       deg.ctypes.data_as(C.POINTER(C.c_uint32)) if degrees else None))
    out = RunStats._from_c(st)
    out.degrees = deg
    return out


def audit_predicate(params: ModelParams, opts: GenOptions = GenOptions()):
    """Predicate audit (rhg_audit_predicate): one generate_stats in which the slab join also
    evaluates the reference predicate (sweep.hpp:531-533) for every pair its FP32 pre-filter
    decided.  Returns (report dict, RunStats); report["disagreements"] must be 0."""
    rep = _native.rhg_audit_report()
    st = _native.rhg_run_stats()
    with _Context.use(opts) as ctx:
        check(lib().rhg_audit_predicate(ctx, C.byref(params._c()), C.byref(_shard(opts)), C.byref(rep),
                                        C.byref(st)))
    return {f: getattr(rep, f) for f, _ in _native.rhg_audit_report._fields_}, RunStats._from_c(st)


def nccl_unique_id() -> bytes:
    """A fresh NCCL unique id (128 bytes) for attach_comm; create it on rank 0 and share it."""
    buf = (C.c_uint8 * 128)()
    check(lib().rhg_nccl_unique_id(buf))
    return bytes(buf)


def attach_comm(world: int, rank: int, uid: bytes, device: int = 0) -> None:
    """Give this process's context on `device` an NCCL communicator (rank of world, one process
    per GPU).  Afterwards generate_stats with GenOptions(rank=rank, world=world) ends with the
    device-side counter all-reduce and returns the whole graph (RunStats.reduced_world = world)."""
    if len(uid) != 128:
        raise ValueError("attach_comm: the NCCL unique id has 128 bytes")
    buf = (C.c_uint8 * 128).from_buffer_copy(uid)
    with _Context.use(device) as ctx:
        check(lib().rhg_attach_comm(ctx, int(world), int(rank), buf))


@dataclass
class ShardExtent:
    """The host-side shard plan (rhg_shard_extent): owned engines (angular chunks) and points."""
    chunk_begin: int
    chunk_end: int
    owned_points: int
    halo_points: int
    global_points: int
    sampled_points: int
    device_point_bytes: int


def shard_extent(params: ModelParams, rank: int = 0, world: int = 1) -> ShardExtent:
    """Which chunks and how many points rank `rank` of `world` draws (no GPU needed)."""
    out = _native.rhg_shard_info()
    check(lib().rhg_shard_extent(C.byref(params._c()), C.byref(_native.rhg_shard(int(rank), int(world))),
                                 C.byref(out)))
    return ShardExtent(*[int(getattr(out, f)) for f, _ in _native.rhg_shard_info._fields_])


@dataclass
class Points:
    """All n vertices in id order (PointDraw fields, sweep.hpp:89-97)."""
    beta: np.ndarray
    r: np.ndarray
    theta: np.ndarray
    half_width: np.ndarray
    coth_r: np.ndarray
    inv_sinh_r: np.ndarray
    cos_theta: np.ndarray
    sin_theta: np.ndarray

    FIELDS = ("beta", "r", "theta", "half_width", "coth_r", "inv_sinh_r", "cos_theta", "sin_theta")

    def _c(self) -> _native.rhg_points:
        arrs = {}
        for k in self.FIELDS:
            a = getattr(self, k)
            if a is None:
                arrs[k] = None
                continue
            if a.dtype != np.float64 or not a.flags.c_contiguous:
                a = np.ascontiguousarray(a, np.float64)
                setattr(self, k, a)
            arrs[k] = a.ctypes.data_as(_native.P_f64)
        return _native.rhg_points(*[arrs[k] for k in self.FIELDS])


def sample_points(params: ModelParams, opts: GenOptions = GenOptions()) -> Points:
    """The device sampler's point set (ChunkPointSource streams, sweep.hpp:102-141)."""
    pts = Points(*[np.empty(params.n, np.float64) for _ in Points.FIELDS])
    with _Context.use(opts) as ctx:
        check(lib().rhg_sample_points(ctx, C.byref(params._c()), C.byref(pts._c())))
    return pts


def sample_uniforms(params: ModelParams, opts: GenOptions = GenOptions()):
    """Raw MT19937-64 uniforms of every point's (angle, radius) streams, id order."""
    ua, ur = np.empty(params.n, np.float64), np.empty(params.n, np.float64)
    with _Context.use(opts) as ctx:
        check(lib().rhg_sample_uniforms(ctx, C.byref(params._c()), ua.ctypes.data_as(_native.P_f64),
                                        ur.ctypes.data_as(_native.P_f64)))
    return ua, ur


def fp64_peak(device: int = 0):
    """Measured non-FMA FP64 DMUL+DADD rate (ops/s), dependent-DMUL latency (cycles), probe ms."""
    a, b, c = C.c_double(), C.c_double(), C.c_double()
    check(lib().rhg_fp64_peak(int(device), C.byref(a), C.byref(b), C.byref(c)))
    return a.value, b.value, c.value


LIBM_FUNCTIONS = ("exp", "log", "log1p", "acosh", "acos", "pow", "sin", "cos")


def libm_eval(fn: str, x, y=None, device: int = 0):
    """The device restatement of the glibc 2.39 routine `fn` (csrc/glibc_libm.cuh; one of
    LIBM_FUNCTIONS, "sin"/"cos" being the outputs of one sincos call) on array x (and y for
    pow), elementwise on `device`.  Equal to the host glibc bit for bit (tests/test_gpu_libm.py)."""
    code = LIBM_FUNCTIONS.index(fn)
    xa = np.ascontiguousarray(x, dtype=np.float64)
    ya = None
    if fn == "pow":
        ya = np.ascontiguousarray(y, dtype=np.float64)
        if ya.shape != xa.shape:
            raise ValueError("pow: x and y must have the same shape")
    out = np.empty_like(xa)
    P = C.POINTER(C.c_double)
    check(lib().rhg_libm_eval(int(device), code, xa.ctypes.data_as(P),
                              ya.ctypes.data_as(P) if ya is not None else None, out.ctypes.data_as(P), xa.size))
    return out


def count_edges_from_points(params: ModelParams, points, opts: GenOptions = GenOptions(),
                            degrees: bool = False) -> RunStats:
    """Parity hook: run the device edge kernels on a given point set (any
    object with the Points fields; r optional)."""
    pts = Points(*[getattr(points, k, None) for k in Points.FIELDS])
    for k in Points.FIELDS:
        a = getattr(pts, k)
        if k != "r" and (a is None or len(a) != params.n):
            raise ValueError(f"count_edges_from_points: field {k} must have n entries")
    st = _native.rhg_run_stats()
    deg = np.zeros(params.n, np.uint32) if degrees else None
    with _Context.use(opts) as ctx:
        check(lib().rhg_count_edges_from_points(ctx, C.byref(params._c()), C.byref(_shard(opts)),
                                                C.byref(pts._c()), C.byref(st),
                                                deg.ctypes.data_as(C.POINTER(C.c_uint32)) if degrees else None))
    out = RunStats._from_c(st)
    out.degrees = deg
    return out


# ------------------------------------------------------- edge streams ---
# the materialised edge stream (generator.hpp:135-215
# generate(params, opts, edge sink)) and its file formats (io.hpp:20-96).

def _edges_call(fn, params: ModelParams, opts: GenOptions, *pre):
    with _Context.use(opts) as ctx:
        return _edges_call_locked(ctx, fn, params, opts, *pre)


def _edges_call_locked(ctx, fn, params: ModelParams, opts: GenOptions, *pre):
    st = _native.rhg_run_stats()
    m = C.c_uint64(0)
    est = expected_avg_degree(params.C, params.alpha) * params.n / 2.0 / max(1, opts.world)
    cap = int(est * 1.25) + 4096
    for _ in range(2):
        buf = np.empty((cap, 2), np.uint64)
        rc = fn(ctx, C.byref(params._c()), C.byref(_shard(opts)), *pre, C.byref(st),
                buf.ctypes.data_as(C.POINTER(C.c_uint64)), cap, C.byref(m))
        if rc == _native.RHG_INVALID_ARGUMENT and m.value > cap:
            cap = int(m.value)  # the estimate was low: rerun with the exact count
            continue
        check(rc)
        return buf[: m.value], RunStats._from_c(st)
    raise RuntimeError("generate_edges: edge count changed between runs")


def generate_edges(params: ModelParams, opts: GenOptions = GenOptions()):
    """Every edge of the graph (or of this shard) as a (m, 2) uint64 array of
    canonical pairs u < v, sorted by (u, v), plus the RunStats of the run.
    The reference's generate() emits the same multiset in its unit order."""
    return _edges_call(lib().rhg_generate_edges, params, opts)


def generate_edges_units(params: ModelParams, opts: GenOptions = GenOptions()):
    """generate() in the reference's unit order (generator.hpp:183-199): the global unit's edges,
    then chunk engine 0, 1, ... (canonical u < v; (u, v) order inside a unit).  Returns the
    (m, 2) uint64 edge array and the unit offsets (chunks + 2 entries)."""
    P64 = C.POINTER(C.c_uint64)
    offs = np.zeros(params.chunks + 2, np.uint64)
    m = C.c_uint64(0)
    with _Context.use(opts) as ctx:
        check(lib().rhg_generate_edges_units(ctx, C.byref(params._c()), None, 0, C.byref(m),
                                             offs.ctypes.data_as(P64)))
        buf = np.empty((m.value, 2), np.uint64)
        check(lib().rhg_generate_edges_units(ctx, C.byref(params._c()), buf.ctypes.data_as(P64), m.value,
                                             C.byref(m), offs.ctypes.data_as(P64)))
    return buf, offs


def unit_stats(params: ModelParams, opts: GenOptions = GenOptions()):
    """RunStats::unit_edges / unit_comps / unit_vertices (generator.hpp:270-284): unit 0 = the
    global unit, unit c + 1 = chunk engine c.  Returns three lists of chunks + 1 entries."""
    P64 = C.POINTER(C.c_uint64)
    e, c, v = (np.zeros(params.chunks + 1, np.uint64) for _ in range(3))
    with _Context.use(opts) as ctx:
        check(lib().rhg_unit_stats(ctx, C.byref(params._c()), e.ctypes.data_as(P64), c.ctypes.data_as(P64),
                                   v.ctypes.data_as(P64)))
    return [int(x) for x in e], [int(x) for x in c], [int(x) for x in v]


def edges_from_points(params: ModelParams, points, opts: GenOptions = GenOptions()):
    """generate_edges for a GIVEN point set ("same points" mode)."""
    pts = Points(*[getattr(points, k, None) for k in Points.FIELDS])
    return _edges_call(lib().rhg_edges_from_points, params, opts, C.byref(pts._c()))


def _io_check(rc: int) -> None:
    if rc != RHG_OK:
        raise ValueError(lib().rhg_io_last_error().decode())


def _edge_ptr(edges):
    e = np.ascontiguousarray(edges, np.uint64).reshape(-1, 2)
    return e, e.ctypes.data_as(C.POINTER(C.c_uint64))


def write_edges_text(path: str, edges) -> None:
    """io.hpp TextEdgeWriter: one "u v" line per edge (decimal)."""
    e, p = _edge_ptr(edges)
    _io_check(lib().rhg_write_edges_text(str(path).encode(), p, len(e)))


def write_edges_binary(path: str, edges) -> None:
    """io.hpp BinaryEdgeWriter: magic "RHGE0001" then little-endian u64 pairs."""
    e, p = _edge_ptr(edges)
    _io_check(lib().rhg_write_edges_binary(str(path).encode(), p, len(e)))


def read_edges_binary(path: str) -> np.ndarray:
    """io.hpp read_binary_edges (bad magic / truncated pair raise ValueError)."""
    m = C.c_uint64(0)
    _io_check(lib().rhg_read_edges_binary(str(path).encode(), None, 0, C.byref(m)))
    buf = np.empty((m.value, 2), np.uint64)
    _io_check(lib().rhg_read_edges_binary(str(path).encode(), buf.ctypes.data_as(C.POINTER(C.c_uint64)), m.value,
                                          C.byref(m)))
    return buf


# ------------------------------------------------- brute-force oracle ---
# the vertex stream (sample_points) and the brute-force
# verifier of oracle.hpp:26-111, with the quadratic all-pairs check on the GPU.

NAIVE_ORACLE_GUARD = 100000  # oracle.hpp:41


def naive_edges(points, R: float, device: int = 0) -> np.ndarray:
    """oracle.hpp:44-54 on the GPU: all pairs u < v (sorted) of the points
    (id order; fields r, theta) with hyperbolic_distance < R."""
    r = np.ascontiguousarray(points.r, np.float64)
    th = np.ascontiguousarray(points.theta, np.float64)
    n = len(r)
    m = C.c_uint64(0)
    P64 = C.POINTER(C.c_uint64)
    with _Context.use(device) as ctx:
        check(lib().rhg_naive_edges(ctx, n, float(R), r.ctypes.data_as(_native.P_f64),
                                    th.ctypes.data_as(_native.P_f64), None, 0, C.byref(m)))
        buf = np.empty((m.value, 2), np.uint64)
        check(lib().rhg_naive_edges(ctx, n, float(R), r.ctypes.data_as(_native.P_f64),
                                    th.ctypes.data_as(_native.P_f64), buf.ctypes.data_as(P64), m.value, C.byref(m)))
    return buf


def hyperbolic_distance(r1, t1, r2, t2):
    """geometry.hpp:117-123 (host, float64, vectorised; canonical r1 <= r2)."""
    a, b = np.minimum(r1, r2), np.maximum(r1, r2)
    arg = np.cosh(b - a) + (1.0 - np.cos(np.abs(t1 - t2))) * np.sinh(a) * np.sinh(b)
    return np.where(arg <= 1.0, 0.0, np.arccosh(np.maximum(arg, 1.0)))


@dataclass
class CompareReport:
    """oracle.hpp:60-63."""
    missing: int = 0
    extra: int = 0
    duplicates: int = 0
    boundary_band: int = 0

    def clean(self) -> bool:
        return self.missing == 0 and self.extra == 0 and self.duplicates == 0


def compare(generated, oracle_edges, points=None, R: float = 0.0) -> CompareReport:
    """oracle.hpp:65-104: exact multiset diff of two edge streams; mismatches
    within 1e-9 R of the threshold count as boundary_band, not as errors."""
    def canon(e):
        e = np.asarray(e, np.uint64).reshape(-1, 2)
        lo, hi = np.minimum(e[:, 0], e[:, 1]), np.maximum(e[:, 0], e[:, 1])
        return lo.astype(np.uint64), hi.astype(np.uint64)

    rep = CompareReport()
    glo, ghi = canon(generated)
    olo, ohi = canon(oracle_edges)
    if (len(ghi) and ghi.max() >= 2**32) or (len(ohi) and ohi.max() >= 2**32):
        raise ValueError("compare: vertex ids must be < 2^32")
    g = np.sort((glo << np.uint64(32)) | ghi)  # one 64-bit key per edge
    o = np.unique((olo << np.uint64(32)) | ohi)
    gu, gc = np.unique(g, return_counts=True)
    rep.duplicates = int((gc - 1).sum())
    only_g = np.setdiff1d(gu, o, assume_unique=True)
    only_o = np.setdiff1d(o, gu, assume_unique=True)

    def band(keys):
        if points is None or R <= 0.0 or len(keys) == 0:
            return np.zeros(len(keys), bool)
        keys = np.asarray(keys, dtype=np.uint64)
        u, v = keys >> np.uint64(32), keys & np.uint64(0xFFFFFFFF)
        d = hyperbolic_distance(points.r[u], points.theta[u], points.r[v], points.theta[v])
        return np.abs(d - R) < 1e-9 * R

    bg, bo = band(only_g), band(only_o)
    rep.boundary_band = int(bg.sum() + bo.sum())
    rep.extra = int((~bg).sum())
    rep.missing = int((~bo).sum())
    return rep


def verify_against_oracle(params: ModelParams, opts: GenOptions = GenOptions()) -> CompareReport:
    """oracle.hpp:106-111: generate with params, diff against the brute-force
    oracle on the generator's own vertex stream (both on the GPU)."""
    if params.n > NAIVE_ORACLE_GUARD:
        raise ValueError("verify_against_oracle: refusing quadratic work above n = 100000")
    edges, _ = generate_edges(params, opts)
    pts = sample_points(params, opts)
    return compare(edges, naive_edges(pts, params.R, opts.device), pts, params.R)


# ------------------------------------------------- degree analytics ---
# the CLI `stats` path (proj/tools/rhg.cpp:144-164) — exact degrees
# (generate_stats(degrees=True)), the power-law fit and the run report (stats.hpp:37-208).

def degree_histogram(degrees) -> np.ndarray:
    """stats.hpp:48-56: hist[d] = number of vertices of degree d."""
    d = np.asarray(degrees, np.uint32)
    return np.bincount(d, minlength=int(d.max()) + 1 if len(d) else 1).astype(np.uint64)


def powerlaw_mle(degrees, d_min: int) -> float:
    """stats.hpp:58-75 (bit-identical: the library sums in id order with glibc log, like the
    reference).  Fewer than 100 tail samples raise ValueError (std::invalid_argument)."""
    d = np.ascontiguousarray(degrees, np.uint32)
    g = C.c_double()
    rc = lib().rhg_powerlaw_mle(d.ctypes.data_as(C.POINTER(C.c_uint32)), len(d), int(d_min), C.byref(g))
    if rc != RHG_OK:
        raise ValueError(lib().rhg_io_last_error().decode())
    return g.value


def _fmt(x) -> str:
    """std::ostream default formatting of a double (%g, 6 significant digits)."""
    if isinstance(x, float):
        if math.isnan(x):
            return "nan" if math.copysign(1.0, x) > 0 else "-nan"
        if math.isinf(x):
            return "inf" if x > 0 else "-inf"
        return f"{x:g}"
    return str(x)


@dataclass
class RunReport:
    """stats.hpp:120-208: the flat run summary of `rhg stats`, per-unit vectors included
    (unit_stats: the P engine shards)."""
    n: int = 0
    m: int = 0
    avg_degree: float = 0.0
    expected_avg_degree: float = 0.0
    gamma_hat: float = float("nan")
    distance_computations: int = 0
    overestimation_ratio: float = 0.0
    fingerprint: int = 0
    global_vertices: int = 0
    r_G: float = 0.0
    seconds: float = 0.0
    edges_per_sec: float = 0.0
    annulus_edges: list = field(default_factory=list)
    annulus_comps: list = field(default_factory=list)
    annulus_vertices: list = field(default_factory=list)
    unit_edges: list = field(default_factory=list)
    unit_comps: list = field(default_factory=list)
    unit_vertices: list = field(default_factory=list)

    @classmethod
    def from_stats(cls, params: ModelParams, stats: RunStats) -> "RunReport":
        return cls(n=params.n, m=stats.total.edges, avg_degree=stats.avg_degree(),
                   expected_avg_degree=expected_avg_degree(params.C, params.alpha),
                   distance_computations=stats.total.comps, overestimation_ratio=stats.overestimation_ratio(),
                   fingerprint=stats.total.fingerprint, global_vertices=stats.global_vertices, r_G=stats.r_G,
                   seconds=stats.seconds,
                   edges_per_sec=stats.total.edges / stats.seconds if stats.seconds > 0 else 0.0,
                   annulus_edges=list(stats.total.edges_by_annulus),
                   annulus_comps=list(stats.total.comps_by_annulus),
                   annulus_vertices=list(stats.total.vertices_by_annulus))

    CSV_HEADER = ("n,m,avg_degree,expected_avg_degree,gamma_hat,distance_computations,overestimation_ratio,"
                  "fingerprint,global_vertices,r_G,seconds,edges_per_sec")

    def csv_row(self) -> str:
        return ",".join(_fmt(v) for v in (self.n, self.m, float(self.avg_degree), float(self.expected_avg_degree),
                                          float(self.gamma_hat), self.distance_computations,
                                          float(self.overestimation_ratio), self.fingerprint, self.global_vertices,
                                          float(self.r_G), float(self.seconds), float(self.edges_per_sec))) + "\n"

    def text(self) -> str:
        j = lambda v: ",".join(str(int(x)) for x in v)  # noqa: E731
        return (f"n={self.n}\nm={self.m}\navg_degree={_fmt(float(self.avg_degree))}\n"
                f"expected_avg_degree={_fmt(float(self.expected_avg_degree))}\n"
                f"gamma_hat={_fmt(float(self.gamma_hat))}\ndistance_computations={self.distance_computations}\n"
                f"overestimation_ratio={_fmt(float(self.overestimation_ratio))}\nfingerprint={self.fingerprint}\n"
                f"global_vertices={self.global_vertices}\nr_G={_fmt(float(self.r_G))}\n"
                f"seconds={_fmt(float(self.seconds))}\nedges_per_sec={_fmt(float(self.edges_per_sec))}\n"
                f"annulus_vertices={j(self.annulus_vertices)}\nannulus_comps={j(self.annulus_comps)}\n"
                f"annulus_edges={j(self.annulus_edges)}\nunit_edges={j(self.unit_edges)}\n"
                f"unit_comps={j(self.unit_comps)}\n")


def stats_report(params: ModelParams, opts: GenOptions = GenOptions(), units: bool = True) -> RunReport:
    """proj/tools/rhg.cpp:144-164 cmd_stats: generate with exact degrees, fit gamma_hat over
    the degrees >= d_min = max(10, round(expected average degree)) (NaN when the tail has fewer
    than 100 samples) and build the run report.  units=True also fills the per-unit vectors
    (P extra engine-shard runs; whole-graph reports only)."""
    st = generate_stats(params, opts, degrees=True)
    rep = RunReport.from_stats(params, st)
    if units and opts.world == 1:
        rep.unit_edges, rep.unit_comps, rep.unit_vertices = unit_stats(params, opts)
    d_min = int(max(10.0, float(math.floor(rep.expected_avg_degree + 0.5))))  # std::llround (x > 0)
    try:
        rep.gamma_hat = powerlaw_mle(st.degrees, d_min)
    except ValueError:
        pass
    return rep
