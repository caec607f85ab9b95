"""ctypes binding of include/rhg_b200.h (librhg_b200.so, built in-tree).

The library is the product: a missing or unloadable .so is an error, never a
silent fallback.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# RHG_LIB_PATH: an alternative build of the same library (A/B timing experiments only)
LIB_PATH = os.environ.get("RHG_LIB_PATH") or os.path.join(HERE, "librhg_b200.so")

RHG_OK, RHG_INVALID_ARGUMENT, RHG_INVARIANT, RHG_CUDA, RHG_NOMEM = range(5)


class rhg_params(C.Structure):
    _fields_ = [("n", C.c_uint64), ("alpha", C.c_double), ("C", C.c_double), ("seed", C.c_uint64),
                ("chunks", C.c_uint32), ("R", C.c_double)]


class rhg_shard(C.Structure):
    _fields_ = [("rank", C.c_uint32), ("world", C.c_uint32)]


class rhg_run_stats(C.Structure):
    _fields_ = [("n", C.c_uint64), ("edges", C.c_uint64), ("fingerprint", C.c_uint64), ("comps", C.c_uint64),
                ("global_vertices", C.c_uint64), ("streaming_vertices", C.c_uint64), ("global_edges", C.c_uint64),
                ("global_comps", C.c_uint64), ("annuli", C.c_uint32), ("first_streaming", C.c_uint32),
                ("R", C.c_double), ("r_G", C.c_double), ("cosh_R", C.c_double), ("device_ms", C.c_double),
                ("sample_ms", C.c_double), ("edges_ms", C.c_double), ("host_ms", C.c_double),
                ("seconds", C.c_double), ("kernel_launches", C.c_uint64), ("device_bytes", C.c_uint64),
                ("h2d_bytes", C.c_uint64), ("d2h_bytes", C.c_uint64), ("pairs_ms", C.c_double),
                ("stream_comps", C.c_uint64), ("dense_comps", C.c_uint64),
                ("per_annulus", C.c_uint32), ("pad_", C.c_uint32), ("annulus_edges", C.c_uint64 * 64), ("annulus_comps", C.c_uint64 * 64),
                ("annulus_vertices", C.c_uint64 * 64), ("reduced_world", C.c_uint32), ("pad2_", C.c_uint32)]


class rhg_audit_report(C.Structure):
    _fields_ = [(k, C.c_uint64) for k in ("slab_pairs", "prefilter_decided", "exact_recheck", "exact_only",
                                          "disagreements", "noise_band_pairs", "exact_engine_pairs")] + [
        ("max_err_over_tau", C.c_double)]


class rhg_shard_info(C.Structure):
    _fields_ = [("chunk_begin", C.c_uint32), ("chunk_end", C.c_uint32), ("owned_points", C.c_uint64),
                ("halo_points", C.c_uint64), ("global_points", C.c_uint64), ("sampled_points", C.c_uint64),
                ("device_point_bytes", C.c_uint64)]


P_f64 = C.POINTER(C.c_double)


class rhg_points(C.Structure):
    _fields_ = [(k, P_f64) for k in
                ("beta", "r", "theta", "half_width", "coth_r", "inv_sinh_r", "cos_theta", "sin_theta")]


class RhgCudaError(RuntimeError):
    """CUDA / device failure (RHG_CUDA)."""


EXPORTS = ["rhg_last_error", "rhg_abi_version", "rhg_alpha_from_gamma", "rhg_radial_const_from_avg_degree",
           "rhg_params_validate", "rhg_params_from_avg_degree", "rhg_create", "rhg_destroy", "rhg_generate_stats",
           "rhg_sample_points", "rhg_sample_uniforms", "rhg_count_edges_from_points",
           "rhg_fp64_peak", "rhg_generate_edges", "rhg_edges_from_points", "rhg_write_edges_text", "rhg_write_edges_binary",
           "rhg_read_edges_binary", "rhg_io_last_error", "rhg_naive_edges", "rhg_powerlaw_mle", "rhg_layout",
           "rhg_libm_eval", "rhg_create_multi", "rhg_context_devices", "rhg_nccl_unique_id", "rhg_attach_comm",
           "rhg_shard_extent", "rhg_audit_predicate", "rhg_unit_stats", "rhg_generate_edges_units"]

_lib = None


def lib():
    """Load librhg_b200.so once; raise if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: build it with `make -C paper_1710_07565_b200/csrc` "
                          "(or __graft_entry__.build()); there is no CPU fallback")
    L = C.CDLL(LIB_PATH)
    L.rhg_last_error.restype = C.c_char_p
    L.rhg_abi_version.restype = C.c_int
    L.rhg_alpha_from_gamma.argtypes = [C.c_double, P_f64]
    L.rhg_radial_const_from_avg_degree.argtypes = [C.c_double, C.c_double, P_f64]
    L.rhg_params_validate.argtypes = [C.POINTER(rhg_params)]
    L.rhg_params_from_avg_degree.argtypes = [C.c_uint64, C.c_double, C.c_double, C.c_uint64, C.c_uint32,
                                             C.POINTER(rhg_params)]
    L.rhg_create.argtypes = [C.c_int, C.POINTER(C.c_void_p)]
    L.rhg_destroy.argtypes = [C.c_void_p]
    L.rhg_destroy.restype = None
    L.rhg_generate_stats.argtypes = [C.c_void_p, C.POINTER(rhg_params), C.POINTER(rhg_shard),
                                     C.POINTER(rhg_run_stats), C.POINTER(C.c_uint32)]
    L.rhg_sample_points.argtypes = [C.c_void_p, C.POINTER(rhg_params), C.POINTER(rhg_points)]
    L.rhg_count_edges_from_points.argtypes = [C.c_void_p, C.POINTER(rhg_params), C.POINTER(rhg_shard),
                                              C.POINTER(rhg_points), C.POINTER(rhg_run_stats),
                                              C.POINTER(C.c_uint32)]
    L.rhg_sample_uniforms.argtypes = [C.c_void_p, C.POINTER(rhg_params), P_f64, P_f64]
    L.rhg_fp64_peak.argtypes = [C.c_int, P_f64, P_f64, P_f64]
    P_u64 = C.POINTER(C.c_uint64)
    L.rhg_generate_edges.argtypes = [C.c_void_p, C.POINTER(rhg_params), C.POINTER(rhg_shard),
                                     C.POINTER(rhg_run_stats), P_u64, C.c_uint64, P_u64]
    L.rhg_edges_from_points.argtypes = [C.c_void_p, C.POINTER(rhg_params), C.POINTER(rhg_shard),
                                        C.POINTER(rhg_points), C.POINTER(rhg_run_stats), P_u64, C.c_uint64, P_u64]
    L.rhg_write_edges_text.argtypes = [C.c_char_p, P_u64, C.c_uint64]
    L.rhg_write_edges_binary.argtypes = [C.c_char_p, P_u64, C.c_uint64]
    L.rhg_read_edges_binary.argtypes = [C.c_char_p, P_u64, C.c_uint64, P_u64]
    L.rhg_io_last_error.restype = C.c_char_p
    L.rhg_powerlaw_mle.argtypes = [C.POINTER(C.c_uint32), C.c_uint64, C.c_uint32, P_f64]
    L.rhg_naive_edges.argtypes = [C.c_void_p, C.c_uint64, C.c_double, P_f64, P_f64, P_u64, C.c_uint64, P_u64]
    L.rhg_layout.argtypes = [C.POINTER(rhg_params), C.POINTER(C.c_uint32), C.POINTER(C.c_uint32), P_u64, P_u64,
                             P_u64, C.POINTER(C.c_uint8)]
    L.rhg_libm_eval.argtypes = [C.c_int, C.c_int, P_f64, P_f64, P_f64, C.c_uint64]
    L.rhg_create_multi.argtypes = [C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_void_p)]
    L.rhg_context_devices.argtypes = [C.c_void_p, C.POINTER(C.c_int)]
    L.rhg_nccl_unique_id.argtypes = [C.POINTER(C.c_uint8)]
    L.rhg_attach_comm.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.POINTER(C.c_uint8)]
    L.rhg_audit_predicate.argtypes = [C.c_void_p, C.POINTER(rhg_params), C.POINTER(rhg_shard),
                                      C.POINTER(rhg_audit_report), C.POINTER(rhg_run_stats)]
    L.rhg_unit_stats.argtypes = [C.c_void_p, C.POINTER(rhg_params), P_u64, P_u64, P_u64]
    L.rhg_generate_edges_units.argtypes = [C.c_void_p, C.POINTER(rhg_params), P_u64, C.c_uint64, P_u64, P_u64]
    L.rhg_shard_extent.argtypes = [C.POINTER(rhg_params), C.POINTER(rhg_shard), C.POINTER(rhg_shard_info)]
    _lib = L
    return L


def check(rc: int) -> None:
    """Map ABI status codes onto the reference's exception classes."""
    if rc == RHG_OK:
        return
    msg = lib().rhg_last_error().decode()
    if rc == RHG_INVALID_ARGUMENT:
        raise ValueError(msg)  # std::invalid_argument
    if rc == RHG_CUDA:
        raise RhgCudaError(msg)
    if rc == RHG_NOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg)  # std::logic_error
