"""ctypes mirror of include/scalarmc_b200.h (the C-ABI drop-in boundary).

The struct layouts below must match the header field for field; tests/
test_abi.py checks sizes against the compiled library.  `load_library()` loads
the in-tree CUDA library and fails loudly when it is missing: there is no CPU
fallback on the product path.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

PKG_DIR = Path(__file__).resolve().parent
# SMC_LIBRARY: an alternative build of the same library (A/B measurements of
# two kernel versions on one box); the default is the in-tree build.
LIB_PATH = Path(os.environ.get("SMC_LIBRARY") or PKG_DIR / "lib" / "libscalarmc_b200.so")

SMC_OK, SMC_EINVAL, SMC_ERANGE, SMC_ERUNTIME, SMC_ECUDA = range(5)
SCALAR_CONSTANT, SCALAR_COSINE, SCALAR_BUMPS, SCALAR_LINEAR = range(4)
DOMAIN_TORUS, DOMAIN_BOX, DOMAIN_DISK = range(3)
EULER_MARUYAMA, MILSTEIN = 0, 1
FP64, FP32, FP64_STRICT = 0, 1, 2
SMC_CHUNK = 1024

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)


class smc_estimate(C.Structure):
    _fields_ = [("mean", C.c_double), ("std_error", C.c_double), ("n_particles", C.c_int64),
                ("n_failed", C.c_int64), ("aux_mean", C.c_double)]


class smc_scalar_field(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n_terms", C.c_int32), ("constant", C.c_double),
                ("gradient", C.c_double * 2), ("sharpness", C.c_double), ("amplitude", _dp),
                ("freq", _dp), ("phase", _dp), ("center", _dp)]


class smc_velocity(C.Structure):
    _fields_ = [("is_constant", C.c_int32), ("max_wavenumber", C.c_int32),
                ("constant", C.c_double * 2), ("n_modes", C.c_int64), ("k", _ip), ("coeff", _dp)]


class smc_ad_problem(C.Structure):
    _fields_ = [("velocity", smc_velocity), ("kappa", C.c_double),
                ("initial_condition", smc_scalar_field), ("n_obs", C.c_int64), ("obs_t", _dp),
                ("obs_x", _dp), ("dt", C.c_double), ("n_particles", C.c_int64),
                ("scheme", C.c_int32), ("precision", C.c_int32)]


class smc_domain(C.Structure):
    _fields_ = [("kind", C.c_int32), ("pad_", C.c_int32), ("lower", C.c_double * 2),
                ("upper", C.c_double * 2), ("center", C.c_double * 2), ("radius", C.c_double)]


class smc_bvp_problem(C.Structure):
    _fields_ = [("velocity", smc_velocity), ("kappa", C.c_double), ("forcing", smc_scalar_field),
                ("boundary_data", smc_scalar_field), ("domain", smc_domain), ("n_obs", C.c_int64),
                ("obs_x", _dp), ("dt", C.c_double), ("n_particles", C.c_int64),
                ("scheme", C.c_int32), ("precision", C.c_int32), ("max_steps", C.c_int64)]


class smc_prior(C.Structure):
    _fields_ = [("cutoff", C.c_int32), ("pad_", C.c_int32), ("s0", C.c_double), ("alpha", C.c_double)]


class smc_chain_config(C.Structure):
    _fields_ = [("n_steps", C.c_int64), ("beta", C.c_double), ("burn_in", C.c_int64), ("thin", C.c_int64)]


class smc_chain_outputs(C.Structure):
    _fields_ = [("final_u", _dp), ("final_phi", _dp), ("map_u", _dp), ("map_objective", _dp),
                ("accepted", C.POINTER(C.c_int64)), ("phi_trace", _dp), ("samples", _dp)]


class smc_galerkin_basis(C.Structure):
    _fields_ = [("kind", C.c_int32), ("cutoff", C.c_int32)]


class smc_galerkin_result(C.Structure):
    _fields_ = [("observation_values", _dp), ("coefficients_at_observations", _dp), ("final_coefficients", _dp),
                ("dt_used", C.c_double), ("steps", C.c_int64)]


class smc_stats(C.Structure):
    _fields_ = [("particle_kernel_ms", C.c_double), ("reduce_ms", C.c_double),
                ("kernel_launches", C.c_int64), ("particle_steps", C.c_int64),
                ("total_launches", C.c_int64)]


class smc_group_desc(C.Structure):
    _fields_ = [("world", C.c_int32), ("rank", C.c_int32), ("n_local", C.c_int32), ("nccl", C.c_int32),
                ("devices", C.c_int32 * 8)]


SMC_UNIQUE_ID_BYTES = 128
# int (*)(void* user, uint8_t* buf, const uint64_t* displ, const uint64_t* bytes, int world)
EXCHANGE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_uint8), C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                          C.c_int)


def dptr(a: np.ndarray | None):
    if a is None:
        return _dp()
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def iptr(a: np.ndarray | None):
    if a is None:
        return _ip()
    assert a.dtype == np.int32 and a.flags.c_contiguous
    return a.ctypes.data_as(_ip)


# Exported symbols: name -> (restype, argtypes).  Kept in sync with the header;
# tests/test_abi.py asserts every header declaration is listed and exported.
_PROTOS = {
    "smc_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "smc_destroy": (None, [C.c_void_p]),
    "smc_nccl_unique_id": (C.c_int, [C.POINTER(C.c_uint8)]),
    "smc_create_multi": (C.c_int, [C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_void_p)]),
    "smc_create_rank": (C.c_int, [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_uint8), C.POINTER(C.c_void_p)]),
    "smc_group_query": (C.c_int, [C.c_void_p, C.POINTER(smc_group_desc)]),
    "smc_create_rank_hosted": (C.c_int, [C.c_int, C.c_int, C.c_int, EXCHANGE_FN, C.c_void_p, C.POINTER(C.c_void_p)]),
    "smc_last_error": (C.c_char_p, []),
    "smc_abi_version": (C.c_int, []),
    "smc_ad_observe": (C.c_int, [C.c_void_p, C.POINTER(smc_ad_problem), C.c_uint64,
                                 C.POINTER(smc_estimate)]),
    "smc_ad_observe_single": (C.c_int, [C.c_void_p, C.POINTER(smc_ad_problem), C.c_uint64,
                                        C.c_uint64, C.POINTER(smc_estimate)]),
    "smc_ad_observe_batched": (C.c_int, [C.c_void_p, C.POINTER(smc_ad_problem),
                                         C.POINTER(smc_prior), C.c_int64, _dp,
                                         C.POINTER(C.c_uint64), C.c_uint64,
                                         C.POINTER(smc_estimate)]),
    "smc_bvp_observe": (C.c_int, [C.c_void_p, C.POINTER(smc_bvp_problem), C.c_uint64,
                                  C.POINTER(smc_estimate)]),
    "smc_bvp_observe_range": (C.c_int, [C.c_void_p, C.POINTER(smc_bvp_problem), C.c_uint64, C.c_int64,
                                        C.c_int64, C.POINTER(smc_estimate)]),
    "smc_bvp_forcing_basis": (C.c_int, [C.c_void_p, C.POINTER(smc_bvp_problem), C.c_uint64, _dp, _dp, _dp,
                                        C.POINTER(C.c_int64)]),
    "smc_pcn_num_samples": (C.c_int64, [C.POINTER(smc_chain_config)]),
    "smc_galerkin_n_basis": (C.c_int64, [C.POINTER(smc_galerkin_basis)]),
    "smc_galerkin_modes": (C.c_int, [C.POINTER(smc_galerkin_basis), C.POINTER(C.c_int32)]),
    "smc_galerkin_spectral_radius": (C.c_int, [C.c_void_p, C.POINTER(smc_ad_problem), C.POINTER(smc_galerkin_basis),
                                               _dp]),
    "smc_galerkin_solve_ad": (C.c_int, [C.c_void_p, C.POINTER(smc_ad_problem), C.POINTER(smc_galerkin_basis),
                                        C.c_double, C.POINTER(smc_galerkin_result)]),
    "smc_galerkin_field_grid": (C.c_int, [C.c_void_p, C.POINTER(smc_galerkin_basis), _dp, C.c_int32, _dp]),
    "smc_pcn_chains": (C.c_int, [C.c_void_p, C.POINTER(smc_ad_problem), C.POINTER(smc_prior), _dp, C.c_double,
                                 C.c_uint64, C.c_int64, C.POINTER(C.c_uint64), _dp, C.POINTER(smc_chain_config),
                                 C.POINTER(smc_chain_outputs)]),
    "smc_ad_resolved_dt": (C.c_int, [C.POINTER(smc_ad_problem), _dp]),
    "smc_bvp_resolved_dt": (C.c_int, [C.POINTER(smc_bvp_problem), _dp]),
    "smc_ad_validate": (C.c_int, [C.POINTER(smc_ad_problem)]),
    "smc_bvp_validate": (C.c_int, [C.POINTER(smc_bvp_problem)]),
    "smc_velocity_validate": (C.c_int, [C.POINTER(smc_velocity)]),
    "smc_num_chunks": (C.c_int64, [C.c_int64]),
    "smc_stream": (C.c_void_p, [C.c_void_p]),
    "smc_set_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "smc_ad_particle_values": (C.c_int, [C.c_void_p, C.POINTER(smc_ad_problem), C.c_uint64,
                                         C.c_uint64, C.c_int64, _dp]),
    "smc_bvp_particle_values": (C.c_int, [C.c_void_p, C.POINTER(smc_bvp_problem), C.c_uint64,
                                          C.c_uint64, C.c_int64, _dp, _dp,
                                          C.POINTER(C.c_uint8)]),
    "smc_philox_device": (C.c_int, [C.c_void_p, C.c_int64, C.POINTER(C.c_uint32),
                                    C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]),
    "smc_normal_pairs_device": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64,
                                          C.c_int64, _dp]),
    "smc_last_stats": (C.c_int, [C.c_void_p, C.POINTER(smc_stats)]),
    "smc_fp64_peak": (C.c_int, [C.c_void_p, C.c_double, _dp]),
    "smc_guard_selftest": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64]),
    "smc_fp32_peak": (C.c_int, [C.c_void_p, C.c_double, _dp]),
    "smc_struct_sizes": (C.c_int, [C.POINTER(C.c_int64), C.c_int]),
}

_lib = None


def load_library(path: str | os.PathLike | None = None) -> C.CDLL:
    """Load the in-tree CUDA library (no fallback: raises if it is missing)."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise RuntimeError(
            f"scalarmc_b200: CUDA library {p} is not built; run "
            "`python -c 'import __graft_entry__ as g; g.build()'` (there is no CPU fallback)")
    lib = C.CDLL(str(p))
    for name, (res, args) in _PROTOS.items():
        if os.environ.get("SMC_LIBRARY") and not hasattr(lib, name):
            continue  # an older A/B build without this entry point
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib
