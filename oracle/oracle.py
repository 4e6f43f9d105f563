"""ctypes bindings of the parity checkers (TEST INFRASTRUCTURE ONLY).

Two CPU checkers share the C-ABI POD structs of include/scalarmc_b200.h:

  Port       oracle/liboracle.so — the plain-C restatement (scalarmc_oracle.c)
  Reference  oracle/_ref/libscalarmc_ref.so — the real reference scalarmc,
             compiled from /root/reference/proj/src (oracle/Makefile) behind
             the extern "C" harness ref_capi.cpp

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
--impl reference) import this module, and only to check or time the
reference — never as the product path.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

from oracle import pods as A  # the checkers' own copy of the ABI PODs (no product import)

HERE = Path(__file__).resolve().parent
PORT_LIB = HERE / "liboracle.so"
REF_LIB = HERE / "_ref" / "libscalarmc_ref.so"

_dp = C.POINTER(C.c_double)
_u32p = C.POINTER(C.c_uint32)
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_u8p = C.POINTER(C.c_uint8)


def _status(lib, prefix: str, rc: int) -> None:
    if rc == 0:
        return
    msg = getattr(lib, prefix + "last_error")().decode()
    if rc == A.SMC_EINVAL:
        raise ValueError(msg)
    if rc == A.SMC_ERANGE:
        raise IndexError(msg)
    raise RuntimeError(msg)


class _Checker:
    prefix = ""
    takes_workers = False

    def __init__(self, path: Path):
        if not path.exists():
            raise FileNotFoundError(f"{path} not built (make -C oracle)")
        self.lib = C.CDLL(str(path))
        L, P = self.lib, self.prefix
        getattr(L, P + "last_error").restype = C.c_char_p
        getattr(L, P + "pairwise_sum").restype = C.c_double
        getattr(L, P + "pairwise_sum").argtypes = [_dp, C.c_int64]
        for name in ("stream_draws", "prior_modes", "prior_draw"):
            getattr(L, P + name).restype = C.c_int64

    def _f(self, name):
        return getattr(self.lib, self.prefix + name)

    def _w(self, workers):
        return (C.c_int(workers),) if self.takes_workers else ()

    # -- rng ----------------------------------------------------------------
    def philox(self, ctr, key) -> np.ndarray:
        ctr = np.ascontiguousarray(ctr, dtype=np.uint32).reshape(-1, 4)
        key = np.ascontiguousarray(key, dtype=np.uint32).reshape(-1, 2)
        out = np.empty_like(ctr)
        f = self._f("philox4x32")
        for i in range(ctr.shape[0]):
            f(ctr[i].ctypes.data_as(_u32p), key[i].ctypes.data_as(_u32p), out[i].ctypes.data_as(_u32p))
        return out

    def normal_pairs(self, seed: int, obs: int, particle: int, n: int) -> np.ndarray:
        out = np.empty((n, 2), dtype=np.float64)
        self._f("normal_pairs")(C.c_uint64(seed), C.c_uint64(obs) if self.takes_workers else C.c_uint32(obs),
                                C.c_uint64(particle) if self.takes_workers else C.c_uint32(particle),
                                C.c_int64(n), out.ctypes.data_as(_dp))
        return out

    def stream_draws(self, seed: int, obs: int, particle: int, ops) -> np.ndarray:
        ops = np.ascontiguousarray(ops, dtype=np.int32)
        out = np.empty(2 * len(ops), dtype=np.float64)
        conv = C.c_uint64 if self.takes_workers else C.c_uint32
        w = self._f("stream_draws")(C.c_uint64(seed), conv(obs), conv(particle), C.c_int64(len(ops)),
                                    ops.ctypes.data_as(_i32p), out.ctypes.data_as(_dp))
        return out[:w]

    # -- fields -------------------------------------------------------------
    def velocity_eval(self, velocity, x) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1, 2)
        out = np.empty_like(x)
        pod = velocity._pod()
        _status(self.lib, self.prefix, self._f("velocity_eval")(C.byref(pod), C.c_int64(x.shape[0]),
                                                                 x.ctypes.data_as(_dp), out.ctypes.data_as(_dp)))
        return out

    def scalar_eval(self, field, x) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1, 2)
        out = np.empty(x.shape[0], dtype=np.float64)
        pod = field._pod()
        rc = self._f("scalar_eval")(C.byref(pod), C.c_int64(x.shape[0]), x.ctypes.data_as(_dp),
                                    out.ctypes.data_as(_dp))
        if self.takes_workers:
            _status(self.lib, self.prefix, rc)
        return out

    def pairwise_sum(self, values) -> float:
        v = np.ascontiguousarray(values, dtype=np.float64)
        return self._f("pairwise_sum")(v.ctypes.data_as(_dp), C.c_int64(v.size))

    # -- forward maps -------------------------------------------------------
    def observe_ad(self, spec, seed: int, workers: int = 0) -> np.ndarray:
        p, keep = spec._pod()
        out = np.zeros(p.n_obs, dtype=_est_dtype())
        rc = self._f("ad_observe")(C.byref(p), C.c_uint64(seed), *self._w(workers),
                                   out.ctypes.data_as(C.POINTER(A.smc_estimate)))
        _status(self.lib, self.prefix, rc)
        return out

    def ad_particle_values(self, spec, obs_index: int, seed: int, n: int, terminal: bool = False):
        p, keep = spec._pod()
        out = np.empty(n, dtype=np.float64)
        term = np.empty((n, 2), dtype=np.float64) if terminal else None
        rc = self._f("ad_particle_values")(C.byref(p), C.c_uint64(obs_index), C.c_uint64(seed), C.c_int64(n),
                                           out.ctypes.data_as(_dp), term.ctypes.data_as(_dp) if terminal else _dp())
        _status(self.lib, self.prefix, rc)
        return (out, term) if terminal else out

    def observe_bvp(self, spec, seed: int, workers: int = 0) -> np.ndarray:
        p, keep = spec._pod()
        out = np.zeros(p.n_obs, dtype=_est_dtype())
        rc = self._f("bvp_observe")(C.byref(p), C.c_uint64(seed), *self._w(workers),
                                    out.ctypes.data_as(C.POINTER(A.smc_estimate)))
        _status(self.lib, self.prefix, rc)
        return out

    def bvp_particle_values(self, spec, obs_index: int, seed: int, n: int):
        p, keep = spec._pod()
        vals = np.empty(n, dtype=np.float64)
        aux = np.empty(n, dtype=np.float64)
        failed = np.empty(n, dtype=np.uint8)
        steps = np.empty(n, dtype=np.int64)
        rc = self._f("bvp_particle_values")(C.byref(p), C.c_uint64(obs_index), C.c_uint64(seed), C.c_int64(n),
                                            vals.ctypes.data_as(_dp), aux.ctypes.data_as(_dp),
                                            failed.ctypes.data_as(_u8p), steps.ctypes.data_as(_i64p))
        _status(self.lib, self.prefix, rc)
        return vals, aux, failed, steps

    # -- u -> field ---------------------------------------------------------
    def prior_modes(self, cutoff: int) -> np.ndarray:
        cap = 4 * (cutoff + 1) ** 2
        out = np.empty((cap, 2), dtype=np.int32)
        n = self._f("prior_modes")(C.c_int(cutoff), out.ctypes.data_as(_i32p), C.c_int64(cap))
        return out[:n].copy()

    def prior_draw(self, prior, seed: int, obs: int, particle: int) -> np.ndarray:
        cap = 8 * (prior.cutoff + 1) ** 2
        out = np.empty(cap, dtype=np.float64)
        n = self._f("prior_draw")(C.byref(prior._pod()), C.c_uint64(seed), C.c_uint64(obs), C.c_uint64(particle),
                                  out.ctypes.data_as(_dp), C.c_int64(cap))
        return out[:n].copy()


def _est_dtype():
    return np.dtype([("mean", "<f8"), ("std_error", "<f8"), ("n_particles", "<i8"), ("n_failed", "<i8"),
                     ("aux_mean", "<f8")])


class Port(_Checker):
    """The plain-C restatement (oracle/scalarmc_oracle.c)."""
    prefix = "orc_"
    takes_workers = False

    def __init__(self, path: Path = PORT_LIB):
        super().__init__(path)
        self.lib.orc_bvp_resolved_dt.restype = C.c_double


class Reference(_Checker):
    """The real reference library compiled from /root/reference sources."""
    prefix = "ref_"
    takes_workers = True

    def __init__(self, path: Path = REF_LIB):
        super().__init__(path)
        self.lib.ref_resolve_workers.restype = C.c_int

    def resolve_workers(self, n: int = 0) -> int:
        return self.lib.ref_resolve_workers(n)

    def observe_ad_single(self, spec, obs_index: int, seed: int, workers: int = 0):
        p, keep = spec._pod()
        out = np.zeros(1, dtype=_est_dtype())
        rc = self.lib.ref_ad_observe_single(C.byref(p), C.c_uint64(obs_index), C.c_uint64(seed), C.c_int(workers),
                                            out.ctypes.data_as(C.POINTER(A.smc_estimate)))
        _status(self.lib, self.prefix, rc)
        return out[0]

    def observe_ad_u(self, spec, prior, u, seed: int, workers: int = 0) -> np.ndarray:
        p, keep = spec._pod()
        u = np.ascontiguousarray(u, dtype=np.float64)
        out = np.zeros(p.n_obs, dtype=_est_dtype())
        rc = self.lib.ref_ad_observe_u(C.byref(p), C.byref(prior._pod()), u.ctypes.data_as(_dp), C.c_uint64(seed),
                                       C.c_int(workers), out.ctypes.data_as(C.POINTER(A.smc_estimate)))
        _status(self.lib, self.prefix, rc)
        return out

    def misfit(self, spec, prior, u, data, noise_std: float, forward_seed: int, workers: int = 0) -> float:
        p, keep = spec._pod()
        u = np.ascontiguousarray(u, dtype=np.float64)
        d = np.ascontiguousarray(data, dtype=np.float64)
        out = C.c_double()
        rc = self.lib.ref_misfit(C.byref(p), C.byref(prior._pod()), u.ctypes.data_as(_dp), d.ctypes.data_as(_dp),
                                 C.c_double(noise_std), C.c_uint64(forward_seed), C.c_int(workers), C.byref(out))
        _status(self.lib, self.prefix, rc)
        return out.value

    def forcing_cost(self, spec, amplitudes, centers, sharpness: float, target, seed: int, workers: int = 0) -> float:
        p, keep = spec._pod()
        a = np.ascontiguousarray(amplitudes, dtype=np.float64)
        c = np.ascontiguousarray(centers, dtype=np.float64).reshape(-1, 2)
        t = np.ascontiguousarray(target, dtype=np.float64)
        out = C.c_double()
        rc = self.lib.ref_forcing_cost(C.byref(p), C.c_int64(a.size), a.ctypes.data_as(_dp), c.ctypes.data_as(_dp),
                                       C.c_double(sharpness), t.ctypes.data_as(_dp), C.c_uint64(seed),
                                       C.c_int(workers), C.byref(out))
        _status(self.lib, self.prefix, rc)
        return out.value

    def run_chain(self, like, prior, n_steps: int, beta: float, burn_in: int, thin: int, seed: int, u0=None,
                  workers: int = 0) -> dict:
        """The reference's run_chain (inference.cpp:170-194) with LikelihoodSpec
        `like` (paper_1808_10580_b200.LikelihoodSpec)."""
        p, keep = like.forward._pod() if like is not None else (None, None)
        dim = prior.dimension()
        # the reference's sample iterations (inference.cpp:183-185)
        n_samples = sum(1 for i in range(1, n_steps + 1) if i > burn_in and (i - burn_in - 1) % thin == 0)
        trace = np.zeros(max(n_steps, 1))
        samples = np.zeros((max(n_samples, 1), dim))
        final_u = np.zeros(dim)
        map_u = np.zeros(dim)
        sc = np.zeros(3)
        d = np.ascontiguousarray(like.data if like is not None else [0.0], dtype=np.float64)
        u0p = np.ascontiguousarray(u0, dtype=np.float64).ctypes.data_as(_dp) if u0 is not None else _dp()
        rc = self.lib.ref_run_chain(C.byref(p) if p is not None else None, C.byref(prior._pod()),
                                    d.ctypes.data_as(_dp), C.c_double(like.noise_std if like is not None else 1.0),
                                    C.c_uint64(like.forward_seed if like is not None else 0), C.c_int64(n_steps),
                                    C.c_double(beta), C.c_int64(burn_in), C.c_int64(thin), C.c_uint64(seed), u0p,
                                    C.c_int(workers), trace.ctypes.data_as(_dp), samples.ctypes.data_as(_dp),
                                    final_u.ctypes.data_as(_dp), map_u.ctypes.data_as(_dp), sc.ctypes.data_as(_dp))
        _status(self.lib, self.prefix, rc)
        return {"phi_trace": trace[:n_steps], "samples": samples[:n_samples], "final_u": final_u, "map_u": map_u,
                "final_phi": sc[0], "map_objective": sc[1], "accepted": int(sc[2])}

    def optimize_forcing(self, spec, initial, centers, sharpness, target, x_tol, f_tol, max_iter, initial_step,
                         seed: int, workers: int = 0) -> dict:
        p, keep = spec._pod()
        ini = np.ascontiguousarray(initial, dtype=np.float64)
        c = np.ascontiguousarray(centers, dtype=np.float64).reshape(-1, 2)
        t = np.ascontiguousarray(target, dtype=np.float64)
        arg = np.zeros(ini.size)
        sc = np.zeros(2)
        reason = C.create_string_buffer(16)
        rc = self.lib.ref_optimize_forcing(C.byref(p), C.c_int64(ini.size), ini.ctypes.data_as(_dp),
                                           c.ctypes.data_as(_dp), C.c_double(sharpness), t.ctypes.data_as(_dp),
                                           C.c_double(x_tol), C.c_double(f_tol), C.c_int(max_iter),
                                           C.c_double(initial_step), C.c_uint64(seed), C.c_int(workers),
                                           arg.ctypes.data_as(_dp), sc.ctypes.data_as(_dp), reason)
        _status(self.lib, self.prefix, rc)
        return {"argmin": arg, "min_value": sc[0], "iterations": int(sc[1]), "stop_reason": reason.value.decode()}

    # ---- spectral Galerkin reference solver: the reference's src/galerkin.cpp
    # compiled against oracle/eigen_shim (its Eigen dependency is absent) ----
    @staticmethod
    def _gbasis(kind: str, L: int):
        return A.smc_galerkin_basis(1 if kind == "disk" else 0, int(L))

    def galerkin_spectral_radius(self, spec, kind: str, L: int) -> float:
        p, keep = spec._pod()
        out = C.c_double()
        rc = self.lib.ref_galerkin_spectral_radius(C.byref(p), C.byref(self._gbasis(kind, L)), C.byref(out))
        _status(self.lib, self.prefix, rc)
        return out.value

    def galerkin_solve_ad(self, spec, kind: str, L: int, dt_ref: float) -> dict:
        """-> {observation_values, coefficients_at_observations [n_obs][nb]
        (complex), final_coefficients [nb], basis_modes, dt_used, steps}."""
        p, keep = spec._pod()
        cap = (2 * L + 1) ** 2
        n_obs = len(spec.observations)
        vals = np.zeros(n_obs)
        cat = np.zeros((n_obs, cap, 2))
        fin = np.zeros((cap, 2))
        modes = np.zeros((cap, 2), dtype=np.int32)
        r = A.smc_galerkin_result(vals.ctypes.data_as(_dp), cat.ctypes.data_as(_dp), fin.ctypes.data_as(_dp), 0.0, 0)
        self.lib.ref_galerkin_solve_ad.argtypes = [C.c_void_p, C.c_void_p, C.c_double, C.c_void_p, C.c_void_p,
                                                   C.c_int64]
        rc = self.lib.ref_galerkin_solve_ad(C.byref(p), C.byref(self._gbasis(kind, L)), C.c_double(dt_ref),
                                            C.byref(r), modes.ctypes.data, C.c_int64(cap))
        _status(self.lib, self.prefix, rc)
        # the basis size: box (2L+1)^2, disk counted like basis_mode_list
        nb = cap if kind == "box" else sum(1 for a in range(-L, L + 1) for b in range(-L, L + 1) if a * a + b * b <= L * L)
        # coefficients_at_observations was written with stride nb
        flat = cat.reshape(-1)[: n_obs * nb * 2].reshape(n_obs, nb, 2)
        return {"observation_values": vals, "coefficients_at_observations": flat[..., 0] + 1j * flat[..., 1],
                "final_coefficients": fin[:nb, 0] + 1j * fin[:nb, 1],
                "basis_modes": [tuple(int(v) for v in m) for m in modes[:nb]], "dt_used": r.dt_used,
                "steps": int(r.steps)}

    def galerkin_field_grid(self, coefficients, modes, n: int) -> np.ndarray:
        c = np.ascontiguousarray(np.stack([np.real(coefficients), np.imag(coefficients)], axis=-1), dtype=np.float64)
        m = np.ascontiguousarray(np.asarray(modes, dtype=np.int32).reshape(-1, 2))
        out = np.zeros(int(n) * int(n)) if n >= 2 else np.zeros(1)
        self.lib.ref_galerkin_field_grid.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p]
        rc = self.lib.ref_galerkin_field_grid(len(m), m.ctypes.data, c.ctypes.data, int(n), out.ctypes.data)
        _status(self.lib, self.prefix, rc)
        return out

    def resolved_dt_ad(self, spec) -> float:
        p, keep = spec._pod()
        out = C.c_double()
        _status(self.lib, self.prefix, self.lib.ref_ad_resolved_dt(C.byref(p), C.byref(out)))
        return out.value

    def resolved_dt_bvp(self, spec) -> float:
        p, keep = spec._pod()
        out = C.c_double()
        _status(self.lib, self.prefix, self.lib.ref_bvp_resolved_dt(C.byref(p), C.byref(out)))
        return out.value


class ReferenceCli:
    """The reference's config parser, record writer and CLI command bodies
    (oracle/ref_cli.cpp over the compiled reference; needs config.cpp, i.e.
    nlohmann::json at build time)."""

    KINDS = {0: None, 1: "ConfigError", 2: "invalid_argument", 3: "out_of_range", 4: "exception"}

    def __init__(self, path: Path = REF_LIB):
        self.lib = C.CDLL(str(path))
        if not hasattr(self.lib, "refcli_config_check"):
            raise RuntimeError("reference built without config.cpp (nlohmann::json not found)")

    def config_check(self, text: str, origin: str = "<config>", stage: int = 0):
        """-> (kind, message): kind None (accepted), "ConfigError",
        "invalid_argument", "out_of_range" or "exception"."""
        buf = C.create_string_buffer(4096)
        rc = self.lib.refcli_config_check(text.encode(), origin.encode(), stage, buf, 4096)
        return self.KINDS[rc], buf.value.decode()

    def format_double(self, v: float) -> str:
        buf = C.create_string_buffer(64)
        self.lib.refcli_format_double(C.c_double(v), buf, 64)
        return buf.value.decode()

    def _run(self, fn, *args):
        msg = C.create_string_buffer(4096)
        rc = fn(*args, msg, 4096)
        if rc:
            raise RuntimeError(f"{self.KINDS[rc]}: {msg.value.decode()}")

    def forward(self, config: str, out: str, fmt: str = "csv", seed: int = -1, bvp: bool = False) -> None:
        self._run(self.lib.refcli_forward, config.encode(), out.encode(), fmt.encode(), C.c_int64(seed), int(bvp))

    def sample(self, config: str, out_dir: str, fmt: str = "csv", seed: int = -1, steps: int = -1,
               beta: float = -1.0) -> str:
        text = C.create_string_buffer(4096)
        self._run(self.lib.refcli_sample, config.encode(), out_dir.encode(), fmt.encode(), C.c_int64(seed),
                  C.c_int64(steps), C.c_double(beta), text, 4096)
        return text.value.decode()

    def optimize(self, config: str, out: str, fmt: str = "csv", seed: int = -1) -> str:
        text = C.create_string_buffer(4096)
        self._run(self.lib.refcli_optimize, config.encode(), out.encode(), fmt.encode(), C.c_int64(seed), text,
                  4096)
        return text.value.decode()


def port_available() -> bool:
    return PORT_LIB.exists()


def reference_available() -> bool:
    return REF_LIB.exists()
