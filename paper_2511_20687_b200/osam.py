"""Thin Python binding of libosam.so (include/osam.h): argument marshalling only.

Every step of the O-SAM time loop runs in the CUDA kernels of libosam.so; this module
only builds the C structs, passes pointers (torch CUDA tensors -> device pointers,
NumPy arrays -> host pointers) and converts error codes to exceptions.  There is no CPU
fallback: if the shared library is missing or no GPU is present, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("OSAM_LIB") or os.path.join(_HERE, "libosam.so")

OSAM_FOM, OSAM_ROM = 0, 1
OSAM_EXPLICIT, OSAM_IMPLICIT = 0, 1
OSAM_LINEAR, OSAM_SVK, OSAM_NEOHOOKEAN = 0, 1, 2
MATERIALS = {"linear": OSAM_LINEAR, "svk": OSAM_SVK, "neohookean": OSAM_NEOHOOKEAN}
OSAM_OK, OSAM_WNOTCONVERGED = 0, 1
ERRORS = {-1: "OSAM_EINVAL", -2: "OSAM_ENOMEM", -3: "OSAM_ECUDA", -4: "OSAM_EOVERLAP", -5: "OSAM_EUNSTABLE"}

# C entry points declared in include/osam.h
EXPORTS = ("osam_create_subdomain", "osam_set_ic", "osam_step", "osam_get_state", "osam_get_accel",
           "osam_get_sizes", "osam_destroy", "osam_last_error", "osam_set_profiling", "osam_reset_profile",
           "osam_get_profile", "osam_opinf_replay", "osam_set_ic_reduced", "osam_set_conv_trace",
           "osam_get_conv_trace", "osam_get_k1_timeline")


class osam_subdomain_desc(C.Structure):
    _fields_ = [("kind", C.c_int32), ("lo", C.c_double * 3), ("hi", C.c_double * 3), ("nel", C.c_int32 * 3),
                ("E", C.c_double), ("nu", C.c_double), ("rho", C.c_double), ("dirichlet", C.c_uint8 * 6),
                ("r", C.c_int32), ("r_b", C.c_int32), ("batch", C.c_int32),
                ("n_free", C.c_int64), ("n_s", C.c_int64),
                ("Phi", C.POINTER(C.c_double)), ("Phi_s", C.POINTER(C.c_double)),
                ("Kbar", C.POINTER(C.c_double)), ("Bbar", C.POINTER(C.c_double)),
                ("e_scale", C.POINTER(C.c_double)),
                ("Hbar", C.POINTER(C.c_double)), ("Cbar", C.POINTER(C.c_double)),
                ("n_substeps", C.c_int32), ("integrator", C.c_int32), ("material", C.c_int32),
                ("phi_rows", C.POINTER(C.c_int64)), ("n_phi_rows", C.c_int64)]


class osam_replay_desc(C.Structure):
    _fields_ = [("r", C.c_int32), ("r_b", C.c_int32), ("order", C.c_int32), ("n_models", C.c_int32),
                ("n_steps", C.c_int32), ("dt", C.c_double), ("O", C.c_void_p), ("Ubar", C.c_void_p),
                ("Ghat", C.c_void_p), ("vh0", C.c_void_p)]


class osam_schwarz_cfg(C.Structure):
    _fields_ = [("dt", C.c_double), ("tol_rel", C.c_double), ("tol_abs", C.c_double),
                ("max_iters", C.c_int32), ("min_iters", C.c_int32)]


class OsamError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code


_lib = None


def lib():
    """Load libosam.so (built in-tree by __graft_entry__.build()); raise if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise OSError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        vp = C.c_void_p
        L.osam_create_subdomain.argtypes = [C.POINTER(osam_subdomain_desc), vp, C.POINTER(vp)]
        L.osam_set_ic.argtypes = [vp, vp, vp]
        L.osam_step.argtypes = [C.POINTER(vp), C.c_int32, C.POINTER(osam_schwarz_cfg), C.c_int32,
                                C.POINTER(C.c_int32)]
        L.osam_get_state.argtypes = [vp, vp, vp]
        L.osam_get_accel.argtypes = [vp, vp]
        L.osam_get_sizes.argtypes = [vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                     C.POINTER(C.c_int32)]
        L.osam_destroy.argtypes = [vp]
        L.osam_destroy.restype = None
        L.osam_last_error.restype = C.c_char_p
        L.osam_set_profiling.argtypes = [C.c_int32]
        L.osam_set_profiling.restype = None
        L.osam_reset_profile.restype = None
        L.osam_get_profile.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_int64), C.POINTER(C.c_double),
                                       C.POINTER(C.c_int64)]
        L.osam_get_profile.restype = None
        L.osam_opinf_replay.argtypes = [C.POINTER(osam_replay_desc), vp, C.POINTER(C.c_int32), vp, vp]
        L.osam_set_ic_reduced.argtypes = [vp, vp, vp, vp]
        L.osam_set_conv_trace.argtypes = [C.c_int32]
        L.osam_set_conv_trace.restype = None
        i32p = C.POINTER(C.c_int32)
        L.osam_get_conv_trace.argtypes = [C.POINTER(vp), C.c_int32, vp, i32p, i32p, i32p]
        L.osam_get_k1_timeline.argtypes = [C.POINTER(vp), C.c_int32, C.c_int32, C.POINTER(C.c_double)]
        for name in ("osam_create_subdomain", "osam_set_ic", "osam_step", "osam_get_state", "osam_get_accel",
                     "osam_get_sizes", "osam_opinf_replay", "osam_set_ic_reduced", "osam_get_conv_trace",
                     "osam_get_k1_timeline"):
            getattr(L, name).restype = C.c_int
        _lib = L
    return _lib


def _check(rc):
    if rc < 0:
        raise OsamError(rc, lib().osam_last_error().decode())
    return rc


def _ptr(x, numel=None):
    """Device pointer of a contiguous float64 torch tensor, host pointer of a C-contiguous float64 ndarray;
    `numel` (if given) is the element count the library will read or write there."""
    if x is None:
        return None
    if hasattr(x, "data_ptr"):
        import torch
        if x.dtype != torch.float64 or not x.is_contiguous():
            raise ValueError("expected a contiguous float64 tensor")
        n = x.numel()
        p = x.data_ptr()
    elif isinstance(x, np.ndarray) and x.dtype == np.float64 and x.flags.c_contiguous:
        n = x.size
        p = x.ctypes.data
    else:
        raise ValueError("expected a contiguous float64 ndarray or torch tensor")
    if numel is not None and n != numel:
        raise ValueError(f"buffer holds {n} doubles, the call needs {numel}")
    return C.c_void_p(p)


def _dptr(a):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_double))


class Subdomain:
    """Owning wrapper of an osam_subdomain handle (osam_create_subdomain / osam_destroy)."""

    def __init__(self, kind, lo, hi, nel, E, nu, rho, dirichlet=(0,) * 6, stream=None, rom=None, e_scale=None,
                 n_substeps=1, integrator=OSAM_EXPLICIT, material=OSAM_LINEAR):
        d = osam_subdomain_desc()
        d.n_substeps = int(n_substeps)
        d.integrator = int(integrator)
        d.material = int(material)
        d.kind = kind
        d.lo[:] = [float(x) for x in lo]
        d.hi[:] = [float(x) for x in hi]
        d.nel[:] = [int(x) for x in nel]
        d.E, d.nu, d.rho = float(E), float(nu), float(rho)
        d.dirichlet[:] = [int(x) for x in dirichlet]
        self._keep = []
        d.batch = 1
        if kind == OSAM_ROM:
            Phi = np.asfortranarray(rom["Phi"], dtype=np.float64)
            Phi_s = np.asfortranarray(rom["Phi_s"], dtype=np.float64)
            Kbar = np.asfortranarray(rom["Kbar"], dtype=np.float64)
            Bbar = np.asfortranarray(rom["Bbar"], dtype=np.float64)
            d.r, d.r_b = Phi.shape[1], Phi_s.shape[1]
            d.n_free, d.n_s = Phi.shape[0], Phi_s.shape[0]
            if rom.get("phi_rows") is not None:   # Phi on a subset of its rows (include/osam.h)
                rows = np.ascontiguousarray(rom["phi_rows"], dtype=np.int64)
                if len(rows) != Phi.shape[0]:
                    raise ValueError("phi_rows must list one free row per row of Phi")
                d.phi_rows = rows.ctypes.data_as(C.POINTER(C.c_int64))
                d.n_phi_rows = len(rows)
                d.n_free = int(rom["n_free"])
                self._keep.append(rows)
            d.Phi, d.Phi_s, d.Kbar, d.Bbar = _dptr(Phi), _dptr(Phi_s), _dptr(Kbar), _dptr(Bbar)
            self._keep += [Phi, Phi_s, Kbar, Bbar]
            for name in ("Hbar", "Cbar"):  # polynomial OpInf terms (optional)
                if rom.get(name) is not None:
                    M = np.asfortranarray(rom[name], dtype=np.float64)
                    setattr(d, name, _dptr(M))
                    self._keep.append(M)
            if e_scale is not None:
                e = np.ascontiguousarray(e_scale, dtype=np.float64)
                d.batch = len(e)
                d.e_scale = _dptr(e)
                self._keep.append(e)
            self.r = d.r
            self.n_s = d.n_s
        self.kind = kind
        self.batch = d.batch
        self.nn = tuple(int(n) + 1 for n in nel)
        self.n_nodes = self.nn[0] * self.nn[1] * self.nn[2]
        h = C.c_void_p()
        _check(lib().osam_create_subdomain(C.byref(d), C.c_void_p(stream or 0), C.byref(h)))
        self.handle = h
        self._keep = []  # the library copied the host arrays

    def _field_size(self):
        """doubles of a state field: batch x 3n (FOM / full ROM field) or r x batch (ROM state)."""
        return 3 * self.n_nodes * self.batch

    def set_ic(self, u0, v0=None):
        n = self._field_size()
        _check(lib().osam_set_ic(self.handle, _ptr(u0, n), _ptr(v0, n)))

    def set_ic_reduced(self, uh0, vh0=None, s0=None):
        """ROM: u^0, v^0 (batch, r) and s0 (batch, n_s) given directly (osam_set_ic_reduced)."""
        n = self.r * self.batch
        _check(lib().osam_set_ic_reduced(self.handle, _ptr(uh0, n), _ptr(vh0, n),
                                         _ptr(s0, None if s0 is None else self.n_s * self.batch)))

    def _state_size(self):
        return 3 * self.n_nodes if self.kind == OSAM_FOM else self.r * self.batch

    def get_state(self, u_out=None, v_out=None):
        n = self._state_size()
        _check(lib().osam_get_state(self.handle, _ptr(u_out, n), _ptr(v_out, n)))

    def get_accel(self, a_out):
        _check(lib().osam_get_accel(self.handle, _ptr(a_out, self._state_size())))

    def sizes(self):
        n, f, s = C.c_int64(), C.c_int64(), C.c_int64()
        b = C.c_int32()
        _check(lib().osam_get_sizes(self.handle, C.byref(n), C.byref(f), C.byref(s), C.byref(b)))
        return n.value, f.value, s.value, b.value

    def close(self):
        if getattr(self, "handle", None):
            lib().osam_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def osam_step(subdomains, dt, tol_rel, n_steps, max_iters=50, min_iters=2, tol_abs=0.0, iters_out=None):
    """osam_step over `subdomains` (sweep order); returns (status, iters [n_steps, batch])."""
    cfg = osam_schwarz_cfg(float(dt), float(tol_rel), float(tol_abs), int(max_iters), int(min_iters))
    arr = (C.c_void_p * len(subdomains))(*[s.handle for s in subdomains])
    B = max(s.batch for s in subdomains)
    if iters_out is None:
        iters_out = np.zeros((max(n_steps, 1), B), dtype=np.int32)
    elif not (isinstance(iters_out, np.ndarray) and iters_out.dtype == np.int32 and iters_out.flags.c_contiguous
              and iters_out.size >= n_steps * B):
        raise ValueError("iters_out must be a contiguous int32 array of at least n_steps x batch entries")
    ip = iters_out.ctypes.data_as(C.POINTER(C.c_int32)) if n_steps > 0 else None
    rc = _check(lib().osam_step(arr, len(subdomains), C.byref(cfg), int(n_steps), ip))
    return rc, iters_out[:n_steps]


def set_conv_trace(max_n):
    """Record (num, den) of every tested Schwarz iteration n <= max_n in later osam_step calls (0: off)."""
    lib().osam_set_conv_trace(int(max_n))


def get_conv_trace(subdomains):
    """Convergence trace of the last osam_step on this list: (n_steps, max_n, batch, 2) float64, NaN = not
    tested."""
    arr = (C.c_void_p * len(subdomains))(*[s.handle for s in subdomains])
    ns, T, B = C.c_int32(), C.c_int32(), C.c_int32()
    _check(lib().osam_get_conv_trace(arr, len(subdomains), None, C.byref(ns), C.byref(T), C.byref(B)))
    out = np.empty((ns.value, T.value, B.value, 2))
    if out.size:
        _check(lib().osam_get_conv_trace(arr, len(subdomains), _ptr(out), None, None, None))
    return out


def k1_timeline(subdomains, reset=False):
    """In-schedule K1 timeline of the group (osam_get_k1_timeline): dict(union_ms, sum_ms, launches, sweeps,
    tested_sweeps, bytes)."""
    arr = (C.c_void_p * len(subdomains))(*[s.handle for s in subdomains])
    out = (C.c_double * 6)()
    _check(lib().osam_get_k1_timeline(arr, len(subdomains), 1 if reset else 0, out))
    return dict(zip(("union_ms", "sum_ms", "launches", "sweeps", "tested_sweeps", "bytes"), list(out)))


def set_profiling(on):
    lib().osam_set_profiling(1 if on else 0)


def reset_profile():
    lib().osam_reset_profile()


def get_profile():
    ms, n, b, k = C.c_double(), C.c_int64(), C.c_double(), C.c_int64()
    lib().osam_get_profile(C.byref(ms), C.byref(n), C.byref(b), C.byref(k))
    return dict(k1_ms=ms.value, k1_launches=n.value, k1_bytes=b.value, kernel_launches=k.value)


def opinf_replay(O, Ubar, Ghat, dt, order=1, vh0=None, trajectories=False, stream=None):
    """osam_opinf_replay: O (n_models, r, r + r_b + nf) candidate operators [-Kbar|Bbar|-Hbar|-Cbar],
    Ubar (r, K) and Ghat (r_b, K) training data.  Returns (errors (n_models,), best index[, U^hat
    (n_models, K, r)])."""
    O = np.asarray(O, dtype=np.float64)
    B, r, _ = O.shape
    Ocm = np.ascontiguousarray(O.transpose(0, 2, 1))               # column-major blocks
    Ub = np.asfortranarray(Ubar, dtype=np.float64)
    Gh = np.asfortranarray(Ghat, dtype=np.float64)
    K = Ub.shape[1]
    v0 = None if vh0 is None else np.ascontiguousarray(vh0, dtype=np.float64)
    d = osam_replay_desc(r, Gh.shape[0], int(order), B, K, float(dt), Ocm.ctypes.data, Ub.ctypes.data,
                         Gh.ctypes.data if Gh.size else None, None if v0 is None else v0.ctypes.data)
    err = np.empty(B)
    best = C.c_int32(-2)
    traj = np.empty((B, K, r)) if trajectories else None
    _check(lib().osam_opinf_replay(C.byref(d), _ptr(err), C.byref(best), _ptr(traj), C.c_void_p(stream or 0)))
    return (err, best.value, traj) if trajectories else (err, best.value)
