"""TEST INFRASTRUCTURE ONLY: ctypes driver for the unmodified reference library.

Wraps ``oracle/_ref/libgeodist_ref.so`` (reference sources + ``ref_capi.cpp``).
Every call mirrors one reference entry point; see ``ref_capi.cpp`` for the
file:line of each.
"""

import ctypes as C
import os

import numpy as np

from . import REF_SO

_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")

_lib = None


def available():
    return os.path.exists(REF_SO)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError(f"reference oracle not built: {REF_SO} (run make -C oracle ref)")
        L = C.CDLL(REF_SO)
        L.ref_last_error.restype = C.c_char_p
        L.ref_max_threads.restype = C.c_int
        L.ref_mesh_create.argtypes = [_f64p, C.c_int, _i32p, C.c_int, C.POINTER(C.c_void_p),
                                      C.POINTER(C.c_double)]
        L.ref_mesh_destroy.argtypes = [C.c_void_p]
        L.ref_load_mesh.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
        L.ref_write_mesh.argtypes = [C.c_void_p, C.c_char_p, C.c_int]
        L.ref_generate_grid.argtypes = [C.c_int, C.c_int, C.c_double, C.POINTER(C.c_void_p)]
        L.ref_generate_icosphere.argtypes = [C.c_int, C.POINTER(C.c_void_p)]
        L.ref_generate_torus.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double,
                                         C.POINTER(C.c_void_p)]
        L.ref_perturb_radial.argtypes = [C.c_void_p, C.c_double, C.c_uint]
        L.ref_heightfield.argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_double]
        L.ref_mesh_sizes.argtypes = [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.ref_mesh_copy.argtypes = [C.c_void_p, _f64p, _i32p]
        L.ref_fan.argtypes = [C.c_void_p, C.c_int, _i32p, _i32p, C.c_int, C.POINTER(C.c_int)]
        L.ref_toplesets.argtypes = [C.c_void_p, _i32p, C.c_int, _i32p, _i32p, _i32p,
                                    C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int),
                                    C.POINTER(C.c_double)]
        L.ref_reorder.argtypes = [C.c_void_p, _i32p, C.c_int, _i32p, _i32p, _i32p]
        L.ref_ptp.argtypes = [C.c_void_p, _i32p, C.c_int, C.c_double, C.c_int, C.c_int, C.c_int,
                              C.c_int, _f64p, _i32p, _i64p, _f64p, _i64p, _f64p, _i32p, C.c_int,
                              _i32p]
        L.ref_ptp_ordered.argtypes = [C.c_void_p, _i32p, C.c_int, _i32p, C.c_int, _i32p, C.c_int,
                                      _i32p, C.c_double, C.c_int, C.c_int, C.c_int, _f64p, _i32p,
                                      _i64p]
        L.ref_fps.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, _i32p,
                              _i32p, C.POINTER(C.c_double), _i64p, _f64p, C.POINTER(C.c_double)]
        L.ref_voronoi.argtypes = [C.c_void_p, _i32p, C.c_int, C.c_double, C.c_int, C.c_int, _i32p]
        L.ref_planar.argtypes = [_f64p, _f64p, C.c_double, C.c_double, C.c_int,
                                 C.POINTER(C.c_double), C.POINTER(C.c_int), C.POINTER(C.c_int)]
        _lib = L
    return _lib


class RefError(Exception):
    pass


def _check(rc):
    if rc == 1:
        raise ValueError(lib().ref_last_error().decode())
    if rc != 0:
        raise RuntimeError(lib().ref_last_error().decode())


def max_threads():
    return lib().ref_max_threads()


def planar(x1, x2, t1, t2, single=False):
    v, s, d = C.c_double(), C.c_int(), C.c_int()
    lib().ref_planar(np.ascontiguousarray(x1, np.float64), np.ascontiguousarray(x2, np.float64),
                     float(t1), float(t2), int(single), C.byref(v), C.byref(s), C.byref(d))
    return v.value, s.value, bool(d.value)


class RefMesh:
    """Reference TriangleMesh + Connectivity (built once, like bindings.cpp:26-31)."""

    def __init__(self, handle):
        self.h = handle
        n, f = C.c_int(), C.c_int()
        lib().ref_mesh_sizes(self.h, C.byref(n), C.byref(f))
        self.n, self.nf = n.value, f.value
        self.build_seconds = None

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ref_mesh_destroy(self.h)
            self.h = None

    @classmethod
    def from_arrays(cls, vertices, faces):
        v = np.ascontiguousarray(vertices, np.float64).reshape(-1)
        f = np.ascontiguousarray(faces, np.int32).reshape(-1)
        h, secs = C.c_void_p(), C.c_double()
        _check(lib().ref_mesh_create(v, len(v) // 3, f, len(f) // 3, C.byref(h), C.byref(secs)))
        m = cls(h)
        m.build_seconds = secs.value
        return m

    @classmethod
    def load(cls, path):
        """geodist::load_mesh (mesh_io.cpp): arrays() only -- no connectivity is built."""
        h = C.c_void_p()
        _check(lib().ref_load_mesh(str(path).encode(), C.byref(h)))
        return cls(h)

    def write(self, path, obj=False):
        _check(lib().ref_write_mesh(self.h, str(path).encode(), int(bool(obj))))

    @classmethod
    def grid(cls, nx, ny, shear=0.0):
        h = C.c_void_p()
        _check(lib().ref_generate_grid(nx, ny, shear, C.byref(h)))
        return cls(h)

    @classmethod
    def icosphere(cls, subdiv):
        h = C.c_void_p()
        _check(lib().ref_generate_icosphere(subdiv, C.byref(h)))
        return cls(h)

    @classmethod
    def torus(cls, nu, nv, R=3.0, r=1.0):
        """SURVEY §8d configs 4/5 torus, generated on the reference's own types (ref_capi.cpp)."""
        h = C.c_void_p()
        _check(lib().ref_generate_torus(nu, nv, float(R), float(r), C.byref(h)))
        return cls(h)

    @classmethod
    def noisy_icosphere(cls, subdiv, sigma, seed=1):
        """generate_icosphere, then p *= 1 + sigma*N(0,1), mt19937(seed)."""
        m = cls.icosphere(subdiv)
        lib().ref_perturb_radial(m.h, float(sigma), int(seed))
        return m

    @classmethod
    def heightfield(cls, nx, ny, amp=20.0, wx=97.0, wy=131.0):
        """generate_grid(nx, ny), z = amp sin(x/wx) cos(y/wy)."""
        m = cls.grid(nx, ny, 0.0)
        lib().ref_heightfield(m.h, float(amp), float(wx), float(wy))
        return m

    def arrays(self):
        v = np.empty(self.n * 3, np.float64)
        f = np.empty(self.nf * 3, np.int32)
        lib().ref_mesh_copy(self.h, v, f)
        return v.reshape(-1, 3), f.reshape(-1, 3)

    def fan(self, v, cap=256):
        a = np.empty(cap, np.int32)
        b = np.empty(cap, np.int32)
        extra = C.c_int()
        c = lib().ref_fan(self.h, v, a, b, cap, C.byref(extra))
        if c < 0:
            raise ValueError("fan larger than cap")
        return a[:c].copy(), b[:c].copy(), extra.value

    def toplesets(self, sources):
        s = np.ascontiguousarray(sources, np.int32)
        srt = np.empty(self.n, np.int32)
        lim = np.empty(self.n + 1, np.int32)
        pos = np.empty(self.n, np.int32)
        rho, unr, reach, secs = C.c_int(), C.c_int(), C.c_int(), C.c_double()
        _check(lib().ref_toplesets(self.h, s, len(s), srt, lim, pos, C.byref(rho), C.byref(unr),
                                   C.byref(reach), C.byref(secs)))
        return {"sorted": srt[:reach.value].copy(), "limits": lim[:rho.value + 1].copy(),
                "position": pos, "rho": rho.value, "unreached": unr.value, "seconds": secs.value}

    def reorder(self, sources):
        s = np.ascontiguousarray(sources, np.int32)
        oon = np.empty(self.n, np.int32)
        noo = np.empty(self.n, np.int32)
        faces = np.empty(self.nf * 3, np.int32)
        _check(lib().ref_reorder(self.h, s, len(s), oon, noo, faces))
        return oon, noo, faces.reshape(-1, 3)

    def ptp(self, sources, epsilon=1e-3, precision="double", labels=False, trace=False,
            workers=0, trace_cap=None):
        s = np.ascontiguousarray(sources, np.int32)
        dist = np.empty(self.n, np.float64)
        lab = np.empty(self.n if labels else 1, np.int32)
        stats = np.zeros(6, np.int64)
        secs = np.zeros(2, np.float64)
        cap = trace_cap if trace_cap is not None else (4 * self.n + 64 if trace else 1)
        ti = np.zeros(4 * cap, np.int64)
        tf = np.zeros(cap, np.float64)
        tc = np.zeros(cap, np.int32)
        lc = np.zeros(self.n if trace else 1, np.int32)
        _check(lib().ref_ptp(self.h, s, len(s), epsilon, int(precision == "single"), int(labels),
                             int(trace), workers, dist, lab, stats, secs, ti, tf, tc, cap, lc))
        out = {"distances": dist, "relax_calls": int(stats[0]), "degenerate_calls": int(stats[1]),
               "iterations": int(stats[2]), "workers": int(stats[3]), "rho": int(stats[4]),
               "unreached": int(stats[5]), "wall_seconds": float(secs[0]),
               "toplesets_seconds": float(secs[1])}
        if labels:
            out["labels"] = lab
        if trace:
            K = min(int(stats[2]), cap)
            out["trace"] = {"kijU": ti[:4 * K].reshape(K, 4), "max_rel": tf[:K],
                            "converged": tc[:K].astype(bool)}
            out["last_change"] = lc
        return out

    def ptp_ordered(self, sources, sorted_, limits, position, epsilon=1e-3, precision="double",
                    labels=False, workers=0):
        s = np.ascontiguousarray(sources, np.int32)
        srt = np.ascontiguousarray(sorted_, np.int32)
        lim = np.ascontiguousarray(limits, np.int32)
        pos = np.ascontiguousarray(position, np.int32)
        dist = np.empty(self.n, np.float64)
        lab = np.empty(self.n if labels else 1, np.int32)
        stats = np.zeros(4, np.int64)
        _check(lib().ref_ptp_ordered(self.h, s, len(s), srt, len(srt), lim, len(lim) - 1, pos,
                                     epsilon, int(precision == "single"), int(labels), workers,
                                     dist, lab, stats))
        out = {"distances": dist, "relax_calls": int(stats[0]), "iterations": int(stats[2])}
        if labels:
            out["labels"] = lab
        return out

    def fps(self, count, seed=0, epsilon=1e-3, precision="double", workers=0):
        samples = np.empty(max(count, 1), np.int32)
        lab = np.empty(self.n, np.int32)
        rad, secs = C.c_double(), C.c_double()
        hi = np.zeros(4 * max(count, 1), np.int64)
        hf = np.zeros(max(count, 1), np.float64)
        _check(lib().ref_fps(self.h, count, seed, epsilon, int(precision == "single"), workers,
                             samples, lab, C.byref(rad), hi, hf, C.byref(secs)))
        hist = [{"sources": int(hi[4 * q]), "rho": int(hi[4 * q + 1]),
                 "relax_calls": int(hi[4 * q + 2]), "picked": int(hi[4 * q + 3]),
                 "radius": float(hf[q])} for q in range(count)]
        return {"samples": samples[:count].copy(), "labels": lab, "radius": rad.value,
                "history": hist, "seconds": secs.value}

    def voronoi(self, samples, epsilon=1e-3, precision="double", workers=0):
        s = np.ascontiguousarray(samples, np.int32)
        lab = np.empty(self.n, np.int32)
        _check(lib().ref_voronoi(self.h, s, len(s), epsilon, int(precision == "single"), workers,
                                 lab))
        return lab
