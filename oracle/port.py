"""TEST INFRASTRUCTURE ONLY: ctypes driver for the C restatement ``ptp_oracle.c``.

The restatement is pinned against the unmodified reference (``oracle.ref``) and
the committed golden vectors in ``tests/golden/``.
"""

import ctypes as C
import os

import numpy as np

from . import PORT_SO

_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_lib = None


def available():
    return os.path.exists(PORT_SO)


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(PORT_SO)
        L.orc_last_error.restype = C.c_char_p
        L.orc_build_fans.argtypes = [C.c_int, _f64p, C.c_int, _i32p, _i32p, _i32p, _i32p, _i32p]
        L.orc_toplesets.argtypes = [C.c_int, _i32p, _i32p, _i32p, _i32p, C.c_int, _i32p, _i32p,
                                    _i32p, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        for sfx in ("f32", "f64"):
            getattr(L, "orc_planar_" + sfx).argtypes = [_f64p, _f64p, C.c_double, C.c_double,
                                                        C.POINTER(C.c_double), C.POINTER(C.c_int),
                                                        C.POINTER(C.c_int)]
        L.orc_ptp.argtypes = [C.c_int, _f64p, _i32p, _i32p, _i32p, _i32p, _i32p, C.c_int, _i32p,
                              _i32p, C.c_int, C.c_double, C.c_int, _f64p, C.c_void_p, _i64p,
                              C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]
        L.orc_fps.argtypes = [C.c_int, _f64p, _i32p, _i32p, _i32p, _i32p, C.c_int, C.c_int,
                              C.c_double, C.c_int, _i32p, _i32p, C.POINTER(C.c_double), _i64p,
                              _f64p]
        _lib = L
    return _lib


def _check(rc):
    if rc == 1:
        raise ValueError(lib().orc_last_error().decode())
    if rc != 0:
        raise RuntimeError(lib().orc_last_error().decode())


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def planar(x1, x2, t1, t2, single=False):
    v, s, d = C.c_double(), C.c_int(), C.c_int()
    fn = lib().orc_planar_f32 if single else lib().orc_planar_f64
    fn(np.ascontiguousarray(x1, np.float64), np.ascontiguousarray(x2, np.float64), float(t1),
       float(t2), C.byref(v), C.byref(s), C.byref(d))
    return v.value, s.value, bool(d.value)


class PortMesh:
    def __init__(self, vertices, faces):
        self.xyz = np.ascontiguousarray(vertices, np.float64).reshape(-1)
        self.faces = np.ascontiguousarray(faces, np.int32).reshape(-1)
        self.n = len(self.xyz) // 3
        self.nf = len(self.faces) // 3
        self.cptr = np.zeros(self.n + 1, np.int32)
        self.cv1 = np.zeros(max(3 * self.nf, 1), np.int32)
        self.cv2 = np.zeros(max(3 * self.nf, 1), np.int32)
        self.extra = np.zeros(max(self.n, 1), np.int32)
        _check(lib().orc_build_fans(self.n, self.xyz, self.nf, self.faces, self.cptr, self.cv1,
                                    self.cv2, self.extra))

    def fan(self, v):
        a, b = self.cptr[v], self.cptr[v + 1]
        return self.cv1[a:b].copy(), self.cv2[a:b].copy(), int(self.extra[v])

    def toplesets(self, sources):
        s = np.ascontiguousarray(sources, np.int32)
        srt = np.empty(self.n, np.int32)
        lim = np.empty(self.n + 1, np.int32)
        pos = np.empty(self.n, np.int32)
        rho, unr = C.c_int(), C.c_int()
        _check(lib().orc_toplesets(self.n, self.cptr, self.cv1, self.extra, s, len(s), srt, lim,
                                   pos, C.byref(rho), C.byref(unr)))
        reach = self.n - unr.value
        return {"sorted": srt[:reach].copy(), "limits": lim[:rho.value + 1].copy(),
                "position": pos, "rho": rho.value, "unreached": unr.value}

    def ptp(self, sources, epsilon=1e-3, precision="double", labels=False, trace=False,
            ordering=None):
        s = np.ascontiguousarray(sources, np.int32)
        o = ordering if ordering is not None else self.toplesets(s)
        dist = np.empty(self.n, np.float64)
        lab = np.empty(self.n, np.int32)
        stats = np.zeros(3, np.int64)
        cap = 4 * self.n + 64 if trace else 0
        ti = np.zeros(4 * cap, np.int64) if trace else None
        tf = np.zeros(cap, np.float64) if trace else None
        tc = np.zeros(cap, np.int32) if trace else None
        lc = np.zeros(self.n, np.int32) if trace else None
        _check(lib().orc_ptp(self.n, self.xyz, self.cptr, self.cv1, self.cv2,
                             np.ascontiguousarray(o["sorted"], np.int32),
                             np.ascontiguousarray(o["limits"], np.int32), len(o["limits"]) - 1,
                             np.ascontiguousarray(o["position"], np.int32), s, len(s), epsilon,
                             int(precision == "single"), dist, _ptr(lab), stats, _ptr(ti), _ptr(tf),
                             _ptr(tc), cap, _ptr(lc)))
        out = {"distances": dist, "relax_calls": int(stats[0]), "degenerate_calls": int(stats[1]),
               "iterations": int(stats[2]), "rho": len(o["limits"]) - 1,
               "unreached": self.n - len(o["sorted"])}
        if labels:
            out["labels"] = lab
        if trace:
            K = int(stats[2])
            out["trace"] = {"kijU": ti[:4 * K].reshape(K, 4), "max_rel": tf[:K],
                            "converged": tc[:K].astype(bool)}
            out["last_change"] = lc
        return out

    def fps(self, count, seed=0, epsilon=1e-3, precision="double"):
        samples = np.empty(max(count, 1), np.int32)
        lab = np.empty(self.n, np.int32)
        rad = C.c_double()
        hi = np.zeros(4 * max(count, 1), np.int64)
        hf = np.zeros(max(count, 1), np.float64)
        _check(lib().orc_fps(self.n, self.xyz, self.cptr, self.cv1, self.cv2, self.extra, count,
                             seed, epsilon, int(precision == "single"), samples, lab,
                             C.byref(rad), hi, hf))
        hist = [{"sources": int(hi[4 * q]), "rho": int(hi[4 * q + 1]),
                 "relax_calls": int(hi[4 * q + 2]), "picked": int(hi[4 * q + 3]),
                 "radius": float(hf[q])} for q in range(count)]
        return {"samples": samples[:count].copy(), "labels": lab, "radius": rad.value,
                "history": hist}
