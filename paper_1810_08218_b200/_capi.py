"""ctypes binding of the C ABI declared in ``include/geodist_b200.h``.

Loads the in-tree ``libgeodist_b200.so`` (built for sm_100a by ``csrc/Makefile``).
There is no fallback: if the library is missing every call raises.
"""

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# GEODIST_B200_LIB: another in-tree build of the same C ABI (the tests load the alternative
# layouts' build, libgeodist_b200_alt.so, this way)
LIB_PATH = os.environ.get("GEODIST_B200_LIB") or os.path.join(HERE, "libgeodist_b200.so")

GEODIST_OK, GEODIST_EINVAL, GEODIST_EMESH, GEODIST_ECUDA, GEODIST_ENOMEM = range(5)

# Every symbol include/geodist_b200.h declares (checked by tests/test_capi_symbols.py).
EXPORTED = [
    "geodist_last_error", "geodist_version", "geodist_device_count", "geodist_mesh_create",
    "geodist_mesh_destroy", "geodist_mesh_sizes", "geodist_mesh_degrees", "geodist_mesh_fan",
    "geodist_mesh_fans",
    "geodist_meshfile_load", "geodist_meshfile_copy", "geodist_meshfile_free", "geodist_write_mesh",
    "geodist_build_fans", "geodist_validate_mesh", "geodist_build_halfedges", "geodist_grid_sizes", "geodist_generate_grid", "geodist_icosphere_sizes",
    "geodist_generate_icosphere", "geodist_perturb_radial", "geodist_torus_sizes",
    "geodist_generate_torus", "geodist_heightfield", "geodist_toplesets",
    "geodist_reorder_for_bands", "geodist_reorder_ordered", "geodist_ptp", "geodist_ptp_ordered",
    "geodist_voronoi",
    "geodist_fps", "geodist_batch_device", "geodist_batch", "geodist_planar_update",
    "geodist_kernel_launches", "geodist_selftest_arith", "geodist_reset_persisting_l2",
]


class PtpConfig(C.Structure):
    _fields_ = [("epsilon", C.c_double), ("precision", C.c_int32), ("workers", C.c_int32),
                ("with_labels", C.c_int32), ("record_trace", C.c_int32)]


class PtpStats(C.Structure):
    _fields_ = [("relax_calls", C.c_int64), ("degenerate_calls", C.c_int64),
                ("vertex_updates", C.c_int64), ("iterations", C.c_int32), ("rho", C.c_int32),
                ("unreached", C.c_int32), ("workers", C.c_int32), ("wall_seconds", C.c_double),
                ("total_seconds", C.c_double)]


class BandRow(C.Structure):
    _fields_ = [("k", C.c_int32), ("i", C.c_int32), ("j", C.c_int32),
                ("front_converged", C.c_int32), ("updated", C.c_int64),
                ("max_rel_change", C.c_double)]


class FpsRow(C.Structure):
    _fields_ = [("sources", C.c_int32), ("rho", C.c_int32), ("relax_calls", C.c_int64),
                ("radius", C.c_double), ("picked", C.c_int32), ("iterations", C.c_int32)]


OBSERVER = C.CFUNCTYPE(None, C.c_void_p, C.c_int32, C.POINTER(C.c_double), C.c_int32)

_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_vp = C.c_void_p
_lib = None


def lib():
    """The loaded C ABI library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                "(the B200 solver has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        L.geodist_last_error.restype = C.c_char_p
        L.geodist_version.restype = C.c_int32
        L.geodist_kernel_launches.restype = C.c_int64
        L.geodist_device_count.argtypes = [C.POINTER(C.c_int32)]
        L.geodist_mesh_create.argtypes = [_f64p, C.c_int32, _i32p, C.c_int32, C.c_int32,
                                          C.POINTER(_vp)]
        L.geodist_mesh_destroy.argtypes = [_vp]
        L.geodist_mesh_sizes.argtypes = [_vp, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                         C.POINTER(C.c_int64)]
        L.geodist_mesh_degrees.argtypes = [_vp, _i32p]
        L.geodist_mesh_fan.argtypes = [_vp, C.c_int32, _i32p, _i32p, C.c_int32,
                                       C.POINTER(C.c_int32)]
        L.geodist_mesh_fans.argtypes = [_vp, _i32p, _i32p, _i32p]
        L.geodist_selftest_arith.argtypes = [C.c_int64, C.c_uint64,
                                             np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")]
        L.geodist_meshfile_load.argtypes = [C.c_char_p, C.POINTER(C.c_void_p),
                                            C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
        L.geodist_meshfile_copy.argtypes = [_vp, _f64p, _i32p]
        L.geodist_meshfile_free.argtypes = [_vp]
        L.geodist_write_mesh.argtypes = [C.c_char_p, _f64p, C.c_int32, _i32p, C.c_int32,
                                         C.c_int32]
        L.geodist_build_fans.argtypes = [_f64p, C.c_int32, _i32p, C.c_int32, _i32p, _i32p, _vp]
        L.geodist_validate_mesh.argtypes = [_f64p, C.c_int32, _i32p, C.c_int32]
        L.geodist_build_halfedges.argtypes = [_vp, C.c_int32, _i32p, C.c_int32, _i32p, _i32p]
        L.geodist_grid_sizes.argtypes = [C.c_int32, C.c_int32, C.POINTER(C.c_int32),
                                         C.POINTER(C.c_int32)]
        L.geodist_generate_grid.argtypes = [C.c_int32, C.c_int32, C.c_double, _f64p, _i32p]
        L.geodist_icosphere_sizes.argtypes = [C.c_int32, C.POINTER(C.c_int32),
                                              C.POINTER(C.c_int32)]
        L.geodist_generate_icosphere.argtypes = [C.c_int32, _f64p, _i32p]
        L.geodist_perturb_radial.argtypes = [_f64p, C.c_int32, C.c_double, C.c_uint32]
        L.geodist_torus_sizes.argtypes = [C.c_int32, C.c_int32, C.POINTER(C.c_int32),
                                          C.POINTER(C.c_int32)]
        L.geodist_generate_torus.argtypes = [C.c_int32, C.c_int32, C.c_double, C.c_double, _f64p,
                                             _i32p]
        L.geodist_heightfield.argtypes = [_f64p, C.c_int32, C.c_double, C.c_double, C.c_double]
        L.geodist_toplesets.argtypes = [_vp, _i32p, C.c_int32, _vp, _vp, _vp,
                                        C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
        L.geodist_reorder_for_bands.argtypes = [_vp, _i32p, C.c_int32, _vp, _vp, _vp]
        L.geodist_reorder_ordered.argtypes = [_vp, _i32p, C.c_int32, _i32p, _vp, _vp, _vp, _vp]
        L.geodist_ptp.argtypes = [_vp, _i32p, C.c_int32, C.POINTER(PtpConfig), _vp, _vp,
                                  C.POINTER(PtpStats), _vp, C.c_int32, _vp, OBSERVER, _vp]
        L.geodist_ptp_ordered.argtypes = [_vp, _i32p, C.c_int32, _i32p, C.c_int32, _i32p,
                                          C.c_int32, _i32p, C.POINTER(PtpConfig), _vp, _vp,
                                          C.POINTER(PtpStats), _vp, C.c_int32, _vp, OBSERVER, _vp]
        L.geodist_voronoi.argtypes = [_vp, _i32p, C.c_int32, C.POINTER(PtpConfig), _i32p]
        L.geodist_fps.argtypes = [_vp, C.c_int32, C.c_int32, C.POINTER(PtpConfig), _i32p, _i32p,
                                  C.POINTER(C.c_double), _vp]
        L.geodist_batch_device.argtypes = [_vp, _i32p, _i32p, C.c_int32, C.POINTER(PtpConfig),
                                           _vp, _vp, _vp, C.c_int32, _vp]
        L.geodist_batch.argtypes = [_vp, _i32p, _i32p, C.c_int32, C.POINTER(PtpConfig), _vp, _vp,
                                    _vp, C.c_int32]
        L.geodist_planar_update.argtypes = [_f64p, _f64p, _f64p, _f64p, C.c_int32, C.c_int32,
                                            _f64p, _i32p, _i32p]
        _lib = L
    return _lib


def check(rc):
    """Map a geodist_status to the reference's Python exception types."""
    if rc == GEODIST_OK:
        return
    msg = lib().geodist_last_error().decode()
    if rc == GEODIST_EINVAL:
        raise ValueError(msg)
    if rc == GEODIST_EMESH:
        raise RuntimeError(msg)
    if rc == GEODIST_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"CUDA: {msg}")


def ptr(a):
    return None if a is None else a.ctypes.data_as(_vp)


def kernel_launches():
    return int(lib().geodist_kernel_launches())
