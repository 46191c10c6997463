"""B200-native Parallel Toplesets Propagation (arXiv 1810.08218).

Drop-in for the reference's Python module ``geodist`` (``python/bindings.cpp``
and ``python/geodist/__init__.py`` of /root/reference/proj): the same entry
points, argument names, defaults, return dictionaries and exception types, but
every distance field is computed by hand-written sm_100a kernels through the
C ABI in ``include/geodist_b200.h`` (``libgeodist_b200.so``).  A ``Mesh`` owns
a device-resident replica (fan-CSR + per-precision geometry tables) built
once, like the reference's ``MeshHandle`` owns its ``Connectivity``.

There is no CPU fallback: without the library or an sm_100 GPU the compute
entry points raise.
"""

import ctypes as C
import os

import numpy as np

from . import _capi
from ._capi import check, lib, ptr

__all__ = [
    "Mesh", "farthest_point_sampling", "generate_grid", "generate_icosphere", "generate_torus",
    "geodesics", "grid_reference", "heightfield_grid", "load_mesh", "read_mesh", "write_mesh",
    "mape", "mesh_from_arrays",
    "noisy_icosphere", "sphere_reference", "toplesets", "voronoi", "reorder_for_bands",
    "batch_geodesics", "planar_update", "device_count",
]

__version__ = "0.1.0"

_PRECISION = {"single": 0, "double": 1}


def device_count():
    c = C.c_int32()
    check(lib().geodist_device_count(C.byref(c)))
    return c.value


class Mesh:
    """Mesh plus its device replica (reference ``MeshHandle``, bindings.cpp:26-31)."""

    def __init__(self, vertices, faces, device=0):
        v = np.ascontiguousarray(vertices, dtype=np.float64).reshape(-1, 3)
        f = np.ascontiguousarray(faces, dtype=np.int32).reshape(-1, 3)
        self._v, self._f = v, f
        self.device = device
        h = C.c_void_p()
        check(lib().geodist_mesh_create(v.reshape(-1), len(v), f.reshape(-1), len(f), device,
                                        C.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _capi is not None and getattr(_capi, "_lib", None) is not None:
            _capi._lib.geodist_mesh_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    @property
    def n_vertices(self):
        return len(self._v)

    @property
    def n_faces(self):
        return len(self._f)

    def vertices(self):
        return self._v.copy()

    def faces(self):
        return self._f.copy()

    def degree_histogram(self):
        deg = np.empty(self.n_vertices, np.int32)
        check(lib().geodist_mesh_degrees(self._h, deg))
        vals, counts = np.unique(deg, return_counts=True)
        return {int(a): int(b) for a, b in zip(vals, counts)}

    def fan(self, v, cap=1024):
        a = np.empty(cap, np.int32)
        b = np.empty(cap, np.int32)
        cnt = C.c_int32()
        check(lib().geodist_mesh_fan(self._h, int(v), a, b, cap, C.byref(cnt)))
        return a[:cnt.value].copy(), b[:cnt.value].copy()

    def fans(self):
        """The mesh's fan-CSR as built (on the device): (cptr[n+1], ring[3F+n], degree[n]),
        the layout of :func:`build_fans`."""
        n = self.n_vertices
        cptr = np.empty(n + 1, np.int32)
        ring = np.empty(3 * self.n_faces + n + 1, np.int32)
        deg = np.empty(max(n, 1), np.int32)
        check(lib().geodist_mesh_fans(self._h, cptr, ring, deg))
        return cptr, ring[:cptr[n] + n], deg[:n]

    def __repr__(self):
        return f"<geodist.Mesh with {self.n_vertices} vertices, {self.n_faces} faces>"


# ---------------------------------------------------------------------------
# generators (host fixtures; grid / icosphere bit-identical to mesh.cpp:36-105)

def build_fans(vertices, faces):
    """Host-only rotational fans (validation + for_each_incident_triangle order):
    returns (cptr[n+1], ring[cptr[n]+n], degree[n]); corner c of v is
    (ring[cptr[v]+v+c], ring[cptr[v]+v+c+1])."""
    v = np.ascontiguousarray(vertices, np.float64).reshape(-1)
    f = np.ascontiguousarray(faces, np.int32).reshape(-1)
    n, nf = len(v) // 3, len(f) // 3
    cptr = np.empty(n + 1, np.int32)
    ring = np.empty(3 * nf + n + 1, np.int32)
    deg = np.empty(max(n, 1), np.int32)
    check(lib().geodist_build_fans(v, n, f, nf, cptr, ring, ptr(deg)))
    return cptr, ring[:cptr[n] + n], deg[:n]


def grid_arrays(nx, ny, shear=0.0):
    n, f = C.c_int32(), C.c_int32()
    check(lib().geodist_grid_sizes(nx, ny, C.byref(n), C.byref(f)))
    v = np.empty(3 * n.value, np.float64)
    fa = np.empty(max(3 * f.value, 1), np.int32)
    check(lib().geodist_generate_grid(nx, ny, float(shear), v, fa))
    return v.reshape(-1, 3), fa[:3 * f.value].reshape(-1, 3)


def icosphere_arrays(subdiv):
    n, f = C.c_int32(), C.c_int32()
    check(lib().geodist_icosphere_sizes(subdiv, C.byref(n), C.byref(f)))
    v = np.empty(3 * n.value, np.float64)
    fa = np.empty(3 * f.value, np.int32)
    check(lib().geodist_generate_icosphere(subdiv, v, fa))
    return v.reshape(-1, 3), fa.reshape(-1, 3)


def torus_arrays(nu, nv, R=3.0, r=1.0):
    n, f = C.c_int32(), C.c_int32()
    check(lib().geodist_torus_sizes(nu, nv, C.byref(n), C.byref(f)))
    v = np.empty(3 * n.value, np.float64)
    fa = np.empty(3 * f.value, np.int32)
    check(lib().geodist_generate_torus(nu, nv, float(R), float(r), v, fa))
    return v.reshape(-1, 3), fa.reshape(-1, 3)


def noisy_icosphere_arrays(subdiv, sigma, seed=1):
    """p *= 1 + sigma*N(0,1), std::mt19937(seed)."""
    v, f = icosphere_arrays(subdiv)
    flat = np.ascontiguousarray(v.reshape(-1))
    check(lib().geodist_perturb_radial(flat, len(v), float(sigma), int(seed)))
    return flat.reshape(-1, 3), f


def heightfield_arrays(nx, ny, amp=20.0, wx=97.0, wy=131.0):
    """z = amp * sin(x/wx) * cos(y/wy) over generate_grid(nx, ny)."""
    v, f = grid_arrays(nx, ny, 0.0)
    flat = np.ascontiguousarray(v.reshape(-1))
    check(lib().geodist_heightfield(flat, len(v), float(amp), float(wx), float(wy)))
    return flat.reshape(-1, 3), f


def generate_grid(nx, ny, shear=0.0, device=0):
    return Mesh(*grid_arrays(nx, ny, shear), device=device)


def generate_icosphere(subdiv, device=0):
    return Mesh(*icosphere_arrays(subdiv), device=device)


def generate_torus(nu, nv, R=3.0, r=1.0, device=0):
    return Mesh(*torus_arrays(nu, nv, R, r), device=device)


def noisy_icosphere(subdiv, sigma, seed=1, device=0):
    return Mesh(*noisy_icosphere_arrays(subdiv, sigma, seed), device=device)


def heightfield_grid(nx, ny, amp=20.0, wx=97.0, wy=131.0, device=0):
    return Mesh(*heightfield_arrays(nx, ny, amp, wx, wy), device=device)


def mesh_from_arrays(vertices, faces, device=0):
    v = np.asarray(vertices)
    f = np.asarray(faces)
    if v.ndim != 2 or v.shape[1] != 3:
        raise ValueError("vertices must have shape (n, 3)")
    if f.ndim != 2 or f.shape[1] != 3:
        raise ValueError("faces must have shape (m, 3)")
    return Mesh(v, f, device=device)


def read_mesh(path):
    """Parse an ASCII OFF / OBJ file (load_mesh, mesh_io.cpp:119-139: format from the
    extension, triangles only, validated) into (vertices float64 (n,3), faces int32 (m,3)).
    Host-only: the native reader in csrc/mesh_io.cpp; errors raise RuntimeError with the
    reference's message."""
    h = C.c_void_p()
    n, nf = C.c_int32(), C.c_int32()
    check(lib().geodist_meshfile_load(os.fsencode(str(path)), C.byref(h), C.byref(n), C.byref(nf)))
    try:
        v = np.empty(3 * n.value + 1, np.float64)
        f = np.empty(3 * nf.value + 1, np.int32)
        check(lib().geodist_meshfile_copy(h, v, f))
    finally:
        lib().geodist_meshfile_free(h)
    return v[:3 * n.value].reshape(-1, 3), f[:3 * nf.value].reshape(-1, 3)


def load_mesh(path, device=0):
    """Mesh from an OFF / OBJ file (bindings.cpp load_mesh)."""
    v, f = read_mesh(path)
    return Mesh(v, f, device=device)


def write_mesh(path, vertices, faces, fmt=None):
    """write_mesh (mesh_io.cpp:141-156): "%.17g" coordinates, OFF or OBJ (from the
    extension unless fmt is 'off' / 'obj')."""
    if fmt is None:
        fmt = "obj" if str(path).lower().endswith(".obj") else "off"
    v = np.ascontiguousarray(vertices, np.float64).reshape(-1)
    f = np.ascontiguousarray(faces, np.int32).reshape(-1)
    check(lib().geodist_write_mesh(os.fsencode(str(path)), v, len(v) // 3, f, len(f) // 3,
                                   1 if fmt == "obj" else 0))


# ---------------------------------------------------------------------------
# solver entry points (bindings.cpp:134-231)

def _config(epsilon, precision, workers, labels, trace=False):
    if precision not in _PRECISION:
        raise ValueError("precision must be 'single' or 'double'")
    return _capi.PtpConfig(float(epsilon), _PRECISION[precision], int(workers), int(bool(labels)),
                           int(bool(trace)))


def _sources(sources):
    s = np.asarray(sources, dtype=np.int64).reshape(-1)
    # index_t is int32 (vec3.hpp:8): a wider value must not wrap onto another vertex
    bad = s[(s < np.iinfo(np.int32).min) | (s > np.iinfo(np.int32).max)]
    if bad.size:
        raise ValueError(f"compute_toplesets: source index {int(bad[0])} out of range")
    return np.ascontiguousarray(s.astype(np.int32))


def geodesics(mesh, sources, method="ptp", epsilon=1e-3, precision="double", workers=0,
              labels=False, trace=False, observer=None, out=None):
    """Distance map from a source set (bindings.cpp:134-175).

    Returns ``{"distances", "unreached", ["labels"], "iterations", "relax_calls",
    "workers"}`` plus the GPU-side counters ``degenerate_calls``,
    ``vertex_updates``, ``rho`` and ``device_seconds``.  ``trace=True`` adds the
    band trace rows and ``last_change`` (PtpConfig.record_trace); ``observer``
    is the IterationObserver ``f(k, distances)`` (double precision only).
    """
    if method != "ptp":
        if method in ("fm", "dijkstra"):
            raise NotImplementedError(
                f"method={method!r}: the sequential CPU baselines are outside the B200 hot path")
        raise ValueError("method must be 'ptp', 'fm' or 'dijkstra'")
    cfg = _config(epsilon, precision, workers, labels, trace)
    src = _sources(sources)
    n = mesh.n_vertices
    dist = np.empty(n, np.float64) if out is None else out
    if dist.dtype != np.float64 or dist.shape != (n,) or not dist.flags.c_contiguous:
        raise ValueError("out must be a contiguous float64 array of n_vertices")
    lab = np.empty(n, np.int32) if labels else None
    stats = _capi.PtpStats()
    cap = 0
    rows = lc = None
    if trace:
        cap = 4 * n + 64
        rows = (_capi.BandRow * cap)()
        lc = np.zeros(n, np.int32)
    cb = _capi.OBSERVER(0)
    if observer is not None:
        def _obs(user, k, data, count):
            observer(int(k), np.ctypeslib.as_array(data, shape=(count,)).copy())
        cb = _capi.OBSERVER(_obs)
    check(lib().geodist_ptp(mesh.handle, src, len(src), C.byref(cfg), ptr(dist), ptr(lab),
                            C.byref(stats), C.cast(rows, C.c_void_p) if rows is not None else None,
                            cap, ptr(lc), cb, None))
    out = {"distances": dist, "unreached": int(stats.unreached)}
    if labels:
        out["labels"] = lab
    out["iterations"] = int(stats.iterations)
    out["relax_calls"] = int(stats.relax_calls)
    out["workers"] = int(stats.workers)
    out["degenerate_calls"] = int(stats.degenerate_calls)
    out["vertex_updates"] = int(stats.vertex_updates)
    out["rho"] = int(stats.rho)
    out["device_seconds"] = float(stats.wall_seconds)
    if trace:
        K = min(int(stats.iterations), cap)
        out["trace"] = [{"k": rows[q].k, "i": rows[q].i, "j": rows[q].j,
                         "updated": int(rows[q].updated), "max_rel_change": rows[q].max_rel_change,
                         "front_converged": bool(rows[q].front_converged)} for q in range(K)]
        out["last_change"] = lc
    return out


def geodesics_ordered(mesh, sources, ordering, epsilon=1e-3, precision="double", labels=False):
    """ptp_run with a caller-supplied ToplesetOrdering (ptp.hpp:70-72)."""
    cfg = _config(epsilon, precision, 0, labels)
    src = _sources(sources)
    srt = np.ascontiguousarray(ordering["sorted"], np.int32)
    lim = np.ascontiguousarray(ordering["limits"], np.int32)
    pos = np.ascontiguousarray(ordering["position"], np.int32)
    n = mesh.n_vertices
    dist = np.empty(n, np.float64)
    lab = np.empty(n, np.int32) if labels else None
    stats = _capi.PtpStats()
    check(lib().geodist_ptp_ordered(mesh.handle, src, len(src), srt, len(srt), lim, len(lim) - 1,
                                    pos, C.byref(cfg), ptr(dist), ptr(lab), C.byref(stats), None, 0,
                                    None, _capi.OBSERVER(0), None))
    out = {"distances": dist, "unreached": int(stats.unreached),
           "iterations": int(stats.iterations), "relax_calls": int(stats.relax_calls)}
    if labels:
        out["labels"] = lab
    return out


def toplesets(mesh, sources):
    """Breadth-first level sets (bindings.cpp:177-188), exact reference order."""
    src = _sources(sources)
    n = mesh.n_vertices
    srt = np.empty(n, np.int32)
    lim = np.empty(n + 1, np.int32)
    pos = np.empty(n, np.int32)
    rho, unr = C.c_int32(), C.c_int32()
    check(lib().geodist_toplesets(mesh.handle, src, len(src), ptr(srt), ptr(lim), ptr(pos),
                                  C.byref(rho), C.byref(unr)))
    reach = n - unr.value
    return {"sorted": srt[:reach].copy(), "limits": lim[:rho.value + 1].copy(), "rho": rho.value,
            "unreached": unr.value, "position": pos}


def reorder_for_bands(mesh, sources=None, ordering=None):
    """reorder_for_bands (toplesets.cpp:60-89): returns (permuted Mesh, old_of_new, new_of_old).

    From a source set (toplesets computed on the device), or from a caller's
    ``ordering`` dict with ``sorted`` and ``position`` (the reference signature's
    ToplesetOrdering, toplesets.hpp:45-46); positions are permuted on the device."""
    n, nf = mesh.n_vertices, mesh.n_faces
    oon = np.empty(n, np.int32)
    noo = np.empty(n, np.int32)
    faces = np.empty(max(3 * nf, 1), np.int32)
    if ordering is not None:
        srt = np.ascontiguousarray(ordering["sorted"], np.int32)
        pos = np.ascontiguousarray(ordering["position"], np.int32)
        if pos.shape != (n,):
            raise ValueError("reorder_for_bands: ordering built for a different mesh")
        verts = np.empty((n, 3), np.float64)
        check(lib().geodist_reorder_ordered(mesh.handle, srt, len(srt), pos, ptr(oon), ptr(noo),
                                            ptr(faces), ptr(verts)))
    else:
        src = _sources(sources)
        check(lib().geodist_reorder_for_bands(mesh.handle, src, len(src), ptr(oon), ptr(noo),
                                              ptr(faces)))
        verts = mesh._v[oon]
    return Mesh(verts, faces[:3 * nf].reshape(-1, 3), device=mesh.device), oon, noo


def farthest_point_sampling(mesh, count, seed=0, epsilon=1e-3, workers=0, precision="double"):
    """Farthest point sampling (bindings.cpp:190-217; sampling.cpp:11-49), on device."""
    cfg = _config(epsilon, precision, workers, True)
    samples = np.empty(max(int(count), 1), np.int32)
    lab = np.empty(mesh.n_vertices, np.int32)
    rad = C.c_double()
    hist = (_capi.FpsRow * max(int(count), 1))()
    check(lib().geodist_fps(mesh.handle, int(count), int(seed), C.byref(cfg), samples, lab,
                            C.byref(rad), C.cast(hist, C.c_void_p)))
    history = [{"sources": hist[q].sources, "rho": hist[q].rho,
                "relax_calls": int(hist[q].relax_calls), "radius": hist[q].radius,
                "picked": hist[q].picked, "iterations": hist[q].iterations}
               for q in range(int(count))]
    return {"samples": samples[:count].copy(), "labels": lab, "radius": rad.value,
            "history": history}


def voronoi(mesh, samples, epsilon=1e-3, workers=0, precision="double"):
    """Nearest-sample label per vertex (bindings.cpp:219-231)."""
    cfg = _config(epsilon, precision, workers, True)
    src = _sources(samples)
    lab = np.empty(mesh.n_vertices, np.int32)
    check(lib().geodist_voronoi(mesh.handle, src, len(src), C.byref(cfg), lab))
    return lab


def batch_geodesics(mesh, queries, epsilon=1e-3, precision="single", labels=False, groups=0):
    """Independent source sets; returns (distances[nq, n], stats list)."""
    qs = [np.asarray(q, np.int64).reshape(-1) for q in queries]
    off = np.zeros(len(qs) + 1, np.int32)
    off[1:] = np.cumsum([len(q) for q in qs])
    src = np.ascontiguousarray(np.concatenate(qs).astype(np.int32)) if qs else np.zeros(1, np.int32)
    n = mesh.n_vertices
    cfg = _config(epsilon, precision, 0, labels)
    dist = np.empty((len(qs), n), np.float64)
    lab = np.empty((len(qs), n), np.int32) if labels else None
    stats = (_capi.PtpStats * max(len(qs), 1))()
    check(lib().geodist_batch(mesh.handle, src, off, len(qs), C.byref(cfg), ptr(dist), ptr(lab),
                              C.cast(stats, C.c_void_p), int(groups)))
    st = [{"iterations": stats[q].iterations, "rho": stats[q].rho,
           "relax_calls": int(stats[q].relax_calls), "vertex_updates": int(stats[q].vertex_updates),
           "unreached": stats[q].unreached} for q in range(len(qs))]
    out = {"distances": dist, "stats": st}
    if labels:
        out["labels"] = lab
    return out


def batch_geodesics_device(mesh, queries, out_dist_ptr, epsilon=1e-3, precision="single",
                           out_labels_ptr=None, groups=0, stream=0):
    """Independent queries with results left in device memory (``out_dist_ptr``:
    nq*n elements of the run precision, e.g. a torch tensor's data_ptr()).
    Returns per-query stats; ``device_seconds`` is the CUDA-event time of the launch."""
    qs = [np.asarray(q, np.int64).reshape(-1) for q in queries]
    off = np.zeros(len(qs) + 1, np.int32)
    off[1:] = np.cumsum([len(q) for q in qs])
    src = np.ascontiguousarray(np.concatenate(qs).astype(np.int32))
    cfg = _config(epsilon, precision, 0, out_labels_ptr is not None)
    stats = (_capi.PtpStats * max(len(qs), 1))()
    check(lib().geodist_batch_device(mesh.handle, src, off, len(qs), C.byref(cfg),
                                     C.c_void_p(int(out_dist_ptr)),
                                     C.c_void_p(int(out_labels_ptr)) if out_labels_ptr else None,
                                     C.cast(stats, C.c_void_p), int(groups),
                                     C.c_void_p(int(stream)) if stream else None))
    return [{"iterations": stats[q].iterations, "rho": stats[q].rho,
             "relax_calls": int(stats[q].relax_calls),
             "vertex_updates": int(stats[q].vertex_updates), "unreached": stats[q].unreached,
             "device_seconds": float(stats[q].wall_seconds)} for q in range(len(qs))]


def planar_update(x1, x2, t1, t2, precision="double"):
    """planar_update<T> on the device for arrays of corners (test hook)."""
    x1 = np.ascontiguousarray(np.asarray(x1, np.float64).reshape(-1, 3))
    x2 = np.ascontiguousarray(np.asarray(x2, np.float64).reshape(-1, 3))
    t1 = np.ascontiguousarray(np.asarray(t1, np.float64).reshape(-1))
    t2 = np.ascontiguousarray(np.asarray(t2, np.float64).reshape(-1))
    cnt = len(t1)
    val = np.empty(cnt, np.float64)
    side = np.empty(cnt, np.int32)
    deg = np.empty(cnt, np.int32)
    check(lib().geodist_planar_update(x1.reshape(-1), x2.reshape(-1), t1, t2, cnt,
                                      _PRECISION[precision], val, side, deg))
    return val, side, deg.astype(bool)


# ---------------------------------------------------------------------------
# accuracy helpers (metrics.cpp:11-65; host post-processing, not on the hot path)

def mape(approx, exact, sources=()):
    approx = np.asarray(approx, np.float64)
    exact = np.asarray(exact, np.float64)
    if approx.shape != exact.shape:
        raise ValueError("mape: reference size mismatch")
    mask = np.ones(len(exact), bool)
    mask[np.asarray(list(sources), np.int64)] = False
    mask &= np.isfinite(approx) & (exact > 0.0)
    if not mask.any():
        raise RuntimeError("mape: no comparable vertices")
    rel = np.abs(approx[mask] - exact[mask]) / exact[mask]
    return {"mape": 100.0 * float(rel.mean()), "max_rel_error": 100.0 * float(rel.max()),
            "compared": int(mask.sum()), "excluded": int(len(exact) - mask.sum())}


def grid_reference(mesh, sources):
    v = mesh._v
    out = np.full(len(v), np.inf)
    for s in np.asarray(sources).reshape(-1):
        d = v - v[s]
        out = np.minimum(out, np.sqrt(d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1] + d[:, 2] * d[:, 2]))
    return out


def sphere_reference(mesh, sources):
    v = mesh._v
    p = v / np.linalg.norm(v, axis=1)[:, None]
    out = np.full(len(v), np.inf)
    for s in np.asarray(sources).reshape(-1):
        c = np.clip(p @ p[s], -1.0, 1.0)
        out = np.minimum(out, np.arccos(c))
    return out
