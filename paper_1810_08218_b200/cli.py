"""Command-line front end on the B200 backend: the reference CLI's
`geodesic`, `fps` and `bench` subcommands (tools/geodist_main.cpp:190-367) with the same
input flags, output files (CSV / PLY / JSON stats formats of src/mesh_io.cpp and
src/reports.cpp) and exit codes (0 success, 2 input error, 3 solver or output error).

    python -m paper_1810_08218_b200 geodesic --sphere 5 --source 0 --out-csv d.csv
    python -m paper_1810_08218_b200 fps --grid 64,64 --count 16 --stats s.json
    python -m paper_1810_08218_b200 bench --mesh m.off --sources-range 1:8

Not on the GPU path (reported as input errors): `--method fm|dijkstra` (sequential
reference solvers) and the `diag` subcommand's bound suite; `bench` reports the PTP
columns (no FM relax counts).
"""
import argparse
import json
import math
import os
import sys
import time

import numpy as np

from . import (Mesh, farthest_point_sampling, geodesics, grid_arrays, grid_reference,
               icosphere_arrays, mape, read_mesh, sphere_reference, toplesets)

EXIT_OK, EXIT_INPUT, EXIT_SOLVER = 0, 2, 3


class InputError(Exception):
    pass


def format_distance(d):
    """format_distance (mesh_io.cpp): "inf", or %.17g with ".0" when it reads as an integer."""
    if math.isinf(d):
        return "inf" if d > 0 else "-inf"
    s = "%.17g" % d
    if not any(c in s for c in ".en"):
        s += ".0"
    return s


def distance_color(d, d_max):
    u = 1.0
    if math.isfinite(d):
        u = d / d_max if d_max > 0.0 else 0.0
        u = min(max(u, 0.0), 1.0)
    ch = lambda x: int(math.floor(255.0 * x + 0.5))  # std::round on non-negative values
    return ch(u), ch(1.0 - abs(2.0 * u - 1.0)), ch(1.0 - u)


def label_color(label):
    if label < 0:
        return 128, 128, 128
    h = label & 0xFFFFFFFF
    h = (h ^ 61) ^ (h >> 16)
    h = (h * 9) & 0xFFFFFFFF
    h ^= h >> 4
    h = (h * 0x27D4EB2D) & 0xFFFFFFFF
    h ^= h >> 15
    return h & 0xFF, (h >> 8) & 0xFF, (h >> 16) & 0xFF


def _open(path):
    try:
        return open(path, "w", newline="\n")
    except OSError:
        raise RuntimeError(f"{path}: cannot open file for writing")


def write_distance_csv(values, labels, path):
    with _open(path) as out:
        out.write("index,distance,label\n")
        lab = labels if labels is not None else None
        out.write("".join(f"{v},{format_distance(float(d))},{int(lab[v]) if lab is not None else -1}\n"
                          for v, d in enumerate(values)))


def write_ply(vertices, faces, colors, path):
    with _open(path) as out:
        out.write("ply\nformat ascii 1.0\n")
        out.write(f"element vertex {len(vertices)}\n")
        out.write("property float x\nproperty float y\nproperty float z\n")
        out.write("property uchar red\nproperty uchar green\nproperty uchar blue\n")
        out.write(f"element face {len(faces)}\n")
        out.write("property list uchar int vertex_indices\nend_header\n")
        f32 = np.asarray(vertices, np.float64).astype(np.float32)
        for v in range(len(f32)):
            r, g_, b = colors(v)
            out.write(f"{_fmt_float(f32[v, 0])} {_fmt_float(f32[v, 1])} {_fmt_float(f32[v, 2])} "
                      f"{r} {g_} {b}\n")
        out.write("".join(f"3 {t[0]} {t[1]} {t[2]}\n" for t in np.asarray(faces)))


def _fmt_float(x):
    """operator<<(float) with the default stream precision (6 significant digits, %g)."""
    return "%g" % float(x)


def write_json(obj, path):
    with _open(path) as out:
        out.write(json.dumps(obj, indent=2, sort_keys=True) + "\n")


def _integer(text, what):
    t = text.strip()
    if not t or not (t.lstrip("-").isdigit()) or t != text:
        raise InputError(f"invalid {what}: '{text}'")
    return int(t)


def resolve_mesh(args):
    """resolve_mesh (geodist_main.cpp:99-136): --mesh / --grid / --sphere."""
    given = [x for x in (args.mesh, args.grid, args.sphere) if x is not None]
    if not given:
        raise InputError("one of --mesh, --grid, --sphere is required")
    kind = None
    if args.mesh is not None:
        try:
            v, f = read_mesh(args.mesh)
        except RuntimeError as e:
            raise InputError(str(e))
    elif args.grid is not None:
        parts = args.grid.split(",")
        if len(parts) not in (2, 3):
            raise InputError("--grid expects NX,NY or NX,NY,SHEAR")
        nx, ny = _integer(parts[0], "grid size"), _integer(parts[1], "grid size")
        shear = 0.0
        if len(parts) == 3:
            try:
                shear = float(parts[2])
            except ValueError:
                raise InputError(f"invalid grid shear: '{parts[2]}'")
        if nx < 2 or ny < 2:
            raise InputError("--grid sizes must be >= 2")
        v, f = grid_arrays(nx, ny, shear)
        kind = "grid" if shear == 0.0 else None
    else:
        sub = _integer(args.sphere, "sphere subdivision")
        if sub < 0 or sub > 9:
            raise InputError("--sphere subdivision must be in [0, 9]")
        v, f = icosphere_arrays(sub)
        kind = "sphere"
    try:
        mesh = Mesh(v, f)
    except RuntimeError as e:
        if str(e).startswith("CUDA"):
            raise
        raise InputError(str(e))  # non-manifold input
    return mesh, kind


def make_config(args):
    if not (args.epsilon > 0):
        raise InputError("--epsilon must be positive")
    if args.precision not in ("single", "double"):
        raise InputError("--precision must be 'single' or 'double'")
    workers = args.workers
    if workers == "auto":
        workers = os.environ.get("GEODIST_WORKERS", "auto")
    w = 0
    if workers != "auto":
        w = _integer(workers, "worker count")
        if w < 1:
            raise InputError("--workers must be >= 1 or 'auto'")
    return w


def manifest(args, command):
    j = {"command": command, "epsilon": args.epsilon, "precision": args.precision,
         "workers": args.workers}
    for k in ("mesh", "grid", "sphere"):
        if getattr(args, k) is not None:
            j[k] = getattr(args, k)
    if getattr(args, "sources", None):
        j["sources"] = args.sources
    if command == "geodesic":
        j["method"] = args.method
    if command == "fps":
        j["count"] = args.count
        j["seed"] = args.seed
    if command == "bench":
        j["sources_range"] = args.sources_range
    return j


def parse_sources(text, n):
    if text is None:
        raise InputError("--source is required")
    src = [_integer(t, "source index") for t in text.split(",")]
    for s in src:
        if s < 0 or s >= n:
            raise InputError(f"source index {s} out of range (mesh has {n} vertices)")
    return src


def cmd_geodesic(args):
    mesh, kind = resolve_mesh(args)
    args.sources = parse_sources(args.source, mesh.n_vertices)
    workers = make_config(args)
    if args.method != "ptp":
        if args.method in ("fm", "dijkstra"):
            raise InputError(f"--method {args.method} is not available on the GPU backend")
        raise InputError("--method must be ptp, fm or dijkstra")
    r = geodesics(mesh, args.sources, epsilon=args.epsilon, precision=args.precision,
                  workers=workers, trace=bool(args.trace))
    d = np.asarray(r["distances"])
    stats = {"manifest": manifest(args, "geodesic"), "n": int(len(d)), "rho": int(r["rho"]),
             "iterations": int(r["iterations"]), "unreached": int(r["unreached"]),
             "precision": args.precision, "epsilon": args.epsilon, "workers": int(r["workers"]),
             "relax_calls": int(r["relax_calls"]), "degenerate_calls": int(r["degenerate_calls"]),
             "wall_seconds": float(r["device_seconds"])}
    if args.trace:
        with _open(args.trace) as out:
            out.write("k,i,j,updated,max_rel_change\n")
            for t in r["trace"]:
                out.write(f"{t['k']},{t['i']},{t['j']},{t['updated']},"
                          f"{format_distance(float(t['max_rel_change']))}\n")
    if kind is not None:
        ref = grid_reference(mesh, args.sources) if kind == "grid" else sphere_reference(mesh, args.sources)
        rep = mape(d, ref, args.sources)
        stats.update({"mape_percent": rep["mape"], "max_rel_error_percent": rep["max_rel_error"],
                      "compared": rep["compared"]})
    if args.out_csv:
        write_distance_csv(d, None, args.out_csv)
    if args.out_ply:
        finite = d[np.isfinite(d)]
        d_max = float(finite.max()) if len(finite) else 0.0
        write_ply(mesh.vertices(), mesh.faces(), lambda v: distance_color(float(d[v]), d_max),
                  args.out_ply)
    if args.stats:
        write_json(stats, args.stats)
    print(f"geodesic: n={len(d)} method={args.method} unreached={int(r['unreached'])}")
    return EXIT_OK


def cmd_fps(args):
    mesh, _ = resolve_mesh(args)
    workers = make_config(args)
    n = mesh.n_vertices
    if args.count < 1:
        raise InputError("--count must be >= 1")
    if args.count > n:
        raise InputError("--count exceeds the vertex count")
    if args.seed < 0 or args.seed >= n:
        raise InputError("--seed vertex out of range")
    s = farthest_point_sampling(mesh, args.count, args.seed, epsilon=args.epsilon, workers=workers,
                                precision=args.precision)
    samples = [int(x) for x in s["samples"]]
    hist = s["history"]
    if args.out_csv:
        with _open(args.out_csv) as out:
            out.write("order,vertex,insertion_radius\n")
            for i, v in enumerate(samples):
                rad = math.inf if i == 0 else hist[i - 1]["radius"]
                out.write(f"{i},{v},{format_distance(rad)}\n")
    if args.out_ply:
        lab = s["labels"]
        write_ply(mesh.vertices(), mesh.faces(), lambda v: label_color(int(lab[v])), args.out_ply)
    if args.out_dist:
        r = geodesics(mesh, samples, epsilon=args.epsilon, precision=args.precision,
                      workers=workers, labels=True)
        write_distance_csv(np.asarray(r["distances"]), r["labels"], args.out_dist)
    if args.stats:
        its = [{"sources": h["sources"], "rho": h["rho"], "relax_calls": h["relax_calls"],
                "radius": h["radius"], "picked": h["picked"]} for h in hist]
        write_json({"manifest": manifest(args, "fps"), "samples": samples,
                    "covering_radius": s["radius"],
                    "total_relax_calls": int(sum(h["relax_calls"] for h in hist)),
                    "iterations": its}, args.stats)
    print(f"fps: samples={len(samples)} covering_radius={s['radius']:.6g}")
    return EXIT_OK


def cmd_bench(args):
    mesh, _ = resolve_mesh(args)
    workers = make_config(args)
    parts = args.sources_range.split(":")
    if len(parts) != 2:
        raise InputError("--sources-range expects A:B")
    lo, hi = _integer(parts[0], "range bound"), _integer(parts[1], "range bound")
    if lo < 1 or hi < lo:
        raise InputError("--sources-range needs 1 <= A <= B")
    if hi > mesh.n_vertices:
        raise InputError("--sources-range exceeds the vertex count")
    spread = farthest_point_sampling(mesh, hi, args.seed, epsilon=args.epsilon, workers=workers,
                                     precision=args.precision)
    samples = [int(x) for x in spread["samples"]]
    rows = []
    out = _open(args.out_csv) if args.out_csv else None
    if out:
        out.write("m,rho,iterations,ptp_relax_calls\n")
    for m in range(lo, hi + 1):
        src = samples[:m]
        rho = toplesets(mesh, src)["rho"]
        r = geodesics(mesh, src, epsilon=args.epsilon, precision=args.precision, workers=workers)
        rows.append({"m": m, "rho": int(rho), "iterations": int(r["iterations"]),
                     "ptp_relax_calls": int(r["relax_calls"]),
                     "device_seconds": float(r["device_seconds"])})
        if out:
            out.write(f"{m},{rho},{r['iterations']},{r['relax_calls']}\n")
    if out:
        out.close()
    if args.stats:
        write_json({"manifest": manifest(args, "bench"), "rows": rows}, args.stats)
    print(f"bench: m in [{lo}, {hi}] done")
    return EXIT_OK


def build_parser():
    p = argparse.ArgumentParser(prog="geodist", description="Geodesic distance fields on triangle "
                                "meshes (B200 backend)")
    sub = p.add_subparsers(dest="command", required=True)

    def inputs(c):
        src = c.add_mutually_exclusive_group()  # (CLI11 excludes)
        src.add_argument("--mesh", help="Mesh file (.off or .obj)")
        src.add_argument("--grid", help="Generate a grid: NX,NY[,SHEAR]")
        src.add_argument("--sphere", help="Generate an icosphere: SUBDIV")
        c.add_argument("--epsilon", type=float, default=1e-3, help="Relative-change threshold")
        c.add_argument("--precision", default="double", help="single|double")
        c.add_argument("--workers", default="auto", help="Worker count or 'auto' (echoed)")
        c.add_argument("--stats", help="Write run statistics JSON")

    g = sub.add_parser("geodesic", help="Compute a geodesic distance map")
    inputs(g)
    g.add_argument("--source", required=True, help="Source vertex indices I[,I...]")
    g.add_argument("--method", default="ptp", help="ptp (fm|dijkstra: reference CPU only)")
    g.add_argument("--out-csv", dest="out_csv", help="Write per-vertex distance CSV")
    g.add_argument("--out-ply", dest="out_ply", help="Write distance-colored PLY")
    g.add_argument("--trace", help="Write band trace CSV")

    f = sub.add_parser("fps", help="Farthest point sampling")
    inputs(f)
    f.add_argument("--count", type=int, required=True, help="Number of samples")
    f.add_argument("--seed", type=int, default=0, help="Seed vertex")
    f.add_argument("--out-csv", dest="out_csv", help="Write sample CSV")
    f.add_argument("--out-ply", dest="out_ply", help="Write label-colored PLY")
    f.add_argument("--out-dist", dest="out_dist", help="Write labeled distance CSV")

    b = sub.add_parser("bench", help="Relax-count sweep over source counts")
    inputs(b)
    b.add_argument("--sources-range", dest="sources_range", required=True, help="Source counts A:B")
    b.add_argument("--seed", type=int, default=0, help="Seed vertex for the source spread")
    b.add_argument("--out-csv", dest="out_csv", help="Write per-m CSV")
    return p


def main(argv=None):
    p = build_parser()
    try:
        args = p.parse_args(argv)
    except SystemExit as e:
        return EXIT_INPUT if e.code not in (0, None) else EXIT_OK
    try:
        return {"geodesic": cmd_geodesic, "fps": cmd_fps, "bench": cmd_bench}[args.command](args)
    except (InputError, ValueError) as e:  # ValueError: the library's invalid_argument
        print(f"error: {e}", file=sys.stderr)
        return EXIT_INPUT
    except (RuntimeError, OSError) as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_SOLVER


if __name__ == "__main__":
    sys.exit(main())
