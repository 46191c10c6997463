// TEST INFRASTRUCTURE ONLY -- never linked into the product.
//
// extern "C" shim over the UNMODIFIED reference library (compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/).  It exposes
// the reference's own hot-path entry points with plain pointers so the Python
// test-suite, the golden-vector generator and bench.py's `cpu_baseline` /
// `--impl reference` arm can drive them through ctypes:
//
//   ref_toplesets   -> geodist::compute_toplesets   (src/toplesets.cpp:16-58)
//   ref_reorder     -> geodist::reorder_for_bands   (src/toplesets.cpp:60-89)
//   ref_ptp         -> geodist::ptp_run             (src/ptp.cpp:152-172)
//   ref_fps         -> geodist::fps                 (src/sampling.cpp:11-49)
//   ref_voronoi     -> geodist::voronoi             (src/sampling.cpp:51-58)
//   ref_planar      -> geodist::planar_update<T>    (include/geodist/update_kernel.hpp:34-79)
//   ref_fan         -> Connectivity::for_each_incident_triangle (connectivity.hpp:35-44)
//   ref_load_mesh   -> geodist::load_mesh             (src/mesh_io.cpp:119-139)
//   ref_write_mesh  -> geodist::write_mesh            (src/mesh_io.cpp:141-156)
//
// Every function returns 0 on success, 1 for std::invalid_argument, 2 for
// std::runtime_error / anything else; the message is kept in ref_last_error().

#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

#include "geodist/connectivity.hpp"
#include "geodist/mesh.hpp"
#include "geodist/mesh_io.hpp"
#include "geodist/ptp.hpp"
#include "geodist/sampling.hpp"
#include "geodist/toplesets.hpp"
#include "geodist/update_kernel.hpp"

using namespace geodist;

namespace {

thread_local std::string g_err;

struct Handle {
    TriangleMesh mesh;
    Connectivity conn;
};

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_max_threads() {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

int ref_mesh_create(const double* xyz, int n, const int* faces, int nf, void** out,
                    double* build_seconds) {
    return guarded([&] {
        auto* h = new Handle;
        h->mesh.vertices.resize(n);
        for (int v = 0; v < n; ++v) h->mesh.vertices[v] = {xyz[3 * v], xyz[3 * v + 1], xyz[3 * v + 2]};
        h->mesh.faces.resize(nf);
        for (int f = 0; f < nf; ++f) h->mesh.faces[f] = {faces[3 * f], faces[3 * f + 1], faces[3 * f + 2]};
        const auto t0 = std::chrono::steady_clock::now();
        try {
            h->conn = build_connectivity(h->mesh);
        } catch (...) {
            delete h;
            throw;
        }
        if (build_seconds)
            *build_seconds =
                std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        *out = h;
    });
}

void ref_mesh_destroy(void* h) { delete static_cast<Handle*>(h); }

// load_mesh into a handle WITHOUT building connectivity (the file reader alone)
int ref_load_mesh(const char* path, void** out) {
    return guarded([&] {
        auto* h = new Handle;
        try {
            h->mesh = load_mesh(std::string(path));
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

int ref_write_mesh(void* hp, const char* path, int obj) {
    return guarded([&] {
        write_mesh(static_cast<Handle*>(hp)->mesh, std::string(path),
                   obj ? MeshFormat::obj : MeshFormat::off);
    });
}

static void* wrap(TriangleMesh m) {
    auto* h = new Handle;
    h->mesh = std::move(m);
    h->conn = build_connectivity(h->mesh);
    return h;
}

int ref_generate_grid(int nx, int ny, double shear, void** out) {
    return guarded([&] { *out = wrap(generate_grid(nx, ny, shear)); });
}

int ref_generate_icosphere(int subdiv, void** out) {
    return guarded([&] { *out = wrap(generate_icosphere(subdiv)); });
}

// SURVEY §8d synthetic inputs the reference does not ship a generator for (it has
// generate_grid / generate_icosphere only, mesh.cpp:36-105).  Written here on the
// reference's own types so the bench's reference arm never loads the product
// library; tests/test_capi_host.py checks they equal the product generators.
//   torus nu x nv, R, r: vertex (i, j) at ((R + r cos w) cos u, (R + r cos w) sin u, r sin w),
//   u = 2 pi i / nu, w = 2 pi j / nv; quad (a, b, c, d) split (a, b, c), (a, c, d).
int ref_generate_torus(int nu, int nv, double R, double r, void** out) {
    return guarded([&] {
        if (nu < 3 || nv < 3) throw std::invalid_argument("generate_torus: nu and nv must be >= 3");
        TriangleMesh m;
        const double two_pi = 2.0 * 3.14159265358979323846;
        m.vertices.reserve(static_cast<size_t>(nu) * nv);
        for (int j = 0; j < nv; ++j)
            for (int i = 0; i < nu; ++i) {
                const double u = two_pi * i / nu, w = two_pi * j / nv;
                m.vertices.push_back({(R + r * std::cos(w)) * std::cos(u),
                                      (R + r * std::cos(w)) * std::sin(u), r * std::sin(w)});
            }
        m.faces.reserve(2 * static_cast<size_t>(nu) * nv);
        for (int j = 0; j < nv; ++j)
            for (int i = 0; i < nu; ++i) {
                const int i1 = (i + 1) % nu, j1 = (j + 1) % nv;
                const int a = j * nu + i, b = j * nu + i1, c = j1 * nu + i1, d = j1 * nu + i;
                m.faces.push_back({a, b, c});
                m.faces.push_back({a, c, d});
            }
        *out = wrap(std::move(m));
    });
}

// p *= 1 + sigma * N(0, 1) per vertex in index order, std::mt19937(seed) (config 2)
void ref_perturb_radial(void* hp, double sigma, unsigned seed) {
    auto* h = static_cast<Handle*>(hp);
    std::mt19937 gen(seed);
    std::normal_distribution<double> normal(0.0, 1.0);
    for (auto& p : h->mesh.vertices) {
        const double f = 1.0 + sigma * normal(gen);
        p.x *= f;
        p.y *= f;
        p.z *= f;
    }
}

// z = amp * sin(x / wx) * cos(y / wy) (config 3, over generate_grid)
void ref_heightfield(void* hp, double amp, double wx, double wy) {
    auto* h = static_cast<Handle*>(hp);
    for (auto& p : h->mesh.vertices) p.z = amp * std::sin(p.x / wx) * std::cos(p.y / wy);
}

void ref_mesh_sizes(void* hp, int* n, int* nf) {
    auto* h = static_cast<Handle*>(hp);
    *n = h->mesh.vertex_count();
    *nf = h->mesh.face_count();
}

void ref_mesh_copy(void* hp, double* xyz, int* faces) {
    auto* h = static_cast<Handle*>(hp);
    for (index_t v = 0; v < h->mesh.vertex_count(); ++v) {
        xyz[3 * v] = h->mesh.vertices[v].x;
        xyz[3 * v + 1] = h->mesh.vertices[v].y;
        xyz[3 * v + 2] = h->mesh.vertices[v].z;
    }
    for (index_t f = 0; f < h->mesh.face_count(); ++f)
        for (int c = 0; c < 3; ++c) faces[3 * f + c] = h->mesh.faces[f][c];
}

// Fan of v in for_each_incident_triangle order; returns the corner count, or
// -1 if cap is too small.  ring_extra receives the closing neighbour of an
// open fan (Connectivity::neighbors' last entry) or -1 for closed fans.
int ref_fan(void* hp, int v, int* v1, int* v2, int cap, int* ring_extra) {
    auto* h = static_cast<Handle*>(hp);
    int count = 0;
    bool overflow = false;
    h->conn.for_each_incident_triangle(v, [&](index_t a, index_t b, index_t) {
        if (count < cap) {
            v1[count] = a;
            v2[count] = b;
        } else {
            overflow = true;
        }
        ++count;
    });
    const auto nb = h->conn.neighbors(v);
    *ring_extra = static_cast<int>(nb.size()) > count ? nb.back() : -1;
    return overflow ? -1 : count;
}

int ref_toplesets(void* hp, const int* src, int m, int* sorted, int* limits, int* position,
                  int* rho, int* unreached, int* reachable, double* seconds) {
    return guarded([&] {
        auto* h = static_cast<Handle*>(hp);
        const auto t0 = std::chrono::steady_clock::now();
        const ToplesetOrdering o =
            compute_toplesets(h->conn, std::span<const index_t>(src, static_cast<size_t>(m)));
        if (seconds)
            *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        std::memcpy(sorted, o.sorted.data(), o.sorted.size() * sizeof(int));
        std::memcpy(limits, o.limits.data(), o.limits.size() * sizeof(int));
        std::memcpy(position, o.position.data(), o.position.size() * sizeof(int));
        *rho = o.rho();
        *unreached = o.unreached;
        *reachable = o.reachable();
    });
}

// reorder_for_bands: old_of_new / new_of_old (n each) and the permuted faces.
int ref_reorder(void* hp, const int* src, int m, int* old_of_new, int* new_of_old, int* faces_out) {
    return guarded([&] {
        auto* h = static_cast<Handle*>(hp);
        const ToplesetOrdering o =
            compute_toplesets(h->conn, std::span<const index_t>(src, static_cast<size_t>(m)));
        const BandReordered re = reorder_for_bands(h->mesh, h->conn, o);
        std::memcpy(old_of_new, re.old_of_new.data(), re.old_of_new.size() * sizeof(int));
        std::memcpy(new_of_old, re.new_of_old.data(), re.new_of_old.size() * sizeof(int));
        for (size_t f = 0; f < re.mesh.faces.size(); ++f)
            for (int c = 0; c < 3; ++c) faces_out[3 * f + c] = re.mesh.faces[f][c];
    });
}

// stats: [0]=relax_calls [1]=degenerate_calls [2]=K [3]=workers [4]=rho [5]=unreached
// seconds: [0]=ptp_run wall_seconds (reference scope) [1]=compute_toplesets
// trace_i64 rows of (k, i, j, updated); trace_f64 max_rel; trace_conv front_converged
int ref_ptp(void* hp, const int* src, int m, double eps, int single, int with_labels,
            int record_trace, int workers, double* dist, int* labels, int64_t* stats,
            double* seconds, int64_t* trace_i64, double* trace_f64, int* trace_conv,
            int trace_cap, int* last_change) {
    return guarded([&] {
        auto* h = static_cast<Handle*>(hp);
        const std::span<const index_t> sources(src, static_cast<size_t>(m));
        const auto t0 = std::chrono::steady_clock::now();
        const ToplesetOrdering o = compute_toplesets(h->conn, sources);
        const double t_bfs =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        PtpConfig cfg;
        cfg.epsilon = eps;
        cfg.precision = single ? Precision::single_fp : Precision::double_fp;
        cfg.with_labels = with_labels != 0;
        cfg.record_trace = record_trace != 0;
        cfg.workers = workers;
        const PtpResult r = ptp_run(h->mesh, h->conn, o, sources, cfg);
        std::memcpy(dist, r.distances.values.data(), r.distances.values.size() * sizeof(double));
        if (with_labels && labels)
            std::memcpy(labels, r.distances.labels.data(), r.distances.labels.size() * sizeof(int));
        stats[0] = r.stats.relax_calls;
        stats[1] = r.stats.degenerate_calls;
        stats[2] = r.trace.iterations;
        stats[3] = r.stats.workers;
        stats[4] = o.rho();
        stats[5] = o.unreached;
        seconds[0] = r.stats.wall_seconds;
        seconds[1] = t_bfs;
        if (record_trace) {
            const int rows = static_cast<int>(r.trace.rows.size());
            for (int q = 0; q < rows && q < trace_cap; ++q) {
                const BandRow& b = r.trace.rows[q];
                trace_i64[4 * q] = b.k;
                trace_i64[4 * q + 1] = b.i;
                trace_i64[4 * q + 2] = b.j;
                trace_i64[4 * q + 3] = b.updated;
                trace_f64[q] = b.max_rel_change;
                trace_conv[q] = b.front_converged ? 1 : 0;
            }
            if (last_change)
                std::memcpy(last_change, r.trace.last_change.data(),
                            r.trace.last_change.size() * sizeof(int));
        }
    });
}

// ptp_run with a caller-supplied ordering (sorted / limits / position arrays).
int ref_ptp_ordered(void* hp, const int* src, int m, const int* sorted, int reachable,
                    const int* limits, int rho, const int* position, double eps, int single,
                    int with_labels, int workers, double* dist, int* labels, int64_t* stats) {
    return guarded([&] {
        auto* h = static_cast<Handle*>(hp);
        ToplesetOrdering o;
        o.sorted.assign(sorted, sorted + reachable);
        o.limits.assign(limits, limits + rho + 1);
        o.position.assign(position, position + h->mesh.vertex_count());
        o.unreached = h->mesh.vertex_count() - reachable;
        PtpConfig cfg;
        cfg.epsilon = eps;
        cfg.precision = single ? Precision::single_fp : Precision::double_fp;
        cfg.with_labels = with_labels != 0;
        cfg.workers = workers;
        const PtpResult r =
            ptp_run(h->mesh, h->conn, o, std::span<const index_t>(src, static_cast<size_t>(m)), cfg);
        std::memcpy(dist, r.distances.values.data(), r.distances.values.size() * sizeof(double));
        if (with_labels && labels)
            std::memcpy(labels, r.distances.labels.data(), r.distances.labels.size() * sizeof(int));
        stats[0] = r.stats.relax_calls;
        stats[1] = r.stats.degenerate_calls;
        stats[2] = r.trace.iterations;
        stats[3] = r.stats.workers;
    });
}

// history rows: (sources, rho, relax_calls, picked) as int64 + radius f64
int ref_fps(void* hp, int m, int seed, double eps, int single, int workers, int* samples,
            int* labels, double* radius, int64_t* hist_i64, double* hist_f64, double* seconds) {
    return guarded([&] {
        auto* h = static_cast<Handle*>(hp);
        PtpConfig cfg;
        cfg.epsilon = eps;
        cfg.precision = single ? Precision::single_fp : Precision::double_fp;
        cfg.workers = workers;
        const auto t0 = std::chrono::steady_clock::now();
        const SamplingResult r = fps(h->mesh, h->conn, m, seed, cfg);
        if (seconds)
            *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        std::memcpy(samples, r.samples.data(), r.samples.size() * sizeof(int));
        std::memcpy(labels, r.labels.data(), r.labels.size() * sizeof(int));
        *radius = r.radius;
        for (size_t q = 0; q < r.history.size(); ++q) {
            hist_i64[4 * q] = r.history[q].sources;
            hist_i64[4 * q + 1] = r.history[q].rho;
            hist_i64[4 * q + 2] = r.history[q].relax_calls;
            hist_i64[4 * q + 3] = r.history[q].picked;
            hist_f64[q] = r.history[q].radius;
        }
    });
}

int ref_voronoi(void* hp, const int* src, int m, double eps, int single, int workers,
                int* labels) {
    return guarded([&] {
        auto* h = static_cast<Handle*>(hp);
        PtpConfig cfg;
        cfg.epsilon = eps;
        cfg.precision = single ? Precision::single_fp : Precision::double_fp;
        cfg.workers = workers;
        const auto out =
            voronoi(h->mesh, h->conn, std::span<const index_t>(src, static_cast<size_t>(m)), cfg);
        std::memcpy(labels, out.data(), out.size() * sizeof(int));
    });
}

// planar_update<T> on one corner; T = float when single != 0 (inputs are
// cast exactly as run_impl casts positions and distances).
void ref_planar(const double* x1, const double* x2, double t1, double t2, int single,
                double* value, int* side, int* degenerate) {
    if (single) {
        const Vec3T<float> a{static_cast<float>(x1[0]), static_cast<float>(x1[1]),
                             static_cast<float>(x1[2])};
        const Vec3T<float> b{static_cast<float>(x2[0]), static_cast<float>(x2[1]),
                             static_cast<float>(x2[2])};
        const auto r = planar_update<float>(a, b, static_cast<float>(t1), static_cast<float>(t2));
        *value = r.value;
        *side = r.side;
        *degenerate = r.degenerate;
    } else {
        const auto r = planar_update<double>({x1[0], x1[1], x1[2]}, {x2[0], x2[1], x2[2]}, t1, t2);
        *value = r.value;
        *side = r.side;
        *degenerate = r.degenerate;
    }
}

}  // extern "C"
