// C++ drop-in for the reference library's hot path, backed by the B200 C ABI.
//
// Compiled against the reference's OWN public headers (proj/include/geodist/*.hpp),
// so every declaration, type layout and default argument is the reference's.  A
// maintainer replaces the reference's src/{mesh,connectivity,toplesets,ptp,sampling}.cpp
// with this file and links libgeodist_b200.so; the remaining reference sources
// (mesh_io, metrics, reference_solvers, reports, the CLI and the pybind module)
// compile and link unchanged (integration/Makefile).
//
//   validate_mesh / generate_grid / generate_icosphere   mesh.hpp:23-32
//   build_connectivity, neighbors, degree, vertex_star,
//   degree_histogram                                     connectivity.hpp:48-83
//   compute_toplesets (GPU), reorder_for_bands (GPU),
//   level_of, classify_sequences, topleset_histogram      toplesets.hpp:26-63
//   band_boundaries, ptp_run (GPU), iteration_bound_check ptp.hpp:60-76
//   fps (GPU), voronoi (GPU)                              sampling.hpp:36-41
//
// Device replicas: the reference API passes (mesh, conn) by reference on every
// call and has no handle.  Replicas are cached per mesh, keyed by the vectors'
// buffers and sizes plus a sampled content signature (GEODIST_B200_CACHE=0
// disables the cache; GEODIST_B200_DEVICE picks the GPU).
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <list>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "geodist/connectivity.hpp"
#include "geodist/mesh.hpp"
#include "geodist/ptp.hpp"
#include "geodist/sampling.hpp"
#include "geodist/toplesets.hpp"
#include "geodist_b200.h"

namespace geodist {
namespace {

void check(int rc) {
    if (rc == GEODIST_OK) return;
    const std::string msg = geodist_last_error();
    if (rc == GEODIST_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

int device_index() {
    const char* e = std::getenv("GEODIST_B200_DEVICE");
    return e ? std::atoi(e) : 0;
}

bool cache_enabled() {
    const char* e = std::getenv("GEODIST_B200_CACHE");
    return !(e && e[0] == '0');
}

// FNV-1a over the sizes and up to 4096 evenly strided 8-byte words.
uint64_t signature(const void* data, size_t bytes, uint64_t h) {
    const unsigned char* p = static_cast<const unsigned char*>(data);
    const size_t words = bytes / 8;
    const size_t step = words > 4096 ? words / 4096 : 1;
    auto mix = [&](uint64_t x) {
        for (int b = 0; b < 8; ++b) {
            h ^= (x >> (8 * b)) & 0xff;
            h *= 1099511628211ull;
        }
    };
    mix(bytes);
    for (size_t w = 0; w < words; w += step) {
        uint64_t x;
        std::memcpy(&x, p + 8 * w, 8);
        mix(x);
    }
    if (words) {
        uint64_t x;
        std::memcpy(&x, p + 8 * (words - 1), 8);
        mix(x);
    }
    return h;
}

// A replica stays alive while any call uses it: the cache and every in-flight call
// hold a reference, so an eviction (or the disabled-cache path) never destroys a
// handle another thread is solving on.
using ReplicaRef = std::shared_ptr<geodist_mesh_s>;

ReplicaRef adopt(geodist_mesh_t h) {
    return ReplicaRef(h, [](geodist_mesh_t p) { geodist_mesh_destroy(p); });
}

struct Replica {
    const void* vbuf;
    const void* fbuf;
    size_t nv, nf;
    uint64_t sig;
    bool geometry;
    ReplicaRef h;
};

struct Cache {
    std::mutex mu;
    std::list<Replica> items;  // most recent first
};
Cache& cache() {
    static Cache c;
    return c;
}

ReplicaRef create(bool geometry, const double* xyz, size_t nv, const int32_t* faces, size_t nf) {
    geodist_mesh_t h = nullptr;
    check(geodist_mesh_create(geometry ? xyz : nullptr, static_cast<int32_t>(nv), faces,
                              static_cast<int32_t>(nf), device_index(), &h));
    return adopt(h);
}

ReplicaRef lookup(const void* vbuf, const void* fbuf, size_t nv, size_t nf, uint64_t sig,
                  bool geometry, const double* xyz, const int32_t* faces) {
    if (!cache_enabled()) return create(geometry, xyz, nv, faces, nf);  // this call's own
    Cache& c = cache();
    {
        std::lock_guard<std::mutex> lock(c.mu);
        for (auto it = c.items.begin(); it != c.items.end(); ++it) {
            if (it->vbuf == vbuf && it->fbuf == fbuf && it->nv == nv && it->nf == nf &&
                it->sig == sig && (it->geometry || !geometry)) {
                c.items.splice(c.items.begin(), c.items, it);
                return it->h;
            }
        }
    }
    ReplicaRef h = create(geometry, xyz, nv, faces, nf);  // built outside the lock
    std::lock_guard<std::mutex> lock(c.mu);
    c.items.push_front({vbuf, fbuf, nv, nf, sig, geometry, h});
    while (c.items.size() > 8) c.items.pop_back();  // users keep their own reference
    return h;
}

// Replica with positions (distance fields).
ReplicaRef replica(const TriangleMesh& mesh) {
    const size_t nv = mesh.vertices.size(), nf = mesh.faces.size();
    static_assert(sizeof(Vec3) == 3 * sizeof(double), "Vec3 layout");
    static_assert(sizeof(std::array<index_t, 3>) == 3 * sizeof(int32_t), "face layout");
    uint64_t sig = signature(mesh.vertices.data(), nv * sizeof(Vec3), 1469598103934665603ull);
    sig = signature(mesh.faces.data(), nf * sizeof(std::array<index_t, 3>), sig);
    return lookup(mesh.vertices.data(), mesh.faces.data(), nv, nf, sig, true,
                  reinterpret_cast<const double*>(mesh.vertices.data()),
                  reinterpret_cast<const int32_t*>(mesh.faces.data()));
}

// Topology-only replica from a Connectivity (compute_toplesets has no mesh).
ReplicaRef replica(const Connectivity& conn) {
    const size_t nhe = static_cast<size_t>(conn.halfedge_count());
    std::vector<int32_t> faces(nhe);
    for (size_t h = 0; h < nhe; ++h) faces[h] = conn.origin(static_cast<index_t>(h));
    const uint64_t sig = signature(faces.data(), nhe * sizeof(int32_t), 7ull);
    return lookup(&conn, nullptr, static_cast<size_t>(conn.vertex_count()), nhe / 3, sig, false,
                  nullptr, faces.data());
}

geodist_ptp_config make_cfg(const PtpConfig& c) {
    geodist_ptp_config g;
    g.epsilon = c.epsilon;
    g.precision = c.precision == Precision::single_fp ? GEODIST_SINGLE : GEODIST_DOUBLE;
    g.workers = c.workers;
    g.with_labels = c.with_labels ? 1 : 0;
    g.record_trace = c.record_trace ? 1 : 0;
    return g;
}

void observer_tramp(void* user, int32_t k, const double* d, int32_t n) {
    const auto* obs = static_cast<const IterationObserver*>(user);
    (*obs)(k, std::span<const double>(d, static_cast<size_t>(n)));
}

}  // namespace

// ---------------------------------------------------------------------------
// mesh.hpp

void validate_mesh(const TriangleMesh& mesh) {
    check(geodist_validate_mesh(reinterpret_cast<const double*>(mesh.vertices.data()),
                                static_cast<int32_t>(mesh.vertices.size()),
                                reinterpret_cast<const int32_t*>(mesh.faces.data()),
                                static_cast<int32_t>(mesh.faces.size())));
}

TriangleMesh generate_grid(index_t nx, index_t ny, double shear) {
    int32_t n = 0, nf = 0;
    check(geodist_grid_sizes(nx, ny, &n, &nf));
    TriangleMesh m;
    m.vertices.resize(static_cast<size_t>(n));
    m.faces.resize(static_cast<size_t>(nf));
    check(geodist_generate_grid(nx, ny, shear, reinterpret_cast<double*>(m.vertices.data()),
                                reinterpret_cast<int32_t*>(m.faces.data())));
    return m;
}

TriangleMesh generate_icosphere(int subdiv) {
    int32_t n = 0, nf = 0;
    check(geodist_icosphere_sizes(subdiv, &n, &nf));
    TriangleMesh m;
    m.vertices.resize(static_cast<size_t>(n));
    m.faces.resize(static_cast<size_t>(nf));
    check(geodist_generate_icosphere(subdiv, reinterpret_cast<double*>(m.vertices.data()),
                                     reinterpret_cast<int32_t*>(m.faces.data())));
    return m;
}

// ---------------------------------------------------------------------------
// connectivity.hpp

Connectivity build_connectivity(const TriangleMesh& mesh) {
    const int32_t n = static_cast<int32_t>(mesh.vertices.size());
    const int32_t nf = static_cast<int32_t>(mesh.faces.size());
    Connectivity conn;
    conn.origin_.resize(3 * static_cast<size_t>(nf));
    std::memcpy(conn.origin_.data(), mesh.faces.data(), sizeof(int32_t) * 3 * nf);
    conn.twin_.assign(3 * static_cast<size_t>(nf), invalid_index);
    conn.vertex_halfedge_.assign(static_cast<size_t>(n), invalid_index);
    check(geodist_build_halfedges(reinterpret_cast<const double*>(mesh.vertices.data()), n,
                                  reinterpret_cast<const int32_t*>(mesh.faces.data()), nf,
                                  conn.twin_.data(), conn.vertex_halfedge_.data()));
    return conn;
}

std::vector<index_t> Connectivity::neighbors(index_t v) const {
    std::vector<index_t> ring;
    index_t last = invalid_index;
    bool open = false;
    const index_t start = vertex_halfedge_[v];
    if (start == invalid_index) return ring;
    index_t h = start;
    do {
        ring.push_back(target(h));
        last = h;
        h = twin(prev(h));
        open = h == invalid_index;
    } while (!open && h != start);
    if (open) ring.push_back(origin(prev(last)));
    return ring;
}

index_t Connectivity::degree(index_t v) const {
    return static_cast<index_t>(neighbors(v).size());
}

VertexStar vertex_star(const Connectivity& conn, index_t v) {
    if (v < 0 || v >= conn.vertex_count())
        throw std::invalid_argument("vertex_star: index out of range");
    VertexStar star;
    conn.for_each_incident_triangle(v, [&](index_t a, index_t, index_t f) {
        star.neighbors.push_back(a);
        star.faces.push_back(f);
    });
    const std::vector<index_t> ring = conn.neighbors(v);
    if (ring.size() > star.neighbors.size()) star.neighbors.push_back(ring.back());
    return star;
}

std::map<index_t, index_t> degree_histogram(const Connectivity& conn) {
    std::map<index_t, index_t> hist;
    for (index_t v = 0; v < conn.vertex_count(); ++v) ++hist[conn.degree(v)];
    return hist;
}

// ---------------------------------------------------------------------------
// toplesets.hpp

index_t ToplesetOrdering::level_of(index_t v) const {
    const index_t p = position[v];
    if (p == invalid_index) return invalid_index;
    return static_cast<index_t>(std::upper_bound(limits.begin(), limits.end(), p) -
                                limits.begin()) - 1;
}

ToplesetOrdering compute_toplesets(const Connectivity& conn, std::span<const index_t> sources) {
    const index_t n = conn.vertex_count();
    ToplesetOrdering out;
    out.sorted.resize(static_cast<size_t>(n));
    out.limits.resize(static_cast<size_t>(n) + 1);
    out.position.resize(static_cast<size_t>(n));
    int32_t rho = 0, unreached = 0;
    if (sources.empty()) throw std::invalid_argument("compute_toplesets: empty source set");
    ReplicaRef h = replica(conn);
    check(geodist_toplesets(h.get(), sources.data(), static_cast<int32_t>(sources.size()),
                            out.sorted.data(), out.limits.data(), out.position.data(), &rho,
                            &unreached));
    out.sorted.resize(static_cast<size_t>(n - unreached));
    out.limits.resize(static_cast<size_t>(rho) + 1);
    out.unreached = unreached;
    return out;
}

BandReordered reorder_for_bands(const TriangleMesh& mesh, const Connectivity& conn,
                                const ToplesetOrdering& ordering) {
    (void)conn;
    const index_t n = mesh.vertex_count();
    if (static_cast<index_t>(ordering.position.size()) != n)
        throw std::invalid_argument("reorder_for_bands: ordering built for a different mesh");
    BandReordered out;
    // GPU: old_of_new (the topleset order, then unreachable vertices in id order),
    // its inverse, the relabelled faces and the permuted positions (toplesets.cpp:60-89)
    out.old_of_new.resize(static_cast<size_t>(n));
    out.new_of_old.resize(static_cast<size_t>(n));
    out.mesh.vertices.resize(static_cast<size_t>(n));
    out.mesh.faces.resize(mesh.faces.size());
    ReplicaRef h = replica(mesh);
    check(geodist_reorder_ordered(h.get(), ordering.sorted.data(),
                                  static_cast<int32_t>(ordering.sorted.size()),
                                  ordering.position.data(), out.old_of_new.data(),
                                  out.new_of_old.data(),
                                  reinterpret_cast<int32_t*>(out.mesh.faces.data()),
                                  reinterpret_cast<double*>(out.mesh.vertices.data())));
    out.conn = build_connectivity(out.mesh);
    out.ordering.limits = ordering.limits;
    out.ordering.unreached = ordering.unreached;
    out.ordering.sorted.resize(ordering.sorted.size());
    for (size_t p = 0; p < ordering.sorted.size(); ++p) out.ordering.sorted[p] = static_cast<index_t>(p);
    out.ordering.position.assign(static_cast<size_t>(n), invalid_index);
    for (size_t p = 0; p < ordering.sorted.size(); ++p) out.ordering.position[p] = static_cast<index_t>(p);
    return out;
}

std::vector<SequenceSegment> classify_sequences(const ToplesetOrdering& ordering) {
    const index_t rho = ordering.rho();
    if (rho < 2) throw std::invalid_argument("classify_sequences: need at least two toplesets");
    auto cls = [&](index_t r) {
        const index_t d = ordering.level_size(r) - ordering.level_size(r - 1);
        return d > 0 ? SequenceClass::increasing
                     : (d < 0 ? SequenceClass::decreasing : SequenceClass::stationary);
    };
    std::vector<SequenceSegment> runs;
    SequenceSegment run{0, 1, cls(1)};
    for (index_t r = 2; r < rho; ++r) {
        if (cls(r) == run.cls) {
            run.end = r;
        } else {
            runs.push_back(run);
            run = {r, r, cls(r)};
        }
    }
    runs.push_back(run);
    return runs;
}

std::vector<index_t> topleset_histogram(const ToplesetOrdering& ordering) {
    std::vector<index_t> sizes(static_cast<size_t>(ordering.rho()));
    for (index_t r = 0; r < ordering.rho(); ++r) sizes[r] = ordering.level_size(r);
    return sizes;
}

const char* to_string(SequenceClass c) {
    return c == SequenceClass::increasing   ? "increasing"
           : c == SequenceClass::stationary ? "stationary"
           : c == SequenceClass::decreasing ? "decreasing"
                                            : "?";
}

// ---------------------------------------------------------------------------
// ptp.hpp

std::pair<index_t, index_t> band_boundaries(int k, index_t prev_i, index_t rho,
                                            bool converged_front) {
    return {converged_front ? prev_i + 1 : prev_i,
            k < rho ? static_cast<index_t>(k) : rho - 1};
}

PtpResult ptp_run(const TriangleMesh& mesh, const Connectivity& conn,
                  const ToplesetOrdering& ordering, std::span<const index_t> sources,
                  const PtpConfig& config, const IterationObserver& observer) {
    (void)conn;
    if (sources.empty()) throw std::invalid_argument("ptp_run: empty source set");
    if (!(config.epsilon > 0)) throw std::invalid_argument("ptp_run: epsilon must be positive");
    if (mesh.vertices.size() != ordering.position.size())
        throw std::invalid_argument("ptp_run: ordering built for a different mesh");
    const index_t n = mesh.vertex_count();
    ReplicaRef h = replica(mesh);
    const geodist_ptp_config cfg = make_cfg(config);
    PtpResult res;
    res.distances.values.resize(static_cast<size_t>(n));
    if (config.with_labels) res.distances.labels.resize(static_cast<size_t>(n));
    std::vector<geodist_band_row> rows;
    if (config.record_trace) {
        rows.resize(static_cast<size_t>(4) * static_cast<size_t>(n) + 64);
        res.trace.last_change.assign(static_cast<size_t>(n), 0);
    }
    geodist_ptp_stats st{};
    const int32_t rho = ordering.rho();
    check(geodist_ptp_ordered(
        h.get(), sources.data(), static_cast<int32_t>(sources.size()), ordering.sorted.data(),
        static_cast<int32_t>(ordering.sorted.size()), ordering.limits.data(), rho < 0 ? 0 : rho,
        ordering.position.data(), &cfg, res.distances.values.data(),
        config.with_labels ? res.distances.labels.data() : nullptr, &st,
        config.record_trace ? rows.data() : nullptr, static_cast<int32_t>(rows.size()),
        config.record_trace ? res.trace.last_change.data() : nullptr,
        observer ? &observer_tramp : nullptr,
        observer ? const_cast<IterationObserver*>(&observer) : nullptr));
    res.trace.iterations = st.iterations;
    if (config.record_trace) {
        const size_t cnt = std::min(rows.size(), static_cast<size_t>(st.iterations));
        res.trace.rows.reserve(cnt);
        for (size_t r = 0; r < cnt; ++r)
            res.trace.rows.push_back({rows[r].k, rows[r].i, rows[r].j, rows[r].updated,
                                      rows[r].max_rel_change, rows[r].front_converged != 0});
    }
    res.stats.relax_calls = st.relax_calls;
    res.stats.degenerate_calls = st.degenerate_calls;
    res.stats.wall_seconds = st.wall_seconds;
    res.stats.epsilon = config.epsilon;
    res.stats.workers = st.workers;
    res.distances.sources.assign(sources.begin(), sources.end());
    res.distances.precision = config.precision;
    res.distances.unreached = ordering.unreached;
    return res;
}

double iteration_bound_check(const BandTrace& trace, const ToplesetOrdering& ordering) {
    return static_cast<double>(trace.iterations) / static_cast<double>(ordering.rho());
}

// ---------------------------------------------------------------------------
// sampling.hpp

SamplingResult fps(const TriangleMesh& mesh, const Connectivity& conn, index_t m, index_t seed,
                   const PtpConfig& config) {
    (void)conn;
    const index_t n = mesh.vertex_count();
    if (m < 1 || m > n)
        throw std::invalid_argument("fps: sample count must be in [1, " + std::to_string(n) + "]");
    if (seed < 0 || seed >= n) throw std::invalid_argument("fps: seed vertex out of range");
    ReplicaRef h = replica(mesh);
    geodist_ptp_config cfg = make_cfg(config);
    cfg.with_labels = 1;
    SamplingResult out;
    out.samples.resize(static_cast<size_t>(m));
    out.labels.resize(static_cast<size_t>(n));
    std::vector<geodist_fps_row> hist(static_cast<size_t>(m));
    check(geodist_fps(h.get(), m, seed, &cfg, out.samples.data(), out.labels.data(), &out.radius,
                      hist.data()));
    for (const auto& r : hist)
        out.history.push_back({r.sources, r.rho, r.relax_calls, r.radius, r.picked});
    return out;
}

std::vector<index_t> voronoi(const TriangleMesh& mesh, const Connectivity& conn,
                             std::span<const index_t> samples, const PtpConfig& config) {
    (void)conn;
    if (samples.empty()) throw std::invalid_argument("voronoi: empty sample set");
    ReplicaRef h = replica(mesh);
    geodist_ptp_config cfg = make_cfg(config);
    cfg.with_labels = 1;
    std::vector<index_t> labels(static_cast<size_t>(mesh.vertex_count()));
    check(geodist_voronoi(h.get(), samples.data(), static_cast<int32_t>(samples.size()), &cfg,
                          labels.data()));
    return labels;
}

}  // namespace geodist
