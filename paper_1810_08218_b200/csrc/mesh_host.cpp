// Host-side mesh preprocessing for the B200 PTP solver.
//
//  * validate()      -- the checks of validate_mesh (reference src/mesh.cpp:11-34),
//                       same error wording.
//  * build_fans()    -- the rotational fan order of build_connectivity +
//                       for_each_incident_triangle (src/connectivity.cpp:19-81,
//                       include/geodist/connectivity.hpp:35-44), computed with
//                       origin buckets (counting sort) instead of a hash map.
//  * generators      -- grid / icosphere bit-identical to src/mesh.cpp:36-105,
//                       plus the SURVEY §8d synthetic inputs (radial noise,
//                       torus, height field).
//
// Output of build_fans is the "fan-CSR" the device packs: for vertex v the
// corners cptr[v]..cptr[v+1] and the ring of cptr[v]+v .. cptr[v+1]+v
// (d+1 entries: r_0..r_{d-1} and r_d = closing neighbour of an open fan, or
// r_0 again for a closed fan), so corner c of v is (ring[c], ring[c+1]).
#include "mesh_host.hpp"

#include <algorithm>
#include <cmath>
#include <map>
#include <random>
#include <stdexcept>
#include <string>
#include <utility>

namespace gdb {

void validate(const double* xyz, int32_t n, const int32_t* faces, int32_t nf) {
    for (int32_t v = 0; xyz != nullptr && v < n; ++v) {
        const double* p = xyz + 3 * static_cast<size_t>(v);
        if (!std::isfinite(p[0]) || !std::isfinite(p[1]) || !std::isfinite(p[2]))
            throw std::runtime_error("vertex " + std::to_string(v) + " has non-finite coordinates");
    }
    for (int32_t f = 0; f < nf; ++f) {
        const int32_t* t = faces + 3 * static_cast<size_t>(f);
        for (int c = 0; c < 3; ++c)
            if (t[c] < 0 || t[c] >= n)
                throw std::runtime_error("face " + std::to_string(f) + ": vertex index " +
                                         std::to_string(t[c]) + " out of range (mesh has " +
                                         std::to_string(n) + " vertices)");
        if (t[0] == t[1] || t[1] == t[2] || t[0] == t[2])
            throw std::runtime_error("face " + std::to_string(f) + " repeats a vertex index");
        for (int c = 0; xyz != nullptr && c < 3; ++c) {
            const int32_t a = t[c], b = t[(c + 1) % 3];
            const double* pa = xyz + 3 * static_cast<size_t>(a);
            const double* pb = xyz + 3 * static_cast<size_t>(b);
            if (pa[0] == pb[0] && pa[1] == pb[1] && pa[2] == pb[2])
                throw std::runtime_error("face " + std::to_string(f) + ": zero-length edge (" +
                                         std::to_string(a) + ", " + std::to_string(b) + ")");
        }
    }
}

namespace {
inline int32_t nxt(int32_t h) { return h - h % 3 + (h % 3 + 1) % 3; }
inline int32_t prv(int32_t h) { return h - h % 3 + (h % 3 + 2) % 3; }
}  // namespace

Fans build_fans(const double* xyz, int32_t n, const int32_t* faces, int32_t nf) {
    validate(xyz, n, faces, nf);
    const int64_t nhe = 3 * static_cast<int64_t>(nf);
    if (nhe > INT32_MAX) throw std::runtime_error("mesh too large for int32 half-edge ids");
    const int32_t* org = faces;  // origin(h) = faces[h]: half-edge h = 3f+c starts at corner c

    // Outgoing half-edges bucketed by origin, ascending half-edge id.
    std::vector<int32_t> bptr(static_cast<size_t>(n) + 1, 0);
    for (int64_t h = 0; h < nhe; ++h) ++bptr[org[h] + 1];
    for (int32_t v = 0; v < n; ++v) bptr[v + 1] += bptr[v];
    std::vector<int32_t> bucket(static_cast<size_t>(nhe));
    {
        std::vector<int32_t> fill(bptr.begin(), bptr.end() - 1);
        for (int64_t h = 0; h < nhe; ++h) bucket[fill[org[h]]++] = static_cast<int32_t>(h);
    }
    // Directed-edge uniqueness, reported at the first repeat in half-edge order
    // (the reference's emplace failure, connectivity.cpp:33-35).
    for (int64_t h = 0; h < nhe; ++h) {
        const int32_t o = org[h], t = org[nxt(static_cast<int32_t>(h))];
        for (int32_t q = bptr[o]; q < bptr[o + 1] && bucket[q] < h; ++q)
            if (org[nxt(bucket[q])] == t)
                throw std::runtime_error("non-manifold edge (" + std::to_string(o) + ", " +
                                         std::to_string(t) + "): same orientation appears twice");
    }
    // twin(h) = the half-edge target(h) -> origin(h), if any.
    std::vector<int32_t> twin(static_cast<size_t>(nhe), -1);
    for (int64_t h = 0; h < nhe; ++h) {
        const int32_t o = org[h], t = org[nxt(static_cast<int32_t>(h))];
        for (int32_t q = bptr[t]; q < bptr[t + 1]; ++q)
            if (org[nxt(bucket[q])] == o) {
                twin[h] = bucket[q];
                break;
            }
    }

    Fans F;
    F.n = n;
    F.cptr.assign(static_cast<size_t>(n) + 1, 0);
    F.ring.clear();
    F.ring.reserve(static_cast<size_t>(nhe) + n);
    F.degree.assign(static_cast<size_t>(n), 0);
    F.vstart.assign(static_cast<size_t>(n), -1);
    int32_t corners = 0;
    for (int32_t v = 0; v < n; ++v) {
        F.cptr[v] = corners;
        const int32_t incident = bptr[v + 1] - bptr[v];
        if (incident == 0) {
            F.ring.push_back(-1);  // isolated vertex: one unused ring slot
            continue;
        }
        // Fan start: the first outgoing half-edge, rotated to the open-fan
        // start (connectivity.cpp:47-60).
        const int32_t h0 = bucket[bptr[v]];
        int32_t h = h0;
        while (twin[h] != -1) {
            h = nxt(twin[h]);
            if (h == h0) break;
        }
        F.vstart[v] = h;
        // Walk h -> twin(prev(h)) (connectivity.hpp:35-44).
        int32_t w = h, last = h, count = 0;
        do {
            F.ring.push_back(org[nxt(w)]);  // v1 = target(w)
            ++count;
            last = w;
            w = twin[prv(w)];
        } while (w != -1 && w != h);
        const bool open = w == -1;
        if (count != incident)
            throw std::runtime_error("non-manifold vertex " + std::to_string(v) +
                                     ": star is not a single fan");
        // Closing ring entry: origin(prev(last)) for an open fan
        // (connectivity.cpp:95), r_0 again for a closed one.
        F.ring.push_back(open ? org[prv(last)] : F.ring[F.ring.size() - count]);
        F.degree[v] = open ? count + 1 : count;
        corners += count;
    }
    F.cptr[n] = corners;
    F.twin = std::move(twin);
    return F;
}

// ---------------------------------------------------------------------------
// generators

void generate_grid(int32_t nx, int32_t ny, double shear, double* xyz, int32_t* faces) {
    if (nx < 2 || ny < 2) throw std::invalid_argument("generate_grid: nx and ny must be >= 2");
    size_t q = 0;
    for (int32_t j = 0; j < ny; ++j)
        for (int32_t i = 0; i < nx; ++i) {
            xyz[q++] = i + shear * j;
            xyz[q++] = static_cast<double>(j);
            xyz[q++] = 0.0;
        }
    q = 0;
    for (int32_t j = 0; j + 1 < ny; ++j)
        for (int32_t i = 0; i + 1 < nx; ++i) {
            const int32_t a = j * nx + i, b = a + 1, c = a + nx + 1, d = a + nx;
            faces[q++] = a; faces[q++] = b; faces[q++] = c;
            faces[q++] = a; faces[q++] = c; faces[q++] = d;
        }
}

void icosphere_sizes(int32_t subdiv, int32_t* n, int32_t* nf) {
    if (subdiv < 0) throw std::invalid_argument("generate_icosphere: subdiv must be >= 0");
    if (subdiv > 12) throw std::invalid_argument("generate_icosphere: subdiv too large for int32");
    int64_t p = 1;
    for (int s = 0; s < subdiv; ++s) p *= 4;
    *n = static_cast<int32_t>(10 * p + 2);
    *nf = static_cast<int32_t>(20 * p);
}

void generate_icosphere(int32_t subdiv, double* xyz, int32_t* faces) {
    int32_t n_final, nf_final;
    icosphere_sizes(subdiv, &n_final, &nf_final);
    const double phi = (1.0 + std::sqrt(5.0)) / 2.0;
    const double s = 1.0 / std::sqrt(1.0 + phi * phi);
    const double a = s, b = phi * s;
    const double base[12][3] = {{-a, b, 0},  {a, b, 0},  {-a, -b, 0}, {a, -b, 0},
                                {0, -a, b},  {0, a, b},  {0, -a, -b}, {0, a, -b},
                                {b, 0, -a},  {b, 0, a},  {-b, 0, -a}, {-b, 0, a}};
    const int32_t tri[20][3] = {{0, 11, 5}, {0, 5, 1},  {0, 1, 7},   {0, 7, 10}, {0, 10, 11},
                                {1, 5, 9},  {5, 11, 4}, {11, 10, 2}, {10, 7, 6}, {7, 1, 8},
                                {3, 9, 4},  {3, 4, 2},  {3, 2, 6},   {3, 6, 8},  {3, 8, 9},
                                {4, 9, 5},  {2, 4, 11}, {6, 2, 10},  {8, 6, 7},  {9, 8, 1}};
    int32_t nv = 12;
    for (int v = 0; v < 12; ++v)
        for (int d = 0; d < 3; ++d) xyz[3 * v + d] = base[v][d];
    std::vector<int32_t> cur(60), nxtf;
    for (int f = 0; f < 20; ++f)
        for (int c = 0; c < 3; ++c) cur[3 * f + c] = tri[f][c];
    for (int32_t level = 0; level < subdiv; ++level) {
        // Midpoints cached per undirected edge; new vertices appended in the
        // order faces request them (ab, bc, ca).
        std::map<std::pair<int32_t, int32_t>, int32_t> mid;
        auto midpoint = [&](int32_t p, int32_t q) {
            const auto key = p < q ? std::make_pair(p, q) : std::make_pair(q, p);
            auto it = mid.find(key);
            if (it != mid.end()) return it->second;
            double m[3];
            for (int d = 0; d < 3; ++d) m[d] = xyz[3 * p + d] + xyz[3 * q + d];
            const double inv = 1.0 / std::sqrt(m[0] * m[0] + m[1] * m[1] + m[2] * m[2]);
            for (int d = 0; d < 3; ++d) xyz[3 * static_cast<size_t>(nv) + d] = inv * m[d];
            mid.emplace(key, nv);
            return nv++;
        };
        const size_t nfc = cur.size() / 3;
        nxtf.resize(cur.size() * 4);
        for (size_t f = 0; f < nfc; ++f) {
            const int32_t t0 = cur[3 * f], t1 = cur[3 * f + 1], t2 = cur[3 * f + 2];
            const int32_t ab = midpoint(t0, t1), bc = midpoint(t1, t2), ca = midpoint(t2, t0);
            const int32_t quad[12] = {t0, ab, ca, t1, bc, ab, t2, ca, bc, ab, bc, ca};
            std::copy(quad, quad + 12, nxtf.begin() + 12 * f);
        }
        cur.swap(nxtf);
    }
    std::copy(cur.begin(), cur.end(), faces);
}

void perturb_radial(double* xyz, int32_t n, double sigma, uint32_t seed) {
    std::mt19937 gen(seed);
    std::normal_distribution<double> normal(0.0, 1.0);
    for (int32_t v = 0; v < n; ++v) {
        const double f = 1.0 + sigma * normal(gen);
        for (int d = 0; d < 3; ++d) xyz[3 * static_cast<size_t>(v) + d] *= f;
    }
}

void generate_torus(int32_t nu, int32_t nv, double R, double r, double* xyz, int32_t* faces) {
    if (nu < 3 || nv < 3) throw std::invalid_argument("generate_torus: nu and nv must be >= 3");
    const double two_pi = 2.0 * 3.14159265358979323846;
    size_t q = 0;
    for (int32_t j = 0; j < nv; ++j)
        for (int32_t i = 0; i < nu; ++i) {
            const double u = two_pi * i / nu, w = two_pi * j / nv;
            xyz[q++] = (R + r * std::cos(w)) * std::cos(u);
            xyz[q++] = (R + r * std::cos(w)) * std::sin(u);
            xyz[q++] = r * std::sin(w);
        }
    q = 0;
    for (int32_t j = 0; j < nv; ++j)
        for (int32_t i = 0; i < nu; ++i) {
            const int32_t i1 = (i + 1) % nu, j1 = (j + 1) % nv;
            const int32_t a = j * nu + i, b = j * nu + i1, c = j1 * nu + i1, d = j1 * nu + i;
            faces[q++] = a; faces[q++] = b; faces[q++] = c;
            faces[q++] = a; faces[q++] = c; faces[q++] = d;
        }
}

void heightfield(double* xyz, int32_t n, double amp, double wx, double wy) {
    for (int32_t v = 0; v < n; ++v) {
        double* p = xyz + 3 * static_cast<size_t>(v);
        p[2] = amp * std::sin(p[0] / wx) * std::cos(p[1] / wy);
    }
}

}  // namespace gdb
