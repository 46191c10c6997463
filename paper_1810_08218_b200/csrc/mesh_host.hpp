// Host-side mesh preprocessing (see mesh_host.cpp).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace gdb {

// Rotational fans in the reference's for_each_incident_triangle order.
struct Fans {
    int32_t n = 0;
    std::vector<int32_t> cptr;    // n+1 corner offsets
    std::vector<int32_t> ring;    // cptr[n] + n entries; vertex v at cptr[v] + v
    std::vector<int32_t> degree;  // graph degree (Connectivity::degree)
    std::vector<int32_t> twin;    // half-edge twins (3 nf), -1 on the boundary
    std::vector<int32_t> vstart;  // fan-start half-edge per vertex, -1 if isolated
    int32_t ring_offset(int32_t v) const { return cptr[v] + v; }
};

void validate(const double* xyz, int32_t n, const int32_t* faces, int32_t nf);

// Mesh files (mesh_io.cpp): ASCII OFF / OBJ by extension, validated.
struct MeshData {
    std::vector<double> xyz;      // 3 n
    std::vector<int32_t> faces;   // 3 nf
};
void load_mesh_file(const std::string& path, MeshData& m);
void write_mesh_file(const std::string& path, const double* xyz, int32_t n, const int32_t* faces,
                     int32_t nf, bool off);
Fans build_fans(const double* xyz, int32_t n, const int32_t* faces, int32_t nf);

void generate_grid(int32_t nx, int32_t ny, double shear, double* xyz, int32_t* faces);
void icosphere_sizes(int32_t subdiv, int32_t* n, int32_t* nf);
void generate_icosphere(int32_t subdiv, double* xyz, int32_t* faces);
void perturb_radial(double* xyz, int32_t n, double sigma, uint32_t seed);
void generate_torus(int32_t nu, int32_t nv, double R, double r, double* xyz, int32_t* faces);
void heightfield(double* xyz, int32_t n, double amp, double wx, double wy);

}  // namespace gdb
