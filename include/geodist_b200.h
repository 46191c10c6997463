/*
 * geodist_b200.h -- C ABI of the B200-native PTP geodesic solver.
 *
 * Drop-in boundary for the reference's hot path (/root/reference/proj).  Each
 * entry point replaces one reference interface; the C++ drop-in
 * (integration/cpp/geodist_b200_dropin.cpp, compiled against the reference's own
 * headers) and the Python package (paper_1810_08218_b200) sit on top of these calls:
 *
 *   geodist_mesh_create    TriangleMesh + build_connectivity, once per mesh
 *                          (include/geodist/mesh.hpp:12-23, connectivity.hpp:69,
 *                          python/bindings.cpp:26-31 MeshHandle) -> device replica
 *   geodist_toplesets      compute_toplesets (include/geodist/toplesets.hpp:32)
 *   geodist_reorder_for_bands  reorder_for_bands (toplesets.hpp:45-46) from a source set
 *   geodist_reorder_ordered    reorder_for_bands (toplesets.hpp:45-46) from a caller's
 *                          ToplesetOrdering (the drop-in's entry point)
 *   geodist_ptp            compute_toplesets + ptp_run (ptp.hpp:70-72) as called by
 *                          python geodesics(method="ptp") (bindings.cpp:134-151)
 *   geodist_ptp_ordered    ptp_run with a caller-supplied ToplesetOrdering (ptp.hpp:70-72)
 *   geodist_voronoi        voronoi (sampling.hpp:40-41)
 *   geodist_fps            fps (sampling.hpp:36-37)
 *   geodist_batch          (no reference symbol) independent queries
 *   geodist_planar_update  planar_update<T> (update_kernel.hpp:34-79), test hook
 *
 * Conventions: plain pointers and sizes, caller-allocated outputs, int32
 * vertex ids (index_t, vec3.hpp:8), -1 = invalid_index.  Every call returns a
 * geodist_status; on failure geodist_last_error() holds a thread-local message
 * worded like the reference's exception text.  GEODIST_EINVAL maps to
 * std::invalid_argument (python ValueError), GEODIST_EMESH to
 * std::runtime_error (python RuntimeError).  Calls are synchronous unless
 * named *_async; host buffers may be pageable or pinned.
 */
#ifndef GEODIST_B200_H
#define GEODIST_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    GEODIST_OK = 0,
    GEODIST_EINVAL = 1, /* invalid argument (std::invalid_argument)            */
    GEODIST_EMESH = 2,  /* invalid / non-manifold mesh (std::runtime_error)     */
    GEODIST_ECUDA = 3,  /* CUDA runtime failure or no sm_100 device             */
    GEODIST_ENOMEM = 4  /* device or host allocation failure                    */
} geodist_status;

typedef enum { GEODIST_SINGLE = 0, GEODIST_DOUBLE = 1 } geodist_precision; /* Precision, distance_map.hpp:12 */

/* PtpConfig (include/geodist/ptp.hpp:15-21). */
typedef struct {
    double epsilon;       /* relative-change threshold retiring the front topleset (> 0) */
    int32_t precision;    /* geodist_precision */
    int32_t workers;      /* accepted and echoed (the GPU ignores it) */
    int32_t with_labels;  /* fill nearest-source labels */
    int32_t record_trace; /* fill the band trace and last_change */
} geodist_ptp_config;

/* PtpStats + BandTrace.iterations + ToplesetOrdering counts (ptp.hpp:43-49). */
typedef struct {
    int64_t relax_calls;      /* planar_update invocations (C)            */
    int64_t degenerate_calls; /* fallback-only triangles                  */
    int64_t vertex_updates;   /* sum of band sizes (U)                     */
    int32_t iterations;       /* K                                         */
    int32_t rho;              /* number of toplesets                       */
    int32_t unreached;        /* vertices the sources cannot reach         */
    int32_t workers;          /* echo of the config (>= 1)                 */
    double wall_seconds;      /* device time of the solve loop (CUDA events) */
    double total_seconds;     /* device time incl. BFS, init, copy-out       */
} geodist_ptp_stats;

/* BandRow (ptp.hpp:27-34). */
typedef struct {
    int32_t k;
    int32_t i;
    int32_t j;
    int32_t front_converged;
    int64_t updated;
    double max_rel_change;
} geodist_band_row;

/* FpsIterationStat (sampling.hpp:17-23). */
typedef struct {
    int32_t sources;
    int32_t rho;
    int64_t relax_calls;
    double radius;
    int32_t picked; /* -1 on the final labelling run */
    int32_t iterations;
} geodist_fps_row;

typedef struct geodist_mesh_s* geodist_mesh_t;

/* IterationObserver (ptp.hpp:64): called after every iteration with the full
 * snapshot in original vertex order (double precision runs only). */
typedef void (*geodist_observer_fn)(void* user, int32_t k, const double* distances, int32_t n);

const char* geodist_last_error(void);
int32_t geodist_version(void);

/* Device queries. */
int geodist_device_count(int32_t* count);

/* ---- meshes ---------------------------------------------------------- */
/* Validates (validate_mesh, mesh.cpp:11-34), builds the rotational fans
 * (build_connectivity, connectivity.cpp:19-81) and keeps the fan-CSR on
 * `device`.  The build runs on the device from the uploaded faces
 * (GEODIST_HOST_BUILD=1 selects the host build); a rejected mesh reports the
 * reference's error text.  xyz: n*3 doubles, faces: nf*3 int32.  xyz may be NULL for a
 * topology-only mesh (toplesets / reorder only; compute_toplesets receives a
 * Connectivity without positions). */
int geodist_mesh_create(const double* xyz, int32_t n, const int32_t* faces, int32_t nf,
                        int32_t device, geodist_mesh_t* out);
int geodist_mesh_destroy(geodist_mesh_t mesh);
int geodist_mesh_sizes(geodist_mesh_t mesh, int32_t* n, int32_t* nf, int64_t* corners);
/* degree (Connectivity::degree, connectivity.cpp:98-109) of every vertex. */
int geodist_mesh_degrees(geodist_mesh_t mesh, int32_t* degree);
/* Rotational fan of v (for_each_incident_triangle order): v1[c], v2[c];
 * returns the corner count in *count (needs cap >= count). */
int geodist_mesh_fan(geodist_mesh_t mesh, int32_t v, int32_t* v1, int32_t* v2, int32_t cap,
                     int32_t* count);
/* The whole fan-CSR of a mesh (the layout of geodist_build_fans): cptr n+1,
 * ring 3*nf + n, degree n; any pointer may be NULL. */
int geodist_mesh_fans(geodist_mesh_t mesh, int32_t* cptr, int32_t* ring, int32_t* degree);

/* Host-only fan build (no device): validation + rotational fans exactly as
 * geodist_mesh_create computes them.  cptr: n+1; ring: 3*nf + n entries
 * (vertex v's ring r_0..r_d at cptr[v]+v); degree: n (or NULL). */
int geodist_build_fans(const double* xyz, int32_t n, const int32_t* faces, int32_t nf,
                       int32_t* cptr, int32_t* ring, int32_t* degree);

/* Mesh files (load_mesh / write_mesh, mesh_io.cpp:119-156): ASCII OFF or OBJ chosen
 * by the extension, triangles only, validated; errors are GEODIST_EMESH with the
 * reference's message ("<path>: ...").  load parses the whole file into a handle
 * (n vertices, nf faces), copy fills caller arrays (xyz 3n doubles, faces 3nf), free
 * releases it.  write uses "%.17g" coordinates (reading back is bit-exact). */
typedef struct geodist_meshfile_s* geodist_meshfile_t;
#define GEODIST_FORMAT_OFF 0
#define GEODIST_FORMAT_OBJ 1
int geodist_meshfile_load(const char* path, geodist_meshfile_t* out, int32_t* n, int32_t* nf);
int geodist_meshfile_copy(geodist_meshfile_t file, double* xyz, int32_t* faces);
int geodist_meshfile_free(geodist_meshfile_t file);
int geodist_write_mesh(const char* path, const double* xyz, int32_t n, const int32_t* faces,
                       int32_t nf, int32_t format);

/* validate_mesh (mesh.cpp:11-34): GEODIST_EMESH with the reference's message. */
int geodist_validate_mesh(const double* xyz, int32_t n, const int32_t* faces, int32_t nf);

/* Host-only half-edge tables of build_connectivity (connectivity.cpp:19-81):
 * twin[3*nf] (-1 on the boundary) and the fan-start half-edge per vertex
 * (vertex_halfedge[n], -1 for isolated vertices); half-edge 3f+c runs from
 * corner c to corner (c+1)%3 of face f.  xyz may be NULL (topology checks only). */
int geodist_build_halfedges(const double* xyz, int32_t n, const int32_t* faces, int32_t nf,
                            int32_t* twin, int32_t* vertex_halfedge);

/* Host-side mesh generators (fixtures; bit-identical to mesh.cpp:36-105 for
 * grid and icosphere).  Sizes first, then fill caller arrays. */
int geodist_grid_sizes(int32_t nx, int32_t ny, int32_t* n, int32_t* nf);
int geodist_generate_grid(int32_t nx, int32_t ny, double shear, double* xyz, int32_t* faces);
int geodist_icosphere_sizes(int32_t subdiv, int32_t* n, int32_t* nf);
int geodist_generate_icosphere(int32_t subdiv, double* xyz, int32_t* faces);
/* Radial noise p *= 1 + sigma * N(0,1), std::mt19937(seed) +
 * std::normal_distribution<double> in vertex order. */
int geodist_perturb_radial(double* xyz, int32_t n, double sigma, uint32_t seed);
/* Torus nu x nv, radii R, r; quads split (a,b,c),(a,c,d). */
int geodist_torus_sizes(int32_t nu, int32_t nv, int32_t* n, int32_t* nf);
int geodist_generate_torus(int32_t nu, int32_t nv, double R, double r, double* xyz,
                           int32_t* faces);
/* z = amp * sin(x / wx) * cos(y / wy) over generate_grid(nx, ny) (config 3). */
int geodist_heightfield(double* xyz, int32_t n, double amp, double wx, double wy);

/* ---- toplesets (compute_toplesets, toplesets.cpp:16-58) --------------- */
/* sorted: n entries (first reachable used), limits: n+1, position: n. */
int geodist_toplesets(geodist_mesh_t mesh, const int32_t* sources, int32_t m, int32_t* sorted,
                      int32_t* limits, int32_t* position, int32_t* rho, int32_t* unreached);

/* reorder_for_bands (toplesets.cpp:60-89): permutation and permuted faces.
 * old_of_new, new_of_old: n; faces_out: nf*3. */
int geodist_reorder_for_bands(geodist_mesh_t mesh, const int32_t* sources, int32_t m,
                              int32_t* old_of_new, int32_t* new_of_old, int32_t* faces_out);

/* reorder_for_bands (toplesets.cpp:60-89) for a caller-supplied ordering: sorted
 * (reachable ids in topleset order) and position (n, -1 = unreachable), as
 * ToplesetOrdering holds them (toplesets.hpp:16-28).  Outputs as above plus
 * xyz_out (n*3 doubles, the permuted positions; NULL to skip; needs a mesh with
 * positions).  A position array inconsistent with sorted is rejected. */
int geodist_reorder_ordered(geodist_mesh_t mesh, const int32_t* sorted, int32_t reachable,
                            const int32_t* position, int32_t* old_of_new, int32_t* new_of_old,
                            int32_t* faces_out, double* xyz_out);

/* ---- distance fields -------------------------------------------------- */
/* compute_toplesets + ptp_run fused on the device.  distances: n doubles
 * (+inf for unreached); labels: n int32 or NULL (requires with_labels);
 * trace: trace_cap rows or NULL; last_change: n or NULL. */
int geodist_ptp(geodist_mesh_t mesh, const int32_t* sources, int32_t m,
                const geodist_ptp_config* config, double* distances, int32_t* labels,
                geodist_ptp_stats* stats, geodist_band_row* trace, int32_t trace_cap,
                int32_t* last_change, geodist_observer_fn observer, void* observer_user);

/* ptp_run with the caller's ordering (sorted: reachable entries, limits:
 * rho+1, position: n) -- validated like ptp.cpp:155-167. */
int geodist_ptp_ordered(geodist_mesh_t mesh, const int32_t* sources, int32_t m,
                        const int32_t* sorted, int32_t reachable, const int32_t* limits,
                        int32_t rho, const int32_t* position, const geodist_ptp_config* config,
                        double* distances, int32_t* labels, geodist_ptp_stats* stats,
                        geodist_band_row* trace, int32_t trace_cap, int32_t* last_change,
                        geodist_observer_fn observer, void* observer_user);

/* voronoi (sampling.cpp:51-58): labels of one multi-source run. */
int geodist_voronoi(geodist_mesh_t mesh, const int32_t* samples, int32_t m,
                    const geodist_ptp_config* config, int32_t* labels);

/* fps (sampling.cpp:11-49): samples (count), labels (n), radius, history
 * (count rows).  The whole sampling loop runs on the device. */
int geodist_fps(geodist_mesh_t mesh, int32_t count, int32_t seed, const geodist_ptp_config* config,
                int32_t* samples, int32_t* labels, double* radius, geodist_fps_row* history);

/* Independent queries: query q uses sources[offsets[q] .. offsets[q+1]).
 * Results land in DEVICE memory of the mesh's device: out_dist (nq*n values
 * of the run precision: float for SINGLE, double for DOUBLE), out_labels
 * (nq*n int32, or NULL), out_stats (nq rows, host).  `groups` queries run
 * concurrently inside one persistent launch; 0 = auto: query 0 runs on the whole
 * GPU and its mean band per CTA picks 1..8 groups for the rest (narrow,
 * latency-bound fields gain from concurrency, wide ones do not); wall_seconds
 * of every row is then the device time of both launches.  `stream` is a
 * cudaStream_t (NULL = the mesh's own stream); the call returns after the
 * launch completes. */
int geodist_batch_device(geodist_mesh_t mesh, const int32_t* sources, const int32_t* offsets,
                         int32_t nq, const geodist_ptp_config* config, void* out_dist,
                         int32_t* out_labels, geodist_ptp_stats* out_stats, int32_t groups,
                         void* stream);

/* Same with host output (nq*n doubles, labels nq*n or NULL). */
int geodist_batch(geodist_mesh_t mesh, const int32_t* sources, const int32_t* offsets,
                  int32_t nq, const geodist_ptp_config* config, double* distances,
                  int32_t* labels, geodist_ptp_stats* stats, int32_t groups);

/* One planar_update<T> on the device (test hook for the kernel arithmetic):
 * x1, x2: count*3 doubles, t1, t2: count doubles; value/side/degenerate out. */
int geodist_planar_update(const double* x1, const double* x2, const double* t1, const double* t2,
                          int32_t count, int32_t precision, double* value, int32_t* side,
                          int32_t* degenerate);

/* Self-test of the kernels' straight-line div/sqrt fast paths against the IEEE
 * intrinsics over n pseudo-random operand pairs: counts[0..7] = (accepted, differing)
 * for fp64 div, fp64 sqrt, fp32 div, fp32 sqrt.  "differing" must be 0. */
int geodist_selftest_arith(int64_t n, uint64_t seed, int64_t* counts);

/* Kernel launches issued by this library since load (evidence counter). */
int64_t geodist_kernel_launches(void);

/* Demote the L2 lines the solver's access-policy window marked persisting on the current
 * device (cudaCtxResetPersistingL2Cache), so that a cache flush evicts them too (benchmarks
 * that flush L2 between timed fields). */
int geodist_reset_persisting_l2(void);

#ifdef __cplusplus
}
#endif
#endif /* GEODIST_B200_H */
