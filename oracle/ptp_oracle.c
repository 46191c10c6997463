/*
 * TEST INFRASTRUCTURE ONLY -- the CPU oracle.  Never linked into, loaded by or
 * called from the product path (paper_1810_08218_b200/).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may use it, and only
 * as the checker.
 *
 * A plain-C restatement of the reference's hot path (/root/reference/proj):
 *
 *   orc_build_fans   build_connectivity + for_each_incident_triangle order
 *                    (src/connectivity.cpp:19-81, include/geodist/connectivity.hpp:35-44,
 *                    src/connectivity.cpp:83-96 for the open-fan closing neighbour)
 *   orc_toplesets    compute_toplesets (src/toplesets.cpp:16-58)
 *   orc_planar_*     planar_update<T> (include/geodist/update_kernel.hpp:34-79)
 *   orc_ptp_*        run_impl<T> + ptp_run validation (src/ptp.cpp:37-43, 45-148, 152-172)
 *   orc_fps          fps (src/sampling.cpp:11-49)
 *
 * Parity of this restatement is pinned against the unmodified reference built
 * by oracle/Makefile into oracle/_ref/ (tests/test_oracle.py) and against the
 * committed golden vectors in tests/golden/ (generated from oracle/_ref by
 * oracle/gen_golden.py).  Compiled with -ffp-contract=off: no FMA, IEEE
 * division and sqrt, left-to-right association exactly as the C++ source.
 *
 * Return codes: 0 ok, 1 invalid argument, 2 invalid/non-manifold mesh.
 */
#include <float.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static char orc_err[256];
const char* orc_last_error(void) { return orc_err; }

#define FAIL(code, ...)                                            \
    do {                                                           \
        snprintf(orc_err, sizeof orc_err, __VA_ARGS__);            \
        return (code);                                             \
    } while (0)

/* ------------------------------------------------------------------------ */
/* Fans (connectivity.cpp:19-81)                                              */
/* ------------------------------------------------------------------------ */

static int he_next(int h) { return 3 * (h / 3) + (h % 3 + 1) % 3; }
static int he_prev(int h) { return 3 * (h / 3) + (h % 3 + 2) % 3; }

typedef struct {
    uint64_t key;
    int he;
} edge_rec;

static int cmp_edge(const void* a, const void* b) {
    const edge_rec* x = (const edge_rec*)a;
    const edge_rec* y = (const edge_rec*)b;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    return x->he - y->he;
}

static uint64_t ekey(int a, int b) { return ((uint64_t)(uint32_t)a << 32) | (uint32_t)b; }

static int find_edge(const edge_rec* e, int ne, uint64_t key) {
    int lo = 0, hi = ne - 1;
    while (lo <= hi) {
        const int mid = (lo + hi) / 2;
        if (e[mid].key == key) return e[mid].he;
        if (e[mid].key < key) lo = mid + 1; else hi = mid - 1;
    }
    return -1;
}

/* validate_mesh (mesh.cpp:11-34) */
static int validate(int n, const double* xyz, int nf, const int* faces) {
    for (int v = 0; v < n; ++v)
        if (!isfinite(xyz[3 * v]) || !isfinite(xyz[3 * v + 1]) || !isfinite(xyz[3 * v + 2]))
            FAIL(2, "vertex %d has non-finite coordinates", v);
    for (int f = 0; f < nf; ++f) {
        const int* t = faces + 3 * f;
        for (int c = 0; c < 3; ++c)
            if (t[c] < 0 || t[c] >= n)
                FAIL(2, "face %d: vertex index %d out of range (mesh has %d vertices)", f, t[c], n);
        if (t[0] == t[1] || t[1] == t[2] || t[0] == t[2]) FAIL(2, "face %d repeats a vertex index", f);
        for (int c = 0; c < 3; ++c) {
            const int a = t[c], b = t[(c + 1) % 3];
            if (xyz[3 * a] == xyz[3 * b] && xyz[3 * a + 1] == xyz[3 * b + 1] &&
                xyz[3 * a + 2] == xyz[3 * b + 2])
                FAIL(2, "face %d: zero-length edge (%d, %d)", f, a, b);
        }
    }
    return 0;
}

/*
 * Per vertex v: corner_ptr[v]..corner_ptr[v+1] lists the incident triangles in
 * for_each_incident_triangle order as (c_v1, c_v2); ring_extra[v] is the
 * closing neighbour of an open fan (-1 for closed fans and isolated vertices).
 * corner arrays must hold 3*nf entries.
 */
int orc_build_fans(int n, const double* xyz, int nf, const int* faces, int* corner_ptr,
                   int* c_v1, int* c_v2, int* ring_extra) {
    int rc = validate(n, xyz, nf, faces);
    if (rc) return rc;
    const int nhe = 3 * nf;
    int* origin = (int*)malloc(sizeof(int) * (size_t)(nhe + 1));
    int* twin = (int*)malloc(sizeof(int) * (size_t)(nhe + 1));
    int* vh = (int*)malloc(sizeof(int) * (size_t)(n + 1));
    int* incident = (int*)calloc((size_t)n + 1, sizeof(int));
    edge_rec* e = (edge_rec*)malloc(sizeof(edge_rec) * (size_t)(nhe + 1));
    for (int h = 0; h < nhe; ++h) origin[h] = faces[h];
    for (int v = 0; v < n; ++v) vh[v] = -1;
    for (int h = 0; h < nhe; ++h) {
        e[h].key = ekey(origin[h], origin[he_next(h)]);
        e[h].he = h;
        if (vh[origin[h]] == -1) vh[origin[h]] = h; /* first outgoing half-edge */
    }
    qsort(e, (size_t)nhe, sizeof(edge_rec), cmp_edge);
    for (int q = 1; q < nhe; ++q)
        if (e[q].key == e[q - 1].key) {
            /* the reference reports the first duplicate in half-edge order */
            int first_dup = nhe;
            for (int r = 1; r < nhe; ++r)
                if (e[r].key == e[r - 1].key && e[r].he < first_dup) first_dup = e[r].he;
            const int o = origin[first_dup], t = origin[he_next(first_dup)];
            free(origin); free(twin); free(vh); free(incident); free(e);
            FAIL(2, "non-manifold edge (%d, %d): same orientation appears twice", o, t);
        }
    for (int h = 0; h < nhe; ++h) twin[h] = find_edge(e, nhe, ekey(origin[he_next(h)], origin[h]));
    for (int f = 0; f < nf; ++f)
        for (int c = 0; c < 3; ++c) ++incident[faces[3 * f + c]];

    int nc = 0;
    rc = 0;
    for (int v = 0; v < n && !rc; ++v) {
        corner_ptr[v] = nc;
        ring_extra[v] = -1;
        int h = vh[v];
        if (h == -1) {
            if (incident[v] != 0) rc = 2;
            continue;
        }
        /* rotate to the open-fan start (connectivity.cpp:47-60) */
        const int h0 = h;
        int guard = 0;
        while (twin[h] != -1) {
            h = he_next(twin[h]);
            if (h == h0) break;
            if (++guard > nhe) { rc = 2; break; }
        }
        if (rc) { snprintf(orc_err, sizeof orc_err, "non-manifold vertex %d: star is not a single fan", v); break; }
        /* fan walk (connectivity.hpp:35-44) */
        int w = h, last = h, count = 0;
        do {
            c_v1[nc] = origin[he_next(w)];
            c_v2[nc] = origin[he_prev(w)];
            ++nc;
            ++count;
            last = w;
            w = twin[he_prev(w)];
        } while (w != -1 && w != h);
        if (w == -1) ring_extra[v] = origin[he_prev(last)]; /* connectivity.cpp:95 */
        if (count != incident[v]) {
            rc = 2;
            snprintf(orc_err, sizeof orc_err, "non-manifold vertex %d: star is not a single fan", v);
        }
    }
    corner_ptr[n] = nc;
    free(origin); free(twin); free(vh); free(incident); free(e);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* Toplesets (toplesets.cpp:16-58)                                            */
/* ------------------------------------------------------------------------ */

static int cmp_int(const void* a, const void* b) {
    const int x = *(const int*)a, y = *(const int*)b;
    return (x > y) - (x < y);
}

/* limits must hold n+1 entries; returns rho through *rho. */
int orc_toplesets(int n, const int* corner_ptr, const int* c_v1, const int* ring_extra,
                  const int* sources, int m, int* sorted, int* limits, int* position, int* rho,
                  int* unreached) {
    if (m <= 0) FAIL(1, "compute_toplesets: empty source set");
    int* level = (int*)malloc(sizeof(int) * (size_t)(n + 1));
    int* next = (int*)malloc(sizeof(int) * (size_t)(n + 1));
    memcpy(level, sources, sizeof(int) * (size_t)m);
    qsort(level, (size_t)m, sizeof(int), cmp_int);
    for (int i = 0; i < m; ++i) {
        if (level[i] < 0 || level[i] >= n) {
            const int s = level[i];
            free(level); free(next);
            FAIL(1, "compute_toplesets: source index %d out of range", s);
        }
        if (i > 0 && level[i] == level[i - 1]) {
            const int s = level[i];
            free(level); free(next);
            FAIL(1, "compute_toplesets: duplicate source index %d", s);
        }
    }
    for (int v = 0; v < n; ++v) position[v] = -1;
    int nl = m, ns = 0, r = 0;
    limits[0] = 0;
    while (nl > 0) {
        for (int q = 0; q < nl; ++q) {
            position[level[q]] = ns;
            sorted[ns++] = level[q];
        }
        limits[++r] = ns;
        int nn = 0;
        for (int q = 0; q < nl; ++q) {
            const int v = level[q];
            /* Connectivity::neighbors: fan v1's in order, then the closing one */
            for (int c = corner_ptr[v]; c <= corner_ptr[v + 1]; ++c) {
                const int u = c < corner_ptr[v + 1] ? c_v1[c] : ring_extra[v];
                if (u < 0) continue;
                if (position[u] == -1) {
                    position[u] = n;
                    next[nn++] = u;
                }
            }
        }
        qsort(next, (size_t)nn, sizeof(int), cmp_int);
        memcpy(level, next, sizeof(int) * (size_t)nn);
        nl = nn;
    }
    *rho = r;
    *unreached = n - ns;
    free(level);
    free(next);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* planar_update / relax_vertex / run_impl, instantiated for float and double */
/* ------------------------------------------------------------------------ */

#define DEFINE_PTP(T, SFX, TINF, TMIN, TSQRT, TABS)                                             \
    typedef struct { T value; int side; int degenerate; } cand_##SFX;                           \
                                                                                                \
    /* update_kernel.hpp:34-79 */                                                               \
    static cand_##SFX planar_##SFX(const T* x1, const T* x2, T t1, T t2) {                     \
        cand_##SFX out;                                                                         \
        const T f1 = t1 + TSQRT(x1[0] * x1[0] + x1[1] * x1[1] + x1[2] * x1[2]);                \
        const T f2 = t2 + TSQRT(x2[0] * x2[0] + x2[1] * x2[1] + x2[2] * x2[2]);                \
        out.degenerate = 0;                                                                     \
        if (f1 <= f2) { out.value = f1; out.side = 0; } else { out.value = f2; out.side = 1; } \
        if (t1 == TINF && t2 == TINF) { out.value = TINF; out.side = -1; return out; }          \
        if (t1 == TINF || t2 == TINF) return out;                                               \
        const T g11 = x1[0] * x1[0] + x1[1] * x1[1] + x1[2] * x1[2];                            \
        const T g22 = x2[0] * x2[0] + x2[1] * x2[1] + x2[2] * x2[2];                            \
        const T g12 = x1[0] * x2[0] + x1[1] * x2[1] + x1[2] * x2[2];                            \
        const T det = g11 * g22 - g12 * g12;                                                    \
        const T sin_tol = (T)1e-12;                                                             \
        if (!(det > sin_tol * sin_tol * g11 * g22)) { out.degenerate = 1; return out; }         \
        const T q11 = g22 / det, q22 = g11 / det, q12 = -g12 / det;                             \
        const T qt1 = q11 * t1 + q12 * t2;                                                      \
        const T qt2 = q12 * t1 + q22 * t2;                                                      \
        const T a = q11 + (T)2 * q12 + q22;                                                     \
        const T b = (T)(-2) * (qt1 + qt2);                                                      \
        const T c = t1 * qt1 + t2 * qt2 - (T)1;                                                 \
        const T disc = b * b - (T)4 * a * c;                                                    \
        if (disc >= (T)0) {                                                                     \
            const T p = (-b + TSQRT(disc)) / ((T)2 * a);                                        \
            const T tmax = t1 < t2 ? t2 : t1; /* std::max(t1, t2) */                            \
            if (p >= tmax) {                                                                    \
                const T m1 = q11 * (t1 - p) + q12 * (t2 - p);                                   \
                const T m2 = q12 * (t1 - p) + q22 * (t2 - p);                                   \
                if (m1 < (T)0 && m2 < (T)0 && p <= out.value) {                                 \
                    out.value = p;                                                              \
                    out.side = t1 <= t2 ? 0 : 1;                                                \
                }                                                                               \
            }                                                                                   \
        }                                                                                       \
        return out;                                                                             \
    }                                                                                           \
                                                                                                \
    void orc_planar_##SFX(const double* x1, const double* x2, double t1, double t2,            \
                          double* value, int* side, int* degenerate) {                         \
        const T a[3] = {(T)x1[0], (T)x1[1], (T)x1[2]};                                          \
        const T b[3] = {(T)x2[0], (T)x2[1], (T)x2[2]};                                          \
        const cand_##SFX r = planar_##SFX(a, b, (T)t1, (T)t2);                                  \
        *value = (double)r.value;                                                               \
        *side = r.side;                                                                         \
        *degenerate = r.degenerate;                                                             \
    }                                                                                           \
                                                                                                \
    /* ptp.cpp:37-43 */                                                                         \
    static T relchange_##SFX(T before, T after) {                                               \
        if (before == TINF) return after == TINF ? (T)0 : TINF;                                 \
        const T denom = before == (T)0 ? TMIN : before;                                         \
        return TABS(after - before) / denom;                                                    \
    }                                                                                           \
                                                                                                \
    /* run_impl<T> loop, ptp.cpp:45-148; relax_vertex, update_kernel.hpp:93-120 */             \
    static void run_##SFX(int n, const double* xyz, const int* cptr, const int* cv1,            \
                          const int* cv2, const int* sorted, const int* limits, int rho,        \
                          const int* sources, int m, double eps_d, double* out_dist,            \
                          int* out_labels, int64_t* stats, int64_t* trace_i64,                  \
                          double* trace_f64, int* trace_conv, int trace_cap, int* last_change) { \
        const T eps = (T)eps_d;                                                                 \
        T* pos = (T*)malloc(sizeof(T) * 3 * (size_t)n);                                         \
        T* dist[2];                                                                             \
        int* lab[2];                                                                            \
        for (int v = 0; v < 3 * n; ++v) pos[v] = (T)xyz[v];                                     \
        for (int s = 0; s < 2; ++s) {                                                           \
            dist[s] = (T*)malloc(sizeof(T) * (size_t)n);                                        \
            lab[s] = (int*)malloc(sizeof(int) * (size_t)n);                                     \
            for (int v = 0; v < n; ++v) { dist[s][v] = TINF; lab[s][v] = -1; }                  \
        }                                                                                       \
        for (int si = 0; si < m; ++si) {                                                        \
            dist[0][sources[si]] = dist[1][sources[si]] = (T)0;                                 \
            lab[0][sources[si]] = lab[1][sources[si]] = si;                                     \
        }                                                                                       \
        if (last_change) memset(last_change, 0, sizeof(int) * (size_t)n);                       \
        int prev = 0, curr = 1, i = 1, k = 0;                                                   \
        int64_t calls = 0, degen = 0;                                                           \
        while (i <= rho - 1) {                                                                  \
            ++k;                                                                                \
            const int j = k < rho ? k : rho - 1;                                                \
            const int bb = limits[i], be = limits[j + 1], fe = limits[i + 1];                   \
            const T* dp = dist[prev];                                                           \
            T* dc = dist[curr];                                                                 \
            const int* lp = lab[prev];                                                          \
            int* lc = lab[curr];                                                                \
            T max_rel = (T)0;                                                                   \
            for (int p = bb; p < be; ++p) {                                                     \
                const int v = sorted[p];                                                        \
                T best = dp[v];                                                                 \
                int best_label = lp[v];                                                         \
                const T* pv = pos + 3 * v;                                                      \
                for (int c = cptr[v]; c < cptr[v + 1]; ++c) {                                   \
                    const int v1 = cv1[c], v2 = cv2[c];                                         \
                    const int mixed = lp[v1] != lp[v2] && isfinite(dp[v1]) && isfinite(dp[v2]); \
                    const T t2 = mixed ? TINF : dp[v2];                                         \
                    T x1[3], x2[3];                                                             \
                    for (int d = 0; d < 3; ++d) {                                               \
                        x1[d] = pos[3 * v1 + d] - pv[d];                                        \
                        x2[d] = pos[3 * v2 + d] - pv[d];                                        \
                    }                                                                           \
                    cand_##SFX cd = planar_##SFX(x1, x2, dp[v1], t2);                           \
                    if (mixed) {                                                                \
                        const T other =                                                         \
                            dp[v2] + TSQRT(x2[0] * x2[0] + x2[1] * x2[1] + x2[2] * x2[2]);      \
                        if (other < cd.value) { cd.value = other; cd.side = 1; cd.degenerate = 0; } \
                    }                                                                           \
                    ++calls;                                                                    \
                    degen += cd.degenerate ? 1 : 0;                                             \
                    if (cd.value < best) {                                                      \
                        best = cd.value;                                                        \
                        best_label = lp[cd.side == 0 ? v1 : v2];                                \
                    }                                                                           \
                }                                                                               \
                dc[v] = best;                                                                   \
                lc[v] = best_label;                                                             \
                const T rc = relchange_##SFX(dp[v], best);                                      \
                if (p < fe && rc > max_rel) max_rel = rc;                                       \
                if (last_change && rc >= eps) last_change[v] = k;                               \
            }                                                                                   \
            const int converged = max_rel < eps;                                                \
            if (trace_i64 && k - 1 < trace_cap) {                                               \
                trace_i64[4 * (k - 1)] = k;                                                     \
                trace_i64[4 * (k - 1) + 1] = i;                                                 \
                trace_i64[4 * (k - 1) + 2] = j;                                                 \
                trace_i64[4 * (k - 1) + 3] = be - bb;                                           \
                trace_f64[k - 1] = (double)max_rel;                                             \
                trace_conv[k - 1] = converged;                                                  \
            }                                                                                   \
            if (converged) {                                                                    \
                for (int p = bb; p < fe; ++p) {                                                 \
                    const int v = sorted[p];                                                    \
                    dist[prev][v] = dc[v];                                                      \
                    lab[prev][v] = lc[v];                                                       \
                }                                                                               \
                ++i;                                                                            \
            }                                                                                   \
            prev ^= 1;                                                                          \
            curr ^= 1;                                                                          \
        }                                                                                       \
        for (int v = 0; v < n; ++v) out_dist[v] = (double)dist[prev][v];                        \
        if (out_labels) memcpy(out_labels, lab[prev], sizeof(int) * (size_t)n);                 \
        stats[0] = calls;                                                                       \
        stats[1] = degen;                                                                       \
        stats[2] = k;                                                                           \
        free(pos);                                                                              \
        for (int s = 0; s < 2; ++s) { free(dist[s]); free(lab[s]); }                            \
    }

DEFINE_PTP(float, f32, INFINITY, FLT_MIN, sqrtf, fabsf)
DEFINE_PTP(double, f64, (double)INFINITY, DBL_MIN, sqrt, fabs)

/*
 * ptp_run with its validation (ptp.cpp:152-167).  The ordering arrays are
 * the caller's (normally from orc_toplesets).  stats: [0] relax_calls,
 * [1] degenerate_calls, [2] K.  Trace rows as (k,i,j,updated) + max_rel + converged.
 */
int orc_ptp(int n, const double* xyz, const int* cptr, const int* cv1, const int* cv2,
            const int* sorted, const int* limits, int rho, const int* position,
            const int* sources, int m, double eps, int single, double* out_dist, int* out_labels,
            int64_t* stats, int64_t* trace_i64, double* trace_f64, int* trace_conv, int trace_cap,
            int* last_change) {
    if (m <= 0) FAIL(1, "ptp_run: empty source set");
    if (!(eps > 0)) FAIL(1, "ptp_run: epsilon must be positive");
    if (rho < 1 || limits[1] != m) FAIL(1, "ptp_run: ordering does not match the source set");
    for (int q = 0; q < m; ++q) {
        const int s = sources[q];
        if (s < 0 || s >= n || position[s] == -1 || position[s] >= limits[1])
            FAIL(1, "ptp_run: ordering does not match the source set");
    }
    if (single)
        run_f32(n, xyz, cptr, cv1, cv2, sorted, limits, rho, sources, m, eps, out_dist, out_labels,
                stats, trace_i64, trace_f64, trace_conv, trace_cap, last_change);
    else
        run_f64(n, xyz, cptr, cv1, cv2, sorted, limits, rho, sources, m, eps, out_dist, out_labels,
                stats, trace_i64, trace_f64, trace_conv, trace_cap, last_change);
    return 0;
}

/*
 * fps (sampling.cpp:11-49): m rounds of {toplesets from all samples, ptp with
 * labels, argmax with strict '>' from v = 0}.  history rows as
 * (sources, rho, relax_calls, picked) + radius.
 */
int orc_fps(int n, const double* xyz, const int* cptr, const int* cv1, const int* cv2,
            const int* ring_extra, int m, int seed, double eps, int single, int* samples,
            int* labels, double* radius, int64_t* hist_i64, double* hist_f64) {
    if (m < 1 || m > n) FAIL(1, "fps: sample count must be in [1, %d]", n);
    if (seed < 0 || seed >= n) FAIL(1, "fps: seed vertex out of range");
    int* sorted = (int*)malloc(sizeof(int) * (size_t)n);
    int* limits = (int*)malloc(sizeof(int) * (size_t)(n + 1));
    int* position = (int*)malloc(sizeof(int) * (size_t)n);
    double* dist = (double*)malloc(sizeof(double) * (size_t)n);
    int ns = 1, rho = 0, unreached = 0;
    samples[0] = seed;
    for (;;) {
        orc_toplesets(n, cptr, cv1, ring_extra, samples, ns, sorted, limits, position, &rho, &unreached);
        int64_t st[3];
        orc_ptp(n, xyz, cptr, cv1, cv2, sorted, limits, rho, position, samples, ns, eps, single,
                dist, labels, st, NULL, NULL, NULL, 0, NULL);
        int far = 0;
        double r = dist[0];
        for (int v = 1; v < n; ++v)
            if (dist[v] > r) { r = dist[v]; far = v; }
        const int final_run = ns == m;
        const int row = ns - 1;
        hist_i64[4 * row] = ns;
        hist_i64[4 * row + 1] = rho;
        hist_i64[4 * row + 2] = st[0];
        hist_i64[4 * row + 3] = final_run ? -1 : far;
        hist_f64[row] = r;
        if (final_run) { *radius = r; break; }
        samples[ns++] = far;
    }
    free(sorted); free(limits); free(position); free(dist);
    return 0;
}
