// C ABI (include/geodist_b200.h) over the sm_100a kernels.
//
// A geodist_mesh_t is the device-resident replica the reference rebuilds per
// call (Python MeshHandle, bindings.cpp:26-31): fan-CSR + per-precision
// geometry tables live in HBM for the mesh's lifetime; every solve reuses
// them.  Errors follow the reference's exception text; nothing here falls
// back to a CPU solve -- without an sm_100 device every compute call fails
// with GEODIST_ECUDA.
#include <algorithm>
#include <atomic>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/geodist_b200.h"
#include "mesh_host.hpp"
#include "ptp_common.cuh"
#include "ptp_launch.hpp"

namespace gdb {

static std::atomic<long long> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

namespace {

thread_local std::string g_err;

struct Fail : std::exception {
    int code;
    std::string msg;
    Fail(int c, std::string m) : code(c), msg(std::move(m)) {}
    const char* what() const noexcept override { return msg.c_str(); }
};

inline void cuda_ok(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw Fail(GEODIST_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return GEODIST_OK;
    } catch (const Fail& f) {
        g_err = f.msg;
        return f.code;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return GEODIST_EINVAL;
    } catch (const std::bad_alloc&) {
        g_err = "out of host memory";
        return GEODIST_ENOMEM;
    } catch (const std::exception& e) {
        g_err = e.what();
        return GEODIST_EMESH;
    }
}

template <typename X>
X* dalloc(size_t count) {
    void* p = nullptr;
    if (count == 0) count = 1;
    const cudaError_t e = cudaMalloc(&p, count * sizeof(X));
    if (e != cudaSuccess) {
        cudaGetLastError();
        throw Fail(GEODIST_ENOMEM, std::string("device allocation of ") +
                                       std::to_string(count * sizeof(X)) + " bytes failed");
    }
    return static_cast<X*>(p);
}

struct DFree {
    void operator()(void* p) const {
        if (p) cudaFree(p);
    }
};

void require_device(int device) {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
        cudaGetLastError();
        throw Fail(GEODIST_ECUDA, "no CUDA device available (the B200 solver has no CPU path)");
    }
    if (device < 0 || device >= count)
        throw Fail(GEODIST_EINVAL, "device " + std::to_string(device) + " out of range");
    cudaDeviceProp prop;
    cuda_ok(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
    if (prop.major != 10)
        throw Fail(GEODIST_ECUDA, std::string("device ") + prop.name +
                                      " is not sm_100 (this library is built for sm_100a only)");
    cuda_ok(cudaSetDevice(device), "cudaSetDevice");
}

}  // namespace

// fp32 multi-source cells pack the label into 24 bits (ptp_common.cuh Cell<float, true>)
constexpr long long kMaxLabels32 = (1 << 24) - 2;
static void check_label_range(int prec, long long m) {
    if (prec == GEODIST_SINGLE && m > kMaxLabels32)
        throw std::invalid_argument(
            "ptp_run: single-precision multi-source fields support at most 16777214 sources "
            "(use double precision)");
}

// Per-query device workspace for `groups` concurrent queries.
struct Workspace {
    int groups = 0;
    long long n = 0;
    void* cell0 = nullptr;  // Jacobi double buffer: Cell<T, LABELS> (<= 16 B) per vertex
    void* cell1 = nullptr;
    void* pcell0 = nullptr;  // the same by BFS position (wide iterations)
    void* pcell1 = nullptr;
    int* posof = nullptr;
    int* dflag = nullptr;    // wide-iteration relaxation marks, 2 per position
    int* level = nullptr;
    int* queue = nullptr;
    int* limits = nullptr;
    GroupCtl* ctl = nullptr;
    unsigned long long* scratch = nullptr;  // FPS argmax, 2 words per CTA
    int scratch_blocks = 0;
    int* pring = nullptr;                  // packed records by BFS position
    void* pL = nullptr;
    void* pquad = nullptr;
    int* blists = nullptr;                 // per-CTA claim lists [blocks][claim_cap]
    int claim_cap = 0;
    int claim_min = 0;                     // raised after a claim-list overflow

    // cell0/cell1/level/queue live in one block (`hot`): the per-vertex
    // arrays every iteration gathers from.  Solver launches mark it L2-persisting so
    // the streaming reads of ELL rows (one per vertex, ~n * 192 B per field) do not
    // evict the distance and level lines of the vertices the wavefront reaches next.
    char* hot = nullptr;
    size_t hot_bytes = 0;
    mutable cudaStream_t persisted_on = nullptr;  // stream whose window covers `hot`

    void release() {
        if (hot) cudaFree(hot);
        persisted_on = nullptr;
        for (void* p : {static_cast<void*>(limits), static_cast<void*>(ctl),
                        static_cast<void*>(scratch), static_cast<void*>(pring), pL, pquad,
                        static_cast<void*>(dflag),
                        static_cast<void*>(blists)})
            if (p) cudaFree(p);
        const int keep = claim_min;
        *this = Workspace();
        claim_min = keep;
    }
    // A CTA claimed more vertices in one iteration than its list holds (the solve
    // reported err 2 and stopped): the next ensure() sizes every list for the
    // worst case (a CTA can never claim more than n vertices in one iteration).
    void grow_claims() {
        claim_min = static_cast<int>(std::min<long long>(n + 1, INT_MAX));
        release();
    }
    void ensure(int g, long long nn, int blocks) {
        if (g <= groups && nn == n && blocks <= scratch_blocks) return;
        release();
        groups = g;
        n = nn;
        const size_t e = static_cast<size_t>(g) * static_cast<size_t>(nn);
        {
            auto up = [](size_t b) { return (b + 255) & ~static_cast<size_t>(255); };
            const size_t bc = up(e * kCellMaxBytes), b4 = up(e * sizeof(int));
            hot_bytes = 4 * bc + 3 * b4;
            hot = dalloc<char>(hot_bytes);
            char* x = hot;
            cell0 = x; x += bc;
            cell1 = x; x += bc;
            pcell0 = x; x += bc;
            pcell1 = x; x += bc;
            level = reinterpret_cast<int*>(x); x += b4;
            posof = reinterpret_cast<int*>(x); x += b4;
            queue = reinterpret_cast<int*>(x);
        }
        limits = dalloc<int>(static_cast<size_t>(g) * (nn + 2));
        ctl = dalloc<GroupCtl>(g);
        cuda_ok(cudaMemset(ctl, 0, sizeof(GroupCtl) * g), "memset ctl");
        scratch_blocks = blocks;
        scratch = dalloc<unsigned long long>(2 * static_cast<size_t>(blocks));
        pring = dalloc<int>(e * kEllW);
        dflag = dalloc<int>(2 * e);
        pL = dalloc<double>(e * kEllW);
        pquad = dalloc<char>(e * kEllW * 4 * sizeof(double));
        // a CTA rarely claims more than a few times its share of a level; beyond the
        // capacity the solve stops with err 2 and is redone with lists of n + 1 entries
        claim_cap = static_cast<int>(std::min<long long>(
            nn + 1, 8 * ((nn + blocks - 1) / std::max(1, blocks / std::max(1, g))) + 4096));
        claim_cap = std::max(claim_cap, claim_min);
        blists = dalloc<int>(static_cast<size_t>(blocks) * claim_cap);
    }
    // L2 access-policy window over the hot block for launches on `st`
    void persist(cudaStream_t st, int device) const {
        static const bool on = [] {
            const char* e = getenv("GEODIST_PERSIST");
            return !(e && e[0] == '0');
        }();
        if (!on || !hot || persisted_on == st) return;  // set once per stream and block
        int max_persist = 0, max_window = 0;
        cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, device);
        cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, device);
        if (max_persist <= 0 || max_window <= 0) return;
        // only when the block fits the set-aside comfortably (measured: 1-2 % faster
        // fields on 0.6-1 M-vertex meshes; a 4 M-vertex block would only thrash it)
        if (hot_bytes > static_cast<size_t>(max_persist)) return;
        const size_t bytes = std::min<size_t>(hot_bytes, static_cast<size_t>(max_window));
        const size_t limit = std::min<size_t>(bytes, static_cast<size_t>(max_persist));
        cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, limit);
        cudaStreamAttrValue v{};
        v.accessPolicyWindow.base_ptr = hot;
        v.accessPolicyWindow.num_bytes = bytes;
        v.accessPolicyWindow.hitRatio = static_cast<float>(static_cast<double>(limit) / bytes);
        v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &v);
        cudaGetLastError();  // the window is a hint: never fail a solve over it
        persisted_on = st;
    }

    void fill(RunArgs& a) const {
        const char* w = getenv("GEODIST_WIDE");
        a.wide_factor = w ? atoi(w) : kWideFactor;
        a.cell0 = cell0;
        a.cell1 = cell1;
        a.pcell0 = pcell0;
        a.pcell1 = pcell1;
        a.posof = posof;
        a.dflag = dflag;
        a.level = level;
        a.queue = queue;
        a.limits = limits;
        a.ctl = ctl;
        a.fps_scratch = scratch;
        a.pring = pring;
        a.pL = pL;
        a.pquad = pquad;
        a.blists = blists;
        a.claim_cap = claim_cap;
    }
};

}  // namespace gdb

using namespace gdb;

struct PrecTables {
    int* ring = nullptr;   // ring with degenerate flags for this precision
    void* ringL = nullptr;
    void* quad = nullptr;
    int* ering = nullptr;  // ELL-8 copies (interleaved)
    void* eL = nullptr;
    void* equad = nullptr;
};

struct geodist_mesh_s {
    int device = 0;
    int n = 0, nf = 0;
    long long corners = 0;
    Fans fans;               // host copy of the fan-CSR, downloaded on first use
    bool host_fans = false;  // (vertex_star / degree queries only; the solver never needs it)
    std::mutex fans_mu;
    int* degree_d = nullptr;
    double* xyz = nullptr;
    int* faces = nullptr;
    int* cptr = nullptr;
    int* ring = nullptr;
    PrecTables prec[2];
    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    Workspace ws;
    // toplesets scratch
    int* t_sorted = nullptr;
    int* t_position = nullptr;
    int* t_scratch = nullptr;
    size_t t_scratch_words = 0;
    int* d_src = nullptr;
    size_t d_src_cap = 0;
    int* d_i32 = nullptr;  // generic n-sized int buffer
    std::mutex mu;
    // grow-only per-call device buffers (no cudaMalloc on the solve path)
    void* pool[8] = {};
    size_t pool_cap[8] = {};
    void* buf(int slot, size_t bytes) {
        if (bytes > pool_cap[slot]) {
            if (pool[slot]) cudaFree(pool[slot]);
            pool[slot] = nullptr;
            pool[slot] = dalloc<char>(bytes);
            pool_cap[slot] = bytes;
        }
        return pool[slot];
    }

    ~geodist_mesh_s() {
        cudaSetDevice(device);
        if (stream) cudaStreamSynchronize(stream);
        ws.release();
        for (void* p : {static_cast<void*>(xyz), static_cast<void*>(faces),
                        static_cast<void*>(cptr), static_cast<void*>(ring),
                        static_cast<void*>(t_sorted), static_cast<void*>(t_position),
                        static_cast<void*>(t_scratch), static_cast<void*>(d_src),
                        static_cast<void*>(d_i32), static_cast<void*>(degree_d)})
            if (p) cudaFree(p);
        for (auto& t : prec)
            for (void* p : {static_cast<void*>(t.ring), t.ringL, t.quad,
                            static_cast<void*>(t.ering), t.eL, t.equad})
                if (p) cudaFree(p);
        for (void* p : pool)
            if (p) cudaFree(p);
        if (ev0) cudaEventDestroy(ev0);
        if (ev1) cudaEventDestroy(ev1);
        if (stream) cudaStreamDestroy(stream);
    }

    bool has_geometry = true;

    void ensure_prec(int p) {
        if (!has_geometry)
            throw Fail(GEODIST_EINVAL, "mesh was created without vertex positions (topology only)");
        PrecTables& t = prec[p];
        if (t.quad) return;
        const size_t ring_len = static_cast<size_t>(corners) + n;
        const size_t tsz = p == 0 ? sizeof(float) : sizeof(double);
        t.ring = dalloc<int>(ring_len);
        t.ringL = dalloc<char>(ring_len * tsz);
        t.quad = dalloc<char>(static_cast<size_t>(corners > 0 ? corners : 1) * 4 * tsz);
        const size_t ell = static_cast<size_t>(n > 0 ? n : 1) * kEllW;
        t.ering = dalloc<int>(ell);
        t.eL = dalloc<char>(ell * tsz);
        t.equad = dalloc<char>(ell * 4 * tsz);
        if (p == 0)
            launch_pack<float>(xyz, n, cptr, ring, t.ring, t.ringL, t.quad, t.ering, t.eL, t.equad,
                               stream);
        else
            launch_pack<double>(xyz, n, cptr, ring, t.ring, t.ringL, t.quad, t.ering, t.eL,
                                t.equad, stream);
        cuda_ok(cudaGetLastError(), "pack_kernel");
        cuda_ok(cudaStreamSynchronize(stream), "pack_kernel");
    }

    int* upload_sources(const int32_t* src, size_t count) {
        if (count > d_src_cap) {
            if (d_src) cudaFree(d_src);
            d_src_cap = std::max<size_t>(count, 1024);
            d_src = dalloc<int>(d_src_cap);
        }
        if (count)
            cuda_ok(cudaMemcpyAsync(d_src, src, count * sizeof(int), cudaMemcpyHostToDevice, stream),
                    "upload sources");
        return d_src;
    }
};

namespace {

geodist_mesh_s* M(geodist_mesh_t h) {
    if (!h) throw Fail(GEODIST_EINVAL, "null mesh handle");
    return static_cast<geodist_mesh_s*>(h);
}

// Host copy of a device-built fan-CSR (downloaded once, on the first host-side query).
const Fans& host_fans(geodist_mesh_s* m) {
    std::lock_guard<std::mutex> lk(m->fans_mu);
    if (m->host_fans) return m->fans;
    cuda_ok(cudaSetDevice(m->device), "cudaSetDevice");
    Fans& f = m->fans;
    f.n = m->n;
    f.cptr.resize(static_cast<size_t>(m->n) + 1);
    f.ring.resize(static_cast<size_t>(m->corners) + m->n);
    f.degree.resize(static_cast<size_t>(m->n));
    cuda_ok(cudaMemcpy(f.cptr.data(), m->cptr, sizeof(int) * f.cptr.size(), cudaMemcpyDeviceToHost),
            "download fans");
    cuda_ok(cudaMemcpy(f.ring.data(), m->ring, sizeof(int) * f.ring.size(), cudaMemcpyDeviceToHost),
            "download fans");
    if (m->n)
        cuda_ok(cudaMemcpy(f.degree.data(), m->degree_d, sizeof(int) * f.degree.size(),
                           cudaMemcpyDeviceToHost), "download fans");
    m->host_fans = true;
    return f;
}

// compute_toplesets source validation (toplesets.cpp:18-34): sorted copy.
std::vector<int> checked_sources(const int32_t* sources, int32_t m, int32_t n,
                                 const char* who = "compute_toplesets") {
    if (m <= 0 || sources == nullptr)
        throw std::invalid_argument(std::string(who) + ": empty source set");
    std::vector<int> s(sources, sources + m);
    std::sort(s.begin(), s.end());
    for (size_t i = 0; i < s.size(); ++i) {
        if (s[i] < 0 || s[i] >= n)
            throw std::invalid_argument(std::string(who) + ": source index " +
                                        std::to_string(s[i]) + " out of range");
        if (i > 0 && s[i] == s[i - 1])
            throw std::invalid_argument(std::string(who) + ": duplicate source index " +
                                        std::to_string(s[i]));
    }
    return s;
}

void check_config(const geodist_ptp_config* c) {
    if (!c) throw Fail(GEODIST_EINVAL, "null config");
    if (!(c->epsilon > 0)) throw std::invalid_argument("ptp_run: epsilon must be positive");
    if (c->precision != GEODIST_SINGLE && c->precision != GEODIST_DOUBLE)
        throw std::invalid_argument("precision must be 'single' or 'double'");
}

// Everything one distance-field solve needs from the caller.
struct Solve {
    const int32_t* sources = nullptr;
    int32_t m = 0;
    const geodist_ptp_config* cfg = nullptr;
    double* distances = nullptr;
    int32_t* labels = nullptr;
    geodist_ptp_stats* stats = nullptr;
    geodist_band_row* trace = nullptr;
    int32_t trace_cap = 0;
    int32_t* last_change = nullptr;
    geodist_observer_fn observer = nullptr;
    void* observer_user = nullptr;
    // caller ordering (ptp_run) or fused BFS
    bool ordered = false;
    const int32_t* sorted = nullptr;
    int32_t reachable = 0;
    const int32_t* limits = nullptr;
    int32_t rho = 0;
};

void run_solve(geodist_mesh_s* mh, const Solve& q) {
    const int prec = q.cfg->precision;
    const bool labels = q.m > 1;  // single source: labels are provably inert
    check_label_range(prec, q.m);
    mh->ensure_prec(prec);
    const int n = mh->n;
    const int maxb = std::min(run_max_blocks(prec, labels, mh->device, 0),
                              std::min(run_max_blocks(prec, labels, mh->device, 1),
                                       run_max_blocks(prec, labels, mh->device, 2)));
    if (maxb <= 0) throw Fail(GEODIST_ECUDA, "run kernel cannot be resident on this device");
    // With an IterationObserver the claim lists are sized for the worst case up front: a
    // claim-list overflow redoes the field, and the observer must see every iteration
    // exactly once (ptp.cpp:118-120).
    if (q.observer != nullptr && q.cfg->precision == GEODIST_DOUBLE &&
        mh->ws.claim_min < n + 1) {
        mh->ws.release();
        mh->ws.claim_min = n + 1;
    }
    mh->ws.ensure(1, n, maxb);
    Workspace& ws = mh->ws;
    cudaStream_t st = mh->stream;

    int* d_src = mh->upload_sources(q.sources, static_cast<size_t>(q.m));
    if (q.ordered) {
        cuda_ok(cudaMemcpyAsync(ws.queue, q.sorted, sizeof(int) * q.reachable,
                                cudaMemcpyHostToDevice, st), "upload ordering");
        cuda_ok(cudaMemcpyAsync(ws.limits, q.limits, sizeof(int) * (q.rho + 1),
                                cudaMemcpyHostToDevice, st), "upload limits");
    }
    const bool want_trace = q.cfg->record_trace && (q.trace || q.last_change);
    const bool stepwise = q.observer != nullptr && prec == GEODIST_DOUBLE;
    const int chunk = stepwise ? 1 : (want_trace ? 4096 : 0);

    double* d_out = static_cast<double*>(mh->buf(0, sizeof(double) * n));
    int* d_lab = q.labels ? static_cast<int*>(mh->buf(1, sizeof(int) * n)) : nullptr;
    int* d_lc = want_trace && q.last_change ? static_cast<int*>(mh->buf(2, sizeof(int) * n))
                                            : nullptr;
    TraceRow* d_tr = want_trace ? static_cast<TraceRow*>(mh->buf(3, sizeof(TraceRow) * chunk))
                                : nullptr;
    QueryStats* d_qs = static_cast<QueryStats*>(mh->buf(4, sizeof(QueryStats)));

    RunArgs a{};
    a.mesh.cptr = mh->cptr;
    a.mesh.ring = mh->prec[prec].ring;
    a.mesh.ringL = mh->prec[prec].ringL;
    a.mesh.quad = mh->prec[prec].quad;
    a.mesh.ering = mh->prec[prec].ering;
    a.mesh.eL = mh->prec[prec].eL;
    a.mesh.equad = mh->prec[prec].equad;
    a.mesh.n = n;
    ws.fill(a);
    ws.persist(st, mh->device);
    a.stride = n;
    a.groups = 1;
    a.blocks_per_group = maxb;
    a.src = d_src;
    a.src_off = nullptr;
    a.src_count = q.m;
    a.nq = 1;
    a.eps = q.cfg->epsilon;
    a.fused_bfs = q.ordered ? 0 : 1;
    a.given_rho = q.rho;
    a.max_iters = chunk;
    a.trace = d_tr;
    a.trace_cap = chunk;
    a.last_change = d_lc;
    a.out_dist = d_out;
    a.out_double = 1;
    a.out_labels = d_lab;
    a.qstats = d_qs;
    a.fps_mode = 0;
    if (const char* e = getenv("GEODIST_DEBUG_TIMING")) {
        a.dbg_iters = atoi(e);
        a.dbg = static_cast<unsigned long long*>(
            mh->buf(5, sizeof(unsigned long long) * kDbgSlots * static_cast<size_t>(a.dbg_iters) * maxb));
        cuda_ok(cudaMemsetAsync(a.dbg, 0, sizeof(unsigned long long) * kDbgSlots * a.dbg_iters * maxb, st),
                "dbg");
    }

    std::vector<TraceRow> rows;
    std::vector<double> snap;
    float total_ms = 0.f;
    GroupCtl hctl{};
    // Without per-iteration host work the narrow-band and wide-band instantiations
    // hand the field to each other at band cross-overs (each carries only its own
    // path's registers); otherwise (trace chunks, observer) the combined kernel.
    const bool switching = chunk <= 0 && !getenv("GEODIST_NO_MODES");
    int mode = switching ? 1 : 0;
    for (int launch = 0;; ++launch) {
        a.phase_init = launch == 0 ? 1 : 0;
        a.trace_k0 = hctl.k + 1;
        if (switching && launch >= 64) mode = 0;  // pathological oscillation
        cuda_ok(cudaEventRecord(mh->ev0, st), "event");
        cuda_ok(launch_run(prec, labels, a, st, mode), "ptp_run_kernel launch");
        cuda_ok(cudaEventRecord(mh->ev1, st), "event");
        cuda_ok(cudaMemcpyAsync(&hctl, ws.ctl, sizeof(GroupCtl), cudaMemcpyDeviceToHost, st),
                "read state");
        cuda_ok(cudaStreamSynchronize(st), "ptp_run_kernel");
        float ms = 0.f;
        cudaEventElapsedTime(&ms, mh->ev0, mh->ev1);
        total_ms += ms;
        static const bool log_launches = getenv("GEODIST_LAUNCH_LOG") != nullptr;
        if (log_launches)
            fprintf(stderr, "launch %d mode %d: %.3f ms, k %d, i %d, exit %d, done %d\n", launch,
                    mode, ms, hctl.k, hctl.i, hctl.mode_exit, hctl.done);
        if (hctl.err >= 2) {
            // a CTA's claim list overflowed (the kernel stopped the field): redo it
            // with lists that cannot overflow, before any observer call sees it
            ws.grow_claims();
            run_solve(mh, q);
            return;
        }
        if (want_trace && q.trace) {
            const int got = hctl.k - a.trace_k0 + 1;
            if (got > 0) {
                const size_t old = rows.size();
                rows.resize(old + got);
                cuda_ok(cudaMemcpy(rows.data() + old, a.trace, sizeof(TraceRow) * got,
                                   cudaMemcpyDeviceToHost), "read trace");
            }
        }
        if (stepwise && hctl.k >= a.trace_k0) {
            // IterationObserver: snapshot of dist[curr] after iteration k (ptp.cpp:118-120);
            // the buffer written last is the one the saved parity names.
            const void* buf = hctl.parity ? ws.cell1 : ws.cell0;
            snap.resize(n);
            // the distance is the first 8 bytes of each fp64 cell
            const size_t pitch = labels ? sizeof(Cell<double, true>) : sizeof(Cell<double, false>);
            cuda_ok(cudaMemcpy2D(snap.data(), sizeof(double), buf, pitch, sizeof(double), n,
                                 cudaMemcpyDeviceToHost), "snapshot");
            q.observer(q.observer_user, hctl.k, snap.data(), n);
        }
        if (hctl.done) break;
        if (switching && hctl.mode_exit != 0) {
            mode = hctl.mode_exit;
            continue;
        }
        if (chunk <= 0) throw Fail(GEODIST_ECUDA, "solver returned before convergence");
    }
    QueryStats qs{};
    cuda_ok(cudaMemcpy(&qs, a.qstats, sizeof(QueryStats), cudaMemcpyDeviceToHost), "stats");
    if (qs.pad >= 2) throw Fail(GEODIST_ECUDA, "solver error " + std::to_string(qs.pad));
    if (a.dbg) {
        std::vector<unsigned long long> h(kDbgSlots * static_cast<size_t>(a.dbg_iters) * maxb);
        cuda_ok(cudaMemcpy(h.data(), a.dbg, h.size() * 8, cudaMemcpyDeviceToHost), "dbg");
        if (FILE* f = fopen("gpurun_out/dbg_timing.bin", "wb")) {
            const int hdr[2] = {a.dbg_iters, maxb};
            fwrite(hdr, sizeof(int), 2, f);
            fwrite(h.data(), 8, h.size(), f);
            fclose(f);
        }
    }
    if (q.distances)
        cuda_ok(cudaMemcpy(q.distances, d_out, sizeof(double) * n, cudaMemcpyDeviceToHost),
                "read distances");
    if (q.labels)
        cuda_ok(cudaMemcpy(q.labels, a.out_labels, sizeof(int) * n, cudaMemcpyDeviceToHost),
                "read labels");
    if (want_trace && q.last_change)
        cuda_ok(cudaMemcpy(q.last_change, a.last_change, sizeof(int) * n, cudaMemcpyDeviceToHost),
                "read last_change");
    if (want_trace && q.trace) {
        const int cnt = std::min<int>(static_cast<int>(rows.size()), q.trace_cap);
        for (int r = 0; r < cnt; ++r) {
            geodist_band_row& o = q.trace[r];
            o.k = rows[r].k;
            o.i = rows[r].i;
            o.j = rows[r].j;
            o.front_converged = rows[r].conv;
            o.updated = rows[r].updated;
            o.max_rel_change = rows[r].max_rel;
        }
    }
    if (q.stats) {
        q.stats->relax_calls = qs.relax;
        q.stats->degenerate_calls = qs.degen;
        q.stats->vertex_updates = qs.updates;
        q.stats->iterations = qs.iterations;
        q.stats->rho = qs.rho;
        q.stats->unreached = qs.unreached;
        q.stats->workers = q.cfg->workers > 0 ? q.cfg->workers : 1;
        q.stats->wall_seconds = total_ms * 1e-3;
        q.stats->total_seconds = total_ms * 1e-3;
    }
}

}  // namespace

extern "C" {

const char* geodist_last_error(void) { return g_err.c_str(); }
int32_t geodist_version(void) { return 100; }
int64_t geodist_kernel_launches(void) { return g_launches.load(); }
int geodist_reset_persisting_l2(void) {
    return guarded([&] { cuda_ok(cudaCtxResetPersistingL2Cache(), "reset persisting L2"); });
}

int geodist_device_count(int32_t* count) {
    return guarded([&] {
        int c = 0;
        if (cudaGetDeviceCount(&c) != cudaSuccess) {
            cudaGetLastError();
            c = 0;
        }
        *count = c;
    });
}

int geodist_mesh_create(const double* xyz, int32_t n, const int32_t* faces, int32_t nf,
                        int32_t device, geodist_mesh_t* out) {
    return guarded([&] {
        if (!out) throw Fail(GEODIST_EINVAL, "null output handle");
        *out = nullptr;
        if (n < 0 || nf < 0 || (nf > 0 && !faces))
            throw Fail(GEODIST_EINVAL, "invalid mesh arrays");
        int count = 0;
        const bool have_gpu = cudaGetDeviceCount(&count) == cudaSuccess && count > 0;
        if (!have_gpu) cudaGetLastError();
        // The fan-CSR is built on the device (mesh_build.cu); the host build runs only
        // when asked for (GEODIST_HOST_BUILD=1), for meshes beyond int32 half-edge ids,
        // and -- for its exact error text -- on a mesh the device build rejects or on a
        // machine without a device (mesh errors before device errors, as before).
        const char* hb = std::getenv("GEODIST_HOST_BUILD");
        const bool host_build = !have_gpu || (hb && hb[0] == '1') || 3LL * nf > INT32_MAX;
        Fans fans;
        if (host_build) fans = build_fans(xyz, n, faces, nf);  // runtime_error -> EMESH
        if (n > kIdMask) throw Fail(GEODIST_EINVAL, "mesh too large: at most 2^27-1 vertices");
        require_device(device);
        std::unique_ptr<geodist_mesh_s> m(new geodist_mesh_s);
        m->device = device;
        m->n = n;
        m->nf = nf;
        m->corners = 3LL * nf;  // every outgoing half-edge of a manifold star is a corner
        cuda_ok(cudaStreamCreateWithFlags(&m->stream, cudaStreamNonBlocking), "stream");
        cuda_ok(cudaEventCreate(&m->ev0), "event");
        cuda_ok(cudaEventCreate(&m->ev1), "event");
        m->xyz = dalloc<double>(3 * static_cast<size_t>(n));
        m->faces = dalloc<int>(3 * static_cast<size_t>(nf));
        m->cptr = dalloc<int>(static_cast<size_t>(n) + 1);
        m->ring = dalloc<int>(3 * static_cast<size_t>(nf) + n);
        m->has_geometry = xyz != nullptr;
        if (xyz)
            cuda_ok(cudaMemcpy(m->xyz, xyz, sizeof(double) * 3 * n, cudaMemcpyHostToDevice),
                    "upload");
        if (nf)
            cuda_ok(cudaMemcpy(m->faces, faces, sizeof(int) * 3 * nf, cudaMemcpyHostToDevice),
                    "upload");
        if (host_build) {
            cuda_ok(cudaMemcpy(m->cptr, fans.cptr.data(), sizeof(int) * (n + 1),
                               cudaMemcpyHostToDevice), "upload");
            cuda_ok(cudaMemcpy(m->ring, fans.ring.data(), sizeof(int) * fans.ring.size(),
                               cudaMemcpyHostToDevice), "upload");
            m->fans = std::move(fans);
            m->host_fans = true;
        } else {
            int sms = 148;
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
            m->degree_d = dalloc<int>(static_cast<size_t>(n));
            std::unique_ptr<int, DFree> scratch(
                dalloc<int>(build_fans_scratch_ints(n, nf) + 3 * static_cast<size_t>(nf)));
            int* twin = scratch.get() + build_fans_scratch_ints(n, nf);
            cudaError_t err = cudaSuccess;
            const unsigned flag =
                build_fans_device(xyz ? m->xyz : nullptr, n, m->faces, nf, m->cptr, m->ring,
                                  m->degree_d, twin, scratch.get(), sms, m->stream, &err);
            cuda_ok(err, "device mesh build");
            if (flag) {
                build_fans(xyz, n, faces, nf);  // throws the reference's message
                throw std::runtime_error("mesh rejected by the device build (flags " +
                                         std::to_string(flag) + ")");
            }
        }
        *out = m.release();
    });
}

int geodist_mesh_destroy(geodist_mesh_t mesh) {
    return guarded([&] { delete static_cast<geodist_mesh_s*>(mesh); });
}

int geodist_mesh_sizes(geodist_mesh_t mesh, int32_t* n, int32_t* nf, int64_t* corners) {
    return guarded([&] {
        auto* m = M(mesh);
        if (n) *n = m->n;
        if (nf) *nf = m->nf;
        if (corners) *corners = m->corners;
    });
}

int geodist_mesh_degrees(geodist_mesh_t mesh, int32_t* degree) {
    return guarded([&] {
        auto* m = M(mesh);
        const Fans& f = host_fans(m);
        std::copy(f.degree.begin(), f.degree.end(), degree);
    });
}

int geodist_mesh_fan(geodist_mesh_t mesh, int32_t v, int32_t* v1, int32_t* v2, int32_t cap,
                     int32_t* count) {
    return guarded([&] {
        auto* m = M(mesh);
        if (v < 0 || v >= m->n) throw std::invalid_argument("vertex_star: index out of range");
        const Fans& f = host_fans(m);
        const int c0 = f.cptr[v], d = f.cptr[v + 1] - c0, r0 = c0 + v;
        *count = d;
        if (d > cap) throw Fail(GEODIST_EINVAL, "fan larger than cap");
        for (int c = 0; c < d; ++c) {
            v1[c] = f.ring[r0 + c];
            v2[c] = f.ring[r0 + c + 1];
        }
    });
}

int geodist_mesh_fans(geodist_mesh_t mesh, int32_t* cptr, int32_t* ring, int32_t* degree) {
    return guarded([&] {
        auto* m = M(mesh);
        const Fans& f = host_fans(m);
        if (cptr) std::copy(f.cptr.begin(), f.cptr.end(), cptr);
        if (ring) std::copy(f.ring.begin(), f.ring.end(), ring);
        if (degree) std::copy(f.degree.begin(), f.degree.end(), degree);
    });
}

int geodist_build_fans(const double* xyz, int32_t n, const int32_t* faces, int32_t nf,
                       int32_t* cptr, int32_t* ring, int32_t* degree) {
    return guarded([&] {
        const Fans f = build_fans(xyz, n, faces, nf);
        std::copy(f.cptr.begin(), f.cptr.end(), cptr);
        std::copy(f.ring.begin(), f.ring.end(), ring);
        if (degree) std::copy(f.degree.begin(), f.degree.end(), degree);
    });
}

struct geodist_meshfile_s {
    MeshData m;
};

int geodist_meshfile_load(const char* path, geodist_meshfile_t* out, int32_t* n, int32_t* nf) {
    return guarded([&] {
        if (!path || !out) throw Fail(GEODIST_EINVAL, "null argument");
        *out = nullptr;
        std::unique_ptr<geodist_meshfile_s> f(new geodist_meshfile_s);
        load_mesh_file(path, f->m);  // runtime_error -> EMESH (the reference's text)
        if (n) *n = static_cast<int32_t>(f->m.xyz.size() / 3);
        if (nf) *nf = static_cast<int32_t>(f->m.faces.size() / 3);
        *out = f.release();
    });
}

int geodist_meshfile_copy(geodist_meshfile_t file, double* xyz, int32_t* faces) {
    return guarded([&] {
        if (!file) throw Fail(GEODIST_EINVAL, "null mesh file handle");
        if (xyz) std::copy(file->m.xyz.begin(), file->m.xyz.end(), xyz);
        if (faces) std::copy(file->m.faces.begin(), file->m.faces.end(), faces);
    });
}

int geodist_meshfile_free(geodist_meshfile_t file) {
    return guarded([&] { delete file; });
}

int geodist_write_mesh(const char* path, const double* xyz, int32_t n, const int32_t* faces,
                       int32_t nf, int32_t format) {
    return guarded([&] {
        if (!path || (n > 0 && !xyz) || (nf > 0 && !faces) || n < 0 || nf < 0)
            throw Fail(GEODIST_EINVAL, "invalid mesh arrays");
        write_mesh_file(path, xyz, n, faces, nf, format == GEODIST_FORMAT_OFF);
    });
}

int geodist_validate_mesh(const double* xyz, int32_t n, const int32_t* faces, int32_t nf) {
    return guarded([&] { validate(xyz, n, faces, nf); });
}

int geodist_build_halfedges(const double* xyz, int32_t n, const int32_t* faces, int32_t nf,
                            int32_t* twin, int32_t* vertex_halfedge) {
    return guarded([&] {
        const Fans f = build_fans(xyz, n, faces, nf);
        std::copy(f.twin.begin(), f.twin.end(), twin);
        std::copy(f.vstart.begin(), f.vstart.end(), vertex_halfedge);
    });
}

int geodist_grid_sizes(int32_t nx, int32_t ny, int32_t* n, int32_t* nf) {
    return guarded([&] {
        if (nx < 2 || ny < 2) throw std::invalid_argument("generate_grid: nx and ny must be >= 2");
        *n = nx * ny;
        *nf = 2 * (nx - 1) * (ny - 1);
    });
}
int geodist_generate_grid(int32_t nx, int32_t ny, double shear, double* xyz, int32_t* faces) {
    return guarded([&] { generate_grid(nx, ny, shear, xyz, faces); });
}
int geodist_icosphere_sizes(int32_t subdiv, int32_t* n, int32_t* nf) {
    return guarded([&] { icosphere_sizes(subdiv, n, nf); });
}
int geodist_generate_icosphere(int32_t subdiv, double* xyz, int32_t* faces) {
    return guarded([&] { generate_icosphere(subdiv, xyz, faces); });
}
int geodist_perturb_radial(double* xyz, int32_t n, double sigma, uint32_t seed) {
    return guarded([&] { perturb_radial(xyz, n, sigma, seed); });
}
int geodist_torus_sizes(int32_t nu, int32_t nv, int32_t* n, int32_t* nf) {
    return guarded([&] {
        if (nu < 3 || nv < 3) throw std::invalid_argument("generate_torus: nu and nv must be >= 3");
        *n = nu * nv;
        *nf = 2 * nu * nv;
    });
}
int geodist_generate_torus(int32_t nu, int32_t nv, double R, double r, double* xyz,
                           int32_t* faces) {
    return guarded([&] { generate_torus(nu, nv, R, r, xyz, faces); });
}
int geodist_heightfield(double* xyz, int32_t n, double amp, double wx, double wy) {
    return guarded([&] { heightfield(xyz, n, amp, wx, wy); });
}

int geodist_toplesets(geodist_mesh_t mesh, const int32_t* sources, int32_t m, int32_t* sorted,
                      int32_t* limits, int32_t* position, int32_t* rho, int32_t* unreached) {
    return guarded([&] {
        auto* mh = M(mesh);
        std::lock_guard<std::mutex> lock(mh->mu);
        const std::vector<int> s = checked_sources(sources, m, mh->n);
        cuda_ok(cudaSetDevice(mh->device), "cudaSetDevice");
        const int n = mh->n;
        const int maxb = std::max(1, topo_max_blocks(mh->device));
        mh->ws.ensure(1, n, run_max_blocks(0, false, mh->device, 0));
        if (!mh->t_sorted) {
            mh->t_sorted = dalloc<int>(n);
            mh->t_position = dalloc<int>(n);
            // the (level, chunk) count table of the exact-order pass (toplesets.cu)
            mh->t_scratch_words = std::max<size_t>(static_cast<size_t>(n) / 16 + 1, 1u << 22);
            mh->t_scratch = dalloc<int>(mh->t_scratch_words);
        }
        int* d_src = mh->upload_sources(s.data(), s.size());
        std::unique_ptr<void, DFree> rho_d(dalloc<int>(1));
        TopoArgs a{};
        a.cptr = mh->cptr;
        a.ring = mh->ring;
        a.n = n;
        a.src = d_src;
        a.m = m;
        a.level = mh->ws.level;
        a.queue = mh->ws.queue;
        a.limits = mh->ws.limits;
        a.sorted = mh->t_sorted;
        a.position = mh->t_position;
        a.ctl = mh->ws.ctl;
        a.rho_out = static_cast<int*>(rho_d.get());
        a.blocks = std::min(maxb, 148 * 2);
        int r = 0;
        cuda_ok(launch_toplesets(a, mh->t_scratch, mh->t_scratch_words, &r, mh->stream),
                "toplesets");
        std::vector<int> lim(static_cast<size_t>(r) + 1);
        cuda_ok(cudaMemcpyAsync(lim.data(), a.limits, sizeof(int) * (r + 1),
                                cudaMemcpyDeviceToHost, mh->stream), "read limits");
        cuda_ok(cudaStreamSynchronize(mh->stream), "toplesets");
        const int reach = lim[r];
        if (sorted)
            cuda_ok(cudaMemcpy(sorted, a.sorted, sizeof(int) * reach, cudaMemcpyDeviceToHost),
                    "read sorted");
        if (limits) std::copy(lim.begin(), lim.end(), limits);
        if (position)
            cuda_ok(cudaMemcpy(position, a.position, sizeof(int) * n, cudaMemcpyDeviceToHost),
                    "read position");
        if (rho) *rho = r;
        if (unreached) *unreached = n - reach;
    });
}

int geodist_reorder_for_bands(geodist_mesh_t mesh, const int32_t* sources, int32_t m,
                              int32_t* old_of_new, int32_t* new_of_old, int32_t* faces_out) {
    int r = 0, unr = 0;
    int rc = geodist_toplesets(mesh, sources, m, nullptr, nullptr, nullptr, &r, &unr);
    if (rc != GEODIST_OK) return rc;
    return guarded([&] {
        auto* mh = M(mesh);
        std::lock_guard<std::mutex> lock(mh->mu);
        cuda_ok(cudaSetDevice(mh->device), "cudaSetDevice");
        const int n = mh->n, nf = mh->nf;
        std::unique_ptr<void, DFree> oon(dalloc<int>(n)), noo(dalloc<int>(n)),
            fo(dalloc<int>(3 * static_cast<size_t>(nf)));
        cuda_ok(launch_reorder(mh->t_position, mh->t_sorted, n - unr, n, mh->faces, nf,
                               static_cast<int*>(oon.get()), static_cast<int*>(noo.get()),
                               static_cast<int*>(fo.get()), mh->stream), "reorder");
        cuda_ok(cudaStreamSynchronize(mh->stream), "reorder");
        if (old_of_new)
            cuda_ok(cudaMemcpy(old_of_new, oon.get(), sizeof(int) * n, cudaMemcpyDeviceToHost), "d2h");
        if (new_of_old)
            cuda_ok(cudaMemcpy(new_of_old, noo.get(), sizeof(int) * n, cudaMemcpyDeviceToHost), "d2h");
        if (faces_out)
            cuda_ok(cudaMemcpy(faces_out, fo.get(), sizeof(int) * 3 * nf, cudaMemcpyDeviceToHost),
                    "d2h");
    });
}

int geodist_reorder_ordered(geodist_mesh_t mesh, const int32_t* sorted, int32_t reachable,
                            const int32_t* position, int32_t* old_of_new, int32_t* new_of_old,
                            int32_t* faces_out, double* xyz_out) {
    return guarded([&] {
        auto* mh = M(mesh);
        std::lock_guard<std::mutex> lock(mh->mu);
        const int n = mh->n, nf = mh->nf;
        if (reachable < 0 || reachable > n || (reachable > 0 && !sorted) || !position)
            throw std::invalid_argument("reorder_for_bands: ordering built for a different mesh");
        // the ordering must be a partial permutation: position[sorted[p]] == p, and
        // exactly `reachable` vertices have a position (toplesets.hpp:16-28)
        int have = 0;
        for (int v = 0; v < n; ++v) have += position[v] >= 0;
        bool ok = have == reachable;
        for (int p = 0; ok && p < reachable; ++p)
            ok = sorted[p] >= 0 && sorted[p] < n && position[sorted[p]] == p;
        if (!ok) throw std::invalid_argument("reorder_for_bands: ordering built for a different mesh");
        if (xyz_out && !mh->has_geometry)
            throw Fail(GEODIST_EINVAL, "mesh was created without vertex positions (topology only)");
        cuda_ok(cudaSetDevice(mh->device), "cudaSetDevice");
        std::unique_ptr<void, DFree> srt(dalloc<int>(std::max(reachable, 1))), pos(dalloc<int>(n)),
            oon(dalloc<int>(n)), noo(dalloc<int>(n)), fo(dalloc<int>(3 * static_cast<size_t>(nf))),
            xo(xyz_out ? dalloc<double>(3 * static_cast<size_t>(n)) : nullptr);
        cudaStream_t st = mh->stream;
        if (reachable)
            cuda_ok(cudaMemcpyAsync(srt.get(), sorted, sizeof(int) * reachable,
                                    cudaMemcpyHostToDevice, st), "h2d");
        cuda_ok(cudaMemcpyAsync(pos.get(), position, sizeof(int) * n, cudaMemcpyHostToDevice, st),
                "h2d");
        cuda_ok(launch_reorder(static_cast<int*>(pos.get()), static_cast<int*>(srt.get()),
                               reachable, n, mh->faces, nf, static_cast<int*>(oon.get()),
                               static_cast<int*>(noo.get()), static_cast<int*>(fo.get()), st,
                               xyz_out ? mh->xyz : nullptr, static_cast<double*>(xo.get())),
                "reorder");
        cuda_ok(cudaStreamSynchronize(st), "reorder");
        if (old_of_new)
            cuda_ok(cudaMemcpy(old_of_new, oon.get(), sizeof(int) * n, cudaMemcpyDeviceToHost), "d2h");
        if (new_of_old)
            cuda_ok(cudaMemcpy(new_of_old, noo.get(), sizeof(int) * n, cudaMemcpyDeviceToHost), "d2h");
        if (faces_out)
            cuda_ok(cudaMemcpy(faces_out, fo.get(), sizeof(int) * 3 * nf, cudaMemcpyDeviceToHost),
                    "d2h");
        if (xyz_out)
            cuda_ok(cudaMemcpy(xyz_out, xo.get(), sizeof(double) * 3 * n, cudaMemcpyDeviceToHost),
                    "d2h");
    });
}

int geodist_ptp(geodist_mesh_t mesh, const int32_t* sources, int32_t m,
                const geodist_ptp_config* config, double* distances, int32_t* labels,
                geodist_ptp_stats* stats, geodist_band_row* trace, int32_t trace_cap,
                int32_t* last_change, geodist_observer_fn observer, void* observer_user) {
    return guarded([&] {
        auto* mh = M(mesh);
        std::lock_guard<std::mutex> lock(mh->mu);
        checked_sources(sources, m, mh->n);  // compute_toplesets runs first (bindings.cpp:143)
        check_config(config);
        cuda_ok(cudaSetDevice(mh->device), "cudaSetDevice");
        Solve q;
        q.sources = sources;
        q.m = m;
        q.cfg = config;
        q.distances = distances;
        q.labels = config->with_labels ? labels : nullptr;
        q.stats = stats;
        q.trace = trace;
        q.trace_cap = trace_cap;
        q.last_change = last_change;
        q.observer = observer;
        q.observer_user = observer_user;
        run_solve(mh, q);
    });
}

int geodist_ptp_ordered(geodist_mesh_t mesh, const int32_t* sources, int32_t m,
                        const int32_t* sorted, int32_t reachable, const int32_t* limits,
                        int32_t rho, const int32_t* position, const geodist_ptp_config* config,
                        double* distances, int32_t* labels, geodist_ptp_stats* stats,
                        geodist_band_row* trace, int32_t trace_cap, int32_t* last_change,
                        geodist_observer_fn observer, void* observer_user) {
    return guarded([&] {
        auto* mh = M(mesh);
        std::lock_guard<std::mutex> lock(mh->mu);
        // ptp_run validation (ptp.cpp:155-167)
        if (m <= 0 || !sources) throw std::invalid_argument("ptp_run: empty source set");
        check_config(config);
        if (!limits || rho < 1 || limits[1] != m)
            throw std::invalid_argument("ptp_run: ordering does not match the source set");
        if (!position || reachable < 0 || reachable > mh->n || limits[rho] != reachable)
            throw std::invalid_argument("ptp_run: ordering built for a different mesh");
        // the kernel indexes positions and packed records through limits: it must be a
        // non-decreasing sequence inside [0, reachable]
        for (int r = 0; r < rho; ++r)
            if (limits[r] < 0 || limits[r] > limits[r + 1])
                throw std::invalid_argument("ptp_run: ordering built for a different mesh");
        for (int q = 0; q < m; ++q) {
            const int s = sources[q];
            if (s < 0 || s >= mh->n || position[s] == -1 || position[s] >= limits[1])
                throw std::invalid_argument("ptp_run: ordering does not match the source set");
        }
        // a vertex at two positions would have two cells in the position-indexed layout
        std::vector<unsigned char> seen(static_cast<size_t>(mh->n), 0);
        for (int p = 0; p < reachable; ++p) {
            if (sorted[p] < 0 || sorted[p] >= mh->n || seen[sorted[p]]++)
                throw std::invalid_argument("ptp_run: ordering built for a different mesh");
        }
        cuda_ok(cudaSetDevice(mh->device), "cudaSetDevice");
        Solve q;
        q.sources = sources;
        q.m = m;
        q.cfg = config;
        q.distances = distances;
        q.labels = config->with_labels ? labels : nullptr;
        q.stats = stats;
        q.trace = trace;
        q.trace_cap = trace_cap;
        q.last_change = last_change;
        q.observer = observer;
        q.observer_user = observer_user;
        q.ordered = true;
        q.sorted = sorted;
        q.reachable = reachable;
        q.limits = limits;
        q.rho = rho;
        run_solve(mh, q);
    });
}

int geodist_voronoi(geodist_mesh_t mesh, const int32_t* samples, int32_t m,
                    const geodist_ptp_config* config, int32_t* labels) {
    return guarded([&] {
        if (m <= 0 || !samples) throw std::invalid_argument("voronoi: empty sample set");
        geodist_ptp_config c = *config;
        c.with_labels = 1;
        c.record_trace = 0;
        const int rc = geodist_ptp(mesh, samples, m, &c, nullptr, labels, nullptr, nullptr, 0,
                                   nullptr, nullptr, nullptr);
        if (rc != GEODIST_OK) throw Fail(rc, g_err);
    });
}

int geodist_fps(geodist_mesh_t mesh, int32_t count, int32_t seed, const geodist_ptp_config* config,
                int32_t* samples, int32_t* labels, double* radius, geodist_fps_row* history) {
    return guarded([&] {
        auto* mh = M(mesh);
        std::lock_guard<std::mutex> lock(mh->mu);
        const int n = mh->n;
        if (count < 1 || count > n)
            throw std::invalid_argument("fps: sample count must be in [1, " + std::to_string(n) +
                                        "]");
        if (seed < 0 || seed >= n) throw std::invalid_argument("fps: seed vertex out of range");
        check_config(config);
        cuda_ok(cudaSetDevice(mh->device), "cudaSetDevice");
        const int prec = config->precision;
        check_label_range(prec, count);  // the last round labels all count samples
        mh->ensure_prec(prec);
    fps_retry:
        int maxb = INT_MAX;
        for (int md = 0; md < 3; ++md)
            maxb = std::min({maxb, run_max_blocks(prec, true, mh->device, md),
                             run_max_blocks(prec, false, mh->device, md)});
        mh->ws.ensure(1, n, maxb);
        Workspace& ws = mh->ws;
        cudaStream_t st = mh->stream;
        std::unique_ptr<void, DFree> smp(dalloc<int>(count)), lab(dalloc<int>(n)),
            hist(dalloc<QueryStats>(count));
        int* d_samples = static_cast<int*>(smp.get());
        cuda_ok(cudaMemcpyAsync(d_samples, &seed, sizeof(int), cudaMemcpyHostToDevice, st), "h2d");
        RunArgs a{};
        a.mesh.cptr = mh->cptr;
        a.mesh.ring = mh->prec[prec].ring;
        a.mesh.ringL = mh->prec[prec].ringL;
        a.mesh.quad = mh->prec[prec].quad;
        a.mesh.ering = mh->prec[prec].ering;
        a.mesh.eL = mh->prec[prec].eL;
        a.mesh.equad = mh->prec[prec].equad;
        a.mesh.n = n;
        ws.fill(a);
        ws.persist(st, mh->device);
        a.stride = n;
        a.groups = 1;
        a.blocks_per_group = maxb;
        a.src = d_samples;
        a.nq = 1;
        a.eps = config->epsilon;
        a.fused_bfs = 1;
        a.phase_init = 1;
        a.max_iters = 0;
        a.fps_mode = 1;
        a.fps_samples = d_samples;
        a.out_dist = nullptr;
        cuda_ok(cudaEventRecord(mh->ev0, st), "event");
        for (int s = 1; s <= count; ++s) {
            a.src_count = s;
            a.fps_final = s == count;
            a.out_labels = s == count ? static_cast<int*>(lab.get()) : nullptr;
            a.qstats = static_cast<QueryStats*>(hist.get()) + (s - 1);
            // no host round trip between rounds: a fixed launch sequence per round,
            // narrow-only -> wide-only -> narrow-only -> combined, each resuming the
            // field where the previous one handed it over (a launch whose field is
            // complete returns at once)
            for (int x = 0; x < 4; ++x) {
                a.phase_init = x == 0 ? 1 : 0;
                const int md = x == 3 ? 0 : (x & 1) ? 2 : 1;
                cuda_ok(launch_run(prec, s > 1, a, st, md), "fps round launch");
            }
            a.phase_init = 1;
        }
        cuda_ok(cudaEventRecord(mh->ev1, st), "event");
        cuda_ok(cudaStreamSynchronize(st), "fps");
        GroupCtl hctl{};
        cuda_ok(cudaMemcpy(&hctl, ws.ctl, sizeof(GroupCtl), cudaMemcpyDeviceToHost), "d2h");
        std::vector<int> hs(count);
        std::vector<QueryStats> hh(count);
        cuda_ok(cudaMemcpy(hs.data(), d_samples, sizeof(int) * count, cudaMemcpyDeviceToHost), "d2h");
        cuda_ok(cudaMemcpy(hh.data(), hist.get(), sizeof(QueryStats) * count,
                           cudaMemcpyDeviceToHost), "d2h");
        if (std::any_of(hh.begin(), hh.end(), [](const QueryStats& x) { return x.pad >= 2; })) {
            ws.grow_claims();  // claim-list overflow: redo the sampling with full-size lists
            goto fps_retry;
        }
        for (int s = 1; s < count; ++s)
            for (int t = 0; t < s; ++t)
                if (hs[s] == hs[t])
                    throw std::invalid_argument("compute_toplesets: duplicate source index " +
                                                std::to_string(hs[s]));
        if (samples) std::copy(hs.begin(), hs.end(), samples);
        if (labels)
            cuda_ok(cudaMemcpy(labels, lab.get(), sizeof(int) * n, cudaMemcpyDeviceToHost), "d2h");
        if (radius) *radius = hh[count - 1].radius;
        if (history)
            for (int s = 0; s < count; ++s) {
                history[s].sources = s + 1;
                history[s].rho = hh[s].rho;
                history[s].relax_calls = hh[s].relax;
                history[s].radius = hh[s].radius;
                history[s].picked = s + 1 < count ? hs[s + 1] : -1;
                history[s].iterations = hh[s].iterations;
            }
    });
}

int geodist_batch_device(geodist_mesh_t mesh, const int32_t* sources, const int32_t* offsets,
                         int32_t nq, const geodist_ptp_config* config, void* out_dist,
                         int32_t* out_labels, geodist_ptp_stats* out_stats, int32_t groups,
                         void* stream) {
    if (groups <= 0 && nq >= 3 && mesh && config && sources && offsets && out_dist) {
        // Automatic grouping: query 0 runs on the whole GPU; its mean band per CTA
        // chooses the number of concurrent fields.  Narrow bands are latency-bound per
        // iteration (16 groups: 2.1x the single-field throughput on the icosphere-8);
        // wide ones gain less but still gain (the 1000^2 torus: 4 groups, 1.2x; the
        // grid barrier is amortised over more work per CTA).  scripts/batch_probe.py.
        geodist_ptp_stats s0{};
        int rc = geodist_batch_device(mesh, sources, offsets, 1, config, out_dist, out_labels,
                                      &s0, 1, stream);
        if (rc != GEODIST_OK) return rc;
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, M(mesh)->device);
        const double band = s0.iterations > 0 ? double(s0.vertex_updates) / s0.iterations : 0.0;
        const double per_cta = band / std::max(1, sms);
        const int g = per_cta < 600 ? 16 : per_cta < 1200 ? 8 : 4;
        if (std::getenv("GEODIST_DEBUG_GROUPS"))
            std::fprintf(stderr, "batch auto-grouping: band per CTA %.0f -> %d groups\n", per_cta, g);
        std::vector<int32_t> off(nq);
        for (int q = 1; q <= nq - 1; ++q) off[q - 1] = offsets[q] - offsets[1];
        off[nq - 1] = offsets[nq] - offsets[1];
        const size_t n = M(mesh)->n;
        const size_t esz = config->precision == GEODIST_DOUBLE ? 8 : 4;
        std::vector<geodist_ptp_stats> rest(nq - 1);
        rc = geodist_batch_device(mesh, sources + offsets[1], off.data(), nq - 1, config,
                                  static_cast<char*>(out_dist) + n * esz,
                                  out_labels ? out_labels + n : nullptr, rest.data(), g, stream);
        if (rc != GEODIST_OK) return rc;
        if (out_stats) {
            const double total = s0.wall_seconds + rest[0].wall_seconds;
            out_stats[0] = s0;
            for (int q = 1; q < nq; ++q) out_stats[q] = rest[q - 1];
            for (int q = 0; q < nq; ++q) out_stats[q].wall_seconds = out_stats[q].total_seconds = total;
        }
        return GEODIST_OK;
    }
    return guarded([&] {
        auto* mh = M(mesh);
        std::lock_guard<std::mutex> lock(mh->mu);
        check_config(config);
        if (nq < 0 || (nq > 0 && (!sources || !offsets)))
            throw std::invalid_argument("batch: invalid query arrays");
        if (nq == 0) return;
        bool multi = false;
        for (int q = 0; q < nq; ++q) {
            checked_sources(sources + offsets[q], offsets[q + 1] - offsets[q], mh->n);
            multi = multi || offsets[q + 1] - offsets[q] > 1;
            check_label_range(config->precision, offsets[q + 1] - offsets[q]);
        }
        cuda_ok(cudaSetDevice(mh->device), "cudaSetDevice");
        const int prec = config->precision;
        mh->ensure_prec(prec);
        const int n = mh->n;
    batch_retry:
        int maxb = INT_MAX;
        for (int md = 0; md < 3; ++md)
            maxb = std::min(maxb, run_max_blocks(prec, multi, mh->device, md));
        int g = groups > 0 ? groups : std::min(nq, 4);
        g = std::max(1, std::min({g, nq, maxb}));
        const int bpg = maxb / g;
        mh->ws.ensure(g, n, maxb);
        Workspace& ws = mh->ws;
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : mh->stream;
        std::unique_ptr<void, DFree> srcb(dalloc<int>(offsets[nq])), offb(dalloc<int>(nq + 1)),
            qs(dalloc<QueryStats>(nq));
        cuda_ok(cudaMemcpyAsync(srcb.get(), sources, sizeof(int) * offsets[nq],
                                cudaMemcpyHostToDevice, st), "h2d");
        cuda_ok(cudaMemcpyAsync(offb.get(), offsets, sizeof(int) * (nq + 1),
                                cudaMemcpyHostToDevice, st), "h2d");
        RunArgs a{};
        a.mesh.cptr = mh->cptr;
        a.mesh.ring = mh->prec[prec].ring;
        a.mesh.ringL = mh->prec[prec].ringL;
        a.mesh.quad = mh->prec[prec].quad;
        a.mesh.ering = mh->prec[prec].ering;
        a.mesh.eL = mh->prec[prec].eL;
        a.mesh.equad = mh->prec[prec].equad;
        a.mesh.n = n;
        ws.fill(a);
        ws.persist(st, mh->device);
        a.stride = n;
        a.groups = g;
        a.blocks_per_group = bpg;
        a.src = static_cast<int*>(srcb.get());
        a.src_off = static_cast<int*>(offb.get());
        a.nq = nq;
        a.eps = config->epsilon;
        a.fused_bfs = 1;
        a.phase_init = 1;
        a.max_iters = 0;
        a.out_dist = out_dist;
        a.out_double = prec == GEODIST_DOUBLE;
        a.out_labels = config->with_labels ? out_labels : nullptr;
        a.qstats = static_cast<QueryStats*>(qs.get());
        float ms_sync = -1.f;  // device time when the launches were timed one by one
        if (g == 1 && nq == 1) {
            // one field: narrow-only first, the other mode only if the field hands over
            // (host-read state; no launches that would return at once)
            ms_sync = 0.f;
            int md = 1;
            for (int launch = 0; launch < 64; ++launch) {
                a.phase_init = launch == 0 ? 1 : 0;
                cuda_ok(cudaEventRecord(mh->ev0, st), "event");
                cuda_ok(launch_run(prec, multi, a, st, launch >= 63 ? 0 : md), "batch launch");
                cuda_ok(cudaEventRecord(mh->ev1, st), "event");
                GroupCtl hc{};
                cuda_ok(cudaMemcpyAsync(&hc, ws.ctl, sizeof(GroupCtl), cudaMemcpyDeviceToHost, st),
                        "read state");
                cuda_ok(cudaStreamSynchronize(st), "batch");
                float ms1 = 0.f;
                cudaEventElapsedTime(&ms1, mh->ev0, mh->ev1);
                ms_sync += ms1;
                if (hc.done || hc.mode_exit == 0 || hc.err >= 2) break;
                md = hc.mode_exit;
            }
        }
        cuda_ok(cudaEventRecord(mh->ev0, st), "event");
        if (ms_sync >= 0.f) {
            // launched and timed above
        } else if (g == 1) {
            // one field at a time on the whole GPU (wide-band meshes): the narrow/wide
            // launch sequence per query, enqueued without host round trips
            const size_t esz = prec == GEODIST_DOUBLE ? 8 : 4;
            for (int q = 0; q < nq; ++q) {
                a.nq = 1;
                a.src_off = static_cast<int*>(offb.get()) + q;
                a.out_dist = static_cast<char*>(out_dist) + static_cast<size_t>(q) * n * esz;
                a.out_labels = config->with_labels && out_labels ? out_labels + static_cast<size_t>(q) * n
                                                                 : nullptr;
                a.qstats = static_cast<QueryStats*>(qs.get()) + q;
                for (int x = 0; x < 4; ++x) {
                    a.phase_init = x == 0 ? 1 : 0;
                    const int md = x == 3 ? 0 : (x & 1) ? 2 : 1;
                    cuda_ok(launch_run(prec, multi, a, st, md), "batch launch");
                }
            }
        } else {
            cuda_ok(launch_run(prec, multi, a, st, 0), "batch launch");
        }
        cuda_ok(cudaEventRecord(mh->ev1, st), "event");
        std::vector<QueryStats> hq(nq);
        cuda_ok(cudaMemcpyAsync(hq.data(), qs.get(), sizeof(QueryStats) * nq,
                                cudaMemcpyDeviceToHost, st), "d2h");
        cuda_ok(cudaStreamSynchronize(st), "batch");
        if (std::any_of(hq.begin(), hq.end(), [](const QueryStats& x) { return x.pad >= 2; })) {
            ws.grow_claims();  // claim-list overflow: redo the batch with full-size lists
            goto batch_retry;
        }
        float ms = 0.f;
        cudaEventElapsedTime(&ms, mh->ev0, mh->ev1);
        if (ms_sync >= 0.f) ms = ms_sync;
        if (out_stats)
            for (int q = 0; q < nq; ++q) {
                geodist_ptp_stats& o = out_stats[q];
                o.relax_calls = hq[q].relax;
                o.degenerate_calls = hq[q].degen;
                o.vertex_updates = hq[q].updates;
                o.iterations = hq[q].iterations;
                o.rho = hq[q].rho;
                o.unreached = hq[q].unreached;
                o.workers = config->workers > 0 ? config->workers : 1;
                o.wall_seconds = ms * 1e-3;
                o.total_seconds = ms * 1e-3;
            }
    });
}

int geodist_batch(geodist_mesh_t mesh, const int32_t* sources, const int32_t* offsets,
                  int32_t nq, const geodist_ptp_config* config, double* distances,
                  int32_t* labels, geodist_ptp_stats* stats, int32_t groups) {
    return guarded([&] {
        auto* mh = M(mesh);
        check_config(config);
        if (nq <= 0) return;
        cuda_ok(cudaSetDevice(mh->device), "cudaSetDevice");
        const size_t n = mh->n;
        const int chunk = std::max<int>(1, std::min<long long>(nq, (1LL << 30) / (8 * n + 1)));
        const size_t tsz = config->precision == GEODIST_DOUBLE ? 8 : 4;
        std::unique_ptr<void, DFree> dout(dalloc<char>(chunk * n * tsz));
        std::unique_ptr<void, DFree> dlab(labels && config->with_labels ? dalloc<int>(chunk * n)
                                                                         : nullptr);
        std::vector<float> fbuf;
        for (int q0 = 0; q0 < nq; q0 += chunk) {
            const int cnt = std::min(chunk, nq - q0);
            std::vector<int> off(cnt + 1);
            for (int q = 0; q <= cnt; ++q) off[q] = offsets[q0 + q] - offsets[q0];
            const int rc = geodist_batch_device(mesh, sources + offsets[q0], off.data(), cnt,
                                                config, dout.get(), static_cast<int*>(dlab.get()),
                                                stats ? stats + q0 : nullptr, groups, nullptr);
            if (rc != GEODIST_OK) throw Fail(rc, g_err);
            if (distances) {
                if (tsz == 8) {
                    cuda_ok(cudaMemcpy(distances + q0 * n, dout.get(), cnt * n * 8,
                                       cudaMemcpyDeviceToHost), "d2h");
                } else {
                    fbuf.resize(cnt * n);
                    cuda_ok(cudaMemcpy(fbuf.data(), dout.get(), cnt * n * 4,
                                       cudaMemcpyDeviceToHost), "d2h");
                    for (size_t x = 0; x < cnt * n; ++x) distances[q0 * n + x] = fbuf[x];
                }
            }
            if (labels && dlab)
                cuda_ok(cudaMemcpy(labels + q0 * n, dlab.get(), cnt * n * sizeof(int),
                                   cudaMemcpyDeviceToHost), "d2h");
        }
    });
}

int geodist_selftest_arith(int64_t n, uint64_t seed, int64_t* counts) {
    return guarded([&] {
        int dev = 0;
        cudaGetDevice(&dev);
        require_device(dev);
        std::unique_ptr<void, DFree> out(dalloc<unsigned long long>(8));
        cuda_ok(cudaMemset(out.get(), 0, 64), "memset");
        launch_arith_selftest(n, seed, static_cast<unsigned long long*>(out.get()), nullptr);
        cuda_ok(cudaGetLastError(), "arith_selftest_kernel");
        cuda_ok(cudaMemcpy(counts, out.get(), 64, cudaMemcpyDeviceToHost), "d2h");
    });
}

int geodist_planar_update(const double* x1, const double* x2, const double* t1, const double* t2,
                          int32_t count, int32_t precision, double* value, int32_t* side,
                          int32_t* degenerate) {
    return guarded([&] {
        if (count <= 0) return;
        int dev = 0;
        cudaGetDevice(&dev);
        require_device(dev);
        std::unique_ptr<void, DFree> a(dalloc<double>(3 * count)), b(dalloc<double>(3 * count)),
            c(dalloc<double>(count)), d(dalloc<double>(count)), v(dalloc<double>(count)),
            s(dalloc<int>(count)), g(dalloc<int>(count));
        cuda_ok(cudaMemcpy(a.get(), x1, 24 * count, cudaMemcpyHostToDevice), "h2d");
        cuda_ok(cudaMemcpy(b.get(), x2, 24 * count, cudaMemcpyHostToDevice), "h2d");
        cuda_ok(cudaMemcpy(c.get(), t1, 8 * count, cudaMemcpyHostToDevice), "h2d");
        cuda_ok(cudaMemcpy(d.get(), t2, 8 * count, cudaMemcpyHostToDevice), "h2d");
        launch_planar_test(precision, static_cast<double*>(a.get()), static_cast<double*>(b.get()),
                           static_cast<double*>(c.get()), static_cast<double*>(d.get()), count,
                           static_cast<double*>(v.get()), static_cast<int*>(s.get()),
                           static_cast<int*>(g.get()), nullptr);
        cuda_ok(cudaGetLastError(), "planar_test_kernel");
        cuda_ok(cudaMemcpy(value, v.get(), 8 * count, cudaMemcpyDeviceToHost), "d2h");
        cuda_ok(cudaMemcpy(side, s.get(), 4 * count, cudaMemcpyDeviceToHost), "d2h");
        cuda_ok(cudaMemcpy(degenerate, g.get(), 4 * count, cudaMemcpyDeviceToHost), "d2h");
    });
}

}  // extern "C"
