// B200 (sm_100a) kernels of the PTP geodesic solver.
//
//   pack_kernel<T>      one-time per mesh & precision: per-ring |x| and per-corner
//                       Gram inverse {q11,q12,q22,a} + degenerate flag, i.e. the
//                       geometry-only half of planar_update<T>
//                       (reference include/geodist/update_kernel.hpp:38-60)
//   ptp_run_kernel<T,L> persistent cooperative kernel; one group of CTAs per
//                       query.  Per query: reset, seed sources (ptp.cpp:61-73),
//                       then the band loop of run_impl<T> (ptp.cpp:79-132) with
//                         * the BFS of compute_toplesets (toplesets.cpp:37-55)
//                           fused in: level k+1 is discovered while level k is
//                           relaxed (one group barrier per iteration serves both)
//                         * relax_vertex (update_kernel.hpp:93-120): 8 lanes per
//                           vertex, one corner per lane, lexicographic
//                           (value, corner) shuffle-min = the strict '<' scan
//                         * the front max relative change (ptp.cpp:107) reduced
//                           into the barrier; retirement + freeze (ptp.cpp:114-131)
//                           decided identically by every CTA after the barrier
//                       then copy-out (ptp.cpp:139-147), optional FPS argmax
//                       (sampling.cpp:29-36).
//   planar_test_kernel  planar_update<T> on raw inputs (parity hook).
//
// All floating point goes through __f*_rn / __d*_rn intrinsics: IEEE rounding,
// no FMA contraction, the reference's left-to-right association -- the CPU
// reference build has no FMA, so results are bit-identical.
#include <climits>
#include <cstdio>

#include "ptp_common.cuh"
#include "ptp_launch.hpp"

namespace gdb {

// ---------------------------------------------------------------------------
// one-time geometry pack (per mesh, per precision)

// CSR tables: per-ring |x|, per-corner Gram inverse, degenerate flag in bit 31.
template <typename T>
__global__ void pack_kernel(const double* __restrict__ xyz, int n, const int* __restrict__ cptr,
                            const int* __restrict__ ring_in, int* __restrict__ ring_out,
                            T* __restrict__ ringL, void* __restrict__ quad) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    const int c0 = cptr[v], d = cptr[v + 1] - c0, r0 = c0 + v;
    if (d == 0) {
        ring_out[r0] = ring_in[r0];
        ringL[r0] = T(0);
        return;
    }
    const T px = to_t<T>(xyz[3 * (size_t)v]), py = to_t<T>(xyz[3 * (size_t)v + 1]),
            pz = to_t<T>(xyz[3 * (size_t)v + 2]);
    T x0 = 0, y0 = 0, z0 = 0, g0 = 0;  // ring entry e-1
    for (int e = 0; e <= d; ++e) {
        const int r = ring_in[r0 + e];
        const T x = sub(to_t<T>(xyz[3 * (size_t)r]), px);
        const T y = sub(to_t<T>(xyz[3 * (size_t)r + 1]), py);
        const T z = sub(to_t<T>(xyz[3 * (size_t)r + 2]), pz);
        const T g = dot3(x, y, z, x, y, z);
        ringL[r0 + e] = sq(g);  // norm(x) = sqrt(dot(x, x)) (vec3.hpp:31-34)
        ring_out[r0 + e] = r;
        if (e > 0) {
            const int c = e - 1;  // corner (ring[c], ring[c+1])
            const T g12 = dot3(x0, y0, z0, x, y, z);
            T q11, q12, q22, a;
            const bool degen = corner_geometry(g0, g, g12, q11, q12, q22, a);
            Quad<T>::store(quad, c0 + c, q11, q12, q22, quad_w<T>(a, degen));
            if (degen) ring_out[r0 + c] = ring_in[r0 + c] | INT_MIN;
        }
        x0 = x; y0 = y; z0 = z; g0 = g;
    }
}

// ELL-8 tables (kEllW ring entries per vertex, interleaved so that lane l of a
// 4-lane group reads entries l and l+4 with one vector load).  Vertices with
// more than kEllW-1 corners are marked overflow and use the CSR tables.
template <typename T>
__global__ void pack_ell_kernel(int n, const int* __restrict__ cptr,
                                const int* __restrict__ ring_f, const T* __restrict__ ringL,
                                const void* __restrict__ quad, int* __restrict__ ering,
                                T* __restrict__ eL, void* __restrict__ equad) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    const int c0 = cptr[v], d = cptr[v + 1] - c0, r0 = c0 + v;
    const size_t b = static_cast<size_t>(v) * kEllW;
    if (d > kEllW - 1) {
        for (int e = 0; e < kEllW; ++e) {
            ering[b + ell_slot(e)] = e == 0 ? (v | (kEllOverflow << kMetaShift)) : v;
            eL[b + ell_slot(e)] = T(0);
            Quad<T>::store(equad, static_cast<int>(b + ell_slot(e)), T(0), T(0), T(0), T(0));
        }
        return;
    }
    for (int e = 0; e < kEllW; ++e) {
        const bool has = d > 0 && e <= d;
        int val = has ? ring_f[r0 + e] : v;  // bit 31: corner e is degenerate
        if (e == 0) val = (val & (INT_MIN | kIdMask)) | (d << kMetaShift);
        ering[b + ell_slot(e)] = val;
        eL[b + ell_slot(e)] = has ? ringL[r0 + e] : T(0);
        Quad<T> q;
        if (e < d) {
            q.load(quad, c0 + e);
        } else {
            q.q11 = q.q12 = q.q22 = q.a = T(0);
        }
        Quad<T>::store(equad, static_cast<int>(b + ell_slot(e)), q.q11, q.q12, q.q22, q.a);
    }
}

// Relax one band vertex per 4-lane group (relax_vertex, update_kernel.hpp:93-120).
// All 32 lanes call this in lock-step; `act` predicates the group.  Lanes
// holding ring ids of a level-k vertex also claim unvisited neighbours for
// level k+1 (toplesets.cpp:44-52), issued right after the ring ids arrive.
template <typename T, bool LABELS>
__device__ __forceinline__ void relax_group(const MeshDev& M, bool act, int p, int kk,
                                            const int* queue, const T* dp, T* dc, const int* lp,
                                            int* lc, int fe, bool expand, int* level,
                                            int* queue_w, int* tail_ptr, T eps, int* last_change,
                                            T& my_max, long long& calls, long long& degs) {
    const T inf = Lim<T>::inf();
    const int gl = threadIdx.x & (kGroup - 1);
    const int g0 = (threadIdx.x & 31) & ~(kGroup - 1);  // group's lane 0 within the warp
    int v = 0;
    if (act) v = ldcg(queue + p);
    const size_t eb = static_cast<size_t>(v) * kEllW;
    // ELL fast path: entries gl and gl+4, corners gl and gl+4 (one vector load each)
    int2 rr = make_int2(0, 0);
    T La = T(0), Lb = T(0);
    Quad<T> qa, qb;
    T tv = inf;
    int lv = -1;
    if (act) {
        rr = __ldg(reinterpret_cast<const int2*>(M.ering) + (eb >> 1) + gl);
        Ell2<T>::load(M.eL, eb + 2 * gl, La, Lb);
        qa.load(M.equad, static_cast<int>(eb + 2 * gl));
        qb.load(M.equad, static_cast<int>(eb + 2 * gl + 1));
        tv = ldcg(dp + v);
        if (LABELS) lv = ldcg(lp + v);
    }
    const int meta = __shfl_sync(kFull, rr.x, g0);
    int d = act ? (meta >> kMetaShift) & 15 : 0;
    const bool ovf = d == kEllOverflow;
    const int ida = rr.x & kIdMask, idb = rr.y & kIdMask;
    const bool hasa = act && !ovf && d > 0 && gl <= d;
    const bool hasb = act && !ovf && d > 0 && gl + kGroup <= d;
    // BFS claims first: they depend on the ring ids only
    bool ca_claim = false, cb_claim = false;
    if (expand) {
        if (hasa) ca_claim = atomicCAS(level + ida, -1, kk + 1) == -1;
        if (hasb) cb_claim = atomicCAS(level + idb, -1, kk + 1) == -1;
    }
    T ta = inf, tb = inf;
    int la = -1, lb_ = -1;
    if (hasa) {
        ta = ldcg(dp + ida);
        if (LABELS) la = ldcg(lp + ida);
    }
    if (hasb) {
        tb = ldcg(dp + idb);
        if (LABELS) lb_ = ldcg(lp + idb);
    }
    T best = gl == 0 ? tv : inf;
    int bidx = gl == 0 ? -1 : INT_MAX;
    int blab = gl == 0 ? lv : -1;
    chunk_candidates<T, LABELS>(gl, 0, ovf ? 0 : d, rr.x, rr.y, La, Lb, ta, tb, la, lb_, qa, qb,
                                best, bidx, blab, degs);
    if (ca_claim) prefetch_ell<T>(M, ida);
    if (cb_claim) prefetch_ell<T>(M, idb);
    append_claims(ca_claim, ida, tail_ptr, queue_w);
    append_claims(cb_claim, idb, tail_ptr, queue_w);

    // overflow vertices (> 7 corners): CSR tables, 7 corners per chunk
    if (__any_sync(kFull, act && ovf)) {
        int c0 = 0;
        if (act && ovf) {
            c0 = __ldg(M.cptr + v);
            d = __ldg(M.cptr + v + 1) - c0;
        }
        const int r0 = c0 + v;
        int nch = act && ovf ? (d + kEllW - 2) / (kEllW - 1) : 0;
        nch = __reduce_max_sync(kFull, nch);
        const int* ring = M.ring;
        const T* ringL = static_cast<const T*>(M.ringL);
        for (int ch = 0; ch < nch; ++ch) {
            const int base = ch * (kEllW - 1);
            const int ea = base + gl, ebb = base + gl + kGroup;
            const bool ha = act && ovf && ea <= d, hb = act && ovf && ebb <= d;
            int xa = 0, xb = 0;
            T LA = T(0), LB = T(0), TA = inf, TB = inf;
            int lA = -1, lB = -1;
            Quad<T> QA, QB;
            QA.q11 = QA.q12 = QA.q22 = QA.a = T(0);
            QB = QA;
            if (ha) {
                xa = __ldg(ring + r0 + ea);
                LA = __ldg(ringL + r0 + ea);
                if (ea < d) QA.load(M.quad, c0 + ea);
            }
            if (hb) {
                xb = __ldg(ring + r0 + ebb);
                LB = __ldg(ringL + r0 + ebb);
                if (ebb < d) QB.load(M.quad, c0 + ebb);
            }
            const int ia = xa & INT_MAX, ib = xb & INT_MAX;
            bool cA = false, cB = false;
            if (expand) {
                if (ha) cA = atomicCAS(level + ia, -1, kk + 1) == -1;
                if (hb) cB = atomicCAS(level + ib, -1, kk + 1) == -1;
            }
            if (ha) {
                TA = ldcg(dp + ia);
                if (LABELS) lA = ldcg(lp + ia);
            }
            if (hb) {
                TB = ldcg(dp + ib);
                if (LABELS) lB = ldcg(lp + ib);
            }
            // corners base+gl and base+gl+4 of this chunk; cap at 7 corners per chunk
            const int dlim = act && ovf ? min(d, base + kEllW - 1) : 0;
            chunk_candidates<T, LABELS>(gl, base, dlim, xa, xb, LA, LB, TA, TB, lA, lB, QA, QB,
                                        best, bidx, blab, degs);
            append_claims(cA, ia, tail_ptr, queue_w);
            append_claims(cB, ib, tail_ptr, queue_w);
        }
    }

    // lexicographic (value, corner) min over the group == first strict-'<' winner
    for (int o = kGroup / 2; o > 0; o >>= 1) {
        const T ob = __shfl_xor_sync(kFull, best, o, kGroup);
        const int oi = __shfl_xor_sync(kFull, bidx, o, kGroup);
        int ol = -1;
        if (LABELS) ol = __shfl_xor_sync(kFull, blab, o, kGroup);
        if (ob < best || (ob == best && oi < bidx)) {
            best = ob;
            bidx = oi;
            if (LABELS) blab = ol;
        }
    }
    if (act && gl == 0) {
        dc[v] = best;
        if (LABELS) lc[v] = blab;
        calls += d;
        const T rc = rel_change(tv, best);
        if (p < fe && rc > my_max) my_max = rc;
        if (last_change != nullptr && rc >= eps) last_change[v] = kk;
    }
}

// Relax one band vertex per THREAD (wide bands): relax_vertex's sequential fan
// scan with strict '<' (update_kernel.hpp:93-120) -- 32 vertices advance per warp
// instruction instead of 8, no shuffles.  All lanes call it (claims are
// warp-aggregated); `act` predicates the lane.
template <typename T, bool LABELS>
__device__ __forceinline__ void relax_thread(const MeshDev& M, bool act, int p, int kk,
                                             const int* queue, const T* dp, T* dc,
                                             const int* lp, int* lc, int fe, bool expand,
                                             int* level, int* queue_w, int* tail_ptr, T eps,
                                             int* last_change, T& my_max, long long& calls,
                                             long long& degs) {
    const T inf = Lim<T>::inf();
    int v = 0, d = 0;
    int raw[kEllW];
    T L[kEllW];
#pragma unroll
    for (int e = 0; e < kEllW; ++e) {
        raw[e] = 0;
        L[e] = T(0);
    }
    if (act) {
        v = ldcg(queue + p);
        const int4* rp = reinterpret_cast<const int4*>(M.ering) + 2 * static_cast<size_t>(v);
        const int4 a = __ldg(rp), b = __ldg(rp + 1);
        raw[0] = a.x; raw[4] = a.y; raw[1] = a.z; raw[5] = a.w;
        raw[2] = b.x; raw[6] = b.y; raw[3] = b.z; raw[7] = b.w;
        RowL<T>::load(M.eL, v, L);
        d = (raw[0] >> kMetaShift) & 15;
    }
    const bool ovf = act && d == kEllOverflow;
    int id[kEllW];
    bool claim[kEllW];
#pragma unroll
    for (int e = 0; e < kEllW; ++e) {
        id[e] = raw[e] & kIdMask;
        claim[e] = false;
    }
    T tv = inf;
    int lv = -1;
    T best = inf;
    int blab = -1;
    if (act) {
        tv = ldcg(dp + v);
        if (LABELS) lv = ldcg(lp + v);
        best = tv;
        blab = lv;
    }
    if (act && !ovf && d > 0) {
        T t[kEllW];
        int l[kEllW];
#pragma unroll
        for (int e = 0; e < kEllW; ++e) {
            t[e] = inf;
            l[e] = -1;
            if (e <= d) {
                if (expand) claim[e] = atomicCAS(level + id[e], -1, kk + 1) == -1;
                t[e] = ldcg(dp + id[e]);
                if (LABELS) l[e] = ldcg(lp + id[e]);
            }
        }
        const size_t qb = static_cast<size_t>(v) * kEllW;
#pragma unroll
        for (int c = 0; c < kEllW - 1; ++c) {
            if (c < d) {
                Quad<T> q;
                q.load(M.equad, static_cast<int>(qb + ell_slot(c)));
                const bool mixed = LABELS && l[c] != l[c + 1] && t[c] != inf && t[c + 1] != inf;
                int side, deg;
                const T val = corner_eval<T>(t[c], t[c + 1], L[c], L[c + 1], q, raw[c] < 0, mixed,
                                             side, deg);
                degs += deg;
                if (val < best) {
                    best = val;
                    if (LABELS) blab = side == 0 ? l[c] : l[c + 1];
                }
            }
        }
    } else if (ovf) {
        // more than 7 corners: CSR tables, sequential fan walk
        const int c0 = __ldg(M.cptr + v);
        d = __ldg(M.cptr + v + 1) - c0;
        const int r0 = c0 + v;
        const T* ringL = static_cast<const T*>(M.ringL);
        int x0 = __ldg(M.ring + r0);
        int i0 = x0 & INT_MAX;
        T t0 = ldcg(dp + i0), L0 = __ldg(ringL + r0);
        int l0 = LABELS ? ldcg(lp + i0) : -1;
        if (expand && atomicCAS(level + i0, -1, kk + 1) == -1) {
            prefetch_ell<T>(M, i0);
            append_one(i0, tail_ptr, queue_w);
        }
        for (int c = 0; c < d; ++c) {
            const int x1 = __ldg(M.ring + r0 + c + 1);
            const int i1 = x1 & INT_MAX;
            const T t1 = ldcg(dp + i1), L1 = __ldg(ringL + r0 + c + 1);
            const int l1 = LABELS ? ldcg(lp + i1) : -1;
            if (expand && atomicCAS(level + i1, -1, kk + 1) == -1) {
                prefetch_ell<T>(M, i1);
                append_one(i1, tail_ptr, queue_w);
            }
            Quad<T> q;
            q.load(M.quad, c0 + c);
            const bool mixed = LABELS && l0 != l1 && t0 != inf && t1 != inf;
            int side, deg;
            const T val = corner_eval<T>(t0, t1, L0, L1, q, x0 < 0, mixed,
                                           side, deg);
            degs += deg;
            if (val < best) {
                best = val;
                if (LABELS) blab = side == 0 ? l0 : l1;
            }
            x0 = x1; i0 = i1; t0 = t1; L0 = L1; l0 = l1;
        }
    }
#pragma unroll
    for (int e = 0; e < kEllW; ++e)
        if (claim[e]) prefetch_ell<T>(M, id[e]);
    append_claims_multi(claim, id, tail_ptr, queue_w);
    if (act) {
        dc[v] = best;
        if (LABELS) lc[v] = blab;
        calls += d;
        const T rc = rel_change(tv, best);
        if (p < fe && rc > my_max) my_max = rc;
        if (last_change != nullptr && rc >= eps) last_change[v] = kk;
    }
}

template <typename T, bool LABELS>
__global__ void __launch_bounds__(kBlock, 1) ptp_run_kernel(RunArgs A) {
    __shared__ Bcast S;
    __shared__ T red_t[kBlock / 32];
    __shared__ long long red_l[kBlock / 32];
    __shared__ double red_v[kBlock / 32];
    __shared__ int red_i[kBlock / 32];

    const int tid = threadIdx.x;
    const int nb = A.blocks_per_group;
    const int g = blockIdx.x / nb;
    const int lb = blockIdx.x - g * nb;
    GroupCtl* ctl = A.ctl + g;
    const long long off = static_cast<long long>(g) * A.stride;
    T* dist[2] = {static_cast<T*>(A.dist0) + off, static_cast<T*>(A.dist1) + off};
    int* lab[2] = {nullptr, nullptr};
    if (LABELS) {
        lab[0] = A.lab0 + off;
        lab[1] = A.lab1 + off;
    }
    int* level = A.level + off;
    int* queue = A.queue + off;
    int* limits = A.limits + off;
    const MeshDev M = A.mesh;
    const int n = M.n;
    const T inf = Lim<T>::inf();
    const T eps = static_cast<T>(A.eps);
    unsigned epoch = 0;
    const int gthreads = nb * kBlock;
    const int gtid = lb * kBlock + tid;
    constexpr int kGroupsPerBlock = kBlock / kGroup;
    const int stride = nb * kGroupsPerBlock;
    const int first_task = lb + nb * (tid / kGroup);

    for (int q = g; q < A.nq; q += A.groups) {
        const int s0 = A.src_off ? A.src_off[q] : 0;
        const int m = A.src_off ? A.src_off[q + 1] - s0 : A.src_count;
        const int* src = A.src + s0;
        // thread-0 loop state (identical in every CTA of the group)
        int k = 0, i = 1, rho = INT_MAX, parity = 0, bfs_open = 0, done = 0;
        int tail = 0, limk = 0, bb = 0, fe = 0, frzb = 0, frze = 0;
        unsigned long long upd = 0;
        int pf = -1;
        // fills S for the iteration after `k` (thread 0)
        auto publish = [&] {
            S.done = done;
            if (done) return;
            const int kk = k + 1;
            const int j = bfs_open ? kk : min(kk, rho - 1);
            S.k = kk;
            S.i = i;
            S.j = j;
            S.bb = bb;
            S.fe = fe;
            S.be = (bfs_open || j + 1 == rho) ? tail : ldcg(limits + j + 1);
            S.expb = bfs_open ? limk : 0;
            S.expe = bfs_open ? tail : 0;
            S.frzb = frzb;
            S.frze = frze;
            S.parity = parity;
            pf = -1;
            if (i + 2 <= kk + 1 && (bfs_open || i + 2 <= rho))
                pf = (bfs_open && i + 2 == kk + 1) ? tail : ldcg(limits + i + 2);
            if (lb == 0) ctl->slot[(kk + 1) % 3] = 0ull;
        };

        if (A.phase_init) {
            // reset (ptp.cpp:61-68)
            for (int v = gtid; v < n; v += gthreads) {
                dist[0][v] = inf;
                dist[1][v] = inf;
                if (LABELS) {
                    lab[0][v] = -1;
                    lab[1][v] = -1;
                }
                if (A.fused_bfs) level[v] = -1;
                if (A.last_change) A.last_change[v] = 0;
            }
            if (gtid == 0) {
                ctl->relax = ctl->degen = ctl->updates = 0;
                ctl->slot[0] = ctl->slot[1] = ctl->slot[2] = 0ull;
                ctl->tail = m;
                ctl->err = 0;
            }
            group_barrier(&ctl->bar, epoch, nb, [] {});
            // seed sources: d = 0, label = index in caller order (ptp.cpp:69-73)
            for (int s = gtid; s < m; s += gthreads) {
                const int v = src[s];
                dist[0][v] = T(0);
                dist[1][v] = T(0);
                if (LABELS) {
                    lab[0][v] = s;
                    lab[1][v] = s;
                }
                if (A.fused_bfs) {
                    level[v] = 0;
                    queue[s] = v;
                }
            }
            if (A.fused_bfs && gtid == 0) {
                limits[0] = 0;
                limits[1] = m;
            }
            group_barrier(&ctl->bar, epoch, nb, [] {});
            if (A.fused_bfs) {
                // iteration 0: level 0 -> level 1 (ring walk only; sources are never relaxed)
                const int gl = tid & (kGroup - 1);
                for (int t = first_task;; t += stride) {
                    const bool act = t < m;
                    if (!__any_sync(kFull, act)) break;
                    int v = 0, c0 = 0, d = 0;
                    if (act) {
                        v = ldcg(queue + t);
                        c0 = __ldg(M.cptr + v);
                        d = __ldg(M.cptr + v + 1) - c0;
                    }
                    int nch = d > 0 ? (d + kGroup) / kGroup : 0;  // ring entries 0..d
                    nch = __reduce_max_sync(kFull, nch);
                    for (int ch = 0; ch < nch; ++ch) {
                        const int e = ch * kGroup + gl;
                        bool claim = false;
                        int id = 0;
                        if (act && d > 0 && e <= d) {
                            id = __ldg(M.ring + c0 + v + e) & INT_MAX;
                            claim = atomicCAS(level + id, -1, 1) == -1;
                        }
                        append_claims(claim, id, &ctl->tail, queue);
                    }
                }
            }
            group_barrier(&ctl->bar, epoch, nb, [&] {
                if (A.fused_bfs) {
                    const int t = ldcg(&ctl->tail);
                    tail = t;
                    limk = m;
                    bb = m;
                    fe = t;
                    if (t == m) {
                        bfs_open = 0;
                        rho = 1;
                    } else {
                        bfs_open = 1;
                        if (lb == 0) limits[2] = t;
                    }
                } else {
                    rho = A.given_rho;
                    bfs_open = 0;
                    tail = ldcg(limits + rho);
                    bb = ldcg(limits + 1);
                    fe = rho >= 2 ? ldcg(limits + 2) : tail;
                }
                done = !bfs_open && i > rho - 1;
                publish();
            });
        } else {
            if (tid == 0) {
                // resume a run stopped by max_iters
                k = ctl->k; i = ctl->i; rho = ctl->rho; parity = ctl->parity;
                bfs_open = ctl->bfs_open; done = ctl->done;
                tail = ctl->s_tail; limk = ctl->s_limk; bb = ctl->s_bb; fe = ctl->s_fe;
                frzb = ctl->s_frzb; frze = ctl->s_frze;
                publish();
            }
            __syncthreads();
        }

        T my_max = T(0);
        long long calls = 0, degs = 0;
        int iters = 0;
        for (;;) {
            // S was filled by thread 0 inside the previous barrier
            if (S.done || (A.max_iters > 0 && iters >= A.max_iters)) break;
            const int kk = S.k;
            const bool dbg = A.dbg != nullptr && tid == 0 && iters < A.dbg_iters;
            unsigned long long* dslot =
                dbg ? A.dbg + kDbgSlots * (static_cast<size_t>(iters) * gridDim.x + blockIdx.x) : nullptr;
            if (dbg) dslot[0] = gtimer();
            const int prv = S.parity, cur = prv ^ 1;
            const T* dp = dist[prv];
            T* dcur = dist[cur];
            const int* lp = LABELS ? lab[prv] : nullptr;
            int* lc = LABELS ? lab[cur] : nullptr;
            const int bb_ = S.bb, ntask = S.be - S.bb, fe_ = S.fe;
            const int expb = S.expb, expe = S.expe;
            const int frzb_ = S.frzb, frze_ = S.frze;
            // deferred freeze of the level retired last iteration (ptp.cpp:121-130)
            for (int p = frzb_ + gtid; p < frze_; p += gthreads) {
                const int v = ldcg(queue + p);
                dcur[v] = ldcg(dp + v);
                if (LABELS) lc[v] = ldcg(lp + v);
            }
            // relax the band [bb, be)   (ptp.cpp:96-110): 4 lanes per vertex while the
            // band fits the CTA groups (latency), one thread per vertex beyond (throughput)
            my_max = T(0);
            if (ntask <= A.wide_factor * stride) {
                for (int t = first_task;; t += stride) {
                    const bool act = t < ntask;
                    if (!__any_sync(kFull, act)) break;
                    const int p = bb_ + t;
                    relax_group<T, LABELS>(M, act, p, kk, queue, dp, dcur, lp, lc, fe_,
                                           p >= expb && p < expe, level, queue, &ctl->tail, eps,
                                           A.last_change, my_max, calls, degs);
                }
            } else {
                for (int t = gtid;; t += gthreads) {
                    const bool act = t < ntask;
                    if (!__any_sync(kFull, act)) break;
                    const int p = bb_ + t;
                    relax_thread<T, LABELS>(M, act, p, kk, queue, dp, dcur, lp, lc, fe_,
                                            p >= expb && p < expe, level, queue, &ctl->tail, eps,
                                            A.last_change, my_max, calls, degs);
                }
            }
            const T bmax = block_max(my_max, red_t);
            if (dbg) dslot[1] = gtimer();
            if (tid == 0 && bmax > T(0)) atomicMax(&ctl->slot[kk % 3], Lim<T>::bits(bmax));
            group_barrier(&ctl->bar, epoch, nb, [&] {
                if (dbg) dslot[2] = gtimer();
                const T mr = Lim<T>::from_bits(__ldcg(&ctl->slot[kk % 3]));
                const int nt = bfs_open ? ldcg(&ctl->tail) : tail;
                const bool conv = mr < eps;  // ptp.cpp:114
                const int ub = bb, ue = S.be;
                upd += static_cast<unsigned long long>(ue - ub);
                if (lb == 0 && A.trace != nullptr) {
                    const int row = kk - A.trace_k0;
                    if (row >= 0 && row < A.trace_cap) {
                        TraceRow r;
                        r.k = kk; r.i = i; r.j = S.j; r.conv = conv ? 1 : 0;
                        r.updated = ue - ub;
                        r.max_rel = static_cast<double>(mr);
                        A.trace[row] = r;
                    }
                }
                if (bfs_open) {
                    if (nt == tail) {
                        bfs_open = 0;
                        rho = kk + 1;
                    } else {
                        if (lb == 0) limits[kk + 2] = nt;
                        limk = tail;
                    }
                }
                if (conv) {
                    frzb = bb;
                    frze = fe;
                    bb = fe;
                    fe = (i + 2 <= kk + 1) ? pf : nt;
                    ++i;
                } else {
                    frzb = frze = 0;
                }
                tail = nt;
                parity ^= 1;
                k = kk;
                done = !bfs_open && i > rho - 1;
                publish();
            });
            ++iters;
        }

        // per-query statistics
        const long long bc = block_sum(calls, red_l);
        const long long bd = block_sum(degs, red_l);
        if (tid == 0) {
            if (bc) atomicAdd(&ctl->relax, static_cast<unsigned long long>(bc));
            if (bd) atomicAdd(&ctl->degen, static_cast<unsigned long long>(bd));
            if (lb == 0) {
                ctl->k = k; ctl->i = i; ctl->rho = rho; ctl->parity = parity;
                ctl->bfs_open = bfs_open; ctl->done = done;
                ctl->s_tail = tail; ctl->s_limk = limk; ctl->s_bb = bb; ctl->s_fe = fe;
                ctl->s_frzb = frzb; ctl->s_frze = frze;
                ctl->updates += upd;
            }
            S.done = done;
            S.parity = parity;
        }
        __syncthreads();
        const int fin_done = S.done;
        const int fin = S.parity;  // buffer written last (ptp.cpp:142)
        if (!fin_done) continue;   // resumable launch ended mid-run

        // copy-out to original vertex order, widened (ptp.cpp:139-147)
        double vmax = -1.0;
        int vidx = INT_MAX;
        if (A.out_dist != nullptr || A.fps_mode || A.out_labels != nullptr) {
            const T* df = dist[fin];
            const int* lf = LABELS ? lab[fin] : nullptr;
            const long long qo = static_cast<long long>(q) * n;
            for (int v = gtid; v < n; v += gthreads) {
                const T x = ldcg(df + v);
                if (A.out_dist != nullptr) {
                    if (A.out_double)
                        static_cast<double*>(A.out_dist)[qo + v] = static_cast<double>(x);
                    else
                        static_cast<float*>(A.out_dist)[qo + v] = static_cast<float>(x);
                }
                if (A.out_labels != nullptr)
                    A.out_labels[qo + v] = LABELS ? ldcg(lf + v) : (x != inf ? 0 : -1);
                const double xd = static_cast<double>(x);
                if (xd > vmax || (xd == vmax && v < vidx)) {
                    vmax = xd;
                    vidx = v;
                }
            }
        }
        if (A.fps_mode) {
            // block argmax: max value, lowest index (sampling.cpp:29-36)
            for (int o = 16; o > 0; o >>= 1) {
                const double ov = __shfl_xor_sync(kFull, vmax, o);
                const int oi = __shfl_xor_sync(kFull, vidx, o);
                if (ov > vmax || (ov == vmax && oi < vidx)) { vmax = ov; vidx = oi; }
            }
            if ((tid & 31) == 0) { red_v[tid >> 5] = vmax; red_i[tid >> 5] = vidx; }
            __syncthreads();
            if (tid == 0) {
                for (int w = 1; w < kBlock / 32; ++w)
                    if (red_v[w] > vmax || (red_v[w] == vmax && red_i[w] < vidx)) {
                        vmax = red_v[w];
                        vidx = red_i[w];
                    }
                A.fps_scratch[2 * blockIdx.x] =
                    static_cast<unsigned long long>(__double_as_longlong(vmax));
                A.fps_scratch[2 * blockIdx.x + 1] = static_cast<unsigned long long>(vidx);
            }
        }
        group_barrier(&ctl->bar, epoch, nb, [&] {
            if (lb != 0) return;
            QueryStats st;
            st.relax = static_cast<long long>(__ldcg(&ctl->relax));
            st.degen = static_cast<long long>(__ldcg(&ctl->degen));
            st.updates = static_cast<long long>(ctl->updates);
            st.iterations = k;
            st.rho = rho;
            st.unreached = n - tail;
            st.done = 1;
            st.radius = 0.0;
            st.argmax = -1;
            st.pad = 0;
            if (A.fps_mode) {
                double bv = -1.0;
                int bi = INT_MAX;
                for (int b = g * nb; b < g * nb + nb; ++b) {
                    const double ov = __longlong_as_double(
                        static_cast<long long>(__ldcg(&A.fps_scratch[2 * b])));
                    const int oi = static_cast<int>(__ldcg(&A.fps_scratch[2 * b + 1]));
                    if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
                }
                st.radius = bv;
                st.argmax = bi;
                if (!A.fps_final) {
                    if (ldcg(level + bi) == 0) ctl->err = 1;  // would repeat a sample
                    A.fps_samples[A.src_count] = bi;
                }
            }
            A.qstats[q] = st;
        });
    }
}

// ===========================================================================
// v3 solver: claimer-first relaxation over BFS-ordered packed records.
//
// A CTA that claims vertices for level k+1 (during iteration k) appends their
// ids to its own global claim list (index from a shared-memory counter, no
// global atomic).  The per-CTA claim counts ride on the grid barrier together
// with the per-CTA max relative change; every CTA turns them into a prefix
// table, which maps the new level's BFS positions to (claimer, index).  At
// iteration k+1 the new level is relaxed round-robin like the rest of the band:
// a task of the new level looks its id up in the claimer's list, relaxes it from
// the id-indexed ELL tables and writes the vertex's packed record (id, ring,
// |x|, Gram quads) at its BFS position; older band levels are relaxed straight
// from those packed records -- the reference's reorder_for_bands layout
// (toplesets.cpp:60-89), built incrementally while the band advances.  A task
// costs two dependent L2 round trips (record, then neighbour distances), three
// for the newest level (claim-list lookup first).
// ===========================================================================

struct Bcast3 {
    int k, i, j, bb, oe, be, fe, frzb, frze, parity, done, cur, expand;
};

__device__ __forceinline__ void ld_acquire_v2(const unsigned long long* p, unsigned long long& a,
                                              unsigned long long& b) {
    asm volatile("ld.acquire.gpu.global.v2.u64 {%0, %1}, [%2];"
                 : "=l"(a), "=l"(b)
                 : "l"(p)
                 : "memory");
}

// Warp-aggregated append of claims (entries a and b of every lane) to the
// CTA's own global claim list for the next level (index from a shared-memory
// counter: no global atomic).
__device__ __forceinline__ void list_claims(bool ca, int ia, bool cb, int ib, int* list,
                                            int* cnt, int cap, int* err) {
    const unsigned ba = __ballot_sync(kFull, ca), bbal = __ballot_sync(kFull, cb);
    if ((ba | bbal) == 0u) return;
    const int l32 = threadIdx.x & 31;
    const int leader = __ffs(ba | bbal) - 1;
    int base = 0;
    if (l32 == leader) base = atomicAdd(cnt, __popc(ba) + __popc(bbal));
    base = __shfl_sync(kFull, base, leader);
    const unsigned lt = (1u << l32) - 1u;
    if (ca) {
        const int at = base + __popc(ba & lt);
        if (at < cap) list[at] = ia; else *err = 2;
    }
    if (cb) {
        const int at = base + __popc(ba) + __popc(bbal & lt);
        if (at < cap) list[at] = ib; else *err = 2;
    }
}

template <typename T, bool LABELS>
__device__ __forceinline__ void relax3(const MeshDev& M, const RunArgs& A, long long off8,
                                       bool act, bool is_new, int v_new, int p, int kk,
                                       int* pv, const T* dp, T* dc, const int* lp, int* lc,
                                       int fe, bool expand, int* level, int* nlist, int* ncnt,
                                       int* err, T eps, T& my_max, long long& calls,
                                       long long& degs, unsigned long long* tdbg) {
    const T inf = Lim<T>::inf();
    const int gl = threadIdx.x & (kGroup - 1);
    const int g0 = (threadIdx.x & 31) & ~(kGroup - 1);
    if (tdbg) tdbg[3] = cyc();
    int* pring = A.pring + off8;
    T* pL = static_cast<T*>(A.pL) + off8;
    char* pquad = static_cast<char*>(A.pquad) + off8 * sizeof(Quad<T>);
    const size_t pb = static_cast<size_t>(p) * kEllW;
    int v = 0;
    int2 rr = make_int2(0, 0);
    T La = T(0), Lb = T(0);
    Quad<T> qa, qb;
    qa.q11 = qa.q12 = qa.q22 = qa.a = T(0);
    qb = qa;
    if (act) {
        if (is_new) {
            v = v_new;
            const size_t eb = static_cast<size_t>(v) * kEllW;
            rr = __ldg(reinterpret_cast<const int2*>(M.ering) + (eb >> 1) + gl);
            Ell2<T>::load(M.eL, eb + 2 * gl, La, Lb);
            qa.load(M.equad, static_cast<int>(eb + 2 * gl));
            qb.load(M.equad, static_cast<int>(eb + 2 * gl + 1));
            // commit the packed record at the vertex's BFS position
            if (gl == 0) pv[p] = v;
            reinterpret_cast<int2*>(pring)[(pb >> 1) + gl] = rr;
            Ell2<T>::store(pL, pb + 2 * gl, La, Lb);
            qa.store_at(pquad, pb + 2 * gl);
            qb.store_at(pquad, pb + 2 * gl + 1);
        } else {
            v = ldcg(pv + p);
            rr = __ldcg(reinterpret_cast<const int2*>(pring) + (pb >> 1) + gl);
            Ell2<T>::load_cg(pL, pb + 2 * gl, La, Lb);
            qa.load_cg(pquad, pb + 2 * gl);
            qb.load_cg(pquad, pb + 2 * gl + 1);
        }
    }
    if (tdbg) tdbg[4] = gtimer_after(rr.x + v);
    const int meta = __shfl_sync(kFull, rr.x, g0);
    int d = act ? (meta >> kMetaShift) & 15 : 0;
    const bool ovf = d == kEllOverflow;
    const int ida = rr.x & kIdMask, idb = rr.y & kIdMask;
    const bool hasa = act && !ovf && d > 0 && gl <= d;
    const bool hasb = act && !ovf && d > 0 && gl + kGroup <= d;
    const bool exp = expand && is_new;
    bool ca_claim = false, cb_claim = false;
    if (exp) {
        if (hasa) ca_claim = atomicCAS(level + ida, -1, kk + 1) == -1;
        if (hasb) cb_claim = atomicCAS(level + idb, -1, kk + 1) == -1;
    }
    T tv = inf;
    int lv = -1;
    if (act) {
        tv = ldcg(dp + v);
        if (LABELS) lv = ldcg(lp + v);
    }
    T ta = inf, tb = inf;
    int la = -1, lb_ = -1;
    if (hasa) {
        ta = ldcg(dp + ida);
        if (LABELS) la = ldcg(lp + ida);
    }
    if (hasb) {
        tb = ldcg(dp + idb);
        if (LABELS) lb_ = ldcg(lp + idb);
    }
    if (tdbg) tdbg[5] = gtimer_after(__float_as_int(static_cast<float>(ta + tb + tv)));
    T best = gl == 0 ? tv : inf;
    int bidx = gl == 0 ? -1 : INT_MAX;
    int blab = gl == 0 ? lv : -1;
    chunk_candidates<T, LABELS>(gl, 0, ovf ? 0 : d, rr.x, rr.y, La, Lb, ta, tb, la, lb_, qa, qb,
                                best, bidx, blab, degs);
    if (tdbg) tdbg[6] = gtimer_after(__float_as_int(static_cast<float>(best)) + ca_claim + cb_claim);
    if (ca_claim) prefetch_ell<T>(M, ida);
    if (cb_claim) prefetch_ell<T>(M, idb);
    list_claims(ca_claim, ida, cb_claim, idb, nlist, ncnt, A.claim_cap, err);

    // overflow vertices (> 7 corners): CSR tables, 7 corners per chunk
    if (__any_sync(kFull, act && ovf)) {
        int c0 = 0;
        if (act && ovf) {
            c0 = __ldg(M.cptr + v);
            d = __ldg(M.cptr + v + 1) - c0;
        }
        const int r0 = c0 + v;
        int nch = act && ovf ? (d + kEllW - 2) / (kEllW - 1) : 0;
        nch = __reduce_max_sync(kFull, nch);
        const int* ring = M.ring;
        const T* ringL = static_cast<const T*>(M.ringL);
        for (int ch = 0; ch < nch; ++ch) {
            const int base = ch * (kEllW - 1);
            const int ea = base + gl, ebb = base + gl + kGroup;
            const bool ha = act && ovf && ea <= d, hb = act && ovf && ebb <= d;
            int xa = 0, xb = 0;
            T LA = T(0), LB = T(0), TA = inf, TB = inf;
            int lA = -1, lB = -1;
            Quad<T> QA, QB;
            QA.q11 = QA.q12 = QA.q22 = QA.a = T(0);
            QB = QA;
            if (ha) {
                xa = __ldg(ring + r0 + ea);
                LA = __ldg(ringL + r0 + ea);
                if (ea < d) QA.load(M.quad, c0 + ea);
            }
            if (hb) {
                xb = __ldg(ring + r0 + ebb);
                LB = __ldg(ringL + r0 + ebb);
                if (ebb < d) QB.load(M.quad, c0 + ebb);
            }
            const int ia = xa & INT_MAX, ib = xb & INT_MAX;
            bool cA = false, cB = false;
            if (exp) {
                if (ha) cA = atomicCAS(level + ia, -1, kk + 1) == -1;
                if (hb) cB = atomicCAS(level + ib, -1, kk + 1) == -1;
            }
            if (ha) {
                TA = ldcg(dp + ia);
                if (LABELS) lA = ldcg(lp + ia);
            }
            if (hb) {
                TB = ldcg(dp + ib);
                if (LABELS) lB = ldcg(lp + ib);
            }
            const int dlim = act && ovf ? min(d, base + kEllW - 1) : 0;
            chunk_candidates<T, LABELS>(gl, base, dlim, xa, xb, LA, LB, TA, TB, lA, lB, QA, QB,
                                        best, bidx, blab, degs);
            list_claims(cA, ia, cB, ib, nlist, ncnt, A.claim_cap, err);
        }
    }

    for (int o = kGroup / 2; o > 0; o >>= 1) {
        const T ob = __shfl_xor_sync(kFull, best, o, kGroup);
        const int oi = __shfl_xor_sync(kFull, bidx, o, kGroup);
        int ol = -1;
        if (LABELS) ol = __shfl_xor_sync(kFull, blab, o, kGroup);
        if (ob < best || (ob == best && oi < bidx)) {
            best = ob;
            bidx = oi;
            if (LABELS) blab = ol;
        }
    }
    if (act && gl == 0) {
        dc[v] = best;
        if (LABELS) lc[v] = blab;
        calls += d;
        const T rc = rel_change(tv, best);
        if (p < fe && rc > my_max) my_max = rc;
        if (A.last_change != nullptr && rc >= eps) A.last_change[v] = kk;
    }
}

template <typename T, bool LABELS>
__global__ void __launch_bounds__(kBlock, 1) ptp_run3_kernel(RunArgs A) {
    __shared__ Bcast3 S;
    __shared__ int s_pref[kMaxGroupBlocks + 1];  // prefix of last iteration's claim counts
    __shared__ T red_t[kBlock / 32];
    __shared__ long long red_l[kBlock / 32];
    __shared__ double red_v[kBlock / 32];
    __shared__ int red_i[kBlock / 32];
    __shared__ int s_ncnt, s_err;

    const int tid = threadIdx.x;
    const int nb = A.blocks_per_group;
    const int g = blockIdx.x / nb;
    const int lb = blockIdx.x - g * nb;
    GroupCtl* ctl = A.ctl + g;
    const long long off = static_cast<long long>(g) * A.stride;
    const long long off8 = off * kEllW;
    T* dist[2] = {static_cast<T*>(A.dist0) + off, static_cast<T*>(A.dist1) + off};
    int* lab[2] = {nullptr, nullptr};
    if (LABELS) {
        lab[0] = A.lab0 + off;
        lab[1] = A.lab1 + off;
    }
    int* level = A.level + off;
    int* pv = A.queue + off;
    int* limits = A.limits + off;
    // this CTA's claim lists (parity 0/1) and the base of all lists of the group
    int* lists[2] = {A.blists + (static_cast<size_t>(0) * gridDim.x + blockIdx.x) * A.claim_cap,
                     A.blists + (static_cast<size_t>(1) * gridDim.x + blockIdx.x) * A.claim_cap};
    auto claim_list = [&](int par, int b) {
        return A.blists + (static_cast<size_t>(par) * gridDim.x + g * nb + b) * A.claim_cap;
    };
    const MeshDev M = A.mesh;
    const int n = M.n;
    const T inf = Lim<T>::inf();
    const T eps = static_cast<T>(A.eps);
    unsigned epoch = 0;
    const int gthreads = nb * kBlock;
    const int gtid = lb * kBlock + tid;
    constexpr int kGroupsPerBlock = kBlock / kGroup;
    BlkSlot* slots = reinterpret_cast<BlkSlot*>(A.blk_slot);  // [2][gridDim.x]

    // grid barrier whose payload (per-CTA max and claim count) is reduced by warp 0
    unsigned long long* bdbg = nullptr;  // barrier3 phase timers (debug)
    auto barrier3 = [&](int par, unsigned long long mybits, int mycnt, auto&& post) {
        if (tid == 0) {
            BlkSlot sl;
            sl.maxbits = mybits;
            sl.count = static_cast<unsigned long long>(mycnt);
            __stcg(reinterpret_cast<ulonglong2*>(&slots[par * gridDim.x + blockIdx.x]),
                   make_ulonglong2(sl.maxbits, sl.count));
        }
        __syncthreads();
        if (tid < 32) {
            // every lane of warp 0 polls with acquire semantics (one coalesced
            // request per poll), so its relaxed slot reads below are ordered
            ++epoch;
            if (tid == 0 && bdbg) bdbg[8] = cyc();
            if (tid == 0) red_release(&ctl->bar, 1u);
            if (tid == 0 && bdbg) bdbg[9] = cyc();
            const unsigned target = epoch * nb;
            while (static_cast<int>(ld_acquire(&ctl->bar) - target) < 0) {
            }
            if (tid == 0 && bdbg) bdbg[10] = cyc();
            // lane l reads CTAs [l*per, (l+1)*per): max, and an exclusive scan of
            // the claim counts into s_pref (block order)
            const int per = (nb + 31) / 32;
            const int b0 = tid * per, b1 = min(nb, b0 + per);
            unsigned long long mx = 0, mine = 0;
            ulonglong2 sv[kSlotsPerLane];
#pragma unroll
            for (int x = 0; x < kSlotsPerLane; ++x)  // all loads in flight at once
                if (b0 + x < b1)
                    sv[x] = __ldcg(reinterpret_cast<const ulonglong2*>(
                        &slots[par * gridDim.x + g * nb + b0 + x]));
#pragma unroll
            for (int x = 0; x < kSlotsPerLane; ++x)
                if (b0 + x < b1) {
                    mx = sv[x].x > mx ? sv[x].x : mx;
                    s_pref[b0 + x] = static_cast<int>(sv[x].y);
                    mine += sv[x].y;
                }
            unsigned long long incl = mine;
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned long long y = __shfl_up_sync(kFull, incl, o);
                if (tid >= o) incl += y;
            }
            unsigned long long run = incl - mine;
            for (int b = b0; b < b1; ++b) {
                const int c = s_pref[b];
                s_pref[b] = static_cast<int>(run);
                run += c;
            }
            const unsigned long long tot = __shfl_sync(kFull, incl, 31);
            if (tid == 0) s_pref[nb] = static_cast<int>(tot);
            for (int o = 16; o > 0; o >>= 1) {
                const unsigned long long y = __shfl_xor_sync(kFull, mx, o);
                mx = y > mx ? y : mx;
            }
            __syncwarp();
            const unsigned long long before = static_cast<unsigned long long>(s_pref[lb]);
            if (tid == 0 && bdbg) bdbg[11] = cyc();
            if (tid == 0) post(mx, static_cast<int>(tot), static_cast<int>(before));
        }
        __syncthreads();
    };

    for (int q = g; q < A.nq; q += A.groups) {
        const int s0 = A.src_off ? A.src_off[q] : 0;
        const int m = A.src_off ? A.src_off[q + 1] - s0 : A.src_count;
        const int* src = A.src + s0;
        int k = 0, i = 1, rho = INT_MAX, parity = 0, bfs_open = 0, done = 0;
        int tail = 0, limk = 0, bb = 0, fe = 0, frzb = 0, frze = 0;
        unsigned long long upd = 0;
        int pf = -1;
        auto publish = [&] {
            S.done = done;
            s_ncnt = 0;
            if (done) return;
            const int kk = k + 1;
            const int j = bfs_open ? kk : min(kk, rho - 1);
            S.k = kk;
            S.i = i;
            S.j = j;
            S.bb = bb;
            S.fe = fe;
            const int be = (bfs_open || j + 1 == rho) ? tail : ldcg(limits + j + 1);
            S.be = be;
            S.oe = bfs_open ? limk : be;  // newest level: ids from the claim lists
            S.expand = bfs_open;
            S.cur = k & 1;                // claim-list parity holding the newest level
            S.frzb = frzb;
            S.frze = frze;
            S.parity = parity;
            pf = -1;
            if (i + 2 <= kk + 1 && (bfs_open || i + 2 <= rho))
                pf = (bfs_open && i + 2 == kk + 1) ? tail : ldcg(limits + i + 2);
        };

        if (tid == 0) s_err = 0;
        if (A.phase_init) {
            for (int v = gtid; v < n; v += gthreads) {
                dist[0][v] = inf;
                dist[1][v] = inf;
                if (LABELS) {
                    lab[0][v] = -1;
                    lab[1][v] = -1;
                }
                if (A.fused_bfs) level[v] = -1;
                if (A.last_change) A.last_change[v] = 0;
            }
            if (gtid == 0) {
                ctl->relax = ctl->degen = ctl->updates = 0;
                ctl->err = 0;
            }
            group_barrier(&ctl->bar, epoch, nb, [] {});
            for (int s = gtid; s < m; s += gthreads) {
                const int v = src[s];
                dist[0][v] = T(0);
                dist[1][v] = T(0);
                if (LABELS) {
                    lab[0][v] = s;
                    lab[1][v] = s;
                }
                if (A.fused_bfs) {
                    level[v] = 0;
                    pv[s] = v;
                }
            }
            if (A.fused_bfs && gtid == 0) {
                limits[0] = 0;
                limits[1] = m;
            }
            if (!A.fused_bfs) {
                // caller ordering: pack every reachable position's record up front
                const int reach = ldcg(limits + A.given_rho);
                int* pring = A.pring + off8;
                T* pL = static_cast<T*>(A.pL) + off8;
                char* pquad = static_cast<char*>(A.pquad) + off8 * sizeof(Quad<T>);
                for (long long x = gtid; x < static_cast<long long>(reach) * kEllW;
                     x += gthreads) {
                    const int p = static_cast<int>(x / kEllW), slot = static_cast<int>(x % kEllW);
                    const int v = ldcg(pv + p);
                    const size_t eb = static_cast<size_t>(v) * kEllW + slot;
                    pring[x] = __ldg(M.ering + eb);
                    pL[x] = __ldg(static_cast<const T*>(M.eL) + eb);
                    Quad<T> qq;
                    qq.load(M.equad, static_cast<int>(eb));
                    qq.store_at(pquad, x);
                }
            }
            if (tid == 0) s_ncnt = 0;
            group_barrier(&ctl->bar, epoch, nb, [] {});
            if (A.fused_bfs) {
                // iteration 0: claim level 1 from the sources into list 0
                const int gl = tid & (kGroup - 1);
                for (int t = lb + nb * (tid / kGroup);; t += nb * kGroupsPerBlock) {
                    const bool act = t < m;
                    if (!__any_sync(kFull, act)) break;
                    int v = 0, c0 = 0, d = 0;
                    if (act) {
                        v = ldcg(pv + t);
                        c0 = __ldg(M.cptr + v);
                        d = __ldg(M.cptr + v + 1) - c0;
                    }
                    int nch = d > 0 ? (d + 2 * kGroup) / (2 * kGroup) : 0;  // entries 0..d
                    nch = __reduce_max_sync(kFull, nch);
                    for (int ch = 0; ch < nch; ++ch) {
                        const int ea = ch * 2 * kGroup + gl, eb2 = ea + kGroup;
                        bool cA = false, cB = false;
                        int ia = 0, ib = 0;
                        if (act && d > 0 && ea <= d) {
                            ia = __ldg(M.ring + c0 + v + ea) & INT_MAX;
                            cA = atomicCAS(level + ia, -1, 1) == -1;
                        }
                        if (act && d > 0 && eb2 <= d) {
                            ib = __ldg(M.ring + c0 + v + eb2) & INT_MAX;
                            cB = atomicCAS(level + ib, -1, 1) == -1;
                        }
                        list_claims(cA, ia, cB, ib, lists[0], &s_ncnt, A.claim_cap, &s_err);
                    }
                }
                __syncthreads();
                const int mycnt = s_ncnt;
                barrier3(0, 0ull, mycnt, [&](unsigned long long, int tot, int) {
                    bb = m;
                    if (tot == 0) {
                        bfs_open = 0;
                        rho = 1;
                        tail = m;
                        fe = m;
                    } else {
                        bfs_open = 1;
                        limk = m;
                        tail = m + tot;
                        fe = tail;
                        if (lb == 0) limits[2] = tail;
                    }
                    done = !bfs_open && i > rho - 1;
                    publish();
                });
            } else {
                if (tid == 0) {
                    rho = A.given_rho;
                    bfs_open = 0;
                    tail = ldcg(limits + rho);
                    bb = ldcg(limits + 1);
                    fe = rho >= 2 ? ldcg(limits + 2) : tail;
                    done = i > rho - 1;
                    publish();
                }
                __syncthreads();
            }
        } else {
            if (tid == 0) {
                k = ctl->k; i = ctl->i; rho = ctl->rho; parity = ctl->parity;
                bfs_open = ctl->bfs_open; done = ctl->done;
                tail = ctl->s_tail; limk = ctl->s_limk; bb = ctl->s_bb; fe = ctl->s_fe;
                frzb = ctl->s_frzb; frze = ctl->s_frze;
                publish();
            }
            __syncthreads();
        }

        T my_max = T(0);
        long long calls = 0, degs = 0;
        int iters = 0;
        for (;;) {
            if (S.done || (A.max_iters > 0 && iters >= A.max_iters)) break;
            const int kk = S.k;
            const bool dbg = A.dbg != nullptr && tid == 0 && iters < A.dbg_iters;
            unsigned long long* dslot =
                dbg ? A.dbg + kDbgSlots * (static_cast<size_t>(iters) * gridDim.x + blockIdx.x) : nullptr;
            if (dbg) dslot[0] = gtimer();
            const int prv = S.parity, cur_b = prv ^ 1;
            const T* dp = dist[prv];
            T* dcur = dist[cur_b];
            const int* lp = LABELS ? lab[prv] : nullptr;
            int* lc = LABELS ? lab[cur_b] : nullptr;
            const int bb_ = S.bb, fe_ = S.fe, oe_ = S.oe;
            const bool expand = S.expand != 0;
            const int* clist_base = claim_list(S.cur, 0);
            int* nlist = lists[kk & 1];
            const int ntask = S.be - bb_;
            my_max = T(0);
            for (int t = lb + nb * (tid / kGroup);; t += nb * kGroupsPerBlock) {
                const bool act = t < ntask;
                if (!__any_sync(kFull, act)) break;
                const int p = bb_ + t;
                const bool is_new = p >= oe_;
                int vn = 0;
                if (act && is_new) {
                    // position -> (claimer CTA, index) through the prefix table
                    const int r = p - oe_;
                    int lo = 0, hi = nb;  // s_pref[lo] <= r < s_pref[hi]
                    while (hi - lo > 1) {
                        const int mid = (lo + hi) >> 1;
                        if (s_pref[mid] <= r) lo = mid; else hi = mid;
                    }
                    vn = ldcg(clist_base + static_cast<size_t>(lo) * A.claim_cap + (r - s_pref[lo]));
                }
                relax3<T, LABELS>(M, A, off8, act, is_new, vn, p, kk, pv, dp, dcur, lp, lc, fe_,
                                  expand, level, nlist, &s_ncnt, &s_err, eps, my_max, calls, degs,
                                  (dbg && t == lb && act) ? dslot : nullptr);
            }
            if (dbg) dslot[7] = cyc();
            // deferred freeze of the level retired last iteration, on the highest
            // (usually idle) threads (ptp.cpp:121-130)
            {
                const int nf = S.frze - S.frzb;
                for (int f = gthreads - 1 - gtid; f < nf; f += gthreads) {
                    const int v = ldcg(pv + S.frzb + f);
                    dcur[v] = ldcg(dp + v);
                    if (LABELS) lc[v] = ldcg(lp + v);
                }
            }
            const T bmax = block_max(my_max, red_t);
            if (dbg) dslot[1] = gtimer();
            bdbg = dslot;
            const int mycnt = s_ncnt;  // after block_max's __syncthreads
            barrier3(kk & 1, Lim<T>::bits(bmax), mycnt,
                     [&](unsigned long long mxb, int tot, int) {
                if (dbg) dslot[2] = gtimer();
                const T mr = Lim<T>::from_bits(mxb);
                const bool conv = mr < eps;  // ptp.cpp:114
                const int ub = bb, ue = S.be;
                upd += static_cast<unsigned long long>(ue - ub);
                if (lb == 0 && A.trace != nullptr) {
                    const int row = kk - A.trace_k0;
                    if (row >= 0 && row < A.trace_cap) {
                        TraceRow r;
                        r.k = kk; r.i = i; r.j = S.j; r.conv = conv ? 1 : 0;
                        r.updated = ue - ub;
                        r.max_rel = static_cast<double>(mr);
                        A.trace[row] = r;
                    }
                }
                int nt = tail;
                if (bfs_open) {
                    if (tot == 0) {
                        bfs_open = 0;
                        rho = kk + 1;
                    } else {
                        nt = tail + tot;
                        if (lb == 0) limits[kk + 2] = nt;
                        limk = tail;
                    }
                }
                if (conv) {
                    frzb = bb;
                    frze = fe;
                    bb = fe;
                    fe = (i + 2 <= kk + 1) ? pf : nt;
                    ++i;
                } else {
                    frzb = frze = 0;
                }
                tail = nt;
                parity ^= 1;
                k = kk;
                done = !bfs_open && i > rho - 1;
                publish();
            });
            ++iters;
        }

        const long long bc = block_sum(calls, red_l);
        const long long bd = block_sum(degs, red_l);
        if (tid == 0) {
            if (bc) atomicAdd(&ctl->relax, static_cast<unsigned long long>(bc));
            if (bd) atomicAdd(&ctl->degen, static_cast<unsigned long long>(bd));
            if (s_err) atomicMax(&ctl->err, s_err);
            if (lb == 0) {
                ctl->k = k; ctl->i = i; ctl->rho = rho; ctl->parity = parity;
                ctl->bfs_open = bfs_open; ctl->done = done;
                ctl->s_tail = tail; ctl->s_limk = limk; ctl->s_bb = bb; ctl->s_fe = fe;
                ctl->s_frzb = frzb; ctl->s_frze = frze;
                ctl->updates += upd;
            }
            S.done = done;
            S.parity = parity;
        }
        __syncthreads();
        const int fin_done = S.done;
        const int fin = S.parity;
        if (!fin_done) continue;

        double vmax = -1.0;
        int vidx = INT_MAX;
        if (A.out_dist != nullptr || A.fps_mode || A.out_labels != nullptr) {
            const T* df = dist[fin];
            const int* lf = LABELS ? lab[fin] : nullptr;
            const long long qo = static_cast<long long>(q) * n;
            for (int v = gtid; v < n; v += gthreads) {
                const T x = ldcg(df + v);
                if (A.out_dist != nullptr) {
                    if (A.out_double)
                        static_cast<double*>(A.out_dist)[qo + v] = static_cast<double>(x);
                    else
                        static_cast<float*>(A.out_dist)[qo + v] = static_cast<float>(x);
                }
                if (A.out_labels != nullptr)
                    A.out_labels[qo + v] = LABELS ? ldcg(lf + v) : (x != inf ? 0 : -1);
                const double xd = static_cast<double>(x);
                if (xd > vmax || (xd == vmax && v < vidx)) {
                    vmax = xd;
                    vidx = v;
                }
            }
        }
        if (A.fps_mode) {
            for (int o = 16; o > 0; o >>= 1) {
                const double ov = __shfl_xor_sync(kFull, vmax, o);
                const int oi = __shfl_xor_sync(kFull, vidx, o);
                if (ov > vmax || (ov == vmax && oi < vidx)) { vmax = ov; vidx = oi; }
            }
            if ((tid & 31) == 0) { red_v[tid >> 5] = vmax; red_i[tid >> 5] = vidx; }
            __syncthreads();
            if (tid == 0) {
                for (int w = 1; w < kBlock / 32; ++w)
                    if (red_v[w] > vmax || (red_v[w] == vmax && red_i[w] < vidx)) {
                        vmax = red_v[w];
                        vidx = red_i[w];
                    }
                A.fps_scratch[2 * blockIdx.x] =
                    static_cast<unsigned long long>(__double_as_longlong(vmax));
                A.fps_scratch[2 * blockIdx.x + 1] = static_cast<unsigned long long>(vidx);
            }
        }
        group_barrier(&ctl->bar, epoch, nb, [&] {
            if (lb != 0) return;
            QueryStats st;
            st.relax = static_cast<long long>(__ldcg(&ctl->relax));
            st.degen = static_cast<long long>(__ldcg(&ctl->degen));
            st.updates = static_cast<long long>(ctl->updates);
            st.iterations = k;
            st.rho = rho;
            st.unreached = n - tail;
            st.done = 1;
            st.radius = 0.0;
            st.argmax = -1;
            st.pad = __ldcg(&ctl->err) >= 2 ? __ldcg(&ctl->err) : 0;  // 2: claim list overflow
            if (A.fps_mode) {
                double bv = -1.0;
                int bi = INT_MAX;
                for (int b = g * nb; b < g * nb + nb; ++b) {
                    const double ov = __longlong_as_double(
                        static_cast<long long>(__ldcg(&A.fps_scratch[2 * b])));
                    const int oi = static_cast<int>(__ldcg(&A.fps_scratch[2 * b + 1]));
                    if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
                }
                st.radius = bv;
                st.argmax = bi;
                if (!A.fps_final) {
                    if (ldcg(level + bi) == 0) ctl->err = 1;
                    A.fps_samples[A.src_count] = bi;
                }
            }
            A.qstats[q] = st;
        });
    }
}

// ---------------------------------------------------------------------------
template <typename T>
__global__ void planar_test_kernel(const double* x1, const double* x2, const double* t1,
                                   const double* t2, int count, double* value, int* side,
                                   int* degen) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= count) return;
    const T ax = to_t<T>(x1[3 * q]), ay = to_t<T>(x1[3 * q + 1]), az = to_t<T>(x1[3 * q + 2]);
    const T bx = to_t<T>(x2[3 * q]), by = to_t<T>(x2[3 * q + 1]), bz = to_t<T>(x2[3 * q + 2]);
    const T g11 = dot3(ax, ay, az, ax, ay, az), g22 = dot3(bx, by, bz, bx, by, bz);
    const T g12 = dot3(ax, ay, az, bx, by, bz);
    T q11, q12, q22, a;
    const bool dg = corner_geometry(g11, g22, g12, q11, q12, q22, a);
    // the solver's own path: the packed quad (4th word per quad_w) and corner_eval
    Quad<T> qd;
    qd.q11 = q11;
    qd.q12 = q12;
    qd.q22 = q22;
    qd.a = quad_w<T>(a, dg);
    int s, d;
    const T v = corner_eval<T>(to_t<T>(t1[q]), to_t<T>(t2[q]), sq(g11), sq(g22), qd, dg, false, s, d);
    value[q] = static_cast<double>(v);
    side[q] = s;
    degen[q] = d;
}

// ---------------------------------------------------------------------------
// host launchers

template <typename T>
void launch_pack(const double* xyz, int n, const int* cptr, const int* ring_in, int* ring_out,
                 void* ringL, void* quad, int* ering, void* eL, void* equad, cudaStream_t st) {
    const int blk = 256;
    const int grid = (n + blk - 1) / blk;
    if (grid == 0) return;
    pack_kernel<T><<<grid, blk, 0, st>>>(xyz, n, cptr, ring_in, ring_out, static_cast<T*>(ringL),
                                         quad);
    note_launch();
    pack_ell_kernel<T><<<grid, blk, 0, st>>>(n, cptr, ring_out, static_cast<const T*>(ringL),
                                             quad, ering, static_cast<T*>(eL), equad);
    note_launch();
}
template void launch_pack<float>(const double*, int, const int*, const int*, int*, void*, void*,
                                 int*, void*, void*, cudaStream_t);
template void launch_pack<double>(const double*, int, const int*, const int*, int*, void*, void*,
                                  int*, void*, void*, cudaStream_t);

void launch_planar_test(int precision, const double* x1, const double* x2, const double* t1,
                        const double* t2, int count, double* value, int* side, int* degen,
                        cudaStream_t st) {
    const int blk = 128;
    const int grid = (count + blk - 1) / blk;
    if (precision == 0)
        planar_test_kernel<float><<<grid, blk, 0, st>>>(x1, x2, t1, t2, count, value, side, degen);
    else
        planar_test_kernel<double><<<grid, blk, 0, st>>>(x1, x2, t1, t2, count, value, side, degen);
    note_launch();
}

// Self-test of the straight-line div/sqrt fast paths (ptp_common.cuh) against the
// IEEE intrinsics on pseudo-random operands spanning the exponent range: counts the
// operands each fast path accepts (checked) and those where it differs (mismatch).
// out[0..7] = fp64 div checked, mismatch, fp64 sqrt checked, mismatch, fp32 div ...,
// fp32 sqrt ...
__device__ __forceinline__ unsigned long long mix64(unsigned long long x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull;
    return x ^ (x >> 33);
}
__global__ void arith_selftest_kernel(long long n, unsigned long long seed,
                                      unsigned long long* out) {
    unsigned long long c[8] = {};
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const unsigned long long h1 = mix64(seed ^ (2 * i)), h2 = mix64(seed ^ (2 * i + 1));
        // doubles: random mantissa and sign, exponent in [-300, 300] (and a few edges)
        auto mk = [](unsigned long long h) {
            const unsigned long long e = 1023 - 300 + (h >> 52) % 601;
            return __longlong_as_double(static_cast<long long>(((h & 1ull) << 63) | (e << 52) |
                                                               (h >> 12 & 0xfffffffffffffull)));
        };
        const double x = mk(h1), y = mk(h2);
        bool ok;
        const double q = div_with_recip64(x, y, div_recip64(y), ok);
        if (ok) {
            ++c[0];
            c[1] += __double_as_longlong(q) != __double_as_longlong(__ddiv_rn(x, y));
        }
        const double ax = fabs(x);
        const double r = sqrt_fast64(ax, ok);
        if (ok) {
            ++c[2];
            c[3] += __double_as_longlong(r) != __double_as_longlong(__dsqrt_rn(ax));
        }
        // floats: exponent in [-80, 80]
        auto mkf = [](unsigned long long h) {
            const unsigned e = 127 - 80 + static_cast<unsigned>((h >> 40) % 161);
            return __uint_as_float(static_cast<unsigned>((h & 1ull) << 31) | (e << 23) |
                                   static_cast<unsigned>(h >> 9 & 0x7fffffu));
        };
        const float xf = mkf(h1), yf = mkf(h2);
        if (div_operand_ok(xf) && div_operand_ok(yf)) {
            ++c[4];
            const float qf = div_with_recip(xf, yf, div_recip(yf));
            c[5] += __float_as_uint(qf) != __float_as_uint(__fdiv_rn(xf, yf));
        }
        const float af = fabsf(xf);
        if (sqrt_fast_ok(af)) {
            ++c[6];
            c[7] += __float_as_uint(sqrt_fast(af)) != __float_as_uint(__fsqrt_rn(af));
        }
    }
    for (int k = 0; k < 8; ++k) atomicAdd(out + k, c[k]);
}

void launch_arith_selftest(long long n, unsigned long long seed, unsigned long long* out,
                           cudaStream_t st) {
    arith_selftest_kernel<<<4 * 148, 256, 0, st>>>(n, seed, out);
    note_launch();
}

__global__ void reset_bars_kernel(GroupCtl* ctl, int groups) {
    for (int g = threadIdx.x; g < groups; g += blockDim.x) {
        ctl[g].bar = 0u;
        for (int w = 0; w < 4; ++w) ctl[g].barw[w] = 0ull;
    }
}

static const void* run_kernel_ptr(int version, int precision, bool labels) {
    if (version >= 4) return run4_kernel_ptr(precision, labels, version - 4);
    if (version == 2) {
        if (precision == 0)
            return labels ? reinterpret_cast<const void*>(&ptp_run_kernel<float, true>)
                          : reinterpret_cast<const void*>(&ptp_run_kernel<float, false>);
        return labels ? reinterpret_cast<const void*>(&ptp_run_kernel<double, true>)
                      : reinterpret_cast<const void*>(&ptp_run_kernel<double, false>);
    }
    if (precision == 0)
        return labels ? reinterpret_cast<const void*>(&ptp_run3_kernel<float, true>)
                      : reinterpret_cast<const void*>(&ptp_run3_kernel<float, false>);
    return labels ? reinterpret_cast<const void*>(&ptp_run3_kernel<double, true>)
                  : reinterpret_cast<const void*>(&ptp_run3_kernel<double, false>);
}

// v4: shared-memory record cache
static size_t run_dyn_smem(int version, int precision, bool labels) {
    return version >= 4 ? run4_dyn_smem(precision, labels) : 0;
}

int run_max_blocks(int precision, bool labels, int device, int version) {
    int per_sm = 0, sms = 0;
    const void* f = run_kernel_ptr(version, precision, labels);
    const size_t dyn = run_dyn_smem(version, precision, labels);
    if (dyn) cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, f, kBlock, dyn);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    const int total = per_sm * sms;
    return version == 3 ? (total < kMaxGroupBlocks ? total : kMaxGroupBlocks) : total;
}

cudaError_t launch_run(int precision, bool labels, const RunArgs& args, cudaStream_t st,
                       int version) {
    const int grid = args.groups * args.blocks_per_group;
    RunArgs a = args;
    void* params[] = {&a};
    reset_bars_kernel<<<1, 32, 0, st>>>(a.ctl, a.groups);
    note_launch();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const void* f = run_kernel_ptr(version, precision, labels);
    const size_t dyn = run_dyn_smem(version, precision, labels);
    if (dyn) cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    e = cudaLaunchCooperativeKernel(f, dim3(grid), dim3(version >= 4 ? run4_block(version - 4) : kBlock),
                                    params, dyn, st);
    note_launch();
    return e;
}

}  // namespace gdb
