// The PTP solver (sm_100a): the band loop of run_impl<T> (reference src/ptp.cpp:79-132) with
// compute_toplesets' BFS (src/toplesets.cpp:37-55) fused in, as one persistent cooperative
// kernel per field (or per group of concurrent fields), bit-identical to the reference.
// Where every dependent memory trip of an iteration goes:
//
//  * the BFS runs one topleset ahead of the band: at iteration k a BFS task per position of
//    level k+1 reads the vertex's ELL row (pulled into L2 by its claimer) into the owner's
//    record cache (narrow iterations) or its packed record (wide ones) and claims level k+2
//    (bfs4); level k+1 is relaxed for the first time at iteration k+1 from the chip.
//  * narrow iterations (MODE 1): BFS position p is owned by CTA p % nb for the whole solve
//    and its record lives in the owner's shared-memory cache (slot p / nb), so a band vertex
//    costs one L2 trip per iteration: its neighbours' cells (by vertex id).
//  * claims go to a per-CTA list; their BFS positions are assigned by the grid barrier
//    itself: the arrival is one atom.acq_rel.add of a 64-bit word whose fields carry the
//    iteration's payload (bits 0-15 arrivals, 16-31 CTAs with a front change >= eps,
//    ptp.cpp:107,114, 32-63 claims = the next topleset's size); the value it returns is the
//    CTA's offset in the new topleset, and warp 0 writes the list to pv[] / posof[] while
//    the CTA waits.  Topleset limits live in a shared-memory ring.
//  * wide iterations (MODE 2; band beyond the record cache) relax one vertex per thread in
//    chunks of 32 positions from records packed by position (slot-major, the
//    reorder_for_bands layout, toplesets.cpp:60-89); single-source fields keep their cells
//    by BFS position there (relayout), and fp64 ones relax only the positions a change
//    marked (the change-driven worklist).
#include "ptp_common.cuh"
#include "ptp_launch.hpp"

namespace gdb {

namespace {

constexpr int kLimRing = 1024;  // topleset limits kept on chip (levels)
// pv[p] flag: the packed record at position p has been written.  Packed records
// are only written once the band approaches the record cache's capacity (they
// serve the wide path); writing them on every first relaxation would stream
// n * 192 B through the L2 and evict the distance and level arrays.
constexpr int kPacked = 1 << 30;
// packed ring entry flag: still a vertex id, its position was not known when the
// record was written (the topleset after the vertex's own, claimed in the same
// iteration); resolved through posof at a later relaxation.  Bit 30 is free in every
// entry of a packed record (entry 0's corner-count field is <= 7 there).
#ifndef GEODIST_POSL
#define GEODIST_POSL 0
#endif
constexpr int kUnres = 1 << 30;
// pv[p] flag: the vertex has a degenerate corner (its degenerate_calls count depends on
// which of its corners are finite, so the change-driven worklist never skips it)
constexpr int kAlways = 1 << 29;
#ifndef GEODIST_WORKLIST
#define GEODIST_WORKLIST 1
#endif
// Position-layout wide iterations relax only positions marked by a change in the
// previous iteration (see the older-band loop); 0: every band position every iteration.
// fp64 only: measured on the 1000^2 torus, fp64 17.3 ms with it vs 18.7 without, fp32
// 15.3 vs 14.6 -- the scan trip costs more than the skipped fp32 relaxations save.
#ifndef GEODIST_WL_MASK
#define GEODIST_WL_MASK 0  // bit 0: fp32 single source, 1: fp32 labels, 2: fp64 single, 3: fp64 labels
#endif
template <typename T, bool L> __host__ __device__ constexpr bool worklist_for() {
    return GEODIST_WORKLIST != 0 &&
           ((GEODIST_WL_MASK >> ((sizeof(T) == 8 ? 2 : 0) + (L ? 1 : 0))) & 1) != 0;
}

// Mark position q for relaxation in the next iteration (mark value kk + 1 in the array
// of the next iteration's parity).  Plain stores: every writer stores the same value.
__device__ __forceinline__ void mark(int* dnext, int q, int kk) { dnext[q] = kk + 1; }

struct T0State {
    int k, i, rho, parity, bfs_open, done, tail, bb, fe, frzb, frze, lim_top;
    bool use_glim;
    unsigned long long upd;
    int sh_p0, sh_a0, sh_f0, sh_fa0, sh_nfz, be_pub, sh_x0, sh_xa0;
};

struct Bcast4 {
    int k, i, j, bb, oe, be, fe, frzb, frze, parity, done, expand;
    int tail;  // positions assigned so far
    // BFS tasks (one topleset ahead of the band): positions [be, xe); this CTA's first one
    // (xp0, cache slot xa0)
    int xe, xp0, xa0;
    // this CTA's share (positions p == lb mod nb): band tasks p0 + t * nb below
    // be (record-cache slot a0 + t), frozen positions f0 + t * nb for t < nfz
    int p0, a0, f0, fa0, nfz;
};

// Record-cache ring (power of two) per CTA; narrow iterations last while the band and the
// BFS tasks' topleset span at most cache_slots - 1 positions per CTA.  The rest of the SM's
// shared memory is L1 (cell gathers).  Measured (icosphere-8 / grid / torus / height):
// fp32 128 slots 3.64 ms vs 256: 3.76 on the icosphere-8, the others equal; fp64 256 slots
// 3.99 ms vs 128: 4.48 (its band spills to the wide path) and vs 512: 4.06.
#ifndef GEODIST_CACHE_SLOTS32
#define GEODIST_CACHE_SLOTS32 128
#endif
#ifndef GEODIST_CACHE_SLOTS64
#define GEODIST_CACHE_SLOTS64 256
#endif
template <typename T> __host__ __device__ constexpr int cache_slots() {
    return sizeof(T) == 4 ? GEODIST_CACHE_SLOTS32 : GEODIST_CACHE_SLOTS64;
}

__device__ __forceinline__ void red_release_u64(unsigned long long* p, unsigned long long x) {
    asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(x) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long atom_acq_rel_add_u64(unsigned long long* p,
                                                                   unsigned long long x) {
    unsigned long long r;
    asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], %2;" : "=l"(r) : "l"(p), "l"(x) : "memory");
    return r;
}
__device__ __forceinline__ int ld_relaxed_i32(const int* p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long x) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(x) : "memory");
}

// Shared-memory record cache: one lane's share (entries gl and gl+4) of slot s
// lives at index s * 4 + gl of each array.
template <typename T> struct Cache {
    int2* rr;    // ring entries (ids | flags; entry 0 carries the corner count)
    int2* pv;    // (position tag, vertex id)
    T* L;        // |x| of the two entries
    Quad<T>* q;  // Gram quads of corners gl and gl+4
    __host__ __device__ static constexpr size_t bytes_per_slot() {
        return 4 * (sizeof(int2) + sizeof(int2) + 2 * sizeof(T) + 2 * sizeof(Quad<T>));
    }
    __device__ void bind(unsigned char* base, int R) {
        rr = reinterpret_cast<int2*>(base);
        pv = rr + 4 * R;
        L = reinterpret_cast<T*>(pv + 4 * R);
        q = reinterpret_cast<Quad<T>*>(L + 8 * R);
    }
};

template <typename T> __device__ __forceinline__ void sm_store_quad(Quad<T>* at, const Quad<T>& x);
template <typename T> __device__ __forceinline__ void sm_load_quad(const Quad<T>* at, Quad<T>& x);
template <> __device__ __forceinline__ void sm_store_quad<float>(Quad<float>* at, const Quad<float>& x) {
    *reinterpret_cast<float4*>(at) = make_float4(x.q11, x.q12, x.q22, x.a);
}
template <> __device__ __forceinline__ void sm_load_quad<float>(const Quad<float>* at, Quad<float>& x) {
    const float4 v = *reinterpret_cast<const float4*>(at);
    x.q11 = v.x; x.q12 = v.y; x.q22 = v.z; x.a = v.w;
}
template <> __device__ __forceinline__ void sm_store_quad<double>(Quad<double>* at, const Quad<double>& x) {
    double2* p = reinterpret_cast<double2*>(at);
    p[0] = make_double2(x.q11, x.q12);
    p[1] = make_double2(x.q22, x.a);
}
template <> __device__ __forceinline__ void sm_load_quad<double>(const Quad<double>* at, Quad<double>& x) {
    const double2* p = reinterpret_cast<const double2*>(at);
    const double2 u = p[0], w = p[1];
    x.q11 = u.x; x.q12 = u.y; x.q22 = w.x; x.a = w.y;
}

// Claims of one warp go to the CTA's claim list (index from a shared-memory
// counter; entries beyond kSmemClaims spill to the CTA's global list).  Their
// BFS positions are assigned at the grid barrier: the arrival atomic returns
// the claims of the CTAs that arrived earlier, and warp 0 writes the list to
// pv[level start + that prefix + index] (claim_list_flush).  The claimer also
// pulls the vertex's ELL row towards L2 for the owner's first relaxation.
constexpr int kSmemClaims = 2048;

template <typename T>
__device__ __forceinline__ void claim_records(bool ca, int ia, bool cb, int ib,
                                              const MeshDev& M, int* s_list, int* g_list,
                                              int g_cap, int* s_ccnt, int* err) {
    const unsigned ba = __ballot_sync(kFull, ca), bbal = __ballot_sync(kFull, cb);
    const int na = __popc(ba);
    const int total = na + __popc(bbal);
    if (total == 0) return;
    if (ca) prefetch_ell<T>(M, ia);
    if (cb) prefetch_ell<T>(M, ib);
    const int l32 = threadIdx.x & 31;
    int base = 0;
    if (l32 == 0) base = atomicAdd(s_ccnt, total);
    base = __shfl_sync(kFull, base, 0);
    const unsigned lt = (1u << l32) - 1u;
    auto put = [&](int at, int id) {
        if (at < kSmemClaims) s_list[at] = id;
        else if (at - kSmemClaims < g_cap) g_list[at - kSmemClaims] = id;
        else *err = 2;
    };
    if (ca) put(base + __popc(ba & lt), ia);
    if (cb) put(base + na + __popc(bbal & lt), ib);
}

struct ClaimCtx {
    int* s_list;
    int* g_list;
    int g_cap;
    int* ccnt;
    int* err;
};

// Relax the vertex at BFS position p (narrow iterations; 4-lane group; relax_vertex,
// update_kernel.hpp:93-120): its record from the CTA's shared-memory cache (left there by
// its BFS task, or by an earlier relaxation), or on a miss from the id-indexed ELL row;
// the cells by vertex id.
template <typename T, bool LABELS>
__device__ __forceinline__ void relax4(const MeshDev& M, const RunArgs& A, const Cache<T>& C,
                                       int sl, bool act, int p, int kk, const int* pv,
                                       const Cell<T, LABELS>* cp, Cell<T, LABELS>* cc, int fe,
                                       T eps, int& nonconv, T& my_max, long long& calls,
                                       long long& degs, unsigned long long* tdbg) {
    const T inf = Lim<T>::inf();
    if (tdbg) tdbg[3] = cyc();
    const int gl = threadIdx.x & (kGroup - 1);
    const int g0 = (threadIdx.x & 31) & ~(kGroup - 1);
    int v = 0;
    int2 rr = make_int2(0, 0);
    T La = T(0), Lb = T(0);
    Quad<T> qa, qb;
    qa.q11 = qa.q12 = qa.q22 = qa.a = T(0);
    qb = qa;
    const int ci = sl * 4 + gl;
    bool hit = false;
    if (act) {
        const int2 tg = C.pv[ci];
        if (tg.x == p) {
            hit = true;
            v = tg.y;
            rr = C.rr[ci];
            La = C.L[2 * ci];
            Lb = C.L[2 * ci + 1];
            sm_load_quad<T>(C.q + 2 * ci, qa);
            sm_load_quad<T>(C.q + 2 * ci + 1, qb);
        }
    }
    if (act && !hit) {
        // cache miss (the first narrow iteration of a launch): position word, ELL row
        v = ldcg(pv + p) & kIdMask;
        const size_t eb = static_cast<size_t>(v) * kEllW;
        rr = __ldg(reinterpret_cast<const int2*>(M.ering) + (eb >> 1) + gl);
        Ell2<T>::load(M.eL, eb + 2 * gl, La, Lb);
        qa.load(M.equad, static_cast<int>(eb + 2 * gl));
        qb.load(M.equad, static_cast<int>(eb + 2 * gl + 1));
        C.pv[ci] = make_int2(p, v);
        C.rr[ci] = rr;
        C.L[2 * ci] = La;
        C.L[2 * ci + 1] = Lb;
        sm_store_quad<T>(C.q + 2 * ci, qa);
        sm_store_quad<T>(C.q + 2 * ci + 1, qb);
    }
    if (tdbg) tdbg[4] = gtimer_after(rr.x + v);
    const int meta = __shfl_sync(kFull, rr.x, g0);
    int d = act ? (meta >> kMetaShift) & 15 : 0;
    const bool ovf = d == kEllOverflow;
    const int ida = rr.x & kIdMask;
    const int idb = rr.y & kIdMask;
    const bool hasa = act && !ovf && d > 0 && gl <= d;
    const bool hasb = act && !ovf && d > 0 && gl + kGroup <= d;
    T tv = inf;
    int lv = -1, sv = 0;
    T ta = inf, tb = inf;
    int la = -1, lb_ = -1;
    if (act && gl == 0) {
        const Cell<T, LABELS> c = ld_cell(cp + v);
        tv = c.d;
        lv = c.lab();
        sv = c.stamp();
    }
    if (hasa) {
        const Cell<T, LABELS> c = ld_cell(cp + ida);
        ta = c.d;
        la = c.lab();
    }
    if (hasb) {
        const Cell<T, LABELS> c = ld_cell(cp + idb);
        tb = c.d;
        lb_ = c.lab();
    }
    if (tdbg) tdbg[5] = gtimer_after(__float_as_int(static_cast<float>(ta + tb + tv)));
    T best = gl == 0 ? tv : inf;
    int bidx = gl == 0 ? -1 : INT_MAX;
    int blab = gl == 0 ? lv : -1;
    chunk_candidates<T, LABELS>(gl, 0, ovf ? 0 : d, rr.x, rr.y, La, Lb, ta, tb, la, lb_, qa, qb,
                                best, bidx, blab, degs);
    if (tdbg) tdbg[6] = gtimer_after(__float_as_int(static_cast<float>(best)));

    // overflow vertices (> 7 corners): CSR tables, 7 corners per chunk (rare: valence > 7)
    if (__any_sync(kFull, act && ovf)) {
        int c0 = 0;
        if (act && ovf) {
            c0 = __ldg(M.cptr + v);
            d = __ldg(M.cptr + v + 1) - c0;
        }
        const int r0 = c0 + v;
        int nch = act && ovf ? (d + kEllW - 2) / (kEllW - 1) : 0;
        nch = __reduce_max_sync(kFull, nch);
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
                xa = __ldg(M.ring + r0 + ea);
                LA = __ldg(ringL + r0 + ea);
                if (ea < d) QA.load(M.quad, c0 + ea);
            }
            if (hb) {
                xb = __ldg(M.ring + r0 + ebb);
                LB = __ldg(ringL + r0 + ebb);
                if (ebb < d) QB.load(M.quad, c0 + ebb);
            }
            const int ia = xa & INT_MAX, ib = xb & INT_MAX;
            if (ha) {
                const Cell<T, LABELS> c = ld_cell(cp + ia);
                TA = c.d;
                lA = c.lab();
            }
            if (hb) {
                const Cell<T, LABELS> c = ld_cell(cp + ib);
                TB = c.d;
                lB = c.lab();
            }
            const int dlim = act && ovf ? min(d, base + kEllW - 1) : 0;
            chunk_candidates<T, LABELS>(gl, base, dlim, xa, xb, LA, LB, TA, TB, lA, lB, QA, QB,
                                        best, bidx, blab, degs);
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
        // the change stamp: this iteration if the distance changed (a label changes
        // only with its distance, update_kernel.hpp:114-117)
        st_cell(cc + v, make_cell<T, LABELS>(best, blab, best != tv ? kk : sv));
        calls += d;
        if (p < fe || A.last_change != nullptr) {
            const T rc = rel_change(tv, best);
            if (p < fe && rc >= eps) nonconv = 1;
            if (p < fe && rc > my_max) my_max = rc;
            if (A.last_change != nullptr && rc >= eps) A.last_change[v] = kk;
        }
    }
}

// BFS one topleset ahead of the band (toplesets.cpp:37-55).  At iteration k the band's
// newest topleset is level k, and a BFS task per position of level k + 1 (positioned at
// the barrier that ended iteration k - 1) reads the vertex's ELL row -- into its record-
// cache slot in narrow iterations, into its packed record in wide ones -- and claims its
// unvisited neighbours for level k + 2 (atomicCAS on `level`; positions are assigned at
// this iteration's barrier).  Level k + 1 is relaxed for the first time at iteration k + 1
// from the row its BFS task left on chip: the relaxation's chain no longer carries the pv
// and row trips nor the claims' atomics.  4-lane group per position, lanes return their
// claims in (ca, ia, cb, ib).
template <typename T>
__device__ __forceinline__ void bfs4(const MeshDev& M, const RunArgs& A, const Cache<T>& C,
                                     int sl, bool act, bool cached, bool pack, bool posm, int p,
                                     int lvl,
                                     int* pv, const int* posof, int* pring, T* pL, char* pquad,
                                     int* level, const ClaimCtx& CC, bool& ca_claim, int& ida,
                                     bool& cb_claim, int& idb) {
    const int gl = threadIdx.x & (kGroup - 1);
    const int g0 = (threadIdx.x & 31) & ~(kGroup - 1);
    int v = 0;
    int2 rr = make_int2(0, 0);
    T La = T(0), Lb = T(0);
    Quad<T> qa, qb;
    qa.q11 = qa.q12 = qa.q22 = qa.a = T(0);
    qb = qa;
    if (act) {
        // the claimer's warp 0 wrote pv[p] right after its barrier arrival
        v = ld_relaxed_i32(pv + p);
        for (int spin = 0; v < 0; ++spin) {
            if (spin > (1 << 22)) {
                *CC.err = 3;
                v = 0;
                break;
            }
            v = ld_relaxed_i32(pv + p);
        }
        const size_t eb = static_cast<size_t>(v) * kEllW;
        rr = __ldg(reinterpret_cast<const int2*>(M.ering) + (eb >> 1) + gl);
        Ell2<T>::load(M.eL, eb + 2 * gl, La, Lb);
        qa.load(M.equad, static_cast<int>(eb + 2 * gl));
        qb.load(M.equad, static_cast<int>(eb + 2 * gl + 1));
    }
    const int meta = __shfl_sync(kFull, rr.x, g0);
    int d = act ? (meta >> kMetaShift) & 15 : 0;
    const bool ovf = d == kEllOverflow;
    ida = rr.x & kIdMask;
    idb = rr.y & kIdMask;
    const bool hasa = act && !ovf && d > 0 && gl <= d;
    const bool hasb = act && !ovf && d > 0 && gl + kGroup <= d;
    ca_claim = hasa && atomicCAS(level + ida, -1, lvl) == -1;
    cb_claim = hasb && atomicCAS(level + idb, -1, lvl) == -1;
    if (cached && act) {
        const int ci = sl * 4 + gl;
        C.pv[ci] = make_int2(p, v);
        C.rr[ci] = rr;
        C.L[2 * ci] = La;
        C.L[2 * ci + 1] = Lb;
        sm_store_quad<T>(C.q + 2 * ci, qa);
        sm_store_quad<T>(C.q + 2 * ci + 1, qb);
    }
    if (!cached || pack) {  // CTA-uniform
        // the packed record: in the position layout ring entries as positions (levels
        // k .. k + 1 are positioned; an entry of level k + 2 keeps its id, flagged kUnres)
        int dg = ((gl < d && rr.x < 0) || (gl + kGroup < d && rr.y < 0)) ? 1 : 0;
        dg |= __shfl_xor_sync(kFull, dg, 1, kGroup);
        dg |= __shfl_xor_sync(kFull, dg, 2, kGroup);
        if (act && !ovf) {
            int ea = rr.x, eb2 = rr.y;
            if (posm) {
                const int pa = hasa ? ldcg(posof + ida) : -1;
                const int pb = hasb ? ldcg(posof + idb) : -1;
                const int fa = rr.x & ~kIdMask, fb = rr.y & ~kIdMask;
                ea = !hasa ? rr.x : pa >= 0 ? (fa | pa) : (fa | kUnres | ida);
                eb2 = !hasb ? rr.y : pb >= 0 ? (fb | pb) : (fb | kUnres | idb);
            }
            const size_t N = static_cast<size_t>(A.stride);
            const size_t s0 = (2 * gl) * N + p, s1 = (2 * gl + 1) * N + p;
            pring[s0] = ea;
            pring[s1] = eb2;
            pL[s0] = La;
            pL[s1] = Lb;
            qa.store_at(pquad, s0);
            qb.store_at(pquad, s1);
            if (gl == 0) pv[p] = v | kPacked | (dg ? kAlways : 0);
        }
    }
    // overflow vertices (> 7 corners): the CSR ring, claims appended chunk by chunk
    if (__any_sync(kFull, act && ovf)) {
        int c0 = 0;
        if (act && ovf) {
            c0 = __ldg(M.cptr + v);
            d = __ldg(M.cptr + v + 1) - c0;
        }
        const int r0 = c0 + v;
        int nch = act && ovf ? (d + kEllW - 2) / (kEllW - 1) : 0;
        nch = __reduce_max_sync(kFull, nch);
        for (int ch = 0; ch < nch; ++ch) {
            const int base = ch * (kEllW - 1);
            const int ea = base + gl, ebb = base + gl + kGroup;
            const bool ha = act && ovf && ea <= d, hb = act && ovf && ebb <= d;
            const int ia = ha ? __ldg(M.ring + r0 + ea) & INT_MAX : 0;
            const int ib = hb ? __ldg(M.ring + r0 + ebb) & INT_MAX : 0;
            const bool cA = ha && atomicCAS(level + ia, -1, lvl) == -1;
            const bool cB = hb && atomicCAS(level + ib, -1, lvl) == -1;
            claim_records<T>(cA, ia, cB, ib, M, CC.s_list, CC.g_list, CC.g_cap, CC.ccnt, CC.err);
        }
    }
}

// Wide iterations: one band vertex per THREAD from its packed record (no
// shuffles, no idle corner slots, record bookkeeping once per vertex): the
// sequential strict-'<' fan scan of relax_vertex (update_kernel.hpp:93-120),
// corners evaluated two at a time.
// Wide relaxation, one vertex per thread, arranged for memory-level parallelism:
// trip 1 loads the position's vertex id AND its packed record's ring entries (both
// addressed by the position: slot s of p at s * N + p), trip 2 the neighbours' cells
// together with |x| and the corner quads of the d live slots only, then the corners are
// evaluated.  Wide iterations keep the Jacobi cells indexed by BFS position (the
// reorder_for_bands layout, toplesets.cpp:60-89): the packed ring entries are the
// neighbours' POSITIONS, so a warp over 32 consecutive positions gathers from a few
// runs of the adjacent toplesets instead of 32 x 7 scattered vertex ids, and its own
// cell loads and stores are coalesced.
// A position without a packed record (its first wide relaxation) reads its ring from
// the id-indexed ELL table, maps the ids to positions (posof) and writes the record
// once every neighbour has a position (the topleset after its own is positioned at the
// barrier that ends its first relaxation, and that flush is visible one iteration later).
#ifndef GEODIST_DYN_CHUNKS
#define GEODIST_DYN_CHUNKS 1
#endif
constexpr bool kDynChunks = GEODIST_DYN_CHUNKS != 0;

struct WidePre {
    int vr;
    int raw[kEllW];
};

// trip 1 of a wide position (issued one position ahead by the caller)
__device__ __forceinline__ void wide_pre(int p, size_t N, const int* pv, const int* pring,
                                         WidePre& w) {
    w.vr = ldcg(pv + p);
#pragma unroll
    for (int e = 0; e < kEllW; ++e) w.raw[e] = __ldcg(pring + ell_slot(e) * N + p);
}

// Change-driven (multi-source runs, whose cells carry change stamps; ptp_common.cuh
// Cell): the vertex is re-evaluated only over corners with an endpoint whose
// distance changed in the previous iteration (stamp kk - 1).  relax_vertex is a pure
// function of the neighbours' previous values and starts from the vertex's own
// previous value, which is already <= every candidate of an unchanged corner, so
// those corners can never be adopted (strict '<', update_kernel.hpp:114): skipping
// them gives the same bits as evaluating them.  A vertex with no changed corner
// keeps its value, and its cell is rewritten only if its value changed in this or
// the previous iteration: otherwise both buffers already hold the same cell.  relax_calls and
// degenerate_calls count every corner as the reference does: the degenerate test
// (update_kernel.hpp:51-57 on finite, unmixed corners) is a function of the flags
// and values already loaded.  |x| and the quads of the evaluated corners are loaded
// after the stamps (a third trip for those only: the 2048^2 height field's band does
// not fit L2, and the skipped loads are DRAM traffic).  Single-source runs evaluate
// every corner with |x| and quads loaded together with the distances.
template <typename T, bool LABELS, bool POS>
__device__ __forceinline__ void relax_wide2(const MeshDev& M, const RunArgs& A, int p, int kk,
                                            const WidePre& w, int* pv, int* pring, T* pL,
                                            char* pquad, const int* posof, int* dnext,
                                            const Cell<T, LABELS>* cp, Cell<T, LABELS>* cc,
                                            int fe, T eps, int& nonconv, T& my_max,
                                            long long& calls, long long& degs) {
    const T inf = Lim<T>::inf();
    const size_t N = static_cast<size_t>(A.stride);
    const int vr = w.vr;
    int raw[kEllW];
#pragma unroll
    for (int e = 0; e < kEllW; ++e) raw[e] = w.raw[e];
    const int v = vr & kIdMask;
    size_t pb = static_cast<size_t>(p), step = N;
    const T* lsrc = pL;
    const char* qsrc = pquad;
    unsigned unk = 0;  // entries whose neighbour has no position yet (+inf cells)
    if (!(vr & kPacked)) {
        pb = static_cast<size_t>(v) * kEllW;
        step = 1;
        lsrc = static_cast<const T*>(M.eL);
        qsrc = static_cast<const char*>(M.equad);
#pragma unroll
        for (int e = 0; e < kEllW; ++e) raw[e] = __ldcg(M.ering + pb + ell_slot(e));
        const int d0 = (raw[0] >> kMetaShift) & 15;
        if (POS && d0 != kEllOverflow) {
            int ps[kEllW];
#pragma unroll
            for (int e = 0; e < kEllW; ++e) ps[e] = e <= d0 ? ldcg(posof + (raw[e] & kIdMask)) : 0;
#pragma unroll
            for (int e = 0; e < kEllW; ++e) {
                if (ps[e] < 0) unk |= 1u << e;
                raw[e] = (raw[e] & ~kIdMask) | (ps[e] & kIdMask);
            }
            if (unk == 0) {
                // the packed record: ring entries as positions (flags kept), |x|, quads
#pragma unroll
                for (int e = 0; e < kEllW; ++e) {
                    const size_t dst = static_cast<size_t>(ell_slot(e)) * N + p;
                    const size_t src = pb + ell_slot(e);
                    pring[dst] = raw[e];
                    pL[dst] = ldcg(lsrc + src);
                    Quad<T> qq;
                    qq.load_cg(qsrc, src);
                    qq.store_at(pquad, dst);
                }
                bool dg = false;
#pragma unroll
                for (int c = 0; c < kEllW - 1; ++c) dg |= c < d0 && raw[c] < 0;
                pv[p] = v | kPacked | (dg ? kAlways : 0);
            }
        }
    } else if (POS) {
        // entries left unresolved by the first relaxation: resolved once their vertex
        // has a position (and written back), +inf cells until then
        unsigned unr = 0;
#pragma unroll
        for (int e = 0; e < kEllW; ++e) unr |= static_cast<unsigned>((raw[e] >> 30) & 1) << e;
        if (unr) {
#pragma unroll
            for (int e = 0; e < kEllW; ++e) {
                if (!((unr >> e) & 1u)) continue;
                raw[e] &= ~kUnres;
                const int ps = ldcg(posof + (raw[e] & kIdMask));
                if (ps >= 0) {
                    raw[e] = (raw[e] & ~kIdMask) | ps;
                    pring[static_cast<size_t>(ell_slot(e)) * N + p] = raw[e];
                } else {
                    unk |= 1u << e;
                }
            }
        }
    }
    constexpr bool kSkip = LABELS;
    const int sidx = POS ? p : v;  // this vertex's cell
    const Cell<T, LABELS> self = ld_cell(cp + sidx);
    const T tv = self.d;
    const int lv = self.lab();
    const int prevk = kk - 1;
    int d = (raw[0] >> kMetaShift) & 15;
    T best = tv;
    int blab = lv;
    const bool ovfl = d == kEllOverflow;
    if (ovfl) {
        // more than 7 corners: CSR tables, sequential fan walk, every corner evaluated
        const int c0 = __ldg(M.cptr + v);
        d = __ldg(M.cptr + v + 1) - c0;
        const int r0 = c0 + v;
        const T* ringL = static_cast<const T*>(M.ringL);
        auto cell_of = [&](int id) {
            const int q = POS ? ldcg(posof + id) : id;
            return q >= 0 ? ld_cell(cp + q) : make_cell<T, LABELS>(inf, -1, 0);
        };
        int x0 = __ldg(M.ring + r0);
        int i0 = x0 & INT_MAX;
        Cell<T, LABELS> n0 = cell_of(i0);
        T t0 = n0.d, L0 = __ldg(ringL + r0);
        int l0 = n0.lab();
        for (int c = 0; c < d; ++c) {
            const int x1 = __ldg(M.ring + r0 + c + 1);
            const int i1 = x1 & INT_MAX;
            const Cell<T, LABELS> n1 = cell_of(i1);
            const T t1 = n1.d, L1 = __ldg(ringL + r0 + c + 1);
            const int l1 = n1.lab();
            Quad<T> q;
            q.load(M.quad, c0 + c);
            const bool mixed = LABELS && l0 != l1 && t0 != inf && t1 != inf;
            int side, deg;
            const T val = corner_eval<T>(t0, t1, L0, L1, q, x0 < 0, mixed, side, deg);
            degs += deg;
            if (val < best) {
                best = val;
                if (LABELS) blab = side == 0 ? l0 : l1;
            }
            x0 = x1; i0 = i1; t0 = t1; L0 = L1; l0 = l1;
        }
    } else if (d > 0) {
        // fp32: every live quad is loaded with the distances (one trip); fp64: the quads
        // of a corner pair are loaded as the pair is reached (register budget)
        constexpr int kQ = sizeof(T) == 4 ? kEllW : 1;
        T t[kEllW + 1], L[kEllW];
        int l[kEllW + 1];
        bool ch[kEllW + 1];
        Quad<T> q[kQ];
#pragma unroll
        for (int e = 0; e <= kEllW; ++e) {
            t[e] = inf;
            l[e] = -1;
            ch[e] = false;
            if (e < kEllW) L[e] = T(0);
            if (e < kQ) q[e].q11 = q[e].q12 = q[e].q22 = q[e].a = T(0);
            if (e < kEllW && e <= d) {
                const Cell<T, LABELS> c = (unk >> e) & 1u ? make_cell<T, LABELS>(inf, -1, 0)
                                                          : ld_cell(cp + (raw[e] & kIdMask));
                t[e] = c.d;
                l[e] = c.lab();
                ch[e] = !kSkip || c.changed_at(prevk);
                // fp64: |x| and the quads are loaded per corner pair below (registers)
                if (!kSkip && sizeof(T) == 4) L[e] = ldcg(lsrc + pb + ell_slot(e) * step);
                if (!kSkip && sizeof(T) == 4 && e < kQ && e < d)
                    q[e].load_cg(qsrc, pb + ell_slot(e) * step);
            }
        }
        if (kSkip && sizeof(T) == 4) {
            // |x| and quads only for the corners that are evaluated (a third trip)
#pragma unroll
            for (int e = 0; e < kEllW; ++e) {
                const bool need_e = e <= d && ((e > 0 && (ch[e - 1] || ch[e])) ||
                                               (e < d && (ch[e] || ch[e + 1])));
                if (need_e) L[e] = ldcg(lsrc + pb + ell_slot(e) * step);
                if (e < kQ && e < d && (ch[e] || ch[e + 1])) q[e].load_cg(qsrc, pb + ell_slot(e) * step);
            }
        }
        // degenerate corners (rare): counted whether or not they are evaluated
        bool anydg = false;
#pragma unroll
        for (int c = 0; c < kEllW - 1; ++c) anydg |= c < d && raw[c] < 0;
        if (anydg) {
#pragma unroll
            for (int c = 0; c < kEllW - 1; ++c) {
                const bool mixed = LABELS && l[c] != l[c + 1] && t[c] != inf && t[c + 1] != inf;
                degs += (c < d && raw[c] < 0 && t[c] != inf && t[c + 1] != inf && !mixed) ? 1 : 0;
            }
        }
#pragma unroll
        for (int c = 0; c < kEllW - 1; c += 2) {
            if (c >= d) break;  // valence 6: three pairs, not four
            // corners c (entries c, c+1) and c+1 (entries c+1, c+2)
            const bool e0 = ch[c] || ch[c + 1];
            const bool e1 = c + 1 < d && (ch[c + 1] || ch[c + 2]);
            if (!(e0 || e1)) continue;
            const bool m0 = LABELS && l[c] != l[c + 1] && t[c] != inf && t[c + 1] != inf;
            const bool m1 = LABELS && l[c + 1] != l[c + 2] && t[c + 1] != inf && t[c + 2] != inf;
            T val[2];
            int side[2], deg[2];
            if constexpr (sizeof(T) == 4) {
                const float t1v[2] = {t[c], t[c + 1]}, t2v[2] = {t[c + 1], t[c + 2]};
                const float L1v[2] = {L[c], L[c + 1]};
                const float L2v[2] = {L[c + 1], c + 2 < kEllW ? L[c + 2] : 0.0f};
                const Quad<float> qv[2] = {q[c % kQ], q[(c + 1) % kQ]};
                const bool dgv[2] = {raw[c] < 0, raw[c + 1] < 0};
                const bool mix[2] = {m0, m1};
                const bool valid[2] = {e0, e1};
                corner_pair_f32(t1v, t2v, L1v, L2v, qv, dgv, mix, valid, val, side, deg);
            } else {
                val[0] = inf;
                val[1] = inf;
                side[0] = side[1] = -1;
                if (e0) {
                    Quad<T> q0;
                    q0.load_cg(qsrc, pb + ell_slot(c) * step);
                    const T L0 = ldcg(lsrc + pb + ell_slot(c) * step);
                    const T L1 = ldcg(lsrc + pb + ell_slot(c + 1) * step);
                    val[0] = corner_eval_f64<true>(t[c], t[c + 1], L0, L1, q0, raw[c] < 0, m0,
                                                   side[0], deg[0]);
                }
                if (e1) {
                    Quad<T> q1;
                    q1.load_cg(qsrc, pb + ell_slot(c + 1) * step);
                    const T L1 = ldcg(lsrc + pb + ell_slot(c + 1) * step);
                    const T L2 = ldcg(lsrc + pb + ell_slot(c + 2 < kEllW ? c + 2 : c + 1) * step);
                    val[1] = corner_eval_f64<true>(t[c + 1], t[c + 2], L1, L2, q1,
                                                   raw[c + 1] < 0, m1, side[1], deg[1]);
                }
            }
            if (e0 && val[0] < best) {
                best = val[0];
                if (LABELS) blab = side[0] == 0 ? l[c] : l[c + 1];
            }
            if (e1 && val[1] < best) {
                best = val[1];
                if (LABELS) blab = side[1] == 0 ? l[c + 1] : l[c + 2];
            }
        }
    }
    calls += d;
    if (worklist_for<T, LABELS>() && dnext != nullptr && best != tv) {
        // worklist marks for the next iteration: this vertex and its positioned neighbours
        // (in the id layout their positions from posof: a neighbour without one yet is the
        // next newest topleset, relaxed anyway)
        mark(dnext, p, kk);
        if (ovfl) {
            const int r0 = __ldg(M.cptr + v) + v;
            for (int e = 0; e <= d; ++e) {
                const int q = ld_c(posof + (__ldg(M.ring + r0 + e) & INT_MAX));
                if (q >= 0) mark(dnext, q, kk);
            }
        } else if (POS) {
#pragma unroll
            for (int e = 0; e < kEllW; ++e)
                if (e <= d && !((unk >> e) & 1u)) mark(dnext, raw[e] & kIdMask, kk);
        } else {
            int q[kEllW];
#pragma unroll
            for (int e = 0; e < kEllW; ++e) q[e] = e <= d ? ld_c(posof + (raw[e] & kIdMask)) : -1;
#pragma unroll
            for (int e = 0; e < kEllW; ++e)
                if (q[e] >= 0) mark(dnext, q[e], kk);
        }
    }
    // The other buffer holds this vertex's cell of two iterations ago: rewrite it only
    // if the value changed now or last iteration.
    if (!kSkip || best != tv || self.changed_at(prevk))
        st_cell(cc + sidx, make_cell<T, LABELS>(best, blab, best != tv ? kk : self.stamp()));
    if (best != tv && (p < fe || A.last_change != nullptr)) {
        const T rc = rel_change(tv, best);
        if (p < fe && rc >= eps) nonconv = 1;
        if (p < fe && rc > my_max) my_max = rc;
        if (A.last_change != nullptr && rc >= eps) A.last_change[v] = kk;
    }
}

}  // namespace

// MODE 0: every iteration (narrow bands through the record cache, wide ones one
// vertex per thread); MODE 1: narrow iterations only, MODE 2: wide only -- each
// exits (state saved in GroupCtl, mode_exit = the other mode) when the band
// crosses over, so each instantiation carries only its own path's registers.
template <typename T, bool LABELS, int MODE>
__global__ void __launch_bounds__(run4_block(MODE), 1) ptp_run4_kernel(RunArgs A) {
    constexpr int kB = run4_block(MODE);
    extern __shared__ __align__(16) unsigned char dsm[];
    __shared__ Bcast4 S;
    __shared__ T0State s_t0;
    __shared__ int s_lim[kLimRing];
    __shared__ int s_list[kSmemClaims];
    __shared__ T red_t[kB / 32];
    __shared__ long long red_l[kB / 32];
    __shared__ double red_v[kB / 32];
    __shared__ int red_i[kB / 32];
    __shared__ int s_ccnt, s_err;
    __shared__ int s_chunk;  // next older-band chunk of this CTA (wide iterations)
    __shared__ int s_qn, s_qh;  // worklist length / next batch (wide iterations)

    const int tid = threadIdx.x;
    constexpr int R = cache_slots<T>();
    constexpr int kNarrowMax = R - 1;
    // Wide iterations keep the cells by vertex id: with L1-cached gathers (and the wide-only
    // instantiation's shared memory given to L1) row-major neighbours share L1 lines (torus
    // fp32 12.7 ms vs 13.9 by position; fp64 14.6 ms vs 17.0 by position with the worklist).
    // GEODIST_POSL=1 puts fp64 single-source fields in the BFS-position layout (with
    // GEODIST_WL_MASK bit 2, the change-driven worklist), the round-2 alternative.
    constexpr bool kPosLayout = !LABELS && sizeof(T) == 8 && GEODIST_POSL;
    Cache<T> C;
    C.bind(dsm, R);
    const int nb = A.blocks_per_group;
    const int g = blockIdx.x / nb;
    const int lb = blockIdx.x - g * nb;
    GroupCtl* ctl = A.ctl + g;
    const long long off = static_cast<long long>(g) * A.stride;
    const long long off8 = off * kEllW;
    using CellT = Cell<T, LABELS>;
    CellT* cells[2] = {static_cast<CellT*>(A.cell0) + off, static_cast<CellT*>(A.cell1) + off};
    // the same double buffer indexed by BFS position (wide iterations)
    CellT* pcells[2] = {static_cast<CellT*>(A.pcell0) + off, static_cast<CellT*>(A.pcell1) + off};
    int* level = A.level + off;
    int* pv = A.queue + off;
    int* posof = A.posof + off;  // BFS position of a vertex (-1: not yet positioned)
    int* dflag = A.dflag + 2 * off;  // worklist marks by position, [parity][n]
    int* limits = A.limits + off;
    int* pring = A.pring + off8;
    T* pL = static_cast<T*>(A.pL) + off8;
    char* pquad = static_cast<char*>(A.pquad) + off8 * sizeof(Quad<T>);
    const MeshDev M = A.mesh;
    const int n = M.n;
    const T inf = Lim<T>::inf();
    const T eps = static_cast<T>(A.eps);
    const int gthreads = nb * kB;
    const int gtid = lb * kB + tid;
    unsigned long long* barw = ctl->barw;
    int* g_list = A.blists + static_cast<size_t>(blockIdx.x) * A.claim_cap;
    const ClaimCtx CC{s_list, g_list, A.claim_cap, &s_ccnt, &s_err};
    unsigned bseq = 0;
    const double inv_nb = 1.0 / nb;

    // Grid barrier with payload; thread 0 runs post(word) before the CTA is
    // released.  The arrival atomic returns the word as it was before this
    // CTA's arrival: its claim field is the number of claims of the CTAs that
    // arrived earlier, i.e. this CTA's offset inside the new topleset, and warp
    // 0 writes the CTA's claim list to those positions.  Readers of the new
    // positions (the owners, next iteration) wait for pv[p] >= 0.
    // The last CTA to arrive learns from its own atomic that the barrier is complete
    // (acq_rel: it also acquires every earlier arrival) and skips the polling trip.
    auto barrier = [&](unsigned long long payload, int level_start, auto&& pre, auto&& post,
                       bool presynced = false) {
        if (!presynced) __syncthreads();
        if (tid < 32) {
            unsigned long long* w = barw + (bseq & 3);
            unsigned long long old = 0;
            if (tid == 0) {
                // word (bseq+2)&3 was last polled at barrier bseq-2; every CTA has
                // arrived at bseq-1 since, so it is free until barrier bseq+2
                if (lb == 0) st_relaxed_u64(barw + ((bseq + 2) & 3), 0ull);
                old = atom_acq_rel_add_u64(w, payload + 1ull);
                pre();  // overlaps the arrival's round trip
            }
            const int cnt = static_cast<int>(payload >> 32);
            if (cnt > 0) {
                // claims beyond the lists' capacity were dropped (err 2: the field is
                // abandoned at this barrier and redone with larger lists); their
                // positions get vertex 0, an in-bounds placeholder
                const int at = level_start + static_cast<int>(__shfl_sync(kFull, old, 0) >> 32);
                for (int x = tid; x < cnt; x += 32) {
                    const bool kept = x < kSmemClaims || x - kSmemClaims < A.claim_cap;
                    const int id = x < kSmemClaims ? s_list[x]
                                   : kept          ? g_list[x - kSmemClaims]
                                                   : 0;
                    pv[at + x] = id;
                    if (kept) posof[id] = at + x;
                }
            }
            if (tid == 0) {
                unsigned long long x = old + payload + 1ull;
                if (static_cast<int>(x & 0xffffull) < nb) {
                    do {
                        x = ld_acquire_u64(w);
                    } while (static_cast<int>(x & 0xffffull) < nb);
                }
                post(x);
            }
        }
        ++bseq;
        __syncthreads();
    };

    // A CTA whose claim list overflowed (s_err 2) or whose new position was never
    // written (3) adds nb + 1 to the barrier word's nonconverged-CTA field (bits
    // 16-31, at most nb <= 255 otherwise): every CTA of the group then sees the
    // same word and ends the field (the host redoes it; the err reaches ctl->err).
    auto abort_bits = [&]() -> unsigned long long {
        return s_err >= 2 ? static_cast<unsigned long long>(nb + 1) << 16 : 0ull;
    };
    auto aborted = [&](unsigned long long x) {
        return static_cast<int>((x >> 16) & 0xffffull) > nb;
    };

    // reset the record cache tags (smem does not survive launches); the wide-only
    // instantiation has no record cache (and no dynamic shared memory unless its worklist
    // queue needs it: the rest goes to L1, which caches the cell gathers)
    if constexpr (MODE != 2)
        for (int x = tid; x < 4 * R; x += kB) C.pv[x] = make_int2(-1, 0);

    for (int q = g; q < A.nq; q += A.groups) {
        const int s0 = A.src_off ? A.src_off[q] : 0;
        const int m = A.src_off ? A.src_off[q + 1] - s0 : A.src_count;
        const int* src = A.src + s0;
        // thread-0 loop state (identical in every CTA of the group)
        // thread-0 loop state: only thread 0 touches it (barrier post / publish).  The
        // wide-only and the fp64 labelled instantiations keep it in shared memory (as
        // registers it is live in every thread: -5 % on the torus, and the fp64 labelled
        // narrow path spilled); the others in registers (it sits on the narrow
        // iteration's critical path: +3 % there from shared memory)
        T0State t0_local;
        T0State& t0 = [&]() -> T0State& {
            if constexpr (MODE == 2 || (sizeof(T) == 8 && LABELS)) return s_t0;
            else return t0_local;
        }();
        int &k = t0.k, &i = t0.i, &rho = t0.rho, &parity = t0.parity, &bfs_open = t0.bfs_open,
            &done = t0.done;
        int &tail = t0.tail, &bb = t0.bb, &fe = t0.fe, &frzb = t0.frzb,
            &frze = t0.frze;
        int& lim_top = t0.lim_top;    // highest topleset limit index held in s_lim
        bool& use_glim = t0.use_glim; // limits read from global memory (ring too short)
        unsigned long long& upd = t0.upd;
        if (tid == 0) {
            k = 0; i = 1; rho = INT_MAX; parity = 0; bfs_open = 0; done = 0;
            tail = 0; bb = 0; fe = 0; frzb = 0; frze = 0;
            lim_top = -1;
            use_glim = false;
            upd = 0;
        }
        auto lim = [&](int r) -> int {
            return (use_glim || r <= lim_top - kLimRing) ? ldcg(limits + r) : s_lim[r % kLimRing];
        };
        auto set_lim = [&](int r, int x) {
            s_lim[r % kLimRing] = x;
            if (r > lim_top) lim_top = r;
        };
        // this CTA's share of a position range: first owned position >= x and its
        // cache slot (x / nb via a double reciprocal, corrected), and the count of
        // owned positions in [x, y).  Thread 0 evaluates these while its barrier
        // arrival is in flight, for both outcomes of the convergence test.
        auto div_nb = [&](int x) {
            int qq = static_cast<int>(static_cast<double>(x) * inv_nb);
            if ((qq + 1) * nb <= x) ++qq;
            if (qq * nb > x) --qq;
            return qq;
        };
        auto first_owned = [&](int x, int& first, int& slot) {
            const int qx = div_nb(x), r = x - qx * nb;
            first = x + (lb >= r ? lb - r : lb - r + nb);
            slot = qx + (lb >= r ? 0 : 1);
        };
        auto owned_count = [&](int first, int y) { return y > first ? div_nb(y - first + nb - 1) : 0; };
        int &sh_p0 = t0.sh_p0, &sh_a0 = t0.sh_a0, &sh_f0 = t0.sh_f0, &sh_fa0 = t0.sh_fa0,
            &sh_nfz = t0.sh_nfz;
        int &sh_x0 = t0.sh_x0, &sh_xa0 = t0.sh_xa0;  // this CTA's first BFS task (next iteration)
        auto shares_now = [&] {
            first_owned(bb, sh_p0, sh_a0);
            first_owned(frzb, sh_f0, sh_fa0);
            sh_nfz = owned_count(sh_f0, frze);
            if (bfs_open) first_owned(lim(k + 2), sh_x0, sh_xa0);  // level k + 2's BFS tasks
        };
        int& be_pub = t0.be_pub;  // the band end publish() wrote to S.be (thread 0's copy)
        if (tid == 0) {
            be_pub = 0;
        }
        const bool tr0 = A.trace != nullptr && lb == 0;
        auto publish = [&] {
            S.done = done;
            S.tail = tail;
            s_ccnt = 0;
            s_chunk = 0;
            s_qn = 0;
            s_qh = 0;
            if (done) return;
            const int kk = k + 1;
            const int j = bfs_open ? kk : min(kk, rho - 1);
            S.k = kk;
            S.i = i;
            S.j = j;
            S.bb = bb;
            S.fe = fe;
            // the BFS runs one topleset ahead: levels through kk + 1 are positioned, so
            // the band end lim(j + 1) is always known (lim(rho) = tail once it closed)
            const int be = lim(j + 1);
            S.be = be;
            be_pub = be;
            S.oe = j == kk ? lim(j) : be;  // the topleset relaxed for the first time
            S.expand = bfs_open;
            // (sh_x0, sh_xa0) = first_owned(be): precomputed by thread 0 during the arrival
            S.xe = bfs_open ? tail : be;
            S.xp0 = bfs_open ? sh_x0 : be;  // no BFS tasks once the BFS has closed
            S.xa0 = sh_xa0;
            S.frzb = frzb;
            S.frze = frze;
            S.parity = parity;
            if (tr0) ctl->slot[(kk + 1) % 3] = 0ull;
            S.p0 = sh_p0;
            S.a0 = sh_a0;
            S.f0 = sh_f0;
            S.fa0 = sh_fa0;
            S.nfz = sh_nfz;
        };

        // BFS tasks of this CTA for the positions [xb, xe) (bfs4), claiming level `lvl`:
        // narrow (cachedv) -- owned positions xp0 + t * nb into cache slots xa0 + t, from the
        // top group down (the band's tasks fill the groups from the bottom up); wide -- chunks
        // of 32 consecutive positions, records packed (ring entries as positions when posm)
        auto bfs_loop = [&](bool cachedv, bool posm, int xb, int xe, int xp0, int xa0, int lvl) {
            constexpr int kGroupsB = kB / kGroup;
            for (int t = tid / kGroup;; t += kGroupsB) {
                const int tb = cachedv ? kGroupsB - 1 - tid / kGroup + (t - tid / kGroup) : t;
                const int p = cachedv ? xp0 + tb * nb
                                      : xb + (lb + (t / 32) * nb) * 32 + (t % 32);
                const bool act = p < xe;
                if (!__any_sync(kFull, act)) break;
                bool ca = false, cb = false;
                int ia = 0, ib = 0;
                bfs4<T>(M, A, C, (xa0 + tb) & (R - 1), act, cachedv, false, posm, p, lvl,
                        pv, posof, pring, pL, pquad, level, CC, ca, ia, cb, ib);
                claim_records<T>(ca, ia, cb, ib, M, CC.s_list, CC.g_list, CC.g_cap, CC.ccnt,
                                 CC.err);
            }
        };

        if (tid == 0) s_err = 0;
        if (MODE != 2 && q != g)
            for (int x = tid; x < 4 * R; x += kB) C.pv[x] = make_int2(-1, 0);
        if (A.phase_init) {
            // reset (ptp.cpp:61-68)
            for (int v = gtid; v < n; v += gthreads) {
                const CellT c = make_cell<T, LABELS>(inf, -1, 0);
                st_cell(cells[0] + v, c);
                st_cell(cells[1] + v, c);
                if (A.fused_bfs) {
                    level[v] = -1;
                    pv[v] = -1;  // position not yet assigned (claim_records)
                }
                posof[v] = -1;
                dflag[v] = 0;
                dflag[n + v] = 0;
                if (A.last_change) A.last_change[v] = 0;
            }
            if (gtid == 0) {
                ctl->relax = ctl->degen = ctl->updates = 0;
                ctl->slot[0] = ctl->slot[1] = ctl->slot[2] = 0ull;
                ctl->err = 0;
            }
            barrier(0ull, 0, [] {}, [](unsigned long long) {});
            // seed sources: d = 0, label = index in caller order (ptp.cpp:69-73)
            for (int s = gtid; s < m; s += gthreads) {
                const int v = src[s];
                const CellT c = make_cell<T, LABELS>(T(0), s, 0);
                st_cell(cells[0] + v, c);
                st_cell(cells[1] + v, c);
                if (A.fused_bfs) {
                    level[v] = 0;
                    pv[s] = v;
                    posof[v] = s;
                }
            }
            if (A.fused_bfs && gtid == 0) {
                limits[0] = 0;
                limits[1] = m;
            }
            if (!A.fused_bfs) {
                // caller ordering: every reachable vertex's position up front
                const int reach = ldcg(limits + A.given_rho);
                for (int p = gtid; p < reach; p += gthreads) posof[ldcg(pv + p) & kIdMask] = p;
            }
            if (tid == 0) s_ccnt = 0;
            barrier(0ull, 0, [] {}, [](unsigned long long) {});
            if (A.fused_bfs) {
                // iteration 0: claim topleset 1 from the sources (ring walk only)
                const int gl = tid & (kGroup - 1);
                for (int t = lb + nb * (tid / kGroup);; t += nb * (kB / kGroup)) {
                    const bool act = t < m;
                    if (!__any_sync(kFull, act)) break;
                    int v = 0, c0 = 0, d = 0;
                    if (act) {
                        v = ldcg(pv + t) & kIdMask;
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
                        claim_records<T>(cA, ia, cB, ib, M, CC.s_list, CC.g_list, CC.g_cap,
                                         CC.ccnt, CC.err);
                    }
                }
                __syncthreads();
                const unsigned long long cnt = static_cast<unsigned long long>(s_ccnt);
                barrier((cnt << 32) | abort_bits(), m, [] {}, [&](unsigned long long x) {
                    const int tot = static_cast<int>(x >> 32);
                    bb = m;
                    set_lim(0, 0);
                    set_lim(1, m);
                    if (tot == 0) {
                        bfs_open = 0;
                        rho = 1;
                        tail = m;
                        fe = m;
                    } else {
                        bfs_open = 1;
                        tail = m + tot;
                        fe = tail;
                        set_lim(2, tail);
                        if (lb == 0) limits[2] = tail;
                    }
                    done = (!bfs_open && i > rho - 1) || aborted(x);
                    shares_now();
                    // the BFS runs one topleset ahead: before iteration 1, claim level 2 from
                    // the positions of level 1 [m, tail) (publish follows the pre-pass)
                    S.done = done;
                    S.expand = bfs_open && !done;
                    S.xe = tail;
                    first_owned(m, sh_x0, sh_xa0);
                    S.xp0 = sh_x0;
                    S.xa0 = sh_xa0;
                    s_ccnt = 0;
                });
                if (S.expand) {
                    const bool cpre = MODE == 1 ||
                                      (MODE == 0 && A.wide_factor != 0 &&
                                       S.xe - m <= (R - 1) * nb);
                    bfs_loop(cpre, kPosLayout, m, S.xe, S.xp0, S.xa0, 2);
                    __syncthreads();
                    const unsigned long long c2 = static_cast<unsigned long long>(s_ccnt);
                    barrier((c2 << 32) | abort_bits(), S.xe, [] {}, [&](unsigned long long x) {
                        const int tot = static_cast<int>(x >> 32);
                        if (tot == 0) {
                            bfs_open = 0;
                            rho = 2;
                        } else {
                            tail += tot;
                            set_lim(3, tail);
                            if (lb == 0) limits[3] = tail;
                        }
                        done = aborted(x);
                        first_owned(lim(2), sh_x0, sh_xa0);  // iteration 1's BFS tasks: level 2
                        publish();
                    });
                } else {
                    if (tid == 0) publish();
                    __syncthreads();
                }
            } else {
                if (A.given_rho + 1 <= kLimRing) {
                    for (int r = tid; r <= A.given_rho; r += kB) s_lim[r] = ldcg(limits + r);
                }
                __syncthreads();
                if (tid == 0) {
                    rho = A.given_rho;
                    use_glim = rho + 1 > kLimRing;
                    lim_top = rho;
                    bfs_open = 0;
                    tail = lim(rho);
                    bb = lim(1);
                    fe = rho >= 2 ? lim(2) : tail;
                    done = i > rho - 1;
                    shares_now();
                    publish();
                }
                __syncthreads();
            }
        } else {
            // resume a run stopped by max_iters or a mode switch: state from ctl, the
            // limits ring reloaded from global memory.  A launch of a fixed launch
            // sequence (FPS rounds, batched fields) whose field is already complete
            // has nothing to do (every CTA reads the same ctl).
            if (__ldcg(&ctl->done)) return;
            const int top = ctl->bfs_open ? ctl->k + 3 : ctl->rho;  // BFS one topleset ahead
            const int lo = top - kLimRing + 1 > 0 ? top - kLimRing + 1 : 0;
            for (int r = lo + tid; r <= top; r += kB) s_lim[r % kLimRing] = ldcg(limits + r);
            __syncthreads();
            if (tid == 0) {
                k = ctl->k; i = ctl->i; rho = ctl->rho; parity = ctl->parity;
                bfs_open = ctl->bfs_open; done = ctl->done;
                tail = ctl->s_tail; bb = ctl->s_bb; fe = ctl->s_fe;
                frzb = ctl->s_frzb; frze = ctl->s_frze;
                lim_top = top;
                shares_now();
                publish();
            }
            __syncthreads();
        }

        // Cell layout: narrow iterations index the double buffer by vertex id (the record
        // cache holds ring ids), wide ones by BFS position (pcells; packed ring entries
        // are positions).  Every launch starts and ends in the id layout; crossing over
        // is one pass over the positions assigned so far, both buffers, and a barrier.
        int layout = 0;
        bool fresh = false, was_wide = false;

        auto relayout = [&](int to) {
            const int top = S.tail;
            const CellT none = make_cell<T, LABELS>(inf, -1, 0);
            for (int x = gtid; x < n; x += gthreads) {
                // a position flushed at the last barrier may not be visible yet (-1): its
                // vertex has not been relaxed, +inf in both layouts
                const int id = x < top ? ldcg(pv + x) : -1;
                const int v = id & kIdMask;
                if (to == 1) {
                    st_cell(pcells[0] + x, id >= 0 ? ld_cell(cells[0] + v) : none);
                    st_cell(pcells[1] + x, id >= 0 ? ld_cell(cells[1] + v) : none);
                } else if (id >= 0) {
                    st_cell(cells[0] + v, ld_cell(pcells[0] + x));
                    st_cell(cells[1] + v, ld_cell(pcells[1] + x));
                }
            }
            // wide iterations reuse the record cache's shared memory as the worklist queue
            if (to == 0 && kPosLayout && worklist_for<T, LABELS>())
                for (int x = tid; x < 4 * R; x += kB) C.pv[x] = make_int2(-1, 0);
            barrier(0ull, 0, [] {}, [](unsigned long long) {});
            layout = to;
            fresh = to == 1;  // no marks yet: the first wide iteration relaxes every position
        };

        long long calls = 0, degs = 0;
        int iters = 0;
        int mode_exit = 0;
        for (;;) {
            if (S.done || (A.max_iters > 0 && iters >= A.max_iters)) break;
            if constexpr (MODE != 0) {
                const int span = S.xe - S.bb;  // the band and the BFS tasks' topleset
                const bool wide = A.wide_factor == 0 || span > kNarrowMax * nb;
                if (MODE == 1 && wide) {
                    mode_exit = 2;
                    break;
                }
                if (MODE == 2 && A.wide_factor != 0 && 2 * span <= kNarrowMax * nb) {
                    mode_exit = 1;  // narrow again (with hysteresis)
                    break;
                }
            }
            const int kk = S.k;
            const bool dbg = A.dbg != nullptr && tid == 0 && S.k - 1 < A.dbg_iters;
            unsigned long long* dslot =
                dbg ? A.dbg + kDbgSlots * (static_cast<size_t>(S.k - 1) * gridDim.x + blockIdx.x) : nullptr;
            if (dbg) {
                dslot[0] = gtimer();
                dslot[18] = 0;
            }
            const unsigned long long it0 = A.dbg != nullptr ? cyc() : 0ull;
            const int prv = S.parity, cur_b = prv ^ 1;
            const int bb_ = S.bb, be_ = S.be, fe_ = S.fe, oe_ = S.oe;
            // BFS tasks: positions [be, xe) (the topleset after the band's newest)
            const int xe_ = S.xe, xp0_ = S.xp0, xa0_ = S.xa0;
            // GEODIST_WIDE=0 (wide_factor 0) forces the wide path (tests)
            const bool cached = MODE == 1   ? true
                                : MODE == 2 ? false
                                            : A.wide_factor != 0 && (xe_ - bb_) <= kNarrowMax * nb;
            // single-source fields relax wide bands in the position layout; labelled ones
            // keep the id layout (measured: the 2048^2 height field's band does not fit L2,
            // and its row-major ids give each vertex's gathers shared sectors)
            const bool posl = kPosLayout && !cached;
            if ((posl ? 1 : 0) != layout) relayout(posl ? 1 : 0);
            const CellT* cp = posl ? pcells[prv] : cells[prv];
            CellT* ccur = posl ? pcells[cur_b] : cells[cur_b];
            // records are also packed by the BFS tasks of narrow iterations once the band
            // approaches the record cache's capacity, ready for the wide path
            const bool pack = 2 * (xe_ - bb_) > kNarrowMax * nb;
            int* dnext = (!cached && worklist_for<T, LABELS>()) ? dflag + ((kk + 1) & 1) * n : nullptr;
            // the first wide iteration after narrow ones has no marks: it relaxes every position;
            // narrow ones after wide ones (combined instantiation, id layout) find the record
            // cache's memory used as the worklist queue: its tags are reset
            if (!cached && !was_wide) fresh = true;
            if constexpr (worklist_for<T, LABELS>() && !kPosLayout) {
                if (cached && was_wide) {
                    for (int x = tid; x < 4 * R; x += kB) C.pv[x] = make_int2(-1, 0);
                    __syncthreads();
                }
            }
            was_wide = !cached;
            // owned positions: band task t at p0 + t * nb; the frozen topleset's
            // positions go to the groups from the top of the CTA down
            const int p0 = S.p0, a0 = S.a0;
            const int f0 = S.f0, fa0 = S.fa0, nfz = S.nfz;
            int nonconv = 0;
            T my_max = T(0);
            constexpr int kGroups = kB / kGroup;
            // Wide iterations (fp32): positions are dealt to CTAs in chunks of 32
            // consecutive positions (chunk c -> CTA c mod nb) instead of one by one, so
            // a warp works on 32 neighbouring positions: their records are adjacent and,
            // since a CTA's claims come from its own chunks, their neighbours' distances
            // share sectors.  The newest topleset keeps the 4-lane groups (BFS claims),
            // the older ones are relaxed one vertex per thread.
            constexpr int kChunk = 32;
            const bool wchunk = !cached;
            if (!wchunk) {
            for (int t = tid / kGroup, tf = kGroups - 1 - tid / kGroup;; t += kGroups, tf += kGroups) {
                const bool act = p0 + t * nb < be_;
                const bool frz = tf < nfz;
                const bool bact = xp0_ + tf * nb < xe_;  // BFS tasks from the top group down
                if (!__any_sync(kFull, act || frz || bact)) break;
                const int p = p0 + t * nb;
                bool ca = false, cb = false;
                int ia = 0, ib = 0;
                if (__any_sync(kFull, bact)) {
                    bfs4<T>(M, A, C, (xa0_ + tf) & (R - 1), bact, true, pack,
                            kPosLayout, xp0_ + tf * nb, kk + 2, pv, posof, pring, pL, pquad,
                            level, CC, ca, ia, cb, ib);
                    claim_records<T>(ca, ia, cb, ib, M, CC.s_list, CC.g_list, CC.g_cap,
                                     CC.ccnt, CC.err);
                }
                unsigned long long* kd =
                    (A.dbg != nullptr && S.k - 1 < A.dbg_iters && act && p >= oe_ && p - nb < oe_ &&
                     (tid & (kGroup - 1)) == 0)
                        ? A.dbg + kDbgSlots * (static_cast<size_t>(S.k - 1) * gridDim.x + blockIdx.x)
                        : nullptr;
                if (__any_sync(kFull, act))
                    relax4<T, LABELS>(M, A, C, (a0 + t) & (R - 1), act, p, kk, pv, cp,
                                      ccur, fe_, eps, nonconv, my_max, calls, degs,
                                      (dbg && t == 0) ? dslot : nullptr);
                if (kd) kd[9] = cyc() - it0;
                if (frz && (tid & (kGroup - 1)) == 0) {
                    // deferred freeze of the topleset retired last iteration (ptp.cpp:121-130)
                    const int fp = f0 + tf * nb;
                    const int2 tg = C.pv[((fa0 + tf) & (R - 1)) * 4];
                    const int v = tg.x == fp ? tg.y : (ldcg(pv + fp) & kIdMask);
                    st_cell(ccur + v, ld_cell(cp + v));
                }
            }
            } else {
            // worklist queue in the record cache's memory, structure of arrays: position,
            // position word, the 8 packed ring entries (40 B per queued position)
            constexpr int kQEnt = 10 * sizeof(int);
            const int qcap = static_cast<int>(R * Cache<T>::bytes_per_slot() / kQEnt);
            int* wq_p = reinterpret_cast<int*>(dsm);
            int* wq_v = wq_p + qcap;
            int* wq_r = wq_v + qcap;  // entry e of queued position x at wq_r[e * qcap + x]
            // this CTA's older positions: chunks lb, lb + nb, ... of 32 from bb up to oe
            const int span0 = be_ - bb_ - lb * kChunk;
            const int nch = span0 > 0 ? (span0 + nb * kChunk - 1) / (nb * kChunk) : 0;
            const int total = nch * kChunk;
            // (a CTA share beyond the queue's capacity relaxes every position this iteration)
            const bool wl = worklist_for<T, LABELS>() && total <= qcap;
            if (wl) {
                // Change-driven worklist (position layout).  relax_vertex is a pure function
                // of the neighbours' previous values and starts from the vertex's own previous
                // value, which is <= every candidate it already evaluated: a position none of
                // whose neighbours (nor itself) changed in the previous iteration would
                // recompute exactly its value, and both buffers already hold it (it was
                // rewritten when it last changed, or relaxed unchanged).  Skipping it is
                // bit-identical (update_kernel.hpp:93-120, ptp.cpp:96-110): its relative
                // change is 0, its corners are still counted (relax_calls, from the record's
                // corner count), and a vertex with a degenerate corner is never skipped
                // (kAlways).  Changed vertices mark themselves and their neighbours (mark());
                // the first wide iteration after a layout switch relaxes everything.
                // The CTA scans all its older positions at once -- one trip: position word,
                // mark and packed ring entries (trip 1 of the relaxation) -- and queues the
                // marked ones with their ring entries in shared memory; relaxing a queued
                // position is then one trip (neighbour cells, |x|, quads).
                const int* dcur = dflag + (kk & 1) * n;
                const int lane = tid & 31;
                const unsigned lt = (1u << lane) - 1u;
                const size_t N = static_cast<size_t>(A.stride);
                constexpr int kU = 4;
                for (int t0 = 0; t0 < total; t0 += kB * kU) {
                    int vr[kU], df[kU], pp[kU], rw[kU][kEllW];
#pragma unroll
                    for (int u = 0; u < kU; ++u) {
                        const int t = t0 + u * kB + tid;
                        pp[u] = bb_ + (lb + (t / kChunk) * nb) * kChunk + (t % kChunk);
                        vr[u] = df[u] = 0;
#pragma unroll
                        for (int e = 0; e < kEllW; ++e) rw[u][e] = 0;
                        if (t < total && pp[u] < be_) {
                            vr[u] = ldcg(pv + pp[u]);
                            df[u] = ldcg(dcur + pp[u]);
#pragma unroll
                            for (int e = 0; e < kEllW; ++e)
                                rw[u][e] = __ldcg(pring + ell_slot(e) * N + pp[u]);
                        }
                    }
#pragma unroll
                    for (int u = 0; u < kU; ++u) {
                        const int t = t0 + u * kB + tid;
                        const bool in = t < total && pp[u] < be_;
                        // the band's newest topleset is relaxed for the first time
                        const bool dirty = in && (fresh || pp[u] >= oe_ || !(vr[u] & kPacked) ||
                                                  (vr[u] & kAlways) || df[u] == kk);
                        if (in && !dirty) calls += (rw[u][0] >> kMetaShift) & 7;
                        const unsigned bal = __ballot_sync(kFull, dirty);
                        int at = 0;
                        if (lane == 0 && bal) at = atomicAdd(&s_qn, __popc(bal));
                        at = __shfl_sync(kFull, at, 0) + __popc(bal & lt);
                        if (dirty) {
                            wq_p[at] = pp[u];
                            wq_v[at] = vr[u];
#pragma unroll
                            for (int e = 0; e < kEllW; ++e) wq_r[e * qcap + at] = rw[u][e];
                        }
                    }
                }
                __syncthreads();
            }
            for (int t = tid / kGroup, tf = kGroups - 1 - tid / kGroup;; t += kGroups, tf += kGroups) {
                // BFS tasks here (the topleset after the band's newest, records packed),
                // the band one vertex per thread below (relax_wide2)
                const int p = be_ + (lb + (t / kChunk) * nb) * kChunk + (t % kChunk);
                const bool act = p < xe_;
                const bool frz = tf < nfz;
                if (!__any_sync(kFull, act || frz)) break;
                bool ca = false, cb = false;
                int ia = 0, ib = 0;
                if (__any_sync(kFull, act)) {
                    bfs4<T>(M, A, C, 0, act, false, false, kPosLayout, p, kk + 2, pv, posof,
                            pring, pL, pquad, level, CC, ca, ia, cb, ib);
                    claim_records<T>(ca, ia, cb, ib, M, CC.s_list, CC.g_list, CC.g_cap,
                                     CC.ccnt, CC.err);
                }
                if (frz && (tid & (kGroup - 1)) == 0) {
                    // deferred freeze of the topleset retired last iteration (ptp.cpp:121-130)
                    const int fp = f0 + tf * nb;
                    const int fv = kPosLayout ? fp : (ldcg(pv + fp) & kIdMask);
                    st_cell(ccur + fv, ld_cell(cp + fv));
                }
            }
            if (dbg) {
                dslot[17] = gtimer();
                dslot[18] = wchunk ? 1 : 0;
            }
            {
                // older band positions [bb, oe): one vertex per thread, chunked.  Warps
                // take this CTA's chunks from a shared counter, so the warps that held the
                // BFS tasks (the longest chain) take fewer.
                // Chunk m of this CTA starts at position bb + (lb + m * nb) * 32; task t
                // below is chunk * 32 + lane.
                const int lane = tid & 31;
                auto grab = [&]() {
                    int m = 0;
                    if (kDynChunks) {
                        if (lane == 0) m = atomicAdd(&s_chunk, 1);
                        m = __shfl_sync(kFull, m, 0);
                    }
                    return m;
                };
                auto pos = [&](int t) { return bb_ + (lb + (t / kChunk) * nb) * kChunk + (t % kChunk); };
                // next task of this thread: the static deal (t + blockDim) or a fresh chunk
                auto next_t = [&](int t) { return kDynChunks ? grab() * kChunk + lane : t + kB; };
                    // software-pipelined: trip 1 of the next position is in flight while
                    // this one's distances are gathered and its corners evaluated
                    // (not with labels: the second record in flight spills registers)
                    const size_t N = static_cast<size_t>(A.stride);
                    if (wl) {
                        // the worklist built by the scan above: batches of 32 queued positions,
                        // one per thread, trip 1 of the next batch in flight during this one
                        const int qn = s_qn;
                        auto grabq = [&]() {
                            int h = 0;
                            if (lane == 0) h = atomicAdd(&s_qh, 32);
                            return __shfl_sync(kFull, h, 0);
                        };
                        while (true) {
                            const int h = grabq();
                            if (h >= qn) break;
                            if (h + lane < qn) {
                                const int x = h + lane;
                                WidePre w;
                                w.vr = wq_v[x];
#pragma unroll
                                for (int e = 0; e < kEllW; ++e) w.raw[e] = wq_r[e * qcap + x];
                                relax_wide2<T, LABELS, kPosLayout>(M, A, wq_p[x], kk, w, pv, pring,
                                                                   pL, pquad, posof, dnext, cp,
                                                                   ccur, fe_, eps, nonconv, my_max,
                                                                   calls, degs);
                            }
                        }
                    } else {
                    int t = kDynChunks ? grab() * kChunk + lane : tid;
                    int p = pos(t);
                    WidePre nx;
                    if constexpr (LABELS || sizeof(T) == 8) {
                        for (;; t = next_t(t)) {
                            p = pos(t);
                            if (p - (t % kChunk) >= be_) break;
                            if (p < be_) {
                                wide_pre(p, N, pv, pring, nx);
                                relax_wide2<T, LABELS, kPosLayout>(M, A, p, kk, nx, pv, pring, pL, pquad,
                                                       posof, dnext, cp, ccur, fe_, eps, nonconv,
                                                       my_max, calls, degs);
                            }
                        }
                    } else {
                    if (p - (t % kChunk) < be_ && p < be_) wide_pre(p, N, pv, pring, nx);
                    while (p - (t % kChunk) < be_) {
                        const WidePre cw = nx;
                        const int pc = p;
                        t = next_t(t);
                        p = pos(t);
                        if (p - (t % kChunk) < be_ && p < be_) wide_pre(p, N, pv, pring, nx);
                        if (pc < be_)
                            relax_wide2<T, LABELS, kPosLayout>(M, A, pc, kk, cw, pv, pring, pL, pquad, posof,
                                                   dnext, cp, ccur, fe_, eps, nonconv, my_max, calls,
                                                   degs);
                    }
                    }
                    }
            }
            }
            if (dbg) dslot[7] = cyc();
            fresh = false;
            nonconv = __syncthreads_or(nonconv);
            if (A.trace != nullptr) {
                const T bmax = block_max(my_max, red_t);
                if (tid == 0 && bmax > T(0)) atomicMax(&ctl->slot[kk % 3], Lim<T>::bits(bmax));
            }
            if (dbg) dslot[1] = gtimer();
            const unsigned long long pay = (nonconv ? (1ull << 16) : 0ull) | abort_bits() |
                                           (static_cast<unsigned long long>(s_ccnt) << 32);
            int c_p0 = 0, c_a0 = 0, n_p0 = 0, n_a0 = 0, c_nfz = 0;
            barrier(pay, xe_, [&] {  // claims: the topleset starting at xe
                first_owned(fe, c_p0, c_a0);  // converged: the band starts at fe
                first_owned(bb, n_p0, n_a0);  // not converged: it stays at bb
                first_owned(tail, sh_x0, sh_xa0);  // next BFS tasks start at the current tail
                c_nfz = owned_count(n_p0, fe);  // converged: [bb, fe) is frozen next
            }, [&](unsigned long long x) {
                if (dbg) dslot[2] = gtimer();
                const int nnc = static_cast<int>((x >> 16) & 0xffffull);  // <= nb unless aborted
                const int tot = static_cast<int>(x >> 32);
                const bool conv = nnc == 0;  // ptp.cpp:114
                const int ub = bb, ue = be_pub;
                upd += static_cast<unsigned long long>(ue - ub);
                if (tr0) {
                    const int row = kk - A.trace_k0;
                    if (row >= 0 && row < A.trace_cap) {
                        TraceRow r;
                        r.k = kk; r.i = i; r.j = S.j; r.conv = conv ? 1 : 0;
                        r.updated = ue - ub;
                        r.max_rel = static_cast<double>(
                            Lim<T>::from_bits(__ldcg(&ctl->slot[kk % 3])));
                        A.trace[row] = r;
                    }
                }
                // the claims of this iteration are level kk + 2 (one topleset ahead)
                int nt = tail;
                if (bfs_open) {
                    if (tot == 0) {
                        bfs_open = 0;
                        rho = kk + 2;
                    } else {
                        nt = tail + tot;
                        set_lim(kk + 3, nt);
                        if (lb == 0) limits[kk + 3] = nt;
                    }
                }
                if (conv) {
                    frzb = bb;
                    frze = fe;
                    bb = fe;
                    fe = (bfs_open || i + 2 <= rho) ? lim(i + 2) : nt;
                    ++i;
                    sh_p0 = c_p0; sh_a0 = c_a0; sh_f0 = n_p0; sh_fa0 = n_a0; sh_nfz = c_nfz;
                } else {
                    frzb = frze = 0;
                    sh_p0 = n_p0; sh_a0 = n_a0; sh_nfz = 0;
                }
                tail = nt;
                parity ^= 1;
                k = kk;
                done = (!bfs_open && i > rho - 1) || aborted(x);
                publish();
                if (dbg) dslot[8] = gtimer();
            }, true);
            ++iters;
        }

        if (layout != 0) relayout(0);  // launches end in the id layout
        // per-query statistics
        const long long bc = block_sum(calls, red_l);
        const long long bd = block_sum(degs, red_l);
        if (tid == 0) {
            if (bc) atomicAdd(&ctl->relax, static_cast<unsigned long long>(bc));
            if (bd) atomicAdd(&ctl->degen, static_cast<unsigned long long>(bd));
            if (s_err) atomicMax(&ctl->err, s_err);
            if (lb == 0) {
                ctl->k = k; ctl->i = i; ctl->rho = rho; ctl->parity = parity;
                ctl->bfs_open = bfs_open; ctl->done = done;
                ctl->mode_exit = mode_exit;
                ctl->s_tail = tail; ctl->s_bb = bb; ctl->s_fe = fe;
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
            const CellT* cf = cells[fin];
            const long long qo = static_cast<long long>(q) * n;
            for (int v = gtid; v < n; v += gthreads) {
                const CellT cx = ld_cell(cf + v);
                const T x = cx.d;
                if (A.out_dist != nullptr) {
                    if (A.out_double)
                        static_cast<double*>(A.out_dist)[qo + v] = static_cast<double>(x);
                    else
                        static_cast<float*>(A.out_dist)[qo + v] = static_cast<float>(x);
                }
                if (A.out_labels != nullptr)
                    A.out_labels[qo + v] = cx.lab();
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
                for (int w = 1; w < kB / 32; ++w)
                    if (red_v[w] > vmax || (red_v[w] == vmax && red_i[w] < vidx)) {
                        vmax = red_v[w];
                        vidx = red_i[w];
                    }
                A.fps_scratch[2 * blockIdx.x] =
                    static_cast<unsigned long long>(__double_as_longlong(vmax));
                A.fps_scratch[2 * blockIdx.x + 1] = static_cast<unsigned long long>(vidx);
            }
        }
        barrier(0ull, 0, [] {}, [&](unsigned long long) {
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
            const int e = __ldcg(&ctl->err);
            st.pad = e >= 2 ? e : 0;  // 2: claim list overflow, 3: position never written
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

// ---------------------------------------------------------------------------
// host side

size_t run4_dyn_smem(int precision, bool labels, int mode) {
    const size_t cache = precision == 0 ? cache_slots<float>() * Cache<float>::bytes_per_slot()
                                        : cache_slots<double>() * Cache<double>::bytes_per_slot();
    if (mode == 2) {  // wide-only: the worklist queue (record cache memory) or nothing
        const bool wl = precision == 0 ? (labels ? worklist_for<float, true>()
                                                 : worklist_for<float, false>())
                                       : (labels ? worklist_for<double, true>()
                                                 : worklist_for<double, false>());
        return wl ? cache : 0;
    }
    return cache;
}

template <int MODE> static const void* run4_ptr(int precision, bool labels) {
    if (precision == 0)
        return labels ? reinterpret_cast<const void*>(&ptp_run4_kernel<float, true, MODE>)
                      : reinterpret_cast<const void*>(&ptp_run4_kernel<float, false, MODE>);
    return labels ? reinterpret_cast<const void*>(&ptp_run4_kernel<double, true, MODE>)
                  : reinterpret_cast<const void*>(&ptp_run4_kernel<double, false, MODE>);
}

const void* run4_kernel_ptr(int precision, bool labels, int mode) {
    return mode == 1 ? run4_ptr<1>(precision, labels)
                     : mode == 2 ? run4_ptr<2>(precision, labels) : run4_ptr<0>(precision, labels);
}

}  // namespace gdb
