// Device-side types and helpers of the B200 PTP solver (sm_100a).
//
// Data layout in HBM (per mesh, built once by pack_fans_kernel):
//   cptr[n+1]            corner offsets, original vertex order (int32)
//   ring[cptr[n]+n]      fan ring per vertex at cptr[v]+v: r_0..r_d (int32);
//                        corner c of v is (ring[c], ring[c+1]); bit 31 of
//                        ring[cptr[v]+v+c] flags corner c as degenerate
//                        (update_kernel.hpp:51-57 test precomputed)
//   ringL<T>[..]         |x| = sqrt(dot(x,x)) per ring entry, x = p[r]-p[v] in T
//   quad<T>[4*cptr[n]]   per corner {q11, q12, q22, a} of the Gram inverse
//                        (update_kernel.hpp:55-60), computed in T with the
//                        reference's operation order (no FMA)
// Per query (per group of CTAs):
//   cell0/cell1[n]       Jacobi double buffer (ptp.cpp:61-63), original order:
//                        Cell<T, LABELS> = distance (+ nearest-source label for
//                        multi-source runs) + change stamp (ptp_common.cuh)
//   level[n]             BFS level (-1 = unvisited), fused topleset discovery
//   pcell0/pcell1[n]     the double buffer indexed by BFS position (wide iterations)
//   queue[n]             vertices in BFS order, level r at [limits[r], limits[r+1])
//   posof[n]             inverse of queue (-1: vertex not yet positioned)
//   limits[n+2]
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace gdb {

constexpr int kBlock = 512;        // threads per CTA
#ifndef GEODIST_WIDE_BLOCK
#define GEODIST_WIDE_BLOCK 512
#endif
// threads per CTA of the wide-only v4 instantiation (a build knob: 640 / 768 threads
// cap registers at 96 / 80 and the spills cost 8 % / 24 % on the torus, measured)
constexpr int kWideBlock = GEODIST_WIDE_BLOCK;
__host__ __device__ constexpr int run4_block(int mode) { return mode == 2 ? kWideBlock : kBlock; }
constexpr int kW = 8;              // lanes per vertex in the BFS-only kernel
constexpr int kGroup = 4;          // lanes per vertex in the solver: 2 ring entries per lane
constexpr int kEllW = 8;           // ELL slot: 8 ring entries (<= 7 corners) per vertex
constexpr int kMetaShift = 27;     // entry 0 bits 27..30 hold the corner count d
constexpr int kIdMask = (1 << kMetaShift) - 1;
constexpr int kEllOverflow = 15;   // d code: more than 7 corners, use the CSR tables
constexpr unsigned kFull = 0xffffffffu;
constexpr int kWideFactor = 2;     // RunArgs.wide_factor default (GEODIST_WIDE=0 forces the
                                   // wide path on every iteration: tests)

// ELL entry e of a vertex lives at slot (e % 4) * 2 + e / 4, so lane l of a
// 4-lane group reads entries l and l + 4 as one 8-byte (or 16-byte) vector.
__host__ __device__ constexpr int ell_slot(int e) { return (e & 3) * 2 + (e >> 2); }

// One group of CTAs runs one query; its control block lives in global memory.
// Hot words sit on separate 128-byte lines.
struct alignas(128) GroupCtl {
    unsigned int bar;              // barrier arrivals (monotonic within a launch)
    unsigned int pad0[31];
    unsigned long long slot[3];    // per-iteration max relative change (bit pattern)
    unsigned long long pad1[13];
    int tail;                      // BFS queue tail (= limits[top+1])
    int err;
    int pad2[30];
    // loop state, saved by CTA 0 of the group when a launch ends mid-run
    int k, i, rho, parity, mode_exit, bfs_open, done, initialized;  // mode_exit: v4 kernel to resume with
    int s_tail, s_limk, s_bb, s_fe, s_frzb, s_frze, pad3[2];
    unsigned long long relax, degen, updates;
    unsigned long long pad4[5];
    // v4 barrier words (ring of 4): bits 0-15 arrivals, 16-31 CTAs with a front
    // change >= eps, 32-63 claims made in the iteration
    unsigned long long barw[4];
    unsigned long long pad5[12];
    // FPS / argmax scratch: per-CTA (value bits, index)
};

struct QueryStats {  // per query, written by CTA 0 of the group
    long long relax, degen, updates;
    int iterations, rho, unreached, done;
    double radius;
    int argmax, pad;
};

struct TraceRow {  // mirrors geodist_band_row
    int k, i, j, conv;
    long long updated;
    double max_rel;
};

struct MeshDev {
    const int* cptr;   // CSR (overflow vertices, BFS seeding)
    const int* ring;   // CSR ring with degenerate flags for this precision
    const void* ringL;
    const void* quad;
    const int* ering;  // ELL-8 ring (interleaved, meta in entry 0)
    const void* eL;    // ELL-8 |x|
    const void* equad; // ELL-8 Gram inverse quads
    int n;
};

struct RunArgs {
    MeshDev mesh;
    // per-group buffers: group g at base + g * stride (elements)
    void* cell0;         // Cell<T, LABELS>[stride] per group
    void* cell1;
    void* pcell0;        // the same cells indexed by BFS position (wide iterations)
    void* pcell1;
    int* posof;          // BFS position of each vertex, -1 before it is positioned
    int* dflag;          // 2 x stride per group: relaxation marks by position (parity k & 1)
    int* level;
    int* queue;
    int* limits;
    long long stride;
    GroupCtl* ctl;
    int groups;
    int blocks_per_group;
    // queries
    const int* src;      // concatenated sources (caller order)
    const int* src_off;  // nq+1 offsets, or NULL with src_count
    int src_count;       // sources of query 0 when src_off == NULL (FPS round)
    int nq;
    double eps;
    int fused_bfs;       // 0: queue/limits preloaded (caller ordering), rho = given_rho
    int given_rho;
    int phase_init;      // start a fresh query (else resume from ctl state)
    int max_iters;       // iterations per launch (<= 0: run to completion)
    // diagnostics
    TraceRow* trace;     // rows indexed by (k - trace_k0), capacity trace_cap
    int trace_k0;
    int trace_cap;
    int* last_change;    // n, or NULL
    // outputs (query q at + q*n)
    void* out_dist;
    int out_double;      // out_dist element: 1 double, 0 float
    int* out_labels;     // or NULL
    QueryStats* qstats;  // nq rows
    // FPS: argmax over the final field, appended to src[src_count]
    int fps_mode;
    unsigned long long* fps_scratch;  // 2 * gridDim.x words
    int* fps_samples;                 // device sample list (== src)
    int fps_final;
    // optional per-iteration timestamps (globaltimer ns): [iter][cta][3] =
    // (work start, work end after the CTA reduction, barrier release)
    unsigned long long* dbg;
    int dbg_iters;
    // packed records by BFS position (slot-major: slot s of position p at s * stride + p)
    int* pring;          // 8 ints per position (ELL interleaved)
    void* pL;            // 8 T per position
    void* pquad;         // 8 Quad<T> per position
    int wide_factor;     // 0 forces the wide (one vertex per thread) path on every iteration
    int* blists;         // [gridDim.x][claim_cap] per-CTA claim lists (beyond the smem list)
    int claim_cap;       // capacity of one claim list
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// SM cycle counter read that cannot issue before `dep` is available
__device__ __forceinline__ unsigned long long gtimer_after(int dep) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t) : "r"(dep));
    return t;
}
__device__ __forceinline__ unsigned long long cyc() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
    return t;
}
// [0] start [1] work end [2] release (globaltimer); [3..6] thread-0 task stages,
// [7] task-loop end, [8..11] barrier3 phases (clock64)
constexpr int kDbgSlots = 20;  // v4: [9..17] stages of the first newest-topleset task

__device__ __forceinline__ int ldcg(const int* p) { return __ldcg(p); }
__device__ __forceinline__ float ldcg(const float* p) { return __ldcg(p); }
__device__ __forceinline__ double ldcg(const double* p) { return __ldcg(p); }

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

template <typename T> struct Lim;
template <> struct Lim<float> {
    __device__ static float inf() { return __int_as_float(0x7f800000); }
    __device__ static float min_normal() { return 1.17549435e-38f; }  // FLT_MIN
    __device__ static unsigned long long bits(float x) {
        return static_cast<unsigned long long>(__float_as_uint(x));
    }
    __device__ static float from_bits(unsigned long long b) {
        return __uint_as_float(static_cast<unsigned>(b));
    }
};
template <> struct Lim<double> {
    __device__ static double inf() { return __longlong_as_double(0x7ff0000000000000LL); }
    __device__ static double min_normal() { return 2.2250738585072014e-308; }  // DBL_MIN
    __device__ static unsigned long long bits(double x) {
        return static_cast<unsigned long long>(__double_as_longlong(x));
    }
    __device__ static double from_bits(unsigned long long b) {
        return __longlong_as_double(static_cast<long long>(b));
    }
};

}  // namespace gdb
