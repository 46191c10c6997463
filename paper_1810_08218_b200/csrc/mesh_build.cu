// On-device mesh build: the rotational fan-CSR the solver packs,
// built from the uploaded face array with no host pass over the mesh.
//
// Same output as the host build_fans (mesh_host.cpp), i.e. the reference's
// build_connectivity + for_each_incident_triangle order (src/connectivity.cpp:19-81,
// include/geodist/connectivity.hpp:35-44):
//   * half-edge h = 3f + c starts at faces[h]; next/prev inside its face;
//   * twin(h) = the half-edge target(h) -> origin(h);
//   * fan start of v: its smallest outgoing half-edge, rotated h -> next(twin(h))
//     back to the open-fan start (connectivity.cpp:47-60);
//   * fan walk h -> twin(prev(h)), ring entry target(h), closing entry
//     origin(prev(last)) for an open fan, r_0 for a closed one (connectivity.cpp:83-96).
// The fan order depends only on the smallest outgoing half-edge and the twins, so the
// outgoing half-edges are bucketed by origin with atomics (order inside a bucket is
// irrelevant) instead of a sort.
//
// Kernels (one pass each, all HBM/L2-latency bound, grid-stride, 148 x k CTAs):
//   validate_count  vertex/face checks of validate_mesh (src/mesh.cpp:11-34) -> flag bits;
//                   outgoing-half-edge count per origin
//   scan            exclusive sum of the counts -> cptr (= corner offsets: every
//                   outgoing half-edge of a manifold vertex is one corner)
//   fill            bucket[cptr[o] + k] = h, btgt[...] = target(h)
//   twins           twin per half-edge from the target's bucket; repeated directed
//                   edges (connectivity.cpp:33-35) -> flag
//   fans            per vertex: fan start, walk, ring + degree; star not a single fan
//                   (connectivity.cpp:76-78) -> flag
// Any flag: the caller re-runs the host build for the reference's exact error text.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "ptp_launch.hpp"

namespace gdb {
namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ int he_next(int h) { return h % 3 == 2 ? h - 2 : h + 1; }
__device__ __forceinline__ int he_prev(int h) { return h % 3 == 0 ? h + 2 : h - 1; }

__global__ void validate_count_kernel(const double* __restrict__ xyz, int n,
                                      const int* __restrict__ faces, int nf,
                                      int* __restrict__ cnt, unsigned* __restrict__ flag) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned f_bits = 0;
    if (xyz)
        for (long long v = tid; v < n; v += stride) {
            const double a = xyz[3 * v], b = xyz[3 * v + 1], c = xyz[3 * v + 2];
            if (!isfinite(a) || !isfinite(b) || !isfinite(c)) f_bits |= 1u;
        }
    for (long long f = tid; f < nf; f += stride) {
        const int t0 = faces[3 * f], t1 = faces[3 * f + 1], t2 = faces[3 * f + 2];
        if (t0 < 0 || t0 >= n || t1 < 0 || t1 >= n || t2 < 0 || t2 >= n) {
            f_bits |= 2u;
            continue;
        }
        if (t0 == t1 || t1 == t2 || t0 == t2) f_bits |= 4u;
        if (xyz) {
            const int t[3] = {t0, t1, t2};
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const double* pa = xyz + 3 * (long long)t[c];
                const double* pb = xyz + 3 * (long long)t[(c + 1) % 3];
                if (pa[0] == pb[0] && pa[1] == pb[1] && pa[2] == pb[2]) f_bits |= 8u;
            }
        }
        atomicAdd(cnt + t0, 1);
        atomicAdd(cnt + t1, 1);
        atomicAdd(cnt + t2, 1);
    }
    if (f_bits) atomicOr(flag, f_bits);
}

// Exclusive scan of x[0..m) in place, three phases (per-tile sums, one-CTA scan of the
// tile sums, tile down-sweep).  Tile = kThreads * 8 items.
constexpr int kScanItems = 8;
constexpr int kTile = kThreads * kScanItems;

__device__ __forceinline__ int block_excl_scan(int v, int* sh, int* total) {
    // warp inclusive scan
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int s = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(~0u, s, o);
        if (lane >= o) s += y;
    }
    if (lane == 31) sh[w] = s;
    __syncthreads();
    if (w == 0) {
        int t = lane < kThreads / 32 ? sh[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(~0u, t, o);
            if (lane >= o) t += y;
        }
        if (lane < kThreads / 32) sh[lane] = t;
    }
    __syncthreads();
    const int before = (w ? sh[w - 1] : 0) + s - v;
    *total = sh[kThreads / 32 - 1];
    __syncthreads();
    return before;
}

__global__ void tile_sum_kernel(const int* __restrict__ x, long long m, int* __restrict__ sums) {
    __shared__ int sh[kThreads / 32];
    const long long base = (long long)blockIdx.x * kTile + threadIdx.x * kScanItems;
    int s = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i)
        if (base + i < m) s += x[base + i];
    int total;
    block_excl_scan(s, sh, &total);
    if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

__global__ void sums_scan_kernel(int* __restrict__ sums, int tiles) {
    __shared__ int sh[kThreads / 32];
    int carry = 0;
    for (int base = 0; base < tiles; base += kThreads) {
        const int i = base + threadIdx.x;
        const int v = i < tiles ? sums[i] : 0;
        int total;
        const int e = block_excl_scan(v, sh, &total);
        if (i < tiles) sums[i] = carry + e;
        carry += total;
    }
}

__global__ void tile_scan_kernel(int* __restrict__ x, long long m, const int* __restrict__ sums) {
    __shared__ int sh[kThreads / 32];
    const long long base = (long long)blockIdx.x * kTile + threadIdx.x * kScanItems;
    int v[kScanItems];
    int s = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        v[i] = base + i < m ? x[base + i] : 0;
        s += v[i];
    }
    int total;
    int run = block_excl_scan(s, sh, &total) + sums[blockIdx.x];
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        if (base + i < m) x[base + i] = run;
        run += v[i];
    }
}

__global__ void fill_kernel(const int* __restrict__ faces, long long nhe, int* __restrict__ cur,
                            int* __restrict__ bucket, int* __restrict__ btgt) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long h = (long long)blockIdx.x * blockDim.x + threadIdx.x; h < nhe; h += stride) {
        const int o = faces[h];
        const int pos = atomicAdd(cur + o, 1);
        bucket[pos] = (int)h;
        btgt[pos] = faces[he_next((int)h)];
    }
}

__global__ void twin_kernel(const int* __restrict__ faces, long long nhe,
                            const int* __restrict__ cptr, const int* __restrict__ bucket,
                            const int* __restrict__ btgt, int* __restrict__ twin,
                            unsigned* __restrict__ flag) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    bool dup = false;
    for (long long h = (long long)blockIdx.x * blockDim.x + threadIdx.x; h < nhe; h += stride) {
        const int o = faces[h], t = faces[he_next((int)h)];
        int tw = -1;
        for (int q = cptr[t], e = cptr[t + 1]; q < e; ++q)
            if (btgt[q] == o) {
                tw = bucket[q];
                break;
            }
        twin[h] = tw;
        int same = 0;  // outgoing half-edges of o with target t (h itself included)
        for (int q = cptr[o], e = cptr[o + 1]; q < e; ++q) same += btgt[q] == t;
        dup |= same > 1;
    }
    if (dup) atomicOr(flag, 16u);
}

__global__ void fans_kernel(const int* __restrict__ faces, int n, const int* __restrict__ cptr,
                            const int* __restrict__ bucket, const int* __restrict__ twin,
                            int* __restrict__ ring, int* __restrict__ degree,
                            unsigned* __restrict__ flag) {
    const int stride = gridDim.x * blockDim.x;
    bool bad = false;
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += stride) {
        const int b0 = cptr[v], incident = cptr[v + 1] - b0;
        int* r = ring + b0 + v;  // incident + 1 slots
        if (incident == 0) {
            r[0] = -1;
            degree[v] = 0;
            continue;
        }
        int h0 = bucket[b0];
        for (int q = 1; q < incident; ++q) h0 = min(h0, bucket[b0 + q]);
        // rotate back to the open-fan start (at most `incident` steps on a valid star)
        int h = h0;
        for (int s = 0; s < incident && twin[h] != -1; ++s) {
            h = he_next(twin[h]);
            if (h == h0) break;
        }
        int w = h, last = h, count = 0;
        do {
            r[count] = faces[he_next(w)];
            ++count;
            last = w;
            w = twin[he_prev(w)];
        } while (w != -1 && w != h && count < incident);
        const bool open = w == -1;
        if (count != incident || (w != -1 && w != h)) {
            bad = true;
            continue;
        }
        r[count] = open ? faces[he_prev(last)] : r[0];
        degree[v] = open ? count + 1 : count;
    }
    if (bad) atomicOr(flag, 32u);
}

int grid_for(long long items, int sms) {
    const long long want = (items + kThreads - 1) / kThreads;
    const long long cap = 8LL * sms;
    return (int)(want < 1 ? 1 : (want < cap ? want : cap));
}

}  // namespace

// faces (3 nf, device), xyz (3 n, device, or null: no coordinate checks).  Outputs:
// cptr (n+1), ring (3 nf + n), degree (n), twin (3 nf).  Scratch: 3 * (3 nf) + tiles
// ints (bucket, btgt, cursor copy of cptr is taken in `scratch` too).  Returns the
// flag word (0 = valid mesh); synchronises `st` twice.
unsigned build_fans_device(const double* xyz, int n, const int* faces, int nf, int* cptr,
                           int* ring, int* degree, int* twin, int* scratch, int sms,
                           cudaStream_t st, cudaError_t* err) {
    const long long nhe = 3LL * nf;
    unsigned* flag = reinterpret_cast<unsigned*>(scratch);
    int* cur = scratch + 32;                  // n + 1
    int* bucket = cur + (n + 1);              // nhe
    int* btgt = bucket + nhe;                 // nhe
    int* sums = btgt + nhe;                   // tiles
    const long long m = (long long)n + 1;
    const int tiles = (int)((m + kTile - 1) / kTile);
    unsigned hflag = 0;
    auto fail = [&](cudaError_t e) {
        *err = e;
        return ~0u;
    };
    cudaError_t e;
    if ((e = cudaMemsetAsync(flag, 0, sizeof(unsigned), st)) != cudaSuccess) return fail(e);
    if ((e = cudaMemsetAsync(cptr, 0, sizeof(int) * m, st)) != cudaSuccess) return fail(e);
    validate_count_kernel<<<grid_for(n > nf ? n : nf, sms), kThreads, 0, st>>>(xyz, n, faces, nf,
                                                                               cptr, flag);
    note_launch();
    if ((e = cudaMemcpyAsync(&hflag, flag, sizeof(unsigned), cudaMemcpyDeviceToHost, st)) !=
        cudaSuccess)
        return fail(e);
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return fail(e);
    if (hflag) return hflag;  // out-of-range indices: stop before any bucket write
    tile_sum_kernel<<<tiles, kThreads, 0, st>>>(cptr, m, sums);
    sums_scan_kernel<<<1, kThreads, 0, st>>>(sums, tiles);
    tile_scan_kernel<<<tiles, kThreads, 0, st>>>(cptr, m, sums);
    for (int i = 0; i < 3; ++i) note_launch();
    if ((e = cudaMemcpyAsync(cur, cptr, sizeof(int) * m, cudaMemcpyDeviceToDevice, st)) !=
        cudaSuccess)
        return fail(e);
    fill_kernel<<<grid_for(nhe, sms), kThreads, 0, st>>>(faces, nhe, cur, bucket, btgt);
    twin_kernel<<<grid_for(nhe, sms), kThreads, 0, st>>>(faces, nhe, cptr, bucket, btgt, twin,
                                                         flag);
    fans_kernel<<<grid_for(n, sms), kThreads, 0, st>>>(faces, n, cptr, bucket, twin, ring, degree,
                                                       flag);
    for (int i = 0; i < 3; ++i) note_launch();
    if ((e = cudaGetLastError()) != cudaSuccess) return fail(e);
    if ((e = cudaMemcpyAsync(&hflag, flag, sizeof(unsigned), cudaMemcpyDeviceToHost, st)) !=
        cudaSuccess)
        return fail(e);
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return fail(e);
    return hflag;
}

size_t build_fans_scratch_ints(int n, int nf) {
    const long long m = (long long)n + 1;
    return 32 + (size_t)m + 2 * 3 * (size_t)nf + (size_t)((m + kTile - 1) / kTile) + 32;
}

}  // namespace gdb
