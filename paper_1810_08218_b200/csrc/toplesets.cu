// Toplesets with the reference's exact ordering, and reorder_for_bands, on sm_100a.
//
//   bfs_kernel          cooperative level-synchronous BFS (compute_toplesets,
//                       reference src/toplesets.cpp:37-55): one group barrier per
//                       level, warp-aggregated queue appends; levels come out
//                       grouped (limits exact) but unordered inside a level
//   level_count/scan/scatter_kernel  ascending vertex id inside every level
//                       (toplesets.cpp:53) and position[sorted[p]] = p
//                       (toplesets.cpp:38-41): a stable counting sort of the vertices
//                       by level over chunks of consecutive ids, all levels at once
//   reorder kernels     reorder_for_bands (toplesets.cpp:60-89): old_of_new =
//                       sorted ++ unreachable in id order, inverse, face rewrite.
//                       The permuted connectivity is a relabelling of the
//                       original one (same half-edge ids), so no rebuild.
#include <climits>
#include <vector>

#include "ptp_device.cuh"
#include "ptp_launch.hpp"

namespace gdb {

constexpr int kTopoBlock = 512;

template <typename Post>
__device__ __forceinline__ void topo_barrier(unsigned* bar, unsigned& epoch, unsigned nblk,
                                             Post&& post) {
    __syncthreads();
    if (threadIdx.x == 0) {
        ++epoch;
        __threadfence();
        atomicAdd(bar, 1u);
        const unsigned target = epoch * nblk;
        while (static_cast<int>(ld_acquire(bar) - target) < 0) {
        }
        __threadfence();
        post();
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kTopoBlock) bfs_kernel(TopoArgs a) {
    __shared__ int s_lo, s_hi, s_r, s_done;
    const int nb = gridDim.x;
    const int tid = threadIdx.x;
    const int gtid = blockIdx.x * kTopoBlock + tid;
    const int gthreads = nb * kTopoBlock;
    unsigned epoch = 0;
    GroupCtl* ctl = a.ctl;
    for (int v = gtid; v < a.n; v += gthreads) {
        a.level[v] = -1;
        a.position[v] = -1;
    }
    if (gtid == 0) ctl->tail = a.m;
    topo_barrier(&ctl->bar, epoch, nb, [] {});
    for (int s = gtid; s < a.m; s += gthreads) {
        a.level[a.src[s]] = 0;
        a.queue[s] = a.src[s];
    }
    int lo = 0, hi = a.m, r = 0, done = 0;
    topo_barrier(&ctl->bar, epoch, nb, [&] {
        s_lo = lo; s_hi = hi; s_r = r; s_done = 0;
        if (blockIdx.x == 0) a.limits[0] = 0;
    });
    const int lane = tid & (kW - 1);
    const int sw = tid / kW;
    const int stride = nb * (kTopoBlock / kW);
    while (!s_done) {
        const int L0 = s_lo, L1 = s_hi, rr = s_r;
        for (int t = blockIdx.x + nb * sw;; t += stride) {
            const bool act = t < L1 - L0;
            if (!__any_sync(kFull, act)) break;
            int v = 0, c0 = 0, d = 0;
            if (act) {
                v = ldcg(a.queue + L0 + t);
                c0 = __ldg(a.cptr + v);
                d = __ldg(a.cptr + v + 1) - c0;
            }
            int nch = d > 0 ? (d + kW) / kW : 0;
            nch = __reduce_max_sync(kFull, nch);
            for (int ch = 0; ch < nch; ++ch) {
                const int e = ch * kW + lane;
                bool claim = false;
                int id = 0;
                if (act && d > 0 && e <= d) {
                    id = __ldg(a.ring + c0 + v + e);
                    if (ldcg(a.level + id) < 0) claim = atomicCAS(a.level + id, -1, rr + 1) == -1;
                }
                const unsigned bal = __ballot_sync(kFull, claim);
                if (bal) {
                    const int l32 = tid & 31;
                    const int leader = __ffs(bal) - 1;
                    int base = 0;
                    if (l32 == leader) base = atomicAdd(&ctl->tail, __popc(bal));
                    base = __shfl_sync(kFull, base, leader);
                    if (claim) a.queue[base + __popc(bal & ((1u << l32) - 1u))] = id;
                }
            }
        }
        topo_barrier(&ctl->bar, epoch, nb, [&] {
            const int nt = ldcg(&ctl->tail);
            if (blockIdx.x == 0) a.limits[rr + 1] = L1;
            if (nt == L1) {
                done = 1;
                if (blockIdx.x == 0) *a.rho_out = rr + 1;
            } else {
                lo = L1;
                hi = nt;
                ++r;
            }
            s_lo = lo; s_hi = hi; s_r = r; s_done = done;
        });
    }
}

// Exact order inside every level (ascending vertex id, toplesets.cpp:53) for all
// levels at once, as a stable counting sort of the vertices by level over chunks of
// consecutive ids: one warp per chunk counts its vertices per level, every level's
// row of chunk counts is scanned into global offsets (limits[r] + earlier chunks),
// and the warp scatters its chunk in id order.  position[v] comes out of the same pass.
__global__ void level_count_kernel(const int* level, int n, int chunk, int nchunks,
                                   int* cnt) {
    const int lane = threadIdx.x & 31;
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int c = w; c < nchunks; c += nw) {
        const int v1 = min(n, (c + 1) * chunk);
        for (int v0 = c * chunk; v0 < v1; v0 += 32) {
            const int v = v0 + lane;
            const int l = v < v1 ? level[v] : -1;
            const unsigned peers = __match_any_sync(kFull, l);
            if (l >= 0 && lane == __ffs(peers) - 1)
                atomicAdd(cnt + static_cast<size_t>(l) * nchunks + c, __popc(peers));
        }
    }
}

// one warp per level: exclusive scan of the level's chunk counts, offset by limits[r]
__global__ void level_scan_kernel(const int* limits, int rho, int nchunks, int* cnt) {
    const int lane = threadIdx.x & 31;
    const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (r >= rho) return;
    int* row = cnt + static_cast<size_t>(r) * nchunks;
    int run = limits[r];
    for (int c0 = 0; c0 < nchunks; c0 += 32) {
        const int c = c0 + lane;
        const int x = c < nchunks ? row[c] : 0;
        int incl = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl += y;
        }
        if (c < nchunks) row[c] = run + incl - x;
        run += __shfl_sync(kFull, incl, 31);
    }
}

__global__ void level_scatter_kernel(const int* level, int n, int chunk, int nchunks,
                                     int* off, int* sorted, int* position) {
    const int lane = threadIdx.x & 31;
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int c = w; c < nchunks; c += nw) {
        const int v1 = min(n, (c + 1) * chunk);
        for (int v0 = c * chunk; v0 < v1; v0 += 32) {
            const int v = v0 + lane;
            const int l = v < v1 ? level[v] : -1;
            const unsigned peers = __match_any_sync(kFull, l);
            const int leader = __ffs(peers) - 1;
            int* slot = off + static_cast<size_t>(l < 0 ? 0 : l) * nchunks + c;
            int base = 0;
            if (l >= 0 && lane == leader) base = *slot;
            base = __shfl_sync(kFull, base, leader);
            if (l >= 0) {
                const int at = base + __popc(peers & ((1u << lane) - 1u));
                sorted[at] = v;
                position[v] = at;
                if (lane == leader) *slot = base + __popc(peers);
            }
            __syncwarp();  // the next step's leader reads the updated offsets
        }
    }
}

int topo_max_blocks(int device) {
    int per_sm = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bfs_kernel, kTopoBlock, 0);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    return per_sm * sms;
}

// scratch: the (level, chunk) count table, at least n / 1024 + 1 words (more words
// allow smaller chunks).  Leaves sorted / limits / position on the device and the
// number of levels in *rho_host.
cudaError_t launch_toplesets(const TopoArgs& a, int* scratch, size_t scratch_words, int* rho_host,
                             cudaStream_t st) {
    int* counts = scratch;
    const long long count_words = static_cast<long long>(scratch_words);
    if (count_words < a.n / 1024 + 1) return cudaErrorInvalidValue;
    cudaError_t e = cudaMemsetAsync(&a.ctl->bar, 0, sizeof(unsigned), st);
    if (e != cudaSuccess) return e;
    TopoArgs args = a;
    void* params[] = {&args};
    e = cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(&bfs_kernel), dim3(a.blocks),
                                    dim3(kTopoBlock), params, 0, st);
    note_launch();
    if (e != cudaSuccess) return e;
    int rho = 0;
    e = cudaMemcpyAsync(&rho, a.rho_out, sizeof(int), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return e;
    std::vector<int> lim(static_cast<size_t>(rho) + 1);
    e = cudaMemcpyAsync(lim.data(), a.limits, sizeof(int) * (rho + 1), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return e;
    const int reach = lim[rho];
    if (reach > 0) {
        // chunks of consecutive ids; the per-(level, chunk) table stays within the
        // scratch the caller provides (count_words)
        long long chunk = 1024;
        while (static_cast<long long>(rho) * ((a.n + chunk - 1) / chunk) > count_words) chunk *= 2;
        const int nchunks = static_cast<int>((a.n + chunk - 1) / chunk);
        e = cudaMemsetAsync(counts, 0, sizeof(int) * static_cast<size_t>(rho) * nchunks, st);
        if (e != cudaSuccess) return e;
        const int wblocks = (nchunks + 7) / 8;  // 8 warps per block, one warp per chunk
        level_count_kernel<<<wblocks, 256, 0, st>>>(a.level, a.n, static_cast<int>(chunk), nchunks,
                                                   counts);
        note_launch();
        level_scan_kernel<<<(rho + 7) / 8, 256, 0, st>>>(a.limits, rho, nchunks, counts);
        note_launch();
        level_scatter_kernel<<<wblocks, 256, 0, st>>>(a.level, a.n, static_cast<int>(chunk),
                                                     nchunks, counts, a.sorted, a.position);
        note_launch();
    }
    *rho_host = rho;
    return cudaGetLastError();
}

// Unreachable vertices in original order after the reachable block
// (toplesets.cpp:67-69): one CTA, chunked stable compaction.
__global__ void __launch_bounds__(1024) unreached_kernel(const int* position, int n, int reachable,
                                                         int* old_of_new) {
    __shared__ int part[1024];
    const int per = (n + blockDim.x - 1) / blockDim.x;
    const int v0 = threadIdx.x * per, v1 = min(n, v0 + per);
    int cnt = 0;
    for (int v = v0; v < v1; ++v) cnt += position[v] < 0;
    part[threadIdx.x] = cnt;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
        const int add = threadIdx.x >= o ? part[threadIdx.x - o] : 0;
        __syncthreads();
        part[threadIdx.x] += add;
        __syncthreads();
    }
    int out = reachable + part[threadIdx.x] - cnt;
    for (int v = v0; v < v1; ++v)
        if (position[v] < 0) old_of_new[out++] = v;
}

__global__ void inverse_kernel(const int* old_of_new, int n, int* new_of_old) {
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x)
        new_of_old[old_of_new[p]] = p;
}

__global__ void relabel_kernel(const int* new_of_old, const int* faces, long long count,
                               int* faces_out) {
    for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < count;
         x += (long long)gridDim.x * blockDim.x)
        faces_out[x] = new_of_old[faces[x]];
}

__global__ void permute_xyz_kernel(const int* old_of_new, int n, const double* xyz,
                                   double* xyz_out) {
    for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < 3LL * n;
         x += (long long)gridDim.x * blockDim.x)
        xyz_out[x] = xyz[3LL * old_of_new[x / 3] + x % 3];
}

cudaError_t launch_reorder(const int* position, const int* sorted, int reachable, int n,
                           const int* faces, int nf, int* old_of_new, int* new_of_old,
                           int* faces_out, cudaStream_t st, const double* xyz, double* xyz_out) {
    cudaError_t e = cudaMemcpyAsync(old_of_new, sorted, sizeof(int) * reachable,
                                    cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return e;
    unreached_kernel<<<1, 1024, 0, st>>>(position, n, reachable, old_of_new);
    note_launch();
    const int g = (n + 255) / 256 < 1184 ? (n + 255) / 256 : 1184;
    inverse_kernel<<<g > 0 ? g : 1, 256, 0, st>>>(old_of_new, n, new_of_old);
    note_launch();
    relabel_kernel<<<1184, 256, 0, st>>>(new_of_old, faces, 3LL * nf, faces_out);
    note_launch();
    if (xyz && xyz_out) {
        permute_xyz_kernel<<<1184, 256, 0, st>>>(old_of_new, n, xyz, xyz_out);
        note_launch();
    }
    return cudaGetLastError();
}

}  // namespace gdb
