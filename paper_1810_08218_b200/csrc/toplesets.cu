// Toplesets with the reference's exact ordering, and reorder_for_bands, on sm_100a.
//
//   bfs_kernel          cooperative level-synchronous BFS (compute_toplesets,
//                       reference src/toplesets.cpp:37-55): one group barrier per
//                       level, warp-aggregated queue appends; levels come out
//                       grouped (limits exact) but unordered inside a level
//   sort_small_kernel   per level, ascending vertex id (toplesets.cpp:53) by an
//                       in-shared-memory bitonic sort (levels <= kSortCap)
//   rank_large_kernel   levels > kSortCap: bitmap of the level + word prefix
//                       popcounts give every vertex its rank among smaller ids
//   position_kernel     position[sorted[p]] = p (toplesets.cpp:38-41)
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
constexpr int kSortCap = 8192;   // ints sorted in shared memory per level
constexpr int kSortBlock = 1024;

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

__global__ void __launch_bounds__(kSortBlock) sort_small_kernel(const int* queue,
                                                                 const int* limits, int rho,
                                                                 int* sorted) {
    __shared__ int buf[kSortCap];
    for (int r = blockIdx.x; r < rho; r += gridDim.x) {
        const int lo = limits[r], sz = limits[r + 1] - lo;
        if (sz > kSortCap) continue;
        if (sz == 1) {
            if (threadIdx.x == 0) sorted[lo] = queue[lo];
            continue;
        }
        int P = 1;
        while (P < sz) P <<= 1;
        for (int x = threadIdx.x; x < P; x += kSortBlock) buf[x] = x < sz ? queue[lo + x] : INT_MAX;
        __syncthreads();
        for (int kk = 2; kk <= P; kk <<= 1) {
            for (int j = kk >> 1; j > 0; j >>= 1) {
                for (int x = threadIdx.x; x < P; x += kSortBlock) {
                    const int y = x ^ j;
                    if (y > x) {
                        const int u = buf[x], w = buf[y];
                        const bool up = (x & kk) == 0;
                        if ((u > w) == up) {
                            buf[x] = w;
                            buf[y] = u;
                        }
                    }
                }
                __syncthreads();
            }
        }
        for (int x = threadIdx.x; x < sz; x += kSortBlock) sorted[lo + x] = buf[x];
        __syncthreads();
    }
}

// One CTA ranks one large level through a bitmap over vertex ids.
__global__ void __launch_bounds__(1024) rank_large_kernel(const int* queue, int lo, int sz, int n,
                                                          unsigned* bitmap, int* wprefix,
                                                          int* sorted) {
    __shared__ int part[1024];
    const int words = (n + 31) / 32;
    for (int x = threadIdx.x; x < sz; x += blockDim.x) {
        const int v = queue[lo + x];
        atomicOr(&bitmap[v >> 5], 1u << (v & 31));
    }
    __syncthreads();
    const int per = (words + blockDim.x - 1) / blockDim.x;
    const int w0 = threadIdx.x * per, w1 = min(words, w0 + per);
    int cnt = 0;
    for (int w = w0; w < w1; ++w) cnt += __popc(bitmap[w]);
    part[threadIdx.x] = cnt;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {  // inclusive scan
        const int add = threadIdx.x >= o ? part[threadIdx.x - o] : 0;
        __syncthreads();
        part[threadIdx.x] += add;
        __syncthreads();
    }
    int run = part[threadIdx.x] - cnt;
    for (int w = w0; w < w1; ++w) {
        wprefix[w] = run;
        run += __popc(bitmap[w]);
    }
    __syncthreads();
    for (int x = threadIdx.x; x < sz; x += blockDim.x) {
        const int v = queue[lo + x];
        const int w = v >> 5;
        const int rank = wprefix[w] + __popc(bitmap[w] & ((1u << (v & 31)) - 1u));
        sorted[lo + rank] = v;
    }
    __syncthreads();
    for (int x = threadIdx.x; x < sz; x += blockDim.x) bitmap[queue[lo + x] >> 5] = 0u;
}

__global__ void position_kernel(const int* sorted, int reachable, int* position) {
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < reachable; p += gridDim.x * blockDim.x)
        position[sorted[p]] = p;
}

int topo_max_blocks(int device) {
    int per_sm = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bfs_kernel, kTopoBlock, 0);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    return per_sm * sms;
}

// scratch: >= 2 * ((n + 31) / 32 + 1) words.  Leaves sorted / limits /
// position on the device and the number of levels in *rho_host.
cudaError_t launch_toplesets(const TopoArgs& a, int* scratch, size_t scratch_words, int* rho_host,
                             cudaStream_t st) {
    const int words = (a.n + 31) / 32 + 1;
    if (scratch_words < static_cast<size_t>(2 * words)) return cudaErrorInvalidValue;
    unsigned* bitmap = reinterpret_cast<unsigned*>(scratch);
    int* wprefix = scratch + words;
    cudaError_t e = cudaMemsetAsync(&a.ctl->bar, 0, sizeof(unsigned), st);
    if (e == cudaSuccess) e = cudaMemsetAsync(bitmap, 0, sizeof(unsigned) * words, st);
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
    const int grid = rho < 4 * 148 ? rho : 4 * 148;
    sort_small_kernel<<<grid, kSortBlock, 0, st>>>(a.queue, a.limits, rho, a.sorted);
    note_launch();
    for (int r = 0; r < rho; ++r) {
        const int sz = lim[r + 1] - lim[r];
        if (sz > kSortCap) {
            rank_large_kernel<<<1, 1024, 0, st>>>(a.queue, lim[r], sz, a.n, bitmap, wprefix,
                                                  a.sorted);
            note_launch();
        }
    }
    const int reach = lim[rho];
    if (reach > 0) {
        position_kernel<<<(reach + 255) / 256 < 1184 ? (reach + 255) / 256 : 1184, 256, 0, st>>>(
            a.sorted, reach, a.position);
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
