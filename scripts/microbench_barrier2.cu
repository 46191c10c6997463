// Grid-barrier cost vs CTA count and with thread-block-cluster pre-aggregation (sm_100a).
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_rel(unsigned* p, unsigned x) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(x) : "memory");
}

// flat: every CTA arrives; clustered: cluster barrier, one CTA per cluster arrives,
// then cluster barrier again to release the others.
template <bool CLUSTER>
__global__ void bar_kernel(int iters, unsigned* bar, unsigned long long* out) {
    unsigned epoch = 0;
    unsigned narr = gridDim.x;
    unsigned rank = 0;
    if (CLUSTER) {
        cg::cluster_group cl = cg::this_cluster();
        narr = gridDim.x / cl.num_blocks();
        rank = cl.block_rank();
    }
    for (int it = 0; it < iters; ++it) {
        if (CLUSTER) {
            cg::this_cluster().sync();
            if (rank == 0 && threadIdx.x == 0) {
                ++epoch;
                red_rel(bar, 1u);
                while ((int)(ld_acq(bar) - epoch * narr) < 0) {
                }
            }
            cg::this_cluster().sync();
        } else {
            __syncthreads();
            if (threadIdx.x == 0) {
                ++epoch;
                red_rel(bar, 1u);
                while ((int)(ld_acq(bar) - epoch * narr) < 0) {
                }
            }
            __syncthreads();
        }
    }
}

template <bool CLUSTER>
float run(int grid, int cluster, int threads, unsigned* bar) {
    cudaMemset(bar, 0, 4);
    int iters = 2000;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(threads);
    cudaLaunchAttribute at[2];
    int na = 0;
    at[na].id = cudaLaunchAttributeCooperative;
    at[na].val.cooperative = 1;
    ++na;
    if (CLUSTER) {
        at[na].id = cudaLaunchAttributeClusterDimension;
        at[na].val.clusterDim.x = cluster;
        at[na].val.clusterDim.y = 1;
        at[na].val.clusterDim.z = 1;
        ++na;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    if (CLUSTER && cluster > 8)
        cudaFuncSetAttribute(bar_kernel<CLUSTER>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    unsigned long long* out = nullptr;
    cudaError_t e = cudaLaunchKernelEx(&cfg, bar_kernel<CLUSTER>, iters, bar, out);
    cudaEventRecord(e1);
    cudaError_t e2 = cudaDeviceSynchronize();
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (e != cudaSuccess || e2 != cudaSuccess) {
        printf("  grid %d cluster %d: launch %s / %s\n", grid, cluster, cudaGetErrorString(e),
               cudaGetErrorString(e2));
        cudaGetLastError();
        return -1;
    }
    return 1e3f * ms / iters;
}

int main() {
    unsigned* bar;
    cudaMalloc(&bar, 4);
    for (int grid : {16, 37, 74, 148})
        printf("flat grid %3d x512: %.3f us\n", grid, run<false>(grid, 1, 512, bar));
    printf("flat grid 296 x256: %.3f us\n", run<false>(296, 1, 256, bar));
    for (int cl : {2, 4, 8, 16}) {
        int grid = (148 / cl) * cl;
        printf("cluster %2d grid %3d x512: %.3f us\n", cl, grid, run<true>(grid, cl, 512, bar));
    }
    return 0;
}
