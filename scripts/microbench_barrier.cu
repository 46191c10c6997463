// Microbenchmark (sm_100a): grid-barrier variants and L2 dependent-load latency
// for a persistent cooperative kernel of 148 CTAs.  Informs the design of the
// PTP iteration loop (one grid barrier per Jacobi iteration).
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a scripts/microbench_barrier.cu -o build/mb
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned ld_rlx(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_rel(unsigned* p, unsigned x) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(x) : "memory");
}
__device__ __forceinline__ void st_rel64(unsigned long long* p, unsigned long long x) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(x) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acq64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_rlx64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// mode 0: __threadfence + atomicAdd + ld.acquire poll + __threadfence (current)
// mode 1: red.release + ld.acquire poll
// mode 2: red.release + ld.relaxed poll (+ fence.acquire after)
// mode 3: per-CTA flag array (st.release epoch), warp 0 polls all flags (ld.relaxed)
__global__ void barrier_kernel(int mode, int iters, unsigned* bar, unsigned long long* flags,
                               unsigned long long* out) {
    const int nb = gridDim.x;
    unsigned epoch = 0;
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        __syncthreads();
        if (mode == 3) {
            if (threadIdx.x == 0) st_rel64(&flags[blockIdx.x * 16], (unsigned long long)(it + 1));
            if (threadIdx.x < 32) {
                for (int b = threadIdx.x; b < nb; b += 32) {
                    while (ld_rlx64(&flags[b * 16]) < (unsigned long long)(it + 1)) {
                    }
                }
                __syncwarp();
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
            }
        } else if (threadIdx.x == 0) {
            ++epoch;
            const unsigned target = epoch * nb;
            if (mode == 0) {
                __threadfence();
                atomicAdd(bar, 1u);
                while ((int)(ld_acq(bar) - target) < 0) {
                }
                __threadfence();
            } else if (mode == 1) {
                red_rel(bar, 1u);
                while ((int)(ld_acq(bar) - target) < 0) {
                }
            } else {
                red_rel(bar, 1u);
                while ((int)(ld_rlx(bar) - target) < 0) {
                }
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
            }
        }
        __syncthreads();
    }
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

// dependent pointer chase through L2-resident memory (ld.cg), 1 thread per CTA
__global__ void chase_kernel(const int* next, int steps, int start, unsigned long long* out,
                             int* sink) {
    if (threadIdx.x != 0) return;
    int p = start + blockIdx.x * 97;
    unsigned long long t0 = clock64();
    for (int s = 0; s < steps; ++s) p = __ldcg(next + p);
    unsigned long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
    sink[blockIdx.x] = p;
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    unsigned* bar;
    unsigned long long *flags, *out;
    cudaMalloc(&bar, 4);
    cudaMalloc(&flags, 8 * 16 * 1024);
    cudaMalloc(&out, 8 * 1024);
    const int iters = 2000;
    for (int threads : {512, 1024}) {
        for (int mode = 0; mode < 4; ++mode) {
            cudaMemset(bar, 0, 4);
            cudaMemset(flags, 0, 8 * 16 * 1024);
            void* args[] = {&mode, (void*)&iters, &bar, &flags, &out};
            int m = mode;
            args[0] = &m;
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            cudaError_t e = cudaLaunchCooperativeKernel((void*)barrier_kernel, sms, threads, args);
            cudaEventRecord(e1);
            cudaDeviceSynchronize();
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("barrier mode %d threads %d: %s  %.3f us per barrier\n", mode, threads,
                   cudaGetErrorString(e), 1e3 * ms / iters);
        }
    }
    // L2 latency: random cyclic permutation over 32 MB
    const int N = 8 << 20;
    int* h = new int[N];
    for (int i = 0; i < N; ++i) h[i] = i;
    unsigned long long x = 88172645463325252ull;
    for (int i = N - 1; i > 0; --i) {
        x ^= x << 13; x ^= x >> 7; x ^= x << 17;
        int j = x % (i + 1);
        int t = h[i]; h[i] = h[j]; h[j] = t;
    }
    int* nxt = new int[N];
    for (int i = 0; i < N; ++i) nxt[h[i]] = h[(i + 1) % N];
    int *d, *sink;
    cudaMalloc(&d, 4ull * N);
    cudaMalloc(&sink, 4 * 1024);
    cudaMemcpy(d, nxt, 4ull * N, cudaMemcpyHostToDevice);
    for (int grid : {1, 148}) {
        chase_kernel<<<grid, 32>>>(d, 2000, 0, out, sink);  // warm L2
        chase_kernel<<<grid, 32>>>(d, 20000, 0, out, sink);
        cudaDeviceSynchronize();
        unsigned long long c[148];
        cudaMemcpy(c, out, 8 * grid, cudaMemcpyDeviceToHost);
        double s = 0;
        for (int b = 0; b < grid; ++b) s += c[b];
        printf("L2 dependent ld.cg latency (grid %d): %.1f cycles (%.1f ns at %d MHz)\n", grid,
               s / grid / 20000, s / grid / 20000 / (clk / 1e6), clk / 1000);
    }
    return 0;
}
