// Microbenchmark (sm_100a): grid-barrier designs for the PTP iteration loop,
// empty and with a one-trip gather+store payload per iteration (the minimum
// work of one Jacobi band iteration: read neighbour distances, write own).
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a scripts/microbench_barrier3.cu -o build/mb3
//
// modes
//   0 flat:    red.release.add on one counter, thread 0 polls with ld.acquire
//   1 master:  every CTA st.release's {epoch,payload} into its own 128-B slot;
//              warp 0 of CTA 0 polls all slots, reduces, st.release's one
//              broadcast line; every other CTA polls that line
//   2 allpoll: every CTA st.release's its slot; warp 0 of every CTA polls all
//              slots (no atomics, no second hop)
//   4 relaxed: red.relaxed.add + ld.relaxed poll, no fences (lower bound; not a
//              valid barrier for plain data, only for epoch-tagged data)
//   5 rel-only: red.release.add + ld.relaxed poll (acquire side omitted)
//   3 tree:    atom.acq_rel.add on one of 16 leaf counters; the last arriver of a
//              leaf red.release's the root; root-last writes the broadcast line
//              (arrivals are spread over 16 L2 lines; one extra hop)
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_rel(unsigned* p, unsigned x) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(x) : "memory");
}
__device__ __forceinline__ unsigned atom_ar(unsigned* p, unsigned x) {
    unsigned r;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "r"(x) : "memory");
    return r;
}
__device__ __forceinline__ void st_rel_v2(unsigned long long* p, unsigned long long a,
                                          unsigned long long b) {
    asm volatile("st.release.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void ld_acq_v2(const unsigned long long* p, unsigned long long& a,
                                          unsigned long long& b) {
    asm volatile("ld.acquire.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
__device__ __forceinline__ void st_rel(unsigned* p, unsigned x) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(x) : "memory");
}

struct Ctl {
    unsigned flat;                 // mode 0
    unsigned pad0[31];
    unsigned bcast_epoch;          // modes 1,3 broadcast line
    unsigned bcast_payload;
    unsigned pad1[30];
    unsigned root;                 // mode 3
    unsigned pad2[31];
    unsigned leaf[16 * 32];        // mode 3, one 128-B line each
};

__global__ void iter_kernel(int mode, int iters, int work, Ctl* ctl, unsigned long long* slots,
                            const int* nbr, float* d0, float* d1, int n, unsigned long long* out) {
    const int nb = gridDim.x;
    const int tid = threadIdx.x;
    __shared__ unsigned s_pay;
    unsigned long long t0 = clock64();
    float acc = 0.f;
    // work < 0: |work| vertices, neighbour ids cached in registers (records resident on chip)
    const bool pre = work < 0;
    if (pre) work = -work;
    int cid[6];
    const int v0 = blockIdx.x * blockDim.x + tid;
#pragma unroll
    for (int e = 0; e < 6; ++e) cid[e] = (pre && v0 < work) ? nbr[6 * v0 + e] : 0;
    for (int it = 1; it <= iters; ++it) {
        // one dependent trip: 6 neighbour gathers, one store (Jacobi)
        if (pre) {
            const float* dp = (it & 1) ? d0 : d1;
            float* dc = (it & 1) ? d1 : d0;
            if (v0 < work) {
                float m = dp[v0];
#pragma unroll
                for (int e = 0; e < 6; ++e) m = fminf(m, __ldcg(dp + cid[e]) + 1.0f);
                dc[v0] = m;
                acc += m;
            }
        } else if (work) {
            const float* dp = (it & 1) ? d0 : d1;
            float* dc = (it & 1) ? d1 : d0;
            for (int v = blockIdx.x * blockDim.x + tid; v < work; v += nb * blockDim.x) {
                float m = dp[v];
#pragma unroll
                for (int e = 0; e < 6; ++e) m = fminf(m, __ldcg(dp + nbr[6 * v + e]) + 1.0f);
                dc[v] = m;
                acc += m;
            }
        }
        __syncthreads();
        const unsigned mine = (blockIdx.x * 2654435761u) ^ it;  // payload
        if (mode == 0) {
            if (tid == 0) {
                red_rel(&ctl->flat, 1u);
                const unsigned target = (unsigned)it * nb;
                while ((int)(ld_acq(&ctl->flat) - target) < 0) {
                }
                s_pay = mine;
            }
        } else if (mode == 1 || mode == 2) {
            if (tid == 0) st_rel_v2(slots + 16 * blockIdx.x, (unsigned long long)it, mine);
            if (mode == 2 || blockIdx.x == 0) {
                if (tid < 32) {
                    unsigned mx = 0;
                    for (int b = tid; b < nb; b += 32) {
                        unsigned long long e, p;
                        do {
                            ld_acq_v2(slots + 16 * b, e, p);
                        } while (e < (unsigned long long)it);
                        mx = max(mx, (unsigned)p);
                    }
                    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(~0u, mx, o));
                    if (tid == 0) {
                        s_pay = mx;
                        if (mode == 1) {
                            ctl->bcast_payload = mx;
                            st_rel(&ctl->bcast_epoch, (unsigned)it);
                        }
                    }
                }
            } else if (tid == 0) {
                while ((int)(ld_acq(&ctl->bcast_epoch) - it) < 0) {
                }
                s_pay = __ldcg(&ctl->bcast_payload);
            }
        } else if (mode == 4 || mode == 5) {
            if (tid == 0) {
                if (mode == 4)
                    asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(&ctl->flat), "r"(1u) : "memory");
                else
                    red_rel(&ctl->flat, 1u);
                const unsigned target = (unsigned)it * nb;
                unsigned v;
                do {
                    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(&ctl->flat) : "memory");
                } while ((int)(v - target) < 0);
                s_pay = mine;
            }
        } else if (mode == 3) {
            if (tid == 0) {
                const int leaves = 16;
                const int lf = blockIdx.x % leaves;
                const unsigned lsize = nb / leaves + (lf < nb % leaves ? 1 : 0);
                const unsigned r = atom_ar(&ctl->leaf[lf * 32], 1u);
                if (r + 1 == (unsigned)it * lsize) {
                    const unsigned r2 = atom_ar(&ctl->root, 1u);
                    if (r2 + 1 == (unsigned)it * leaves) {
                        ctl->bcast_payload = mine;
                        st_rel(&ctl->bcast_epoch, (unsigned)it);
                    }
                }
                while ((int)(ld_acq(&ctl->bcast_epoch) - it) < 0) {
                }
                s_pay = __ldcg(&ctl->bcast_payload);
            }
        }
        __syncthreads();
        acc += (float)(s_pay & 1);
    }
    unsigned long long t1 = clock64();
    if (tid == 0) out[blockIdx.x] = t1 - t0;
    if (acc == -1.f) out[0] = 0;
}

int main(int argc, char** argv) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int n = 1 << 20;
    int* h = (int*)malloc(sizeof(int) * 6 * n);
    unsigned long long x = 88172645463325252ull;
    for (int i = 0; i < 6 * n; ++i) {
        x ^= x << 13; x ^= x >> 7; x ^= x << 17;
        h[i] = (int)(x % n);
    }
    int* nbr;
    float *d0, *d1;
    Ctl* ctl;
    unsigned long long *slots, *out;
    cudaMalloc(&nbr, sizeof(int) * 6 * n);
    cudaMemcpy(nbr, h, sizeof(int) * 6 * n, cudaMemcpyHostToDevice);
    cudaMalloc(&d0, 4 * n);
    cudaMalloc(&d1, 4 * n);
    cudaMemset(d0, 0, 4 * n);
    cudaMemset(d1, 0, 4 * n);
    cudaMalloc(&ctl, sizeof(Ctl));
    cudaMalloc(&slots, 8 * 16 * 1024);
    cudaMalloc(&out, 8 * 1024);
    const int iters = 3000;
    const char* names[] = {"flat", "master", "allpoll", "tree", "relaxed", "rel-only"};
    for (int threads : {512, 1024}) {
        for (int work : {0, 16384, -16384}) {
            for (int mode : {0, 3, 4, 5}) {
                cudaMemset(ctl, 0, sizeof(Ctl));
                cudaMemset(slots, 0, 8 * 16 * 1024);
                int m = mode, it = iters, w = work, nn = n;
                void* args[] = {&m, &it, &w, &ctl, &slots, &nbr, &d0, &d1, &nn, &out};
                cudaEvent_t e0, e1;
                cudaEventCreate(&e0);
                cudaEventCreate(&e1);
                cudaEventRecord(e0);
                cudaError_t e = cudaLaunchCooperativeKernel((void*)iter_kernel, sms, threads, args);
                cudaEventRecord(e1);
                cudaDeviceSynchronize();
                float ms = 0;
                cudaEventElapsedTime(&ms, e0, e1);
                printf("%-8s threads %d work %6d: %s  %.3f us per iteration\n", names[mode],
                       threads, work, cudaGetErrorString(e), 1e3 * ms / iters);
            }
        }
    }
    return 0;
}
