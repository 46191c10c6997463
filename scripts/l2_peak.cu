// L2 read bandwidth of this B200 (the denominator of roofline.l2): every SM streams
// an L2-resident buffer with ld.global.cg (L1 bypassed) in 16-byte vectors, several
// passes per launch, best of 10 launches (CUDA events).  Buffer sizes 16-96 MiB
// (L2 = 126 MB on two dies).  Writes JSON to stdout.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a scripts/l2_peak.cu -o /tmp/l2_peak
#include <cstdio>
#include <cuda_runtime.h>

__global__ void sweep(const int4* __restrict__ p, size_t n16, int passes, int* sink) {
    int acc = 0;
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    for (int r = 0; r < passes; ++r)
        for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n16;
             i += stride) {
            int4 v;
            asm volatile("ld.global.cg.v4.s32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p + i));
            acc ^= v.x ^ v.y ^ v.z ^ v.w;
        }
    if (acc == 0x7fffffff) *sink = acc;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const size_t sizes_mib[] = {16, 32, 48, 64, 96};
    int* sink;
    cudaMalloc(&sink, 4);
    printf("{\"sms\": %d, \"results\": [", sms);
    double best_all = 0;
    for (int s = 0; s < 5; ++s) {
        const size_t bytes = sizes_mib[s] << 20;
        int4* buf;
        cudaMalloc(&buf, bytes);
        cudaMemset(buf, 1, bytes);
        const int passes = 8;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        double best = 0;
        for (int it = 0; it < 11; ++it) {
            cudaEventRecord(e0);
            sweep<<<sms * 4, 512>>>(buf, bytes / 16, passes, sink);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            const double gbs = double(bytes) * passes / (ms * 1e-3) / 1e9;
            if (it > 0 && gbs > best) best = gbs;  // launch 0 warms L2
        }
        if (sizes_mib[s] <= 64 && best > best_all) best_all = best;
        printf("%s{\"mib\": %zu, \"gbs\": %.1f}", s ? ", " : "", sizes_mib[s], best);
        cudaFree(buf);
    }
    printf("], \"l2_read_gbs\": %.1f, \"how\": \"ld.global.cg.v4 sweeps of an L2-resident "
           "buffer (16-64 MiB), 8 passes per launch, %d CTAs x 512 threads, best of 10 "
           "launches after one warm-up, CUDA events\"}\n", best_all, sms * 4);
    return 0;
}
