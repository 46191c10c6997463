// Microbenchmark (sm_100a): latency of one 4-lane group's candidate evaluation
// (chunk_candidates: 2 corners per lane + neighbour shuffles) as used by the
// solver kernels, one warp per SM, dependent chain across calls.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a --fmad=false \
//        -Ipaper_1810_08218_b200/csrc scripts/microbench_corner.cu -o build/microbench_corner
#include <cstdio>

#include "ptp_common.cuh"

using namespace gdb;

template <typename T>
__global__ void corner_lat(const float* in, int iters, float* out, unsigned long long* cyc_out) {
    const int gl = threadIdx.x & 3;
    // a plausible valence-6 star: |x| ~ 3e-3, Gram inverse ~ 1e5
    T La = T(in[0]) + gl * T(1e-5), Lb = T(in[1]) + gl * T(1e-5);
    Quad<T> qa, qb;
    qa.q11 = in[2]; qa.q12 = in[3]; qa.q22 = in[4];
    qa.a = sizeof(T) == 4 ? T(in[5]) : add(add(qa.q11, mul(T(2), qa.q12)), qa.q22);
    qb = qa;
    T ta = T(in[6]) + gl * T(1e-4), tb = T(in[7]) + gl * T(1e-4);
    const int d = 6;
    long long degs = 0;
    T acc = 0;
    __syncwarp();
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        T best = gl == 0 ? T(1e30) : Lim<T>::inf();
        int bidx = gl == 0 ? -1 : INT_MAX, blab = -1;
        chunk_candidates<T, false>(gl, 0, d, 1, 1, La, Lb, ta, tb, -1, -1, qa, qb, best, bidx,
                                   blab, degs);
        // make the next call depend on this one (tiny perturbation)
        ta = add(ta, mul(best, T(1e-12)));
        acc += best;
    }
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0) cyc_out[blockIdx.x] = t1 - t0;
    out[blockIdx.x * blockDim.x + threadIdx.x] = float(acc) + (float)degs;
}

int main() {
    float h[8] = {3e-3f, 3.1e-3f, 1.2e5f, -0.55e5f, 1.1e5f, 4.2e-6f, 0.50f, 0.5012f};
    float *in, *out;
    unsigned long long* cyc;
    cudaMalloc(&in, sizeof(h));
    cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
    cudaMalloc(&out, 4 << 20);
    cudaMalloc(&cyc, 8 * 1024);
    const int iters = 2000;
    for (int prec : {0, 1})
    for (int warps : {1, 16}) {
        if (prec == 0) corner_lat<float><<<148, 32 * warps>>>(in, iters, out, cyc);
        else corner_lat<double><<<148, 32 * warps>>>(in, iters, out, cyc);
        cudaDeviceSynchronize();
        unsigned long long c[148];
        cudaMemcpy(c, cyc, 8 * 148, cudaMemcpyDeviceToHost);
        double s = 0;
        for (int b = 0; b < 148; ++b) s += c[b];
        printf("%s warps/SM %2d: %.0f cycles per chunk_candidates call (2 corners/lane)\n",
               prec ? "fp64" : "fp32", warps, s / 148 / iters);
    }
    return 0;
}
