// B200 (sm_100a) kernels of the PTP geodesic solver.
//
//   pack_kernel<T>      one-time per mesh & precision: per-ring |x| and per-corner
//                       Gram inverse {q11,q12,q22,a} + degenerate flag, i.e. the
//                       geometry-only half of planar_update<T>
//                       (reference include/geodist/update_kernel.hpp:38-60)
//   (the solver itself, ptp_run4_kernel, is in ptp_run4.cu)
//   planar_test_kernel  planar_update<T> on raw inputs (parity hook).
//
// All floating point goes through __f*_rn / __d*_rn intrinsics: IEEE rounding,
// no FMA contraction, the reference's left-to-right association -- the CPU
// reference build has no FMA, so results are bit-identical.
#include <climits>
#include <cstdio>

#include "ptp_common.cuh"
#include "ptp_launch.hpp"

namespace gdb {

// ---------------------------------------------------------------------------
// one-time geometry pack (per mesh, per precision)

// CSR tables: per-ring |x|, per-corner Gram inverse, degenerate flag in bit 31.
template <typename T>
__global__ void pack_kernel(const double* __restrict__ xyz, int n, const int* __restrict__ cptr,
                            const int* __restrict__ ring_in, int* __restrict__ ring_out,
                            T* __restrict__ ringL, void* __restrict__ quad) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    const int c0 = cptr[v], d = cptr[v + 1] - c0, r0 = c0 + v;
    if (d == 0) {
        ring_out[r0] = ring_in[r0];
        ringL[r0] = T(0);
        return;
    }
    const T px = to_t<T>(xyz[3 * (size_t)v]), py = to_t<T>(xyz[3 * (size_t)v + 1]),
            pz = to_t<T>(xyz[3 * (size_t)v + 2]);
    T x0 = 0, y0 = 0, z0 = 0, g0 = 0;  // ring entry e-1
    for (int e = 0; e <= d; ++e) {
        const int r = ring_in[r0 + e];
        const T x = sub(to_t<T>(xyz[3 * (size_t)r]), px);
        const T y = sub(to_t<T>(xyz[3 * (size_t)r + 1]), py);
        const T z = sub(to_t<T>(xyz[3 * (size_t)r + 2]), pz);
        const T g = dot3(x, y, z, x, y, z);
        ringL[r0 + e] = sq(g);  // norm(x) = sqrt(dot(x, x)) (vec3.hpp:31-34)
        ring_out[r0 + e] = r;
        if (e > 0) {
            const int c = e - 1;  // corner (ring[c], ring[c+1])
            const T g12 = dot3(x0, y0, z0, x, y, z);
            T q11, q12, q22, a;
            const bool degen = corner_geometry(g0, g, g12, q11, q12, q22, a);
            Quad<T>::store(quad, c0 + c, q11, q12, q22, quad_w<T>(a, degen));
            if (degen) ring_out[r0 + c] = ring_in[r0 + c] | INT_MIN;
        }
        x0 = x; y0 = y; z0 = z; g0 = g;
    }
}

// ELL-8 tables (kEllW ring entries per vertex, interleaved so that lane l of a
// 4-lane group reads entries l and l+4 with one vector load).  Vertices with
// more than kEllW-1 corners are marked overflow and use the CSR tables.
template <typename T>
__global__ void pack_ell_kernel(int n, const int* __restrict__ cptr,
                                const int* __restrict__ ring_f, const T* __restrict__ ringL,
                                const void* __restrict__ quad, int* __restrict__ ering,
                                T* __restrict__ eL, void* __restrict__ equad) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    const int c0 = cptr[v], d = cptr[v + 1] - c0, r0 = c0 + v;
    const size_t b = static_cast<size_t>(v) * kEllW;
    if (d > kEllW - 1) {
        for (int e = 0; e < kEllW; ++e) {
            ering[b + ell_slot(e)] = e == 0 ? (v | (kEllOverflow << kMetaShift)) : v;
            eL[b + ell_slot(e)] = T(0);
            Quad<T>::store(equad, static_cast<int>(b + ell_slot(e)), T(0), T(0), T(0), T(0));
        }
        return;
    }
    for (int e = 0; e < kEllW; ++e) {
        const bool has = d > 0 && e <= d;
        int val = has ? ring_f[r0 + e] : v;  // bit 31: corner e is degenerate
        if (e == 0) val = (val & (INT_MIN | kIdMask)) | (d << kMetaShift);
        ering[b + ell_slot(e)] = val;
        eL[b + ell_slot(e)] = has ? ringL[r0 + e] : T(0);
        Quad<T> q;
        if (e < d) {
            q.load(quad, c0 + e);
        } else {
            q.q11 = q.q12 = q.q22 = q.a = T(0);
        }
        Quad<T>::store(equad, static_cast<int>(b + ell_slot(e)), q.q11, q.q12, q.q22, q.a);
    }
}


// ---------------------------------------------------------------------------
template <typename T>
__global__ void planar_test_kernel(const double* x1, const double* x2, const double* t1,
                                   const double* t2, int count, double* value, int* side,
                                   int* degen) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= count) return;
    const T ax = to_t<T>(x1[3 * q]), ay = to_t<T>(x1[3 * q + 1]), az = to_t<T>(x1[3 * q + 2]);
    const T bx = to_t<T>(x2[3 * q]), by = to_t<T>(x2[3 * q + 1]), bz = to_t<T>(x2[3 * q + 2]);
    const T g11 = dot3(ax, ay, az, ax, ay, az), g22 = dot3(bx, by, bz, bx, by, bz);
    const T g12 = dot3(ax, ay, az, bx, by, bz);
    T q11, q12, q22, a;
    const bool dg = corner_geometry(g11, g22, g12, q11, q12, q22, a);
    // the solver's own path: the packed quad (4th word per quad_w) and corner_eval
    Quad<T> qd;
    qd.q11 = q11;
    qd.q12 = q12;
    qd.q22 = q22;
    qd.a = quad_w<T>(a, dg);
    int s, d;
    const T v = corner_eval<T>(to_t<T>(t1[q]), to_t<T>(t2[q]), sq(g11), sq(g22), qd, dg, false, s, d);
    value[q] = static_cast<double>(v);
    side[q] = s;
    degen[q] = d;
}

// ---------------------------------------------------------------------------
// host launchers

template <typename T>
void launch_pack(const double* xyz, int n, const int* cptr, const int* ring_in, int* ring_out,
                 void* ringL, void* quad, int* ering, void* eL, void* equad, cudaStream_t st) {
    const int blk = 256;
    const int grid = (n + blk - 1) / blk;
    if (grid == 0) return;
    pack_kernel<T><<<grid, blk, 0, st>>>(xyz, n, cptr, ring_in, ring_out, static_cast<T*>(ringL),
                                         quad);
    note_launch();
    pack_ell_kernel<T><<<grid, blk, 0, st>>>(n, cptr, ring_out, static_cast<const T*>(ringL),
                                             quad, ering, static_cast<T*>(eL), equad);
    note_launch();
}
template void launch_pack<float>(const double*, int, const int*, const int*, int*, void*, void*,
                                 int*, void*, void*, cudaStream_t);
template void launch_pack<double>(const double*, int, const int*, const int*, int*, void*, void*,
                                  int*, void*, void*, cudaStream_t);

void launch_planar_test(int precision, const double* x1, const double* x2, const double* t1,
                        const double* t2, int count, double* value, int* side, int* degen,
                        cudaStream_t st) {
    const int blk = 128;
    const int grid = (count + blk - 1) / blk;
    if (precision == 0)
        planar_test_kernel<float><<<grid, blk, 0, st>>>(x1, x2, t1, t2, count, value, side, degen);
    else
        planar_test_kernel<double><<<grid, blk, 0, st>>>(x1, x2, t1, t2, count, value, side, degen);
    note_launch();
}

// Self-test of the straight-line div/sqrt fast paths (ptp_common.cuh) against the
// IEEE intrinsics on pseudo-random operands spanning the exponent range: counts the
// operands each fast path accepts (checked) and those where it differs (mismatch).
// out[0..7] = fp64 div checked, mismatch, fp64 sqrt checked, mismatch, fp32 div ...,
// fp32 sqrt ...
__device__ __forceinline__ unsigned long long mix64(unsigned long long x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull;
    return x ^ (x >> 33);
}
__global__ void arith_selftest_kernel(long long n, unsigned long long seed,
                                      unsigned long long* out) {
    unsigned long long c[8] = {};
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const unsigned long long h1 = mix64(seed ^ (2 * i)), h2 = mix64(seed ^ (2 * i + 1));
        // doubles: random mantissa and sign, exponent in [-300, 300] (and a few edges)
        auto mk = [](unsigned long long h) {
            const unsigned long long e = 1023 - 300 + (h >> 52) % 601;
            return __longlong_as_double(static_cast<long long>(((h & 1ull) << 63) | (e << 52) |
                                                               (h >> 12 & 0xfffffffffffffull)));
        };
        const double x = mk(h1), y = mk(h2);
        bool ok;
        const double q = div_with_recip64(x, y, div_recip64(y), ok);
        if (ok) {
            ++c[0];
            c[1] += __double_as_longlong(q) != __double_as_longlong(__ddiv_rn(x, y));
        }
        const double ax = fabs(x);
        const double r = sqrt_fast64(ax, ok);
        if (ok) {
            ++c[2];
            c[3] += __double_as_longlong(r) != __double_as_longlong(__dsqrt_rn(ax));
        }
        // floats: exponent in [-80, 80]
        auto mkf = [](unsigned long long h) {
            const unsigned e = 127 - 80 + static_cast<unsigned>((h >> 40) % 161);
            return __uint_as_float(static_cast<unsigned>((h & 1ull) << 31) | (e << 23) |
                                   static_cast<unsigned>(h >> 9 & 0x7fffffu));
        };
        const float xf = mkf(h1), yf = mkf(h2);
        if (div_operand_ok(xf) && div_operand_ok(yf)) {
            ++c[4];
            const float qf = div_with_recip(xf, yf, div_recip(yf));
            c[5] += __float_as_uint(qf) != __float_as_uint(__fdiv_rn(xf, yf));
        }
        const float af = fabsf(xf);
        if (sqrt_fast_ok(af)) {
            ++c[6];
            c[7] += __float_as_uint(sqrt_fast(af)) != __float_as_uint(__fsqrt_rn(af));
        }
    }
    for (int k = 0; k < 8; ++k) atomicAdd(out + k, c[k]);
}

void launch_arith_selftest(long long n, unsigned long long seed, unsigned long long* out,
                           cudaStream_t st) {
    arith_selftest_kernel<<<4 * 148, 256, 0, st>>>(n, seed, out);
    note_launch();
}

__global__ void reset_bars_kernel(GroupCtl* ctl, int groups) {
    for (int g = threadIdx.x; g < groups; g += blockDim.x) {
        ctl[g].bar = 0u;
        for (int w = 0; w < 4; ++w) ctl[g].barw[w] = 0ull;
    }
}

// mode 0: combined, 1: narrow-band only, 2: wide-band only (ptp_run4.cu)
static const void* run_kernel_ptr(int mode, int precision, bool labels) {
    return run4_kernel_ptr(precision, labels, mode);
}

int run_max_blocks(int precision, bool labels, int device, int mode) {
    int per_sm = 0, sms = 0;
    const void* f = run_kernel_ptr(mode, precision, labels);
    const size_t dyn = run4_dyn_smem(precision, labels, mode);
    if (dyn) cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    // prefer L1: the shared-memory carveout is then the smallest that fits the record cache
    // (none in the wide-only instantiation), and the rest of the SM's 256 KB caches the cell
    // gathers
    cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, f, run4_block(mode), dyn);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    // a group's CTA count must fit the barrier word's 8-bit-safe nonconverged-CTA
    // field (ptp_run4.cu: abort_bits); 148 on a B200 (one CTA per SM)
    return per_sm * sms < 255 ? per_sm * sms : 255;
}

cudaError_t launch_run(int precision, bool labels, const RunArgs& args, cudaStream_t st,
                       int mode) {
    const int grid = args.groups * args.blocks_per_group;
    RunArgs a = args;
    void* params[] = {&a};
    reset_bars_kernel<<<1, 32, 0, st>>>(a.ctl, a.groups);
    note_launch();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const void* f = run_kernel_ptr(mode, precision, labels);
    const size_t dyn = run4_dyn_smem(precision, labels, mode);
    if (dyn) cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 0);
    e = cudaLaunchCooperativeKernel(f, dim3(grid), dim3(run4_block(mode)), params, dyn, st);
    note_launch();
    return e;
}

}  // namespace gdb
