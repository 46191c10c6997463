// Host-side launch interface of the device kernels (ptp_kernels.cu, toplesets.cu).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "ptp_device.cuh"

namespace gdb {

void note_launch();  // evidence counter (capi.cu)

template <typename T>
void launch_pack(const double* xyz, int n, const int* cptr, const int* ring_in, int* ring_out,
                 void* ringL, void* quad, int* ering, void* eL, void* equad, cudaStream_t st);

void launch_planar_test(int precision, const double* x1, const double* x2, const double* t1,
                        const double* t2, int count, double* value, int* side, int* degen,
                        cudaStream_t st);

void launch_arith_selftest(long long n, unsigned long long seed, unsigned long long* out,
                           cudaStream_t st);

// The solver (ptp_run4.cu) in three instantiations: mode 0 handles every iteration,
// mode 1 narrow-band iterations only, mode 2 wide-band iterations only (each hands
// the field to the other at a band cross-over, GroupCtl.mode_exit).
// Max co-resident CTAs of the run kernel on `device` (cooperative launch bound).
int run_max_blocks(int precision, bool labels, int device, int mode = 0);
// record-cache bytes (dynamic shared memory) and kernel entry
size_t run4_dyn_smem(int precision, bool labels, int mode);
const void* run4_kernel_ptr(int precision, bool labels, int mode = 0);
cudaError_t launch_run(int precision, bool labels, const RunArgs& args, cudaStream_t st,
                       int mode = 0);

// Toplesets with the reference's exact ordering (toplesets.cu).
struct TopoArgs {
    const int* cptr;
    const int* ring;  // unflagged ring
    int n;
    const int* src;   // m sorted sources
    int m;
    int* level;       // n scratch
    int* queue;       // n: BFS order, then sorted in place per level
    int* limits;      // n+2
    int* sorted;      // n (output: exact reference order)
    int* position;    // n (output)
    GroupCtl* ctl;
    int* rho_out;     // device scalar
    int blocks;
};
int topo_max_blocks(int device);
cudaError_t launch_toplesets(const TopoArgs& a, int* scratch, size_t scratch_words, int* rho_host,
                             cudaStream_t st);

// reorder_for_bands: old_of_new / new_of_old / permuted faces (toplesets.cu).
// xyz / xyz_out: optional position permutation (xyz_out[p] = xyz[old_of_new[p]]).
cudaError_t launch_reorder(const int* position, const int* sorted, int reachable, int n,
                           const int* faces, int nf, int* old_of_new, int* new_of_old,
                           int* faces_out, cudaStream_t st, const double* xyz = nullptr,
                           double* xyz_out = nullptr);

// On-device fan-CSR build (mesh_build.cu).  Returns 0 for a valid mesh, else the
// validation flag bits (~0u with *err set on a CUDA error).
size_t build_fans_scratch_ints(int n, int nf);
unsigned build_fans_device(const double* xyz, int n, const int* faces, int nf, int* cptr,
                           int* ring, int* degree, int* twin, int* scratch, int sms,
                           cudaStream_t st, cudaError_t* err);

}  // namespace gdb
