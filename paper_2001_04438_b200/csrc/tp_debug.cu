// Unit-test kernels: expose the device building blocks (tp_common.cuh) element by element so
// tests can check them against the oracle's plain definitions and exact pair arithmetic.
#include "tp_common.cuh"
#include "tp_internal.h"

namespace tp {

__global__ void debug_kernel(int what, const float* a, const float* b, float* o0, float* o1, int64_t count) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    switch (what) {
        case 0: {
            const Pair p = ext_exp(a[i]);
            o0[i] = p.m;
            o1[i] = p.n;
            break;
        }
        case 1: o0[i] = pow2_flush(a[i]); break;
        case 2: {
            const Pair p = pair_merge(Pair{a[2 * i], a[2 * i + 1]}, Pair{b[2 * i], b[2 * i + 1]});
            o0[i] = p.m;
            o1[i] = p.n;
            break;
        }
        case 3: o0[i] = exp_flush2(make_float2(a[i], a[i])).x; break;
        case 4: o0[i] = ex2_ftz(a[i]); break;
        default: break;
    }
}

cudaError_t launch_debug(int what, const float* a, const float* b, float* o0, float* o1, int64_t count,
                         cudaStream_t s) {
    if (count <= 0) return cudaSuccess;
    const int64_t grid = (count + 255) / 256;
    debug_kernel<<<(unsigned)grid, 256, 0, s>>>(what, a, b, o0, o1, count);
    return cudaGetLastError();
}

}  // namespace tp
