// One-sided exchange of the per-rank (m, n) partials over NVLink (the
// rank merge a7 of BASELINE.json north_star without a collective library).
//
// Every rank owns a mailbox in its own HBM (layout in include/twopass.h): per epoch parity, a
// flag per rank and a [world][rows] array of pairs (tp_internal.h: why two halves suffice).
// After pass 1, rank r's push kernel stores its pairs into slot r of EVERY rank's mailbox (peer pointers from CUDA IPC: plain st.global over NVLink,
// P2P), makes them visible system-wide (fence.sc.sys) and then release-stores the epoch into
// flag r of each mailbox.  The wait kernel acquires the world flags of the local mailbox for
// this epoch; the finish kernel then reads the pairs from the local mailbox and merges them
// with the canonical tree over rank index (reading G8), exactly as after an all_gather.
// Flags are epoch-tagged, so mailboxes are never reset between calls.
#include <cstdint>

#include "tp_sched.cuh"

namespace tp {


__global__ void pairs_push_kernel(const float2* pairs, int64_t rows, char* const* mailboxes, int rank, int world,
                                  unsigned epoch) {
    const size_t off = mailbox_pairs_offset(world, rows, epoch);
    for (int p = 0; p < world; ++p) {
        float2* dst = reinterpret_cast<float2*>(mailboxes[p] + off) + (int64_t)rank * rows;
        for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) dst[i] = pairs[i];
    }
    __threadfence_system();  // the pairs reach every peer before any flag does
    __syncthreads();
    if (threadIdx.x < (unsigned)world)
        st_release_sys(reinterpret_cast<unsigned*>(mailboxes[threadIdx.x] + mailbox_flag_offset(epoch, rank)), epoch);
}

__global__ void pairs_wait_kernel(const char* mailbox, int world, unsigned epoch, unsigned long long timeout_ns) {
    if (threadIdx.x >= (unsigned)world) return;
    const unsigned* flag = reinterpret_cast<const unsigned*>(mailbox + mailbox_flag_offset(epoch, threadIdx.x));
    const unsigned long long t0 = globaltimer_ns();
    while (ld_acquire_sys(flag) != epoch) {
        if (globaltimer_ns() - t0 > timeout_ns) {  // never hang the GPU on a missing peer
            atomicOr(reinterpret_cast<unsigned*>(const_cast<char*>(mailbox) + kMailboxErrorWord), 1u << (threadIdx.x & 31));
            return;
        }
        __nanosleep(64);
    }
}

size_t mailbox_bytes(int world, int64_t rows) {
    return mailbox_pairs_offset(world, rows, 1u) + sizeof(float2) * (size_t)world * (size_t)rows;
}

cudaError_t launch_pairs_push(const float* pairs, int64_t rows, void* const* mailboxes, int rank, int world,
                              unsigned epoch, cudaStream_t s) {
    pairs_push_kernel<<<1, 256, 0, s>>>(reinterpret_cast<const float2*>(pairs), rows,
                                         reinterpret_cast<char* const*>(mailboxes), rank, world, epoch);
    return cudaGetLastError();
}

cudaError_t launch_pairs_wait(const void* mailbox, int world, unsigned epoch, unsigned long long timeout_ns,
                              cudaStream_t s) {
    pairs_wait_kernel<<<1, 64, 0, s>>>(static_cast<const char*>(mailbox), world, epoch, timeout_ns);
    return cudaGetLastError();
}

}  // namespace tp
