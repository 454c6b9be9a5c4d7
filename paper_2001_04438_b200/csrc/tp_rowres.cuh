// Shared pieces of the resident-row kernels (tp_rowres.cu: Two-Pass, tp_rowres3.cu: the
// Three-Pass comparators): limits, role warps, staging depth, tagged 64-bit slot accesses.
#pragma once
#include "tp_ops.cuh"

namespace tp {

constexpr int kResMaxLocal = 3;           // blocks staged per CTA and row
constexpr int kResMaxBuf = 7;             // rows staged per CTA (bf16 rows of one block per CTA)
constexpr int kResSlots = 8;              // staged blocks per CTA (nbuf x nloc <= 7 for every dtype)
constexpr int kResThreads = kThreads + 128;  // 16 compute warps + 4 service warps
constexpr int kResMaxNb = kGroupBlocks;   // rows of at most one canonical group (one warp tree)
constexpr int kResSmemMax = 227 * 1024 - 1792;  // dynamic shared memory (static arrays ~1.5 KB)

template <typename In>
constexpr int res_max_local() {  // blocks per row and CTA (at least two rows staged)
    const int b = kResSmemMax / (2 * kBlockElems * (int)sizeof(In));
    return b < kResMaxLocal ? b : kResMaxLocal;
}
// rows staged per CTA for shares of `per` blocks
template <typename In>
inline int res_nbuf(int per) {
    int n = kResSmemMax / (per * kBlockElems * (int)sizeof(In));
    if (n > kResMaxBuf) n = kResMaxBuf;
    return n * per <= kResSlots ? n : kResSlots / per;
}

__device__ __forceinline__ void st_relaxed_gpu_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_gpu_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// k / d and k % d for the staging ring (d = rows staged, 2..8; k = a group's row index, < 2^29:
// launch_rowres* refuse more rows per group) by one multiply-high with a magic computed once per
// thread.  The 64-bit `k % nbuf`, `k / nbuf` by a runtime divisor used here first are subroutines
// of ~100 dependent instructions, several per row on every compute warp at once: measured,
// C4 bf16 300 -> see DESIGN (they were 13% of the kernel's stall samples).
constexpr int64_t kResMaxRowsPerGroup = (int64_t)1 << 29;
struct ResDiv {
    unsigned magic;
    int d;
    __device__ __forceinline__ explicit ResDiv(int d_) : magic(0xffffffffu / (unsigned)d_ + 1u), d(d_) {}
    __device__ __forceinline__ int quot(int64_t k) const { return (int)__umulhi((unsigned)k, magic); }
    __device__ __forceinline__ int rem(int64_t k) const { return (int)((unsigned)k - (unsigned)quot(k) * (unsigned)d); }
};

constexpr int kResPostWarp = kWarps, kResStatsWarp = kWarps + 1, kResLoadWarp = kWarps + 3;

}  // namespace tp
