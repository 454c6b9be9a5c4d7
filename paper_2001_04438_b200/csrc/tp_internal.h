// Internal (C++) interface between the C ABI (tp_api.cu) and the kernels (tp_kernels.cu).
#pragma once
#include <atomic>
#include <cstddef>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

namespace tp {

// Development overrides (environment variables) exist only in builds compiled with
// -DTP_DEV_OVERRIDES (tools/ A/B experiments); a release build always takes the default.
inline int dev_env_int(const char* name, int dflt) {
#ifdef TP_DEV_OVERRIDES
    const char* e = getenv(name);
    return e ? atoi(e) : dflt;
#else
    (void)name;
    return dflt;
#endif
}

// Per-device launch-configuration caches, filled on first use (benign to compute twice; the
// slots are atomics so concurrent host threads never race on them).
constexpr int kMaxDevices = 64;
using DevCache = std::atomic<int>;

// Workspace header: the persistent kernels' work queue and launch epoch.  Zero-filled once at
// allocation; every launch leaves it reusable (the last CTA resets the queue).
struct WsHeader {
    unsigned long long counter;  // next work item
    unsigned exit_ticket;        // CTAs that left the kernel
    unsigned epoch;              // launches completed; row flags are valid when == epoch + 1
    unsigned rows_done;          // kPartial with a fused push: rows whose pair has been pushed
    // watchdog: bit 0 = a wait for a row flag timed out.  Its own 128-byte line: every role
    // polls it while waiting, and the work-queue atomics on `counter` must not queue behind them
    alignas(128) unsigned error;
    unsigned pad_;
    // host-mapped abort word of this device (written by every launch before any wait can time
    // out): raise_abort stores 1 into it so that the next C-ABI call reports TP_EWATCHDOG
    unsigned* abort_host;
};

// The host-mapped abort word of device `dev` (tp_api.cu; allocated on first use).
unsigned* abort_word_device(int dev);

// Mailbox of the one-sided pair exchange, double-buffered by epoch parity (an exchange of epoch e
// uses half e & 1): uint32 flags[2][64] (half h at byte h * kMailboxFlagStride), the error word
// at byte kMailboxErrorWord, then float2 pairs[2][world][rows] from byte kMailboxHeader (half h
// at kMailboxHeader + h * world * rows * 8; rank-major, the layout kFinish's pairs_in reads).
// Two halves suffice: a rank pushes epoch e + 2 only after its finish of e + 1, which waited
// for every rank's push of e + 1, which each rank issues after its own finish of e; so no push
// ever overwrites a half a peer's finish has not read.
constexpr size_t kMailboxFlagStride = 256;
constexpr size_t kMailboxErrorWord = 512;
constexpr size_t kMailboxHeader = 1024;
constexpr int kMailboxMaxWorld = 56;
__host__ __device__ inline size_t mailbox_pairs_offset(int world, int64_t rows, unsigned epoch) {
    return kMailboxHeader + (size_t)(epoch & 1u) * sizeof(float) * 2 * (size_t)world * (size_t)rows;
}
__host__ __device__ inline size_t mailbox_flag_offset(unsigned epoch, int rank) {
    return (size_t)(epoch & 1u) * kMailboxFlagStride + sizeof(unsigned) * (size_t)rank;
}

constexpr unsigned long long kWaitTimeoutNs = 4000000000ull;  // 4 s: only a bug can wait this long

struct WsLayout {
    size_t group_tickets, row_tickets, row_ready, row_clamp;  // control region [0, ctrl_bytes)
    size_t res_vals;  // resident-row kernel: epoch-tagged block values, 16 B per (row, block)
    size_t ctrl_bytes;
    size_t row_stats, block_vals, block_clamp, group_vals, bytes;  // data region
};

struct LaunchOpts {
    int64_t grid_ctas = 0;       // 0 = one full wave of resident CTAs
    int64_t lookahead_rows = 0;  // 0 = automatic
    int force_persistent = 0;    // two-phase schedule even for single-block rows
    int no_tma = 0;              // global loads instead of TMA staging (testing)
    int schedule = 0;            // 0 automatic, 1 stream (re-read), 2 hold, 3 cluster (twopass.h TP_SCHED_*)
    int cluster_size = 0;        // cluster schedule: CTAs per row (0 = automatic)
};

// What the last launch on this thread ran (softmax_last_plan in twopass.h).
struct Plan {
    int kernel = 0;           // 1 general, 2 stream, 3 cluster
    int variant = 0;          // tp_sched.cuh Algo of the kernel instance
    int64_t grid_ctas = 0;
    int cluster_size = 0;
    int64_t lookahead_rows = 0;
    int hold = 0;
};
Plan& last_plan();
// development: cycle counters of the cluster kernel's roles (kProf* in tp_rowcl.cu), or null
void set_profile_buffer(void* p);
unsigned long long* profile_buffer();

size_t workspace_bytes(int64_t rows, int64_t cols);
// The control region's layout depends on (rows, cols): it must be re-zeroed whenever a
// workspace is used with a different shape than its previous launch (tp_api.cu does that).
size_t workspace_ctrl_bytes(int64_t rows, int64_t cols);
// the tail layout of a workspace (a concurrent launch on a cluster launch's last rows)
size_t tail_ws_offset(int64_t rows, int64_t cols);
size_t tail_ctrl_bytes(int64_t rows, int64_t cols);
bool softmax_needs_workspace(int algo, int64_t cols, const LaunchOpts& o);
cudaError_t launch_softmax(int algo, int in_bf16, const void* x, float* y, int64_t rows, int64_t cols, void* ws,
                           const LaunchOpts& o, cudaStream_t s);
// Fused one-sided exchange (tp_ops.cuh push_row_pair / finish_wait): the partial launch pushes
// its row pairs into every mailbox and releases `epoch`; the finish launch awaits the epoch in
// the local mailbox and reads the pairs from it.
struct Exchange {
    void* const* peers = nullptr;  // device array of world mailbox pointers (partial)
    int rank = 0, world = 1;
    unsigned epoch = 0;
    const void* mailbox = nullptr;  // local mailbox (finish)
    unsigned long long wait_ns = 0;
};
cudaError_t launch_partial(int in_bf16, const void* x, int64_t rows, int64_t cols, float* pair_out, void* ws,
                           const LaunchOpts& o, cudaStream_t s, const Exchange* xc = nullptr);
cudaError_t launch_finish(int in_bf16, const void* x, float* y, int64_t rows, int64_t cols, const float* pairs,
                          int world, void* ws, const LaunchOpts& o, cudaStream_t s, const Exchange* xc = nullptr);

// debug / unit-test kernels (tp_debug.cu)
cudaError_t launch_debug(int what, const float* a, const float* b, float* out0, float* out1, int64_t count,
                         cudaStream_t s);
cudaError_t launch_stream_baseline(int what, float* x, float* y, int64_t n, float a, int64_t ctas, cudaStream_t s);
cudaError_t launch_phase_only(int algo, int in_bf16, int phase, const void* x, float* y, int64_t rows, int64_t cols,
                              void* ws, const LaunchOpts& o, cudaStream_t s);
// Sharded Three-Pass (softmax3_max_partial_ex / _sum_partial_ex / _finish_ex): one phase of the
// comparator over the local chunk, statistics from the world's gathered partials.
struct Shard3 {
    const float* maxes = nullptr;  // world x rows (phases 1, 2)
    const float* sums = nullptr;   // world x rows (phase 2)
    int world = 1;
    float* out = nullptr;          // rows: this chunk's max (phase 0) / sum (phase 1)
};
cudaError_t launch_shard3(int algo, int in_bf16, int phase, const void* x, float* y, int64_t rows, int64_t cols,
                          void* ws, const Shard3& sh, const LaunchOpts& o, cudaStream_t s);
cudaError_t launch_copy_probe(const void* x, void* y, int64_t bytes, int64_t chunk_bytes, int stages, int64_t ctas,
                              int backward, cudaStream_t s);
cudaError_t launch_read_probe(const void* x, int64_t bytes, int64_t chunk_bytes, int stages, int64_t ctas, float* y,
                              cudaStream_t s);
cudaError_t launch_exp_sweep(int what, uint32_t bits0, int64_t count, float* o0, float* o1, cudaStream_t s);
cudaError_t launch_exp_fit(const float* c, uint32_t bits0, int64_t count, int stride, unsigned* max_bits,
                           unsigned long long* n_over2, cudaStream_t s);
size_t mailbox_bytes(int world, int64_t rows);
cudaError_t launch_pairs_push(const float* pairs, int64_t rows, void* const* mailboxes, int rank, int world,
                              unsigned epoch, cudaStream_t s);
cudaError_t launch_pairs_wait(const void* mailbox, int world, unsigned epoch, unsigned long long timeout_ns,
                              cudaStream_t s);
cudaError_t launch_bench_compute(int what, int in_bf16, int64_t ctas, int reps, float* sink, cudaStream_t s);

}  // namespace tp
