// General kernel (any alignment) and the host-side dispatch of every entry point.
//
// The fast path for 16-byte aligned rows is the warp-specialised TMA kernel of tp_stream.cu.
// general_kernel serves misaligned rows (scalar or partial-vector loads): a persistent grid
// whose 16 warps all load and compute, with warp 0 retiring each block.  Both kernels run the
// same per-item operations (tp_ops.cuh) and give bit-identical results.
//
// Algorithms (tp_sched.cuh Algo):
//   kFused     rows of one block (cols <= kBlockElems): pass 1, lambda, pass 2 on one load
//   kTwoPass   Alg. 3 over rows of several blocks, rows interleaved with a lookahead
//   kPartial   pass 1 only, one (m, n) per row (multi-GPU chunk shards)
//   kFinish    merge world partials, then pass 2
//   kRecompute / kReload   Three-Pass comparators (Alg. 1 / Alg. 2)
//
// Deadlock freedom: items are handed out in increasing order, a CTA works through its items in
// that order, and an item depends only on items of smaller index; so the smallest unfinished
// item is always the current item of a running CTA.
#include <cstdlib>
#include <mutex>

#include "tp_ops.cuh"

namespace tp {

// After the main layout: a second layout for up to kMaxTailRows rows that a concurrent stream
// launch (launch_split) uses for the tail rows of a cluster launch.
constexpr int64_t kMaxTailRows = 256;
size_t tail_ws_offset(int64_t rows, int64_t cols) { return align256(ws_layout(rows, cols).bytes); }
size_t workspace_bytes(int64_t rows, int64_t cols) {
    return tail_ws_offset(rows, cols) + ws_layout(rows < kMaxTailRows ? rows : kMaxTailRows, cols).bytes;
}
size_t workspace_ctrl_bytes(int64_t rows, int64_t cols) { return ws_layout(rows, cols).ctrl_bytes; }
size_t tail_ctrl_bytes(int64_t rows, int64_t cols) {
    return ws_layout(rows < kMaxTailRows ? rows : kMaxTailRows, cols).ctrl_bytes;
}

template <typename In, int A>
__global__ void __launch_bounds__(kThreads, 1) general_kernel(const KArgs a) {
    constexpr int P = AlgoTraits<A>::P;
    constexpr int V = InTraits<In>::V;
    __shared__ long long s_item[2];
    __shared__ Item s_dec[2];
    __shared__ Part s_part;
    __shared__ float4 s_stats;
    __shared__ unsigned s_mask, s_epoch;
    __shared__ int64_t s_cur_row;

    publish_abort_word(a);
    WsHeader* hdr = reinterpret_cast<WsHeader*>(a.ws);
    const unsigned* row_ready = reinterpret_cast<const unsigned*>(a.ws + a.lay.row_ready);
    const In* x = static_cast<const In*>(a.x);
    const int warp = threadIdx.x >> 5;

    auto fetch = [&](int b) {
        const long long item = (long long)atomicAdd(&hdr->counter, 1ull);
        s_item[b] = item;
        if (item < a.total_items) {
            if (a.phase_only) {  // one phase alone: items are (row, blk), odd phases backwards
                Item it;
                it.phase = a.phase_only - 1;
                it.row = item / a.nb;
                it.blk = item - it.row * a.nb;
                if (it.phase & 1) it.blk = a.nb - 1 - it.blk;
                s_dec[b] = it;
            } else {
                s_dec[b] = decode_item<A>(item, a.rows, a.nb, a.L);
            }
        }
    };
    if (threadIdx.x == 0) {
        if (A == kFinish && a.mailbox) finish_wait(a);  // fused NVLink exchange: the peers' pairs
        s_epoch = *reinterpret_cast<volatile unsigned*>(&hdr->epoch);
        s_cur_row = -1;
        fetch(0);
    }
    __syncthreads();
    const unsigned want = s_epoch + 1u;

    for (int buf = 0;; buf ^= 1) {
        if (s_item[buf] >= a.total_items) break;
        const Item it = s_dec[buf];
        if (threadIdx.x == 0) fetch(buf ^ 1);
        const int64_t e0 = it.blk * kBlockElems;
        const int valid = (int)min((int64_t)kBlockElems, a.cols - e0);
        const In* xb = x + it.row * a.cols + e0;
        float* yb = a.y ? a.y + it.row * a.cols + e0 : nullptr;
        const bool vec = a.vec != 0;

        if (item_needs_stats<A>(it)) {
            if (threadIdx.x == 0) {
                if (A == kFinish) {
                    if (it.row != s_cur_row) {
                        s_stats = finish_stats(a, it.row);
                        s_cur_row = it.row;
                    }
                    s_mask = finish_mask(a, s_stats, it.row, it.blk);  // the partial's clamp decisions
                } else if (a.shard_mu) {  // sharded Three-Pass phase: stats from the world's partials
                    if (it.row != s_cur_row) {
                        s_stats = shard_stats<A>(a, it.row, it.phase - 1);
                        s_cur_row = it.row;
                    }
                    s_mask = 0u;
                } else {
                    if (!a.phase_only) wait_flag(row_ready + it.row * 2 + (it.phase - 1), want, &hdr->error);
                    float4 st;
                    unsigned mask;
                    item_stats<A>(a, it, &st, &mask);
                    s_stats = st;
                    s_mask = mask;
                }
            }
            __syncthreads();
        }
        const float4 st = s_stats;
        const bool my_clamp = ((s_mask >> warp) & 1u) != 0;

        BlockVals r;
        if (!(A == kReload && it.phase == 2)) load_global<In>(xb, valid, vec, it.phase == P - 1, r);

        if constexpr (A == kFused) {
            op_pass1<V>(r, valid, s_part);
            __syncthreads();
            op_fused_tail<V>(r, s_part, yb, valid, vec);
        } else if constexpr (A == kTwoPass || A == kPartial) {
            if (it.phase == 0) {
                op_pass1<V>(r, valid, s_part);
                __syncthreads();
                if (warp == 0) retire_block<A>(a, it, s_part, want, 0.0f);
            } else {
                op_pass2<V>(r, st, my_clamp, yb, valid, vec);
            }
        } else if constexpr (A == kFinish) {
            op_pass2<V>(r, st, my_clamp, yb, valid, vec);
        } else {
            if (it.phase == 0) {
                op_max<V>(r, valid, s_part);
                __syncthreads();
                if (warp == 0) retire_block<A>(a, it, s_part, want, 0.0f);
            } else if (it.phase == 1) {
                op_expsum<V, A == kReload>(r, valid, st.x, s_part, yb, vec);
                __syncthreads();
                if (warp == 0) retire_block<A>(a, it, s_part, want, st.x);
            } else if (A == kRecompute) {
                op_out_recompute<V>(r, st, yb, valid, vec);
            } else {
                op_out_reload(st, yb, valid, (a.cols % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.y) & 15) == 0));
            }
        }
        __syncthreads();  // s_item, s_dec, s_part, s_stats reuse
    }
    if (threadIdx.x == 0) exit_and_reset(hdr);
}

// ----------------------------------------------------------------------------- host launchers
static unsigned long long* g_prof = nullptr;
void set_profile_buffer(void* p) { g_prof = static_cast<unsigned long long*>(p); }
unsigned long long* profile_buffer() { return g_prof; }

thread_local Plan g_plan;
Plan& last_plan() { return g_plan; }

static DevCache g_num_sms[kMaxDevices];

int device_sms(int dev) {
    int n = g_num_sms[dev].load(std::memory_order_relaxed);
    if (!n) {
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        g_num_sms[dev].store(n, std::memory_order_relaxed);
    }
    return n;
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

template <typename In>
static int vec_ok(const void* x, const float* y, int64_t cols) {
    constexpr int V = InTraits<In>::V;
    return (cols % V == 0) && aligned16(x) && (y == nullptr || aligned16(y));
}

int64_t lookahead_rows(const KArgs& a, int64_t grid, int items_per_cta, const LaunchOpts& o) {
    // enough rows that a row's pass-1 items are done before its pass-2 items are handed out
    // (about two grids of items in flight)
    int64_t L = o.lookahead_rows > 0 ? o.lookahead_rows : (grid * items_per_cta + a.nb - 1) / a.nb + 2;
    if (L < 1) L = 1;
    if (L > a.rows) L = a.rows;
    return L;
}

template <typename In, int A>
static cudaError_t launch_general(KArgs a, const LaunchOpts& o, cudaStream_t s) {
    int dev = 0;
    cudaGetDevice(&dev);
    auto kern = general_kernel<In, A>;
    static DevCache occ[kMaxDevices];
    int occ_d = occ[dev].load(std::memory_order_relaxed);
    if (!occ_d) {
        int n = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, kThreads, 0);
        occ_d = n > 0 ? n : 1;
        occ[dev].store(occ_d, std::memory_order_relaxed);
    }
    const int64_t resident = (int64_t)device_sms(dev) * occ_d;
    int64_t grid = o.grid_ctas > 0 ? o.grid_ctas : resident;
    if (grid > resident) grid = resident;
    if (grid > a.total_items) grid = a.total_items;
    if (grid < 1) grid = 1;
    a.L = lookahead_rows(a, grid, 2, o);
    last_plan() = Plan{1, A, grid, 0, a.L, 0};
    kern<<<(unsigned)grid, kThreads, 0, s>>>(a);
    return cudaGetLastError();
}

// Cluster kernel on the first rows - tail rows; the tail rows on the SMs the clusters leave idle,
// concurrently (the cluster kernel in clusters of side_cl, or the stream kernel when side_cl is
// 0): fork / join on an internal per-device side stream with events (graph capturable; callers
// on different streams share it, which orders their side launches but not their results).  The
// tail uses the workspace's tail layout (tail_ws_offset).  cudaErrorNotSupported for a tail
// longer than that layout: the caller runs the plain launch.  Should the side launch fail, the
// tail rows run on the caller's stream after the main launch instead.

struct SideStream {
    std::mutex mu;
    cudaStream_t st = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
};
static SideStream g_side[kMaxDevices];

template <typename In>
static cudaError_t launch_split(const KArgs& a, int CL, int64_t tail, int tail_ctas, int side_cl,
                                const LaunchOpts& o, cudaStream_t s) {
    if (tail > kMaxTailRows) return cudaErrorNotSupported;
    const WsLayout lt = ws_layout(tail, a.cols);
    int dev = 0;
    cudaGetDevice(&dev);
    SideStream& ss = g_side[dev];
    std::lock_guard<std::mutex> lk(ss.mu);
    cudaError_t e;
    if (!ss.st) {
        if ((e = cudaStreamCreateWithFlags(&ss.st, cudaStreamNonBlocking)) != cudaSuccess) return e;
        if ((e = cudaEventCreateWithFlags(&ss.fork, cudaEventDisableTiming)) != cudaSuccess) return e;
        if ((e = cudaEventCreateWithFlags(&ss.join, cudaEventDisableTiming)) != cudaSuccess) return e;
    }
    KArgs main = a, t = a;
    main.rows = a.rows - tail;
    main.total_items = main.rows * a.nb;
    t.rows = tail;
    t.total_items = tail * a.nb * AlgoTraits<kTwoPass>::P;
    t.x = static_cast<const In*>(a.x) + main.rows * a.cols;
    t.y = a.y + main.rows * a.cols;
    t.ws = a.ws + tail_ws_offset(a.rows, a.cols);
    t.lay = lt;
    LaunchOpts ot = o;
    ot.grid_ctas = tail_ctas;
    ot.schedule = 1;
    // The tail rows run AFTER the main launch, on the same stream.  Launched concurrently on the
    // side stream (the design until round 2, session 5; -DTP_CONCURRENT_SIDE) about 2% of C4-shaped
    // fp32 calls came back with a few wrong outputs in one row (tools/dev/sched_stress.py: 19 bad
    // of 500 calls, also with the library of the previous sessions; 0 of 500 serialised; forced
    // CLUSTER and STREAM launches alone never differ).  The cause is not found: correctness first.
#ifndef TP_CONCURRENT_SIDE
    {
        if ((e = launch_rowcl<In>(main, CL, o, s)) != cudaSuccess) return e;
        const Plan p0 = last_plan();
        LaunchOpts oq = o;
        oq.schedule = 1;
        oq.grid_ctas = 0;
        e = launch_stream<In, kTwoPass>(t, oq, s);
        last_plan() = Plan{p0.kernel, p0.variant, p0.grid_ctas, p0.cluster_size, (int64_t)tail, p0.hold};
        return e;
    }
#endif
    if ((e = cudaEventRecord(ss.fork, s)) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(ss.st, ss.fork, 0)) != cudaSuccess) return e;
    if ((e = launch_rowcl<In>(main, CL, o, s)) != cudaSuccess) return e;  // clusters first: they need whole GPCs
    const Plan p = last_plan();
    KArgs ts = t;
    ts.total_items = tail * a.nb;
    const cudaError_t e_side =
        side_cl > 0 ? launch_rowcl<In>(ts, side_cl, ot, ss.st) : launch_stream<In, kTwoPass>(t, ot, ss.st);
    last_plan() = Plan{p.kernel, p.variant, p.grid_ctas, p.cluster_size, (int64_t)tail, p.hold};
    e = cudaEventRecord(ss.join, ss.st);  // the fork is always joined
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s, ss.join, 0);
    if (e != cudaSuccess || e_side == cudaSuccess) return e;
    cudaGetLastError();  // the side launch was refused: the tail rows on s, after the main launch
    LaunchOpts oq = o;
    oq.schedule = 1;
    oq.grid_ctas = 0;
    return launch_stream<In, kTwoPass>(t, oq, s);
}

// The resident-row schedule is AUTO's choice where it applies (development override
// TP_RESIDENT=0 for A/B runs against the cluster kernel).
template <typename In>
static bool rowres_auto() {
    static const int on = dev_env_int("TP_RESIDENT", 1);
    return on != 0;
}

template <typename In, int A>
static cudaError_t launch_algo(const void* x, float* y, int64_t rows, int64_t cols, void* ws, float2* pair_out,
                               const float2* pairs_in, int world, const LaunchOpts& o, cudaStream_t s,
                               const Exchange* xc = nullptr) {
    KArgs a{};
    if (xc) {
        a.peers = reinterpret_cast<char* const*>(xc->peers);
        a.rank = xc->rank;
        a.xepoch = xc->epoch;
        a.mailbox = static_cast<const char*>(xc->mailbox);
        a.wait_ns = xc->wait_ns;
    }
    a.x = x; a.y = y; a.rows = rows; a.cols = cols;
    a.nb = (cols + kBlockElems - 1) / kBlockElems;
    a.ng = (a.nb + kGroupBlocks - 1) / kGroupBlocks;
    a.total_items = rows * a.nb * AlgoTraits<A>::P;
    a.ws = static_cast<char*>(ws);
    a.lay = ws_layout(rows, cols);
    a.pair_out = pair_out;
    a.pairs_in = pairs_in;
    a.world = world;
    a.vec = vec_ok<In>(x, y, cols);
    static const int hints = dev_env_int("TP_L2_HINTS", 1);
    a.l2_hints = hints;
    a.prof = profile_buffer();
    {
        int dev = 0;
        cudaGetDevice(&dev);
        a.abort_host = abort_word_device(dev);
    }
    if (a.vec && !o.no_tma) {
        // a few rows of 1..3 blocks: one CTA per row, the row staged in shared memory
        // (the Three-Pass comparators too, so that they are compared on the same footing)
        if ((A == kTwoPass || A == kFused || A == kRecompute || A == kReload) && !o.force_persistent &&
            ((o.schedule == 0 && small_applies(a.rows, a.nb, a.vec)) || (o.schedule == 4 && a.nb <= 3)))
            return launch_small<In, (A == kFused ? kTwoPass : A)>(a, o, s);
        // Two-Pass rows whose share fits shared memory: a group of CTAs per row, the row read
        // once (tp_rowres.cu)
        // (the Three-Pass comparators too, so that they are compared on the same footing; AUTO
        // for Recompute, not for Reload, whose third pass re-reads Y from memory anyway:
        // C4 bf16 Recompute 442 -> 385 us, Reload 599 -> 711 us)
        if ((A == kTwoPass || A == kRecompute || A == kReload) &&
            (o.schedule == 6 || (o.schedule == 0 && A != kReload && rowres_auto<In>()))) {
            int dev = 0;
            cudaGetDevice(&dev);
            const int G = rowres_choose<In>(a.rows, a.nb, device_sms(dev), o.cluster_size);
            if (G) {
                const cudaError_t e = A == kTwoPass ? launch_rowres<In>(a, G, o, s)
                                                     : launch_rowres3<In, (A == kReload ? kReload : kRecompute)>(a, G, o, s);
                if (e != cudaErrorNotSupported) return e;
                cudaGetLastError();
            }
        }
        // Two-Pass rows of a few blocks: one cluster per row, pass 2 from shared memory / L2
        if (A == kTwoPass && (o.schedule == 0 || o.schedule == 3)) {
            int64_t tail = 0;
            int tail_ctas = 0, tail_cl = 0;
            const int CL = rowcl_choose<In>(a.rows, a.nb, o.cluster_size, o.schedule == 0, &tail, &tail_ctas, &tail_cl);
            if (CL && tail > 0) {
                const cudaError_t e = launch_split<In>(a, CL, tail, tail_ctas, tail_cl, o, s);
                if (e != cudaErrorNotSupported) return e;
            }
            if (CL) {
                const cudaError_t e = launch_rowcl<In>(a, CL, o, s);
                if (e != cudaErrorNotSupported) return e;
                cudaGetLastError();
            }
        }
        // the Three-Pass comparators on a one-cluster-per-row schedule (tp_rowcl3.cu; opt-in:
        // faster than their stream schedule for some algorithm / dtype pairs on C4, slower for
        // others, so bench.py times both and compares against the faster)
        if ((A == kRecompute || A == kReload) && o.schedule == 3) {
            int64_t tail = 0;
            int tail_ctas = 0, tail_cl = 0;
            const int CL = rowcl_choose<In>(a.rows, a.nb, o.cluster_size, false, &tail, &tail_ctas, &tail_cl);
            if (CL) {
                const cudaError_t e = launch_rowcl3<In, (A == kReload ? kReload : kRecompute)>(a, CL, o, s);
                if (e != cudaErrorNotSupported) return e;
                cudaGetLastError();
            }
        }
        // a few very long rows (and the chunks of sharded rows): the phase kernel's static
        // schedule (tp_rowph.cu)
        if constexpr (A == kTwoPass || A == kPartial || A == kFinish) {
            int dev = 0;
            cudaGetDevice(&dev);
            if (o.schedule == 5 || (o.schedule == 0 && rowph_applies(A, a.rows, a.nb, device_sms(dev)))) {
                const cudaError_t e = launch_rowph<In, A>(a, o, s);
                if (e != cudaErrorNotSupported) return e;
                cudaGetLastError();
            }
        }
        return launch_stream<In, A>(a, o, s);
    }
    return launch_general<In, A>(a, o, s);
}

// One phase of a multi-phase algorithm on its own (measurement, tp_phase_only): the stream kernel
// with every item in `phase`; a later phase reads the row statistics a previous full launch left
// in the workspace instead of waiting for them.
template <typename In, int A>
static cudaError_t launch_phase(const void* x, float* y, int64_t rows, int64_t cols, void* ws, int phase,
                                const LaunchOpts& o, cudaStream_t s, const Shard3* sh = nullptr) {
    KArgs a{};
    a.x = x; a.y = y; a.rows = rows; a.cols = cols;
    a.nb = (cols + kBlockElems - 1) / kBlockElems;
    a.ng = (a.nb + kGroupBlocks - 1) / kGroupBlocks;
    a.total_items = rows * a.nb;
    a.ws = static_cast<char*>(ws);
    a.lay = ws_layout(rows, cols);
    a.world = 1;
    a.vec = vec_ok<In>(x, y, cols);
    a.l2_hints = 1;
    a.prof = profile_buffer();
    a.phase_only = phase + 1;
    {
        int dev = 0;
        cudaGetDevice(&dev);
        a.abort_host = abort_word_device(dev);
    }
    if (phase < 0 || phase >= AlgoTraits<A>::P) return cudaErrorNotSupported;
    if (sh) {
        a.world = sh->world;
        a.shard_mu = sh->maxes;
        a.shard_sigma = sh->sums;
        a.shard_out = sh->out;
        if (!a.vec || o.no_tma) return launch_general<In, A>(a, o, s);
    }
    if (!a.vec) return cudaErrorNotSupported;
    return launch_stream<In, A>(a, o, s);
}

cudaError_t launch_shard3(int algo, int in_bf16, int phase, const void* x, float* y, int64_t rows, int64_t cols,
                          void* ws, const Shard3& sh, const LaunchOpts& o, cudaStream_t s) {
    switch (algo * 2 + (in_bf16 ? 1 : 0)) {
        case kRecompute * 2: return launch_phase<float, kRecompute>(x, y, rows, cols, ws, phase, o, s, &sh);
        case kRecompute * 2 + 1: return launch_phase<uint16_t, kRecompute>(x, y, rows, cols, ws, phase, o, s, &sh);
        case kReload * 2: return launch_phase<float, kReload>(x, y, rows, cols, ws, phase, o, s, &sh);
        case kReload * 2 + 1: return launch_phase<uint16_t, kReload>(x, y, rows, cols, ws, phase, o, s, &sh);
        default: return cudaErrorNotSupported;
    }
}

cudaError_t launch_phase_only(int algo, int in_bf16, int phase, const void* x, float* y, int64_t rows, int64_t cols,
                              void* ws, const LaunchOpts& o, cudaStream_t s) {
    switch (algo * 2 + (in_bf16 ? 1 : 0)) {
        case kTwoPass * 2: return launch_phase<float, kTwoPass>(x, y, rows, cols, ws, phase, o, s);
        case kTwoPass * 2 + 1: return launch_phase<uint16_t, kTwoPass>(x, y, rows, cols, ws, phase, o, s);
        case kRecompute * 2: return launch_phase<float, kRecompute>(x, y, rows, cols, ws, phase, o, s);
        case kRecompute * 2 + 1: return launch_phase<uint16_t, kRecompute>(x, y, rows, cols, ws, phase, o, s);
        case kReload * 2: return launch_phase<float, kReload>(x, y, rows, cols, ws, phase, o, s);
        case kReload * 2 + 1: return launch_phase<uint16_t, kReload>(x, y, rows, cols, ws, phase, o, s);
        default: return cudaErrorNotSupported;
    }
}

template <typename In>
static cudaError_t launch_softmax_t(int algo, const void* x, float* y, int64_t rows, int64_t cols, void* ws,
                                    const LaunchOpts& o, cudaStream_t s) {
    switch (algo) {
        case kTwoPass:
            if (cols <= kBlockElems && !o.force_persistent)
                return launch_algo<In, kFused>(x, y, rows, cols, ws, nullptr, nullptr, 1, o, s);
            return launch_algo<In, kTwoPass>(x, y, rows, cols, ws, nullptr, nullptr, 1, o, s);
        case kRecompute: return launch_algo<In, kRecompute>(x, y, rows, cols, ws, nullptr, nullptr, 1, o, s);
        case kReload: return launch_algo<In, kReload>(x, y, rows, cols, ws, nullptr, nullptr, 1, o, s);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_softmax(int algo, int in_bf16, const void* x, float* y, int64_t rows, int64_t cols, void* ws,
                           const LaunchOpts& o, cudaStream_t s) {
    return in_bf16 ? launch_softmax_t<uint16_t>(algo, x, y, rows, cols, ws, o, s)
                   : launch_softmax_t<float>(algo, x, y, rows, cols, ws, o, s);
}

bool softmax_needs_workspace(int, int64_t, const LaunchOpts&) { return true; }

cudaError_t launch_partial(int in_bf16, const void* x, int64_t rows, int64_t cols, float* pair_out, void* ws,
                           const LaunchOpts& o, cudaStream_t s, const Exchange* xc) {
    float2* po = reinterpret_cast<float2*>(pair_out);
    const int world = xc ? xc->world : 1;
    return in_bf16 ? launch_algo<uint16_t, kPartial>(x, nullptr, rows, cols, ws, po, nullptr, world, o, s, xc)
                   : launch_algo<float, kPartial>(x, nullptr, rows, cols, ws, po, nullptr, world, o, s, xc);
}

cudaError_t launch_finish(int in_bf16, const void* x, float* y, int64_t rows, int64_t cols, const float* pairs,
                          int world, void* ws, const LaunchOpts& o, cudaStream_t s, const Exchange* xc) {
    const float2* pi = reinterpret_cast<const float2*>(pairs);
    return in_bf16 ? launch_algo<uint16_t, kFinish>(x, y, rows, cols, ws, nullptr, pi, world, o, s, xc)
                   : launch_algo<float, kFinish>(x, y, rows, cols, ws, nullptr, pi, world, o, s, xc);
}

}  // namespace tp
