// C ABI of libtwopass.so (declared and documented in include/twopass.h): argument checks,
// the internal per-device workspace, the host-buffer (end-to-end) pipeline.  No arithmetic of
// the method lives here; every step runs in the kernels of tp_kernels.cu.
#include <cstdlib>
#include <cstring>

#include <cuda.h>
#include <mutex>
#include <vector>
#include <unordered_map>
#include <utility>

#include "../../include/twopass.h"
#include "tp_internal.h"

namespace {

thread_local int g_last_cuda_error = 0;

int cuda_fail(cudaError_t e) {
    g_last_cuda_error = (int)e;
    return TP_ECUDA;
}

constexpr int kMaxDev = 64;
constexpr int kHostStreams = 4;                // host pipeline: stream slots (default use: 2)
constexpr size_t kHostSlabBytes = 64ull << 20;  // host pipeline: input bytes per slab
// Measured on B200 (tools/pcie_probe.py, C4): H2D 14.8 ms and D2H 15.2 ms alone, 17.0 ms at
// once; 2 streams x 64 MB slabs 18.1 ms end to end; smaller slabs or more streams are slower.

// One in-flight host-buffer call: its streams, events and device staging (cached between calls).
struct HostSlot {
    // row slabs: one staging slot per stream
    void* hx_dev[kHostStreams] = {};
    float* hy_dev[kHostStreams] = {};
    size_t stage_bytes_x = 0, stage_bytes_y = 0;
    void* hws[kHostStreams] = {};
    size_t hws_bytes = 0;
    // host pipeline, single long row: whole-row buffers, chunk workspace, chunk pairs
    void* row_x = nullptr;
    void* row_y = nullptr;
    size_t row_x_bytes = 0, row_y_bytes = 0;
    void* row_ws = nullptr;
    size_t row_ws_bytes = 0;
    void* pairs = nullptr;
    size_t pairs_bytes = 0;
    cudaStream_t st[kHostStreams] = {};
    cudaEvent_t ev[64];
    bool ev_init = false;
};
// slot 0: the synchronous call; 1 and 2: submitted calls in turn, so that one call's uploads
// overlap the previous call's downloads (the two PCIe directions at once)
constexpr int kHostSlots = 3;
constexpr int kTicketEvents = 16;  // submitted calls that can be waited for individually
struct DevState {
    std::mutex mu;
    void* ws = nullptr;
    size_t ws_bytes = 0;
    HostSlot hs[kHostSlots];
    unsigned long long tickets = 0;
    cudaEvent_t tev[kTicketEvents];
    bool tev_init = false;
};
DevState g_dev[kMaxDev];

int current_device(int* dev) {
    cudaError_t e = cudaGetDevice(dev);
    if (e != cudaSuccess) return e == cudaErrorNoDevice ? TP_ENODEV : cuda_fail(e);
    if (*dev < 0 || *dev >= kMaxDev) return TP_EINVAL;
    return TP_OK;
}

// Last (rows, cols) each workspace was launched with.  The kernels leave the control region
// reusable for the same shape; a different shape moves the tickets and flags, so the control
// region is zeroed (stream-ordered memset) before the launch.
std::mutex g_shape_mu;
std::unordered_map<const void*, std::pair<int64_t, int64_t>> g_ws_shape;

int prepare_ws(void* ws, int64_t rows, int64_t cols, cudaStream_t s) {
    {
        std::lock_guard<std::mutex> lk(g_shape_mu);
        auto it = g_ws_shape.find(ws);
        if (it != g_ws_shape.end() && it->second == std::make_pair(rows, cols)) return TP_OK;
        g_ws_shape[ws] = std::make_pair(rows, cols);
    }
    cudaError_t e = cudaMemsetAsync(ws, 0, tp::workspace_ctrl_bytes(rows, cols), s);
    if (e == cudaSuccess)
        e = cudaMemsetAsync((char*)ws + tp::tail_ws_offset(rows, cols), 0, tp::tail_ctrl_bytes(rows, cols), s);
    return e == cudaSuccess ? TP_OK : cuda_fail(e);
}

void forget_ws(const void* ws) {
    std::lock_guard<std::mutex> lk(g_shape_mu);
    g_ws_shape.erase(ws);
}

// ---- watchdog aborts (include/twopass.h TP_EWATCHDOG).  A launch that gives up on a wait
// stores 1 into its device's word of this host-mapped array (tp_sched.cuh raise_abort); the
// next call on that device sees it, clears it, forgets every workspace's shape (so every
// control region, the header's error word included, is re-zeroed before its next launch) and
// returns TP_EWATCHDOG without launching anything.
std::once_flag g_abort_once;
unsigned* g_abort_host = nullptr;   // kMaxDev words, host view
unsigned* g_abort_dev = nullptr;    // the same words, device view

void abort_init() {
    std::call_once(g_abort_once, [] {
        void* p = nullptr;
        if (cudaHostAlloc(&p, sizeof(unsigned) * kMaxDev, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess) {
            cudaGetLastError();
            return;  // no abort reporting (the workspace flags still record aborts)
        }
        memset(p, 0, sizeof(unsigned) * kMaxDev);
        void* d = nullptr;
        if (cudaHostGetDevicePointer(&d, p, 0) != cudaSuccess) {
            cudaGetLastError();
            d = p;  // unified addressing: the host pointer is valid on the device
        }
        g_abort_host = static_cast<unsigned*>(p);
        g_abort_dev = static_cast<unsigned*>(d);
    });
}

bool take_abort(int dev) {
    abort_init();
    if (!g_abort_host || !__atomic_load_n(&g_abort_host[dev], __ATOMIC_ACQUIRE)) return false;
    __atomic_store_n(&g_abort_host[dev], 0u, __ATOMIC_RELEASE);
    std::lock_guard<std::mutex> lk(g_shape_mu);
    g_ws_shape.clear();
    return true;
}

// Grow-only zero-filled device buffer.  Growth synchronises the device (documented).
int ensure_zeroed(void** p, size_t* have, size_t need) {
    if (*have >= need && *p) return TP_OK;
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_fail(e);
    if (*p) {
        cudaFree(*p);
        forget_ws(*p);
    }
    *p = nullptr;
    *have = 0;
    e = cudaMalloc(p, need);
    if (e != cudaSuccess) return cuda_fail(e);
    e = cudaMemset(*p, 0, need);
    if (e != cudaSuccess) return cuda_fail(e);
    *have = need;
    return TP_OK;
}

int internal_workspace(size_t need, void** ws) {
    int dev;
    int st = current_device(&dev);
    if (st) return st;
    DevState& d = g_dev[dev];
    std::lock_guard<std::mutex> lk(d.mu);
    st = ensure_zeroed(&d.ws, &d.ws_bytes, need < 4096 ? 4096 : need);
    if (st) return st;
    *ws = d.ws;
    return TP_OK;
}

bool overlap_bad(const void* x, size_t xbytes, const void* y, size_t ybytes, bool allow_exact) {
    const uintptr_t x0 = (uintptr_t)x, x1 = x0 + xbytes, y0 = (uintptr_t)y, y1 = y0 + ybytes;
    if (x1 <= y0 || y1 <= x0) return false;
    return !(allow_exact && x0 == y0 && xbytes == ybytes);
}

int check_args(int in_dtype, const void* x, const float* y, int64_t rows, int64_t cols, bool need_y) {
    if (!x || (need_y && !y)) return TP_EINVAL;
    int dev;  // a usable device, and one the per-device tables (kMaxDev entries) cover
    if (const int st = current_device(&dev)) return st;
    if (rows < 1 || cols < 1) return TP_EINVAL;
    if (in_dtype != TP_IN_F32 && in_dtype != TP_IN_BF16) return TP_EINVAL;
    if (rows > (int64_t(1) << 40) / cols) return TP_EINVAL;  // 2^40 elements: far beyond HBM
    if (need_y) {
        const size_t esz = in_dtype == TP_IN_BF16 ? 2 : 4;
        if (overlap_bad(x, (size_t)(rows * cols) * esz, y, (size_t)(rows * cols) * 4, in_dtype == TP_IN_F32))
            return TP_EINVAL;
    }
    if (take_abort(dev)) return TP_EWATCHDOG;  // an earlier launch on this device gave up
    return TP_OK;
}

tp::LaunchOpts to_opts(const softmax_opts* o) {
    tp::LaunchOpts L;
    if (o) {
        L.grid_ctas = o->grid_ctas;
        L.lookahead_rows = o->lookahead_rows;
        L.force_persistent = o->force_persistent;
        L.no_tma = o->disable_tma;
        L.schedule = o->schedule;
        L.cluster_size = o->cluster_size;
    }
    return L;
}

int run_softmax(int algo, int in_dtype, const void* x, float* y, int64_t rows, int64_t cols, void* ws,
                size_t ws_bytes, const softmax_opts* opts, cudaStream_t s) {
    int st = check_args(in_dtype, x, y, rows, cols, true);
    if (st) return st;
    if (algo != TP_ALGO_TWO_PASS && algo != TP_ALGO_THREE_PASS_RECOMPUTE && algo != TP_ALGO_THREE_PASS_RELOAD)
        return TP_EINVAL;
    const tp::LaunchOpts lo = to_opts(opts);
    if (tp::softmax_needs_workspace(algo, cols, lo)) {
        const size_t need = tp::workspace_bytes(rows, cols);
        if (ws) {
            if (ws_bytes < need) return TP_EINVAL;
        } else {
            st = internal_workspace(need, &ws);
            if (st) return st;
        }
    }
    if (tp::softmax_needs_workspace(algo, cols, lo) && (st = prepare_ws(ws, rows, cols, s))) return st;
    cudaError_t e = tp::launch_softmax(algo, in_dtype == TP_IN_BF16, x, y, rows, cols, ws, lo, s);
    return e == cudaSuccess ? TP_OK : cuda_fail(e);
}

int run_partial(int in_dtype, const void* x, int64_t rows, int64_t cols, float* pair_out, void* ws,
                size_t ws_bytes, const softmax_opts* opts, cudaStream_t s) {
    int st = check_args(in_dtype, x, nullptr, rows, cols, false);
    if (st) return st;
    if (!pair_out) return TP_EINVAL;
    const size_t need = tp::workspace_bytes(rows, cols);
    if (ws) {
        if (ws_bytes < need) return TP_EINVAL;
    } else {
        st = internal_workspace(need, &ws);
        if (st) return st;
    }
    if ((st = prepare_ws(ws, rows, cols, s))) return st;
    cudaError_t e = tp::launch_partial(in_dtype == TP_IN_BF16, x, rows, cols, pair_out, ws, to_opts(opts), s);
    return e == cudaSuccess ? TP_OK : cuda_fail(e);
}

// A workspace argument (or the internal one for NULL), checked and prepared for (rows, cols).
int workspace_for(void** ws, size_t ws_bytes, int64_t rows, int64_t cols, cudaStream_t s) {
    const size_t need = tp::workspace_bytes(rows, cols);
    int st;
    if (*ws) {
        if (ws_bytes < need) return TP_EINVAL;
    } else if ((st = internal_workspace(need, ws))) {
        return st;
    }
    return prepare_ws(*ws, rows, cols, s);
}

int run_finish(int in_dtype, const void* x, float* y, int64_t rows, int64_t cols, const float* pairs, int world,
               void* ws, size_t ws_bytes, const softmax_opts* opts, cudaStream_t s) {
    int st = check_args(in_dtype, x, y, rows, cols, true);
    if (st) return st;
    if (!pairs || world < 1 || (!ws && ws_bytes)) return TP_EINVAL;
    if ((st = workspace_for(&ws, ws_bytes, rows, cols, s))) return st;
    cudaError_t e = tp::launch_finish(in_dtype == TP_IN_BF16, x, y, rows, cols, pairs, world, ws, to_opts(opts), s);
    return e == cudaSuccess ? TP_OK : cuda_fail(e);
}

// ---------------------------------------------------------------- host-buffer pipeline
// Enqueue one call on the slot's streams (caller holds the device lock); *last = the stream
// whose completion completes the call.
int host_enqueue(HostSlot& d, int in_dtype, const void* hx, float* hy, int64_t rows, int64_t cols,
                 cudaStream_t* last) {
    int st = TP_OK;
    cudaError_t e;
    if (!d.st[0]) {
        for (int i = 0; i < kHostStreams; ++i) {
            e = cudaStreamCreateWithFlags(&d.st[i], cudaStreamNonBlocking);
            if (e != cudaSuccess) return cuda_fail(e);
        }
    }
    if (!d.ev_init) {
        for (auto& ev : d.ev) {
            e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
            if (e != cudaSuccess) return cuda_fail(e);
        }
        d.ev_init = true;
    }
    const size_t esz = in_dtype == TP_IN_BF16 ? 2 : 4;
    const int64_t n = rows * cols;
    const int64_t kBlock = 16384;  // tp::kBlockElems
    const int64_t nb = (cols + kBlock - 1) / kBlock;

    if (rows == 1 && cols % kBlock == 0 && nb >= 64) {
        // Single long row: stream it in K equal block-aligned chunks (K a power of two, so the
        // chunk partials merged by the finish kernel's tree reproduce softmax_f32 bit for bit).
        int K = 32;
        while (K > 1 && nb % K) K >>= 1;
        const int64_t cl = cols / K;
        if ((st = ensure_zeroed(&d.row_x, &d.row_x_bytes, (size_t)n * esz))) return st;
        if ((st = ensure_zeroed(&d.row_y, &d.row_y_bytes, (size_t)n * 4))) return st;
        // one workspace per chunk: a chunk's finish reads the per-block clamp decisions its
        // partial left there (reading G11)
        const size_t wstride = (tp::workspace_bytes(1, cl) + 255) & ~size_t(255);
        if ((st = ensure_zeroed(&d.row_ws, &d.row_ws_bytes, wstride * K))) return st;
        if ((st = ensure_zeroed(&d.pairs, &d.pairs_bytes, sizeof(float) * 2 * K))) return st;
        char* dx = (char*)d.row_x;
        float* dy = (float*)d.row_y;
        float* pairs = (float*)d.pairs;
        cudaStream_t cp = d.st[0], cm = d.st[1];
        const tp::LaunchOpts lo;
        for (int c = 0; c < K; ++c) {  // H2D chunk c || pass 1 of chunk c-1
            e = cudaMemcpyAsync(dx + (size_t)c * cl * esz, (const char*)hx + (size_t)c * cl * esz, (size_t)cl * esz,
                                cudaMemcpyHostToDevice, cp);
            if (e != cudaSuccess) return cuda_fail(e);
            cudaEventRecord(d.ev[c], cp);
            cudaStreamWaitEvent(cm, d.ev[c], 0);
            void* wsc = (char*)d.row_ws + wstride * c;
            if ((st = prepare_ws(wsc, 1, cl, cm))) return st;
            e = tp::launch_partial(in_dtype == TP_IN_BF16, dx + (size_t)c * cl * esz, 1, cl, pairs + 2 * c, wsc, lo,
                                   cm);
            if (e != cudaSuccess) return cuda_fail(e);
        }
        for (int c = 0; c < K; ++c) {  // pass 2 of chunk c || D2H chunk c-1
            e = tp::launch_finish(in_dtype == TP_IN_BF16, dx + (size_t)c * cl * esz, dy + (size_t)c * cl, 1, cl,
                                  pairs, K, (char*)d.row_ws + wstride * c, lo, cm);
            if (e != cudaSuccess) return cuda_fail(e);
            cudaEventRecord(d.ev[32 + c], cm);
            cudaStreamWaitEvent(cp, d.ev[32 + c], 0);
            e = cudaMemcpyAsync(hy + (size_t)c * cl, dy + (size_t)c * cl, (size_t)cl * 4, cudaMemcpyDeviceToHost, cp);
            if (e != cudaSuccess) return cuda_fail(e);
        }
        *last = cp;
        return TP_OK;
    }

    // Row slabs of ~64 MB round-robin over 2 streams: the H2D copy of the next slab, the kernel
    // and the D2H copy of the previous slab overlap (the two copy directions run concurrently,
    // so the pipeline approaches the bidirectional PCIe rate).
    static const size_t slab_bytes = (size_t)tp::dev_env_int("TP_HOST_SLAB_MB", (int)(kHostSlabBytes >> 20)) << 20;
    static const int nstreams = [] {  // development override TP_HOST_STREAMS (1..kHostStreams)
        const int v = tp::dev_env_int("TP_HOST_STREAMS", 2);
        return v < 1 ? 1 : (v > kHostStreams ? kHostStreams : v);
    }();
    int64_t slab = (int64_t)(slab_bytes / ((size_t)cols * esz));
    if (slab < 1) slab = 1;
    if (slab > rows) slab = rows;
    const size_t need_x = (size_t)(slab * cols) * esz, need_y = (size_t)(slab * cols) * 4;
    if (d.stage_bytes_x < need_x || d.stage_bytes_y < need_y || !d.hx_dev[nstreams - 1] ||
        !d.hy_dev[nstreams - 1]) {
        e = cudaDeviceSynchronize();
        if (e != cudaSuccess) return cuda_fail(e);
        for (int i = 0; i < kHostStreams; ++i) {
            if (d.hx_dev[i]) cudaFree(d.hx_dev[i]);
            if (d.hy_dev[i]) cudaFree(d.hy_dev[i]);
            d.hx_dev[i] = nullptr;
            d.hy_dev[i] = nullptr;
        }
        const size_t bx = need_x > d.stage_bytes_x ? need_x : d.stage_bytes_x;
        const size_t by = need_y > d.stage_bytes_y ? need_y : d.stage_bytes_y;
        for (int i = 0; i < nstreams; ++i) {  // one staging slot per stream in use
            if ((e = cudaMalloc(&d.hx_dev[i], bx)) != cudaSuccess) return cuda_fail(e);
            if ((e = cudaMalloc((void**)&d.hy_dev[i], by)) != cudaSuccess) return cuda_fail(e);
        }
        d.stage_bytes_x = bx;
        d.stage_bytes_y = by;
    }
    const tp::LaunchOpts lo;
    const bool needs_ws = tp::softmax_needs_workspace(TP_ALGO_TWO_PASS, cols, lo);
    if (needs_ws) {
        const size_t wsb = tp::workspace_bytes(slab, cols);
        if (d.hws_bytes < wsb || !d.hws[nstreams - 1]) {
            e = cudaDeviceSynchronize();
            if (e != cudaSuccess) return cuda_fail(e);
            for (int i = 0; i < kHostStreams; ++i) {
                if (d.hws[i]) {
                    cudaFree(d.hws[i]);
                    forget_ws(d.hws[i]);
                    d.hws[i] = nullptr;
                }
                if (i >= nstreams) continue;
                if ((e = cudaMalloc(&d.hws[i], wsb)) != cudaSuccess) return cuda_fail(e);
                if ((e = cudaMemset(d.hws[i], 0, wsb)) != cudaSuccess) return cuda_fail(e);
            }
            d.hws_bytes = wsb;
        }
    }
    // Slab sizes: full slabs in the middle, a doubling ramp at both ends (slab/8, /4, /2 ...) so
    // that the first H2D copy and the last D2H copy, which nothing overlaps, are short.
    static const int ramp = tp::dev_env_int("TP_HOST_RAMP", 1);  // development: 0 = equal slabs
    std::vector<int64_t> sizes;
    {
        std::vector<int64_t> up;
        int64_t ramp_rows = 0;
        // (bf16 inputs: the D2H direction carries twice the H2D bytes and bounds the pipeline,
        // so its start and end are what matter; measured: bf16 C4 16.4 -> 15.7 ms, fp32 C4
        // 18.1 -> 18.4 ms, so fp32 keeps equal slabs)
        if (ramp && esz == 2)
            for (int64_t z = slab / 8 > 0 ? slab / 8 : 1; z < slab; z *= 2) up.push_back(z), ramp_rows += 2 * z;
        if (!ramp || rows < ramp_rows + 2 * slab) {
            for (int64_t r0 = 0; r0 < rows; r0 += slab) sizes.push_back(rows - r0 < slab ? rows - r0 : slab);
        } else {
            sizes = up;
            int64_t mid = rows - ramp_rows;
            for (; mid > 0; mid -= slab) sizes.push_back(mid < slab ? mid : slab);
            sizes.insert(sizes.end(), up.rbegin(), up.rend());
        }
    }
    int64_t r0 = 0;
    for (size_t i = 0; i < sizes.size(); r0 += sizes[i], ++i) {
        const int k = (int)(i % (size_t)nstreams);
        const int64_t nr = sizes[i];
        cudaStream_t s = d.st[k];
        e = cudaMemcpyAsync(d.hx_dev[k], (const char*)hx + (size_t)(r0 * cols) * esz, (size_t)(nr * cols) * esz,
                            cudaMemcpyHostToDevice, s);
        if (e != cudaSuccess) return cuda_fail(e);
        if (needs_ws && (st = prepare_ws(d.hws[k], nr, cols, s))) return st;
        e = tp::launch_softmax(TP_ALGO_TWO_PASS, in_dtype == TP_IN_BF16, d.hx_dev[k], d.hy_dev[k], nr, cols,
                               d.hws[k], lo, s);
        if (e != cudaSuccess) return cuda_fail(e);
        e = cudaMemcpyAsync(hy + (size_t)(r0 * cols), d.hy_dev[k], (size_t)(nr * cols) * 4, cudaMemcpyDeviceToHost, s);
        if (e != cudaSuccess) return cuda_fail(e);
    }
    for (int i = 1; i < kHostStreams; ++i) {  // the call ends on stream 0
        cudaEventRecord(d.ev[i], d.st[i]);
        cudaStreamWaitEvent(d.st[0], d.ev[i], 0);
    }
    *last = d.st[0];
    return TP_OK;
}

int host_pipeline(int in_dtype, const void* hx, float* hy, int64_t rows, int64_t cols) {
    int st = check_args(in_dtype, hx, hy, rows, cols, true);
    if (st) return st;
    int dev;
    st = current_device(&dev);
    if (st) return st;
    DevState& d = g_dev[dev];
    std::lock_guard<std::mutex> lk(d.mu);
    cudaStream_t last = nullptr;
    if ((st = host_enqueue(d.hs[0], in_dtype, hx, hy, rows, cols, &last))) return st;
    const cudaError_t e = cudaStreamSynchronize(last);
    return e == cudaSuccess ? TP_OK : cuda_fail(e);
}

int host_submit(int in_dtype, const void* hx, float* hy, int64_t rows, int64_t cols, unsigned long long* ticket) {
    int st = check_args(in_dtype, hx, hy, rows, cols, true);
    if (st) return st;
    if (!ticket) return TP_EINVAL;
    int dev;
    st = current_device(&dev);
    if (st) return st;
    DevState& d = g_dev[dev];
    std::lock_guard<std::mutex> lk(d.mu);
    if (!d.tev_init) {
        for (auto& ev : d.tev) {
            const cudaError_t e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
            if (e != cudaSuccess) return cuda_fail(e);
        }
        d.tev_init = true;
    }
    const unsigned long long t = ++d.tickets;
    cudaStream_t last = nullptr;
    if ((st = host_enqueue(d.hs[1 + (t & 1)], in_dtype, hx, hy, rows, cols, &last))) return st;
    const cudaError_t e = cudaEventRecord(d.tev[t % kTicketEvents], last);
    if (e != cudaSuccess) return cuda_fail(e);
    *ticket = (unsigned long long)dev << 48 | t;
    return TP_OK;
}

int host_wait(unsigned long long ticket) {
    const int dev = (int)(ticket >> 48);
    const unsigned long long t = ticket & ((1ull << 48) - 1);
    if (dev < 0 || dev >= kMaxDev || t == 0) return TP_EINVAL;
    DevState& d = g_dev[dev];
    cudaEvent_t ev;
    {
        std::lock_guard<std::mutex> lk(d.mu);
        if (!d.tev_init || t > d.tickets || d.tickets - t >= (unsigned long long)kTicketEvents) return TP_EINVAL;
        ev = d.tev[t % kTicketEvents];
    }
    const cudaError_t e = cudaEventSynchronize(ev);
    return e == cudaSuccess ? TP_OK : cuda_fail(e);
}

}  // namespace

namespace tp {
unsigned* abort_word_device(int dev) {
    abort_init();
    return g_abort_dev && dev >= 0 && dev < kMaxDev ? g_abort_dev + dev : nullptr;
}
}  // namespace tp

// mapped pointer -> base of the IPC mapping it was opened from (tp_ipc_open / tp_ipc_close)
std::mutex g_ipc_mu;
std::unordered_map<void*, void*> g_ipc_base;

extern "C" {

int softmax_f32(const float* x, float* y, int64_t rows, int64_t cols, cudaStream_t stream) {
    return run_softmax(TP_ALGO_TWO_PASS, TP_IN_F32, x, y, rows, cols, nullptr, 0, nullptr, stream);
}
int softmax_bf16_f32(const uint16_t* x, float* y, int64_t rows, int64_t cols, cudaStream_t stream) {
    return run_softmax(TP_ALGO_TWO_PASS, TP_IN_BF16, x, y, rows, cols, nullptr, 0, nullptr, stream);
}
int softmax3_recompute_f32(const float* x, float* y, int64_t rows, int64_t cols, cudaStream_t stream) {
    return run_softmax(TP_ALGO_THREE_PASS_RECOMPUTE, TP_IN_F32, x, y, rows, cols, nullptr, 0, nullptr, stream);
}
int softmax3_reload_f32(const float* x, float* y, int64_t rows, int64_t cols, cudaStream_t stream) {
    return run_softmax(TP_ALGO_THREE_PASS_RELOAD, TP_IN_F32, x, y, rows, cols, nullptr, 0, nullptr, stream);
}
int softmax3_recompute_bf16_f32(const uint16_t* x, float* y, int64_t rows, int64_t cols, cudaStream_t stream) {
    return run_softmax(TP_ALGO_THREE_PASS_RECOMPUTE, TP_IN_BF16, x, y, rows, cols, nullptr, 0, nullptr, stream);
}
int softmax3_reload_bf16_f32(const uint16_t* x, float* y, int64_t rows, int64_t cols, cudaStream_t stream) {
    return run_softmax(TP_ALGO_THREE_PASS_RELOAD, TP_IN_BF16, x, y, rows, cols, nullptr, 0, nullptr, stream);
}
int softmax_f32_partial(const float* x, int64_t rows, int64_t cols, float* pair_out, cudaStream_t stream) {
    return run_partial(TP_IN_F32, x, rows, cols, pair_out, nullptr, 0, nullptr, stream);
}
int softmax_bf16_partial(const uint16_t* x, int64_t rows, int64_t cols, float* pair_out, cudaStream_t stream) {
    return run_partial(TP_IN_BF16, x, rows, cols, pair_out, nullptr, 0, nullptr, stream);
}
int softmax_f32_finish(const float* x, float* y, int64_t rows, int64_t cols, const float* pairs, int world,
                       cudaStream_t stream) {
    return run_finish(TP_IN_F32, x, y, rows, cols, pairs, world, nullptr, 0, nullptr, stream);
}
int softmax_bf16_f32_finish(const uint16_t* x, float* y, int64_t rows, int64_t cols, const float* pairs, int world,
                            cudaStream_t stream) {
    return run_finish(TP_IN_BF16, x, y, rows, cols, pairs, world, nullptr, 0, nullptr, stream);
}
size_t softmax_workspace_bytes(int64_t rows, int64_t cols) {
    if (rows < 1 || cols < 1) return 0;
    return tp::workspace_bytes(rows, cols);
}
int softmax_ex(int algo, int in_dtype, const void* x, float* y, int64_t rows, int64_t cols, void* workspace,
               size_t workspace_bytes, const softmax_opts* opts, cudaStream_t stream) {
    if (!workspace && workspace_bytes) return TP_EINVAL;
    return run_softmax(algo, in_dtype, x, y, rows, cols, workspace, workspace_bytes, opts, stream);
}
int softmax_partial_ex(int in_dtype, const void* x, int64_t rows, int64_t cols, float* pair_out, void* workspace,
                       size_t workspace_bytes, const softmax_opts* opts, cudaStream_t stream) {
    return run_partial(in_dtype, x, rows, cols, pair_out, workspace, workspace_bytes, opts, stream);
}
int softmax_finish_ex(int in_dtype, const void* x, float* y, int64_t rows, int64_t cols, const float* pairs,
                      int world, void* workspace, size_t workspace_bytes, const softmax_opts* opts,
                      cudaStream_t stream) {
    return run_finish(in_dtype, x, y, rows, cols, pairs, world, workspace, workspace_bytes, opts, stream);
}
int softmax_partial_push_ex(int in_dtype, const void* x, int64_t rows, int64_t cols, void* const* peer_mailboxes,
                            int rank, int world, unsigned epoch, float* pair_out, void* workspace,
                            size_t workspace_bytes, const softmax_opts* opts, cudaStream_t stream) {
    int st = check_args(in_dtype, x, nullptr, rows, cols, false);
    if (st) return st;
    if (!peer_mailboxes || world < 1 || world > tp::kMailboxMaxWorld || rank < 0 || rank >= world || epoch == 0)
        return TP_EINVAL;
    void* ws = workspace;
    const size_t need = tp::workspace_bytes(rows, cols);
    if (ws) {
        if (workspace_bytes < need) return TP_EINVAL;
    } else if ((st = internal_workspace(need, &ws))) {
        return st;
    }
    if ((st = prepare_ws(ws, rows, cols, stream))) return st;
    tp::Exchange xc;
    xc.peers = peer_mailboxes;
    xc.rank = rank;
    xc.world = world;
    xc.epoch = epoch;
    cudaError_t e = tp::launch_partial(in_dtype == TP_IN_BF16, x, rows, cols, pair_out, ws, to_opts(opts), stream, &xc);
    return e == cudaSuccess ? TP_OK : cuda_fail(e);
}

int softmax_finish_mailbox_ex(int in_dtype, const void* x, float* y, int64_t rows, int64_t cols, const void* mailbox,
                              int world, unsigned epoch, unsigned long long timeout_ns, void* workspace,
                              size_t workspace_bytes, const softmax_opts* opts, cudaStream_t stream) {
    int st = check_args(in_dtype, x, y, rows, cols, true);
    if (st) return st;
    if (!mailbox || world < 1 || world > tp::kMailboxMaxWorld || epoch == 0 ||
        (reinterpret_cast<uintptr_t>(mailbox) & 15) || (!workspace && workspace_bytes))
        return TP_EINVAL;
    void* ws = workspace;
    if ((st = workspace_for(&ws, workspace_bytes, rows, cols, stream))) return st;
    tp::Exchange xc;
    xc.world = world;
    xc.epoch = epoch;
    xc.mailbox = mailbox;
    xc.wait_ns = timeout_ns;
    const float* pairs = reinterpret_cast<const float*>(static_cast<const char*>(mailbox) +
                                                        tp::mailbox_pairs_offset(world, rows, epoch));
    cudaError_t e = tp::launch_finish(in_dtype == TP_IN_BF16, x, y, rows, cols, pairs, world, ws, to_opts(opts),
                                      stream, &xc);
    return e == cudaSuccess ? TP_OK : cuda_fail(e);
}

// ---- sharded Three-Pass comparators (multi-GPU Alg. 1 / Alg. 2)
namespace {
int run_shard3(int algo, int phase, int in_dtype, const void* x, float* y, int64_t rows, int64_t cols,
               const float* maxes, const float* sums, int world, float* out, void* ws, size_t ws_bytes,
               cudaStream_t s) {
    const bool need_y = phase == 2 || (phase == 1 && algo == TP_ALGO_THREE_PASS_RELOAD);
    int st = check_args(in_dtype, x, y, rows, cols, need_y);
    if (st) return st;
    if (algo != TP_ALGO_THREE_PASS_RECOMPUTE && algo != TP_ALGO_THREE_PASS_RELOAD) return TP_EINVAL;
    if (world < 1 || (phase >= 1 && !maxes) || (phase == 2 && !sums) || (phase < 2 && !out) || (!ws && ws_bytes))
        return TP_EINVAL;
    if ((st = workspace_for(&ws, ws_bytes, rows, cols, s))) return st;
    tp::Shard3 sh;
    sh.maxes = phase >= 1 ? maxes : nullptr;
    sh.sums = phase == 2 ? sums : nullptr;
    sh.world = world;
    sh.out = phase < 2 ? out : nullptr;
    cudaError_t e = tp::launch_shard3(algo, in_dtype == TP_IN_BF16, phase, x, need_y ? y : nullptr, rows, cols, ws,
                                      sh, tp::LaunchOpts{}, s);
    return e == cudaSuccess ? TP_OK : cuda_fail(e);
}
}  // namespace

int softmax3_max_partial_ex(int in_dtype, const void* x, int64_t rows, int64_t cols, float* max_out, void* workspace,
                            size_t workspace_bytes, cudaStream_t stream) {
    return run_shard3(TP_ALGO_THREE_PASS_RECOMPUTE, 0, in_dtype, x, nullptr, rows, cols, nullptr, nullptr, 1, max_out,
                      workspace, workspace_bytes, stream);
}
int softmax3_sum_partial_ex(int algo, int in_dtype, const void* x, float* y, int64_t rows, int64_t cols,
                            const float* maxes, int world, float* sum_out, void* workspace, size_t workspace_bytes,
                            cudaStream_t stream) {
    return run_shard3(algo, 1, in_dtype, x, y, rows, cols, maxes, nullptr, world, sum_out, workspace, workspace_bytes,
                      stream);
}
int softmax3_finish_ex(int algo, int in_dtype, const void* x, float* y, int64_t rows, int64_t cols, const float* maxes,
                       const float* sums, int world, void* workspace, size_t workspace_bytes, cudaStream_t stream) {
    return run_shard3(algo, 2, in_dtype, x, y, rows, cols, maxes, sums, world, nullptr, workspace, workspace_bytes,
                      stream);
}

int softmax_f32_host(const float* hx, float* hy, int64_t rows, int64_t cols) {
    return host_pipeline(TP_IN_F32, hx, hy, rows, cols);
}
int softmax_bf16_f32_host(const uint16_t* hx, float* hy, int64_t rows, int64_t cols) {
    return host_pipeline(TP_IN_BF16, hx, hy, rows, cols);
}
int softmax_host_submit(int in_dtype, const void* hx, float* hy, int64_t rows, int64_t cols,
                        unsigned long long* ticket) {
    return host_submit(in_dtype, hx, hy, rows, cols, ticket);
}
int softmax_host_wait(unsigned long long ticket) { return host_wait(ticket); }
const char* softmax_status_str(int status) {
    switch (status) {
        case TP_OK: return "ok";
        case TP_EINVAL: return "invalid argument";
        case TP_ECUDA: return "CUDA error";
        case TP_ENODEV: return "no CUDA device";
        case TP_EWATCHDOG:
            return "watchdog abort: an earlier launch on this device gave up waiting (its outputs are invalid); "
                   "state reset, call again";
        default: return "unknown status";
    }
}
int softmax_last_cuda_error(void) { return g_last_cuda_error; }

int softmax_last_plan(softmax_plan* out) {
    if (!out) return TP_EINVAL;
    const tp::Plan& p = tp::last_plan();
    out->kernel = p.kernel;
    out->variant = p.variant;
    out->grid_ctas = p.grid_ctas;
    out->cluster_size = p.cluster_size;
    out->lookahead_rows = p.lookahead_rows;
    out->hold = p.hold;
    return TP_OK;
}

int softmax_watchdog_flags(const void* workspace, int reset) {
    const void* ws = workspace;
    if (!ws) {
        int dev;
        if (current_device(&dev)) return -1;
        ws = g_dev[dev].ws;
        if (!ws) return 0;
    }
    // the main header, and the tail layout's header (a concurrent tail launch), found through
    // the shape the workspace was last prepared for
    size_t toff = 0;
    {
        std::lock_guard<std::mutex> lk(g_shape_mu);
        auto it = g_ws_shape.find(ws);
        if (it != g_ws_shape.end()) toff = tp::tail_ws_offset(it->second.first, it->second.second);
    }
    tp::WsHeader h, ht{};
    if (cudaMemcpy(&h, ws, sizeof(h), cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
    if (toff && cudaMemcpy(&ht, (const char*)ws + toff, sizeof(ht), cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
    const unsigned err = h.error | ht.error;
    if (reset) {  // also acknowledges a pending TP_EWATCHDOG of this device
        int dev;
        if (!current_device(&dev) && g_abort_host) __atomic_store_n(&g_abort_host[dev], 0u, __ATOMIC_RELEASE);
    }
    if (reset && err) {
        unsigned z = 0;
        cudaMemcpy((char*)ws + offsetof(tp::WsHeader, error), &z, sizeof(z), cudaMemcpyHostToDevice);
        if (toff) cudaMemcpy((char*)ws + toff + offsetof(tp::WsHeader, error), &z, sizeof(z), cudaMemcpyHostToDevice);
        forget_ws(ws);  // the aborted launch may have left tickets behind: re-zero on next use
    }
    return (int)err;
}

int tp_set_profile_buffer(void* p) {
    tp::set_profile_buffer(p);
    return TP_OK;
}

int tp_stream_baseline(int what, float* x, float* y, int64_t n, float a, int64_t ctas, cudaStream_t stream) {
    if (what < 0 || what > 5 || n < 0 || (n & 3) || !x || (what != 2 && !y) ||
        ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15))
        return TP_EINVAL;
    if (n == 0) return TP_OK;
    if (ctas <= 0) {
        int dev = 0, sms = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        ctas = 4 * (int64_t)sms;
    }
    cudaError_t e = tp::launch_stream_baseline(what, x, y, n, a, ctas, stream);
    return e == cudaSuccess ? TP_OK : cuda_fail(e);
}

int tp_phase_only(int algo, int in_dtype, int phase, const void* x, float* y, int64_t rows, int64_t cols,
                  void* workspace, size_t workspace_bytes, cudaStream_t stream) {
    int st = check_args(in_dtype, x, y, rows, cols, algo != TP_ALGO_TWO_PASS || phase > 0);
    if (st) return st;
    if (algo != TP_ALGO_TWO_PASS && algo != TP_ALGO_THREE_PASS_RECOMPUTE && algo != TP_ALGO_THREE_PASS_RELOAD)
        return TP_EINVAL;
    if (!workspace || workspace_bytes < tp::workspace_bytes(rows, cols)) return TP_EINVAL;
    if ((st = prepare_ws(workspace, rows, cols, stream))) return st;
    cudaError_t e = tp::launch_phase_only(algo, in_dtype == TP_IN_BF16, phase, x, y, rows, cols, workspace,
                                          tp::LaunchOpts{}, stream);
    if (e == cudaErrorNotSupported) {
        cudaGetLastError();
        return TP_EINVAL;
    }
    return e == cudaSuccess ? TP_OK : cuda_fail(e);
}

int tp_read_probe(const void* x, int64_t bytes, int64_t chunk_bytes, int stages, int64_t ctas, float* sink,
                  cudaStream_t stream) {
    if (!x || !sink || bytes < 0 || chunk_bytes < 16 || (chunk_bytes & 15) || stages < 1 || stages > 32 ||
        chunk_bytes * stages > 227 * 1024 || ctas < 1 || (reinterpret_cast<uintptr_t>(x) & 15))
        return TP_EINVAL;
    if (bytes < chunk_bytes) return TP_OK;
    cudaError_t e = tp::launch_read_probe(x, bytes, chunk_bytes, stages, ctas, sink, stream);
    return e == cudaSuccess ? TP_OK : cuda_fail(e);
}

int tp_copy_probe(const void* x, void* y, int64_t bytes, int64_t chunk_bytes, int stages, int64_t ctas, int backward,
                  cudaStream_t stream) {
    if (!x || !y || bytes < 0 || chunk_bytes < 16 || (chunk_bytes & 15) || stages < 1 || stages > 32 ||
        chunk_bytes * stages > 227 * 1024 || ctas < 1 || (reinterpret_cast<uintptr_t>(x) & 15) ||
        (reinterpret_cast<uintptr_t>(y) & 15))
        return TP_EINVAL;
    if (bytes < chunk_bytes) return TP_OK;
    cudaError_t e = tp::launch_copy_probe(x, y, bytes, chunk_bytes, stages, ctas, backward, stream);
    return e == cudaSuccess ? TP_OK : cuda_fail(e);
}

int tp_exp_sweep(int what, uint32_t bits0, int64_t count, float* out0, float* out1, cudaStream_t stream) {
    if (what < 0 || what > 1 || count < 0 || (count > 0 && (!out0 || (what == 0 && !out1))) ||
        (uint64_t)bits0 + (uint64_t)count > 0x100000000ull)
        return TP_EINVAL;
    cudaError_t e = tp::launch_exp_sweep(what, bits0, count, out0, out1, stream);
    return e == cudaSuccess ? TP_OK : cuda_fail(e);
}

int tp_exp_fit(const float* coeffs, uint32_t bits0, int64_t count, int stride, unsigned* max_ulp_bits,
               unsigned long long* n_over2, cudaStream_t stream) {
    if (!coeffs || count < 0 || stride < 1 || (count > 0 && (!max_ulp_bits || !n_over2)) ||
        (uint64_t)bits0 + (uint64_t)count * (uint64_t)stride > 0x100000000ull)
        return TP_EINVAL;
    cudaError_t e = tp::launch_exp_fit(coeffs, bits0, count, stride, max_ulp_bits, n_over2, stream);
    return e == cudaSuccess ? TP_OK : cuda_fail(e);
}

size_t tp_mailbox_bytes(int world, int64_t rows) {
    return (world < 1 || world > tp::kMailboxMaxWorld || rows < 0) ? 0 : tp::mailbox_bytes(world, rows);
}
size_t tp_mailbox_pairs_offset(int world, int64_t rows, unsigned epoch) {
    return (world < 1 || world > tp::kMailboxMaxWorld || rows < 0) ? 0 : tp::mailbox_pairs_offset(world, rows, epoch);
}

int tp_pairs_push(const float* pairs, int64_t rows, void* const* peer_mailboxes, int rank, int world,
                  unsigned epoch, cudaStream_t stream) {
    if (!pairs || !peer_mailboxes || rows < 1 || world < 1 || world > 56 || rank < 0 || rank >= world)
        return TP_EINVAL;
    cudaError_t e = tp::launch_pairs_push(pairs, rows, peer_mailboxes, rank, world, epoch, stream);
    return e == cudaSuccess ? TP_OK : cuda_fail(e);
}

int tp_pairs_wait(const void* mailbox, int world, unsigned epoch, uint64_t timeout_ns, cudaStream_t stream) {
    if (!mailbox || world < 1 || world > 56) return TP_EINVAL;
    cudaError_t e = tp::launch_pairs_wait(mailbox, world, epoch, (unsigned long long)timeout_ns, stream);
    return e == cudaSuccess ? TP_OK : cuda_fail(e);
}

int tp_ipc_get_handle(const void* dev_ptr, void* handle64, uint64_t* offset) {
    if (!dev_ptr || !handle64 || !offset) return TP_EINVAL;
    // the handle names the whole allocation (e.g. a caching-allocator segment): report where
    // dev_ptr sits inside it
    // driver entry point through the runtime (no link-time dependency on libcuda)
    using GetRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
    static GetRange get_range = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
        return reinterpret_cast<GetRange>(fn);
    }();
    if (!get_range) return TP_ECUDA;
    CUdeviceptr base = 0;
    size_t size = 0;
    if (get_range(&base, &size, (CUdeviceptr)dev_ptr) != CUDA_SUCCESS) return TP_EINVAL;
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
    if (e != cudaSuccess) return cuda_fail(e);
    static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
    memcpy(handle64, &h, sizeof(h));
    *offset = (uint64_t)((CUdeviceptr)dev_ptr - base);
    return TP_OK;
}

int tp_ipc_open(const void* handle64, uint64_t offset, void** dev_ptr) {
    if (!handle64 || !dev_ptr) return TP_EINVAL;
    cudaIpcMemHandle_t h;
    memcpy(&h, handle64, sizeof(h));
    void* base = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return cuda_fail(e);
    *dev_ptr = static_cast<char*>(base) + offset;
    std::lock_guard<std::mutex> g(g_ipc_mu);
    g_ipc_base[*dev_ptr] = base;
    return TP_OK;
}

int tp_ipc_close(void* dev_ptr) {
    if (!dev_ptr) return TP_EINVAL;
    void* base = nullptr;
    {
        std::lock_guard<std::mutex> g(g_ipc_mu);
        auto it = g_ipc_base.find(dev_ptr);
        if (it == g_ipc_base.end()) return TP_EINVAL;
        base = it->second;
        g_ipc_base.erase(it);
    }
    cudaError_t e = cudaIpcCloseMemHandle(base);
    return e == cudaSuccess ? TP_OK : cuda_fail(e);
}

int tp_bench_compute(int what, int in_dtype, int64_t ctas, int reps, float* sink, cudaStream_t stream) {
    if (what < 0 || what > 11 || ctas < 1 || reps < 1 || !sink || (in_dtype != TP_IN_F32 && in_dtype != TP_IN_BF16))
        return TP_EINVAL;
    cudaError_t e = tp::launch_bench_compute(what, in_dtype == TP_IN_BF16, ctas, reps, sink, stream);
    return e == cudaSuccess ? TP_OK : cuda_fail(e);
}

int tp_debug_op(int what, const float* a, const float* b, float* out0, float* out1, int64_t count,
                cudaStream_t stream) {
    if (count < 0 || what < 0 || what > 8 || (count > 0 && (!a || !out0))) return TP_EINVAL;
    if (what == 8 && count % 32 != 0) return TP_EINVAL;  // whole warps
    if ((what == 0 || what == 2 || what == 6) && count > 0 && !out1) return TP_EINVAL;
    if (what == 2 && count > 0 && !b) return TP_EINVAL;
    cudaError_t e = tp::launch_debug(what, a, b, out0, out1, count, stream);
    return e == cudaSuccess ? TP_OK : cuda_fail(e);
}

}  // extern "C"
