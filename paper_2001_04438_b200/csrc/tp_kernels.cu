// sm_100a kernels of the Two-Pass softmax (Alg. 3) and of the in-house
// Three-Pass comparators (Alg. 1 and 2).
//
// Kernels
//   rowblock_kernel      rows with cols <= kBlockElems: one CTA per row, the row stays in
//                        registers between the passes (no re-read at all)
//   persistent_kernel    everything else: a persistent grid pulls work items (row, phase,
//                        block) from an in-order atomic queue.  Pass-1 blocks publish their
//                        pair; the last block of each group of 64 reduces the group, the last
//                        group reduces the row (canonical tree, reading G8) and releases the
//                        row's flag; pass-2 blocks of that row wait for the flag.  Rows are
//                        interleaved with a lookahead of L rows so that a row's pass 2 runs
//                        while its data is still in L2 (multi-row) / runs the single-row
//                        pass 2 in reverse block order (L2-resident tail first).
//   finish_kernel        multi-GPU chunk finish: merge `world` rank partials (canonical tree
//                        over rank index), then pass 2 of the local chunk
//
// Deadlock freedom of the persistent kernel: items are handed out in increasing order and a
// pass-k item depends only on items of smaller index, so the smallest unfinished item is
// always being executed by a running CTA (a CTA holds its current item and at most one
// prefetched item of larger index).
#include "tp_internal.h"
#include "tp_io.cuh"

namespace tp {

// ----------------------------------------------------------------------------- workspace
__host__ __device__ inline size_t align256(size_t v) { return (v + 255) & ~size_t(255); }

// Control region first (header, tickets, row flags: must be zero when a launch starts; the
// kernels leave it that way except for the epoch-tagged flags), then the data region.
__host__ __device__ inline WsLayout ws_layout(int64_t rows, int64_t cols) {
    WsLayout L{};
    const int64_t nb = (cols + kBlockElems - 1) / kBlockElems;
    const int64_t ng = (nb + kGroupBlocks - 1) / kGroupBlocks;
    size_t off = align256(sizeof(WsHeader));
    L.group_tickets = off; off = align256(off + sizeof(unsigned) * rows * ng);
    L.row_tickets = off;   off = align256(off + sizeof(unsigned) * rows);
    L.row_ready = off;     off = align256(off + sizeof(unsigned) * rows * 2);
    L.ctrl_bytes = off;
    L.row_stats = off;     off = align256(off + sizeof(float4) * rows * 2);
    L.block_vals = off;    off = align256(off + sizeof(float2) * rows * nb);
    L.group_vals = off;    off = align256(off + sizeof(float2) * rows * ng);
    L.bytes = off;
    return L;
}

size_t workspace_bytes(int64_t rows, int64_t cols) { return ws_layout(rows, cols).bytes; }
size_t workspace_ctrl_bytes(int64_t rows, int64_t cols) { return ws_layout(rows, cols).ctrl_bytes; }

struct KArgs {
    const void* x;
    float* y;
    int64_t rows, cols, nb, ng;
    int64_t L;            // lookahead in rows
    int64_t total_items;  // rows * nb * phases
    char* ws;
    WsLayout lay;
    float2* pair_out;     // partial mode: one (m, n) per row
    int vec;              // 16-byte aligned rows
};

enum Algo : int { kTwoPass = 0, kTwoPassPartial = 1, kRecompute = 2, kReload = 3 };

template <int A> struct AlgoTraits;
template <> struct AlgoTraits<kTwoPass> { static constexpr int P = 2; };
template <> struct AlgoTraits<kTwoPassPartial> { static constexpr int P = 1; };
template <> struct AlgoTraits<kRecompute> { static constexpr int P = 3; };
template <> struct AlgoTraits<kReload> { static constexpr int P = 3; };

// number of (phase, row) units in schedule slots < s (slot s holds phase p of row s - p*L)
__device__ __forceinline__ int64_t units_before(int64_t s, int64_t R, int64_t L, int P) {
    int64_t c = 0;
    for (int p = 0; p < P; ++p) {
        int64_t v = s - p * L;
        c += v < 0 ? 0 : (v > R ? R : v);
    }
    return c;
}

struct Item {
    int phase;
    int64_t row, blk;
};

template <int P>
__device__ __forceinline__ Item decode_item(int64_t item, int64_t R, int64_t nb, int64_t L) {
    Item it;
    const int64_t unit = item / nb;
    const int64_t bi = item - unit * nb;
    if (P == 1) {
        it.phase = 0; it.row = unit; it.blk = bi;
        return it;
    }
    // binary search the slot s with units_before(s) <= unit < units_before(s + 1)
    int64_t lo = 0, hi = R + (P - 1) * L;  // answer in [lo, hi)
    while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (units_before(mid, R, L, P) <= unit) lo = mid; else hi = mid;
    }
    const int64_t s = lo;
    int p_hi = (int)((s / L) < (P - 1) ? (s / L) : (P - 1));
    const int64_t idx = unit - units_before(s, R, L, P);
    it.phase = p_hi - (int)idx;              // within a slot: oldest row (highest phase) first
    it.row = s - it.phase * L;
    it.blk = it.phase > 0 ? nb - 1 - bi : bi;  // later passes walk the row backwards
    return it;
}

struct SmemState {
    long long item[2];
    int flag;
    unsigned epoch;
    float4 stats;
    Pair red[kThreads / 32];
    float redf[kThreads / 32];
};

// Publish one block value; if it completes its group (and then its row), reduce it.
// Returns true in the CTA that finished the row (row result valid in thread 0: *root).
template <int A>
__device__ bool publish_and_reduce(const KArgs& a, SmemState& sm, int phase, int64_t row, int64_t blk,
                                   float2 val, float2* root) {
    float2* block_vals = reinterpret_cast<float2*>(a.ws + a.lay.block_vals);
    float2* group_vals = reinterpret_cast<float2*>(a.ws + a.lay.group_vals);
    unsigned* gt = reinterpret_cast<unsigned*>(a.ws + a.lay.group_tickets);
    unsigned* rt = reinterpret_cast<unsigned*>(a.ws + a.lay.row_tickets);
    const int64_t g = blk / kGroupBlocks;
    const int64_t gsize = min((int64_t)kGroupBlocks, a.nb - g * kGroupBlocks);
    if (threadIdx.x == 0) {
        block_vals[row * a.nb + blk] = val;
        __threadfence();
        const unsigned t = atomicAdd(&gt[row * a.ng + g], 1u);
        sm.flag = (t == (unsigned)(gsize - 1));
    }
    __syncthreads();
    if (!sm.flag) return false;
    __threadfence();
    const float2* gv = block_vals + row * a.nb + g * kGroupBlocks;
    // phase 0 of the Three-Pass algorithms reduces a max, phase 1 a sum; Two-Pass reduces pairs
    const bool is_max = (A == kRecompute || A == kReload) && phase == 0;
    const bool is_sum = (A == kRecompute || A == kReload) && phase == 1;
    float2 gres;
    if (is_max) {
        float m = -__int_as_float(0x7f800000);
        for (int64_t j = threadIdx.x; j < gsize; j += kThreads) m = fmaxf(m, __ldcg(gv + j).x);
        m = cta_max(m, sm.redf);
        gres = make_float2(m, 0.0f);
    } else if (is_sum) {
        const float s = cta_canonical_sum(gsize, [&](int64_t j) { return __ldcg(gv + j).x; }, sm.redf);
        gres = make_float2(s, 0.0f);
    } else {
        const Pair p = cta_canonical_tree(gsize, [&](int64_t j) {
            const float2 v = __ldcg(gv + j);
            return Pair{v.x, v.y};
        }, sm.red);
        gres = make_float2(p.m, p.n);
    }
    if (threadIdx.x == 0) {
        gt[row * a.ng + g] = 0u;  // ticket reset for the next phase / launch
        group_vals[row * a.ng + g] = gres;
        __threadfence();
        const unsigned t = atomicAdd(&rt[row], 1u);
        sm.flag = (t == (unsigned)(a.ng - 1));
    }
    __syncthreads();
    if (!sm.flag) return false;
    __threadfence();
    const float2* rv = group_vals + row * a.ng;
    if (is_max) {
        float m = -__int_as_float(0x7f800000);
        for (int64_t j = threadIdx.x; j < a.ng; j += kThreads) m = fmaxf(m, __ldcg(rv + j).x);
        m = cta_max(m, sm.redf);
        *root = make_float2(m, 0.0f);
    } else if (is_sum) {
        const float s = cta_canonical_sum(a.ng, [&](int64_t j) { return __ldcg(rv + j).x; }, sm.redf);
        *root = make_float2(s, 0.0f);
    } else {
        const Pair p = cta_canonical_tree(a.ng, [&](int64_t j) {
            const float2 v = __ldcg(rv + j);
            return Pair{v.x, v.y};
        }, sm.red);
        *root = make_float2(p.m, p.n);
    }
    if (threadIdx.x == 0) rt[row] = 0u;
    return true;
}

template <typename In, int A>
__global__ void __launch_bounds__(kThreads, 2) persistent_kernel(KArgs a) {
    constexpr int P = AlgoTraits<A>::P;
    __shared__ SmemState sm;
    WsHeader* hdr = reinterpret_cast<WsHeader*>(a.ws);
    float4* row_stats = reinterpret_cast<float4*>(a.ws + a.lay.row_stats);
    unsigned* row_ready = reinterpret_cast<unsigned*>(a.ws + a.lay.row_ready);
    const In* x = static_cast<const In*>(a.x);

    if (threadIdx.x == 0) {
        sm.epoch = *reinterpret_cast<volatile unsigned*>(&hdr->epoch);
        sm.item[0] = (long long)atomicAdd(&hdr->counter, 1ull);
    }
    __syncthreads();
    const unsigned want = sm.epoch + 1u;
    int buf = 0;
    while (true) {
        const long long item = sm.item[buf];
        if (item >= a.total_items) break;
        if (threadIdx.x == 0) sm.item[buf ^ 1] = (long long)atomicAdd(&hdr->counter, 1ull);
        const Item it = decode_item<P>(item, a.rows, a.nb, a.L);
        const int64_t e0 = it.blk * kBlockElems;
        const int valid = (int)min((int64_t)kBlockElems, a.cols - e0);
        const In* xb = x + it.row * a.cols + e0;
        float* yb = a.y ? a.y + it.row * a.cols + e0 : nullptr;
        BlockRegs<In> r;

        if (it.phase > 0) {  // wait for the row's previous phase
            if (threadIdx.x == 0) {
                const unsigned* f = row_ready + it.row * 2 + (it.phase - 1);
                unsigned ns = 32;
                const unsigned long long t0 = globaltimer_ns();
                while (ld_acquire_gpu(f) != want) {
                    __nanosleep(ns);
                    ns = ns < 1024 ? ns * 2 : ns;
                    if (globaltimer_ns() - t0 > kWaitTimeoutNs) {  // never hang the GPU on a bug
                        atomicOr(&hdr->error, 1u);
                        break;
                    }
                }
                sm.stats = __ldcg(row_stats + it.row * 2 + (it.phase - 1));
            }
            __syncthreads();
        }
        const float4 st = sm.stats;

        if constexpr (A == kTwoPass || A == kTwoPassPartial) {
            if (it.phase == 0) {
                load_block<In, false>(xb, valid, a.vec != 0, false, r);
                const Pair acc = valid == kBlockElems ? pass1_thread<In, true>(r, valid)
                                                      : pass1_thread<In, false>(r, valid);
                const Pair bp = cta_tree_pairs(acc, sm.red);
                float2 root;
                if (publish_and_reduce<A>(a, sm, 0, it.row, it.blk, make_float2(bp.m, bp.n), &root) &&
                    threadIdx.x == 0) {
                    if (A == kTwoPassPartial) {
                        a.pair_out[it.row] = root;
                    } else {
                        // lambda' = 0.5 / m_sum, correctly rounded (readings G9, G10)
                        row_stats[it.row * 2] = make_float4(__fsub_rn(root.y, 1.0f), __fdiv_rn(0.5f, root.x),
                                                            root.x, root.y);
                        st_release_gpu(row_ready + it.row * 2, want);
                    }
                }
            } else {
                load_block<In, false>(xb, valid, a.vec != 0, true, r);
                pass2_thread<In>(r, st.x, st.y);
                store_block<In, false>(yb, valid, a.vec != 0, r);
            }
        } else {
            // Three-Pass: phase 0 max (Pass 1), phase 1 sum of Exp(x - mu) (Pass 2),
            // phase 2 output (Pass 3).  Alg. 1, Alg. 2 PAPER.md:110-123.
            if (it.phase == 0) {
                load_block<In, false>(xb, valid, a.vec != 0, false, r);
                float mx = valid == kBlockElems ? max_thread<In, true>(r, valid) : max_thread<In, false>(r, valid);
                mx = cta_max(mx, sm.redf);
                float2 root;
                if (publish_and_reduce<A>(a, sm, 0, it.row, it.blk, make_float2(mx, 0.0f), &root) &&
                    threadIdx.x == 0) {
                    row_stats[it.row * 2] = make_float4(root.x, 0.0f, 0.0f, 0.0f);
                    st_release_gpu(row_ready + it.row * 2, want);
                }
            } else if (it.phase == 1) {
                load_block<In, false>(xb, valid, a.vec != 0, A == kReload, r);
                float s = valid == kBlockElems ? exp_sum_thread<In, true>(r, valid, st.x)
                                               : exp_sum_thread<In, false>(r, valid, st.x);
                if (A == kReload) store_block<In, false>(yb, valid, a.vec != 0, r);  // Y_i <- Exp(X_i - mu)
                s = cta_tree_sum(s, sm.redf);
                float2 root;
                if (publish_and_reduce<A>(a, sm, 1, it.row, it.blk, make_float2(s, 0.0f), &root) &&
                    threadIdx.x == 0) {
                    row_stats[it.row * 2 + 1] = make_float4(st.x, __fdiv_rn(1.0f, root.x), root.x, 0.0f);
                    st_release_gpu(row_ready + it.row * 2 + 1, want);
                }
            } else {
                if constexpr (A == kRecompute) {
                    load_block<In, false>(xb, valid, a.vec != 0, true, r);
                    exp_sum_thread<In, false>(r, valid, st.x);
                    scale_thread<In>(r, st.y);  // Y_i <- lambda * Exp(X_i - mu)
                    store_block<In, false>(yb, valid, a.vec != 0, r);
                } else {
                    BlockRegs<float> ry;  // Y_i <- lambda * Y_i  (read Y, write Y)
                    const bool yvec = (a.cols % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.y) & 15) == 0);
                    load_block_y(yb, valid, yvec, ry);
                    scale_thread<float>(ry, st.y);
                    store_block<float, false>(yb, valid, yvec, ry);
                }
            }
        }
        __syncthreads();  // sm.item[buf], sm.stats, sm.red reuse
        buf ^= 1;
    }

    // last CTA out resets the queue and advances the epoch (graph-replay safe)
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned t = atomicAdd(&hdr->exit_ticket, 1u);
        if (t == gridDim.x - 1) {
            hdr->counter = 0ull;
            hdr->exit_ticket = 0u;
            __threadfence();
            atomicAdd(&hdr->epoch, 1u);
        }
    }
}

// One CTA per row for rows that fit one block: the row never leaves registers.
template <typename In>
__global__ void __launch_bounds__(kThreads, 2) rowblock_kernel(const In* __restrict__ x, float* y, int64_t rows,
                                                               int64_t cols, int vec) {
    __shared__ Pair red[kThreads / 32];
    __shared__ float2 stats;
    const int64_t row = blockIdx.x;
    const int valid = (int)cols;
    BlockRegs<In> r;
    load_block<In, false>(x + row * cols, valid, vec != 0, true, r);
    const Pair acc = valid == kBlockElems ? pass1_thread<In, true>(r, valid) : pass1_thread<In, false>(r, valid);
    const Pair root = cta_tree_pairs(acc, red);
    if (threadIdx.x == 0) stats = make_float2(__fsub_rn(root.n, 1.0f), __fdiv_rn(0.5f, root.m));
    __syncthreads();
    const float2 st = stats;
    pass2_thread<In>(r, st.x, st.y);
    store_block<In, false>(y + row * cols, valid, vec != 0, r);
}

// Multi-GPU finish: merge the world partials of every row (canonical tree over rank index,
// reading G8), then pass 2 over the local chunk, blocks in reverse order.
template <typename In>
__global__ void __launch_bounds__(kThreads, 2) finish_kernel(const In* __restrict__ x, float* y, int64_t rows,
                                                             int64_t cols, const float2* __restrict__ pairs,
                                                             int world, int vec) {
    __shared__ float2 stats;
    __shared__ int64_t cur_row;
    const int64_t nb = (cols + kBlockElems - 1) / kBlockElems;
    const int64_t total = rows * nb;
    if (threadIdx.x == 0) cur_row = -1;
    __syncthreads();
    for (int64_t it = blockIdx.x; it < total; it += gridDim.x) {
        const int64_t row = it / nb;
        const int64_t blk = nb - 1 - (it - row * nb);
        if (row != cur_row) {
            if (threadIdx.x == 0) {
                const Pair root = seq_tree_pairs((int)next_pow2(world), [&](int i) {
                    if (i >= world) return pair_identity();
                    const float2 v = pairs[(int64_t)i * rows + row];
                    return Pair{v.x, v.y};
                });
                stats = make_float2(__fsub_rn(root.n, 1.0f), __fdiv_rn(0.5f, root.m));
                cur_row = row;
            }
            __syncthreads();
        }
        const float2 st = stats;
        const int64_t e0 = blk * kBlockElems;
        const int valid = (int)min((int64_t)kBlockElems, cols - e0);
        BlockRegs<In> r;
        load_block<In, false>(x + row * cols + e0, valid, vec != 0, true, r);
        pass2_thread<In>(r, st.x, st.y);
        store_block<In, false>(y + row * cols + e0, valid, vec != 0, r);
        __syncthreads();
    }
}

// ----------------------------------------------------------------------------- host launchers
static int g_num_sms[64];
static int g_occ[64][10];

static int device_sms(int dev) {
    if (!g_num_sms[dev]) cudaDeviceGetAttribute(&g_num_sms[dev], cudaDevAttrMultiProcessorCount, dev);
    return g_num_sms[dev];
}

template <typename K>
static int occupancy(K kernel, int dev, int slot) {
    if (!g_occ[dev][slot]) {
        int n = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, kThreads, 0);
        g_occ[dev][slot] = n > 0 ? n : 1;
    }
    return g_occ[dev][slot];
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

template <typename In>
static int vec_ok(const void* x, const float* y, int64_t cols) {
    constexpr int V = InTraits<In>::V;
    return (cols % V == 0) && aligned16(x) && (y == nullptr || aligned16(y));
}

template <typename In, int A>
static cudaError_t launch_persistent(const void* x, float* y, int64_t rows, int64_t cols, void* ws,
                                     float2* pair_out, const LaunchOpts& o, cudaStream_t s) {
    int dev = 0;
    cudaGetDevice(&dev);
    constexpr int P = AlgoTraits<A>::P;
    KArgs a{};
    a.x = x; a.y = y; a.rows = rows; a.cols = cols;
    a.nb = (cols + kBlockElems - 1) / kBlockElems;
    a.ng = (a.nb + kGroupBlocks - 1) / kGroupBlocks;
    a.total_items = rows * a.nb * P;
    a.ws = static_cast<char*>(ws);
    a.lay = ws_layout(rows, cols);
    a.pair_out = pair_out;
    a.vec = vec_ok<In>(x, y, cols);
    auto kern = persistent_kernel<In, A>;
    const int slot = (int)(sizeof(In) == 4 ? 0 : 4) + A;  // 0..7; finish uses 8, 9
    const int64_t resident = (int64_t)device_sms(dev) * occupancy(kern, dev, slot);
    int64_t grid = o.grid_ctas > 0 ? o.grid_ctas : resident;
    if (grid > resident) grid = resident;  // every CTA must be co-resident (deadlock freedom)
    if (grid > a.total_items) grid = a.total_items;
    if (grid < 1) grid = 1;
    // lookahead: enough rows that a row's pass-1 items finish before its pass-2 items are
    // handed out (~2 grids of items), and at least 2 rows
    int64_t L = o.lookahead_rows > 0 ? o.lookahead_rows : (2 * grid + a.nb - 1) / a.nb + 1;
    if (L < 1) L = 1;
    if (L > rows) L = rows;
    a.L = L;
    kern<<<(unsigned)grid, kThreads, 0, s>>>(a);
    return cudaGetLastError();
}

template <typename In>
static cudaError_t launch_softmax_t(int algo, const void* x, float* y, int64_t rows, int64_t cols, void* ws,
                                    const LaunchOpts& o, cudaStream_t s) {
    if (algo == kTwoPass && cols <= kBlockElems && !o.force_persistent) {
        rowblock_kernel<In><<<(unsigned)rows, kThreads, 0, s>>>(static_cast<const In*>(x), y, rows, cols,
                                                               vec_ok<In>(x, y, cols));
        return cudaGetLastError();
    }
    switch (algo) {
        case kTwoPass: return launch_persistent<In, kTwoPass>(x, y, rows, cols, ws, nullptr, o, s);
        case kRecompute: return launch_persistent<In, kRecompute>(x, y, rows, cols, ws, nullptr, o, s);
        case kReload: return launch_persistent<In, kReload>(x, y, rows, cols, ws, nullptr, o, s);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_softmax(int algo, int in_bf16, const void* x, float* y, int64_t rows, int64_t cols, void* ws,
                           const LaunchOpts& o, cudaStream_t s) {
    return in_bf16 ? launch_softmax_t<uint16_t>(algo, x, y, rows, cols, ws, o, s)
                   : launch_softmax_t<float>(algo, x, y, rows, cols, ws, o, s);
}

bool softmax_needs_workspace(int algo, int64_t cols, const LaunchOpts& o) {
    return !(algo == kTwoPass && cols <= kBlockElems && !o.force_persistent);
}

cudaError_t launch_partial(int in_bf16, const void* x, int64_t rows, int64_t cols, float* pair_out, void* ws,
                           const LaunchOpts& o, cudaStream_t s) {
    return in_bf16 ? launch_persistent<uint16_t, kTwoPassPartial>(x, nullptr, rows, cols, ws,
                                                                   reinterpret_cast<float2*>(pair_out), o, s)
                   : launch_persistent<float, kTwoPassPartial>(x, nullptr, rows, cols, ws,
                                                                reinterpret_cast<float2*>(pair_out), o, s);
}

template <typename In>
static cudaError_t launch_finish_t(const void* x, float* y, int64_t rows, int64_t cols, const float* pairs, int world,
                                   const LaunchOpts& o, cudaStream_t s) {
    int dev = 0;
    cudaGetDevice(&dev);
    auto kern = finish_kernel<In>;
    const int64_t nb = (cols + kBlockElems - 1) / kBlockElems;
    const int64_t resident = (int64_t)device_sms(dev) * occupancy(kern, dev, sizeof(In) == 4 ? 8 : 9);
    int64_t grid = o.grid_ctas > 0 ? o.grid_ctas : resident;
    if (grid > rows * nb) grid = rows * nb;
    if (grid < 1) grid = 1;
    kern<<<(unsigned)grid, kThreads, 0, s>>>(static_cast<const In*>(x), y, rows, cols,
                                             reinterpret_cast<const float2*>(pairs), world, vec_ok<In>(x, y, cols));
    return cudaGetLastError();
}

cudaError_t launch_finish(int in_bf16, const void* x, float* y, int64_t rows, int64_t cols, const float* pairs,
                          int world, const LaunchOpts& o, cudaStream_t s) {
    return in_bf16 ? launch_finish_t<uint16_t>(x, y, rows, cols, pairs, world, o, s)
                   : launch_finish_t<float>(x, y, rows, cols, pairs, world, o, s);
}

}  // namespace tp
