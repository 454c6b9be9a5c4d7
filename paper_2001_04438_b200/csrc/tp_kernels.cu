// sm_100a kernels of the Two-Pass softmax (Alg. 3) and of the in-house
// Three-Pass comparators (Alg. 1 and 2).
//
// One kernel template, stream_kernel<In, Algo, TMA>, runs every entry point.  It is a
// persistent grid (one CTA per SM) that pulls work items (phase, row, block) from an in-order
// atomic queue in the workspace.  With TMA (16-byte aligned rows) each CTA keeps a ring of
// S shared-memory stages, each holding one block, filled by cp.async.bulk (TMA) copies issued
// S items ahead by thread 0 and completed on an mbarrier; all 16 warps compute from the stage.
// Without TMA (misaligned rows) the warps load from global memory directly.
//
//   kFused     rows of one block (cols <= kBlockElems): pass 1, the CTA tree, lambda, pass 2,
//              all on the staged row: the row is read from HBM once
//   kTwoPass   pass-1 blocks publish their pair; the last block of each group of 64 reduces the
//              group, the last group reduces the row (canonical tree, reading G8) and releases
//              the row's flag; pass-2 blocks of that row wait on the flag.  Rows interleave with
//              a lookahead of L rows so that a row's pass 2 re-reads it from L2; pass 2 walks
//              the blocks backwards (most recently loaded first)
//   kPartial   pass 1 only, one (m, n) per row to pair_out (multi-GPU chunk shards)
//   kFinish    merge `world` partials per row (canonical tree over rank index), then pass 2
//   kRecompute / kReload   Three-Pass: max, sum of Exp(x - mu) (Reload also writes it to y),
//              output (Reload rescales y)
//
// Pass 1 runs without the [-2^21, 2^21] input clamp (reading G11) and checks the block result:
// a block whose pair is not finite or whose exponent leaves the clamp domain is recomputed
// with the clamp, and its row's pass 2 then clamps too.  Inside the domain the clamp is the
// identity, so this only changes which instructions run, never a result.
//
// Deadlock freedom: items are handed out in increasing order, a CTA works through its items in
// that order, and an item depends only on items of smaller index; so the smallest unfinished
// item is always the current item of a running CTA.
#include "tp_block.cuh"
#include "tp_internal.h"

namespace tp {

// ----------------------------------------------------------------------------- workspace
__host__ __device__ inline size_t align256(size_t v) { return (v + 255) & ~size_t(255); }

// Control region first (header, tickets, row flags: zero when a launch starts; the kernels
// leave it that way except for the epoch-tagged ready flags), then the data region.
__host__ __device__ inline WsLayout ws_layout(int64_t rows, int64_t cols) {
    WsLayout L{};
    const int64_t nb = (cols + kBlockElems - 1) / kBlockElems;
    const int64_t ng = (nb + kGroupBlocks - 1) / kGroupBlocks;
    size_t off = align256(sizeof(WsHeader));
    L.group_tickets = off; off = align256(off + sizeof(unsigned) * rows * ng);
    L.row_tickets = off;   off = align256(off + sizeof(unsigned) * rows);
    L.row_ready = off;     off = align256(off + sizeof(unsigned) * rows * 2);
    L.row_clamp = off;     off = align256(off + sizeof(unsigned) * rows);
    L.ctrl_bytes = off;
    L.row_stats = off;     off = align256(off + sizeof(float4) * rows * 2);
    L.block_vals = off;    off = align256(off + sizeof(float2) * rows * nb);
    L.group_vals = off;    off = align256(off + sizeof(float2) * rows * ng);
    L.bytes = off;
    return L;
}

size_t workspace_bytes(int64_t rows, int64_t cols) { return ws_layout(rows, cols).bytes; }
size_t workspace_ctrl_bytes(int64_t rows, int64_t cols) { return ws_layout(rows, cols).ctrl_bytes; }

enum Algo : int { kTwoPass = 0, kPartial = 1, kRecompute = 2, kReload = 3, kFused = 4, kFinish = 5 };

template <int A> struct AlgoTraits { static constexpr int P = 1; };
template <> struct AlgoTraits<kTwoPass> { static constexpr int P = 2; };
template <> struct AlgoTraits<kRecompute> { static constexpr int P = 3; };
template <> struct AlgoTraits<kReload> { static constexpr int P = 3; };

template <typename In> struct Stages { static constexpr int S = 3; };     // 3 x 64 KB
template <> struct Stages<uint16_t> { static constexpr int S = 6; };       // 6 x 32 KB

struct KArgs {
    const void* x;
    float* y;
    int64_t rows, cols, nb, ng;
    int64_t L;            // lookahead in rows
    int64_t total_items;  // rows * nb * phases
    char* ws;
    WsLayout lay;
    float2* pair_out;       // kPartial: one (m, n) per row
    const float2* pairs_in; // kFinish: world x rows pairs, rank-major
    int world;
    int vec;                // 16-byte aligned rows
};

// number of (phase, row) units in schedule slots < s (slot s holds phase p of row s - p*L)
__device__ __forceinline__ int64_t units_before(int64_t s, int64_t R, int64_t L, int P) {
    int64_t c = 0;
    for (int p = 0; p < P; ++p) {
        const int64_t v = s - p * L;
        c += v < 0 ? 0 : (v > R ? R : v);
    }
    return c;
}

struct Item {
    int phase;
    int64_t row, blk;
};

template <int A>
__device__ __forceinline__ Item decode_item(int64_t item, int64_t R, int64_t nb, int64_t L) {
    constexpr int P = AlgoTraits<A>::P;
    Item it;
    const int64_t unit = item / nb;
    const int64_t bi = item - unit * nb;
    if (P == 1) {
        it.phase = 0;
        it.row = unit;
        it.blk = (A == kFinish) ? nb - 1 - bi : bi;  // pass 2 walks backwards (L2 tail first)
        return it;
    }
    int64_t lo = 0, hi = R + (P - 1) * L;  // slot s with units_before(s) <= unit < units_before(s+1)
    while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (units_before(mid, R, L, P) <= unit) lo = mid; else hi = mid;
    }
    const int64_t s = lo;
    const int p_hi = (int)((s / L) < (P - 1) ? (s / L) : (P - 1));
    const int64_t idx = unit - units_before(s, R, L, P);
    it.phase = p_hi - (int)idx;  // within a slot: oldest row (highest phase) first
    it.row = s - it.phase * L;
    it.blk = it.phase > 0 ? nb - 1 - bi : bi;
    return it;
}

template <int S>
struct SmemState {
    long long item[S];
    Item dec[S];
    int flag;
    int flag2;
    unsigned epoch;
    int64_t cur_row;
    float4 stats;
    Pair red[kThreads / 32];
    float redf[kThreads / 32];
};

// Publish one block value; if it completes its group (and then its row), reduce it.
// Returns true in the CTA that finished the row (row result valid in thread 0: *root).
template <int A, int S>
__device__ bool publish_and_reduce(const KArgs& a, SmemState<S>& sm, int phase, int64_t row, int64_t blk,
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
    // the Three-Pass algorithms reduce a max in phase 0 and a sum in phase 1; Two-Pass pairs
    const bool is_max = (A == kRecompute || A == kReload) && phase == 0;
    const bool is_sum = (A == kRecompute || A == kReload) && phase == 1;
    float2 gres;
    if (is_max) {
        float m = -__int_as_float(0x7f800000);
        for (int64_t j = threadIdx.x; j < gsize; j += kThreads) m = fmaxf(m, __ldcg(gv + j).x);
        gres = make_float2(cta_max(m, sm.redf), 0.0f);
    } else if (is_sum) {
        gres = make_float2(cta_canonical_sum(gsize, [&](int64_t j) { return __ldcg(gv + j).x; }, sm.redf), 0.0f);
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
        *root = make_float2(cta_max(m, sm.redf), 0.0f);
    } else if (is_sum) {
        *root = make_float2(cta_canonical_sum(a.ng, [&](int64_t j) { return __ldcg(rv + j).x; }, sm.redf), 0.0f);
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

// Pass 1 of a block with the out-of-domain fallback; returns the block pair (thread 0) and
// whether the clamped path was needed (all threads).
template <int V, int S>
__device__ __forceinline__ Pair block_pass1(const BlockVals& r, int valid, SmemState<S>& sm, bool* clamped) {
    Pair acc = valid == kBlockElems ? pass1_thread<V, true, false>(r, valid) : pass1_thread<V, false, false>(r, valid);
    Pair bp = cta_tree_pairs(acc, sm.red);
    if (threadIdx.x == 0) sm.flag2 = pair_out_of_domain(bp);
    __syncthreads();
    *clamped = sm.flag2 != 0;
    if (*clamped) {
        acc = pass1_thread<V, false, true>(r, valid);
        bp = cta_tree_pairs(acc, sm.red);
    }
    return bp;
}

template <typename In, int A, bool TMA>
__global__ void __launch_bounds__(kThreads, 1) stream_kernel(const KArgs a) {
    constexpr int P = AlgoTraits<A>::P;
    constexpr int V = InTraits<In>::V;
    constexpr int S = TMA ? Stages<In>::S : 2;  // without TMA: 2 item slots, no data staging
    extern __shared__ __align__(128) unsigned char dsm[];
    __shared__ SmemState<S> sm;
    __shared__ uint64_t full_bar[S];

    WsHeader* hdr = reinterpret_cast<WsHeader*>(a.ws);
    float4* row_stats = reinterpret_cast<float4*>(a.ws + a.lay.row_stats);
    unsigned* row_ready = reinterpret_cast<unsigned*>(a.ws + a.lay.row_ready);
    unsigned* row_clamp = reinterpret_cast<unsigned*>(a.ws + a.lay.row_clamp);
    const In* x = static_cast<const In*>(a.x);
    uint64_t pol_keep = 0, pol_drop = 0;

    // thread 0: take the next item from the queue into slot s and start its TMA copy
    auto fetch_and_issue = [&](int s) {
        const long long item = (long long)atomicAdd(&hdr->counter, 1ull);
        sm.item[s] = item;
        if (item >= a.total_items) return;
        const Item it = decode_item<A>(item, a.rows, a.nb, a.L);
        sm.dec[s] = it;
        if constexpr (TMA) {
            In* stage = reinterpret_cast<In*>(dsm) + (size_t)s * kBlockElems;
            const bool reload_y = (A == kReload && it.phase == 2);  // reads Y after its flag: no prefetch
            if (reload_y) {
                asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full_bar[s]))
                             : "memory");
            } else {
                const int64_t e0 = it.blk * kBlockElems;
                const uint32_t bytes = (uint32_t)(min((int64_t)kBlockElems, a.cols - e0) * sizeof(In));
                const bool last = (it.phase == P - 1) && A != kPartial;
                mbar_arrive_expect_tx(&full_bar[s], bytes);
                tma_load_1d(stage, x + it.row * a.cols + e0, bytes, &full_bar[s], last ? pol_drop : pol_keep);
            }
        }
    };

    if (threadIdx.x == 0) {
        sm.epoch = *reinterpret_cast<volatile unsigned*>(&hdr->epoch);
        sm.cur_row = -1;
        if constexpr (TMA) {
            pol_keep = policy_evict_last();
            pol_drop = policy_evict_first();
            for (int s = 0; s < S; ++s) mbar_init(&full_bar[s], 1);
            fence_mbar_init();
        }
        for (int s = 0; s < S; ++s) fetch_and_issue(s);
    }
    __syncthreads();
    const unsigned want = sm.epoch + 1u;

    for (uint32_t iter = 0;; ++iter) {
        const int s = (int)(iter % S);
        const long long item = sm.item[s];
        if (item >= a.total_items) break;
        const Item it = sm.dec[s];
        const int64_t e0 = it.blk * kBlockElems;
        const int valid = (int)min((int64_t)kBlockElems, a.cols - e0);
        const In* xb = x + it.row * a.cols + e0;
        float* yb = a.y ? a.y + it.row * a.cols + e0 : nullptr;

        // ---- stats of the row's previous phase (or of the world partials)
        if (P > 1 && it.phase > 0) {
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
        if (A == kFinish && it.row != sm.cur_row) {
            __syncthreads();
            if (threadIdx.x == 0) {
                const Pair root = seq_tree_pairs((int)next_pow2(a.world), [&](int i) {
                    if (i >= a.world) return pair_identity();
                    const float2 v = a.pairs_in[(int64_t)i * a.rows + it.row];
                    return Pair{v.x, v.y};
                });
                sm.stats = make_float4(__fsub_rn(root.n, 1.0f), __fdiv_rn(0.5f, root.m), 1.0f, 0.0f);
                sm.cur_row = it.row;
            }
            __syncthreads();
        }
        const float4 st = sm.stats;

        // ---- this thread's 32 values of the block
        BlockVals r;
        const bool reload_y = (A == kReload && it.phase == 2);
        if (!reload_y) {
            if constexpr (TMA) {
                mbar_wait_parity(&full_bar[s], (iter / S) & 1u);
                load_stage<In>(reinterpret_cast<const In*>(dsm) + (size_t)s * kBlockElems, r);
            } else {
                load_global<In>(xb, valid, a.vec != 0, it.phase == P - 1, r);
            }
        } else {
            if constexpr (TMA) mbar_wait_parity(&full_bar[s], (iter / S) & 1u);
            const bool yvec = (a.cols % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.y) & 15) == 0);
            load_global_y(yb, valid, yvec, r);
        }

        if constexpr (A == kFused) {
            bool clamped;
            const Pair root = block_pass1<V>(r, valid, sm, &clamped);
            if (threadIdx.x == 0) sm.stats = make_float4(__fsub_rn(root.n, 1.0f), __fdiv_rn(0.5f, root.m), 0.f, 0.f);
            __syncthreads();
            const float4 fs = sm.stats;
            if (clamped) pass2_thread<true>(r, fs.x, fs.y);
            else pass2_thread<false>(r, fs.x, fs.y);
            store_block<V>(yb, valid, a.vec != 0, r);
        } else if constexpr (A == kTwoPass || A == kPartial) {
            if (it.phase == 0) {
                bool clamped;
                const Pair bp = block_pass1<V>(r, valid, sm, &clamped);
                if (clamped && threadIdx.x == 0) atomicOr(&row_clamp[it.row], 1u);
                float2 root;
                if (publish_and_reduce<A>(a, sm, 0, it.row, it.blk, make_float2(bp.m, bp.n), &root) &&
                    threadIdx.x == 0) {
                    const unsigned cl = __ldcg(&row_clamp[it.row]);
                    row_clamp[it.row] = 0u;
                    if (A == kPartial) {
                        a.pair_out[it.row] = root;
                    } else {
                        // lambda' = 0.5 / m_sum, correctly rounded (readings G9, G10)
                        row_stats[it.row * 2] = make_float4(__fsub_rn(root.y, 1.0f), __fdiv_rn(0.5f, root.x),
                                                            cl ? 1.0f : 0.0f, root.y);
                        st_release_gpu(row_ready + it.row * 2, want);
                    }
                }
            } else {
                if (st.z != 0.0f) pass2_thread<true>(r, st.x, st.y);
                else pass2_thread<false>(r, st.x, st.y);
                store_block<V>(yb, valid, a.vec != 0, r);
            }
        } else if constexpr (A == kFinish) {
            pass2_thread<true>(r, st.x, st.y);  // the local chunk's clamp state is unknown: always clamp
            store_block<V>(yb, valid, a.vec != 0, r);
        } else {
            // Three-Pass: phase 0 max (Pass 1), phase 1 sum of Exp(x - mu) (Pass 2),
            // phase 2 output (Pass 3).  Alg. 1, Alg. 2 PAPER.md:110-123.
            if (it.phase == 0) {
                const float mx = cta_max(valid == kBlockElems ? max_thread<V, true>(r, valid)
                                                              : max_thread<V, false>(r, valid), sm.redf);
                float2 root;
                if (publish_and_reduce<A>(a, sm, 0, it.row, it.blk, make_float2(mx, 0.0f), &root) &&
                    threadIdx.x == 0) {
                    row_stats[it.row * 2] = make_float4(root.x, 0.0f, 0.0f, 0.0f);
                    st_release_gpu(row_ready + it.row * 2, want);
                }
            } else if (it.phase == 1) {
                float s1 = valid == kBlockElems ? exp_sum_thread<V, true>(r, valid, st.x)
                                                : exp_sum_thread<V, false>(r, valid, st.x);
                if (A == kReload) store_block<V>(yb, valid, a.vec != 0, r);  // Y_i <- Exp(X_i - mu)
                s1 = cta_tree_sum(s1, sm.redf);
                float2 root;
                if (publish_and_reduce<A>(a, sm, 1, it.row, it.blk, make_float2(s1, 0.0f), &root) &&
                    threadIdx.x == 0) {
                    row_stats[it.row * 2 + 1] = make_float4(st.x, __fdiv_rn(1.0f, root.x), root.x, 0.0f);
                    st_release_gpu(row_ready + it.row * 2 + 1, want);
                }
            } else {
                if constexpr (A == kRecompute) {
                    exp_sum_thread<V, false>(r, valid, st.x);
                    scale_thread(r, st.y);  // Y_i <- lambda * Exp(X_i - mu)
                    store_block<V>(yb, valid, a.vec != 0, r);
                } else {
                    scale_thread(r, st.y);  // Y_i <- lambda * Y_i  (read Y, write Y)
                    const bool yvec = (a.cols % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.y) & 15) == 0);
                    store_block<4>(yb, valid, yvec, r);
                }
            }
        }

        __syncthreads();  // stage s, sm.item[s], sm.stats and sm.red are free again
        if (threadIdx.x == 0) {
            if constexpr (TMA) fence_proxy_async_smem();
            fetch_and_issue(s);
        }
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

// ----------------------------------------------------------------------------- host launchers
static int g_num_sms[64];

static int device_sms(int dev) {
    if (!g_num_sms[dev]) cudaDeviceGetAttribute(&g_num_sms[dev], cudaDevAttrMultiProcessorCount, dev);
    return g_num_sms[dev];
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

template <typename In>
static int vec_ok(const void* x, const float* y, int64_t cols) {
    constexpr int V = InTraits<In>::V;
    return (cols % V == 0) && aligned16(x) && (y == nullptr || aligned16(y));
}

template <typename In, int A, bool TMA>
static cudaError_t launch_t(KArgs a, const LaunchOpts& o, cudaStream_t s) {
    int dev = 0;
    cudaGetDevice(&dev);
    auto kern = stream_kernel<In, A, TMA>;
    const size_t dyn = TMA ? (size_t)Stages<In>::S * kBlockElems * sizeof(In) : 0;
    static int configured[64];
    static int occ[64];
    if (!configured[dev]) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
        int n = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, kThreads, dyn);
        occ[dev] = n > 0 ? n : 1;
        configured[dev] = 1;
    }
    const int64_t resident = (int64_t)device_sms(dev) * occ[dev];
    int64_t grid = o.grid_ctas > 0 ? o.grid_ctas : resident;
    if (grid > resident) grid = resident;
    if (grid > a.total_items) grid = a.total_items;
    if (grid < 1) grid = 1;
    // lookahead: enough rows that a row's pass-1 items are done before its pass-2 items are
    // handed out (~2 grids of items in flight, S items per CTA)
    int64_t L = o.lookahead_rows > 0 ? o.lookahead_rows : (2 * grid * (TMA ? Stages<In>::S : 2) + a.nb - 1) / a.nb + 1;
    if (L < 1) L = 1;
    if (L > a.rows) L = a.rows;
    a.L = L;
    kern<<<(unsigned)grid, kThreads, dyn, s>>>(a);
    return cudaGetLastError();
}

template <typename In, int A>
static cudaError_t launch_algo(const void* x, float* y, int64_t rows, int64_t cols, void* ws, float2* pair_out,
                               const float2* pairs_in, int world, const LaunchOpts& o, cudaStream_t s) {
    KArgs a{};
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
    if (a.vec && !o.no_tma) return launch_t<In, A, true>(a, o, s);
    return launch_t<In, A, false>(a, o, s);
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
                           const LaunchOpts& o, cudaStream_t s) {
    float2* po = reinterpret_cast<float2*>(pair_out);
    return in_bf16 ? launch_algo<uint16_t, kPartial>(x, nullptr, rows, cols, ws, po, nullptr, 1, o, s)
                   : launch_algo<float, kPartial>(x, nullptr, rows, cols, ws, po, nullptr, 1, o, s);
}

cudaError_t launch_finish(int in_bf16, const void* x, float* y, int64_t rows, int64_t cols, const float* pairs,
                          int world, void* ws, const LaunchOpts& o, cudaStream_t s) {
    const float2* pi = reinterpret_cast<const float2*>(pairs);
    return in_bf16 ? launch_algo<uint16_t, kFinish>(x, y, rows, cols, ws, nullptr, pi, world, o, s)
                   : launch_algo<float, kFinish>(x, y, rows, cols, ws, nullptr, pi, world, o, s);
}

}  // namespace tp
